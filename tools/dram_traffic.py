"""Per-op DRAM traffic of one training epoch from an ncu launch list.

Capture (on the GPU box; GRD_NVTX=1 makes every op an NVTX range "<op>#<n>"
and --print-nvtx-rename attributes each CUDA kernel to its op call):

  GRD_NVTX=1 ncu --nvtx --print-nvtx-rename kernel --profile-from-start off \
      --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
      --clock-control none --csv --log-file gpurun_out/dram_W.csv \
      python tools/profile_epoch.py W

Then:  python tools/dram_traffic.py gpurun_out/dram_W.csv W [profiles/traffic.json]

Writes traffic[W][op] = DRAM bytes (read + write) per op call, averaged over
the epoch's calls — the figure bench.py's roofline divides by the live
per-call time — and prints a per-op table.
"""
import collections
import csv
import json
import sys

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1, "ns": 1e-9,
         "us": 1e-6, "ms": 1e-3}


def main():
    path, workload = sys.argv[1], sys.argv[2]
    out_path = sys.argv[3] if len(sys.argv) > 3 else "profiles/traffic.json"
    lines = [l for l in open(path) if l.startswith('"')]
    rows = list(csv.DictReader(lines))
    per_launch = collections.defaultdict(dict)
    for r in rows:
        v = float(r["Metric Value"].replace(",", "")) * SCALE.get(r["Metric Unit"], 1)
        per_launch[(r["ID"], r["Kernel Name"])][r["Metric Name"]] = v
    ops = collections.OrderedDict()
    for (_, name), m in per_launch.items():
        # renamed kernels read "<op>#<call>/<kernel signature>"
        op, _, call = name.partition("#")
        call = call.split("/", 1)[0]
        if not call:                  # a kernel outside any op range
            op = "(outside ops) " + name.split("(")[0][:60]
        o = ops.setdefault(op, dict(calls=set(), kernels=0, dram=0.0, s=0.0))
        o["calls"].add(call)
        o["kernels"] += 1
        o["dram"] += m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)
        o["s"] += m.get("gpu__time_duration.sum", 0)
    try:
        traffic = json.load(open(out_path))
    except FileNotFoundError:
        traffic = {}
    entry = {"_source": f"ncu DRAM bytes of one eager epoch ({path.split('/')[-1]}), "
                        "per op call (GRD_NVTX ranges)"}
    print(f"{'op':22s} {'calls':>6s} {'kernels':>8s} {'ms':>10s} {'GB':>9s} {'GB/s':>8s}")
    for op, o in sorted(ops.items(), key=lambda kv: -kv[1]["s"]):
        calls = len(o["calls"])
        entry[op] = int(o["dram"] / calls)
        print(f"{op:22s} {calls:6d} {o['kernels']:8d} {o['s'] * 1e3:10.3f} {o['dram'] / 1e9:9.3f} "
              f"{o['dram'] / max(o['s'], 1e-12) / 1e9:8.1f}")
    traffic[workload] = entry
    json.dump(traffic, open(out_path, "w"), indent=1)


if __name__ == "__main__":
    main()
