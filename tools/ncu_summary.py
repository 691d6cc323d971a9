"""Summarise an `ncu --set full` report (raw CSV export) per launch:
duration, DRAM bytes, L2 hit rate, occupancy, registers.  Also emits the
per-kernel DRAM traffic per launch that bench.py reports as roofline.traffic.

  ncu -i X.ncu-rep --page raw --csv > X.csv
  python tools/ncu_summary.py X.csv profiles/rNN_ncu_epoch_W.json W
"""
import csv, json, sys, collections
path, out_path = sys.argv[1], sys.argv[2]
workload = sys.argv[3] if len(sys.argv) > 3 else None
rows = list(csv.reader(open(path)))
hdr, units = rows[0], rows[1]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "nsecond": 1e-9, "s": 1}
def val(r, name):
    i = hdr.index(name)
    v = r[i].replace(",", "")
    try:
        return float(v) * SCALE.get(units[i], 1)
    except ValueError:
        return None
def short(n):
    n = n.split("(")[0].replace("void ", "").replace("<unnamed>::", "").replace("grd_tc::", "")
    return n
launches = []
for r in rows[2:]:
    k = r[hdr.index("Kernel Name")]
    d = dict(id=int(r[hdr.index("ID")]), kernel=short(k),
             ms=round(val(r, "gpu__time_duration.sum") * 1e3, 4),
             dram_read_GB=round(val(r, "dram__bytes_read.sum") / 1e9, 4),
             dram_write_GB=round(val(r, "dram__bytes_write.sum") / 1e9, 4))
    for key, metric in (("l2_hit_pct", "lts__t_sector_hit_rate.pct"),
                        ("occupancy_pct", "sm__warps_active.avg.pct_of_peak_sustained_active"),
                        ("registers", "launch__registers_per_thread"),
                        ("tensor_pipe_pct", "sm__pipe_tensor_op_tmem_cycles_active.avg.pct_of_peak_sustained_active")):
        if metric in hdr:
            v = val(r, metric)
            if v is not None:
                d[key] = round(v, 2)
    d["dram_GBs"] = round((d["dram_read_GB"] + d["dram_write_GB"]) / (d["ms"] * 1e-3), 1)
    launches.append(d)
per = collections.OrderedDict()
for d in launches:
    base = d["kernel"].split("<")[0]
    p = per.setdefault(base, dict(launches=0, ms=0.0, dram_GB=0.0))
    p["launches"] += 1
    p["ms"] += d["ms"]
    p["dram_GB"] += d["dram_read_GB"] + d["dram_write_GB"]
for p in per.values():
    p["dram_bytes_per_launch"] = round(p["dram_GB"] * 1e9 / p["launches"])
    p["ms"] = round(p["ms"], 4)
    p["dram_GB"] = round(p["dram_GB"], 4)
json.dump(dict(workload=workload, note="ncu --set full --clock-control none, one eager epoch "
               "(tools/profile_epoch.py); cold-cache serialised launches", per_kernel=per,
               launches=launches), open(out_path, "w"), indent=1)
for k, p in per.items():
    print(f"{k:28s} {p['launches']:3d} {p['ms']:9.3f} ms {p['dram_GB']:8.3f} GB")
