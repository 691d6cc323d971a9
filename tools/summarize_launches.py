"""Summarise an ncu --csv launch list: per kernel name, count, total time, DRAM bytes."""
import csv, collections, sys, json
path = sys.argv[1]
rows = list(csv.reader(open(path)))
hi = next(i for i, r in enumerate(rows) if r and r[0] == 'ID')
hdr = rows[hi]
ki, mi, vi, idi = hdr.index('Kernel Name'), hdr.index('Metric Name'), hdr.index('Metric Value'), hdr.index('ID')
per = collections.OrderedDict()
for r in rows[hi + 1:]:
    per.setdefault(r[idi], {'name': r[ki]})[r[mi]] = float(r[vi].replace(',', ''))
agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
for v in per.values():
    n = v['name'].split('(')[0].replace('void ', '').replace('<unnamed>::', '')[:70]
    agg[n][0] += 1
    agg[n][1] += v.get('gpu__time_duration.sum', 0)
    agg[n][2] += v.get('dram__bytes_read.sum', 0) + v.get('dram__bytes_write.sum', 0)
tot = sum(a[1] for a in agg.values())
out = []
for n, (c, t, b) in sorted(agg.items(), key=lambda x: -x[1][1]):
    out.append(dict(kernel=n, launches=c, ms=round(t / 1e6, 3), share=round(t / tot, 4),
                    dram_GB=round(b / 1e9, 3), dram_GBs=round(b / t, 1) if t else None))
    print(f"{c:5d} {t/1e6:9.3f}ms {t/tot*100:5.1f}% {b/1e9:8.3f}GB {b/t if t else 0:8.1f}GB/s  {n}")
if len(sys.argv) > 2:
    json.dump(out, open(sys.argv[2], 'w'), indent=1)
