"""Aggregate an ncu --csv launch list (gpu__time_duration.sum) by kernel name.
usage: python tools/launch_table.py gpurun_out/launches.csv [top]"""
import collections, csv, sys
rows = list(csv.reader(open(sys.argv[1])))
i = next(k for k, r in enumerate(rows) if r and r[0] == "ID")
hdr = rows[i]
ik, iv, im = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name")
t = collections.defaultdict(float); c = collections.Counter()
for r in rows[i + 1:]:
    if len(r) > iv and r[im] == "gpu__time_duration.sum":
        name = r[ik].split("(")[0].split("<")[0].replace("void ", "")
        t[name] += float(r[iv].replace(",", "")) / 1e3; c[name] += 1
tot = sum(t.values())
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
for k, v in sorted(t.items(), key=lambda x: -x[1])[:top]:
    print(f"{k:40s} {c[k]:5d} {v:10.1f} us {100*v/tot:5.1f}%")
print(f"total {tot:.1f} us")
