"""Summarise an ncu capture (run here, no GPU needed):

    python profiles/summarize_ncu.py gpurun_out/prof.ncu-rep gpurun_out/launches.csv rNN

Writes profiles/ncu_<tag>.md (per-kernel table + launch-share table) and
updates profiles/ncu_traffic.json (dram bytes per launch, read by bench.py for
roofline.traffic).
"""
import csv
import io
import json
import os
import re
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
METRICS = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "mem_thr_%"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram_%"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "l1tex_%"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_%"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "fma_pipe_%"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps_active_%"),
    ("launch__registers_per_thread", "regs"),
    ("launch__shared_mem_per_block_static", "smem_static"),
    ("launch__shared_mem_per_block_dynamic", "smem_dyn"),
    ("smsp__inst_executed.sum", "inst"),
]
SCALE = {"ms": 1e-3, "us": 1e-6, "usecond": 1e-6, "msecond": 1e-3, "nsecond": 1e-9, "ns": 1e-9,
         "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1.0}


def short(name):
    base = re.sub(r"^void ", "", name).split("(")[0].split("<")[0]
    return base.split("::")[-1]


def main(rep, launches, tag):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    kern = []
    for r in rows[2:]:
        d = {"kernel": short(r[hdr.index("Kernel Name")]), "full": r[hdr.index("Kernel Name")]}
        for m, k in METRICS:
            if m in hdr:
                i = hdr.index(m)
                v = r[i].replace(",", "")
                try:
                    v = float(v) * SCALE.get(units[i], 1.0)
                except ValueError:
                    pass
                d[k] = v
        kern.append(d)
    traffic_path = os.path.join(HERE, "ncu_traffic.json")
    traffic = json.load(open(traffic_path)) if os.path.exists(traffic_path) else {}
    lines = [f"# ncu summary {tag}", "", f"source: `{os.path.basename(rep)}` (`--set full "
             "--clock-control none`, cold-cache replay); bench workload L1 160x192x224.", "",
             "| kernel | time us | DRAM MB (r+w) | GB/s | mem thr % | L1 % | SM % | FMA % | "
             "warps % | regs |", "|---|---|---|---|---|---|---|---|---|---|"]
    for d in kern:
        t = d.get("time", 0)
        b = d.get("dram_read", 0) + d.get("dram_write", 0)
        traffic[d["kernel"]] = int(b)
        lines.append(
            f"| {d['kernel']} | {t * 1e6:.1f} | {b / 1e6:.1f} | {b / t / 1e9 if t else 0:.0f} | "
            f"{d.get('mem_thr_%', 0):.1f} | {d.get('l1tex_%', 0):.1f} | {d.get('sm_%', 0):.1f} | "
            f"{d.get('fma_pipe_%', 0):.1f} | {d.get('warps_active_%', 0):.1f} | "
            f"{d.get('regs', 0):.0f} |")
    if launches and os.path.exists(launches):
        txt = open(launches).read()
        txt = txt[txt.index('"ID"'):] if '"ID"' in txt else txt
        lr = list(csv.DictReader(io.StringIO(txt)))
        tot = {}
        for r in lr:
            if r.get("Metric Name") != "gpu__time_duration.sum":
                continue
            k = short(r["Kernel Name"])
            v = float(r["Metric Value"].replace(",", "")) * SCALE.get(r.get("Metric Unit", "ns"), 1)
            tot.setdefault(k, [0.0, 0])
            tot[k][0] += v
            tot[k][1] += 1
        all_t = sum(v[0] for v in tot.values())
        lines += ["", "Launch list (`--metrics gpu__time_duration.sum`, every launch of the "
                  "profiled command incl. warm-up):", "", "| kernel | launches | total us | share |",
                  "|---|---|---|---|"]
        for k, (t, c) in sorted(tot.items(), key=lambda kv: -kv[1][0]):
            lines.append(f"| {k} | {c} | {t * 1e6:.1f} | {t / all_t * 100:.1f}% |")
    out = os.path.join(HERE, f"ncu_{tag}.md")
    open(out, "w").write("\n".join(lines) + "\n")
    json.dump(traffic, open(traffic_path, "w"), indent=1, sort_keys=True)
    print("\n".join(lines))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None, sys.argv[3] if len(sys.argv) > 3 else "r01")
