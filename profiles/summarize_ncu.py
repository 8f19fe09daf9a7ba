"""Summarise one profiles/ncu_cmds.sh capture (run here, no GPU needed):

    python profiles/summarize_ncu.py <tag>        # reads gpurun_out/ncu_<tag>/

Writes profiles/ncu_<tag>.md:
  * the bench step: every kernel with launches, avg us, DRAM bytes per launch
    (read + write), achieved DRAM GB/s and its fraction of the measured HBM
    peak, and per op the SURVEY §8(d) algorithmic bytes and their fraction;
  * one PO iteration: the same columns for every kernel it launches;
  * the --set full captures: registers, issue activity, resident warps,
    L1/TEX throughput, executed instructions per voxel;
and profiles/ncu_traffic.json (per-kernel DRAM bytes per launch, read by
bench.py for roofline.traffic).  ncu replays kernels with cold caches, so the
absolute times are above the bench's CUDA-event times; shares agree.
"""
import collections
import csv
import io
import json
import os
import re
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
NVOX = 160 * 192 * 224
S, HD, CH = 1, 6, 8
ALG = {  # SURVEY §8(d), bytes per voxel
    "modet_fwd": 4 * (2 * S * HD + 3 * S), "modet_bwd": 4 * (4 * S * HD + 3 * S),
    "warp_fwd": 4 * (3 + 2 * CH), "warp_bwd": 4 * (6 + 3 * CH)}
OPS = {"modet_fwd": ["modet_fwd_tiled_k", "modet_fwd_fixup_k"],
       "modet_bwd": ["modet_bwd_row_k", "modet_bwd_col_k", "modet_bwd_fused_k", "reduce_db_k"],
       "warp_fwd": ["warp_fwd_k"], "warp_bwd": ["warp_bwd_k"]}
SCALE = {"ms": 1e-3, "us": 1e-6, "usecond": 1e-6, "msecond": 1e-3, "nsecond": 1e-9, "ns": 1e-9,
         "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}


def peak():
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:
        return 6551.0


def short(name):
    name = re.sub(r"^void ", "", name).replace("(anonymous namespace)::", "")
    name = name.replace("<unnamed>::", "")
    return name.split("(")[0].split("<")[0].split("::")[-1]


def launches(path):
    """{launch id: {kernel, time s, dram bytes}} from an ncu --csv --metrics log."""
    if not os.path.exists(path):
        return []
    txt = open(path).read()
    if '"ID"' not in txt:
        return []
    txt = txt[txt.index('"ID"'):]
    out = collections.OrderedDict()
    for r in csv.DictReader(io.StringIO(txt)):
        d = out.setdefault(r["ID"], {"kernel": short(r["Kernel Name"]), "t": 0.0, "b": 0.0})
        v = float(r["Metric Value"].replace(",", "")) * SCALE.get(r.get("Metric Unit", ""), 1.0)
        if r["Metric Name"] == "gpu__time_duration.sum":
            d["t"] = v
        elif r["Metric Name"].startswith("dram__bytes"):
            d["b"] += v
    return list(out.values())


def per_kernel(ls):
    agg = collections.OrderedDict()
    for d in ls:
        a = agg.setdefault(d["kernel"], [0, 0.0, 0.0])
        a[0] += 1
        a[1] += d["t"]
        a[2] += d["b"]
    return agg


def table(agg, pk, lines, share=True):
    tot = sum(a[1] for a in agg.values()) or 1.0
    lines += ["| kernel | launches | avg us | DRAM MB / launch | DRAM GB/s | frac of peak |"
              + (" share |" if share else ""),
              "|---|---|---|---|---|---|" + ("---|" if share else "")]
    for k, (n, t, b) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        gbs = b / t / 1e9 if t else 0.0
        lines.append(f"| {k} | {n} | {t / n * 1e6:.1f} | {b / n / 1e6:.1f} | {gbs:.0f} | "
                     f"{gbs / pk:.3f} |" + (f" {t / tot * 100:.1f}% |" if share else ""))


def full_rows(d):
    rows = []
    for f in sorted(os.listdir(d)):
        if not (f.startswith("full_") and f.endswith(".raw.csv")):
            continue
        raw = open(os.path.join(d, f)).read()
        r = list(csv.reader(io.StringIO(raw)))
        if len(r) < 3:
            continue
        h, u, v = r[0], r[1], r[2]

        def g(n):
            try:
                i = h.index(n)
                return float(v[i].replace(",", "")) * SCALE.get(u[i], 1.0)
            except (ValueError, IndexError):
                return float("nan")
        rows.append((short(v[h.index("Kernel Name")]), g("launch__registers_per_thread"),
                     g("smsp__issue_active.avg.pct_of_peak_sustained_active"),
                     g("sm__warps_active.avg.per_cycle_active"),
                     g("l1tex__throughput.avg.pct_of_peak_sustained_active"),
                     g("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
                     g("smsp__inst_executed.sum") * 32 / NVOX,
                     (g("dram__bytes_read.sum") + g("dram__bytes_write.sum")) / 1e6))
    return rows


def main(tag):
    d = os.path.join(ROOT, "gpurun_out", f"ncu_{tag}")
    pk = peak()
    lines = [f"# ncu summary {tag}", "",
             f"Captured by `bash profiles/ncu_cmds.sh {tag}` on one B200; peak = measured "
             f"{pk:.0f} GB/s (MEASURED_PEAKS.json).  ncu replays each kernel with cold caches, "
             "so its times run above the bench's CUDA-event times; the shares agree.", ""]
    step = launches(os.path.join(d, "step_launches.csv"))
    traffic = {"source": f"profiles/ncu_{tag}.md", "kernels": {}}
    if step:
        agg = per_kernel(step)
        lines += ["## Bench step (L1 160x192x224; 5 steps: 3 warm-up + 2 timed)", ""]
        table(agg, pk, lines)
        lines += ["", "Per op, SURVEY §8(d) algorithmic bytes against the kernels' time "
                  "(the roofline the bench reports):", "",
                  "| op | kernels | alg. MB | ncu DRAM MB | DRAM / alg. | us | alg. frac of peak |",
                  "|---|---|---|---|---|---|---|"]
        nsteps = max(1, agg.get("warp_bwd_k", [5])[0])
        for op, ks in OPS.items():
            ks = [k for k in ks if k in agg]
            if not ks:
                continue
            t = sum(agg[k][1] for k in ks) / nsteps
            b = sum(agg[k][2] for k in ks) / nsteps
            alg = ALG[op] * NVOX
            lines.append(f"| {op} | {' + '.join(ks)} | {alg / 1e6:.1f} | {b / 1e6:.1f} | "
                         f"{b / alg:.2f} | {t * 1e6:.1f} | {alg / t / 1e9 / pk:.3f} |")
        for k, (n, t, b) in agg.items():
            traffic["kernels"][k] = {"dram_bytes": int(b / n), "time_us": round(t / n * 1e6, 1)}
    po = launches(os.path.join(d, "po_launches.csv"))
    if po:
        agg = per_kernel(po)
        tot = sum(a[1] for a in agg.values())
        lines += ["", f"## One PO iteration (160x192x224, eager launches): {len(po)} launches, "
                  f"{tot * 1e3:.2f} ms summed kernel time under ncu", ""]
        table(agg, pk, lines)
    rows = full_rows(d)
    if rows:
        lines += ["", "## --set full captures (one launch each)", "",
                  "| kernel | regs | issue active % | warps/SM | L1/TEX % | DRAM % | "
                  "instr / voxel | DRAM MB |", "|---|---|---|---|---|---|---|---|"]
        for r in rows:
            lines.append("| " + " | ".join([r[0]] + [f"{x:.1f}" for x in r[1:]]) + " |")
    out = os.path.join(HERE, f"ncu_{tag}.md")
    open(out, "w").write("\n".join(lines) + "\n")
    if traffic["kernels"]:
        json.dump(traffic, open(os.path.join(HERE, "ncu_traffic.json"), "w"), indent=1,
                  sort_keys=True)
    print("\n".join(lines))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "r02")
