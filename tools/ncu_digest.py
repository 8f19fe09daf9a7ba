"""Digest of one ncu-rep kernel capture (run here, no GPU): key counters,
stall-reason shares and the SASS opcode histogram.

    python tools/ncu_digest.py gpurun_out/x.ncu-rep [kernel-regex] [n_voxels]
"""
import collections
import csv
import io
import subprocess
import sys


def ncu(rep, *args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


def main(rep, kern=None, nvox=160 * 192 * 224):
    sel = ["--kernel-name", f"regex:{kern}"] if kern else []
    raw = list(csv.reader(io.StringIO(ncu(rep, *sel, "--page", "raw", "--csv"))))
    h, v = raw[0], raw[2]
    get = lambda n: float(v[h.index(n)].replace(",", "")) if n in h else float("nan")  # noqa
    inst = get("smsp__inst_executed.sum")
    dur = get("gpu__time_duration.sum")
    print(f"duration {dur:.1f} (ncu units)  inst {inst/1e6:.1f} M  ({inst*32/nvox:.0f} thread-instr/voxel)"
          f"  regs {get('launch__registers_per_thread'):.0f}"
          f"  warps/SM {get('sm__warps_active.avg.per_cycle_active'):.1f}"
          f"  issue {get('smsp__issue_active.avg.pct_of_peak_sustained_active'):.1f}%"
          f"  dram {(get('dram__bytes_read.sum')+get('dram__bytes_write.sum'))/1e6:.0f} MB")
    st = [(float(v[i].replace(",", "")), n[len("smsp__pcsamp_warps_issue_stalled_"):])
          for i, n in enumerate(h) if n.startswith("smsp__pcsamp_warps_issue_stalled")
          and not n.endswith("not_issued")]
    tot = sum(x for x, _ in st) or 1
    print("stalls: " + ", ".join(f"{n} {100*x/tot:.0f}%" for x, n in sorted(st, reverse=True)[:8]))
    src = list(csv.reader(io.StringIO(ncu(rep, *sel, "--page", "source", "--csv",
                                          "--print-source", "sass"))))
    sh = src[1]
    iS, iE = sh.index("Source"), sh.index("Instructions Executed")
    ops, tot = collections.Counter(), 0
    for r in src[2:]:
        try:
            e = int(float(r[iE] or 0))
        except (ValueError, IndexError):
            continue
        t = r[iS].strip().split()
        if not t:
            continue
        o = t[1] if t[0].startswith("@") else t[0]
        ops[o.split(".")[0]] += e
        tot += e
    print(f"SASS lines {len(src) - 2}; per voxel: " + ", ".join(
        f"{o} {c*32/nvox:.0f}" for o, c in ops.most_common(16)))


if __name__ == "__main__":
    a = sys.argv[1:]
    main(a[0], a[1] if len(a) > 1 else None, *(int(x) for x in a[2:]))
