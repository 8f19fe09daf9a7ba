"""Print stall breakdown + key counters for every kernel in an ncu report."""
import csv, subprocess, sys
rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines())); hdr = rows[0]
idx = [i for i, h in enumerate(hdr) if 'pcsamp_warps_issue_stalled' in h and not h.endswith('not_issued')]
for r in rows[2:]:
    name = r[hdr.index('Kernel Name')].split('(')[0][-34:]
    vals = []
    for i in idx:
        try: vals.append((float(r[i].replace(',', '')), hdr[i].replace('smsp__pcsamp_warps_issue_stalled_', '')))
        except ValueError: pass
    tot = sum(v for v, _ in vals) or 1
    print(name, ' '.join(f'{h}={v/tot*100:.0f}%' for v, h in sorted(vals, reverse=True)[:7]))
    for m in ['smsp__inst_executed.sum', 'smsp__issue_active.avg.pct_of_peak_sustained_active',
              'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum', 'sm__warps_active.avg.pct_of_peak_sustained_active']:
        if m in hdr: print('   ', m, r[hdr.index(m)])
