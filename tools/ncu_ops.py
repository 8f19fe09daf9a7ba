"""SASS opcode histogram (instructions executed) for one kernel of an ncu report."""
import collections, csv, subprocess, sys
rep, rx = sys.argv[1], sys.argv[2]
nvox = float(sys.argv[3]) if len(sys.argv) > 3 else 6881280
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass", "-k", "regex:" + rx],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr = rows[1]; i_src = hdr.index('Source'); i_ex = hdr.index('Instructions Executed')
ops = collections.Counter(); tot = 0
for r in rows[2:]:
    if len(r) <= i_ex: continue
    try: n = float(r[i_ex] or 0)
    except ValueError: continue
    t = r[i_src].split()
    if not t: continue
    op = t[1] if t[0].startswith('@') else t[0]
    ops[op.split('.')[0]] += n; tot += n
print(f'total warp-instrs {tot:.3e}  thread-instrs/voxel {tot*32/nvox:.0f}')
for k, v in ops.most_common(22): print(f'  {k:10s} {v/tot*100:5.1f}%  {v*32/nvox:6.1f}/voxel')
