"""Compile a .cu with -Xptxas -v and print regs/spills per kernel (dev tool).
usage: python tools/ptxas_summary.py <file.cu> [name-filter]"""
import re, subprocess, sys
src = sys.argv[1]; filt = sys.argv[2] if len(sys.argv) > 2 else ""
out = subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17",
                      "-Xcompiler", "-fPIC", "-Iinclude", "-c", src, "-o", "/tmp/ptxas_sum.o",
                      "-Xptxas", "-v"], capture_output=True, text=True).stderr
cur = None
for line in out.splitlines():
    m = re.search(r"Compiling entry function '(\S+)'", line)
    if m:
        cur = m.group(1); spill = ""
        continue
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m and cur:
        spill = f"spill st/ld {m.group(1)}/{m.group(2)}"
    m = re.search(r"Used (\d+) registers", line)
    if m and cur:
        if filt in cur:
            dem = subprocess.run(["c++filt", cur], capture_output=True, text=True).stdout.strip()
            dem = re.sub(r"\(.*", "", dem).replace("mdg::tiled::", "").replace("mdg::", "")
            print(f"{dem:55s} regs {m.group(1):>4s}  {spill}")
        cur = None
for line in out.splitlines():
    if "error" in line: print(line)
