import time, numpy as np, torch, os
n = 330_000_000 // 4
a = torch.zeros(n).pin_memory().numpy(); b = torch.ones(n).pin_memory().numpy()
for _ in range(2):
    t = time.perf_counter(); np.add(a, b, out=a); dt = time.perf_counter() - t
    print(f"1-thread add 330MB: {dt*1e3:.1f} ms  ({3*330/dt/1e3:.1f} GB/s traffic)")
from concurrent.futures import ThreadPoolExecutor
for T in (4, 8, 16):
    ex = ThreadPoolExecutor(T)
    sl = [slice(i * n // T, (i + 1) * n // T) for i in range(T)]
    def f(s): np.add(a[s], b[s], out=a[s])
    list(ex.map(f, sl))
    t = time.perf_counter(); list(ex.map(f, sl)); dt = time.perf_counter() - t
    print(f"{T}-thread add 330MB: {dt*1e3:.1f} ms ({3*330/dt/1e3:.1f} GB/s)")
print(os.cpu_count(), open('/proc/cpuinfo').read().count('processor'))
