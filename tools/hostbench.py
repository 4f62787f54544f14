import numpy as np, time, os, sys
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from harness import gen
from paper_2403_01164_b200 import hg
N,K=28672,7168
for B in (1,2,4,8):
    x, W, b = gen.linear_inputs(45, 0, "fc1", B, N, K)
    y = np.zeros((B, N), np.float32)
    with hg.Context(-1, cpu_threads=int(os.environ.get("THREADS", 16))) as c:
        c.hg_host_gemv(x, B, N, K, W, b, y)
        ts=[]
        for _ in range(7):
            t=time.perf_counter(); c.hg_host_gemv(x, B, N, K, W, b, y); ts.append(time.perf_counter()-t)
    print(os.environ.get("HG_AMX_MIN_BATCH"), B, round(2*N*K/np.median(ts)/1e9,1), "GB/s")
