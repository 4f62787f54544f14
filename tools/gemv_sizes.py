"""GEMV per-launch time vs rows (K, B=1): mean of back-to-back launches with CUDA events (L2 warm
for small n -- this isolates the fixed per-launch cost), or an ncu driver with NCU=1."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2403_01164_b200 import hg

K = int(os.environ.get("K", 7168))
ctx = hg.Context(0, max_k=K, max_n=32768)
W = torch.empty((28672, K), dtype=torch.int16, device="cuda").random_(-3000, 3000)
x = torch.empty((1, K), dtype=torch.int16, device="cuda").random_(-3000, 3000)
y = torch.empty((1, 28672), device="cuda")
s = torch.cuda.current_stream()
for n in (128, 512, 2048, 8192, 28672):
    reps = 2 if os.environ.get("NCU") else 200
    for _ in range(3):
        ctx.hg_gemv(x, 1, n, K, W, None, y)
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record(s)
    for _ in range(reps):
        ctx.hg_gemv(x, 1, n, K, W, None, y)
    e1.record(s)
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) * 1e3 / reps
    print(f"rows {n:6d}  {2*n*K/1e6:8.2f} MB  {t:7.2f} us/launch  {2*n*K/t/1e3:7.0f} GB/s", flush=True)
