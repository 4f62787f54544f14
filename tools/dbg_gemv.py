"""Debug driver: one hg_gemv / hg_linear per (B, N, K) given on the command line."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np, torch
import oracle
from harness import gen
from paper_2403_01164_b200 import hg
from gpu_util import dev, dev_f32, split_weight

B, N, K = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
mode = sys.argv[4] if len(sys.argv) > 4 else "gemv"
ctx = hg.Context(0, chunk_bytes=1 << 20, ring_bytes=64 << 20, max_k=65536, max_n=65536)
x, W, b = gen.linear_inputs(7, 0, "fc1", B, N, K)
y = torch.full((B, N), float("nan"), device="cuda")
if mode == "gemv":
    ctx.hg_gemv(dev(x), B, N, K, dev(W), dev_f32(b), y)
else:
    n_res = int(sys.argv[5]); alpha = float(sys.argv[6])
    Wd, Wh = split_weight(W, n_res)
    ctx.hg_linear(dev(x), B, N, K, Wd, n_res, Wh, alpha, dev_f32(b), y)
torch.cuda.synchronize()
ok, worst = oracle.within_tol(y.cpu().numpy(), oracle.linear(x, W, b))
print(B, N, K, mode, "ok" if ok else "FAIL", worst)
