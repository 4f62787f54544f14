import sys, os, time
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np, torch
import oracle
from harness import gen
from paper_2403_01164_b200 import hg
from test_gpu_linear import _linear
B = int(os.environ.get("B", 1))
with hg.Context(0, chunk_bytes=64 << 10, ring_bytes=int(os.environ.get("RING", 128 << 10)), max_k=256, max_n=8192, timeout_s=5.0) as c:
    x, W, b = gen.linear_inputs(31, 0, "fc1", B, 4096, 256)
    for n_res, alpha in ((0, 1.0), (512, 1.0), (0, 0.6)):
        t0 = time.time()
        try:
            y = _linear(c, x, W, b, B, n_res, alpha)
            ok, worst = oracle.within_tol(y, oracle.linear(x, W, b))
            print(n_res, alpha, "ok" if ok else "BAD", worst, "%.2fs" % (time.time() - t0), flush=True)
        except Exception as e:
            print(n_res, alpha, "EXC", e, "%.2fs" % (time.time() - t0), flush=True)
            break
