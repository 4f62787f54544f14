"""Tiny driver for ncu captures of the device GEMV kernels (OPT-30B fc1 shape, resident)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2403_01164_b200 import hg  # noqa: E402


def main():
    N, K = int(os.environ.get("N", 28672)), int(os.environ.get("K", 7168))
    batches = [int(b) for b in os.environ.get("BATCHES", "1,4,8").split(",")]
    ctx = hg.Context(0, max_k=max(K, 8), max_n=max(N, 8))
    W = torch.empty((N, K), dtype=torch.int16, device="cuda").random_(-20000, 20000)
    for B in batches:
        x = torch.empty((B, K), dtype=torch.int16, device="cuda").random_(-2000, 2000)
        y = torch.empty((B, N), device="cuda")
        for _ in range(3):
            ctx.hg_gemv(x, B, N, K, W, None, y)
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
