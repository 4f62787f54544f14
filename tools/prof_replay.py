"""ncu driver: the step's persistent GEMV launch per OPT-30B linear (hg_gemv_replay), r = 0,
alpha given (default 0.23), batch 1, 32 MiB chunks -- the bench's launch configuration.
Prints CUDA-event times per linear (L2 flushed between launches)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2403_01164_b200 import hg  # noqa: E402

H, F = 7168, 28672
SHAPES = {"qkv": (3 * H, H), "o": (H, H), "fc1": (F, H), "fc2": (H, F)}


def main():
    alpha = float(os.environ.get("ALPHA", 0.23))
    B = int(os.environ.get("B", 1))
    reps = int(os.environ.get("REPS", 5))
    ctx = hg.Context(0, chunk_bytes=32 << 20, ring_bytes=4096 << 20, max_k=F, max_n=F)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    s = torch.cuda.current_stream()
    for name, (N, K) in SHAPES.items():
        p = ctx.plan(hg.make_rates(1, 1, 1), N, K, B, 0, hg.FIXED, alpha)
        x = torch.empty((B, K), dtype=torch.int16, device="cuda").random_(-3000, 3000)
        y = torch.empty((B, N), device="cuda")
        ts = []
        for _ in range(reps):
            flush.zero_()
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            e0.record(s)
            ctx.hg_gemv_replay(p, x, None, None, y, stream=s, seq0=0)
            e1.record(s)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3)
        nb = 2 * K * (p.n_res + p.n_str)
        t = sorted(ts)[len(ts) // 2]
        print(f"{name}: rows {p.n_str} chunks {p.n_chunks} {nb/1e6:.1f} MB  {t:.2f} us  {nb/t/1e3:.0f} GB/s", flush=True)


if __name__ == "__main__":
    main()
