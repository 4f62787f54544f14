"""Per-CTA globaltimer stamps of the step's per-linear GEMV launch (hg_gemv_replay) at batch B:
CTA entry spread, first stage consumed (tcgen05: first MMA stage full; SIMT: first row), consumers
done and CTA exit, against the launch's CUDA-event time.  Measurement only.
  B=8 python tools/tc_stamps.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2403_01164_b200 import hg  # noqa: E402

H, F = 7168, 28672
SHAPES = {"qkv": (3 * H, H), "o": (H, H), "fc1": (F, H), "fc2": (H, F)}


def main():
    B = int(os.environ.get("B", 8))
    alpha = float(os.environ.get("ALPHA", 0.24))
    ctx = hg.Context(0, chunk_bytes=32 << 20, ring_bytes=4096 << 20, max_k=F, max_n=F)
    s = torch.cuda.current_stream()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda").view(torch.float32)
    for name, (N, K) in SHAPES.items():
        p = ctx.plan(hg.make_rates(1, 1, 1), N, K, B, 0, hg.FIXED, alpha)
        x = torch.empty((B, K), dtype=torch.int16, device="cuda").random_(-3000, 3000)
        y = torch.empty((B, N), device="cuda")
        for i in range(3):
            ctx.hg_gemv_replay(p, x, None, None, y, stream=s, seq0=i * 4)
        st = hg.hg_debug_gemv_stamps(4096)
        st[:] = 0
        flush.sum()
        torch.cuda._sleep(200_000)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        ctx.hg_gemv_replay(p, x, None, None, y, stream=s, seq0=40)
        e1.record(s)
        torch.cuda.synchronize()
        hg.hg_debug_gemv_stamps(0, on=False)
        ev = e0.elapsed_time(e1) * 1e3
        n = int((st[:, 0] > 0).sum())
        t0 = st[:n, 0].min()
        rel = (st[:n].astype(np.int64) - int(t0)) / 1e3
        first = rel[:, 1][st[:n, 1] > 0] - rel[:, 0][st[:n, 1] > 0]
        print(f"B={B} {name:4s} rows {p.n_str:5d} chunks {p.n_chunks} ctas {n:3d} | event {ev:6.2f} us | entry spread "
              f"{rel[:, 0].max():5.2f} | first stage after entry med {np.median(first):5.2f} max {first.max():5.2f} | "
              f"work done med {np.median(rel[:, 2]):6.2f} max {rel[:, 2].max():6.2f} | exit max {rel[:, 3].max():6.2f} us",
              flush=True)


if __name__ == "__main__":
    main()
