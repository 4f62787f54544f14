"""Per-CTA globaltimer stamps of the step's per-linear tcgen05 GEMV launch (hg_gemv_replay) at batch B,
cold (one launch after an L2 flush) and warm (the 2nd of two back-to-back launches).  Stamps (us after
the earliest CTA entry, medians and max over CTAs): 0 entry, 1 producer past the tensor-map
prefetches, 2 first W TMA issued, 3 first MMA stage full, 4 first accumulator handed to the epilogue,
5 epilogue done, 6 exit, 7 producer done issuing.  Measurement only.
  B=8 python tools/tc_stamps.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2403_01164_b200 import hg  # noqa: E402

H, F = 7168, 28672
SHAPES = {"qkv": (3 * H, H), "o": (H, H), "fc1": (F, H), "fc2": (H, F)}
NAMES = ["entry", "prefetched", "1stTMA", "1stFull", "1stAcc", "epiDone", "exit", "prodDone"]


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
        for mode in ("cold", "warm"):
            st = hg.hg_debug_gemv_stamps(4096)
            st[:] = 0
            flush.sum()
            torch.cuda._sleep(200_000)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            if mode == "warm":
                hg.hg_debug_gemv_stamps(0, on=False)
                ctx.hg_gemv_replay(p, x, None, None, y, stream=s, seq0=60)
                hg.hg_debug_gemv_stamps(4096)
            e0.record(s)
            ctx.hg_gemv_replay(p, x, None, None, y, stream=s, seq0=40)
            e1.record(s)
            torch.cuda.synchronize()
            hg.hg_debug_gemv_stamps(0, on=False)
            ev = e0.elapsed_time(e1) * 1e3
            flat = st.reshape(-1)
            n = int((flat[0::8] > 0).sum())
            stm = flat[: n * 8].reshape(n, 8).astype(np.int64)
            t0 = stm[:, 0].min()
            rel = (stm - t0) / 1e3
            cols = " ".join(f"{NAMES[j]} {np.median(rel[:, j]):6.2f}/{rel[:, j].max():6.2f}" for j in range(8))
            print(f"B={B} {name:4s} {mode} rows {p.n_str:5d} chunks {p.n_chunks} ctas {n:3d} | event {ev:6.2f} us | {cols}",
                  flush=True)


if __name__ == "__main__":
    main()
