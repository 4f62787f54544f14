"""Quick lane microbenchmarks on one GPU (development tool, not the bench contract).

  resident GEMV GB/s (hg_gemv) for B in 1,2,4,8 on OPT-30B fc1 / fc2 shapes
  hg_measure rates on a pinned OPT-30B fc1 weight
  hg_linear ms at an alpha sweep (C4 fc1, B=1)
"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from harness import gen  # noqa: E402
from paper_2403_01164_b200 import hg  # noqa: E402


def gemv_bw(ctx, N, K, B, iters=20):
    W = torch.empty((N, K), dtype=torch.int16, device="cuda").random_(-20000, 20000)
    x = torch.empty((B, K), dtype=torch.int16, device="cuda").random_(-20000, 20000)
    y = torch.empty((B, N), device="cuda")
    s = torch.cuda.current_stream()
    for _ in range(3):
        ctx.hg_gemv(x, B, N, K, W, None, y, stream=s)
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    ts = []
    for _ in range(iters):
        flush.zero_()
        e0.record(s)
        ctx.hg_gemv(x, B, N, K, W, None, y, stream=s)
        e1.record(s)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e-3)
    t = float(np.median(ts))
    return 2 * N * K / t / 1e9, t


def main():
    out = {}
    ctx = hg.Context(0, cpu_threads=int(os.environ.get("HG_THREADS", "0")))
    for (N, K) in ((28672, 7168), (7168, 28672), (21504, 7168)):
        for B in (1, 2, 4, 8):
            gbs, t = gemv_bw(ctx, N, K, B)
            out[f"gemv_{N}x{K}_B{B}"] = {"GB/s": round(gbs, 1), "us": round(t * 1e6, 1)}
            print(f"gemv {N}x{K} B={B}: {gbs:.1f} GB/s  {t*1e6:.1f} us", flush=True)
    N, K = 28672, 7168
    Wh = torch.empty((N, K), dtype=torch.int16, pin_memory=True)
    gen.uniform_bf16(1164, 2, N * K, gen.w_scale(K), out=Wh.data_ptr())
    for B in (1, 8):
        for load in (False, True):
            r = ctx.hg_measure(Wh, N, K, B, under_load=load)
            out[f"measure_B{B}_load{int(load)}"] = {k: v / 1e9 for k, v in r.as_dict().items()}
            print(f"measure B={B} under_load={load}: " +
                  " ".join(f"{k}={v/1e9:.1f}" for k, v in r.as_dict().items()), flush=True)
    r = ctx.hg_measure(Wh, N, K, 1, under_load=True)
    x = torch.empty((1, K), dtype=torch.int16, device="cuda").random_(-2000, 2000)
    y = torch.empty((1, N), device="cuda")
    bias = torch.zeros(N, device="cuda")
    s = torch.cuda.current_stream()
    for a in (0.0, 0.2, 0.3, 0.35, 0.4, 0.5, 1.0, "plan"):
        if a == "plan":
            p = ctx.plan(r, N, K, 1, 0, hg.EXACT)
        else:
            p = ctx.plan(r, N, K, 1, 0, hg.FIXED, a)
        for _ in range(2):
            ctx.hg_linear_planned(p, x, None, Wh, bias, y, stream=s)
        torch.cuda.synchronize()
        ts = []
        for _ in range(10):
            t0 = time.perf_counter()
            ctx.hg_linear_planned(p, x, None, Wh, bias, y, stream=s)
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - t0)
        t = float(np.median(ts))
        out[f"linear_alpha_{a}"] = {"ms": t * 1e3, "alpha": p.alpha_eff, "t_pred_ms": p.t_pred * 1e3,
                                    "t_roof_ms": p.t_roof * 1e3}
        print(f"hg_linear fc1 alpha={a} ({p.alpha_eff:.3f}): {t*1e3:.3f} ms  pred {p.t_pred*1e3:.3f}  "
              f"roof {p.t_roof*1e3:.3f}", flush=True)
    os.makedirs("gpurun_out", exist_ok=True)
    json.dump(out, open("gpurun_out/microbench.json", "w"), indent=1)


if __name__ == "__main__":
    main()
