"""C5 (BJ:11) on one GPU: rank 0's row shard of the OPT-175B linears (P = 8), r = 0.1 resident per
shard (fc1 n_res = 640 of 6144, fc2 128 of 1536), alpha from Eq. (5) with rates measured
on this box, batch 1.  Each linear runs as hg_linear_planned calls (host-blocking for the CPU slice),
rotating over 4 weight copies so the CPU lane's reads come from DRAM, not the 60 MB L3.  The NCCL
all-gather of the 8 shards needs 8 GPUs and is not in these numbers; with all host cores on one
rank the CPU lane is faster than it would be with 8 ranks sharing the host.

  python tools/c5_shard.py [--reps 10]     -> one JSON line per linear + a per-layer summary
"""
import argparse
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from harness import gen  # noqa: E402
from paper_2403_01164_b200 import hg  # noqa: E402

H, F, P, LAYERS = 12288, 49152, 8, 96
SHAPES = {"qkv": (3 * H, H), "o": (H, H), "fc1": (F, H), "fc2": (H, F)}
SEED = 1164 + 4


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--copies", type=int, default=4)
    ap.add_argument("--r", type=float, default=0.1)
    args = ap.parse_args()
    torch.cuda.set_device(0)
    ctx = hg.Context(0, chunk_bytes=32 << 20, ring_bytes=4096 << 20, max_k=F, max_n=F)
    s = torch.cuda.current_stream()
    out, tot_ms, tot_roof = {}, 0.0, 0.0
    rates = None
    for name, (N, K) in SHAPES.items():
        n = N // P  # rank 0's rows [0, N/P)
        n_res = bench.resident_rows(args.r, n)
        copies = []
        for c in range(args.copies):
            W = torch.empty((n, K), dtype=torch.int16, pin_memory=True)
            gen.uniform_bf16(SEED + c, gen.tensor_id(0, name, "W"), n * K, gen.w_scale(K), out=W.data_ptr())
            copies.append((W[:n_res].cuda() if n_res else None, W[n_res:]))
        b = torch.from_numpy(gen.bf16_bits_to_f32(gen.uniform_bf16(SEED, gen.tensor_id(0, name, "bias"), n,
                                                                   gen.BIAS_SCALE))).cuda()
        x = torch.from_numpy(gen.uniform_bf16(SEED, gen.tensor_id(0, name, "x"), K, 1.7320508).view("int16")
                             ).reshape(1, K).cuda()
        if rates is None or name == "fc1":
            rates = ctx.hg_measure(copies[0][1], n - n_res, K, 1, under_load=True)
        p = ctx.plan(rates, n, K, 1, n_res, hg.EXACT)
        y = torch.empty((1, n), device="cuda")
        for c in range(2):
            ctx.hg_linear_planned(p, x, copies[c][0], copies[c][1], b, y, stream=s)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for i in range(args.reps):
            Wd, Wh = copies[i % args.copies]
            ctx.hg_linear_planned(p, x, Wd, Wh, b, y, stream=s)
        torch.cuda.synchronize()
        ms = (time.perf_counter() - t0) / args.reps * 1e3
        pd = p.as_dict()
        roof_ms = pd["t_roof"] * 1e3
        out[name] = {"rows": n, "K": K, "n_res": p.n_res, "n_str": p.n_str, "n_cpu": p.n_cpu,
                     "alpha": round(p.alpha_eff, 4), "ms": round(ms, 4), "t_roof_ms": round(roof_ms, 4),
                     "frac": round(roof_ms / ms, 4), "t_pred_ms": round(pd["t_pred"] * 1e3, 4)}
        print(json.dumps({"linear": name, **out[name]}), flush=True)
        tot_ms += ms
        tot_roof += roof_ms
        del copies
    rd = rates.as_dict()
    print(json.dumps({"config": "C5 OPT-175B rank 0 of 8 (row shard), r=%.2f, batch 1, one GPU, no all-gather"
                      % args.r, "ms_per_layer_shard": round(tot_ms, 4), "roof_ms_per_layer_shard": round(tot_roof, 4),
                      "frac": round(tot_roof / tot_ms, 4), "ms_per_token_shard_x96": round(tot_ms * LAYERS, 2),
                      "rates_GBps": {k: round(v / 1e9, 2) for k, v in rd.items() if k.startswith(("v_", "b_"))
                                     and v == v and v != float("inf")},
                      "note": "per-linear hg_linear_planned calls (no cross-linear prefetch); the stack's "
                              "all-gather needs 8 GPUs"}), flush=True)


if __name__ == "__main__":
    main()
