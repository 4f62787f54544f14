"""C4 (BJ:10) alpha sweep and C1 (BJ:7) per-call time, one B200 (SURVEY 8(c) c4 "alpha sweep on B200":
the argmin of the measured time over the alpha grid should sit within one grid step of hg_plan's
alpha).

  C4: OPT-30B fc1 [28672, 7168] and fc2 [7168, 28672], r = 0, batch 1 and 8, alpha in {0, 0.1, ...,
      1} plus the Eq. (5) alpha from rates measured on this box; ms per hg_linear_planned call
      (median of --reps, host-blocking for the CPU slice), beside the plan's predicted and roofline
      times.
  C1: OPT-125M fc1 [3072, 768], batch 1, alpha 0.5: us per hg_linear call (overhead-dominated).

  python tools/alpha_sweep.py [--reps 7]    -> JSON lines, then a markdown table
"""
import argparse
import json
import os
import statistics
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from harness import gen  # noqa: E402
from paper_2403_01164_b200 import hg  # noqa: E402

SEED = 1164 + 3


def time_calls(fn, reps):
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    return statistics.median(ts)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=7)
    args = ap.parse_args()
    torch.cuda.set_device(0)
    s = torch.cuda.current_stream()
    ctx = hg.Context(0, chunk_bytes=32 << 20, ring_bytes=4096 << 20, max_k=28672, max_n=28672)
    rows = []
    for name, (N, K) in (("fc1", (28672, 7168)), ("fc2", (7168, 28672))):
        Wh = torch.empty((N, K), dtype=torch.int16, pin_memory=True)
        gen.uniform_bf16(SEED, gen.tensor_id(0, name, "W"), N * K, gen.w_scale(K), out=Wh.data_ptr())
        b = torch.from_numpy(gen.bf16_bits_to_f32(gen.uniform_bf16(SEED, gen.tensor_id(0, name, "bias"), N,
                                                                   gen.BIAS_SCALE))).cuda()
        for B in (1, 8):
            x = torch.from_numpy(gen.uniform_bf16(SEED, gen.tensor_id(0, name, "x"), B * K, 1.7320508)
                                 .view("int16")).reshape(B, K).cuda()
            y = torch.empty((B, N), device="cuda")
            rates = ctx.hg_measure(Wh, N, K, B, under_load=True)
            p_plan = ctx.plan(rates, N, K, B, 0, hg.EXACT)
            grid = [round(0.1 * i, 1) for i in range(11)]
            pts = []
            for a in grid + [None]:
                p = p_plan if a is None else ctx.plan(rates, N, K, B, 0, hg.FIXED, a)
                run = lambda: ctx.hg_linear_planned(p, x, None, Wh, b, y, stream=s)  # noqa: E731
                run()
                t = time_calls(run, args.reps)
                pd = p.as_dict()
                pt = {"linear": name, "B": B, "alpha": "plan" if a is None else a, "alpha_eff": round(p.alpha_eff, 4),
                      "ms": round(t * 1e3, 4), "pred_ms": round(pd["t_pred"] * 1e3, 4),
                      "roof_ms": round(pd["t_roof"] * 1e3, 4)}
                print(json.dumps(pt), flush=True)
                pts.append(pt)
            sweep = [q for q in pts if q["alpha"] != "plan"]
            best = min(sweep, key=lambda q: q["ms"])
            plan = pts[-1]
            rows.append((name, B, plan, best, abs(best["alpha_eff"] - plan["alpha_eff"]) <= 0.1 + 1e-9, sweep))
        del Wh
    # C1
    x1, W1, b1 = gen.linear_inputs(1164, 0, "fc1", 1, 3072, 768)
    W1h = torch.empty((3072, 768), dtype=torch.int16, pin_memory=True)
    W1h.numpy()[...] = W1.view("int16")
    xd = torch.from_numpy(x1.view("int16")).cuda()
    bd = torch.from_numpy(b1).cuda()
    y1 = torch.empty((1, 3072), device="cuda")
    c1 = lambda: ctx.hg_linear(xd, 1, 3072, 768, None, 0, W1h, 0.5, bd, y1, stream=s)  # noqa: E731
    for _ in range(20):
        c1()
    t1 = time_calls(c1, 200)
    print(json.dumps({"config": "C1 OPT-125M fc1 768->3072, batch 1, alpha 0.5", "us_per_call": round(t1 * 1e6, 1)}),
          flush=True)
    print("\n| linear | B | plan alpha | plan ms | pred ms | roofline ms | grid argmin alpha | argmin ms | within one step |")
    print("|---|---|---|---|---|---|---|---|---|")
    for name, B, plan, best, ok, _ in rows:
        print(f"| {name} | {B} | {plan['alpha_eff']:.3f} | {plan['ms']:.3f} | {plan['pred_ms']:.3f} | {plan['roof_ms']:.3f} "
              f"| {best['alpha_eff']:.1f} | {best['ms']:.3f} | {'yes' if ok else 'no'} |")
    print("\n| linear | B | " + " | ".join(f"a={a/10:.1f}" for a in range(11)) + " |")
    print("|---|---|" + "---|" * 11)
    for name, B, _, _, _, sweep in rows:
        print(f"| {name} | {B} | " + " | ".join(f"{q['ms']:.2f}" for q in sweep) + " |")
    print(f"\nC1: {t1 * 1e6:.1f} us per hg_linear call (OPT-125M fc1, batch 1, alpha 0.5; median of 200)")


if __name__ == "__main__":
    main()
