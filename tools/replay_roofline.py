"""The bench's GEMV roofline (bench.gemv_roofline: the step's per-linear GEMV launches, 20 back to
back walking the ring) for OPT-30B at a fixed alpha and batch, without the rest of the bench.
  B=8 ALPHA=0.24 python tools/replay_roofline.py        (A/B knobs: HG_TC_SLICE, HG_GEMV_PDL, ...)"""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2403_01164_b200 import hg  # noqa: E402

H, F = int(os.environ.get("H", 7168)), int(os.environ.get("F", 0)) or 4 * int(os.environ.get("H", 7168))
SHAPES = {"qkv": (3 * H, H), "o": (H, H), "fc1": (F, H), "fc2": (H, F)}


def main():
    B = int(os.environ.get("B", 1))
    alpha = float(os.environ.get("ALPHA", 0.24))
    extra = {"gemv_tc_min_batch": int(os.environ["TCMIN"])} if "TCMIN" in os.environ else {}
    ctx = hg.Context(0, chunk_bytes=32 << 20, ring_bytes=4096 << 20, max_k=F, max_n=F, **extra)
    plans = {n: ctx.plan(hg.make_rates(1, 1, 1), N, K, B, 0, hg.FIXED, alpha) for n, (N, K) in SHAPES.items()}
    r = bench.gemv_roofline(ctx, plans, 48, B, torch, bench.peaks())
    print(json.dumps({"B": B, "alpha": alpha, "env": {k: v for k, v in os.environ.items() if k.startswith("HG_") or k == "TCMIN"},
                      "achieved": r.get("achieved"), "frac": r.get("frac"),
                      "per_linear": {k: (v["us"], v["GBps"]) for k, v in r.get("per_linear", {}).items()}}))


if __name__ == "__main__":
    main()
