"""Small workload for compute-sanitizer (memcheck / racecheck / synccheck; SURVEY 4 tier 4): the
persistent tag-gated GEMVs (SIMT at B = 1, tcgen05 at B = 4 and K > 8192) with a ring SMALLER than a
linear (cooperative launch, slots refilled inside one launch), resident + streamed + CPU rows, and a
2-layer mirrored stack with prefetch into the next step.  Checks results against the fp64 oracle."""
import os
import sys

os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
from gpu_util import bits, dev, dev_f32, split_weight  # noqa: E402
from harness import gen  # noqa: E402
from paper_2403_01164_b200 import hg  # noqa: E402
from test_gpu_layer import make_layer_mirror  # noqa: E402

bad = 0
with hg.Context(0, chunk_bytes=256 << 10, ring_bytes=1 << 20, max_k=16384, max_n=4096, timeout_s=600.0) as c:
    for B, N, K, n_res, alpha in ((1, 1024, 2048, 128, 0.7), (4, 768, 2048, 0, 0.9), (1, 512, 12288, 128, 0.6)):
        x, W, b = gen.linear_inputs(91, 0, "fc1", B, N, K)
        Wd, Wh = split_weight(W, n_res)
        y = torch.full((B, N), float("nan"), device="cuda")
        c.hg_linear(dev(x), B, N, K, Wd, n_res, Wh, alpha, dev_f32(b), y)
        torch.cuda.synchronize()
        ok, worst = oracle.within_tol(y.cpu().numpy(), oracle.linear(x, W, b))
        print("linear", B, N, K, n_res, alpha, "ok" if ok else "BAD", worst, flush=True)
        bad += not ok
with hg.Context(0, chunk_bytes=256 << 10, ring_bytes=2 << 20, max_k=4096, max_n=8192, wrap_prefetch=1,
                timeout_s=600.0) as c:
    H, F = 256, 1024
    for B in (1, 4):
        keep = []
        layers = [make_layer_mirror(c, H, F, B, layer=l, alpha=0.6, keep=keep, ln=True) for l in range(2)]
        h0 = gen.uniform_bf16(92, 988, B * H, 1.0).reshape(B, H)
        outs = []
        for _ in range(2):
            h = dev(h0)
            c.hg_stack(layers, h, B)
            torch.cuda.synchronize()
            outs.append(bits(h))
        same = np.array_equal(outs[0], outs[1]) and c.hg_stats().mirror_linears > 0
        print("stack B", B, "repeatable" if same else "BAD", flush=True)
        bad += not same
print("WORKLOAD", "OK" if not bad else "BAD")
