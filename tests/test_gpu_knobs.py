"""The library's A/B switches (environment variables read once per process) keep parity with the
oracle: each combination runs in a fresh subprocess on a small hetero linear and a fully streamed
one, at a SIMT and a tcgen05 batch, and compares against the fp64 oracle (same tolerance)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, %(root)r); sys.path.insert(0, %(tests)r)
import oracle
from harness import gen
from paper_2403_01164_b200 import hg
from gpu_util import dev, dev_f32, split_weight
bad = []
with hg.Context(0, chunk_bytes=1 << 20, ring_bytes=64 << 20, max_k=32768, max_n=8192) as c:
    for B in (1, 3, 4, 8):
        for (N, K, n_res, alpha) in ((1024, 7168, 128, 0.6), (640, 12288, 0, 1.0), (512, 1000, 256, 0.0)):
            x, W, b = gen.linear_inputs(77, 0, "fc1", B, N, K)
            Wd, Wh = split_weight(W, n_res)
            y = torch.full((B, N), float("nan"), device="cuda")
            c.hg_linear(dev(x), B, N, K, Wd, n_res, Wh, alpha, dev_f32(b), y)
            torch.cuda.synchronize()
            ok, worst = oracle.within_tol(y.cpu().numpy(), oracle.linear(x, W, b))
            if not ok:
                bad.append((B, N, K, n_res, alpha, worst))
print("BAD" if bad else "OK", bad)
"""


@pytest.mark.parametrize("env", [
    {"HG_TC_LONG_K": "0"},
    {"HG_GEMV_PDL": "0"},
    {"HG_TC_STREAM": "0"},
    {"HG_GEMV_TC_MIN_BATCH": "0"},
    {"HG_TC_CLUSTER": "0"},
    {"HG_GEMV_ROW": "0"},
    {"HG_GEMV_ROW": "0", "HG_GEMV_CPS": "1"},
    {"HG_GEMV_PROW": "0"},
    {"HG_ROW_BMAX": "1"},
    {"HG_ROW_BMAX": "4"},
    {"HG_ROW_B4_KMAX": "8192"},
    {"HG_TC_ST": "6"},
    {"HG_TC_ST": "4"},
], ids=lambda e: ",".join(f"{k}={v}" for k, v in e.items()))
def test_switch_keeps_parity(env):
    code = SCRIPT % {"root": ROOT, "tests": os.path.join(ROOT, "tests")}
    r = subprocess.run([sys.executable, "-c", code], env={**os.environ, **env}, capture_output=True, text=True,
                       timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    assert r.stdout.strip().startswith("OK"), r.stdout[-2000:]


BITS_SCRIPT = r"""
import sys, hashlib, numpy as np, torch
sys.path.insert(0, %(root)r); sys.path.insert(0, %(tests)r)
from harness import gen
from paper_2403_01164_b200 import hg
from gpu_util import dev, dev_f32, split_weight
out = []
with hg.Context(0, chunk_bytes=1 << 20, ring_bytes=64 << 20, max_k=32768, max_n=8192) as c:
    for (N, K, n_res, alpha) in ((1024, 7168, 128, 1.0), (640, 28672, 0, 1.0), (512, 1000, 256, 1.0),
                                 (768, 4096, 0, 0.7), (384, 12288, 128, 1.0)):
        x, W, b = gen.linear_inputs(78, 0, "fc1", 1, N, K)
        Wd, Wh = split_weight(W, n_res)
        y = torch.full((1, N), float("nan"), device="cuda")
        c.hg_linear(dev(x), 1, N, K, Wd, n_res, Wh, alpha, dev_f32(b), y)
        torch.cuda.synchronize()
        out.append(hashlib.sha256(y.cpu().numpy().tobytes()).hexdigest()[:16])
print("BITS", " ".join(out))
"""


def test_row_kernels_bit_equal_staged_kernel():
    """B = 1: the warp-per-row kernel (K <= 8192) and the part-row kernel (K > 8192, part sums folded in
    part order) compute the same bits as the staged TMA kernel with its workspace fold (HG_GEMV_ROW=0,
    HG_GEMV_PROW=0, HG_TC_LONG_K=0 keeps long rows on it): same per-lane order, butterfly and fold, and
    fma.rn.f32.bf16 equals fmaf of the converted values (an exact product, one rounding)."""
    code = BITS_SCRIPT % {"root": ROOT, "tests": os.path.join(ROOT, "tests")}
    digests = []
    for env in ({}, {"HG_GEMV_ROW": "0", "HG_GEMV_PROW": "0", "HG_TC_LONG_K": "0"}):
        r = subprocess.run([sys.executable, "-c", code], env={**os.environ, **env}, capture_output=True, text=True,
                           timeout=600, cwd=ROOT)
        assert r.returncode == 0, r.stderr[-2000:]
        line = [ln for ln in r.stdout.splitlines() if ln.startswith("BITS")]
        assert line, r.stdout[-2000:]
        digests.append(line[0])
    assert digests[0] == digests[1], digests
