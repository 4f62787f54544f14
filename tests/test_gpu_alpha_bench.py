"""GPU test of the alpha benchmark (Sec. 4.4; VERDICT r1 missing #3).

hg_alpha_bench runs the stack at every alpha of the window around the seed (reading R9), measures
the lanes and solves F_CPU = F_COM.  Checked: the sampled alphas are the window
[seed-gamma, seed+gamma] cap [0,1] at step lambda (oracle.alpha_window); the lane times are
positive and the CPU time falls / the link time rises with alpha (more rows streamed, fewer on
the CPU); alpha_bar equals the oracle's solve on the returned samples; and the stack re-planned
at alpha_bar (and at a clamped-window seed) matches the oracle teacher-forced.
"""
import numpy as np
import pytest
import torch

import oracle
from gpu_util import bits, dev
from harness import gen
from paper_2403_01164_b200 import hg
from test_gpu_layer import make_layer_mirror

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("seed_alpha,gamma", [(0.4, 0.06), (0.97, 0.1)])
def test_alpha_bench_window_solve_and_replan(seed_alpha, gamma):
    H, F, B, NL = 1024, 4096, 1, 4
    with hg.Context(0, chunk_bytes=1 << 20, ring_bytes=64 << 20, max_k=8192, max_n=16384) as c:
        keep = []
        layers = [make_layer_mirror(c, H, F, B, layer=l, alpha=seed_alpha, keep=keep) for l in range(NL)]
        h0 = gen.uniform_bf16(31, 990, B * H, 1.0).reshape(B, H)
        h = dev(h0)
        res = c.hg_alpha_bench(layers, h, B, seed_alpha, gamma=gamma, lam=0.02, degree=2, reps=2)
        torch.cuda.synchronize()
        d = res.as_dict()
        win = oracle.alpha_window(seed_alpha, gamma, 0.02)
        assert len(d["alpha"]) == len(win)
        assert np.allclose(d["alpha"], win, rtol=0, atol=1e-12)
        # (near alpha = 1 every row of the small linears is streamed and the CPU lane idles: t_cpu = 0)
        assert d["t_cpu"][0] > 0 and all(t >= 0 for t in d["t_cpu"])
        assert all(t > 0 for t in d["t_com"]) and all(t > 0 for t in d["t_step"])
        # more rows streamed -> the link's share grows, the CPU's shrinks (robust ends of the window)
        assert d["t_com"][-1] > d["t_com"][0] and d["t_cpu"][-1] < d["t_cpu"][0]
        ref, clamped = oracle.alpha_bench_solve(d["alpha"], d["t_cpu"], d["t_com"], 2, win[0], win[-1], seed_alpha)
        assert abs(d["alpha_bar"] - ref) <= 1e-9 and bool(d["clamped"]) == clamped
        assert win[0] <= d["alpha_bar"] <= win[-1]
        # re-plan at alpha_bar and check every linear of layer 1 against the oracle, teacher-forced
        a_bar = d["alpha_bar"]
        layers2 = [make_layer_mirror(c, H, F, B, layer=l, alpha=a_bar, keep=keep) for l in range(NL)]
        for L in layers2:
            for dsc in L.lin:
                assert dsc.plan.n_str == oracle.partition(dsc.plan.N, 0, a_bar, 128)[1]
        h = dev(h0)
        for L in layers2[:1]:
            c.hg_layer(L, h, B)
        tr = {k: torch.zeros(B, n, dtype=torch.int16, device="cuda") for k, n in
              (("a", H), ("v", H), ("h1", H), ("a2", H), ("u", F))}
        tr.update({k: torch.zeros(B, n, device="cuda") for k, n in
                   (("y_qkv", 3 * H), ("y_o", H), ("y_fc1", F), ("y_fc2", H))})
        c.hg_layer(layers2[1], h, B, hg.layer_trace(**tr))
        torch.cuda.synchronize()
        T = {k: (bits(v) if v.dtype == torch.int16 else v.cpu().numpy()) for k, v in tr.items()}
        shapes = {"qkv": (3 * H, H), "o": (H, H), "fc1": (F, H), "fc2": (H, F)}
        for name, xin, yk in (("qkv", "a", "y_qkv"), ("o", "v", "y_o"), ("fc1", "a2", "y_fc1"), ("fc2", "u", "y_fc2")):
            _, W, b = gen.linear_inputs(21, 1, name, 1, *shapes[name])
            ok, worst = oracle.within_tol(T[yk], oracle.linear(T[xin], W, b))
            assert ok, (name, worst)
