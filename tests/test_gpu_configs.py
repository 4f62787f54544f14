"""GPU parity at BASELINE.json's configurations (BJ:7-11), full sizes, production
launch configuration (16 MiB chunks, 1 GiB ring, G = 128), against the fp64 oracle.

C1 OPT-125M fc1 (test_gpu_linear.py), C2 OPT-6.7B layer r=0.5, C3 OPT-13B 40-layer
stack (layers {0, 20, 39} teacher-forced; hg_stack bit-identical to layer calls),
C4 OPT-30B fc1/fc2 alpha sweep at batch 1 and 8, C5 OPT-175B per-rank shard (P=8,
r=0.1).  Tolerance: elementwise |y - y_ref| <= 1e-2 max(1, |y_ref|) (BJ:5).
"""
import math

import numpy as np
import pytest
import torch

import oracle
from gpu_util import bits, dev, dev_f32, pinned
from harness import gen
from paper_2403_01164_b200 import hg

pytestmark = pytest.mark.gpu

NAMES = ("qkv", "o", "fc1", "fc2")


def shapes(H, F):
    return {"qkv": (3 * H, H), "o": (H, H), "fc1": (F, H), "fc2": (H, F)}


@pytest.fixture(scope="module")
def ctx():
    c = hg.Context(0, max_k=65536, max_n=65536)  # production defaults otherwise
    yield c
    c.close()


RATES = hg.make_rates(170e9, 5e12, 55e9, b_hbm=6.5e12, b_link=55e9, b_cpu=180e9)


def run_linear(ctx, x, W, b, B, n_res, alpha=None):
    N, K = W.shape
    p = ctx.plan(RATES, N, K, B, n_res, hg.EXACT if alpha is None else hg.FIXED, alpha or 0.0)
    Wd = dev(W[:n_res]) if n_res else None
    Wh = pinned(W[n_res:]) if n_res < N else None
    y = torch.full((B, N), float("nan"), device="cuda")
    ctx.hg_linear_planned(p, dev(x), Wd, Wh, dev_f32(b), y)
    torch.cuda.synchronize()
    return y.cpu().numpy(), p


@pytest.mark.parametrize("B", [1, 8])
@pytest.mark.parametrize("name", ["fc1", "fc2"])
def test_c4_opt30b_mlp_alpha_sweep(ctx, B, name):
    N, K = shapes(7168, 28672)[name]
    x, W, b = gen.linear_inputs(1164 + 3, 0, name, B, N, K)
    ref = oracle.linear(x, W, b, nthreads=16)
    for alpha in (0.0, 0.25, 0.5, 0.75, 1.0, None):
        y, p = run_linear(ctx, x, W, b, B, 0, alpha)
        ok, worst = oracle.within_tol(y, ref)
        assert ok, (alpha, p.n_str, worst)


def test_c5_opt175b_rank_shards(ctx):
    """C5: OPT-175B fc1 [49152, 12288] / fc2 [12288, 49152] at P = 8: rank 3's shard, r = 0.1."""
    for name, (N, K) in (("fc1", (49152, 12288)), ("fc2", (12288, 49152))):
        r0, r1 = oracle.shard(N, 8, 3, 128)
        x, _, _ = gen.linear_inputs(1164 + 4, 0, name, 1, 8, K, bias=False)
        W = gen.uniform_bf16(1164 + 4, gen.tensor_id(0, name, "W"), (r1 - r0) * K, gen.w_scale(K),
                             offset=r0 * K).reshape(r1 - r0, K)
        b = gen.bf16_bits_to_f32(gen.uniform_bf16(1164 + 4, gen.tensor_id(0, name, "bias"), r1 - r0,
                                                  gen.BIAS_SCALE, offset=r0))
        n_res = oracle.resident_rows(0.1, r1 - r0, 128)
        assert n_res == {"fc1": 640, "fc2": 128}[name]
        y, p = run_linear(ctx, x, W, b, 1, n_res)
        assert p.n_res + p.n_str + p.n_cpu == r1 - r0
        ok, worst = oracle.within_tol(y, oracle.linear(x, W, b, nthreads=16))
        assert ok, (name, worst)


def build_layer(ctx, H, F, B, layer, seed, r, rates=RATES, keep=None):
    descs, Wd, bd = [], {}, {}
    for name in NAMES:
        N, K = shapes(H, F)[name]
        _, W, b = gen.linear_inputs(seed, layer, name, 1, N, K)
        Wd[name], bd[name] = W, b
        n_res = oracle.resident_rows(r, N, 128)
        p = ctx.plan(rates, N, K, B, n_res, hg.EXACT)
        W_dev = dev(W[:n_res]) if n_res else None
        W_host = pinned(W[n_res:]) if n_res < N else None
        bias = dev_f32(b)
        keep += [W_dev, W_host, bias]
        descs.append(hg.linear_desc(p, W_dev, W_host, bias))
    return hg.opt_layer(H, F, descs), Wd, bd


def trace_bufs(B, H, F):
    tr = {k: torch.zeros(B, n, dtype=torch.int16, device="cuda") for k, n in
          (("a", H), ("v", H), ("h1", H), ("a2", H), ("u", F))}
    tr.update({k: torch.zeros(B, n, device="cuda") for k, n in
               (("y_qkv", 3 * H), ("y_o", H), ("y_fc1", F), ("y_fc2", H))})
    return tr


def check_layer_trace(tr, h_in, Wd, bd, H):
    T = {k: (bits(v) if v.dtype == torch.int16 else v.cpu().numpy()) for k, v in tr.items()}
    for name, xin, yk in (("qkv", "a", "y_qkv"), ("o", "v", "y_o"), ("fc1", "a2", "y_fc1"), ("fc2", "u", "y_fc2")):
        ok, worst = oracle.within_tol(T[yk], oracle.linear(T[xin], Wd[name], bd[name], nthreads=16))
        assert ok, (name, worst)
    chk = lambda got, ref: oracle.within_tol(oracle.bf16_to_f64(got), oracle.bf16_to_f64(ref))[0]
    assert chk(T["a"], oracle.layernorm(h_in))
    assert chk(T["v"], oracle.attention_pos0(T["y_qkv"], H))
    assert chk(T["h1"], oracle.residual(h_in, T["y_o"]))
    assert chk(T["a2"], oracle.layernorm(T["h1"]))
    assert chk(T["u"], oracle.relu_bf16(T["y_fc1"]))
    return T


def test_c2_opt6p7b_layer_half_resident(ctx):
    """C2: OPT-6.7B decoder layer (h=4096, ffn=16384), batch 1, 50% of each weight resident."""
    H, F, B = 4096, 16384, 1
    keep = []
    L, Wd, bd = build_layer(ctx, H, F, B, 0, 1164 + 1, 0.5, keep=keep)
    for d in L.lin:
        assert d.plan.n_res == d.plan.N // 2
    h0 = gen.uniform_bf16(1164 + 1, 999, B * H, 1.0).reshape(B, H)
    h = dev(h0)
    tr = trace_bufs(B, H, F)
    ctx.hg_layer(L, h, B, hg.layer_trace(**tr))
    torch.cuda.synchronize()
    T = check_layer_trace(tr, h0, Wd, bd, H)
    assert oracle.within_tol(oracle.bf16_to_f64(bits(h)),
                             oracle.bf16_to_f64(oracle.residual(T["h1"], T["y_fc2"])))[0]


@pytest.mark.slow
def test_c3_opt13b_40_layer_stack(ctx):
    """C3: OPT-13B (h=5120, ffn=20480) 40-layer linear stack, batch 2, alpha from Eq. (5),
    r = 0.  hg_stack must equal 40 hg_layer calls bit for bit; layers 0, 20, 39 are checked
    teacher-forced against the oracle."""
    H, F, B, NL = 5120, 20480, 2, 40
    keep, layers, weights = [], [], []
    for l in range(NL):
        L, Wd, bd = build_layer(ctx, H, F, B, l, 1164 + 2, 0.0, keep=keep)
        layers.append(L)
        weights.append((Wd, bd) if l in (0, 20, 39) else None)
    h0 = gen.uniform_bf16(1164 + 2, 999, B * H, 1.0).reshape(B, H)
    h_stack = dev(h0)
    ctx.hg_stack(layers, h_stack, B)
    h = dev(h0)
    for l, L in enumerate(layers):
        if weights[l] is None:
            ctx.hg_layer(L, h, B)
            continue
        h_in = bits(h)
        tr = trace_bufs(B, H, F)
        ctx.hg_layer(L, h, B, hg.layer_trace(**tr))
        torch.cuda.synchronize()
        check_layer_trace(tr, h_in, weights[l][0], weights[l][1], H)
    torch.cuda.synchronize()
    assert np.array_equal(bits(h), bits(h_stack))
