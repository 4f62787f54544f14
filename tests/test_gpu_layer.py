"""GPU parity of hg_layer / hg_stack.

Teacher-forced per linear: each linear's fp32 output is compared with the
oracle fed the GPU's own bf16 input to that linear (from the layer trace); each
glue step likewise.  bf16 glue outputs may differ from the fp64 oracle by the
rounding of an fp32 intermediate, so they use the same elementwise tolerance.
"""
import ctypes

import numpy as np
import pytest
import torch

import oracle
from harness import gen
from paper_2403_01164_b200 import hg
from gpu_util import bits, dev, dev_f32, pinned

pytestmark = pytest.mark.gpu

NAMES = ("qkv", "o", "fc1", "fc2")


def make_layer(ctx, H, F, B, layer=0, seed=21, r=0.0, alpha=0.5, keep=None):
    shapes = {"qkv": (3 * H, H), "o": (H, H), "fc1": (F, H), "fc2": (H, F)}
    descs, Wd, bd = [], {}, {}
    keep = keep if keep is not None else []
    for name in NAMES:
        N, K = shapes[name]
        _, W, b = gen.linear_inputs(seed, layer, name, 1, N, K)
        Wd[name], bd[name] = W, b
        n_res = oracle.resident_rows(r, N, ctx.config.granule)
        p = ctx.plan(hg.make_rates(1, 1, 1), N, K, B, n_res, hg.FIXED, alpha)
        W_dev = dev(W[:n_res]) if n_res else None
        W_host = pinned(W[n_res:]) if n_res < N else None
        bias = dev_f32(b)
        keep += [W_dev, W_host, bias]
        descs.append(hg.linear_desc(p, W_dev, W_host, bias))
    return hg.opt_layer(H, F, descs), Wd, bd


@pytest.fixture(scope="module")
def ctx():
    c = hg.Context(0, chunk_bytes=1 << 20, ring_bytes=64 << 20, max_k=32768, max_n=65536)
    yield c
    c.close()


@pytest.mark.parametrize("B,r,alpha", [(1, 0.0, 0.5), (3, 0.5, 0.3), (8, 0.25, 1.0), (2, 0.0, 0.0)])
def test_layer_teacher_forced(ctx, B, r, alpha):
    H, F = 512, 2048
    keep = []
    L, Wd, bd = make_layer(ctx, H, F, B, r=r, alpha=alpha, keep=keep)
    h0 = gen.uniform_bf16(5, 999, B * H, 1.0).reshape(B, H)
    h = dev(h0)
    tr = {k: torch.zeros(B, n, dtype=torch.int16, device="cuda") for k, n in
          (("a", H), ("v", H), ("h1", H), ("a2", H), ("u", F))}
    tr.update({k: torch.zeros(B, n, device="cuda") for k, n in
               (("y_qkv", 3 * H), ("y_o", H), ("y_fc1", F), ("y_fc2", H))})
    ctx.hg_layer(L, h, B, hg.layer_trace(**tr))
    torch.cuda.synchronize()
    T = {k: (bits(v) if v.dtype == torch.int16 else v.cpu().numpy()) for k, v in tr.items()}
    out = bits(h)
    # linears, teacher-forced on the GPU's own inputs
    for name, xin, yk in (("qkv", "a", "y_qkv"), ("o", "v", "y_o"), ("fc1", "a2", "y_fc1"), ("fc2", "u", "y_fc2")):
        ok, worst = oracle.within_tol(T[yk], oracle.linear(T[xin], Wd[name], bd[name]))
        assert ok, (name, worst)
    # glue, teacher-forced
    chk = lambda got, ref: oracle.within_tol(oracle.bf16_to_f64(got), oracle.bf16_to_f64(ref))[0]
    assert chk(T["a"], oracle.layernorm(h0))
    assert chk(T["v"], oracle.attention_pos0(T["y_qkv"], H))
    assert chk(T["h1"], oracle.residual(h0, T["y_o"]))
    assert chk(T["a2"], oracle.layernorm(T["h1"]))
    assert chk(T["u"], oracle.relu_bf16(T["y_fc1"]))
    assert chk(out, oracle.residual(T["h1"], T["y_fc2"]))
    # end to end (secondary, looser report): the full fp64 oracle layer
    full = oracle.layer(h0, Wd, bd, H)
    assert oracle.within_tol(oracle.bf16_to_f64(out), oracle.bf16_to_f64(full["out"]), rtol=5e-2)[0]


def test_stack_two_layers_matches_two_layer_calls(ctx):
    """hg_stack (cross-linear prefetch) gives the same bits as layer-by-layer calls."""
    H, F, B = 256, 1024, 2
    keep = []
    layers = [make_layer(ctx, H, F, B, layer=l, alpha=0.6, keep=keep)[0] for l in range(3)]
    h0 = gen.uniform_bf16(6, 998, B * H, 1.0).reshape(B, H)
    h_a, h_b = dev(h0), dev(h0)
    ctx.hg_stack(layers, h_a, B)
    for L in layers:
        ctx.hg_layer(L, h_b, B)
    torch.cuda.synchronize()
    assert np.array_equal(bits(h_a), bits(h_b))


def test_stack_wrap_prefetch_repeatable():
    H, F, B = 256, 1024, 1
    with hg.Context(0, chunk_bytes=1 << 20, ring_bytes=32 << 20, max_k=4096, max_n=8192,
                    wrap_prefetch=1) as c:
        keep = []
        layers = [make_layer(c, H, F, B, layer=l, alpha=0.7, keep=keep)[0] for l in range(2)]
        h0 = gen.uniform_bf16(7, 997, B * H, 1.0).reshape(B, H)
        outs = []
        for _ in range(3):
            h = dev(h0)
            c.hg_stack(layers, h, B)
            torch.cuda.synchronize()
            outs.append(bits(h))
        assert np.array_equal(outs[0], outs[1]) and np.array_equal(outs[0], outs[2])


def test_stack_wrap_then_other_calls():
    """wrap_prefetch streams the next token's first chunks; a different call in between drops them
    (their slots are released) and later stacks still match layer-by-layer results."""
    H, F, B = 256, 1024, 1
    with hg.Context(0, chunk_bytes=256 << 10, ring_bytes=2 << 20, max_k=4096, max_n=8192,
                    wrap_prefetch=1) as c:
        keep = []
        layers = [make_layer(c, H, F, B, layer=l, alpha=0.8, keep=keep)[0] for l in range(2)]
        h0 = gen.uniform_bf16(8, 996, B * H, 1.0).reshape(B, H)
        ref = dev(h0)
        for L in layers:
            c.hg_layer(L, ref, B)
        for _ in range(2):
            h = dev(h0)
            c.hg_stack(layers, h, B)
            torch.cuda.synchronize()
            assert np.array_equal(bits(h), bits(ref))
            h2 = dev(h0)
            c.hg_layer(layers[1], h2, B)  # diverges from the wrapped schedule
            torch.cuda.synchronize()


def make_layer_mirror(ctx, H, F, B, layer=0, seed=21, r=0.0, alpha=0.5, keep=None, ln=False):
    """make_layer with host copies of the biases (and LN parameters) for the mirrored glue."""
    shapes = {"qkv": (3 * H, H), "o": (H, H), "fc1": (F, H), "fc2": (H, F)}
    descs = []
    for name in NAMES:
        N, K = shapes[name]
        _, W, b = gen.linear_inputs(seed, layer, name, 1, N, K)
        n_res = oracle.resident_rows(r, N, ctx.config.granule)
        p = ctx.plan(hg.make_rates(1, 1, 1), N, K, B, n_res, hg.FIXED, alpha)
        W_dev = dev(W[:n_res]) if n_res else None
        W_host = pinned(W[n_res:]) if n_res < N else None
        bias, bias_h = dev_f32(b), torch.from_numpy(np.ascontiguousarray(b, np.float32))
        keep += [W_dev, W_host, bias, bias_h]
        descs.append(hg.linear_desc(p, W_dev, W_host, bias, bias_h))
    lnp = {}
    if ln:
        for k, sd in (("g1", 1), ("b1", 2), ("g2", 3), ("b2", 4)):
            v = gen.bf16_bits_to_f32(gen.uniform_bf16(seed + sd, 900 + layer, H, 0.5)) + (1.0 if k[0] == "g" else 0.0)
            lnp[k] = (dev_f32(v), torch.from_numpy(np.ascontiguousarray(v, np.float32)))
            keep += list(lnp[k])
        return hg.opt_layer(H, F, descs, lnp["g1"][0], lnp["b1"][0], lnp["g2"][0], lnp["b2"][0],
                            ln_host=(lnp["g1"][1], lnp["b1"][1], lnp["g2"][1], lnp["b2"][1]))
    return hg.opt_layer(H, F, descs)


@pytest.mark.parametrize("B,r,alpha,ln", [(1, 0.0, 0.5, False), (3, 0.25, 0.3, True), (2, 0.0, 0.0, True),
                                          (1, 0.5, 1.0, False), (8, 0.0, 0.6, True)])
def test_mirrored_glue_bit_exact(B, r, alpha, ln):
    """The CPU lane's mirrored glue (reading R24) reproduces every GPU glue output bit for bit
    (verify_mirror counts mismatching activation elements), and the stack output equals the
    GPU-only glue path's."""
    H, F = 512, 2048
    outs = {}
    for mirror in (1, 0):
        with hg.Context(0, chunk_bytes=1 << 20, ring_bytes=64 << 20, max_k=4096, max_n=8192,
                        mirror_glue=mirror, verify_mirror=mirror) as c:
            keep = []
            layers = [make_layer_mirror(c, H, F, B, layer=l, r=r, alpha=alpha, keep=keep, ln=ln) for l in range(3)]
            h0 = gen.uniform_bf16(9, 995, B * H, 1.0).reshape(B, H)
            h = dev(h0)
            c.hg_stack(layers, h, B)
            torch.cuda.synchronize()
            st = c.hg_stats()
            if mirror:
                expect = 12 if alpha < 1.0 else 0  # no CPU rows at alpha = 1: nothing to mirror
                assert st.mirror_linears == expect and st.mirror_mismatch == 0, (st.mirror_linears, st.mirror_mismatch)
            else:
                assert st.mirror_linears == 0
            outs[mirror] = bits(h)
    assert np.array_equal(outs[0], outs[1])


def test_mirror_falls_back_without_host_bias():
    """Device biases without host copies on a plan with CPU rows: the GPU-only glue is used."""
    H, F, B = 256, 1024, 1
    with hg.Context(0, chunk_bytes=1 << 20, ring_bytes=32 << 20, max_k=4096, max_n=8192) as c:
        keep = []
        L = make_layer(c, H, F, B, alpha=0.5, keep=keep)[0]
        h = dev(gen.uniform_bf16(10, 994, B * H, 1.0).reshape(B, H))
        c.hg_layer(L, h, B)
        torch.cuda.synchronize()
        assert c.hg_stats().mirror_linears == 0


def test_mirrored_glue_mixed_residency():
    """Scheduler-style placement: some linears fully GPU-resident (no CPU rows), others split.  The
    host catches up on the glue of the resident ones lazily; activations stay bit-exact and the
    output equals the GPU-only glue path's."""
    H, F, B = 512, 2048, 2
    shapes = {"qkv": (3 * H, H), "o": (H, H), "fc1": (F, H), "fc2": (H, F)}
    resident = [{"qkv", "o"}, {"qkv", "o", "fc1"}, set(), {"fc2"}, {"qkv", "o", "fc1", "fc2"}, {"o"}]
    outs = {}
    for mirror in (1, 0):
        with hg.Context(0, chunk_bytes=1 << 20, ring_bytes=64 << 20, max_k=4096, max_n=8192,
                        mirror_glue=mirror, verify_mirror=mirror) as c:
            keep, layers = [], []
            for l, res in enumerate(resident):
                descs = []
                for name in NAMES:
                    N, K = shapes[name]
                    _, W, b = gen.linear_inputs(41, l, name, 1, N, K)
                    n_res = N if name in res else 0
                    p = c.plan(hg.make_rates(1, 1, 1), N, K, B, n_res, hg.FIXED, 0.4)
                    W_dev = dev(W[:n_res]) if n_res else None
                    W_host = pinned(W[n_res:]) if n_res < N else None
                    bias, bias_h = dev_f32(b), torch.from_numpy(np.ascontiguousarray(b, np.float32))
                    keep += [W_dev, W_host, bias, bias_h]
                    descs.append(hg.linear_desc(p, W_dev, W_host, bias, bias_h))
                layers.append(hg.opt_layer(H, F, descs))
            h0 = gen.uniform_bf16(11, 993, B * H, 1.0).reshape(B, H)
            for rep in range(2):
                h = dev(h0)
                c.hg_stack(layers, h, B)
                torch.cuda.synchronize()
            st = c.hg_stats()
            if mirror:
                cpu_linears = sum(1 for res in resident for name in NAMES if name not in res)
                assert st.mirror_linears == 2 * cpu_linears and st.mirror_mismatch == 0
            outs[mirror] = bits(h)
    assert np.array_equal(outs[0], outs[1])


@pytest.mark.parametrize("strategy", [hg.HYBRID, hg.NAIVE, hg.PINNED_BLOCKING])
def test_stack_pageable_weights_equal_pinned(strategy):
    """A stack whose host weights are pageable gives the same bits as pinned under every strategy of
    Fig. 5 (hybrid: pin lane, Sec. 4.3; naive: copies from un-pinned rows; pinned-blocking: pin first
    on the CPU lane's threads)."""
    H, F, B = 256, 1024, 2
    outs = []
    for pageable in (1, 0):
        with hg.Context(0, chunk_bytes=256 << 10, ring_bytes=4 << 20, max_k=4096, max_n=8192, pageable=pageable,
                        staging_bytes=1 << 20, wrap_prefetch=1, strategy=strategy) as c:
            keep, layers = [], []
            for l in range(2):
                L = make_layer_mirror(c, H, F, B, layer=l, alpha=0.6, keep=keep)
                if pageable:  # swap every pinned host weight for a pageable copy
                    for i in range(4):
                        d = L.lin[i]
                        if d.W_host:
                            n = d.plan.N - d.plan.n_res
                            t = torch.empty((n, d.plan.K), dtype=torch.int16)
                            ctypes_src = torch.from_numpy(np.ctypeslib.as_array(
                                (ctypes.c_int16 * (n * d.plan.K)).from_address(d.W_host)).reshape(n, d.plan.K).copy())
                            t.copy_(ctypes_src)
                            keep.append(t)
                            L.lin[i].W_host = t.data_ptr()
                layers.append(L)
            h0 = gen.uniform_bf16(13, 991, B * H, 1.0).reshape(B, H)
            for _ in range(2):
                h = dev(h0)
                c.hg_stack(layers, h, B)
                torch.cuda.synchronize()
            outs.append(bits(h))
            if pageable:
                assert (c.hg_stats().bytes_pinned > 0) == (strategy != hg.NAIVE)
                assert c.hg_stats().mirror_linears > 0
    assert np.array_equal(outs[0], outs[1])
