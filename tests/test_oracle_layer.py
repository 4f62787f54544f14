"""Pins for the oracle's layer pieces (reading R22).

Library routines serve as the independent check: torch float64 layer_norm,
scaled_dot_product_attention (for the position-0 reading), and a bit-trick
float32->bf16 rounding for the rounding helper.
"""
import numpy as np
import torch

import oracle
from harness import gen


def test_round_to_bf16_ties_and_library_agreement():
    # exact ties: 1 + 2^-8 lies halfway between 1 and 1 + 2^-7 -> even (1.0)
    vals = np.array([1 + 2**-8, 1 + 3 * 2**-8, -(1 + 2**-8), 0.0, -0.0, 2.0**-130, 3.0e38, 1e39])
    bits = oracle.round_to_bf16(vals)
    back = oracle.bf16_to_f64(bits)
    assert back[0] == 1.0 and back[1] == 1 + 2**-6 and back[2] == -1.0
    assert back[3] == 0.0 and np.signbit(back[4])
    assert back[5] == 2.0**-130                 # subnormal bf16 is exact here
    assert np.isinf(back[7])
    # values already exact in float32: must match the float32 bit-trick RNE
    rng = np.random.default_rng(0)
    f32 = (rng.standard_normal(4000) * 10.0 ** rng.uniform(-6, 6, 4000)).astype(np.float32)
    assert np.array_equal(oracle.round_to_bf16(f32.astype(np.float64)), gen.f32_to_bf16_bits(f32))
    # and torch's own fp64 -> bf16 conversion
    t = torch.from_numpy(f32.astype(np.float64)).to(torch.bfloat16).view(torch.int16).numpy()
    assert np.array_equal(oracle.round_to_bf16(f32.astype(np.float64)), t.view(np.uint16))


def test_layernorm_matches_torch_float64():
    h = gen.uniform_bf16(1, 2, 3 * 512, 2.0).reshape(3, 512)
    a = oracle.layernorm(h)
    ref = torch.nn.functional.layer_norm(torch.from_numpy(oracle.bf16_to_f64(h)), (512,), eps=oracle.LN_EPS)
    assert np.array_equal(a, oracle.round_to_bf16(ref.numpy()))
    # normalised statistics
    av = oracle.bf16_to_f64(a)
    assert np.all(np.abs(av.mean(axis=1)) < 1e-2) and np.all(np.abs(av.var(axis=1) - 1) < 2e-2)


def test_layernorm_constant_row_is_zero():
    h = np.full((1, 64), 0x4040, dtype=np.uint16)  # 3.0
    assert np.all(oracle.bf16_to_f64(oracle.layernorm(h)) == 0.0)


def test_position0_attention_is_v():
    """Reading R22: with a single key, softmax = 1 and the attention output is V."""
    B, H, heads = 2, 64, 4
    rng = np.random.default_rng(1)
    y_qkv = rng.standard_normal((B, 3 * H))
    q, k, v = (torch.from_numpy(y_qkv[:, i * H:(i + 1) * H]).reshape(B, heads, 1, H // heads)
               for i in range(3))
    ctx = torch.nn.functional.scaled_dot_product_attention(q, k, v).reshape(B, H).numpy()
    assert np.array_equal(oracle.attention_pos0(y_qkv, H), oracle.round_to_bf16(ctx))


def test_layer_matches_torch_composition():
    B, H, F = 2, 64, 256
    seed = 9
    Wd, bd = {}, {}
    for name, (n, k) in {"qkv": (3 * H, H), "o": (H, H), "fc1": (F, H), "fc2": (H, F)}.items():
        _, Wd[name], bd[name] = gen.linear_inputs(seed, 0, name, 1, n, k)
    h = gen.uniform_bf16(seed, 99, B * H, 1.0).reshape(B, H)
    o = oracle.layer(h, Wd, bd, H)

    T = lambda bits: torch.from_numpy(oracle.bf16_to_f64(bits))
    rb = lambda t: torch.from_numpy(oracle.bf16_to_f64(oracle.round_to_bf16(t.numpy())))
    lin = lambda a, n: torch.nn.functional.linear(a, T(Wd[n]), torch.from_numpy(bd[n].astype(np.float64)))
    x = T(h)
    a = rb(torch.nn.functional.layer_norm(x, (H,), eps=oracle.LN_EPS))
    v = rb(lin(a, "qkv")[:, 2 * H:])
    h1 = rb(x + lin(v, "o"))
    u = rb(torch.relu(lin(rb(torch.nn.functional.layer_norm(h1, (H,), eps=oracle.LN_EPS)), "fc1")))
    out = rb(h1 + lin(u, "fc2"))
    assert np.allclose(oracle.bf16_to_f64(o["out"]), out.numpy(), rtol=0, atol=0)
