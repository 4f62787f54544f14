"""Parity of the exact path bench.py times (SURVEY 8(a) a1-a7 at the headline, BJ:10).

The OPT-30B 48-layer stack is built by bench.py's own setup functions: the same context
configuration (mirrored glue with host bias copies, wrap_prefetch, 32 MiB chunks, 4 GiB ring,
CPU-lane threads), the same seeded weights and biases, rates from hg_measure and alpha from
Eq. (5), at batch 1 and 8.  Checks:
  * the mirrored glue (reading R24) ran on every linear and the CPU lane's activations equal the
    GPU's bit for bit over all 192 linears (verify_mirror: 0 mismatches);
  * the traced step (hg_stack_trace) gives the same output bits as the untraced step, as the
    verify_mirror context and as the GPU-only glue (mirror_glue = 0);
  * layers 0, 24 and 47 are teacher-forced against the fp64 oracle on every output element of
    their four linears (BJ:5 tolerance) and their glue against the oracle's LN / V / residual /
    ReLU.
"""
import numpy as np
import pytest
import torch

import bench
import oracle
from paper_2403_01164_b200 import hg

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

TRACED = (0, 24, 47)


@pytest.fixture(scope="module")
def weights():
    args = bench.parse_args([])
    w = bench.make_weights(args, 0, 1)
    yield w
    del w
    torch.cuda.synchronize()
    torch._C._host_emptyCache()


def run_step(ctx, layers, h0_pinned, B, stream):
    h = h0_pinned.cuda()
    ctx.hg_stack(layers, h, B, stream=stream)
    torch.cuda.synchronize()
    return h.cpu().numpy().view(np.uint16).copy()


@pytest.mark.parametrize("B", [1, 8])
def test_bench_path_opt30b_stack(weights, B):
    args = bench.parse_args(["--batch", str(B)])
    st = bench.prepare(args, weights=weights)
    ctx, s = st["ctx"], st["stream"]
    try:
        cfg = ctx.config
        assert (cfg.chunk_bytes, cfg.ring_bytes, cfg.wrap_prefetch, cfg.mirror_glue, cfg.verify_mirror) == \
            (32 << 20, 4096 << 20, 1, 1, 0)
        layers, plans, all_plans = bench.build_layers(st, args, hg.EXACT, 0.0, {}, {})
        assert len(all_plans) == 4 * 48 and all(p.n_cpu > 0 and p.n_str > 0 for p in all_plans), \
            [(p.n_str, p.n_cpu) for p in all_plans[:4]]
        # warm-up as in the bench, then the traced step and an untraced step on the same context
        for _ in range(2):
            run_step(ctx, layers, st["h_host"], B, s)
        tr = bench.trace_layers(st, layers, list(TRACED))
        assert tr["mirror_linears"] == 4 * 48
        out_plain = run_step(ctx, layers, st["h_host"], B, s)
        assert np.array_equal(tr["h_out"], out_plain)

        # the CPU lane's mirrored activations equal the GPU's on every linear
        cv, _ = bench.make_context(args, 0, 1, 0, verify_mirror=1)
        try:
            run_step(cv, layers, st["h_host"], B, s)
            cv.hg_reset_stats()
            out_v = run_step(cv, layers, st["h_host"], B, s)
            sv = cv.hg_stats()
            assert sv.mirror_linears == 4 * 48 and sv.mirror_mismatch == 0, (sv.mirror_linears, sv.mirror_mismatch)
        finally:
            cv.close()
        assert np.array_equal(out_v, out_plain)
        # GPU-only glue gives the same bits
        cg, _ = bench.make_context(args, 0, 1, 0, mirror_glue=0)
        try:
            out_g = run_step(cg, layers, st["h_host"], B, s)
            assert cg.hg_stats().mirror_linears == 0
        finally:
            cg.close()
        assert np.array_equal(out_g, out_plain)

        # teacher-forced fp64 oracle on layers 0, 24, 47: every output of every linear
        H = bench.H
        for l in TRACED:
            T = tr["layers"][l]
            for name, xin, yk in bench.LIN_IO:
                W = st["host"][l][name].numpy().view(np.uint16)
                ref = oracle.linear(T[xin], W, st["biases_h"][l][name].numpy(), nthreads=16)
                ok, worst = oracle.within_tol(T[yk], ref)
                assert ok, (B, l, name, worst)
            chk = lambda got, ref: oracle.within_tol(oracle.bf16_to_f64(got), oracle.bf16_to_f64(ref))
            assert chk(T["v"], oracle.attention_pos0(T["y_qkv"], H))[0], l
            assert chk(T["a2"], oracle.layernorm(T["h1"]))[0], l
            assert chk(T["u"], oracle.relu_bf16(T["y_fc1"]))[0], l
            if l == 0:
                assert chk(T["a"], oracle.layernorm(tr["h_in"]))[0]
                assert chk(T["h1"], oracle.residual(tr["h_in"], T["y_o"]))[0]
        # the bench's parity leg on this trace agrees
        _, parity = bench.cpu_baseline_and_parity(st, {**tr, "layers": {l: tr["layers"][l] for l in (0, 47)}})
        assert parity["ok"], parity
    finally:
        ctx.close()
