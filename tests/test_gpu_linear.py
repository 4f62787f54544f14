"""GPU parity for the device GEMV and the heterogeneous linear
through the C ABI, against the fp64 oracle on identical generated inputs.

Tolerance (BJ:5, R13): elementwise |y - y_ref| <= 1e-2 * max(1, |y_ref|).
Bit-exact: small-integer inputs (fp32 sums exact), identity / one-hot / zero W,
and GPU split invariance (every partition with n_cpu = 0 gives identical bits).
"""
import numpy as np
import pytest
import torch

import oracle
from harness import gen
from paper_2403_01164_b200 import hg
from gpu_util import bits, dev, dev_f32, pinned, split_weight

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    c = hg.Context(0, chunk_bytes=1 << 20, ring_bytes=64 << 20, max_k=65536, max_n=65536)
    yield c
    c.close()


@pytest.fixture(scope="module")
def ctx_g1():
    c = hg.Context(0, granule=1, chunk_bytes=4096, ring_bytes=1 << 20, max_k=1024, max_n=4096)
    yield c
    c.close()


def _gemv(ctx, x, W, b, B):
    N, K = W.shape
    y = torch.full((B, N), float("nan"), device="cuda")
    ctx.hg_gemv(dev(x), B, N, K, dev(W), None if b is None else dev_f32(b), y)
    torch.cuda.synchronize()
    return y.cpu().numpy()


@pytest.mark.parametrize("B", range(1, 9))
@pytest.mark.parametrize("N,K", [(1, 8), (33, 768), (300, 4104), (129, 7168), (70, 28672)])
def test_gemv_parity(ctx, B, N, K):
    x, W, b = gen.linear_inputs(7, 0, "fc1", B, N, K)
    y = _gemv(ctx, x, W, b, B)
    ok, worst = oracle.within_tol(y, oracle.linear(x, W, b))
    assert ok, worst


@pytest.fixture(scope="module")
def ctx_simt():
    """Same kernels with the tcgen05 path disabled (B >= 5 on the SIMT kernel)."""
    c = hg.Context(0, chunk_bytes=1 << 20, ring_bytes=64 << 20, max_k=65536, max_n=65536,
                   gemv_tc_min_batch=0)
    yield c
    c.close()


@pytest.mark.parametrize("B", range(5, 9))
@pytest.mark.parametrize("N,K", [(1, 8), (128, 64), (300, 4104), (129, 7168), (1000, 28672)])
def test_gemv_simt_path_for_large_batch(ctx_simt, B, N, K):
    x, W, b = gen.linear_inputs(17, 0, "fc2", B, N, K)
    y = _gemv(ctx_simt, x, W, b, B)
    ok, worst = oracle.within_tol(y, oracle.linear(x, W, b))
    assert ok, worst


@pytest.mark.parametrize("B", [5, 8])
@pytest.mark.parametrize("N,K", [(128, 64), (256, 1024), (4096, 7168), (3, 200)])
def test_gemv_tcgen05_small_integer_exact(ctx, B, N, K):
    """tcgen05 path: fp32 accumulation of small integers is exact -> bit-equal to the oracle."""
    x, W, b = gen.linear_inputs(18, 0, "fc1", B, N, K, integer=2 if K > 256 else 8)
    y = _gemv(ctx, x, W, b, B)
    assert np.array_equal(y.astype(np.float64), oracle.linear(x, W, b))


@pytest.mark.parametrize("B", [1, 3, 8])
@pytest.mark.parametrize("K", [256, 8192])
def test_gemv_small_integer_exact(ctx, B, K):
    m = 16 if K <= 256 else 2  # keep every partial sum < 2^24
    x, W, b = gen.linear_inputs(8, 0, "o", B, 77, K, integer=m)
    y = _gemv(ctx, x, W, b, B)
    assert np.array_equal(y.astype(np.float64), oracle.linear(x, W, b))


def _linear(ctx, x, W, b, B, n_res, alpha, stream=None):
    N, K = W.shape
    W_dev, W_host = split_weight(W, n_res)
    y = torch.full((B, N), float("nan"), device="cuda")
    ctx.hg_linear(dev(x), B, N, K, W_dev, n_res, W_host, alpha, None if b is None else dev_f32(b), y,
                  stream=stream)
    torch.cuda.synchronize()
    return y.cpu().numpy()


def test_c1_opt125m_fc1_alpha_half(ctx):
    """BJ:7: OPT-125M fc1 768->3072, batch 1, alpha = 0.5 -> partition (0, 1536, 1536)."""
    x, W, b = gen.linear_inputs(1164, 0, "fc1", 1, 3072, 768)
    p = ctx.plan(hg.make_rates(1, 1, 1), 3072, 768, 1, 0, hg.FIXED, 0.5)
    assert (p.n_res, p.n_str, p.n_cpu) == (0, 1536, 1536)
    y = _linear(ctx, x, W, b, 1, 0, 0.5)
    ok, worst = oracle.within_tol(y, oracle.linear(x, W, b))
    assert ok, worst


@pytest.mark.parametrize("B", [1, 2, 5, 8])
@pytest.mark.parametrize("n_res,alpha", [(0, 0.0), (0, 1.0), (0, 0.37), (1024, 0.5), (2048, 0.0),
                                         (2048, 1.0), (3072, 0.5)])
def test_linear_partitions(ctx, B, n_res, alpha):
    x, W, b = gen.linear_inputs(2, 0, "fc2", B, 3072, 1000)
    y = _linear(ctx, x, W, b, B, n_res, alpha)
    ok, worst = oracle.within_tol(y, oracle.linear(x, W, b))
    assert ok, worst


def test_linear_no_bias_many_chunks(ctx):
    # 1 MiB chunks at K=4096 -> 128-row chunks; 20 chunks ride a 64-slot ring
    x, W, _ = gen.linear_inputs(3, 0, "qkv", 2, 3840, 4096, bias=False)
    y = _linear(ctx, x, W, None, 2, 256, 0.8)
    assert oracle.within_tol(y, oracle.linear(x, W))[0]


def test_split_invariance_gpu_bit_exact(ctx):
    """All partitions with n_cpu = 0 run the same kernel and reduction order: identical bits."""
    x, W, b = gen.linear_inputs(4, 0, "fc1", 3, 2048, 7168)
    ref = _linear(ctx, x, W, b, 3, 2048, 0.0)  # fully resident
    for n_res in (0, 128, 1024, 1920):
        y = _linear(ctx, x, W, b, 3, n_res, 1.0)  # the rest streamed
        assert np.array_equal(y, ref), n_res
    assert np.array_equal(_gemv(ctx, x, W, b, 3), ref)


@pytest.mark.parametrize("B", [5, 8])
def test_split_invariance_tcgen05_bit_exact(ctx, B):
    """tcgen05 batches: the persistent per-linear launch (resident block + up to 16 chunks, each
    its own tensor map) and the plain resident GEMV give identical bits for every partition with
    n_cpu = 0 (rows never depend on the tile they share)."""
    x, W, b = gen.linear_inputs(14, 0, "fc1", B, 2048, 7168)
    ref = _linear(ctx, x, W, b, B, 2048, 0.0)  # fully resident
    assert oracle.within_tol(ref, oracle.linear(x, W, b))[0]
    for n_res in (0, 128, 1024, 1920):
        y = _linear(ctx, x, W, b, B, n_res, 1.0)  # the rest streamed: 128-row chunks
        assert np.array_equal(y, ref), n_res
    assert np.array_equal(_gemv(ctx, x, W, b, B), ref)


@pytest.mark.parametrize("B", [2, 4, 8])
@pytest.mark.parametrize("K", [64, 200, 1032])
def test_tcgen05_persistent_few_stages(ctx, B, K):
    """Persistent tcgen05 launch with fewer k-stages per CTA than ring stages (K = 64: one stage)
    and a K that is not a multiple of the 64-wide tile (zero-filled tail): the x tiles deferred
    behind griddepcontrol.wait are still issued; resident + streamed rows match the oracle."""
    x, W, b = gen.linear_inputs(19, 0, "o", B, 1536, K)
    for n_res, alpha in ((0, 1.0), (128, 1.0), (512, 0.5)):
        y = _linear(ctx, x, W, b, B, n_res, alpha)
        ok, worst = oracle.within_tol(y, oracle.linear(x, W, b))
        assert ok, (n_res, alpha, worst)


def test_cpu_rows_equal_host_lane(ctx):
    x, W, b = gen.linear_inputs(5, 0, "fc1", 2, 1024, 512)
    y = _linear(ctx, x, W, b, 2, 0, 0.0)  # everything on the CPU lane
    yh = np.zeros((2, 1024), np.float32)
    with hg.Context(-1, cpu_threads=3) as hc:
        hc.hg_host_gemv(x, 2, 1024, 512, W, b, yh)
    assert np.array_equal(y, yh)


@pytest.mark.parametrize("n_res,alpha", [(0, 0.5), (512, 0.3), (0, 0.0), (0, 1.0)])
def test_linear_small_integer_exact(ctx, n_res, alpha):
    x, W, b = gen.linear_inputs(6, 0, "o", 4, 1024, 256, integer=16)
    y = _linear(ctx, x, W, b, 4, n_res, alpha)
    assert np.array_equal(y.astype(np.float64), oracle.linear(x, W, b))


def test_identity_onehot_zero_weights(ctx):
    K = 1024
    x, _, b = gen.linear_inputs(9, 0, "o", 3, K, K)
    eye = np.zeros((K, K), np.uint16)
    eye[np.arange(K), np.arange(K)] = 0x3F80
    y = _linear(ctx, x, eye, None, 3, 256, 0.5)
    assert np.array_equal(y.astype(np.float64), oracle.bf16_to_f64(x))
    perm = np.random.default_rng(0).integers(0, K, size=K)
    oh = np.zeros((K, K), np.uint16)
    oh[np.arange(K), perm] = 0x3F80
    y = _linear(ctx, x, oh, None, 3, 0, 0.25)
    assert np.array_equal(y.astype(np.float64), oracle.bf16_to_f64(x)[:, perm])
    y = _linear(ctx, x, np.zeros((K, K), np.uint16), b, 3, 384, 0.5)
    assert np.array_equal(y, np.broadcast_to(b, y.shape))


def test_brute_force_all_partitions_tiny(ctx_g1):
    """G = 1, N = 12, K = 16: every (n_res, alpha-grid) partition matches the oracle."""
    N, K = 12, 16
    x, W, b = gen.linear_inputs(10, 0, "fc1", 2, N, K, integer=8)
    ref = oracle.linear(x, W, b)
    for n_res in range(N + 1):
        m = N - n_res
        for g in range(m + 1):
            alpha = g / m if m else 0.0
            y = _linear(ctx_g1, x, W, b, 2, n_res, alpha)
            assert np.array_equal(y.astype(np.float64), ref), (n_res, g)


def test_nondefault_stream_and_reuse(ctx):
    s = torch.cuda.Stream()
    x, W, b = gen.linear_inputs(11, 0, "fc1", 1, 2048, 1024)
    ref = oracle.linear(x, W, b)
    for _ in range(3):
        y = _linear(ctx, x, W, b, 1, 512, 0.4, stream=s)
        assert oracle.within_tol(y, ref)[0]


def test_errors(ctx):
    x, W, b = gen.linear_inputs(12, 0, "o", 1, 256, 64)
    xd, Wd, bd = dev(x), dev(W), dev_f32(b)
    y = torch.zeros(1, 256, device="cuda")
    pageable = torch.from_numpy(W.view(np.int16).copy())
    with pytest.raises(hg.HgError) as e:
        ctx.hg_linear(xd, 1, 256, 64, None, 0, pageable, 0.5, bd, y)
    assert e.value.status == hg.HG_ENOTPINNED
    with pytest.raises(hg.HgError) as e:
        ctx.hg_linear(xd, 1, 256, 64, None, 0, pinned(W), 1.5, bd, y)
    assert e.value.status == hg.HG_EINVAL
    with pytest.raises(hg.HgError) as e:
        ctx.hg_linear(xd.data_ptr() + 2, 1, 256, 64, None, 0, pinned(W), 0.5, bd, y)
    assert e.value.status == hg.HG_EALIGN
    with pytest.raises(hg.HgError) as e:
        ctx.hg_linear(torch.from_numpy(x.view(np.int16)), 1, 256, 64, None, 0, pinned(W), 0.5, bd, y)
    assert e.value.status == hg.HG_ENOTDEVICE
    with pytest.raises(hg.HgError) as e:
        ctx.hg_linear(xd, 1, 200, 64, None, 0, pinned(W[:200]), 0.5, bd, y)  # N % G
    assert e.value.status == hg.HG_EINVAL
    # the context is still usable after argument errors
    ok, _ = oracle.within_tol(_linear(ctx, x, W, b, 1, 128, 0.5), oracle.linear(x, W, b))
    assert ok


def test_stats_lane_breakdown():
    with hg.Context(0, chunk_bytes=2 << 20, ring_bytes=64 << 20, collect_stats=1) as c:
        x, W, b = gen.linear_inputs(13, 0, "fc1", 1, 4096, 4096)
        _linear(c, x, W, b, 1, 1024, 0.5)
        s = c.hg_stats()
        assert s.n_linears == 1 and s.bytes_res == 1024 * 4096 * 2
        assert s.bytes_str == 1536 * 4096 * 2 and s.bytes_cpu == 1536 * 4096 * 2
        assert s.n_chunks == 6 and s.link_busy_s > 0 and s.gpu_busy_s > 0 and s.cpu_busy_s > 0
        assert s.wall_s > 0 and s.gpu_launches >= 2


@pytest.mark.parametrize("B", [1, 3, 6])
def test_tags_ring_smaller_than_linear(B):
    """Device-tag pipeline with 2 ring slots and 32 chunks per linear: the copy stream refills a
    slot only after every CTA of the (cooperative) GEMV drained it; results match the oracle."""
    with hg.Context(0, chunk_bytes=64 << 10, ring_bytes=128 << 10, max_k=256, max_n=8192) as c:
        assert c.config.handshake == 1
        x, W, b = gen.linear_inputs(31, 0, "fc1", B, 4096, 256)
        for n_res, alpha in ((0, 1.0), (512, 1.0), (0, 0.6)):
            y = _linear(c, x, W, b, B, n_res, alpha)
            ok, worst = oracle.within_tol(y, oracle.linear(x, W, b))
            assert ok, (n_res, alpha, worst)


@pytest.mark.parametrize("B,K", [(1, 7168), (2, 7168), (1, 12288), (1, 28672)])
def test_tags_ring_smaller_than_linear_row_kernels(B, K):
    """The warp-per-row (B <= 2, K <= 8192) and part-row (B = 1, K <= 32768) kernels with the ring
    smaller than the linear (3 slots, >= 9 chunks refilled inside one launch): a warp / CTA counts a
    chunk out only after it landed (the per-slot count must not mix occupants), with rows of this
    launch's warps in only some of the chunks; results match the oracle and equal a roomy ring's bits."""
    N = 1280
    row = 2 * K
    chunk = 128 * row  # 128 rows per chunk: most warps have no row in most chunks
    x, W, b = gen.linear_inputs(35, 0, "fc1", B, N, K)
    ys = []
    for ring in (3 * chunk, 64 * chunk):
        with hg.Context(0, chunk_bytes=chunk, ring_bytes=ring, max_k=K, max_n=N, timeout_s=20.0) as c:
            for n_res, alpha in ((0, 1.0), (128, 0.8)):
                y = _linear(c, x, W, b, B, n_res, alpha)
                ok, worst = oracle.within_tol(y, oracle.linear(x, W, b))
                assert ok, (ring, n_res, alpha, worst)
                ys.append(y)
    assert np.array_equal(ys[0], ys[2]) and np.array_equal(ys[1], ys[3])  # same kernel, same bits


@pytest.mark.parametrize("B", [1, 2, 4, 8])
def test_event_path_equals_tag_path(ctx, B):
    """handshake=0 (host events, one GEMV per chunk) and the default device-tag pipeline compute
    identical bits: same kernel arithmetic, only the synchronisation differs."""
    x, W, b = gen.linear_inputs(32, 0, "fc2", B, 2048, 7168)
    with hg.Context(0, chunk_bytes=1 << 20, ring_bytes=16 << 20, max_k=8192, max_n=4096, handshake=0) as ce:
        y_ev = _linear(ce, x, W, b, B, 256, 0.7)
    y_tag = _linear(ctx, x, W, b, B, 256, 0.7)
    assert np.array_equal(y_ev, y_tag)
    assert oracle.within_tol(y_tag, oracle.linear(x, W, b))[0]


def test_schedule_divergence_drops_prefetch():
    """Chunks prefetched for a call that never comes are released (tags written) and the
    next, different linear restarts the schedule without stalling the copy stream."""
    with hg.Context(0, chunk_bytes=64 << 10, ring_bytes=512 << 10, max_k=1024, max_n=8192) as c:
        x1, W1, b1 = gen.linear_inputs(33, 0, "fc1", 1, 2048, 1024)
        x2, W2, b2 = gen.linear_inputs(34, 0, "fc2", 1, 1024, 1024)
        for it in range(3):
            y1 = _linear(c, x1, W1, b1, 1, 0, 0.9)
            y2 = _linear(c, x2, W2, b2, 1, 128, 0.5)
            assert oracle.within_tol(y1, oracle.linear(x1, W1, b1))[0], it
            assert oracle.within_tol(y2, oracle.linear(x2, W2, b2))[0], it


@pytest.mark.parametrize("B", [1, 3])
def test_zero_copy_stream_mode_equals_ring(ctx, B):
    """stream_mode 1: the GEMV reads the streamed rows straight from pinned host memory over the
    link (TMA bulk copies from mapped memory) -- same kernel arithmetic, identical bits."""
    x, W, b = gen.linear_inputs(35, 0, "fc1", B, 3072, 7168)
    with hg.Context(0, chunk_bytes=1 << 20, ring_bytes=16 << 20, max_k=8192, max_n=4096, stream_mode=1) as cz:
        y_zc = _linear(cz, x, W, b, B, 512, 0.6)
    y_ring = _linear(ctx, x, W, b, B, 512, 0.6)
    assert np.array_equal(y_zc, y_ring)
    assert oracle.within_tol(y_zc, oracle.linear(x, W, b))[0]


def _pageable(bits):
    """uint16 bits -> a plain (pageable) host int16 tensor."""
    return torch.from_numpy(np.ascontiguousarray(bits, np.uint16).view(np.int16).copy())


@pytest.mark.parametrize("strategy", [hg.HYBRID, hg.NAIVE, hg.PINNED_BLOCKING])
@pytest.mark.parametrize("B,stage_mb", [(1, 512), (2, 2), (8, 2)])
def test_pageable_weights_pin_lane(B, stage_mb, strategy):
    """hg_config.pageable: streamed chunks of a pageable weight go through the pin lane (pinned staging
    ring, tags in mapped memory) -- results bit-identical to the pinned-weight path; a 2-slot staging
    ring (1 MiB chunks) forces slot reuse."""
    N, K = 3072, 1024
    x, W, b = gen.linear_inputs(36, 0, "fc1", B, N, K)
    with hg.Context(0, chunk_bytes=1 << 20, ring_bytes=16 << 20, max_k=4096, max_n=4096, pageable=1,
                    staging_bytes=stage_mb << 20, strategy=strategy) as cp, \
            hg.Context(0, chunk_bytes=1 << 20, ring_bytes=16 << 20, max_k=4096, max_n=4096) as cq:
        for n_res, alpha in ((0, 0.7), (512, 1.0)):
            Wd = dev(W[:n_res]) if n_res else None
            y_pg = torch.full((B, N), float("nan"), device="cuda")
            # the caller keeps every buffer alive until the stream has passed the call (hg.h): the
            # pageable rows are copied asynchronously by the pin lane / naive transfer thread
            W_pg = _pageable(W[n_res:])
            cp.hg_linear(dev(x), B, N, K, Wd, n_res, W_pg, alpha, dev_f32(b), y_pg)
            y_pin = torch.full((B, N), float("nan"), device="cuda")
            W_pin = pinned(W[n_res:])
            cq.hg_linear(dev(x), B, N, K, Wd, n_res, W_pin, alpha, dev_f32(b), y_pin)
            torch.cuda.synchronize()
            del W_pg, W_pin
            assert np.array_equal(y_pg.cpu().numpy(), y_pin.cpu().numpy()), (n_res, alpha)
            assert oracle.within_tol(y_pg.cpu().numpy(), oracle.linear(x, W, b))[0]
        s = cp.hg_stats()
        if strategy == hg.NAIVE:  # Fig. 5a: no pin lane; the driver stages the pageable rows
            assert s.bytes_pinned == 0
        else:
            assert s.bytes_pinned > 0 and s.pin_busy_s > 0


def test_strategy_config_validated():
    with pytest.raises(hg.HgError) as e:
        hg.Context(0, max_k=1024, max_n=1024, strategy=3)
    assert e.value.status == hg.HG_EINVAL


def test_pageable_measure_reports_pin_rate():
    N, K = 4096, 2048
    _, W, _ = gen.linear_inputs(37, 0, "fc1", 1, N, K)
    with hg.Context(0, chunk_bytes=4 << 20, ring_bytes=64 << 20, max_k=4096, max_n=8192, pageable=1,
                    staging_bytes=64 << 20) as c:
        r = c.hg_measure(_pageable(W), N, K, 1)
        assert np.isfinite(r.v_pin) and r.v_pin > 0 and r.v_link > 0 and r.v_cpu > 0


@pytest.mark.parametrize("B,K", [(1, 28672), (3, 12288), (1, 7168)])
def test_back_to_back_gemv_pdl_ordering(ctx, B, K):
    """Back-to-back GEMV launches (programmatic dependent launch) where a torch kernel rewrites x
    right before each one: every launch must see its own x (griddepcontrol.wait before the x copy)
    and, for P > 1, the per-row-group part counters must reset between launches.  Each result is
    bit-identical to the same GEMV launched alone."""
    N = 640
    xs = [gen.linear_inputs(40 + i, 0, "fc2", B, N, K)[0] for i in range(4)]
    _, W, b = gen.linear_inputs(40, 0, "fc2", B, N, K)
    Wd, bd = dev(W), dev_f32(b)
    alone = []
    for x in xs:
        y = torch.empty((B, N), device="cuda")
        ctx.hg_gemv(dev(x), B, N, K, Wd, bd, y)
        torch.cuda.synchronize()
        alone.append(y.cpu().numpy())
        assert oracle.within_tol(alone[-1], oracle.linear(x, W, b))[0]
    src = [dev(x) for x in xs]
    xbuf = torch.empty_like(src[0])
    ys = [torch.empty((B, N), device="cuda") for _ in range(24)]
    torch.cuda.synchronize()
    torch.cuda._sleep(2_000_000)  # queue everything behind a spin so launches run back to back
    for i, y in enumerate(ys):
        torch.bitwise_or(src[i % 4], 0, out=xbuf)  # a kernel (not a memcpy) writing x right before the GEMV
        ctx.hg_gemv(xbuf, B, N, K, Wd, bd, y, stream=torch.cuda.current_stream())
    torch.cuda.synchronize()
    for i, y in enumerate(ys):
        assert np.array_equal(y.cpu().numpy().view(np.uint32), alone[i % 4].view(np.uint32)), i
