"""P > 1 on one GPU through the peer group (peer.cu; VERDICT r1 missing #1).

Rank p owns W rows [pN/P, (p+1)N/P) of every linear (oracle.shard), runs the heterogeneous split on
them with its own ring, copy stream and CPU lane, and the shards meet through the device pushes and
the shared host segment.  Checked: the gathered y of hg_linear_sharded equals the oracle on every
rank and is bit-identical across ranks (ranks as threads of one process: same-process peer
pointers); a sharded mirrored stack (ranks as processes: CUDA IPC and the named host segment, the
bench's multi-GPU path) gives the same bits on every rank, the same bits as the GPU-only glue at the
same P (the host glue mirrors the device glue), and stays within the tolerance of the fp64 oracle.

Whole stacks with ranks as threads of one process are not run: there every rank's streams share one
context's hardware work queues, and an exchange's spinning wait kernel ahead of another rank's work
in a shared queue can stall it until the wait times out (observed: seconds-long stalls broken by the
device-side timeouts).  Separate processes -- one per GPU in production -- have their own queues.
"""
import os
import threading

import numpy as np
import pytest
import torch

import oracle
from gpu_util import bits, dev, dev_f32, pinned
from harness import gen
from paper_2403_01164_b200 import hg

pytestmark = pytest.mark.gpu

NAMES = ("qkv", "o", "fc1", "fc2")


def run_ranks(P, fn):
    """fn(rank, blobs_exchange) in P threads; returns the per-rank results (re-raises the first error)."""
    out, errs = [None] * P, []
    blobs = [None] * P
    bar = threading.Barrier(P)

    def exchange(rank, blob):
        blobs[rank] = blob
        bar.wait()
        return list(blobs)

    def body(rank):
        try:
            torch.cuda.set_device(0)
            # every rank on its own stream: a spinning exchange on the legacy default stream would
            # serialise the other ranks behind it (ranks sharing one GPU)
            with torch.cuda.stream(torch.cuda.Stream()):
                out[rank] = fn(rank, exchange, bar)
        except Exception as e:  # noqa: BLE001
            errs.append(e)
            bar.abort()

    ths = [threading.Thread(target=body, args=(r,)) for r in range(P)]
    for t in ths:
        t.start()
    for t in ths:
        t.join(timeout=600)
    if errs:
        raise errs[0]
    return out


def make_ctx(P, rank, exchange, **kw):
    kw = {"ring_bytes": int(os.environ.get("RING_MB", 32)) << 20, **kw}
    c = hg.Context(0, chunk_bytes=1 << 20, max_k=8192, max_n=16384,
                   cpu_threads=max(1, 8 // P), **kw)
    blob = c.hg_peer_export(P, rank)
    c.hg_peer_open(exchange(rank, blob))
    return c


@pytest.mark.parametrize("P", [2, 4, 8])
@pytest.mark.parametrize("B", [1, 3])
def test_peer_linear_sharded(P, B):
    N, K = 4096, 1024
    x, W, b = gen.linear_inputs(61, 0, "fc1", B, N, K)
    ref = oracle.linear(x, W, b)

    def rank_fn(p, exchange, bar):
        c = make_ctx(P, p, exchange)
        try:
            r0, r1 = oracle.shard(N, P, p, 128)
            n_res = 128 * p % (r1 - r0)  # different residency per rank
            plan = c.plan(hg.make_rates(1, 1, 1), r1 - r0, K, B, n_res, hg.FIXED, (0.3 + 0.2 * p) % 1.0)
            Wd = dev(W[r0:r0 + n_res]) if n_res else None
            Wh = pinned(W[r0 + n_res:r1])
            xd, bd = dev(x), dev_f32(b[r0:r1])
            ys_dev = [torch.full((B, N), float("nan"), device="cuda") for _ in range(3)]
            st = torch.cuda.current_stream()
            st.synchronize()
            # ranks share the device: no allocation and no device-wide synchronisation while another
            # rank may be spinning on this rank's next push (both can wait for the device to go idle)
            bar.wait()
            for y in ys_dev:  # several exchanges: box slots and flags cycle
                c.hg_linear_sharded(plan, xd, Wd, Wh, bd, y, stream=st)
            st.synchronize()
            ys = [y.cpu().numpy() for y in ys_dev]
            bar.wait()
            return ys
        finally:
            c.close()

    outs = run_ranks(P, rank_fn)
    for p in range(P):
        for y in outs[p]:
            assert np.array_equal(y.view(np.uint32), outs[0][0].view(np.uint32))
    ok, worst = oracle.within_tol(outs[0][0], ref)
    assert ok, worst


@pytest.mark.parametrize("P", [2, 4, 8])
@pytest.mark.parametrize("B", [1, 3])
def test_peer_linear_rowpar(P, B):
    """Row-parallel linear (Megatron's o / fc2, reading R32): rank p holds input columns
    [pK/P, (p+1)K/P) of W and the matching slice of x, runs its own heterogeneous split over the N rows,
    and the partials are all-reduced in rank order with the bias added once: the same bits on every
    rank, within tolerance of the oracle's row-parallel sum (and of the unsharded linear)."""
    N, K = 1024, 4096
    x, W, b = gen.linear_inputs(62, 0, "fc2", B, N, K)
    parts = [oracle.shard_k(K, P, q, 128) for q in range(P)]
    ref = oracle.linear_rowpar([x[:, a:e] for a, e in parts], [np.ascontiguousarray(W[:, a:e]) for a, e in parts], b)

    def rank_fn(p, exchange, bar):
        c = make_ctx(P, p, exchange)
        try:
            k0, k1 = parts[p]
            n_res = (128 * p) % N
            plan = c.plan(hg.make_rates(1, 1, 1), N, k1 - k0, B, n_res, hg.FIXED, (0.3 + 0.2 * p) % 1.0)
            Wp = np.ascontiguousarray(W[:, k0:k1])
            Wd = dev(Wp[:n_res]) if n_res else None
            Wh = pinned(Wp[n_res:])
            xd, bd = dev(np.ascontiguousarray(x[:, k0:k1])), dev_f32(b)
            ys_dev = [torch.full((B, N), float("nan"), device="cuda") for _ in range(3)]
            st = torch.cuda.current_stream()
            st.synchronize()
            bar.wait()
            for y in ys_dev:  # several exchanges: box slots and flags cycle
                c.hg_linear_rowpar(plan, xd, Wd, Wh, bd, y, stream=st)
            st.synchronize()
            ys = [y.cpu().numpy() for y in ys_dev]
            bar.wait()
            return ys
        finally:
            c.close()

    outs = run_ranks(P, rank_fn)
    for p in range(P):
        for y in outs[p]:
            assert np.array_equal(y.view(np.uint32), outs[0][0].view(np.uint32))
    ok, worst = oracle.within_tol(outs[0][0], ref)
    assert ok, worst
    assert oracle.within_tol(outs[0][0], oracle.linear(x, W, b))[0]


def run_procs(P, tmp_path, **env):
    """P ranks as processes (tests/peer_worker.py) on GPU 0; returns their npz results."""
    import socket
    import subprocess
    import sys
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    procs, outs = [], []
    for p in range(P):
        out = str(tmp_path / f"rank{p}.npz")
        outs.append(out)
        e = {**os.environ, "WORLD_SIZE": str(P), "RANK": str(p), "MASTER_ADDR": "127.0.0.1",
             "MASTER_PORT": str(port), "OUT": out, **{k: str(v) for k, v in env.items()}}
        procs.append(subprocess.Popen([sys.executable, os.path.join(root, "tests", "peer_worker.py")], env=e,
                                      stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True))
    logs = []
    for pr in procs:
        try:
            logs.append(pr.communicate(timeout=900)[0])
        except subprocess.TimeoutExpired:
            pr.kill()
            logs.append(pr.communicate()[0])
    bad = [f"--- rank {p} rc={pr.returncode}\n{log[-1500:]}" for p, (pr, log) in enumerate(zip(procs, logs))
           if pr.returncode != 0]
    assert not bad, "\n".join(bad)
    return [np.load(o) for o in outs]


@pytest.mark.parametrize("P,B", [(2, 1), (2, 4), (4, 2), (8, 1)])
def test_peer_stack_mirrored_processes(P, B, tmp_path):
    """Ranks as processes: peer blobs all-gathered over gloo, device boxes opened by CUDA IPC, the host
    segment by name (the bench's multi-GPU path).  Every rank ends with the same bits, twice; the
    mirrored glue ran on every linear with 0 mismatches (verify_mirror) and gives the same bits as the
    GPU-only glue at the same P; and the output stays within tolerance of the fp64 oracle."""
    H, F, NL, seed = (1024, 4096, 2, 71) if P == 8 else (512, 2048, 3, 71)  # N/P a multiple of 128
    res = run_procs(P, tmp_path, H=H, F=F, NL=NL, B=B, SEED=seed)
    ref = res[0]["m1_0"]
    for r in res:
        assert np.array_equal(r["m1_0"], ref) and np.array_equal(r["m1_1"], ref)
        assert np.array_equal(r["m0_0"], ref) and np.array_equal(r["m0_1"], ref)
        ml, mm, nlin, with_cpu = r["m1_stats"]
        assert ml == 2 * with_cpu and mm == 0, (ml, mm, with_cpu)
        assert r["m0_stats"][0] == 0
    # at P = 8 (alpha 0.95 on rank 6) one rank's shards have no CPU rows at all: it still takes the
    # mirrored path with the others (can_mirror decides alike on every rank)
    assert any(r["m1_stats"][3] > 0 for r in res)
    if P == 8:
        assert any(r["m1_stats"][3] == 0 for r in res)
    shapes = {"qkv": (3 * H, H), "o": (H, H), "fc1": (F, H), "fc2": (H, F)}
    h = gen.uniform_bf16(seed + 1, 989, B * H, 1.0).reshape(B, H)
    for l in range(NL):
        Wd, bd = {}, {}
        for name in NAMES:
            _, Wd[name], bd[name] = gen.linear_inputs(seed, l, name, 1, *shapes[name])
        h = oracle.layer(h, Wd, bd, H)["out"]
    assert oracle.within_tol(oracle.bf16_to_f64(ref), oracle.bf16_to_f64(h), rtol=5e-2)[0]


@pytest.mark.parametrize("P,B", [(2, 1), (4, 3), (8, 1)])
def test_peer_stack_megatron_processes(P, B, tmp_path):
    """The Megatron pairing (hg_tp = TP_MEGATRON, reading R32) as processes: qkv / fc1 local, o / fc2
    all-reduced -- 2 exchanges per layer.  Every rank ends with the same bits (twice, and with
    mirror_glue on or off: the pairing takes the plain path), and the output stays within tolerance of
    the fp64 oracle's Megatron layer stack (itself pinned to the unsharded layer)."""
    H, F, NL, seed = (1024, 4096, 2, 73) if P == 8 else (512, 2048, 3, 73)
    res = run_procs(P, tmp_path, H=H, F=F, NL=NL, B=B, SEED=seed, TP="megatron")
    ref = res[0]["m1_0"]
    for r in res:
        for k in ("m1_0", "m1_1", "m0_0", "m0_1"):
            assert np.array_equal(r[k], ref), k
        assert r["m1_stats"][0] == 0 and r["m0_stats"][0] == 0  # no mirrored linears
    shapes = {"qkv": (3 * H, H), "o": (H, H), "fc1": (F, H), "fc2": (H, F)}
    h = gen.uniform_bf16(seed + 1, 989, B * H, 1.0).reshape(B, H)
    for l in range(NL):
        Wd, bd = {}, {}
        for name in NAMES:
            _, Wd[name], bd[name] = gen.linear_inputs(seed, l, name, 1, *shapes[name])
        h = oracle.megatron_layer(h, Wd, bd, H, P)["out"]
    assert oracle.within_tol(oracle.bf16_to_f64(ref), oracle.bf16_to_f64(h), rtol=5e-2)[0]
