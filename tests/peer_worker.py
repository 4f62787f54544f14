"""One rank of a multi-process peer-group run (tests/test_gpu_peer.py): ranks are separate processes
(on one GPU here: one CUDA context each, time-sliced), exchanging their 512-byte peer blobs through a
gloo process group -- the way bench.py's ranks do -- so the device boxes are opened with CUDA IPC and
the host segment by name.  Writes the step outputs to OUT (npz)."""
import os
import sys

os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import oracle  # noqa: E402
from gpu_util import bits, dev, dev_f32, pinned  # noqa: E402
from harness import gen  # noqa: E402
from paper_2403_01164_b200 import hg  # noqa: E402

NAMES = ("qkv", "o", "fc1", "fc2")


def shard_layer(c, H, F, B, layer, P, p, alpha, keep, seed, tp="column"):
    """This rank's descriptors: column shards (rows [pN/P, (p+1)N/P) of every linear), or the Megatron
    pairing (qkv: its heads' q/k/v rows, fc1: its rows, o / fc2: its input columns, full bias)."""
    shapes = {"qkv": (3 * H, H), "o": (H, H), "fc1": (F, H), "fc2": (H, F)}
    descs = []
    for name in NAMES:
        N, K = shapes[name]
        _, W, bfull = gen.linear_inputs(seed, layer, name, 1, N, K)
        if tp == "megatron" and name in ("o", "fc2"):
            k0, k1 = oracle.shard_k(K, P, p, 128)
            Wp, bp = np.ascontiguousarray(W[:, k0:k1]), bfull
        elif tp == "megatron" and name == "qkv":
            rows = oracle.megatron_qkv_rows(H, P, p, 128)
            Wp, bp = np.ascontiguousarray(W[rows]), bfull[rows]
        else:
            r0, r1 = oracle.shard(N, P, p, 128)
            Wp, bp = W[r0:r1], bfull[r0:r1]
        plan = c.plan(hg.make_rates(1, 1, 1), Wp.shape[0], Wp.shape[1], B, 0, hg.FIXED, alpha)
        Wh = pinned(Wp)
        bias, bias_h = dev_f32(bp), torch.from_numpy(np.ascontiguousarray(bp, np.float32))
        keep += [Wh, bias, bias_h]
        descs.append(hg.linear_desc(plan, None, Wh, bias, bias_h))
    return hg.opt_layer(H, F, descs, tp=hg.TP_MEGATRON if tp == "megatron" else hg.TP_COLUMN)


def main():
    P, p = int(os.environ["WORLD_SIZE"]), int(os.environ["RANK"])
    H, F, NL, B = (int(os.environ[k]) for k in ("H", "F", "NL", "B"))
    seed, out = int(os.environ.get("SEED", 71)), os.environ["OUT"]
    tp = os.environ.get("TP", "column")
    dist.init_process_group("gloo")
    torch.cuda.set_device(0)
    st = torch.cuda.Stream()
    results = {}
    with torch.cuda.stream(st):
        for mirror in (1, 0):
            c = hg.Context(0, chunk_bytes=1 << 20, ring_bytes=32 << 20, max_k=8192, max_n=16384,
                           cpu_threads=max(1, 8 // P), mirror_glue=mirror, verify_mirror=mirror, wrap_prefetch=1)
            blobs = [None] * P
            dist.all_gather_object(blobs, c.hg_peer_export(P, p))
            c.hg_peer_open(blobs)
            keep = []
            layers = [shard_layer(c, H, F, B, l, P, p, (0.35 + 0.1 * p) % 1.0, keep, seed, tp) for l in range(NL)]
            h0 = gen.uniform_bf16(seed + 1, 989, B * H, 1.0).reshape(B, H)
            hs = [dev(h0) for _ in range(2)]
            st.synchronize()
            dist.barrier()
            for h in hs:
                c.hg_stack(layers, h, B, stream=st)
            st.synchronize()
            s = c.hg_stats()
            results[f"m{mirror}_0"], results[f"m{mirror}_1"] = bits(hs[0]), bits(hs[1])
            with_cpu = sum(1 for L in layers for d in L.lin if d.plan.n_cpu > 0)
            results[f"m{mirror}_stats"] = np.array([s.mirror_linears, s.mirror_mismatch, s.n_linears, with_cpu],
                                                   np.int64)
            dist.barrier()
            c.close()
    np.savez(out, **results)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
