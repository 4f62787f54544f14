#!/usr/bin/env python
"""bench.py -- ms/token of the offloaded OPT-30B decode linear stack (BJ:2, BJ:10).

One step = one decode token through all 48 OPT-30B layers (h=7168, ffn=28672):
every QKV / O / fc1 / fc2 linear runs HeteGen's heterogeneous split (resident
r=0, so every weight lives in pinned host memory; alpha from Eq. (5) with rates
measured by hg_measure in this process; streamed rows copied in chunks over the
host link into a device ring and GEMV'd on the GPU; the rest computed by the
host thread pool), with the glue (LN, attention at position 0, ReLU, residual)
on the GPU.  59,190,018,048 weight bytes per token per job.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference] [--batch B]

N > 1: launched under torchrun; rank p owns W rows [pN/P,(p+1)N/P) of every
linear (column-sharded TP), outputs all-gathered with NCCL after each linear.
--impl reference: the fp64 oracle (oracle/) on the host cores, on a bounded
sample of the same workload (one layer's four linears), scaled to ms/token.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
# one hardware work queue per stream (see tests/conftest.py): the peer exchange's wait kernel spins,
# and an unrelated copy queued behind it in a shared queue would wait for it
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

# OPT decoder dimensions (hidden, ffn, layers) and BASELINE.json config index (seed offset)
MODELS = {"opt-6.7b": (4096, 16384, 32, 1), "opt-13b": (5120, 20480, 40, 2), "opt-30b": (7168, 28672, 48, 3),
          "opt-66b": (9216, 36864, 64, 3)}
MODEL = "opt-30b"
H, F, LAYERS = 7168, 28672, 48
SHAPES = {"qkv": (3 * H, H), "o": (H, H), "fc1": (F, H), "fc2": (H, F)}
NAMES = ("qkv", "o", "fc1", "fc2")
STACK_BYTES = LAYERS * sum(2 * n * k for n, k in SHAPES.values())  # 59,190,018,048
METRIC = "ms/token offloaded OPT-30B decode linears; HBM & H2D GB/s vs roofline"
SEED = 1164 + 3  # base seed + config index (BJ:10 is configs[3])
# hg_strategy: Fig. 5c hybrid (default), 5a naive, 5b pinned-blocking (pageable weights only)
STRATEGIES = {"hybrid": 0, "naive": 1, "blocking": 2}


def set_model(name):
    """Select the OPT shape the stack is built from (default opt-30b: the headline, BJ:10)."""
    global MODEL, H, F, LAYERS, SHAPES, STACK_BYTES, METRIC, SEED
    H, F, LAYERS, cfg = MODELS[name]
    MODEL = name
    SHAPES = {"qkv": (3 * H, H), "o": (H, H), "fc1": (F, H), "fc2": (H, F)}
    STACK_BYTES = LAYERS * sum(2 * n * k for n, k in SHAPES.values())
    METRIC = "ms/token offloaded %s decode linears; HBM & H2D GB/s vs roofline" % name.upper().replace("OPT-", "OPT-")
    if name == "opt-30b":
        METRIC = "ms/token offloaded OPT-30B decode linears; HBM & H2D GB/s vs roofline"
    SEED = 1164 + cfg


def env_rank():
    """(rank, world, local device).  HG_BENCH_ONE_GPU=1 (functional check of the N > 1 flow on a one-GPU
    box: every rank on device 0, gloo for the process group; timings meaningless) maps every rank to
    device 0."""
    local = 0 if os.environ.get("HG_BENCH_ONE_GPU") == "1" else int(os.environ.get("LOCAL_RANK", "0"))
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), local


def coll_device():
    """Device of the small tensors the bench's collectives carry (gloo: CPU)."""
    return "cpu" if os.environ.get("HG_BENCH_ONE_GPU") == "1" else "cuda"


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


# ---------------------------------------------------------------- clocks sampler
class Clocks:
    def __init__(self, index=0):
        self.samples = []
        self.proc = None
        self.index = index

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index),
                 "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.samples.append([s.strip() for s in line.split(",")])

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(5)
        except Exception:
            self.proc.kill()
        sm = [float(s[0]) for s in self.samples if s and s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if len(s) > 1 and s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for s in self.samples:
            for nm, v in zip(names, s[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.samples)}


# ---------------------------------------------------------------- reference arm / cpu baseline
def host_info():
    """lscpu's model name, sockets and cores of the host the oracle runs on."""
    info = {"model": None, "sockets": None, "cores_per_socket": None, "threads_online": os.cpu_count()}
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for ln in out.splitlines():
            k, _, v = ln.partition(":")
            k, v = k.strip(), v.strip()
            if k == "Model name":
                info["model"] = v
            elif k == "Socket(s)":
                info["sockets"] = int(v)
            elif k == "Core(s) per socket":
                info["cores_per_socket"] = int(v)
    except Exception:  # noqa: BLE001
        pass
    return info


def oracle_layer_inputs(layer, batch):
    """Layer `layer`'s weights and biases (bf16 bits / fp32) from the seeded generator, and the step's
    input activation."""
    from harness import gen
    Wd, bd = {}, {}
    for name in NAMES:
        N, K = SHAPES[name]
        _, Wd[name], bd[name] = gen.linear_inputs(SEED, layer, name, 1, N, K)
    return Wd, bd


def oracle_layer_time(h_bits, Wd, bd, nthreads):
    """Seconds for one OPT layer through the fp64 oracle end to end (LN, QKV, V, O, residual, LN, fc1,
    ReLU, fc2, residual with the oracle's exact bf16 rounding points)."""
    import oracle
    t0 = time.perf_counter()
    out = oracle.layer(h_bits, Wd, bd, H, nthreads=nthreads)
    return time.perf_counter() - t0, out


def run_reference(args):
    """--impl reference: the oracle as it stands on the host cores.  A step is a bounded sample of the
    token: `--ref-layers` consecutive OPT layers end to end (each layer's output is the next one's
    input), ms/token = the median step time x LAYERS / ref_layers; ms_per_step is the step's own
    measured time."""
    rank, world, _ = env_rank()
    if rank != 0:
        return 0
    nthr = os.cpu_count() or 1
    L = max(1, min(args.ref_layers, LAYERS))
    weights = [oracle_layer_inputs(l, args.batch) for l in range(L)]
    h0 = initial_h(args.batch)
    ts = []
    for _ in range(args.warmup + args.steps):
        h, t = h0, 0.0
        for Wd, bd in weights:
            dt, out = oracle_layer_time(h, Wd, bd, nthr)
            h, t = out["out"], t + dt
        ts.append(t)
    step_s = statistics.median(ts[args.warmup:])
    ms_tok = step_s * LAYERS / L * 1e3
    line = {
        "impl": "reference", "metric": METRIC, "value": round(ms_tok, 1), "unit": "ms/token", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(step_s * 1e3, 1),
        "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "%s %d-layer decode linear stack (qkv,o,fc1,fc2 x%d), batch %d" % (
                       MODEL.upper(), LAYERS, LAYERS, args.batch), "model": MODEL,
                   "sample": "%d of %d layers end to end per step; value = step x %g" % (L, LAYERS, LAYERS / L),
                   "batch": args.batch, "hidden": H, "ffn": F, "layers": LAYERS},
        "cpu_baseline": {"value": round(ms_tok, 1), "unit": "ms/token", "cores": nthr, "kind": "oracle",
                         "sample": "%d OPT layer(s) end to end per step (LN, 4 linears, V, residuals, ReLU; %.3f GB "
                                   "of weights per layer) through the fp64 oracle (C loops for the linears, exact "
                                   "bf16 rounding in Python), all host threads; scaled x%g to a token"
                                   % (L, STACK_BYTES / LAYERS / 1e9, LAYERS / L),
                         "host": host_info()},
        "e2e": {"value": round(ms_tok, 1), "unit": "ms/token", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def gemv_roofline(ctx, plans, layers, B, torch, pk, iters=20, W_dev=None):
    """Average device time of the step's GEMV launches -- one persistent launch per linear over
    its resident rows and all its streamed chunks (hg_gemv_replay: same kernel, grid and
    per-chunk work split as in the step, arrival tags skipped) -- timed with CUDA events on the
    launching stream over `iters` back-to-back launches.  Each launch reads its chunks from the
    next ring slots (seq0 rotates through the 4 GiB ring), so the launches together read far
    more than L2 holds and every chunk comes from HBM; a GPU spin kernel holds the stream while
    the host enqueues them, so the device never waits for the host.  The per-launch time thus
    includes the launch gap, as in the step.  (The older single-launch-after-L2-flush figure is
    kept as `single_launch`: it is dominated by event/launch latency -- a 1-element torch kernel
    times 11-13 us that way, profiles/r01/gemv_latency.md.)

    Algorithmic bytes per launch = 2*K*(n_res + n_str) (the W rows the GPU lanes must read;
    x, bias and y are < 0.1%).  Returns None when the GEMV runs on the tcgen05 path.
    """
    hbm_peak = pk.get("hbm_gbs", 6650.0)
    s = torch.cuda.current_stream()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    tot_bytes, tot_time, tot_time1, detail = 0.0, 0.0, 0.0, {}
    for name, p in plans.items():
        n_gpu = p.n_res + p.n_str
        if n_gpu <= 0:
            continue
        x = torch.empty((B, p.K), dtype=torch.int16, device="cuda").random_(-3000, 3000)
        y = torch.empty((B, p.N), device="cuda")
        Wd = (W_dev or {}).get(name)
        step = max(1, p.n_chunks)
        seqs = [i * step for i in range(iters)]  # slot = seq mod nslots (128 slots in the bench's ring)
        try:
            for q in seqs[:3]:
                ctx.hg_gemv_replay(p, x, Wd, None, y, stream=s, seq0=q)
        except Exception as e:  # noqa: BLE001
            return {"unavailable": str(e)}
        torch.cuda.synchronize()
        # back to back, GPU held by a spin kernel while the host enqueues
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(4_000_000)
        e0.record(s)
        for q in seqs:
            ctx.hg_gemv_replay(p, x, Wd, None, y, stream=s, seq0=q)
        e1.record(s)
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) * 1e-3 / iters
        # single launch after an L2 flush (reported beside it)
        ts1 = []
        for i in range(5):
            flush.zero_()
            torch.cuda._sleep(200_000)
            f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            f0.record(s)
            ctx.hg_gemv_replay(p, x, Wd, None, y, stream=s, seq0=seqs[i])
            f1.record(s)
            torch.cuda.synchronize()
            ts1.append(f0.elapsed_time(f1) * 1e-3)
        t1 = statistics.mean(ts1)
        nbytes = 2 * p.K * n_gpu
        tot_bytes += nbytes * layers
        tot_time += t * layers
        tot_time1 += t1 * layers
        detail[name] = {"rows": n_gpu, "chunks": p.n_chunks, "K": p.K, "us": round(t * 1e6, 2),
                        "GBps": round(nbytes / t / 1e9, 1), "single_launch_us": round(t1 * 1e6, 2)}
    del flush
    if tot_time <= 0:
        return None
    gbps = tot_bytes / tot_time / 1e9
    traffic, traffic_detail = ncu_traffic() if B == 1 else (None, None)
    # which kernel each linear runs (the library's choice depends on (batch, K) only; R26)
    if B <= 3:
        kernel = ("gemv_row_kernel (persistent per-linear GEMV, warp per row, W straight into registers, "
                  "half-row double buffering, bf16 FMA, PDL) for K <= 8192; "
                  + ("gemv_prow_kernel (a CTA of P warps per row, parts in registers) for fc2 (K = 28672)" if B == 1
                     else "gemv_tc_stream_kernel (tcgen05) for fc2 (K = 28672)"))
    else:
        kernel = "gemv_tc_stream_kernel (tcgen05 M=128 N=16, TMA 2-D tiles; one persistent launch per linear)"
    return {"bound": "hbm", "kernel": kernel,
            "achieved": round(gbps, 1), "peak": hbm_peak, "unit": "GB/s", "frac": round(gbps / hbm_peak, 4),
            "traffic": traffic, "traffic_detail": traffic_detail,
            "peak_source": "MEASURED_PEAKS.json hbm_gbs (copy BW)" if "hbm_gbs" in pk else "fallback 6650 GB/s",
            "per_linear": detail,
            "isolated_ncu": None if not traffic_detail else {
                "GBps": traffic_detail["isolated_GBps"], "frac": round(traffic_detail["isolated_GBps"] / hbm_peak, 4),
                "note": "the four launches under ncu (serialised, caches flushed): sum of algorithmic bytes / sum of "
                        "gpu__time_duration"},
            "single_launch": {"GBps": round(tot_bytes / tot_time1 / 1e9, 1),
                              "frac": round(tot_bytes / tot_time1 / 1e9 / hbm_peak, 4),
                              "note": "one launch after a 256 MiB L2 flush, event to event"},
            "note": "bytes = 2*K*(n_res+n_str) per launch; CUDA events around %d back-to-back hg_gemv_replay "
                    "launches (the step's launch configuration, arrival tags skipped) whose chunks walk the "
                    "ring (inputs larger than L2); mean per launch" % iters}


def ncu_traffic():
    """DRAM traffic per launch of the dominant kernel from the committed `ncu --set full` capture
    of the same launch configuration (profiles/r02/ncu_gemv_replay_traffic.json): mean over the
    four linears of dram__bytes_read.sum + dram__bytes_write.sum, beside their algorithmic bytes."""
    try:
        d = json.load(open(os.path.join(ROOT, "profiles", "r02", "ncu_gemv_replay_traffic.json")))
    except Exception:
        return None, None
    per = d["per_launch"]
    traffic = statistics.mean((v["dram_read_MB"] + v["dram_write_MB"]) * 1e6 for v in per.values())
    alg = statistics.mean(v["algorithmic_MB"] * 1e6 for v in per.values())
    # the same launches in isolation (ncu serialises them and flushes caches between): no launch
    # overlap, every ramp and tail exposed -- reported beside the back-to-back figure
    iso = sum(v["algorithmic_MB"] * 1e6 for v in per.values()) / sum(v["duration_us"] * 1e-6 for v in per.values())
    return round(traffic), {"algorithmic_bytes_per_launch": round(alg), "ratio": round(traffic / alg, 4),
                            "isolated_GBps": round(iso / 1e9, 1), "source": d["source"]}


# ---------------------------------------------------------------- our arm
def pct(sorted_vals, q):
    """q-th percentile of sorted values, linear interpolation between closest ranks."""
    if not sorted_vals:
        return float("nan")
    x = (len(sorted_vals) - 1) * q / 100.0
    i = int(math.floor(x))
    j = min(i + 1, len(sorted_vals) - 1)
    return sorted_vals[i] + (sorted_vals[j] - sorted_vals[i]) * (x - i)


def placement(args, world, local):
    """Host placement of this rank: (NUMA node of its GPU or -1, its share of cores, index
    of its first core in the node's cpulist or -1).  Ranks whose GPUs hang off the same node split that
    node's cores; with one rank (or --numa off, or no sysfs) the pool is not pinned."""
    from paper_2403_01164_b200 import hg
    ncores = os.cpu_count() or 1
    if args.numa == "off":
        return -1, max(1, ncores // world), (local * max(1, ncores // world)) if world > 1 else -1
    try:
        nodes = [hg.hg_numa_node(d) for d in range(world)]
        node = nodes[local]
        cpus = hg.hg_numa_cpus(node) if node >= 0 else []
    except Exception:  # noqa: BLE001
        node, cpus, nodes = -1, [], []
    if node < 0 or not cpus:
        return -1, max(1, ncores // world), (local * max(1, ncores // world)) if world > 1 else -1
    same = [d for d in range(world) if nodes[d] == node]
    per = max(1, len(cpus) // len(same))
    return node, per, (same.index(local) * per) if world > 1 else -1


def pool_placement(args, world, local):
    """(NUMA node, cores per rank, first core the CPU-lane pool's workers are pinned from or -1, threads)."""
    node, per, first = placement(args, world, local)
    pin_threads = 4 if args.pageable else 0  # the pin lane's memcpy threads get their own cores
    # leave cores for the API thread (it enqueues the GPU lanes and joins the CPU rows) and the CUDA
    # driver's threads: with all 16 cores of the GPU box in the pool, a preempted worker stalls the
    # lane now and then (measured: 14 threads 283.6 / 285.8 ms/token, 16 threads 283.0 / 329.7 / 298.0,
    # the slow runs with the link at ~46 GB/s -- profiles/r01/threads.md)
    reserve = 2 if per >= 12 else (1 if per >= 4 else 0)
    pinned_one = world == 1 and first < 0 and args.numa != "off" and reserve == 2 and not args.pageable
    if pinned_one:
        # one rank: the pool's workers pinned to the last cores, core 0 (and the floating API thread's
        # share) left to the API thread, the driver and the clock sampler.  Pinned, 15 threads beat 14:
        # 280.6 vs 285.8 ms/token over seven alternating pairs, without 14's slow episodes (p90 up to
        # 304); unpinned, 16 threads were bimodal (profiles/r02/pin_ab.txt, profiles/r01/threads.md)
        reserve = 1
    threads = args.threads or max(1, per - pin_threads - reserve)
    if pinned_one:
        first = per - threads
    if os.environ.get("HG_BENCH_PIN"):  # development A/B (-1: no pinning)
        first = int(os.environ["HG_BENCH_PIN"])
    return node, per, first, threads


def make_context(args, rank, world, local, **extra):
    """The bench's hg context: one per rank, its CPU lane on this rank's share of the host cores (those
    of its GPU's NUMA node when known)."""
    from paper_2403_01164_b200 import hg
    node, per, first, threads = pool_placement(args, world, local)
    pin_threads = 4 if args.pageable else 0
    cfg = dict(cpu_threads=threads, cpu_first=first, numa_node=node if first >= 0 else -1,
               chunk_bytes=args.chunk_mb << 20, ring_bytes=args.ring_mb << 20,
               max_k=F, max_n=F, wrap_prefetch=1, collect_stats=0,
               pageable=int(args.pageable), pin_threads=max(1, pin_threads),
               strategy=STRATEGIES[args.strategy], staging_bytes=args.staging_mb << 20)
    cfg.update(extra)
    return hg.Context(local, **cfg), threads


def make_weights(args, rank, world):
    """This rank's row shard of every linear: W in host memory (pinned unless --pageable; bound to the
    GPU's NUMA node before first touch, hg_host_alloc), bias on the device and its host copy (the CPU
    lane adds its rows' bias in the mirrored glue)."""
    import torch
    from harness import gen
    from paper_2403_01164_b200 import hg
    local = env_rank()[2]
    node = placement(args, world, local)[0] if torch.cuda.is_available() else -1
    t_setup = time.perf_counter()
    host, biases, biases_h = [], [], []
    for l in range(args.layers):
        hl, bl, bh = {}, {}, {}
        for name in NAMES:
            N, K = SHAPES[name]
            r0, r1 = rank * N // world, (rank + 1) * N // world
            if args.pageable:
                Wt = torch.empty((r1 - r0, K), dtype=torch.int16)
            else:
                Wt = hg.HostBuffer((r1 - r0, K), torch.int16, node=node, lock=True).tensor
            gen.uniform_bf16(SEED, gen.tensor_id(l, name, "W"), (r1 - r0) * K, gen.w_scale(K),
                             offset=r0 * K, out=Wt.data_ptr())
            b = gen.bf16_bits_to_f32(gen.uniform_bf16(SEED, gen.tensor_id(l, name, "bias"), r1 - r0,
                                                      gen.BIAS_SCALE, offset=r0))
            hl[name] = Wt
            bh[name] = torch.from_numpy(b)
            bl[name] = bh[name].cuda()
        host.append(hl)
        biases.append(bl)
        biases_h.append(bh)
    return host, biases, biases_h, time.perf_counter() - t_setup


def initial_h(B):
    """The decode step's input activation h [B, H] (bf16 bits)."""
    from harness import gen
    return gen.uniform_bf16(SEED + 1, 999, B * H, 1.0).reshape(B, H)


def prepare(args, weights=None, **ctx_extra):
    """Process-wide setup: context, this rank's host weights, measured rates."""
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2403_01164_b200 import hg

    rank, world, local = env_rank()
    torch.cuda.set_device(local)
    if world > 1 and not dist.is_initialized():
        if os.environ.get("HG_BENCH_ONE_GPU") == "1":
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    ctx, threads = make_context(args, rank, world, local, **ctx_extra)
    if world > 1 and args.exchange == "peer":
        # a8 over peer memory (peer.cu): device boxes opened by CUDA IPC over NVLink, one host segment
        # shared by the ranks' CPU lanes (mirrored glue at any P)
        blobs = [None] * world
        dist.all_gather_object(blobs, ctx.hg_peer_export(world, rank))
        ctx.hg_peer_open(blobs)
    elif world > 1:
        uid = hg.hg_dist_unique_id() if rank == 0 else None
        obj = [uid]
        dist.broadcast_object_list(obj, src=0)
        ctx.hg_dist_init(world, rank, obj[0])
    B = args.batch
    host, biases, biases_h, t_setup = weights or make_weights(args, rank, world)

    # ---- a1: measured rates (Fig. 1's "parameter size divided by processing time") ----
    fc1 = host[0]["fc1"]
    rates = ctx.hg_measure(fc1, fc1.shape[0], H, B, under_load=True)

    h_host = torch.empty((B, H), dtype=torch.int16, pin_memory=True)
    h_host.numpy()[...] = initial_h(B).view(np.int16)
    return {"torch": torch, "dist": dist, "hg": hg, "rank": rank, "world": world, "local": local,
            "threads": threads, "ctx": ctx, "B": B, "host": host, "biases": biases, "biases_h": biases_h,
            "rates": rates, "t_setup": t_setup, "h_host": h_host, "h_dev": h_host.cuda(),
            "placement": pool_placement(args, world, local)[:3],
            "h_out": torch.empty_like(h_host, pin_memory=True), "stream": torch.cuda.Stream(), "v_kind": None}


def cpu_rate_per_kind(st):
    """The CPU lane's GEMV rate on layer 0's weight of each kind (bytes/s, hg_module_tcpu: median of
    3, measured like Fig. 1) -- T-bar_CPU per module for the scheduler's gain."""
    if st["v_kind"] is None:
        ctx, B = st["ctx"], st["B"]
        v = {}
        for name in NAMES:
            W = st["host"][0][name]
            n, K = W.shape
            v[name] = ctx.hg_module_tcpu(W, n, K, B, 0.0)[1]
        st["v_kind"] = v
    return st["v_kind"]


def resident_rows(r, n, G=128):
    """Rows of an n-row linear kept in HBM for a resident fraction r: G * floor(r * (n / G) + 1/2)
    (the library's hg_resident_rows)."""
    from paper_2403_01164_b200 import hg
    return hg.hg_resident_rows(r, n, G)


def build_layers(st, args, mode, af, n_res_map, W_dev_map):
    hg = st["hg"]
    ctx, world, B = st["ctx"], st["world"], st["B"]
    layers, plans_l0, all_plans = [], {}, []
    for l in range(args.layers):
        descs = []
        for name in NAMES:
            N, K = SHAPES[name]
            n_res = n_res_map.get((l, name), 0)
            p = ctx.plan(st["rates"], N // world, K, B, n_res, mode, af)
            if l == 0:
                plans_l0[name] = p
            all_plans.append(p)
            W_h = st["host"][l][name][n_res:] if n_res < N // world else None
            descs.append(hg.linear_desc(p, W_dev_map.get((l, name)), W_h, st["biases"][l][name],
                                        st["biases_h"][l][name]))
        layers.append(hg.opt_layer(H, F, descs))
    return layers, plans_l0, all_plans


def run_point(st, args, budget_gb=0.0):
    """One measured configuration: schedule (HBM budget), plan, alpha benchmark, timed steps."""
    torch, dist, hg = st["torch"], st["dist"], st["hg"]
    rank, world, local, B = st["rank"], st["world"], st["local"], st["B"]
    ctx, s, h_host, h_dev, h_out = st["ctx"], st["stream"], st["h_host"], st["h_dev"], st["h_out"]
    rates = st["rates"]
    rd = rates.as_dict()
    pk = peaks()
    if args.alpha is not None:
        mode, af = hg.FIXED, args.alpha
    else:  # pageable weights: Eq. (9), T_COM = max(T_PIN, T_TRANS); pinned: Eq. (5)
        mode, af = (hg.ASYNC if args.pageable else hg.EXACT), 0.0

    # ---- NEXT(3): heterogeneous module scheduler under an HBM budget (Sec. 4.5) ----
    n_res_map, W_dev_map, sched = {}, {}, None
    if budget_gb > 0:
        p0 = ctx.plan(rates, SHAPES["fc1"][0] // world, H, B, 0, mode, af)
        alpha0 = p0.alpha_eff
        v_kind = cpu_rate_per_kind(st)
        mods, keys = [], []
        for l in range(args.layers):
            for name in NAMES:
                N, K = SHAPES[name]
                n = N // world
                mods.append((n, K, (1.0 - alpha0) * 2 * n * K / v_kind[name]))  # T-bar_CPU at alpha
                keys.append((l, name))
        if args.scheduler == "rows":  # one resident fraction for every linear (reading R31)
            n_res_list, used = hg.hg_schedule_rows(mods, int(budget_gb * 1e9), 128)
        else:  # Sec. 4.5's module greedy
            n_res_list, used = hg.hg_schedule(mods, int(budget_gb * 1e9), 128, True)
        for key, nr in zip(keys, n_res_list):
            if nr > 0:
                n_res_map[key] = nr
                W_dev_map[key] = st["host"][key[0]][key[1]][:nr].cuda()
        torch.cuda.synchronize()
        sched = {"scheduler": args.scheduler, "budget_GB": budget_gb, "placed_GB": round(used / 1e9, 3),
                 "alpha_for_gain": alpha0,
                 "gain_s_per_GB": {k: round((1.0 - alpha0) / v_kind[k] * 1e9, 6) for k in NAMES},
                 "cpu_GBps_by_kind": {k: round(v_kind[k] / 1e9, 2) for k in NAMES},
                 "resident_modules": sum(1 for (n, _, _), nr in zip(mods, n_res_list) if nr == n),
                 "partial_modules": sum(1 for (n, _, _), nr in zip(mods, n_res_list) if 0 < nr < n)}
    if getattr(args, "resident", 0.0) > 0 and budget_gb <= 0:
        # C2 (BJ:8): a fixed fraction r of every linear's rows resident in HBM,
        # n_res = G * floor(r * (N / G) + 1/2)
        for l in range(args.layers):
            for name in NAMES:
                nr = resident_rows(args.resident, SHAPES[name][0] // world)
                if nr > 0:
                    n_res_map[(l, name)] = nr
                    W_dev_map[(l, name)] = st["host"][l][name][:nr].cuda()
        torch.cuda.synchronize()
    layers, plans, all_plans = build_layers(st, args, mode, af, n_res_map, W_dev_map)
    h_dev.copy_(h_host)

    # ---- a1 refinement: the alpha benchmark (Sec. 4.4) around the Eq. (5) alpha: lane
    # times measured in this pipeline under real interference, fitted and solved F_CPU = F_COM ----
    abench = None
    # Eq. (5) alpha from the measured rates (the same for every module: rates are per byte)
    alpha_seed = ctx.plan(rates, SHAPES["fc1"][0] // world, H, B, 0, mode, af).alpha_req
    any_host = any(p.n_res < p.N for p in all_plans)
    if args.alpha is None and args.abench and any_host:
        if world > 1:  # every rank must sample the same alpha grid (the stack all-gathers)
            t = torch.tensor([alpha_seed], dtype=torch.float64, device=coll_device())
            dist.broadcast(t, 0)
            alpha_seed = float(t.item())
        def agreed(r):
            # every rank must run the same number of alpha-benchmark rounds over the same window (each
            # round runs the stack, whose all-gathers need every rank): take rank 0's decision
            if world == 1:
                return r.alpha_bar, bool(r.clamped)
            t = torch.tensor([r.alpha_bar, 1.0 if r.clamped else 0.0], dtype=torch.float64, device=coll_device())
            dist.broadcast(t, 0)
            return float(t[0].item()), bool(t[1].item() > 0.5)

        # no balance point inside the window: re-centre it on the clamped edge (up to 4 rounds) -- in the
        # library at N = 1; with N > 1 every rank must run the same rounds, so rank 0's decision is
        # broadcast between one-round calls
        res = ctx.hg_alpha_bench(layers, h_dev, B, alpha_seed, gamma=args.abench_gamma, lam=0.02, degree=2,
                                 reps=1, stream=s, max_rounds=4 if world == 1 else 1)
        alpha_bar, clamped = agreed(res)
        rounds = res.rounds
        while world > 1 and clamped and rounds < 4 and 0.0 < alpha_bar < 1.0:
            res = ctx.hg_alpha_bench(layers, h_dev, B, alpha_bar, gamma=args.abench_gamma, lam=0.02,
                                     degree=2, reps=1, stream=s)
            alpha_bar, clamped = agreed(res)
            rounds += 1
        abench = res.as_dict()
        abench["rounds"] = rounds
        abench["alpha_used"] = alpha_bar
        layers, plans, all_plans = build_layers(st, args, hg.FIXED, alpha_bar, n_res_map, W_dev_map)
        h_dev.copy_(h_host)

    def barrier():
        if world > 1:
            dist.barrier()

    def step_device():
        ctx.hg_stack(layers, h_dev, B, stream=s)

    def step_e2e():
        with torch.cuda.stream(s):
            h_dev.copy_(h_host, non_blocking=True)
        ctx.hg_stack(layers, h_dev, B, stream=s)
        with torch.cuda.stream(s):
            h_out.copy_(h_dev, non_blocking=True)

    # ---- warm-up ----
    for _ in range(args.warmup):
        step_device()
    torch.cuda.synchronize()

    # ---- timed region (device events on the launching stream; max over ranks) ----
    clocks = Clocks(local)
    clocks.start()
    ctx.hg_reset_stats()
    barrier()
    torch.cuda.synchronize()
    # one event per step boundary on the launching stream: the distribution of step times (recording
    # an event between steps adds no synchronisation)
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    w0 = time.perf_counter()
    torch.cuda.nvtx.range_push("hg_timed")  # ncu --nvtx --nvtx-include hg_timed/ selects these launches
    evs[0].record(s)
    for i in range(args.steps):
        step_device()
        evs[i + 1].record(s)
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_pop()
    wall = time.perf_counter() - w0
    barrier()
    launches = ctx.hg_stats().gpu_launches
    ck = clocks.stop()
    dev_s = evs[0].elapsed_time(evs[-1]) * 1e-3
    step_ms = sorted(evs[i].elapsed_time(evs[i + 1]) for i in range(args.steps))

    # ---- e2e: public API with host buffers, H2D of the step input + D2H of the result ----
    barrier()
    torch.cuda.synchronize()
    e2, e3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e2.record(s)
    for _ in range(args.steps):
        step_e2e()
    e3.record(s)
    torch.cuda.synchronize()
    e2e_s = e2.elapsed_time(e3) * 1e-3

    # ---- lane breakdown (Table 2 analogue): instrumented steps after the timed region ----
    sctx_stats = None
    if args.breakdown and world == 1:
        sctx = hg.Context(local, cpu_threads=st["threads"], cpu_first=-1, chunk_bytes=args.chunk_mb << 20,
                          ring_bytes=args.ring_mb << 20, max_k=F, max_n=F, wrap_prefetch=1, collect_stats=1,
                          pageable=int(args.pageable), pin_threads=4, strategy=STRATEGIES[args.strategy],
                          staging_bytes=args.staging_mb << 20)
        sctx.hg_stack(layers, h_dev, B, stream=s)  # fill the prefetch pipeline
        sctx.hg_reset_stats()
        for _ in range(2):
            sctx.hg_stack(layers, h_dev, B, stream=s)
        torch.cuda.synchronize()
        sctx_stats = sctx.hg_stats().as_dict()
        sctx.close()

    # ---- dominant kernel: the per-linear GEMV launch, replayed with CUDA events on cold data ----
    roof = None
    if rank == 0:
        roof = gemv_roofline(ctx, plans, args.layers, B, torch, pk,
                             W_dev={name: W_dev_map.get((0, name)) for name in NAMES})

    # ---- parity leg, part 1: one more step of the timed path (same context, plans and layers) with
    # layers 0 and L-1 traced; the oracle side runs in the cpu_baseline leg (main_arm) ----
    trace = None
    if rank == 0 and world == 1 and args.parity and not args.no_cpu_baseline:
        trace = trace_layers(st, layers, sorted({0, args.layers - 1}))

    # ---- rates re-probed after the timed region: the path roofline takes the larger of the two probes
    # of each peak (a probe that under-reads would flatter the fraction) ----
    rates_post = ctx.hg_measure(st["host"][0]["fc1"], st["host"][0]["fc1"].shape[0], H, B, under_load=True)
    rdp = rates_post.as_dict()

    times = torch.tensor([dev_s, e2e_s, wall], device=coll_device())
    if world > 1:
        dist.all_reduce(times, op=dist.ReduceOp.MAX)
    dev_s, e2e_s, wall = times.tolist()
    ms_tok = dev_s / args.steps * 1e3
    e2e_ms = e2e_s / args.steps * 1e3

    # ---- roofline numbers ----
    hbm_peak = pk.get("hbm_gbs", 6650.0)
    plan_tot = {"t_pred": 0.0, "bytes_str": 0, "bytes_cpu": 0, "bytes_res": 0}
    for p in all_plans:
        plan_tot["t_pred"] += p.t_pred
        plan_tot["bytes_str"] += 2 * p.K * p.n_str
        plan_tot["bytes_cpu"] += 2 * p.K * p.n_cpu
        plan_tot["bytes_res"] += 2 * p.K * p.n_res
    # stack roofline: the link runs ahead across linears, so lanes add up over the stack
    peak = {k: max(rd[k], rdp[k]) for k in ("b_link", "b_cpu", "b_host")}
    t_link_roof = plan_tot["bytes_str"] / peak["b_link"]
    t_cpu_roof = plan_tot["bytes_cpu"] / peak["b_cpu"]
    t_hbm_roof = (plan_tot["bytes_res"] + 2 * plan_tot["bytes_str"]) / (hbm_peak * 1e9)
    # 4th term: every offloaded byte is read from host DRAM once, by the DMA or by the
    # CPU lane, so the joint host-DRAM rate measured with both running bounds the sum
    b_host = peak["b_host"] or 0.0
    t_host_roof = (plan_tot["bytes_str"] + plan_tot["bytes_cpu"]) / b_host if b_host > 0 else 0.0
    # best achievable over alpha: all host bytes shared by link + CPU at their peaks
    shard_bytes = STACK_BYTES / world * args.layers / LAYERS
    host_bytes = plan_tot["bytes_str"] + plan_tot["bytes_cpu"]
    t_opt = max(host_bytes / min(peak["b_link"] + peak["b_cpu"], b_host if b_host > 0 else math.inf), t_hbm_roof)
    t_roof = max(t_link_roof, t_cpu_roof, t_hbm_roof, t_host_roof)
    lanes = None
    if sctx_stats:
        wall_i = sctx_stats["wall_s"] or 1
        lanes = {"link_GBps": round(sctx_stats["bytes_str"] / max(sctx_stats["link_busy_s"], 1e-9) / 1e9, 2),
                 "link_peak_GBps": round(rd["b_link"] / 1e9, 2),
                 "cpu_GBps": round(sctx_stats["bytes_cpu"] / max(sctx_stats["cpu_busy_s"], 1e-9) / 1e9, 2),
                 "cpu_peak_GBps": round(rd["b_cpu"] / 1e9, 2),
                 "busy_frac": {"cpu": round(sctx_stats["cpu_busy_s"] / wall_i, 3),
                               "link": round(sctx_stats["link_busy_s"] / wall_i, 3),
                               "gpu": round(sctx_stats["gpu_busy_s"] / wall_i, 4)},
                 "x_wait_ms": round(sctx_stats["x_wait_s"] * 1e3, 2),
                 "pin_GBps": round(sctx_stats["bytes_pinned"] / sctx_stats["pin_busy_s"] / 1e9, 2)
                 if sctx_stats["pin_busy_s"] > 0 else None,
                 "glue_ms": round(sctx_stats["glue_s"] * 1e3, 2),
                 "steps": 2, "mirror_linears": sctx_stats["mirror_linears"]}
        # overlap fraction = (sum busy - wall) / (sum busy - max busy); 1 = the lanes fully
        # overlap, 0 = they run one after another
        busy = [sctx_stats["cpu_busy_s"], sctx_stats["link_busy_s"], sctx_stats["gpu_busy_s"]]
        den = sum(busy) - max(busy)
        lanes["overlap_frac"] = round((sum(busy) - sctx_stats["wall_s"]) / den, 4) if den > 0 else None
    line = {
        "metric": METRIC, "value": round(ms_tok, 3), "unit": "ms/token", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_tok, 3),
        "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (seeded counter-based generator; random-init OPT-30B-shaped weights)",
        "config": {"workload": "%s %d-layer decode linear stack (qkv,o,fc1,fc2 x%d), batch %d" % (
                       MODEL.upper().replace("OPT-", "OPT-"), args.layers, args.layers, B),
                   "model": MODEL,
                   "batch": B, "hidden": H, "ffn": F, "layers": args.layers,
                   "r_resident": round(plan_tot["bytes_res"] / shard_bytes, 4),
                   "hbm_budget_GB": budget_gb,
                   "alpha_mode": "fixed" if args.alpha is not None else (
                       ("Eq9" if args.pageable else "Eq5") + (" (measured rates) refined by the alpha benchmark "
                                                              "(Sec. 4.4)" if abench else " (measured rates)")),
                   "host_weights": ("pageable, strategy %s (Fig. 5%s)" % (args.strategy, {"hybrid": "c, pin lane of "
                                    "Sec. 4.3", "naive": "a", "blocking": "b"}[args.strategy])) if args.pageable
                   else "pinned once at load",
                   "alpha": next((p.alpha_eff for p in all_plans if p.n_res < p.N), 0.0),
                   "alpha_seed_eq5": alpha_seed,
                   "parallelism": (f"tp{world} column shards, %s exchange" % args.exchange) if world > 1 else "1 GPU",
                   "chunk_MiB": args.chunk_mb, "ring_MiB": args.ring_mb, "cpu_threads": st["threads"],
                   "numa": {"node": st["placement"][0], "cores_per_rank": st["placement"][1],
                            "pool_pinned_from": st["placement"][2],
                            "weights": "hg_host_alloc, bound to the node" if st["placement"][0] >= 0
                            else "hg_host_alloc (no NUMA node reported)"},
                   "l2": "inputs larger than L2: %.1f GB of weights streamed/computed per step" % (shard_bytes / 1e9)},
        "gpu_launches": int(launches),
        "e2e": {"value": round(e2e_ms, 3), "unit": "ms/token", "h2d_bytes_per_step": B * H * 2,
                "d2h_bytes_per_step": B * H * 2},
        "roofline": roof,
        "path_roofline": {"bound": "max(host link, host CPU, HBM, joint host DRAM)",
                          "terms_ms": {"link": round(t_link_roof * 1e3, 3), "cpu": round(t_cpu_roof * 1e3, 3),
                                       "hbm": round(t_hbm_roof * 1e3, 3), "host_dram": round(t_host_roof * 1e3, 3)},
                          "t_roof_ms_at_plan_alpha": round(t_roof * 1e3, 3),
                          "t_opt_ms_best_alpha": round(t_opt * 1e3, 3),
                          "frac_of_roof_at_plan": round(t_roof * 1e3 / ms_tok, 4),
                          "frac_of_best": round(t_opt * 1e3 / ms_tok, 4),
                          "t_pred_ms_sum": round(plan_tot["t_pred"] * 1e3, 3),
                          "peaks_GBps": {k: round(v / 1e9, 2) for k, v in peak.items()},
                          "peaks_source": "max of the hg_measure probes before and after the timed region",
                          "probe_under_read": bool(t_roof * 1e3 / ms_tok > 1.0)},
        "step_ms": {"min": round(step_ms[0], 3), "p10": round(pct(step_ms, 10), 3), "p50": round(pct(step_ms, 50), 3),
                    "p90": round(pct(step_ms, 90), 3), "max": round(step_ms[-1], 3),
                    "note": "per-step CUDA events on the launching stream inside the timed region"},
        "rates_GBps": {k: (round(v / 1e9, 2) if math.isfinite(v) else None) for k, v in rd.items()},
        "rates_post_GBps": {k: (round(v / 1e9, 2) if math.isfinite(v) else None) for k, v in rdp.items()},
        "lanes": lanes,
        "scheduler": sched,
        "alpha_bench": None if abench is None else {
            "alpha_bar": abench["alpha_bar"], "clamped": abench["clamped"], "rounds": abench["rounds"],
            "points": [[round(a, 4), round(tc * 1e3, 3), round(tl * 1e3, 3), round(ts * 1e3, 3)] for a, tc, tl, ts in
                       zip(abench["alpha"], abench["t_cpu"], abench["t_com"], abench["t_step"])],
            "points_cols": ["alpha", "t_cpu_ms", "t_link_ms", "t_step_ms"]},
        "clocks": ck,
        "wall_ms_per_step": round(wall / args.steps * 1e3, 3),
        "setup_s": round(st["t_setup"], 1),
        "_trace": trace,
    }
    del W_dev_map, layers
    torch.cuda.empty_cache()
    return line


def trace_layers(st, layers, which):
    """Run one step through hg_stack_trace (the timed path, mirrored glue included) with `which`
    layers traced; returns {layer: {name: host ndarray}} plus the step's input h of layer 0."""
    import numpy as np
    torch, hg, ctx, B, s = st["torch"], st["hg"], st["ctx"], st["B"], st["stream"]
    bufs = {}
    for l in which:
        tr = {k: torch.zeros(B, n, dtype=torch.int16, device="cuda") for k, n in
              (("a", H), ("v", H), ("h1", H), ("a2", H), ("u", F))}
        tr.update({k: torch.zeros(B, n, device="cuda") for k, n in
                   (("y_qkv", 3 * H), ("y_o", H), ("y_fc1", F), ("y_fc2", H))})
        bufs[l] = tr
    h_in = st["h_host"].numpy().view(np.uint16).copy()
    st["h_dev"].copy_(st["h_host"])
    torch.cuda.synchronize()
    ctx.hg_reset_stats()
    ctx.hg_stack_trace(layers, st["h_dev"], B, {l: hg.layer_trace(**tr) for l, tr in bufs.items()}, stream=s)
    torch.cuda.synchronize()
    stats = ctx.hg_stats()
    out = {l: {k: (v.cpu().numpy().view(np.uint16) if v.dtype == torch.int16 else v.cpu().numpy())
               for k, v in tr.items()} for l, tr in bufs.items()}
    return {"layers": out, "h_in": h_in, "mirror_linears": int(stats.mirror_linears),
            "h_out": st["h_dev"].cpu().numpy().view(np.uint16).copy()}


LIN_IO = (("qkv", "a", "y_qkv"), ("o", "v", "y_o"), ("fc1", "a2", "y_fc1"), ("fc2", "u", "y_fc2"))


def cpu_baseline_and_parity(st, trace, sample_rows=256):
    """The cpu_baseline leg: the fp64 oracle timed on layer 0 end to end on the host cores (and one
    linear on one thread).  With a trace of the timed path the oracle is also fed the GPU's own bf16
    inputs to layer 0's linears (teacher-forced) and its outputs are compared with
    the GPU's element by element (BJ:5 tolerance); the last layer is compared on `sample_rows` seeded
    rows per linear (oracle.linear_rows); layer 0's glue against the oracle's LN / V / residual / ReLU;
    and the oracle's own end-to-end layer 0 (not teacher-forced) against the GPU's outputs (looser,
    secondary, as in tests/test_gpu_layer.py)."""
    import numpy as np
    import oracle
    B, nthr = st["B"], os.cpu_count() or 1
    W = lambda l, n: st["host"][l][n].numpy().view(np.uint16)
    bias = lambda l, n: st["biases_h"][l][n].numpy()
    # the baseline: layer 0 end to end through the oracle on all host threads, on the step's input h
    Wd0 = {n: W(0, n) for n in NAMES}
    bd0 = {n: bias(0, n) for n in NAMES}
    h_in = trace["h_in"] if trace is not None else initial_h(B)
    t_layer, ref0 = oracle_layer_time(h_in, Wd0, bd0, nthr)
    # single thread: the o projection of layer 0 (its share of the token's bytes scales it)
    t0 = time.perf_counter()
    oracle.linear(ref0["v"], Wd0["o"], bd0["o"], nthreads=1)
    t_o1 = time.perf_counter() - t0
    o_bytes = 2 * SHAPES["o"][0] * SHAPES["o"][1]
    cb = {"value": round(t_layer * LAYERS * 1e3, 1), "unit": "ms/token", "cores": nthr, "kind": "oracle",
          "sample": "layer 0 end to end (LN, 4 linears, V, residuals, ReLU; %.3f GB of weights) through the fp64 "
                    "oracle on all host threads, scaled x%d to a token" % (STACK_BYTES / LAYERS / 1e9, LAYERS),
          "single_thread": {"value": round(t_o1 * STACK_BYTES / o_bytes * 1e3, 1), "unit": "ms/token", "cores": 1,
                            "sample": "layer 0's o projection (%.1f MB) on one thread, scaled by bytes to a token"
                                      % (o_bytes / 1e6)},
          "host": host_info()}
    if trace is not None:
        T0 = trace["layers"][0]
        ys = {}
        for n, xin, _ in LIN_IO:  # teacher-forced: the GPU's own bf16 inputs
            ys[n] = oracle.linear(T0[xin], W(0, n), bias(0, n), nthreads=nthr)
    if trace is None:
        return cb, None
    worst, ok, checked, per = 0.0, True, 0, {}
    for n, _, yk in LIN_IO:
        good, w = oracle.within_tol(T0[yk], ys[n])
        per["L0." + n] = round(w, 6)
        ok &= good
        worst = max(worst, w)
        checked += T0[yk].size
    rng = np.random.default_rng(SEED)
    for l, T in trace["layers"].items():
        if l == 0:
            continue
        for n, xin, yk in LIN_IO:
            rows = np.sort(rng.choice(SHAPES[n][0], size=min(sample_rows, SHAPES[n][0]), replace=False))
            ref = oracle.linear_rows(T[xin], W(l, n), rows, bias(l, n), nthreads=nthr)
            good, w = oracle.within_tol(T[yk][:, rows], ref)
            per["L%d.%s" % (l, n)] = round(w, 6)
            ok &= good
            worst = max(worst, w)
            checked += ref.size
    chk = lambda got, ref: oracle.within_tol(oracle.bf16_to_f64(got), oracle.bf16_to_f64(ref))
    glue = [chk(T0["a"], oracle.layernorm(trace["h_in"])), chk(T0["v"], oracle.attention_pos0(T0["y_qkv"], H)),
            chk(T0["h1"], oracle.residual(trace["h_in"], T0["y_o"])), chk(T0["a2"], oracle.layernorm(T0["h1"])),
            chk(T0["u"], oracle.relu_bf16(T0["y_fc1"]))]
    glue_ok = all(g for g, _ in glue)
    e2e = [oracle.within_tol(T0[yk], ref0[yk], rtol=5e-2) for _, _, yk in LIN_IO]
    parity = {"ok": bool(ok and glue_ok), "worst": round(worst, 6), "glue_ok": glue_ok,
              "glue_worst": round(max(w for _, w in glue), 6),
              "tolerance": "|y - y_ref| <= 1e-2 max(1, |y_ref|) elementwise (BJ:5); worst = max err/bound",
              "checked_outputs": int(checked), "per_linear": per, "mirror_linears": trace["mirror_linears"],
              "layer0_end_to_end": {"ok": all(g for g, _ in e2e), "worst": round(max(w for _, w in e2e), 6),
                                    "rtol": 5e-2},
              "what": "one extra step of the timed path (same context/plans, hg_stack_trace); layer 0 all "
                      "outputs + glue, layer %d on %d seeded rows per linear, teacher-forced fp64 oracle"
                      % (max(trace["layers"]), sample_rows)}
    return cb, parity


def main_arm(args):
    st = prepare(args)
    line = run_point(st, args, args.hbm_budget_gb)
    rank, world = st["rank"], st["world"]
    trace = line.pop("_trace", None)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"], line["parity"] = cpu_baseline_and_parity(st, trace)
    if rank == 0:
        print(json.dumps(line), flush=True)
    st["ctx"].close()
    if world > 1:
        st["dist"].destroy_process_group()
    return 0


def parse_args(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=8)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--batch", type=int, default=1)
    ap.add_argument("--model", default="opt-30b", choices=sorted(MODELS),
                    help="OPT shape (default opt-30b, the headline; opt-6.7b = C2, opt-13b = C3)")
    ap.add_argument("--layers", type=int, default=None, help="(development only; the metric needs all layers)")
    ap.add_argument("--alpha", type=float, default=None)
    ap.add_argument("--chunk-mb", type=int, default=32)
    ap.add_argument("--ring-mb", type=int, default=4096)
    ap.add_argument("--threads", type=int, default=0)
    ap.add_argument("--no-breakdown", dest="breakdown", action="store_false")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-abench", dest="abench", action="store_false", help="use Eq. (5) alpha unrefined")
    ap.add_argument("--abench-gamma", type=float, default=0.06)
    ap.add_argument("--pageable", action="store_true",
                    help="NEXT(1): host weights not page-locked; streamed chunks go through the pin lane")
    ap.add_argument("--strategy", default="hybrid", choices=sorted(STRATEGIES),
                    help="with --pageable: how streamed rows reach the device (Fig. 5c hybrid, 5a naive, "
                         "5b pinned-blocking)")
    ap.add_argument("--staging-mb", type=int, default=512,
                    help="with --pageable: the pin lane's pinned staging ring (MiB)")
    ap.add_argument("--scheduler", default="module", choices=["module", "rows"],
                    help="with --hbm-budget-gb: Sec. 4.5's module greedy, or one resident fraction for every "
                         "linear (hg_schedule_rows)")
    ap.add_argument("--resident", type=float, default=0.0,
                    help="fraction r of every linear's rows resident in HBM (C2: r = 0.5)")
    ap.add_argument("--hbm-budget-gb", type=float, default=0.0,
                    help="NEXT(3): GPU memory for resident weights, placed by the module scheduler (Sec. 4.5)")
    ap.add_argument("--exchange", default="peer", choices=["peer", "nccl"],
                    help="N > 1: the shard exchange after each linear -- peer-memory pushes + shared host segment "
                         "(default) or NCCL all-gather (GPU-only glue)")
    ap.add_argument("--numa", default="auto", choices=["auto", "off"],
                    help="host placement: weights bound to the GPU's NUMA node; with N > 1 each rank's CPU "
                         "lane pinned to its share of that node's cores")
    ap.add_argument("--ref-layers", type=int, default=2,
                    help="--impl reference: OPT layers per step through the oracle (a bounded sample of the token)")
    ap.add_argument("--no-parity", dest="parity", action="store_false",
                    help="skip the parity leg (one traced step checked against the oracle)")
    args = ap.parse_args(argv)
    set_model(args.model)
    if args.layers is None:
        args.layers = LAYERS
    if args.warmup < 3:
        args.warmup = 3
    return args


def main():
    args = parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return main_arm(args)


if __name__ == "__main__":
    sys.exit(main())
