"""Where the per-launch time of the SIMT GEMV goes, at the step's launch sizes (OPT-30B linears,
B=1, GPU rows of each linear at the bench's alpha).  Measurement only (GPU box):

  flushW   one launch after a 256 MiB zero_() (the bench's L2 flush: leaves dirty lines)
  flushR   one launch after a 256 MiB read (clean L2)
  b2b      20 back-to-back launches rotating over distinct W copies (> L2 in total), per launch
  held     the same 20 launches enqueued while a GPU spin kernel holds the stream, per launch
  stamps   per-CTA globaltimer stamps of one launch after a read flush: CTA entry spread, first
           stage full (latency from the CTA's entry), consumer / producer done (from first entry)
  floor    a 1-element torch kernel back to back (the GPU's launch floor)
"""
import os
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2403_01164_b200 import hg  # noqa: E402

B = int(os.environ.get("B", 1))
ALPHA_ROWS = {  # GPU rows of each OPT-30B linear at alpha ~0.24 (bench), and K
    "qkv": (5376, 7168), "o": (1792, 7168), "fc1": (7040, 7168), "fc2": (1792, 28672)}
if os.environ.get("SHAPES") == "sizes":
    ALPHA_ROWS = {f"r{n}": (n, 7168) for n in (128, 512, 2048, 8192, 28672)}


def ev_time(fn, s):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    fn()
    e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e-3


def main():
    torch.cuda.set_device(0)
    s = torch.cuda.current_stream()
    ctx = hg.Context(0, max_k=28672, max_n=32768)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    flushf = flush.view(torch.float32)
    one = torch.zeros(1, device="cuda")
    for _ in range(10):
        one.add_(1)
    torch.cuda.synchronize()
    floor = ev_time(lambda: [one.add_(1) for _ in range(200)], s) / 200
    print(f"floor: torch 1-element kernel back to back {floor*1e6:.2f} us/launch (CPU-bound)")
    fl = []
    for _ in range(10):
        flushf.sum()
        fl.append(ev_time(lambda: one.add_(1), s))
    print(f"floor: one torch 1-element kernel after a read flush, event to event {statistics.mean(fl)*1e6:.2f} us")
    for name, (n, K) in ALPHA_ROWS.items():
        nbytes = 2 * n * K
        ncopy = max(2, int(np.ceil(300e6 / nbytes)))
        Ws = [torch.empty((n, K), dtype=torch.int16, device="cuda").random_(-3000, 3000) for _ in range(ncopy)]
        x = torch.empty((B, K), dtype=torch.int16, device="cuda").random_(-3000, 3000)
        y = torch.empty((B, n), device="cuda")
        g = lambda W: ctx.hg_gemv(x, B, n, K, W, None, y, stream=s)  # noqa: E731
        for W in Ws:
            g(W)
        torch.cuda.synchronize()
        tw, tr = [], []
        for i in range(10):
            flush.zero_()
            tw.append(ev_time(lambda: g(Ws[i % ncopy]), s))
            flushf.sum()
            tr.append(ev_time(lambda: g(Ws[i % ncopy]), s))
        reps = 20
        b2b = ev_time(lambda: [g(Ws[i % ncopy]) for i in range(reps)], s) / reps
        torch.cuda._sleep(4_000_000)  # hold the GPU while the host enqueues (device-side b2b)
        tg = ev_time(lambda: [g(Ws[i % ncopy]) for i in range(reps)], s) / reps
        st = hg.hg_debug_gemv_stamps(4096)
        st[:] = 0
        flushf.sum()
        torch.cuda.synchronize()
        g(Ws[0])
        torch.cuda.synchronize()
        hg.hg_debug_gemv_stamps(0, on=False)
        nct = int((st[:, 0] > 0).sum())
        t0 = st[:nct, 0].min()
        entry = (st[:nct, 0] - t0) / 1e3
        has = st[:nct, 1] > 0
        first = (st[:nct, 1][has] - st[:nct, 0][has]) / 1e3
        cons = (st[:nct, 2] - t0) / 1e3
        prod = (st[:nct, 3][st[:nct, 3] > 0] - t0) / 1e3
        gb = lambda t: nbytes / t / 1e9  # noqa: E731
        print(f"{name:5s} n={n:6d} K={K:6d} {nbytes/1e6:7.2f} MB | flushW {statistics.mean(tw)*1e6:7.2f} us "
              f"({gb(statistics.mean(tw)):6.0f} GB/s) | flushR {statistics.mean(tr)*1e6:7.2f} us "
              f"({gb(statistics.mean(tr)):6.0f}) | b2b {b2b*1e6:7.2f} us ({gb(b2b):6.0f}) | held {tg*1e6:7.2f} us "
              f"({gb(tg):6.0f})")
        print(f"      stamps: ctas={nct} entry spread {entry.max():.2f} us | first stage full after "
              f"{np.median(first):.2f} (p90 {np.percentile(first, 90):.2f}) us | consumers done med "
              f"{np.median(cons):.2f} max {cons.max():.2f} us | producer done max {prod.max() if len(prod) else 0:.2f} us")
        del Ws
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
