"""Development aid: host enqueue time vs device time of the bench's GEMV replay loop (o projection)."""
import os, sys, time
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2403_01164_b200 import hg  # noqa: E402
H = 7168
ctx = hg.Context(0, chunk_bytes=32 << 20, ring_bytes=4096 << 20, max_k=4 * H, max_n=4 * H)
for name, (N, K) in {"o": (H, H), "qkv": (3 * H, H)}.items():
    p = ctx.plan(hg.make_rates(1, 1, 1), N, K, 1, 0, hg.FIXED, 0.24)
    x = torch.empty((1, K), dtype=torch.int16, device="cuda").random_(-3000, 3000)
    y = torch.empty((1, N), device="cuda")
    s = torch.cuda.current_stream()
    step = max(1, p.n_chunks)
    for spin in (4_000_000, 40_000_000):
        for it in range(3):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda._sleep(spin)
            e0.record(s)
            t0 = time.perf_counter()
            for i in range(20):
                ctx.hg_gemv_replay(p, x, None, None, y, stream=s, seq0=i * step)
            th = time.perf_counter() - t0
            e1.record(s)
            torch.cuda.synchronize()
            print(name, "spin", spin, "host us/call %.1f" % (th / 20 * 1e6), "gpu us/launch %.2f" % (e0.elapsed_time(e1) * 1e3 / 20), flush=True)
