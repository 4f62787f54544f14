"""Development aid: hg_gemv (one resident block) back to back over a flat 4 GiB buffer at the replay's
sizes -- the same launch sequence as tools/probes/read_ceiling.cu's per-linear loop, through the library."""
import os, sys, time
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2403_01164_b200 import hg  # noqa: E402
K = 7168
ctx = hg.Context(0, chunk_bytes=32 << 20, ring_bytes=64 << 20, max_k=4 * K, max_n=4 * K)
buf = torch.ones((4 << 30) // 2, dtype=torch.int16, device="cuda")
x = torch.empty((1, K), dtype=torch.int16, device="cuda").random_(-3000, 3000)
y = torch.empty((1, 64 << 10), device="cuda")
s = torch.cuda.Stream()
tb = tt = 0.0
for name, rows in (("qkv", 5376), ("o", 1792), ("fc1", 7040), ("fc2-like", 7168)):
    n = rows
    best = 1e9
    for t in range(5):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):
            torch.cuda._sleep(4_000_000)
            e0.record(s)
            off = 0
            for i in range(20):
                if off + n * K > buf.numel():
                    off = 0
                ctx.hg_gemv(x, 1, n, K, buf[off:], None, y, stream=s)
                off += n * K
            e1.record(s)
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) * 1e3 / 20)
    tb += 2 * n * K
    tt += best
    print(name, rows, "%.2f us" % best, "%.1f GB/s" % (2 * n * K / best / 1e3), flush=True)
print("frac %.3f" % (tb / tt / 1e3 / 6542.4))
