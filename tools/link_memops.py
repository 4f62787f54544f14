"""Copy-engine cost of stream memory operations between H2D chunk copies (development probe)."""
import sys, time
import torch
from cuda.bindings import driver as drv

def main():
    chunk_mb = [int(a) for a in (sys.argv[1:] or ["16", "32", "64"])]
    total = 2 << 30
    src = torch.empty(total, dtype=torch.uint8, pin_memory=True)
    dst = torch.empty(total, dtype=torch.uint8, device="cuda")
    tags = torch.zeros(1024, dtype=torch.int32, device="cuda")
    s = torch.cuda.Stream()
    h = drv.CUstream(s.cuda_stream)
    base = tags.data_ptr()
    for cm in chunk_mb:
        cb = cm << 20
        n = total // cb
        for mode in ("plain", "write", "wait", "both"):
            best = 0
            for rep in range(3):
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
                e0.record(s)
                with torch.cuda.stream(s):
                    for i in range(n):
                        if mode in ("wait", "both"):
                            drv.cuStreamWaitValue32(h, drv.CUdeviceptr(base + 4 * (i % 512)), 0, 0)
                        dst[i * cb:(i + 1) * cb].copy_(src[i * cb:(i + 1) * cb], non_blocking=True)
                        if mode in ("write", "both"):
                            drv.cuStreamWriteValue32(h, drv.CUdeviceptr(base + 4 * (512 + i % 512)), i + 1, 0)
                e1.record(s)
                torch.cuda.synchronize()
                gbps = total / (e0.elapsed_time(e1) * 1e-3) / 1e9
                best = max(best, gbps)
            print(f"chunk {cm:3d} MiB {mode:6s}: {best:6.2f} GB/s", flush=True)

main()
