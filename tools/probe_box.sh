#!/bin/bash
# One-shot probe of the GPU box host: CPU, RAM, NUMA, link, pin speed.
out=gpurun_out/probe
mkdir -p $out
{
echo "== lscpu"; lscpu
echo "== nproc"; nproc
echo "== cgroup cpu"; cat /sys/fs/cgroup/cpu.max 2>/dev/null; cat /sys/fs/cgroup/cpuset.cpus.effective 2>/dev/null
echo "== cgroup mem"; cat /sys/fs/cgroup/memory.max 2>/dev/null
echo "== free"; free -g
echo "== numa"; ls /sys/devices/system/node/; for n in /sys/devices/system/node/node*; do echo $n; cat $n/cpulist; grep MemTotal $n/meminfo; done
echo "== ulimit -l"; ulimit -l
echo "== nvidia-smi"; nvidia-smi; nvidia-smi topo -m
echo "== pcie"; nvidia-smi --query-gpu=pcie.link.gen.current,pcie.link.gen.max,pcie.link.width.current,pcie.link.width.max --format=csv
echo "== flags"; grep -o -w -E 'avx512_bf16|amx_bf16|amx_tile|avx512f|avx512_fp16|avx2|fma' /proc/cpuinfo | sort | uniq -c
} > $out/host.txt 2>&1
python - > $out/torch_probe.txt 2>&1 <<'PY'
import torch, time
d = torch.device('cuda:0')
print(torch.cuda.get_device_properties(0))
print("L2", torch.cuda.get_device_properties(0).L2_cache_size)
for gb in [1, 8]:
    t0=time.time(); h = torch.empty(gb<<30, dtype=torch.uint8, pin_memory=True); t1=time.time()
    print(f"pin alloc {gb} GiB: {t1-t0:.3f}s")
    dbuf = torch.empty(gb<<30, dtype=torch.uint8, device=d)
    h.fill_(1)
    for chunk_mb in [1, 4, 8, 32, 256]:
        n = chunk_mb<<20; s = torch.cuda.Stream()
        torch.cuda.synchronize()
        e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):
            e0.record()
            off=0
            while off + n <= h.numel():
                dbuf[off:off+n].copy_(h[off:off+n], non_blocking=True); off+=n
            e1.record()
        torch.cuda.synchronize()
        print(f"H2D {gb}GiB chunk {chunk_mb}MB: {off/e0.elapsed_time(e1)/1e6:.2f} GB/s")
    e0.record(); h.copy_(dbuf, non_blocking=True); e1.record(); torch.cuda.synchronize()
    print(f"D2H {gb}GiB: {h.numel()/e0.elapsed_time(e1)/1e6:.2f} GB/s")
    del h, dbuf
t0=time.time(); h = torch.empty(32<<30, dtype=torch.uint8, pin_memory=True); print(f"pin alloc 32 GiB: {time.time()-t0:.3f}s")
del h
# host read bandwidth via torch (multi-thread sum)
import os
print("threads", torch.get_num_threads())
a = torch.ones(2<<30, dtype=torch.uint8)
a32 = a.view(torch.int32)
t0=time.time()
for _ in range(3): s = a32.sum()
print(f"host read BW (torch sum int32 {torch.get_num_threads()} thr): {3*a.numel()/(time.time()-t0)/1e9:.1f} GB/s")
PY
echo done
