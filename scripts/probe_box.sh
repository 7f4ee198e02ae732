#!/bin/bash
# One-off probe of the GPU box: host cores, memory, GPU, PCIe bandwidth.
mkdir -p gpurun_out
{
nvidia-smi; nvidia-smi -q | grep -iE 'PCIe|Link|Gen|Width' | head -30
nproc; lscpu | head -25; free -g
python - <<'PY'
import torch, time
print(torch.cuda.get_device_properties(0))
n = 1 << 28  # 2 GiB fp64... use bytes
for nbytes in [64<<20, 512<<20, 2<<30]:
    h = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(nbytes, dtype=torch.uint8, device='cuda')
    for _ in range(2): d.copy_(h, non_blocking=True); h.copy_(d, non_blocking=True)
    torch.cuda.synchronize()
    e0, e1, e2 = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    e0.record(); d.copy_(h, non_blocking=True); e1.record(); h.copy_(d, non_blocking=True); e2.record(); torch.cuda.synchronize()
    print(f"pinned {nbytes>>20} MiB: H2D {nbytes/e0.elapsed_time(e1)/1e6:.1f} GB/s  D2H {nbytes/e1.elapsed_time(e2)/1e6:.1f} GB/s")
    p = torch.empty(nbytes, dtype=torch.uint8)
    e0.record(); d.copy_(p); e1.record(); p.copy_(d); e2.record(); torch.cuda.synchronize()
    print(f"pageable {nbytes>>20} MiB: H2D {nbytes/e0.elapsed_time(e1)/1e6:.1f} GB/s  D2H {nbytes/e1.elapsed_time(e2)/1e6:.1f} GB/s")
# HBM read/copy
x = torch.empty(1<<28, dtype=torch.float64, device='cuda'); y = torch.empty_like(x)
for _ in range(3): y.copy_(x)
torch.cuda.synchronize(); e0.record()
for _ in range(10): y.copy_(x)
e1.record(); torch.cuda.synchronize()
print(f"copy {2*x.numel()*8*10/e0.elapsed_time(e1)/1e6:.1f} GB/s")
e0.record()
for _ in range(10): s = x.sum()
e1.record(); torch.cuda.synchronize()
print(f"read(sum) {x.numel()*8*10/e0.elapsed_time(e1)/1e6:.1f} GB/s")
PY
} > gpurun_out/probe_box.txt 2>&1
