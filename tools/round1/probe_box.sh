#!/bin/bash
# Box probe: host resources, PCIe/NVLink topology, pinned host<->device bandwidth.
set -x
nvidia-smi
nvidia-smi topo -m
nproc; python -c 'import os;print("affinity",len(os.sched_getaffinity(0)))'
free -g; cat /sys/fs/cgroup/memory.max 2>/dev/null; ulimit -l
lscpu | head -30
numactl -H 2>/dev/null
nvidia-smi -q | grep -i -A3 "PCIe Generation\|Link Width"
python - <<'PY'
import torch, time
d = torch.device('cuda:0')
for gb in [0.25, 1, 4]:
    n = int(gb*2**30)
    h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    g = torch.empty(n, dtype=torch.uint8, device=d)
    for name, fn in [('H2D', lambda: g.copy_(h, non_blocking=True)), ('D2H', lambda: h.copy_(g, non_blocking=True))]:
        fn(); torch.cuda.synchronize()
        e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True)
        e0.record(); 
        for _ in range(5): fn()
        e1.record(); torch.cuda.synchronize()
        print(name, gb, 'GiB', 5*n/ (e0.elapsed_time(e1)/1e3)/1e9, 'GB/s')
    # bidirectional
    h2 = torch.empty(n, dtype=torch.uint8, pin_memory=True); g2 = torch.empty(n, dtype=torch.uint8, device=d)
    s1=torch.cuda.Stream(); s2=torch.cuda.Stream(); torch.cuda.synchronize()
    t=time.time()
    for _ in range(5):
        with torch.cuda.stream(s1): g.copy_(h, non_blocking=True)
        with torch.cuda.stream(s2): h2.copy_(g2, non_blocking=True)
    torch.cuda.synchronize(); dt=time.time()-t
    print('BIDIR', gb, 'GiB', 2*5*n/dt/1e9, 'GB/s total')
t=time.time(); x = torch.empty(16*2**30, dtype=torch.uint8, pin_memory=True); print('pin 16GiB alloc s', time.time()-t)
PY
