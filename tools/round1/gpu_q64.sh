#!/bin/bash
# attn_bwd_q64_kernel at d = 64/80/128: parity (forced for every head_dim), then pair-kernel speed vs attn_bwd_pipe
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
FPDT_BWD_KERNEL=q64 timeout 300 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pytest_q64.log 2>&1; echo "parity(q64 all d) rc=$?"; tail -15 gpurun_out/pytest_q64.log
for d in 128 80 64; do
  timeout 60 env FPDT_BWD_KERNEL=q64 python tools/trace_pair.py bwd 65536 32 $d 100 2>&1 | head -1
done
timeout 60 env FPDT_BWD_KERNEL=q64 python tools/trace_pair.py bwd 65536 8 128 100 2>&1 | head -1
