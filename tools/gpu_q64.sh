#!/bin/bash
# d = 128 backward (attn_bwd_q64_kernel): parity, then pair-kernel speed vs the atomics kernel
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "128" > gpurun_out/pytest_q64.log 2>&1; echo "parity128 rc=$?"; tail -15 gpurun_out/pytest_q64.log
timeout 60 python tools/trace_pair.py bwd 65536 32 128 100 2>&1 | head -1
timeout 60 env FPDT_BWD_KERNEL=v2 python tools/trace_pair.py bwd 65536 32 128 100 2>&1 | head -1
timeout 60 python tools/trace_pair.py bwd 65536 8 128 100 2>&1 | head -1
