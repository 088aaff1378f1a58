#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_kernel_variants.py -q 2>&1 | tail -5
for k in 2 5 3; do timeout 120 python tools/trace_pair.py bwd 65536 32 80 0 $k x 2>&1 | tail -1; done
for k in 2 5 3; do timeout 120 python tools/trace_pair.py bwd 65536 32 64 0 $k x 2>&1 | tail -1; done
timeout 120 python tools/trace_pair.py bwd 65536 32 80 0 5 2>&1 | tail -16
