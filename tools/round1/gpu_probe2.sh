#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 600 python -m pytest tests/test_gpu_multirank.py -x -q > gpurun_out/pytest_multirank.log 2>&1; echo "multirank rc=$?"; tail -15 gpurun_out/pytest_multirank.log
timeout 300 python tools/microbench.py > gpurun_out/microbench.log 2>&1; echo "microbench rc=$?"; cat gpurun_out/microbench.log
timeout 300 python tools/trace_pair.py bwd 65536 32 80 100 > gpurun_out/trace_bwd.log 2>&1; cat gpurun_out/trace_bwd.log
timeout 300 python tools/trace_pair.py fwd 65536 32 80 100 > gpurun_out/trace_fwd.log 2>&1; cat gpurun_out/trace_fwd.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_bwd_kernel -s 1 -c 1 -o gpurun_out/prof_bwd3 python bench.py --seq 131072 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/ncu_bwd3.log 2>&1; echo "ncu rc=$?"
