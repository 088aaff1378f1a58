#!/bin/bash
# build + full GPU test suite + bwd trace (d=80, d=64) + fwd timing
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/pytest_gpu.log
timeout 120 python tools/trace_pair.py bwd 65536 32 80 100 > gpurun_out/trace_bwd.log 2>&1; grep -v "^it " gpurun_out/trace_bwd.log
timeout 120 python tools/trace_pair.py bwd 65536 32 64 100 2>&1 | head -1
timeout 120 python tools/trace_pair.py fwd 65536 32 80 100 2>&1 | head -1
if [ -n "$RUN_BENCH" ]; then timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench.log; fi
