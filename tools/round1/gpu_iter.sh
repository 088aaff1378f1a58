#!/bin/bash
# Iteration loop on the GPU: build, bf16 parity subset, pair-kernel traces, short bench.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_parity.log 2>&1; echo "parity rc=$?"; tail -15 gpurun_out/pytest_parity.log
timeout 120 python tools/trace_pair.py bwd 65536 32 80 100 > gpurun_out/trace_bwd.log 2>&1; echo "trace rc=$?"; cat gpurun_out/trace_bwd.log
timeout 120 env FPDT_BWD_KERNEL=v2 python tools/trace_pair.py bwd 65536 32 80 100 2>&1 | head -1
timeout 120 python tools/trace_pair.py bwd 65536 32 64 100 2>&1 | head -1
if [ -n "$RUN_BENCH" ]; then timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench.log; fi
timeout 120 env FPDT_BWD_DQ=red python tools/trace_pair.py bwd 65536 32 80 100 > gpurun_out/trace_bwd_red.log 2>&1; echo "red:"; grep -v "^it " gpurun_out/trace_bwd_red.log
