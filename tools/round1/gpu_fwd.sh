#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 240 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pytest_parity.log 2>&1; echo "parity rc=$?"; tail -4 gpurun_out/pytest_parity.log
for d in 80 64 128; do timeout 60 python tools/trace_pair.py fwd 65536 32 $d 100 > gpurun_out/trace_fwd$d.log 2>&1; head -1 gpurun_out/trace_fwd$d.log; done
grep -v "^it " gpurun_out/trace_fwd80.log | tail -16
