#!/bin/bash
# GPU test suite, then per-rank workloads of configs[2..4] on one B200 (tools/rank_workloads.py)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 600 python tools/rank_workloads.py --only c5 c3 --steps 2 > gpurun_out/rank_workloads.jsonl 2> gpurun_out/rank_workloads.err
echo "c3/c5 rc=$?"
timeout 1500 python tools/rank_workloads.py --only c4 --steps 1 ${C4_CHUNKS:+--chunks $C4_CHUNKS} >> gpurun_out/rank_workloads.jsonl 2>> gpurun_out/rank_workloads.err
echo "c4 rc=$?"
cut -c1-300 gpurun_out/rank_workloads.jsonl; tail -5 gpurun_out/rank_workloads.err
