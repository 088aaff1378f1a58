#!/bin/bash
# Per-rank workloads of configs[2..4] on one B200 (tools/rank_workloads.py) -> gpurun_out/rank_workloads.jsonl
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 600 python tools/rank_workloads.py --only c5 c3 --steps 2 > gpurun_out/rank_workloads.jsonl 2> gpurun_out/rank_workloads.err
echo "c3/c5 rc=$?"
timeout 1500 python tools/rank_workloads.py --only c4 --steps 1 >> gpurun_out/rank_workloads.jsonl 2>> gpurun_out/rank_workloads.err
echo "c4 rc=$?"
cat gpurun_out/rank_workloads.jsonl | cut -c1-400; tail -5 gpurun_out/rank_workloads.err
