#!/bin/bash
# Q-outer backward (fpdt_set_bwd_order): its GPU tests, then c3/c5 per-rank workloads in both orders
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_bwd_order.py tests/test_gpu_residency.py tests/test_gpu_multirank.py -x -q -m gpu > gpurun_out/pytest_bwd_order.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_bwd_order.log
for o in q kv; do
  timeout 600 python tools/rank_workloads.py --only c5 c3 --steps 2 --bwd-order $o >> gpurun_out/rank_workloads_order.jsonl 2>> gpurun_out/rank_workloads_order.err
  echo "order $o rc=$?"
done
cut -c1-400 gpurun_out/rank_workloads_order.jsonl; tail -5 gpurun_out/rank_workloads_order.err
