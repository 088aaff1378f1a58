#!/bin/bash
# Q-outer backward with two compute streams: its GPU tests, then c5/c3 per-rank workloads: Q-outer 2 streams,
# Q-outer 1 stream, KV-outer (paper)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_bwd_order.py -x -q -m gpu > gpurun_out/pytest_bwd_order.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_bwd_order.log
FPDT_BWD_QO_STREAMS=1 timeout 600 python -m pytest tests/test_gpu_bwd_order.py -x -q -m gpu -k "matches or multirank" > gpurun_out/pytest_bwd_order1.log 2>&1; echo "pytest (1 stream) rc=$?"; tail -2 gpurun_out/pytest_bwd_order1.log
rm -f gpurun_out/rank_workloads_order2.jsonl
timeout 400 python tools/rank_workloads.py --only c5 c3 --steps 2 --bwd-order q >> gpurun_out/rank_workloads_order2.jsonl 2>> gpurun_out/rank_workloads_order2.err; echo "q2 rc=$?"
FPDT_BWD_QO_STREAMS=1 timeout 400 python tools/rank_workloads.py --only c5 --steps 2 --bwd-order q >> gpurun_out/rank_workloads_order2.jsonl 2>> gpurun_out/rank_workloads_order2.err; echo "q1 rc=$?"
python - <<'PY'
import json
for l in open('gpurun_out/rank_workloads_order2.jsonl'):
    r = json.loads(l)
    print(r['config'], r.get('bwd_order'), round(r['step_s'], 3), round(r['tflops_per_gpu'], 1), 'bwd', round(r['bwd_kernel_tflops'], 1), 'h2d GB', round(r['h2d_bytes'] / 1e9, 1))
PY
tail -3 gpurun_out/rank_workloads_order2.err
