#!/bin/bash
# Per-rank workloads of configs[1..4] on one B200 (tools/rank_workloads.py, steady state) and the e2e probe.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python tools/e2e_probe.py > gpurun_out/e2e_probe.jsonl 2> gpurun_out/e2e_probe.err; echo "e2e probe rc=$?"; cat gpurun_out/e2e_probe.jsonl
rm -f gpurun_out/rank_workloads.jsonl
timeout 1200 python tools/rank_workloads.py --only c5 c3 --steps 2 --bwd-order auto >> gpurun_out/rank_workloads.jsonl 2>> gpurun_out/rank_workloads.err; echo "c3/c5 rc=$?"
timeout 1200 python tools/rank_workloads.py --only c2p8 --steps 2 >> gpurun_out/rank_workloads.jsonl 2>> gpurun_out/rank_workloads.err; echo "c2p8 rc=$?"
python - <<'PY'
import json
for l in open('gpurun_out/rank_workloads.jsonl'):
    r = json.loads(l)
    print(r['config'], r.get('chunk'), r.get('bwd_order'), 'step %.2f s' % r['step_s'], 'TFLOPS/GPU %.0f' % r['tflops_per_gpu'])
PY
