#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
rm -f gpurun_out/rank_c3c5.jsonl
for o in auto kv; do
  timeout 600 python tools/rank_workloads.py --only c5 c3 --steps 2 --bwd-order $o >> gpurun_out/rank_c3c5.jsonl 2>> gpurun_out/rank_c3c5.err; echo "order $o rc=$?"
done
python - <<'PY'
import json
for l in open('gpurun_out/rank_c3c5.jsonl'):
    r = json.loads(l)
    print(r['config'], r.get('bwd_order'), 'step %.2f s' % r['step_s'], 'TFLOPS/GPU %.0f' % r['tflops_per_gpu'], 'fwd %.0f' % r['fwd_kernel_tflops'], 'h2d %.0f GB' % (r['h2d_bytes'] / 1e9))
PY
