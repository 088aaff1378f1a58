#!/bin/bash
# configs[3] per-rank chunk sweep, two steps each (the second is the steady state)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
rm -f gpurun_out/c4_steady.jsonl
timeout 2700 python tools/rank_workloads.py --only c4 --steps 2 > gpurun_out/c4_steady.jsonl 2> gpurun_out/c4_steady.err; echo "rc=$?"
python - <<'PY'
import json
for l in open('gpurun_out/c4_steady.jsonl'):
    r = json.loads(l)
    print(r['config'], r['chunk'], 'first %.1f s' % r['first_step_s'], 'steady %.1f s' % r['step_s'], 'TFLOPS/GPU %.0f' % r['tflops_per_gpu'],
          'fwd %.0f bwd %.0f' % (r['fwd_kernel_tflops'], r['bwd_kernel_tflops']), 'h2d %.1f GB/s d2h %.1f GB/s' % (r['h2d_GBps'], r['d2h_GBps']))
PY
tail -3 gpurun_out/c4_steady.err
