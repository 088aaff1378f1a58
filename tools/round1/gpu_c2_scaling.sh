#!/bin/bash
# compute side of configs[1]'s strong scaling: the per-rank work at p = 1, 2, 4, 8 on one B200
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
rm -f gpurun_out/c2_scaling.jsonl
timeout 1200 python tools/rank_workloads.py --only c2p1 c2p2 c2p4 c2p8 --steps 3 > gpurun_out/c2_scaling.jsonl 2> gpurun_out/c2_scaling.err; echo "rc=$?"
python - <<'PY'
import json
rows = [json.loads(l) for l in open('gpurun_out/c2_scaling.jsonl')]
t1 = rows[0]['step_s']
for r in rows:
    p = r['world_size_emulated']
    print(r['config'], p, 'step %.3f s' % r['step_s'], 'TFLOPS/GPU %.1f' % r['tflops_per_gpu'],
          'fwd %.0f bwd %.0f' % (r['fwd_kernel_tflops'], r['bwd_kernel_tflops']), 'eff %.3f' % (t1 / (p * r['step_s'])))
PY
tail -3 gpurun_out/c2_scaling.err
