#!/bin/bash
# PAPER.md Table "MFU at different attention sparsity" on B200: 2.7B shape (32 x 80), S = 256K, chunk 64K, 1 GPU.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
: > gpurun_out/sparsity_sweep.jsonl
for rho in 0.5 0.4 0.3 0.2 0.1 0.0; do
  timeout 600 python bench.py --seq 262144 --sparsity $rho --steps 3 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 >> gpurun_out/sparsity_sweep.jsonl
done
python - <<'PY'
import json
for l in open("gpurun_out/sparsity_sweep.jsonl"):
    d = json.loads(l)
    print(f"rho={d['config']['sparsity']:.1f}  {d['tflops_per_gpu']:7.1f} TFLOPS/GPU  frac_of_peak(sustained)={d['frac_of_peak']:.3f}  {d['value']:9.0f} tok/s  h2d {d['host_link']['h2d_GBps']:.1f} GB/s")
PY
