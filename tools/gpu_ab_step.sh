#!/bin/bash
# Same-box A/B of compile-time variants inside the bench step: for each ';'-separated define set in $VARIANTS, rebuild
# and run the default bench configuration (no e2e, no CPU baseline); print step TFLOPS/GPU, the pair kernels' in-step
# TFLOP/s and the clock.
mkdir -p gpurun_out
IFS=';' read -ra VS <<< "${VARIANTS:-}"
for V in "${VS[@]}"; do
  FPDT_NVCC_DEFINES="$V" python -c "from paper_2408_16978_b200 import build as b; b.build_all(force=True)" > /dev/null 2>&1 || { echo "build [$V] failed"; continue; }
  timeout 600 python bench.py --steps ${STEPS:-3} --no-e2e --no-cpu-baseline > gpurun_out/ab_step.log 2>&1 || { echo "bench [$V] failed"; tail -3 gpurun_out/ab_step.log; continue; }
  tail -1 gpurun_out/ab_step.log | python -c "
import json,sys; r=json.loads(sys.stdin.read()); rf=r['roofline']
print('[$V] step %.1f TFLOPS/GPU  bwd %.1f  fwd %.1f  sm %s MHz' % (r['tflops_per_gpu'], rf['achieved'], rf['fwd_kernel']['achieved'], r['clocks']['sm_mhz']))"
done
