#!/bin/bash
# same-box A/B on the c5 per-rank workload (8 q / 1 kv head, d = 128, S = 1M, Q-outer): exponential splits at d = 128
mkdir -p gpurun_out
python -c "from paper_2408_16978_b200 import build; build.build_generator()" > /dev/null 2>&1
run() {
  FPDT_NVCC_DEFINES="$1" python -c "from paper_2408_16978_b200 import build; build.build_product(force=True)" > gpurun_out/build_ab.log 2>&1 || { tail -5 gpurun_out/build_ab.log; return; }
  timeout 300 python tools/rank_workloads.py --only c5 --steps 2 --bwd-order q 2>/dev/null | python -c "
import json,sys; r=json.loads(sys.stdin.read()); print('[$2]', 'step %.3f s' % r['step_s'], 'TFLOPS/GPU %.1f' % r['tflops_per_gpu'], 'fwd %.0f' % r['fwd_kernel_tflops'])"
}
run "" "final: fwd 1/8, q64 bwd 1/4"
run "-DFPDT_FWD_POLY_EVERY_D128=4" "fwd 1/4"
run "-DFPDT_BWD_POLY_EVERY=0" "q64 bwd all-MUFU (and pipe)"
run "" "final again"
