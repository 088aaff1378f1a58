#!/bin/bash
# same-box A/B/A inside the bench step: forward K/V ring depth at d = 80 (FPDT_FWD_STAGES 3 vs 4)
mkdir -p gpurun_out
python -c "from paper_2408_16978_b200 import build; build.build_generator()" > /dev/null 2>&1
bench() {
  FPDT_NVCC_DEFINES="$1" python -c "from paper_2408_16978_b200 import build; build.build_product(force=True)" > gpurun_out/build_ab.log 2>&1 || { tail -5 gpurun_out/build_ab.log; return; }
  timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; r=json.loads(sys.stdin.read()); print('[$2]', round(r['tflops_per_gpu'],1), 'bwd', round(r['roofline']['achieved'],1), 'fwd', round(r['roofline']['fwd_kernel']['achieved'],1), r['clocks']['sm_mhz'])"
}
bench "" "stages 3"
bench "-DFPDT_FWD_STAGES=4" "stages 4"
bench "" "stages 3 again"
bench "-DFPDT_FWD_STAGES=4" "stages 4 again"
