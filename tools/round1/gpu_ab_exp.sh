#!/bin/bash
# same-box A/B/A of the exponential splits inside the bench step (device-timed, no e2e / cpu baseline)
mkdir -p gpurun_out
bench() {
  FPDT_NVCC_DEFINES="$1" python -c "from paper_2408_16978_b200 import build; build.build_product(force=True)" > gpurun_out/build_ab.log 2>&1 || { tail -5 gpurun_out/build_ab.log; return; }
  python -c "from paper_2408_16978_b200 import build; build.build_generator()" > /dev/null 2>&1
  timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; r=json.loads(sys.stdin.read()); print('[$2]', round(r['tflops_per_gpu'],1), 'bwd', round(r['roofline']['achieved'],1), 'fwd', round(r['roofline']['fwd_kernel']['achieved'],1), r['clocks']['sm_mhz'])"
}
bench "" "final: fwd 1/5, bwd all-MUFU"
bench "-DFPDT_FWD_POLY_EVERY=4 -DFPDT_BWD_POLY_EVERY=4" "v9: fwd 1/4, bwd 1/4"
bench "" "final again"
bench "-DFPDT_FWD_POLY_EVERY=4 -DFPDT_BWD_POLY_EVERY=4" "v9 again"
python -c "from paper_2408_16978_b200 import build; build.build_product(force=True)" > /dev/null 2>&1
