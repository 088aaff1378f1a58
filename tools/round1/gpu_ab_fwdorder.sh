#!/bin/bash
# (archived: the FPDT_FWD_MMA_ORDER variant was measured with it in round 2 and removed)
# same-box A/B/A/B: forward MMA issue order at d <= 80 (FPDT_FWD_MMA_ORDER 1: S_0(j+1), PV_1(j-1), S_1(j+1), PV_0(j);
# 0: S_0(j+1), S_1(j+1), PV_0(j), PV_1(j)); standalone C = 64K pair, 32 heads, d = 80 and 64, and in the bench step
mkdir -p gpurun_out
python -c "from paper_2408_16978_b200 import build; build.build_generator()" > /dev/null 2>&1
ab() {
  FPDT_NVCC_DEFINES="$1" python -c "from paper_2408_16978_b200 import build; build.build_product(force=True); build.build_diag(force=True)" > gpurun_out/build_ab.log 2>&1 || { tail -5 gpurun_out/build_ab.log; return; }
  for d in 80 64; do for i in 1 2; do echo "[$2] $(timeout 120 python tools/trace_pair.py fwd 65536 32 $d 0 1 x 2>&1 | tail -1)"; done; done
  if [ -n "$3" ]; then
    timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; r=json.loads(sys.stdin.read()); print('[$2 bench]', round(r['tflops_per_gpu'],1), 'bwd', round(r['roofline']['achieved'],1), 'fwd', round(r['roofline']['fwd_kernel']['achieved'],1), r['clocks']['sm_mhz'])"
  fi
}
ab "-DFPDT_FWD_MMA_ORDER=1" "new"
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_extreme.py tests/test_gpu_sparse.py -q -x -m gpu 2>&1 | tail -3
timeout 120 python tools/trace_pair.py fwd 65536 32 80 0 > gpurun_out/trace_fwd80_new.txt 2>&1; tail -16 gpurun_out/trace_fwd80_new.txt
ab "-DFPDT_FWD_MMA_ORDER=0" "old" bench
ab "-DFPDT_FWD_MMA_ORDER=1" "new" bench
ab "-DFPDT_FWD_MMA_ORDER=0" "old again"
