#!/bin/bash
# (archived: the FPDT_PIPE_RING / FPDT_PIPE_QS64 variants were measured with it in round 2 and removed, see the
# PipeCfg comment in attn_bwd_pipe_sm100.cu)
# same-box A/B/A/B: backward pipe kernel, Q ring depth 2 + 2 x 20 KB dQ staging (default) against 3 Q stages + an
# R-slot 16-column dQ staging ring (FPDT_PIPE_RING=1); standalone C = 64K diagonal pair, 32 heads, d = 80 and 64;
# parity of the ring variant through the kernel-variant / parity tests
mkdir -p gpurun_out
python -c "from paper_2408_16978_b200 import build; build.build_generator()" > /dev/null 2>&1
ab() {
  FPDT_NVCC_DEFINES="$1" python -c "from paper_2408_16978_b200 import build; build.build_product(force=True); build.build_diag(force=True)" > gpurun_out/build_ab.log 2>&1 || { tail -5 gpurun_out/build_ab.log; return; }
  for d in 80 64; do for i in 1 2 3; do echo "[$2] $(timeout 120 python tools/trace_pair.py bwd 65536 32 $d 0 2 x 2>&1 | tail -1)"; done; done
}
ab "" "default"
ab "-DFPDT_PIPE_RING=1" "ring"
timeout 900 python -m pytest tests/test_gpu_kernel_variants.py tests/test_gpu_parity.py tests/test_gpu_extreme.py -q -x -m gpu 2>&1 | tail -3
timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; r=json.loads(sys.stdin.read()); print('[ring bench]', round(r['tflops_per_gpu'],1), 'bwd', round(r['roofline']['achieved'],1), 'fwd', round(r['roofline']['fwd_kernel']['achieved'],1), r['clocks']['sm_mhz'])"
ab "" "default again"
timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; r=json.loads(sys.stdin.read()); print('[default bench]', round(r['tflops_per_gpu'],1), 'bwd', round(r['roofline']['achieved'],1), 'fwd', round(r['roofline']['fwd_kernel']['achieved'],1), r['clocks']['sm_mhz'])"
ab "-DFPDT_PIPE_RING=1" "ring again"
