#!/bin/bash
# setmaxnreg splits of the d = 128 q64 backward (C = 64K, 32-head diagonal pair) and its exponential split
mkdir -p gpurun_out
run() {
  FPDT_NVCC_DEFINES="$1" python -c "from paper_2408_16978_b200 import build; build.build_product(force=True)" > gpurun_out/build_rg.log 2>&1 || { tail -5 gpurun_out/build_rg.log; return; }
  for rep in 1 2 3; do
    echo -n "[$1] rep=$rep: "; timeout 120 python tools/trace_pair.py bwd 65536 32 128 0 2>&1 | head -1
  done
}
run ""
run "-DFPDT_Q64_REGS_SOFTMAX=176 -DFPDT_Q64_REGS_DQ=96 -DFPDT_Q64_REGS_CTL=64"
run "-DFPDT_Q64_REGS_SOFTMAX=160 -DFPDT_Q64_REGS_DQ=120 -DFPDT_Q64_REGS_CTL=72"
run "-DFPDT_Q64_REGS_SOFTMAX=184 -DFPDT_Q64_REGS_DQ=88 -DFPDT_Q64_REGS_CTL=56"
python -c "from paper_2408_16978_b200 import build; build.build_product(force=True)" > /dev/null 2>&1
