#!/bin/bash
# setmaxnreg splits of the d = 80 pair kernels (C = 64K, 32-head diagonal pairs)
mkdir -p gpurun_out
run() {
  FPDT_NVCC_DEFINES="$1" python -c "from paper_2408_16978_b200 import build; build.build_product(force=True)" > gpurun_out/build_rg.log 2>&1 || { tail -5 gpurun_out/build_rg.log; return; }
  for rep in 1 2 3; do
    echo -n "[$1] rep=$rep: "; timeout 120 python tools/trace_pair.py $2 65536 32 80 0 2>&1 | head -1
  done
}
run "" fwd
run "-DFPDT_FWD_REGS_SOFTMAX=208 -DFPDT_FWD_REGS_OTHER=88" fwd
run "" bwd
run "-DFPDT_BWD_REGS_SOFTMAX=176 -DFPDT_BWD_REGS_DQ=96 -DFPDT_BWD_REGS_CTL=64" bwd
run "-DFPDT_BWD_REGS_SOFTMAX=160 -DFPDT_BWD_REGS_DQ=120 -DFPDT_BWD_REGS_CTL=72" bwd
python -c "from paper_2408_16978_b200 import build; build.build_product(force=True)" > /dev/null 2>&1
