#!/bin/bash
# forward K/V ring depth at d = 80 (FPDT_FWD_STAGES), C = 64K 32-head diagonal pair
mkdir -p gpurun_out
for st in 3 4 2; do
  FPDT_NVCC_DEFINES="-DFPDT_FWD_STAGES=$st" python -c "from paper_2408_16978_b200 import build; build.build_product(force=True)" > gpurun_out/build_st.log 2>&1 || { tail -5 gpurun_out/build_st.log; exit 1; }
  for rep in 1 2 3; do
    echo -n "fwd d80 stages=$st rep=$rep: "; timeout 120 python tools/trace_pair.py fwd 65536 32 80 0 2>&1 | head -1
  done
done
python -c "from paper_2408_16978_b200 import build; build.build_product(force=True)" > /dev/null 2>&1
