#!/bin/bash
# forward exponential split sweep: FPDT_FWD_POLY_EVERY (d <= 80) / FPDT_FWD_POLY_EVERY_D128 (one pair in N on the
# FMA-pipe polynomial, 0 = all MUFU); C = 64K, 32-head diagonal pair via tools/trace_pair.py
mkdir -p gpurun_out
for pe in "5 8" "4 16" "5 0" "6 12"; do
  set -- $pe
  FPDT_NVCC_DEFINES="-DFPDT_FWD_POLY_EVERY=$1 -DFPDT_FWD_POLY_EVERY_D128=$2" python -c "from paper_2408_16978_b200 import build; build.build_product(force=True)" > gpurun_out/build_fpe.log 2>&1 || { tail -5 gpurun_out/build_fpe.log; exit 1; }
  for rep in 1 2; do
    echo -n "fwd d80 every=$1 rep=$rep: "; timeout 120 python tools/trace_pair.py fwd 65536 32 80 0 2>&1 | head -1
    echo -n "fwd d128 every=$2 rep=$rep: "; timeout 120 python tools/trace_pair.py fwd 65536 32 128 0 2>&1 | head -1
  done
done
python -c "from paper_2408_16978_b200 import build; build.build_product(force=True)" > /dev/null 2>&1
