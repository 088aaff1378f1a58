#!/bin/bash
# backward exponential split sweep: FPDT_BWD_POLY_EVERY (one exponential pair in N on the FMA-pipe polynomial; 0 = all
# MUFU); the C = 64K, 32-head diagonal pair via tools/trace_pair.py, d = 80 (pipe kernel) and d = 128 (q64 kernel)
mkdir -p gpurun_out
for pe in 4 8 16 0; do
  FPDT_NVCC_DEFINES="-DFPDT_BWD_POLY_EVERY=$pe" python -c "from paper_2408_16978_b200 import build; build.build_product(force=True)" > gpurun_out/build_pe$pe.log 2>&1 || { tail -5 gpurun_out/build_pe$pe.log; exit 1; }
  for rep in 1 2; do
    echo -n "poly_every=$pe rep=$rep: "; timeout 120 python tools/trace_pair.py bwd 65536 32 80 0 2>&1 | head -1
    echo -n "poly_every=$pe rep=$rep: "; timeout 120 python tools/trace_pair.py bwd 65536 32 128 0 2>&1 | head -1
  done
done
python -c "from paper_2408_16978_b200 import build; build.build_product(force=True)" > /dev/null 2>&1
