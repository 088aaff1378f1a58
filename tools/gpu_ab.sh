#!/bin/bash
# Same-box A/B of compile-time kernel variants: for each ';'-separated define set in $VARIANTS, rebuild, print the
# oracle errors at d = $D (default 80; unless NOERR) and the standalone C = 64K, 32 x d pair speeds (backward kernel $K,
# default 2 = pipe; 1 = dispatch) (causal diagonal pair and a
# full pair, forward and backward).
mkdir -p gpurun_out
IFS=';' read -ra VS <<< "${VARIANTS:-}"
i=0
for V in "${VS[@]}"; do
  i=$((i+1))
  FPDT_NVCC_DEFINES="$V" python -c "from paper_2408_16978_b200 import build as b; b.build_all(force=True)" > gpurun_out/build_ab_$i.log 2>&1 || { echo "build [$V] failed"; tail -20 gpurun_out/build_ab_$i.log; continue; }
  echo "== [$V]"
  [ -z "$NOERR" ] && timeout 300 python tools/err_report.py ${D:-80} 2>&1 | tail -7
  for which in ${WHICH:-fwd bwd}; do
    for c in 1 0; do
      CAUSAL=$c timeout 120 python tools/trace_pair.py $which 65536 32 ${D:-80} 0 ${K:-2} x 2>&1 | tail -1
    done
  done
done
