for V in ${VARIANTS:-"-DFPDT_FWD_THROTTLE=0"}; do
  FPDT_NVCC_DEFINES="$V" python -c "from paper_2408_16978_b200 import build as b; b.build_all(force=True)" > /dev/null 2>&1 || { echo "build $V failed"; continue; }
  echo "== $V"
  python tools/trace_pair.py fwd 65536 32 80 0 | grep -v "^it "
  CAUSAL=0 python tools/trace_pair.py fwd 65536 32 80 0 1 x | tail -1
done
