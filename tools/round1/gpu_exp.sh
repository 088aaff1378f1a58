#!/bin/bash
# timing experiments: rebuild with each define set, trace the bwd pair kernel (results are NOT checked)
for defs in "$@"; do
  rm -rf paper_2408_16978_b200/build paper_2408_16978_b200/libfpdt.so
  FPDT_NVCC_DEFINES="$defs" python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || { echo "build failed: $defs"; continue; }
  echo "=== $defs"; timeout 120 python tools/trace_pair.py ${TRACE_ARGS:-bwd 65536 32 80 100} 2>&1 | grep -v "^it "
done
rm -rf paper_2408_16978_b200/build paper_2408_16978_b200/libfpdt.so
