#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck on configs[0] shapes; logs to gpurun_out/sanitizer_*.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck synccheck racecheck; do
  for w in bf16 fp32 p2; do
    timeout 1200 $CS --tool $tool --error-exitcode 9 --print-limit 50 python tools/sanitize_run.py $w \
      > gpurun_out/sanitizer_${tool}_${w}.log 2>&1
    echo "$tool $w rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|ok$" gpurun_out/sanitizer_${tool}_${w}.log | tail -3
  done
done
