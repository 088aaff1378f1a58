#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
for d in 128 64; do
timeout 60 env FPDT_BWD_KERNEL=q64 python tools/trace_pair.py bwd 65536 32 $d 100 > gpurun_out/trace_q64_$d.log 2>&1; head -1 gpurun_out/trace_q64_$d.log; grep -v "^it " gpurun_out/trace_q64_$d.log | tail -16
done
