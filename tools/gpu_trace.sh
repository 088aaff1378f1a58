#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 120 python tools/trace_pair.py fwd 65536 32 80 0 > gpurun_out/trace_fwd80.txt 2>&1
timeout 120 python tools/trace_pair.py fwd 65536 32 80 4000 > gpurun_out/trace_fwd80_mid.txt 2>&1
timeout 120 python tools/trace_pair.py fwd 65536 32 128 0 > gpurun_out/trace_fwd128.txt 2>&1
timeout 120 python tools/trace_pair.py bwd 65536 32 80 0 2 > gpurun_out/trace_bwd80.txt 2>&1
tail -3 gpurun_out/trace_fwd80.txt
