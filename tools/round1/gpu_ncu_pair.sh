#!/bin/bash
# ncu --set full of one isolated pair kernel (tools/trace_pair.py launch): $1 = fwd|bwd, $2 = d, $3 = out name
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
K=${KREGEX:-attn_}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s 2 -c 1 -o gpurun_out/$3 python tools/trace_pair.py $1 65536 32 $2 100 > gpurun_out/$3.log 2>&1; echo "ncu rc=$?"; tail -3 gpurun_out/$3.log
