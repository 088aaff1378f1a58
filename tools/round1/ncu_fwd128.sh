#!/bin/bash
# ncu --set full of the d = 128 forward pair kernel at the c3 per-rank shape (8 q / 8 kv heads used here, C = 64K,
# full pair via tools/op_latency-style direct launch through fpdt_debug_pair)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_fwd -s 2 -c 1 -o gpurun_out/prof_fwd128 \
  python tools/trace_pair.py fwd 65536 8 128 0 > gpurun_out/ncu_fwd128.log 2>&1; echo "ncu fwd128 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_bwd -s 2 -c 1 -o gpurun_out/prof_bwd128 \
  python tools/trace_pair.py bwd 65536 8 128 0 > gpurun_out/ncu_bwd128.log 2>&1; echo "ncu bwd128 rc=$?"
ls -la gpurun_out/*.ncu-rep
