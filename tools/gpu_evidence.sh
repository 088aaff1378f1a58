#!/bin/bash
# Round evidence on one B200: bench line, ncu launch list of the bench command, ncu --set full of the backward and
# forward pair kernels (the full (1,0) chunk pair at the bench's launch shape) and of the projection GEMM.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python bench.py --steps 5 > gpurun_out/bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench.log | cut -c1-300
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch_bench.log 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_bwd -s 1 -c 1 -o gpurun_out/prof_bwd_bench \
  python bench.py --seq 131072 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/ncu_bwd_bench.log 2>&1; echo "ncu bwd rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_fwd -s 1 -c 1 -o gpurun_out/prof_fwd_bench \
  python bench.py --seq 131072 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/ncu_fwd_bench.log 2>&1; echo "ncu fwd rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_bf16 -s 2 -c 1 -o gpurun_out/prof_gemm \
  python tools/block_bench.py --seq 131072 --steps 1 --warmup 0 > gpurun_out/ncu_gemm.log 2>&1; echo "ncu gemm rc=$?"
