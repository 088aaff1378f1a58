#!/bin/bash
# Round evidence on one B200: bench line, ncu launch list of the bench command, ncu --set full of the dominant
# (backward pair) and forward pair kernels in the bench's launch configuration.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch_bench.log 2>&1; echo "ncu launches rc=$?"
# bwd pair kernel: skip the diagonal (0,0) launch of the first step -> the full (1,0) pair, as in the bench
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_bwd -s 1 -c 1 -o gpurun_out/prof_bwd_bench \
  python bench.py --seq 131072 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/ncu_bwd_bench.log 2>&1; echo "ncu bwd rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_fwd -s 1 -c 1 -o gpurun_out/prof_fwd_bench \
  python bench.py --seq 131072 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/ncu_fwd_bench.log 2>&1; echo "ncu fwd rc=$?"
timeout 120 python tools/trace_pair.py bwd 65536 32 128 100 2>&1 | head -1
timeout 120 python tools/trace_pair.py fwd 65536 32 128 100 2>&1 | head -1
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
