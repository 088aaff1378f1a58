#!/bin/bash
# One-box round validation + evidence: build, every GPU test, smoke, the default bench line, then the ncu launch list of
# the bench command and ncu --set full of the backward and forward pair kernels at the bench's launch shape.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests -q -m gpu --durations=10 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench.log | cut -c1-300
[ -n "$NONCU" ] && exit 0
timeout 900 python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/plain_launch.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch_bench.log 2>&1; echo "ncu launches rc=$?"
timeout 900 python bench.py --seq 131072 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/plain_small.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_bwd -s 1 -c 1 -o gpurun_out/prof_bwd_bench \
  python bench.py --seq 131072 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/ncu_bwd_bench.log 2>&1; echo "ncu bwd rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_fwd -s 1 -c 1 -o gpurun_out/prof_fwd_bench \
  python bench.py --seq 131072 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/ncu_fwd_bench.log 2>&1; echo "ncu fwd rc=$?"
