set -x
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r01.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch_bench.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:attn_bwd_kernel -s 1 -c 1 -o gpurun_out/prof_bwd python bench.py --seq 131072 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_bwd.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:attn_fwd_kernel -s 1 -c 1 -o gpurun_out/prof_fwd python bench.py --seq 131072 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_fwd.log 2>&1
ls -la gpurun_out
