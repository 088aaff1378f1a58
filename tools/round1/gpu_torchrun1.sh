#!/bin/bash
# the driver's launch path at N=1 through torchrun, and the bench flags
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_bwd_order.py -q -m gpu -k multirank > gpurun_out/pytest_qo8.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_qo8.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_torchrun1.log 2>&1; echo "torchrun rc=$?"
tail -1 gpurun_out/bench_torchrun1.log | cut -c1-200
timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --bwd-order auto --residency 2 2 > gpurun_out/bench_flags.log 2>&1; echo "flags rc=$?"
tail -1 gpurun_out/bench_flags.log | cut -c1-200
