#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_bwd_order.py tests/test_gpu_multirank.py tests/test_gpu_residency.py tests/test_gpu_sparse.py -q -m gpu > gpurun_out/pytest_bwd_order.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_bwd_order.log
