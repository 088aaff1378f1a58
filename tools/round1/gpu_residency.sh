#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 600 python -m pytest tests/test_gpu_residency.py tests/test_gpu_multirank.py tests/test_gpu_parity.py tests/test_gpu_sparse.py -x -q > gpurun_out/pytest_res.log 2>&1; echo "rc=$?"; tail -25 gpurun_out/pytest_res.log
