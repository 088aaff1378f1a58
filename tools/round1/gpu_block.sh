#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_block.py -q -m gpu -x > gpurun_out/pytest_block.log 2>&1; echo "pytest rc=$?"; tail -30 gpurun_out/pytest_block.log
