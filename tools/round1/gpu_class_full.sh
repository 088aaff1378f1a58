#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_fullsize_class.py -q -m gpu --durations=2 -s > gpurun_out/pytest_class.log 2>&1; echo "pytest rc=$?"; tail -12 gpurun_out/pytest_class.log
