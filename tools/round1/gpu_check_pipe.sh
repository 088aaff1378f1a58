#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kernel_variants.py tests/test_gpu_fullsize.py tests/test_gpu_sparse.py -q -m gpu > gpurun_out/pytest_pipe.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_pipe.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/bench.log | python -c "
import json,sys; r=json.loads(sys.stdin.read()); print({k:r[k] for k in ['value','ms_per_step','tflops_per_gpu']}, 'bwd', r['roofline']['achieved'], 'fwd', r['roofline']['fwd_kernel']['achieved'], 'e2e', r['e2e']['value'], r['clocks'])"
