#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python bench.py ${BENCH_ARGS} > gpurun_out/bench.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/bench.log | python -c "
import json,sys; r=json.loads(sys.stdin.read()); print({k:r[k] for k in ['value','ms_per_step','tflops_per_gpu']}, r['e2e']['value'], r['e2e']['ms_per_step'], r['clocks'])"
