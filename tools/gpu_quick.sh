#!/bin/bash
# quick GPU check of a subset: $1 = pytest args (default: the host-I/O tests), then (unless NOBENCH) the bench
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest ${1:-tests/test_gpu_hostio.py} -q -x 2>&1 | tail -15
[ -n "$NOBENCH" ] && exit 0
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench.log | python -c "
import json,sys; r=json.loads(sys.stdin.read()); print('value', round(r['value']), 'tflops', round(r['tflops_per_gpu'],1), 'e2e', r['e2e'], 'clk', r['clocks'])"
