#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 1200 python -m pytest tests/test_gpu_block.py tests/test_gpu_stress.py tests/test_gpu_fetch_strategy.py -q 2>&1 | tail -4
timeout 600 python tools/block_bench.py > gpurun_out/block_bench.log 2>&1; echo "block rc=$?"; tail -1 gpurun_out/block_bench.log | cut -c1-400
timeout 600 python tools/sdpa_context.py > gpurun_out/sdpa.jsonl 2>&1; echo "sdpa rc=$?"; cat gpurun_out/sdpa.jsonl | cut -c1-300
