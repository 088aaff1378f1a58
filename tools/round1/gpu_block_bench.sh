#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 600 python tools/block_bench.py --steps 2 --warmup 1 > gpurun_out/block_bench.jsonl 2> gpurun_out/block_bench.err; echo "rc=$?"
cat gpurun_out/block_bench.jsonl; tail -5 gpurun_out/block_bench.err
