#!/bin/bash
# One-box validation on a B200: build, GPU tests (optionally a subset: $1 = pytest args), smoke, bench, block bench,
# overlap probe.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 2400 python -m pytest ${1:-tests} -q -m gpu --durations=10 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -16 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
[ -n "$NOBENCH" ] && exit 0
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench.log | cut -c1-400
timeout 600 python tools/block_bench.py > gpurun_out/block_bench.log 2>&1; echo "block rc=$?"; tail -1 gpurun_out/block_bench.log | cut -c1-300
timeout 900 python tools/overlap_probe.py > gpurun_out/overlap.jsonl 2> gpurun_out/overlap.err; echo "overlap rc=$?"
timeout 900 python tools/e2e_probe.py --one-set --steps 3 > gpurun_out/e2e_probe.jsonl 2> gpurun_out/e2e_probe.err; echo "e2e probe rc=$?"
