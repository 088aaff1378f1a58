#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
show() { python -c "
import json,sys
for l in open('$1'):
    try: d=json.loads(l)
    except Exception: continue
    print('$2', d.get('variant','bench'), d.get('steps'), round(d['ms_per_step'],1), d['clocks'])"; }
timeout 900 python tools/e2e_probe.py --one-set --steps 4 --variants none --warmup-copies 0 --no-pinned > gpurun_out/p1.jsonl 2>&1; show gpurun_out/p1.jsonl nocopy_nopinned
timeout 900 python tools/e2e_probe.py --one-set --steps 4 --variants none --warmup-copies 0 > gpurun_out/p2.jsonl 2>&1; show gpurun_out/p2.jsonl nocopy_pinned
timeout 900 python tools/e2e_probe.py --one-set --steps 4 --variants none --warmup-copies 1 > gpurun_out/p3.jsonl 2>&1; show gpurun_out/p3.jsonl copy_pinned
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_a.log 2>&1; tail -1 gpurun_out/bench_a.log > gpurun_out/b.jsonl; show gpurun_out/b.jsonl bench_with_e2e
