#!/bin/bash
# Why the bench step and the e2e probe's device-only loop differ: same box, back to back, clocks sampled in each.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python bench.py --steps 5 --no-e2e --no-cpu-baseline > gpurun_out/bench_a.log 2>&1; tail -1 gpurun_out/bench_a.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench timing on', d['ms_per_step'], d['clocks'])"
timeout 900 python bench.py --steps 5 --no-e2e --no-cpu-baseline --no-kernel-timing > gpurun_out/bench_b.log 2>&1; tail -1 gpurun_out/bench_b.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench timing off', d['ms_per_step'], d['clocks'])"
timeout 900 python tools/e2e_probe.py > gpurun_out/e2e_probe2.jsonl 2>&1; python -c "
import json
for l in open('gpurun_out/e2e_probe2.jsonl'):
    try: d=json.loads(l)
    except Exception: print(l.strip()); continue
    print(d['variant'], round(d['ms_per_step'],1), d['clocks'])"
