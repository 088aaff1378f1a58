#!/bin/bash
# configs[1] under HBM residency budgets: tokens/s, host bytes, library device bytes -> gpurun_out/residency.jsonl
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
: > gpurun_out/residency.jsonl
for r in "0 0" "2 2" "4 4" "8 8"; do
  timeout 600 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --residency $r >> gpurun_out/residency.jsonl 2> gpurun_out/residency.err; echo "res $r rc=$?"
done
timeout 600 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --offload 0 >> gpurun_out/residency.jsonl 2>> gpurun_out/residency.err; echo "offload0 rc=$?"
python - <<'PY'
import json
for l in open("gpurun_out/residency.jsonl"):
    r = json.loads(l)
    print(r["config"]["residency"], r["config"]["offload"], round(r["value"]), round(r["tflops_per_gpu"]), r["pcie_bytes_per_step"], r["device_bytes_library"])
PY
