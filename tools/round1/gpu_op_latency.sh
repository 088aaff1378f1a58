#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
rm -f gpurun_out/op_latency.jsonl
timeout 300 python tools/op_latency.py --heads 4 --d 80 >> gpurun_out/op_latency.jsonl 2> gpurun_out/op_latency.err; echo "2.7B p=8 rc=$?"
timeout 300 python tools/op_latency.py --heads 32 --d 80 --lens 4096 16384 65536 >> gpurun_out/op_latency.jsonl 2>> gpurun_out/op_latency.err; echo "2.7B p=1 rc=$?"
timeout 300 python tools/op_latency.py --heads 8 --kv-heads 2 --d 128 >> gpurun_out/op_latency.jsonl 2>> gpurun_out/op_latency.err; echo "8B p=4 rc=$?"
python - <<'PY'
import json
for l in open('gpurun_out/op_latency.jsonl'):
    r = json.loads(l)
    print(r['heads_q'], r['heads_kv'], r['head_dim'], r['s'], 'fwd diag %.3f full %.3f bwd full %.3f | h2d qkv %.3f (%.1f GB/s) kv %.3f qside %.3f | ratios %.2f %.2f %.2f' % (
        r['attn_fwd_diag_ms'], r['attn_fwd_full_ms'], r['attn_bwd_full_ms'], r['h2d_qkv_ms'], r['h2d_qkv_GBps'],
        r['h2d_kv_fwd_ms'], r['h2d_q_side_bwd_ms'], r['attn_fwd_diag_over_h2d_qkv'], r['pair_fwd_over_kv_fetch'],
        r['pair_bwd_over_q_side_fetch']))
PY
tail -3 gpurun_out/op_latency.err
