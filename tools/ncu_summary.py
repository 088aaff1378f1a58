#!/usr/bin/env python
"""Summarise ncu captures for profiles/ (run here, on the CPU box, on files gpurun brought back).

    python tools/ncu_summary.py rep  <file.ncu-rep>            -> key metrics + top stall sites (markdown)
    python tools/ncu_summary.py launches <launches.csv>        -> per-kernel time shares of the launch list
"""
import collections
import csv
import io
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second", "launch__grid_size", "launch__block_size",
    "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_uniform.avg.pct_of_peak_sustained_active",
    "dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
]


def ncu(*args):
    return subprocess.run(["ncu", *args], capture_output=True, text=True, check=True).stdout


def rep(path):
    rows = list(csv.reader(io.StringIO(ncu("-i", path, "--page", "raw", "--csv"))))
    hdr, units = rows[0], rows[1]
    out = [f"# ncu summary: {path}", ""]
    for vals in rows[2:]:
        d = dict(zip(hdr, vals))
        u = dict(zip(hdr, units))
        out.append(f"## {d.get('Kernel Name', '?')[:120]}")
        for k in KEYS:
            if k in d:
                out.append(f"- {k}: {d[k]} {u.get(k, '')}")
        stalls = {k: d[k] for k in hdr if k.startswith("smsp__pcsamp_warps_issue_stalled_") and
                  not k.endswith("not_issued") and d[k] not in ("", "0")}
        tot = sum(float(v.replace(",", "")) for v in stalls.values()) or 1
        top = sorted(stalls.items(), key=lambda kv: -float(kv[1].replace(",", "")))[:8]
        out.append("- top stall reasons (pc samples): " + ", ".join(
            f"{k.replace('smsp__pcsamp_warps_issue_stalled_', '')} {100 * float(v.replace(',', '')) / tot:.1f}%"
            for k, v in top))
        out.append("")
    src = list(csv.reader(io.StringIO(ncu("-i", path, "--page", "source", "--csv", "--print-source", "sass"))))
    if len(src) > 2:
        h = src[1]
        i_s, i_src = h.index("Warp Stall Sampling (All Samples)"), h.index("Source")
        data = src[2:]
        tot = sum(float(r[i_s] or 0) for r in data) or 1
        out.append("### top SASS stall sites")
        for r in sorted(data, key=lambda r: -float(r[i_s] or 0))[:15]:
            out.append(f"- {100 * float(r[i_s]) / tot:5.1f}%  `{r[i_src].strip()[:100]}`")
        ops = collections.Counter()
        for r in data:
            op = r[i_src].strip().split()
            if op:
                opname = op[1] if op[0].startswith("@") and len(op) > 1 else op[0]
                if opname.startswith(("UTC", "UTMA", "UBLKCP", "LDTM", "STTM", "HMMA", "UTCBAR")):
                    ops[opname.split(".")[0]] += 1
        out.append("")
        out.append("### Blackwell-native instructions present (static count in SASS): " +
                   ", ".join(f"{k} x{v}" for k, v in sorted(ops.items())))
    print("\n".join(out))


def launches(path):
    text = open(path).read()
    i = text.find('"ID"')
    rows = list(csv.DictReader(io.StringIO(text[i:])))
    per = collections.defaultdict(lambda: [0, 0.0])
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"].split("(")[0]
        v = float(r["Metric Value"].replace(",", ""))
        scale = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "s": 1e3, "second": 1e3}.get(r["Metric Unit"], 1.0)
        per[name][0] += 1
        per[name][1] += v * scale
    tot = sum(v[1] for v in per.values()) or 1
    print(f"# launch list summary: {path} (ncu gpu__time_duration.sum, cold-cache, serialised)")
    print("| kernel | launches | total ms | share |")
    print("|---|---|---|---|")
    for k, (n, ms) in sorted(per.items(), key=lambda kv: -kv[1][1]):
        print(f"| {k[:90]} | {n} | {ms:.1f} | {100 * ms / tot:.1f}% |")


if __name__ == "__main__":
    {"rep": rep, "launches": launches}[sys.argv[1]](sys.argv[2])
