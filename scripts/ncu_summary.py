"""Summarise an ncu report (--set full) and a launch list into profiles/.

    python scripts/ncu_summary.py REPORT.ncu-rep LAUNCHES.csv OUT.md [--traffic-key c2]

Reads the report with `ncu -i ... --page raw --csv`, keeps the metrics the
DESIGN.md roofline discussion cites, and aggregates the launch list
(gpu__time_duration.sum per kernel).  With --traffic-key, also writes
dram read+write bytes per launch of the attention kernel into
profiles/attn_traffic.json (read by bench.py for roofline.traffic).
"""
import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
    "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
    "launch__shared_mem_per_block_dynamic", "launch__occupancy_limit_shared_mem",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__cycles_active.avg",
    "sm__cycles_elapsed.avg.per_second",
]


def _csv_after_header(text, first):
    lines = text.splitlines()
    i = [j for j, l in enumerate(lines) if l.startswith(first)][0]
    return list(csv.reader(io.StringIO("\n".join(lines[i:]))))


def short(name):
    for k in ("select_trees", "walk_commit", "argmax_rows", "tree_attn_tc", "tree_attn_simt"):
        if k in name:
            return k
    return "torch/other"


def main():
    rep, launches, out = sys.argv[1:4]
    tkey = sys.argv[sys.argv.index("--traffic-key") + 1] if "--traffic-key" in sys.argv else None
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = _csv_after_header(raw, '"ID"')
    h, units = rows[0], rows[1]
    md = [f"# ncu summary: {os.path.basename(rep)}", ""]
    traffic = None
    for r in rows[2:]:
        d = dict(zip(h, r))
        u = dict(zip(h, units))
        md.append(f"## {d.get('Kernel Name', '?')[:120]}")
        for k in KEYS:
            if k in d:
                md.append(f"- `{k}` = {d[k]} {u[k]}")
        if tkey and "tree_attn" in d.get("Kernel Name", ""):
            def mb(k):
                s = float(d[k].replace(",", ""))
                return s * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[u[k]]
            traffic = int(mb("dram__bytes_read.sum") + mb("dram__bytes_write.sum"))
            md.append(f"- dram read+write per launch = {traffic} bytes")
        md.append("")
    lrows = _csv_after_header(open(launches).read(), '"ID"')
    lh = lrows[0]
    ki, vi, ui = lh.index("Kernel Name"), lh.index("Metric Value"), lh.index("Metric Unit")
    agg = defaultdict(list)
    for r in lrows[1:]:
        agg[short(r[ki])].append(float(r[vi].replace(",", "")) * (1e-3 if r[ui] == "ns" else 1.0))
    ours = {k: v for k, v in agg.items() if k != "torch/other"}
    per_step = {k: sum(v) / len(v) for k, v in ours.items()}
    tot = sum(per_step.values())
    md += ["## launch list (gpu__time_duration.sum, cold-cache, serialised)", "",
           "| kernel | launches | mean us | share of one step |", "|---|---|---|---|"]
    for k, v in sorted(per_step.items(), key=lambda kv: -kv[1]):
        md.append(f"| {k} | {len(ours[k])} | {v:.2f} | {v / tot:.3f} |")
    md.append(f"| torch/other (input generation, outside the timed step) | {len(agg.get('torch/other', []))} | - | - |")
    open(out, "w").write("\n".join(md) + "\n")
    if tkey and traffic:
        p = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "attn_traffic.json")
        cur = json.load(open(p)) if os.path.exists(p) else {}
        cur[tkey] = traffic
        json.dump(cur, open(p, "w"), indent=1, sort_keys=True)
    print("\n".join(md))


if __name__ == "__main__":
    main()
