#!/usr/bin/env python
"""Render tools/results_table.py's JSON as the BASELINE.md §4 table (markdown on stdout).

  python tools/results_md.py gpurun_out/r2b_results_table.json [--issue C5a=0.711,...]
"""
import json
import sys

d = json.load(open(sys.argv[1]))
issue = {}
if len(sys.argv) > 3 and sys.argv[2] == "--issue":
    issue = {k: float(v) for k, v in (x.split("=") for x in sys.argv[3].split(","))}
print("| Config | QBER | GPUs | Frames | FER | Mean iters | f | Processed Mbps | Corrected Mbps | HBM roofline frac "
      "| Int-issue frac | Oracle Mbps (1T / all cores, N cores) | Bit-exact |")
print("|---|---|---|---|---|---|---|---|---|---|---|---|---|")
for r in d["rows"]:
    name = r["workload"].split("@")[0]
    print(f"| {name} | {100 * r['qber']:g} % | 1 | {r['frames']} | {r['FER']:.4f} | {r['mean_iters']:.2f} | {r['f']:.3f} "
          f"| {r['processed_mbps']:.0f} | {r['corrected_mbps']:.0f} | {r['hbm_frac']:.3f} "
          f"| {issue.get(r['workload'], float('nan')):.3f} ".replace("nan", "—")
          + f"| {r['oracle_mbps_1T']:.3f} / {r['oracle_mbps_all']:.2f} ({r['oracle_cores']}) | {r.get('bit_exact', '—')} |")
