#!/usr/bin/env python
"""Summarise ncu outputs brought back by gpurun into tracked files under profiles/.

  python tools/ncu_summary.py --tag r1 --launches gpurun_out/launches.csv \
         --full gpurun_out/prof_r1.ncu-rep [--algo-bytes B]

Writes profiles/<tag>_launches.md (per-kernel share of the step, from the
`--metrics gpu__time_duration.sum --clock-control none` launch list: cold-cache and
serialised, so compare SHARES) and profiles/<tag>_decode_full.md (+ .csv) with the
DRAM traffic, pipe utilisation and stall reasons of the captured decode launches, and
profiles/traffic.json (DRAM bytes per launch of the dominant decode launch, read by bench.py).
"""
import argparse
import collections
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SCALE = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "s": 1e3, "second": 1e3}


def launches(path):
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[h]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = collections.OrderedDict()
    for r in rows[h + 1:]:
        if len(r) <= vi or not r[vi]:
            continue
        ms = float(r[vi].replace(",", "")) * SCALE.get(r[ui], 1.0)
        name = r[ki].split("(")[0].replace("void ", "").replace("<unnamed>::", "")
        agg.setdefault(name, []).append(ms)
    return agg


def raw(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("lts__t_bytes.sum", "L2 bytes"),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "ALU pipe % of peak"),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "FMA pipe % of peak"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe % of peak"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__inst_executed.avg.per_cycle_active", "IPC (warp inst / SM cycle)"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
    ("smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio", "stall: math pipe throttle"),
    ("smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio", "stall: not selected"),
    ("smsp__average_warps_issue_stalled_wait_per_issue_active.ratio", "stall: wait"),
    ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", "stall: long scoreboard"),
    ("smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio", "stall: barrier"),
    ("smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio", "stall: short scoreboard"),
    ("smsp__cycles_active.avg", "SM cycles active (avg)"),
    ("smsp__sass_inst_executed_op_local_ld.sum", "local loads (spills)"),
]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tag", required=True)
    ap.add_argument("--launches")
    ap.add_argument("--full")
    ap.add_argument("--algo-bytes", type=float, default=None, help="algorithmic bytes of the first decode launch")
    ap.add_argument("--note", default="")
    ap.add_argument("--workload", default="C5a", help="workload of the captured decode launch (bench.py matches it)")
    ap.add_argument("--no-traffic", action="store_true", help="do not rewrite profiles/traffic.json")
    a = ap.parse_args()
    prof = os.path.join(ROOT, "profiles")
    os.makedirs(prof, exist_ok=True)
    if a.launches:
        agg = launches(a.launches)
        tot = sum(sum(v) for v in agg.values())
        with open(os.path.join(prof, f"{a.tag}_launches.md"), "w") as f:
            f.write(f"# {a.tag}: kernel launch list ({os.path.basename(a.launches)})\n\n")
            f.write("`ncu --metrics gpu__time_duration.sum --clock-control none` over the bench command "
                    "(cold-cache, serialised: compare shares, not absolutes).\n\n")
            if a.note:
                f.write(a.note + "\n\n")
            f.write("| kernel | launches | total ms | mean ms | share |\n|---|---|---|---|---|\n")
            for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
                f.write(f"| `{k}` | {len(v)} | {sum(v):.3f} | {sum(v) / len(v):.3f} | {100 * sum(v) / tot:.2f}% |\n")
        print(open(os.path.join(prof, f"{a.tag}_launches.md")).read())
    if a.full:
        hdr, units, rows = raw(a.full)
        name_i = hdr.index("Kernel Name")
        lines = [f"# {a.tag}: `ncu --set full` capture ({os.path.basename(a.full)})\n"]
        table = []
        for r in rows:
            kname = r[name_i].split("(")[0].replace("void ", "").replace("<unnamed>::", "")
            lines.append(f"\n## {kname}\n\n| metric | value | unit |\n|---|---|---|")
            rec = {"kernel": kname}
            for key, label in KEYS:
                if key in hdr:
                    v = r[hdr.index(key)]
                    lines.append(f"| {label} (`{key}`) | {v} | {units[hdr.index(key)]} |")
                    rec[key] = v
            table.append(rec)
        first = table[0]

        def gb(key):
            u = units[hdr.index(key)]
            v = float(first[key])
            return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}[u]

        dram = gb("dram__bytes_read.sum") + gb("dram__bytes_write.sum")
        lines.append(f"\nDRAM bytes (read + write) of the first captured launch: {dram:.4g} B")
        if a.algo_bytes:
            lines.append(f"Algorithmic bytes of that launch: {a.algo_bytes:.4g} B -> traffic/algorithmic = "
                         f"{dram / a.algo_bytes:.3f}")
        if a.note:
            lines.append("\n" + a.note)
        with open(os.path.join(prof, f"{a.tag}_decode_full.md"), "w") as f:
            f.write("\n".join(lines) + "\n")
        def num(key):
            try:
                return float(first[key])
            except (KeyError, ValueError):
                return None

        dur_ms = num("gpu__time_duration.sum")
        counters = {   # DRAM GB/s, integer-issue fraction and the ALU/FMA pipe split
            "dram_GBps": dram / (dur_ms * 1e-3) / 1e9 if dur_ms else None,
            "issue_active_frac": (num("smsp__issue_active.avg.pct_of_peak_sustained_active") or 0) / 100,
            "alu_pipe_frac": (num("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active") or 0) / 100,
            "fma_pipe_frac": (num("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active") or 0) / 100,
            "warp_instructions": num("smsp__inst_executed.sum"),
            "duration_ms_under_ncu": dur_ms,
        }
        if not a.no_traffic:
            with open(os.path.join(prof, "traffic.json"), "w") as f:
                json.dump({"decode_dram_bytes_per_launch": dram, "ncu": counters,
                           "source": f"profiles/{a.tag}_decode_full.md", "kernel": first["kernel"],
                           "workload": a.workload}, f, indent=1)
        print("\n".join(lines))


if __name__ == "__main__":
    sys.exit(main())
