#!/usr/bin/env python
"""Static SASS report of the hot loops of one kernel in a built library (no GPU needed).

  python tools/sass_loops.py [--lib paper_1903_10107_b200/libqkdldpc.so] [--kernel ILi20ELb1ELb1ELb0E]
                             [--min-len 150]

For every backward branch whose body has >= --min-len instructions, prints the body length,
the ALU-pipe / FMA-pipe / other split (sm_100a: LOP3, PRMT, SHF, VABSDIFF4, VIADDMNMX, IADD3,
LEA, ISETP, SEL on the ALU pipe; IMAD*, VIADD on the FMA pipe), shared/local/global memory ops
and the tau count (VABSDIFF4).  Used to check each kernel change before spending GPU time.
"""
from __future__ import annotations

import argparse
import collections
import os
import re
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ALU = {"LOP3", "PRMT", "VABSDIFF4", "VIADDMNMX", "IADD3", "SHF", "LEA", "ISETP", "SEL", "VIMNMX", "IMNMX",
       "PLOP3", "LOP"}
FMA = {"IMAD", "VIADD", "IDP", "HFMA2", "FFMA", "IMUL"}


def functions(lib: str) -> dict[str, list[tuple[int, str]]]:
    txt = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True, check=True).stdout
    out: dict[str, list[tuple[int, str]]] = {}
    cur = None
    for line in txt.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            cur = m.group(1)
            out[cur] = []
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
        if m and cur:
            out[cur].append((int(m.group(1), 16), m.group(2).strip()))
    return out


def opname(t: str) -> str:
    return [o for o in t.split() if not o.startswith("@")][0]


def loops(ins, min_len):
    idx = {a: i for i, (a, _) in enumerate(ins)}
    for i, (a, t) in enumerate(ins):
        m = re.search(r"BRA (0x[0-9a-f]+)", t)
        if m:
            tgt = int(m.group(1), 16)
            if tgt < a and tgt in idx and i + 1 - idx[tgt] >= min_len:
                yield ins[idx[tgt]:i + 1]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--lib", default=os.path.join(ROOT, "paper_1903_10107_b200", "libqkdldpc.so"))
    ap.add_argument("--kernel", default="decode_kernelILi20ELb1ELb1ELb0E")
    ap.add_argument("--min-len", type=int, default=150)
    ap.add_argument("--max-len", type=int, default=4000)
    a = ap.parse_args()
    for name, ins in functions(a.lib).items():
        if a.kernel not in name:
            continue
        print(name)
        for body in loops(ins, a.min_len):
            if len(body) > a.max_len:
                continue
            c = collections.Counter(opname(t).split(".")[0] for _, t in body)
            alu = sum(v for k, v in c.items() if k in ALU)
            fma = sum(v for k, v in c.items() if k in FMA)
            print(f"  len {len(body):5d}  tau/VABS {c['VABSDIFF4']:3d}  ALU {alu:4d}  FMA {fma:4d}  "
                  f"other {len(body) - alu - fma:4d}  LDS {c['LDS']:3d} STS {c['STS']:3d} LDG {c['LDG']:2d} "
                  f"STG {c['STG']:2d} LDL {c['LDL']:2d} STL {c['STL']:2d} SHFL {c['SHFL']}")


if __name__ == "__main__":
    main()
