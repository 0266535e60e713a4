#!/usr/bin/env python
"""Stall profile of a kernel by 100-instruction blocks from an ncu source-page CSV
(`ncu -i X.ncu-rep --page source --csv --print-source sass > src.csv`): per block the share of
warp samples, the ALU share of its instructions and the top stall reasons.  Finds which phase
of the row update (gather, chains, emit) or which barrier the time goes to."""
import collections
import csv
import sys

ALU = {"LOP3", "PRMT", "VABSDIFF4", "VIADDMNMX", "IADD3", "SHF", "LEA", "ISETP", "SEL", "VIMNMX", "IMNMX"}
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
idx = {h: i for i, h in enumerate(hdr)}
blk = int(sys.argv[2]) if len(sys.argv) > 2 else 100
blocks = collections.OrderedDict()
tot_st = collections.Counter()
for i, r in enumerate(rows[2:]):
    src = r[idx["Source"]].strip()
    op = [o for o in src.split() if not o.startswith("@")][0].split(".")[0] if src else ""
    st = {h[6:]: float(r[idx[h]] or 0) for h in hdr if h.startswith("stall_") and "Not Issued" not in h}
    d = blocks.setdefault(i // blk, [0.0, collections.Counter(), collections.Counter(), 0.0])
    d[0] += float(r[idx["Warp Stall Sampling (All Samples)"]] or 0)
    d[1].update(st)
    d[2][op] += 1
    d[3] += float(r[idx["Instructions Executed"]] or 0)
    tot_st.update(st)
tot = sum(v[0] for v in blocks.values())
s = sum(tot_st.values())
print("overall:", ", ".join(f"{k}:{v / s:.3f}" for k, v in tot_st.most_common(8)))
for b, (smp, st, ops, ex) in blocks.items():
    if smp / tot < 0.008:
        continue
    n = sum(ops.values())
    alu = sum(v for k, v in ops.items() if k in ALU) / n
    top = ", ".join(f"{k}:{v / smp:.2f}" for k, v in st.most_common(5))
    print(f"blk {b:4d} samp {smp / tot:.3f} alu {alu:.2f} exec {ex:.2e} | {top}")
