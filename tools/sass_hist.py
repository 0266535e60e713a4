#!/usr/bin/env python
"""Opcode histogram of the hot loop bodies of a kernel (static SASS, no GPU): compare two builds.

  python tools/sass_hist.py --lib A.so [--lib2 B.so] --kernel decode_kernelILi20ELb1ELb1ELb0ELb0E --vabs 84
Selects the loop whose VABSDIFF4 count is closest to --vabs (e.g. the degree-18 row of C5a: 84 =
48 tau + 18 magnitudes + 18 guards)."""
import argparse, collections, os, sys
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from sass_loops import functions, loops, opname  # noqa: E402


def pick(lib, kernel, vabs, min_len=150):
    for name, ins in functions(lib).items():
        if kernel in name:
            best = None
            for body in loops(ins, min_len):
                c = collections.Counter(opname(t).split(".")[0] for _, t in body)
                if best is None or abs(c["VABSDIFF4"] - vabs) < abs(best[0]["VABSDIFF4"] - vabs):
                    best = (c, body)
            return best


ap = argparse.ArgumentParser()
ap.add_argument("--lib", required=True)
ap.add_argument("--lib2")
ap.add_argument("--kernel", default="decode_kernelILi20ELb1ELb1ELb0ELb0E")
ap.add_argument("--vabs", type=int, default=84)
ap.add_argument("--dump", action="store_true")
a = ap.parse_args()
c1, b1 = pick(a.lib, a.kernel, a.vabs)
if a.dump:
    for ad, t in b1:
        print(hex(ad), t)
c2 = pick(a.lib2, a.kernel, a.vabs)[0] if a.lib2 else collections.Counter()
keys = sorted(set(c1) | set(c2), key=lambda k: -(c1[k] + c2[k]))
print(f"{'op':12s} {'A':>6s} {'B':>6s}")
for k in keys:
    print(f"{k:12s} {c1[k]:6d} {c2[k]:6d}")
print(f"{'total':12s} {sum(c1.values()):6d} {sum(c2.values()):6d}")
