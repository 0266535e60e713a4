#!/usr/bin/env python
"""Build the product library with extra nvcc flags into another path (A/B experiments).

  python tools/build_variant.py build_ab/x.so -DQKD_KEEP_ADDR=20 ... [--only decode_inst_20.cu,...]
(--only: recompile just those translation units, link the product build's objects for the rest)
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import _build  # noqa: E402

out, extra = sys.argv[1], sys.argv[2:]
only = None
if "--only" in extra:
    i = extra.index("--only")
    only = extra[i + 1].split(",")
    extra = extra[:i] + extra[i + 2:]
_build.build_cuda(force=True, extra=extra, out=os.path.abspath(out), only=only)
