#!/usr/bin/env python
"""Build the product library with extra nvcc flags into another path (A/B experiments).

  python tools/build_variant.py build_ab/x.so -DQKD_KEEP_ADDR=20 ...
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import _build  # noqa: E402

out, extra = sys.argv[1], sys.argv[2:]
cu = [s for s in _build.cuda_sources() if s.endswith(".cu")]
cmd = [_build.NVCC, *extra, *_build.ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-shared",
       "-I", os.path.join(ROOT, "include"), "-o", out, *cu]
sys.exit(subprocess.run(cmd, cwd=ROOT).returncode)
