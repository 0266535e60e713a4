"""In-tree build of the three native libraries (no JIT cache; the .so files travel with
the repo snapshot to the GPU box).

  synth/libsynth.so                      seeded input generators (gcc)
  oracle/liboracle.so                    scalar CPU oracle (gcc; test infrastructure only)
  paper_1903_10107_b200/libqkdldpc.so    the product: sm_100a kernels + C ABI (nvcc)
"""
from __future__ import annotations

import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.abspath(__file__))
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _stale(target: str, sources: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(s) > t for s in sources)


def _run(cmd: list[str]) -> None:
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("build failed: " + " ".join(cmd))


def build_synth(force: bool = False) -> str:
    src = os.path.join(ROOT, "synth", "synth.c")
    out = os.path.join(ROOT, "synth", "libsynth.so")
    if force or _stale(out, [src]):
        _run(["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-pthread", "-o", out, src])
    return out


def build_oracle(force: bool = False) -> str:
    src = os.path.join(ROOT, "oracle", "oracle.c")
    out = os.path.join(ROOT, "oracle", "liboracle.so")
    if force or _stale(out, [src]):
        # -O2, scalar, no intrinsics, no -ffast-math (SURVEY §8(d) oracle build)
        _run(["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-pthread", "-o", out, src, "-lm"])
    return out


def cuda_sources() -> list[str]:
    d = os.path.join(ROOT, "paper_1903_10107_b200", "csrc")
    srcs = [os.path.join(d, f) for f in sorted(os.listdir(d)) if f.endswith((".cu", ".cuh", ".h"))]
    srcs.append(os.path.join(ROOT, "include", "qkd_ldpc.h"))
    return srcs


def build_cuda(force: bool = False, extra: list[str] | None = None, out: str | None = None,
               only: list[str] | None = None) -> str:
    """Compile every .cu of csrc/ to an object in parallel (the decode kernel variants are spread over
    several translation units), then link the shared library.  `only` (A/B builds): compile just these
    translation units (basenames) with `extra` and link the product build's objects for the rest."""
    srcs = cuda_sources()
    out = out or os.path.join(ROOT, "paper_1903_10107_b200", "libqkdldpc.so")
    if not (force or extra or _stale(out, srcs + [__file__])):
        return out
    cu = [s for s in srcs if s.endswith(".cu")]
    objdir = os.path.join(os.path.dirname(out), "build_obj") if only is None and not extra else out + ".obj"
    os.makedirs(objdir, exist_ok=True)
    common = [NVCC, *(extra or []), *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xfatbin", "-compress-all",
              "-Xptxas", "-v", "-I", os.path.join(ROOT, "include")]
    jobs = []
    main_objdir = os.path.join(ROOT, "paper_1903_10107_b200", "build_obj")
    for src in cu:
        obj = os.path.join(objdir, os.path.basename(src)[:-3] + ".o")
        if only is not None and os.path.basename(src) not in only:
            jobs.append((src, os.path.join(main_objdir, os.path.basename(obj)), None))
            continue
        jobs.append((src, obj, subprocess.Popen([*common, "-c", "-o", obj, src], cwd=ROOT,
                                                stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)))
    logs, failed = [], []
    for src, obj, proc in jobs:
        if proc is None:
            continue
        text = proc.communicate()[0]
        logs.append(f"==== {os.path.basename(src)}\n{text}")
        if proc.returncode != 0:
            failed.append(src)
    log_path = os.path.join(ROOT, "paper_1903_10107_b200", "ptxas.log") if out.endswith(
        os.path.join("paper_1903_10107_b200", "libqkdldpc.so")) else out + ".ptxas.log"
    with open(log_path, "w") as f:
        f.write("\n".join(logs))
    if failed:
        sys.stderr.write("\n".join(logs))
        raise RuntimeError("nvcc build failed: " + ", ".join(failed))
    r = subprocess.run([NVCC, *ARCH, "-shared", "-o", out, *[o for _, o, _ in jobs]], cwd=ROOT,
                       capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc link failed")
    return out


def build_all(force: bool = False) -> None:
    build_synth(force)
    build_oracle(force)
    build_cuda(force)


if __name__ == "__main__":
    build_all(force="--force" in sys.argv)
    print("built")
