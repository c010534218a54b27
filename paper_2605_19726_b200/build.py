"""Build libbaatt.so in-tree with nvcc for sm_100a (no JIT cache, no torch types).

    python -m paper_2605_19726_b200.build [--debug]
"""
from __future__ import annotations

import os
import subprocess
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libbaatt.so")
SOURCES = ["api.cu", "select_kernels.cu", "attn_simt.cu", "attn_sm100.cu", "attn_sm100_pp.cu", "attn_sm100_pp2.cu", "block_mass_sm100.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc"):
        if c and os.path.exists(c):
            return c
    return "nvcc"


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(ROOT, "include", "ba_attn.h")]
    return any(os.path.getmtime(p) > t for p in deps)


def build(force: bool = False, debug: bool = False, verbose: bool = True, extra_flags=None, out: str = None,
          profiling: bool = False) -> str:
    """extra_flags / out: A/B builds (e.g. -DBA_PP_PSPLIT=4 into another .so, loaded via BA_LIB_PATH).
    profiling: also compile the profiling-only kernel variants (no-softmax skeleton, clock64 tile
    traces with device printf; BA_ATTN_DEBUG=1|2) — never part of the product library."""
    lib = out or LIB
    if not force and not needs_build() and out is None:
        return LIB
    objs = []
    flags = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
                    "-I", os.path.join(ROOT, "include"), "-Xptxas", "-v" if verbose and debug else "-O3"]
    if debug:
        flags += ["-DBA_DEBUG=1"]
    if profiling:
        flags += ["-DBA_PROFILING=1"]
    flags += list(extra_flags or [])
    t0 = time.time()
    procs = []
    for src in SOURCES:
        obj = os.path.join(CSRC, src.replace(".cu", ".o" if out is None else "_ab.o"))
        objs.append(obj)
        cmd = [nvcc()] + flags + ["-c", os.path.join(CSRC, src), "-o", obj]
        procs.append((src, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)))
    for src, p in procs:
        out, _ = p.communicate()
        if p.returncode != 0:
            sys.stderr.write(out)
            raise RuntimeError(f"nvcc failed on {src}")
        if verbose and out.strip():
            sys.stderr.write(out)
    cmd = [nvcc()] + ARCH + ["-shared", "-o", lib] + objs + ["-lcuda" if False else "-lcudart_static", "-ldl", "-lrt", "-lpthread"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("link failed")
    for o in objs:
        os.remove(o)
    if verbose:
        print(f"built {lib} in {time.time() - t0:.1f}s")
    return lib


if __name__ == "__main__":
    build(force=True, debug="--debug" in sys.argv, profiling="--profiling" in sys.argv,
          out=sys.argv[sys.argv.index("--out") + 1] if "--out" in sys.argv else None)
