"""Build the in-tree CUDA library libdeepinverse.so (sm_100a only) with nvcc.

No torch extension machinery: the library is a plain C-ABI shared object (include/deepinverse.h)
loaded with ctypes, so the same .so serves C callers, the Python binding, tests and bench.py.
"""
from __future__ import annotations

import json
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libdeepinverse.so")
SOURCES = ["api.cu", "k_proxy.cu", "k_conv_simt.cu", "k_conv2_tc.cu", "k_conv13_tc.cu", "k_conv2_tf32.cu", "k_sense.cu", "k_train.cu",
           "k_wgrad2_tc.cu", "k_wgrad13_tc.cu", "k_conv3_r4.cu"]
HEADERS = ["sm100.cuh", "kernels.cuh"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
         "-Xptxas", "-warn-spills", "--expt-relaxed-constexpr", "-diag-suppress", "177"]
# Experiment builds (e.g. DI_NVCC_EXTRA=-DDI_PROF_CONV2 for the conv2 issuer cycle breakdown) go to a SEPARATE library,
# libdeepinverse_exp.so with its own object directory, compiled with -DDI_EXPERIMENT_BUILD (kernels.cuh refuses the
# instrumentation macros without it).  The product library is never built with extra flags; a stamp file next to it
# records the exact flags and nvcc version, and any difference forces a rebuild.
EXTRA = os.environ.get("DI_NVCC_EXTRA", "").split()
_EXP_NAME = os.environ.get("DI_EXP_NAME", "")   # several experiment libraries side by side (A/B runs)
EXP_LIB = os.path.join(HERE, f"libdeepinverse_exp{'_' + _EXP_NAME if _EXP_NAME else ''}.so")


def _target(extra: list[str]) -> tuple[str, str, list[str]]:
    if extra:
        return (EXP_LIB, os.path.join(HERE, "build_exp" + ("_" + _EXP_NAME if _EXP_NAME else "")),
                FLAGS + ["-DDI_EXPERIMENT_BUILD"] + extra)
    return LIB, os.path.join(HERE, "build"), list(FLAGS)


def _nvcc_version() -> str:
    try:
        return subprocess.run([NVCC, "--version"], capture_output=True, text=True).stdout.strip().splitlines()[-1]
    except OSError:
        return "?"


def _stamp(flags: list[str]) -> str:
    return json.dumps({"flags": flags, "nvcc": _nvcc_version()}, sort_keys=True)


def read_stamp(lib: str = LIB) -> dict | None:
    try:
        return json.load(open(lib + ".stamp"))
    except (OSError, ValueError):
        return None


def _stale(target: str, deps: list[str], stamp: str) -> bool:
    if not os.path.exists(target):
        return True
    try:
        if open(target + ".stamp").read() != stamp:
            return True
    except OSError:
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    """Build if stale.  Serialised across processes by an exclusive lock (torchrun ranks of bench.py, pytest
    workers), so concurrent callers never write the same object files; a waiter finds the library fresh."""
    import fcntl
    os.makedirs(os.path.join(HERE, "build"), exist_ok=True)
    with open(os.path.join(HERE, "build", ".lock"), "w") as lk:
        fcntl.flock(lk, fcntl.LOCK_EX)
        try:
            return _build_locked(force, verbose)
        finally:
            fcntl.flock(lk, fcntl.LOCK_UN)


def _build_locked(force: bool, verbose: bool) -> str:
    lib, objdir, flags = _target(EXTRA)
    deps = [os.path.join(CSRC, s) for s in SOURCES + HEADERS] + [os.path.join(ROOT, "include", "deepinverse.h"),
                                                                 os.path.abspath(__file__)]
    stamp = _stamp(flags)
    if not force and not _stale(lib, deps, stamp):
        return lib
    os.makedirs(objdir, exist_ok=True)
    objs = []
    procs = []
    for s in SOURCES:
        o = os.path.join(objdir, s.replace(".cu", ".o"))
        objs.append(o)
        cmd = [NVCC, *flags, "-I", os.path.join(ROOT, "include"), "-I", CSRC, "-c", os.path.join(CSRC, s), "-o", o]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        procs.append((s, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)))
    for s, p in procs:
        out, _ = p.communicate()
        if p.returncode != 0:
            raise RuntimeError(f"nvcc failed on {s}:\n{out}")
        if verbose and out.strip():
            print(out, file=sys.stderr)
    tmp = lib + f".tmp{os.getpid()}"
    cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", tmp, *objs, "-cudart", "static"]
    r = subprocess.run(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}")
    os.replace(tmp, lib)
    with open(lib + ".stamp", "w") as f:
        f.write(stamp)
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
