"""C-ABI library checks that need no GPU: it builds, loads, exports every symbol include/deepinverse.h
declares, and refuses to create a context without an sm_100 device (there is no CPU fallback)."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_1701_03891_b200 import build, binding
    build.build()
    return binding.load()


def _declared_symbols():
    hdr = open(os.path.join(ROOT, "include", "deepinverse.h")).read()
    hdr = re.sub(r"/\*.*?\*/", "", hdr, flags=re.S)
    return sorted(set(re.findall(r"\b(di_[a-z_]+)\s*\(", hdr)))


def test_header_declares_expected_calls():
    syms = _declared_symbols()
    for s in ("di_create", "di_recover", "di_destroy"):   # SURVEY.md §8(b) boundary
        assert s in syms


def test_every_declared_symbol_is_exported(lib):
    from paper_1701_03891_b200 import binding
    syms = _declared_symbols()
    assert sorted(binding.EXPORTS) == syms
    for s in syms:
        assert hasattr(lib, s), s


def test_status_strings(lib):
    from paper_1701_03891_b200 import binding
    assert binding.di_status_string(0) == "DI_OK"
    assert binding.di_status_string(4) == "DI_ERR_DEVICE"


def test_kernels_are_sm100a_tcgen05(lib):
    """The shipped object carries sm_100a SASS with tcgen05 MMA (UTCHMMA) and TMA (UTMALDG) instructions."""
    import subprocess
    from paper_1701_03891_b200 import binding
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", binding.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert "UTCHMMA" in out and "UTMALDG" in out and "LDTM" in out


def test_no_cpu_fallback_without_gpu(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import synth
    from paper_1701_03891_b200 import binding
    phi = synth.make_phi(64, 256)
    p = synth.make_params()
    ws = [np.ascontiguousarray(w) for w in p.w]
    a = binding.di_create_args(64, 16, 16, phi.ctypes.data, 0, ws[0].ctypes.data, None, ws[1].ctypes.data, None,
                               ws[2].ctypes.data, None, 2, 0, 0, 4)
    h = ctypes.c_void_p()
    st = lib.di_create(ctypes.byref(a), ctypes.byref(h))
    assert st == binding.DI_ERR_DEVICE
    assert h.value is None


def test_argument_validation_before_device(lib):
    from paper_1701_03891_b200 import binding
    h = ctypes.c_void_p()
    assert lib.di_create(None, ctypes.byref(h)) == binding.DI_ERR_ARG
    phi = np.zeros((5, 4), np.float32)
    w = np.zeros(64 * 121 * 64, np.float32)
    a = binding.di_create_args(5, 2, 2, phi.ctypes.data, 0, w.ctypes.data, None, w.ctypes.data, None,
                               w.ctypes.data, None, 2, 0, 0, 4)
    assert lib.di_create(ctypes.byref(a), ctypes.byref(h)) == binding.DI_ERR_DOMAIN     # m > N
    a.m, a.n1 = 0, 3
    assert lib.di_create(ctypes.byref(a), ctypes.byref(h)) == binding.DI_ERR_DOMAIN     # m < 1
    a.m, a.flags = 4, 1 << 9
    assert lib.di_create(ctypes.byref(a), ctypes.byref(h)) == binding.DI_ERR_ARG        # unknown flag
    assert lib.di_recover(None, None, 0, 1, None, None) == binding.DI_ERR_ARG
    assert lib.di_destroy(None) == binding.DI_OK


def test_product_library_is_not_an_experiment_build(lib):
    """Instrumentation / wrong-result experiment switches live only in libdeepinverse_exp.so (build.py); the library
    the tests and bench load was built with exactly the product flags (stamp) and exports no experiment marker."""
    from paper_1701_03891_b200 import binding, build
    if os.environ.get("DI_LIB"):
        pytest.skip("DI_LIB selects another build on purpose (the DI_DEBUG run, DESIGN.md §3)")
    assert binding.LIB_PATH == build.LIB, "DI_LIB points the binding at another library"
    assert not hasattr(lib, "di_experiment_build")
    st = build.read_stamp(build.LIB)
    assert st is not None and st["flags"] == build.FLAGS, st
    assert not any(f.startswith("-D") for f in st["flags"])


def test_instrumentation_macros_refused_outside_experiment_build():
    """kernels.cuh: -DDI_PROF_CONV2 (or a geometry override) without -DDI_EXPERIMENT_BUILD is a compile error."""
    import subprocess
    from paper_1701_03891_b200 import build
    src = os.path.join(build.CSRC, "k_conv2_tc.cu")
    base = [build.NVCC, "-E", "-std=c++17", "-I", os.path.join(ROOT, "include"), "-I", build.CSRC, src, "-o", os.devnull]
    bad = subprocess.run(base + ["-DDI_PROF_CONV2"], capture_output=True, text=True)
    assert bad.returncode != 0 and "DI_EXPERIMENT_BUILD" in bad.stderr
    ok = subprocess.run(base + ["-DDI_PROF_CONV2", "-DDI_EXPERIMENT_BUILD"], capture_output=True, text=True)
    assert ok.returncode == 0, ok.stderr[-2000:]


def _build_c_example(tmp_path):
    import subprocess
    from paper_1701_03891_b200 import build
    build.build()
    exe = str(tmp_path / "recover_c")
    libdir = os.path.dirname(build.LIB)
    r = subprocess.run(["gcc", "-std=c99", "-O2", "-Wall", "-Wextra", "-Werror", "-I", os.path.join(ROOT, "include"),
                        os.path.join(ROOT, "examples", "recover.c"), "-L", libdir, "-ldeepinverse",
                        f"-Wl,-rpath,{libdir}", "-lm", "-o", exe], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return exe


def test_c_example_builds_and_refuses_without_gpu(tmp_path):
    """examples/recover.c: the header is plain C (gcc -std=c99 -Werror) and the library links from C; without an
    sm_100 device di_create returns DI_ERR_DEVICE (exit 2) -- there is no CPU fallback."""
    import subprocess
    import torch
    exe = _build_c_example(tmp_path)
    if torch.cuda.is_available():
        pytest.skip("GPU present: tests/test_gpu_parity.py::test_c_example_on_gpu runs it")
    r = subprocess.run([exe], capture_output=True, text=True)
    assert r.returncode == 2 and "DI_ERR_DEVICE" in r.stderr
