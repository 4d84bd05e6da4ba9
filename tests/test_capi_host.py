"""C ABI without a GPU: the in-tree library loads, exports every symbol that
include/laptomo_gpu.h declares, its host-only entry points (contour, step transform,
preconditioner schedule) agree with the oracle, and compute entry points fail loudly when
no sm_100 device is present (there is no CPU fallback)."""
import ctypes as C
import re
from pathlib import Path

import numpy as np
import pytest

from oracle import shifted_solver as oss
from oracle import talbot as otal
from paper_1409_2556_b200 import capi
from paper_1409_2556_b200 import laptomo as L

HEADER = Path(__file__).resolve().parents[1] / "include" / "laptomo_gpu.h"


def header_symbols():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(lt_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = capi.lib()
    syms = header_symbols()
    assert len(syms) >= 35
    for s in syms:
        assert hasattr(lib, s), s
    assert sorted(capi.SIGNATURES) == syms


def test_version_string():
    assert b"sm_100a" in capi.lib().lt_version()


@pytest.mark.parametrize("n,t", [(24, 1.0), (32, 100.0), (20, 300.0), (40, 1e5)])
def test_contour_matches_oracle(n, t):
    got = L.build_contour(n, t)
    ref = otal.build_contour(n, t)
    assert np.allclose(got.thetas, ref.thetas, rtol=0, atol=0)
    assert np.max(np.abs(got.nodes - ref.nodes) / np.abs(ref.nodes)) <= 1e-15
    assert np.max(np.abs(got.weights - ref.weights) / np.abs(ref.weights)) <= 1e-13
    assert np.max(np.abs(got.dnodes - ref.dnodes) / np.abs(ref.dnodes)) <= 1e-15


def test_contour_and_qhat_errors():
    with pytest.raises(ValueError):
        L.build_contour(7, 1.0)
    with pytest.raises(ValueError):
        L.build_contour(8, -1.0)
    with pytest.raises(ValueError):
        L.qhat_step(1.0, 0.0)
    assert L.qhat_step(1.0, 2.0) == 0.5


def test_inverse_laplace_kats_through_capi_contour():
    c = L.build_contour(24, 1.0)
    assert abs(L.inverse_laplace_sum(c, 1.0 / (c.nodes + 1.0)) - np.exp(-1.0)) <= 1e-8
    c = L.build_contour(32, 7.0)
    assert abs(L.inverse_laplace_sum(c, 1.0 / c.nodes) - 1.0) <= 1e-8


@pytest.mark.parametrize("shifts", [
    [1 + 1j, 5 + 2j], [2 + 3j], [1 + 2j, 1 + 1j, 3 + 0j, 3 - 1j, 3 - 1j],
    list(otal.build_contour(32, 100.0).nodes)])
def test_schedule_matches_oracle(shifts):
    got = L.select_preconditioner_shifts(shifts)
    ref = oss.select_preconditioner_shifts(shifts)
    assert got.taus == ref.taus and got.pattern == ref.pattern


def test_empty_schedule_rejected():
    with pytest.raises(ValueError):
        L.select_preconditioner_shifts([])


def _has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.mark.skipif(_has_gpu(), reason="checks the no-GPU failure path")
def test_compute_fails_loudly_without_gpu():
    h = C.c_void_p()
    st = capi.lib().lt_ctx_create(0, C.byref(h))
    assert st == capi.LT_ERR_CUDA
    with pytest.raises(capi.CudaError):
        L.Context(0)


def test_cpp_mirror_compiles_links_and_runs(tmp_path):
    """include/laptomo/laptomo.hpp (the C++ mirror of the reference API) compiles with g++,
    links the library and its host-only calls work; device calls raise DeviceError without
    a GPU."""
    import subprocess
    root = Path(__file__).resolve().parents[1]
    exe = tmp_path / "demo"
    libdir = root / "paper_1409_2556_b200" / "_lib"
    cmd = ["g++", "-std=c++17", "-O1", f"-I{root / 'include'}", str(root / "examples" / "cpp_mirror_demo.cpp"),
           f"-L{libdir}", "-llaptomo_gpu", f"-Wl,-rpath,{libdir}", "-o", str(exe)]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    out = subprocess.run([str(exe)], check=True, capture_output=True, text=True).stdout
    assert "invalid_argument ok" in out and "taus 2 pattern 5" in out
    err = float(out.split("= ")[1].split()[0])
    assert abs(err) <= 1e-8
    assert ("no device" in out) or ("device: head" in out)
