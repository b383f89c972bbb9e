"""The C++ drop-in API (include/mpmg/*.hpp, namespace mpmg) -- the interface
the reference's users call. CPU: the layer builds, links the
sm_100a library, its host-side setup matches the reference's golden
fixtures bitwise, and device calls fail loudly without a GPU. GPU: the
reference's own kernel known-answer tests and end-to-end solves, restated
in C++ (tests/cpp/test_api.cpp)."""
import os
import subprocess

import numpy as np
import pytest

from oracle import Oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2007_07539_b200", "_lib")
GOLD = os.path.join(ROOT, "tests", "golden")
EXE = os.path.join(ROOT, "tests", "cpp", "_build", "test_api")


def build_exe():
    subprocess.run(["make", "-C", os.path.join(ROOT, "paper_2007_07539_b200", "cpp")], check=True,
                   capture_output=True)
    os.makedirs(os.path.dirname(EXE), exist_ok=True)
    src = os.path.join(ROOT, "tests", "cpp", "test_api.cpp")
    deps = [src, os.path.join(LIB, "libmpmg_cpp.so"), os.path.join(LIB, "libmpmg_b200.so")]
    deps += [os.path.join(ROOT, "include", "mpmg", f) for f in os.listdir(os.path.join(ROOT, "include", "mpmg"))]
    if not os.path.exists(EXE) or os.path.getmtime(EXE) < max(os.path.getmtime(d) for d in deps if os.path.exists(d)):
        subprocess.run(["g++", "-std=c++20", "-O1", "-I" + os.path.join(ROOT, "include"), src, "-L" + LIB, "-lmpmg_cpp",
                        "-lmpmg_b200", "-Wl,-rpath," + LIB, "-o", EXE], check=True)
    return EXE


@pytest.fixture(scope="module")
def exe():
    return build_exe()


def same_bits(a, b):
    a = np.asarray(a, dtype=np.float64); b = np.asarray(b, dtype=np.float64)
    return a.shape == b.shape and np.array_equal(a.view(np.uint64), b.view(np.uint64))


def test_host_setup_matches_reference(exe, tmp_path):
    out = subprocess.run([exe, "--host-dump", str(tmp_path)], capture_output=True, text=True)
    assert out.returncode == 0, out.stdout + out.stderr
    g = np.load(os.path.join(GOLD, "hierarchy.npz"))
    for dim, n, L in ((2, 17, 4), (3, 9, 3)):
        key = f"{dim}_{n}_d_mg_0"
        rw = 9 if dim == 2 else 27
        cols = np.fromfile(tmp_path / f"A_{dim}_{n}_cols.bin", dtype=np.int32).reshape(-1, rw)
        vals = np.fromfile(tmp_path / f"A_{dim}_{n}_vals.bin", dtype=np.float64).reshape(-1, rw)
        assert np.array_equal(cols, g[f"{key}_l{L - 1}_A_cols"])
        assert same_bits(vals, g[f"{key}_l{L - 1}_A_vals"])
        for nm, w in (("P", 1 << dim), ("R", rw)):
            c = np.fromfile(tmp_path / f"{nm}_{dim}_{n}_cols.bin", dtype=np.int32).reshape(-1, w)
            v = np.fromfile(tmp_path / f"{nm}_{dim}_{n}_vals.bin", dtype=np.float64).reshape(-1, w)
            assert np.array_equal(c, g[f"{key}_l{L - 2}_{nm}_cols"]), nm
            assert same_bits(v, g[f"{key}_l{L - 2}_{nm}_vals"]), nm
    for dim, n in ((2, 33), (3, 17)):
        assert same_bits(np.fromfile(tmp_path / f"rhs_{dim}_{n}.bin"), g[f"rhs_{dim}_{n}"])
        assert same_bits(np.fromfile(tmp_path / f"exact_{dim}_{n}.bin"), g[f"exact_{dim}_{n}"])
    O = Oracle()
    rows = np.fromfile(tmp_path / "fp16_fma.bin").reshape(-1, 6)
    ref = [O.fma16(a, b, c, bool(f), bool(m)) for a, b, c, f, m, _ in rows]
    assert same_bits(rows[:, 5], ref)


def test_device_calls_fail_loudly_without_gpu(exe):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    out = subprocess.run([exe], capture_output=True, text=True)
    assert out.returncode == 2 and "no CUDA device" in out.stdout


@pytest.mark.gpu
def test_cpp_api_on_device(exe):
    out = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    print(out.stdout)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "0 failed" in out.stdout
