"""CPU checks of the product library's C ABI (no GPU needed):
  * libmpmg_b200.so loads and exports every function include/mpmg_gpu.h
    declares;
  * the host-side setup entry points (per-level stencil, binary16 rounding of
    level scalars, manufactured right-hand side) are bitwise identical to the
    reference's hierarchy (oracle, itself pinned to the reference);
  * without a CUDA device the product fails loudly (no CPU fallback).
"""
import ctypes as C
import os
import re

import numpy as np
import pytest

import paper_2007_07539_b200 as mg
from oracle import FP16, FP32, FP64, Oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "mpmg_gpu.h")
O = Oracle()


def same_bits(a, b):
    a = np.asarray(a, dtype=np.float64); b = np.asarray(b, dtype=np.float64)
    return a.shape == b.shape and np.array_equal(a.view(np.uint64), b.view(np.uint64))


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"^[A-Za-z_][\w\s\*]*?\b(mpmg_\w+)\s*\(", src, flags=re.M)
    return sorted(set(names))


def test_library_exports_every_declared_symbol():
    L = mg.lib()
    names = declared_functions()
    assert len(names) >= 30, names
    missing = [n for n in names if not hasattr(L, n)]
    assert not missing, missing


def test_library_is_sm100a_only():
    so = open(mg.LIB_PATH, "rb").read()
    assert b"sm_100a" in so or b"sm_100" in so


@pytest.mark.parametrize("variant", ["h_mg", "hsd_mg", "dsh_mg", "d_mg"])
@pytest.mark.parametrize("dim,n,L", [(3, 33, 5), (2, 65, 6), (3, 65, 6)])
@pytest.mark.parametrize("ftz", [True, False])
def test_level_stencils_bitwise(variant, dim, n, L, ftz):
    """MgHierarchy::build per level (multigrid.cpp:282-323): the product's
    constant stencil equals every interior row of the reference's ELL operator
    and its D^-1 equals the reference's inv_diag, bitwise."""
    ho = O.hierarchy(dim, n, L, variant, ftz=ftz)
    for l in range(L):
        nl = ((n - 1) >> (L - 1 - l)) + 1
        s = mg.level_stencil(dim, nl, ho.prec(l), ftz)
        taps = s.taps_array()
        cols, vals = ho.matrix(l, 0)
        m = nl - 2
        # rows whose 3^dim neighbourhood is interior carry the full stencil in slot order
        idx = np.arange(m ** dim)
        coords = [(idx // m ** k) % m for k in range(dim)]
        inner = np.all([(c > 0) & (c < m - 1) for c in coords], axis=0)
        if inner.any():
            rows = vals[inner]
            assert np.all(rows.view(np.uint64) == taps.view(np.uint64)), (l, "stencil")
        assert np.all(ho.invdiag(l).view(np.uint64) == np.float64(s.inv_diag).view(np.uint64)), (l, "invdiag")


def test_binary16_overflow_raises_build_error():
    # cast_checked (multigrid.cpp:25-33): a coefficient above 65504 in binary16
    # is impossible for Poisson stencils (|a| <= 8/3), so probe the host rounding
    assert mg.lib().mpmg_round_fp16(65520.0, 1) == float("inf")
    assert mg.lib().mpmg_round_fp16(65519.0, 1) == 65504.0


def test_round_fp16_matches_oracle():
    rng = np.random.default_rng(3)
    xs = np.concatenate([rng.standard_normal(20000) * 10.0 ** rng.integers(-9, 5, 20000),
                         [0.0, -0.0, 2.0 ** -25, 3 * 2.0 ** -25, 65504.0, 65520.0]])
    for ftz in (0, 1):
        mine = [mg.lib().mpmg_round_fp16(x, ftz) for x in xs]
        ref = [O.q16(x, ftz) for x in xs]
        assert same_bits(mine, ref)


@pytest.mark.parametrize("dim,n", [(2, 33), (3, 17), (3, 33), (2, 129)])
def test_problem_rhs_bitwise(dim, n):  # assemble_rhs, mesh_fem.cpp:157-202
    assert same_bits(mg.problem_rhs(dim, n), O.rhs(dim, n))


@pytest.mark.parametrize("threads", ["1", "3", "16"])
@pytest.mark.parametrize("dim,n", [(3, 129), (2, 1025), (3, 41)])
def test_problem_rhs_threaded_bitwise(dim, n, threads, monkeypatch):
    """The layer-split threaded assembly adds every node's terms in the
    sequential element order: bitwise the reference's sum for any thread
    count (mesh_fem.cpp:157-202)."""
    monkeypatch.setenv("MPMG_RHS_THREADS", threads)
    assert same_bits(mg.problem_rhs(dim, n), O.rhs(dim, n))


def test_padded_layout_sizes():
    L = mg.lib()
    assert L.mpmg_padded_len(3, 257) == 256 ** 3 + 256 ** 2 + 256 + 1
    assert L.mpmg_padded_len(2, 9) == 64 + 8 + 1
    assert L.mpmg_interior_len(3, 257) == 255 ** 3
    assert [L.mpmg_bytes_per_value(p) for p in (FP16, FP32, FP64)] == [2, 4, 8]


def test_invalid_arguments_rejected_without_device():
    L = mg.lib()
    s = mg.Stencil()
    # stencil with a bad precision code -> EINVAL before any CUDA call
    assert L.mpmg_gpu_jacobi(C.byref(s), None, None, None, 2.0 / 3.0, 0, None) == -1
    assert L.mpmg_gpu_restrict(3, 4, 0, 0, None, None, None, 0, None) == -1
    cfg = mg.SolverConfig()
    L.mpmg_solver_default_config(C.byref(cfg))
    cfg.nodes = 66  # (n-1) not divisible by 2^(L-1): ProblemSpec::validate
    err, lvl = C.c_int(0), C.c_int(0)
    assert not L.mpmg_solver_create(C.byref(cfg), C.byref(err), C.byref(lvl))
    assert err.value == -1


def test_no_cpu_fallback():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(RuntimeError):
        mg.Hierarchy(3, 17, 4, "h_mg")
