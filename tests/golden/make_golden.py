"""Generates tests/golden/*.npz from the UNMODIFIED reference library.

Test infrastructure only. Runs in the build container, where /root/reference
exists and `make -C oracle` has compiled it into oracle/_ref/libmpmg_ref.so
(the reference's own six source files, its own flags). The fixtures pin the
oracle restatement (oracle/mpmg_oracle.c) and, through it, the GPU path, on
machines without /root/reference (the GPU box).

    python tests/golden/make_golden.py

Contents (all values in the binary64 value domain, every binary16/32 value
exact):
  kernels.npz     random-ELL spmv per precision/policy (test_kernels.cpp:108-145
                  restated: n in {3, 8, 17, 32}, SplitMix64 seed 42), fused
                  update_residuum_correction (kernels.cpp:300-341), scaled cast
                  (kernels.cpp:343-360)
  hierarchy.npz   per-level precision, stencil taps, inv_diag, full A/P/R ELL
                  arrays of small hierarchies (MgHierarchy::build,
                  multigrid.cpp:282-323; assemble_* mesh_fem.cpp:71-295)
  cycles.npz      V-cycle outputs (multigrid.cpp:354-393) and CG base solves
  solves.npz      ir_solve residual histories / iteration counts
                  (ir_solver.cpp:51-127), incl. BASELINE configs[0]
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import FP16, FP32, FP64, Reference  # noqa: E402

VARIANTS = ["d_mg", "h_mg", "dsh_mg", "hsd_mg"]


class SplitMix64:
    """rng.hpp:9-25 (SplitMix64; next_double = top 53 bits * 2^-53)."""

    def __init__(self, seed):
        self.s = seed & 0xFFFFFFFFFFFFFFFF

    def next_u64(self):
        self.s = (self.s + 0x9E3779B97F4A7C15) & 0xFFFFFFFFFFFFFFFF
        z = self.s
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & 0xFFFFFFFFFFFFFFFF
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & 0xFFFFFFFFFFFFFFFF
        return z ^ (z >> 31)

    def next_double(self):
        return (self.next_u64() >> 11) * 2.0 ** -53


def random_ell(rng, n, per_row):
    """Random sparse system: per row up to `per_row` distinct columns
    (ascending) with values in [-1, 1); padded with (col=row, 0)."""
    rw = per_row
    cols = np.zeros((n, rw), dtype=np.int32)
    vals = np.zeros((n, rw))
    for i in range(n):
        cs = sorted({int(rng.next_u64() % n) for _ in range(per_row)})
        for s, c in enumerate(cs):
            cols[i, s] = c
            vals[i, s] = 2.0 * rng.next_double() - 1.0
        for s in range(len(cs), rw):
            cols[i, s] = min(i, n - 1)
    return cols, vals


def kernels(R):
    out = {}
    rng = SplitMix64(42)
    k = 0
    for prec in (FP16, FP32, FP64):
        for n in (3, 8, 17, 32):
            for rep in range(8):
                cols, vals = random_ell(rng, n, 6)
                x = np.array([2.0 * rng.next_double() - 1.0 for _ in range(n)])
                # magnitudes spanning the binary16 subnormal range on half the reps
                if rep % 2:
                    x *= 1e-4
                out[f"spmv_{k}_cols"] = cols
                out[f"spmv_{k}_vals"] = vals
                out[f"spmv_{k}_x"] = x
                out[f"spmv_{k}_prec"] = np.array(prec)
                for ftz in (0, 1):
                    for fma in (0, 1):
                        for acc32 in ((0, 1) if prec == FP16 else (0,)):
                            y = R.ell_spmv(cols, vals, prec, x, ftz=ftz, fma=fma, acc32=acc32)
                            out[f"spmv_{k}_y_{ftz}{fma}{acc32}"] = y
                k += 1
    out["spmv_count"] = np.array(k)
    # fused outer update on a real 3D operator (9^3 grid), c in 3 precisions
    rng = SplitMix64(11)
    dim, n = 3, 9
    N = (n - 2) ** 3
    j = 0
    for cp in (FP16, FP32, FP64):
        for ftz in (0, 1):
            c = np.array([(2.0 * rng.next_double() - 1.0) for _ in range(N)])
            c = R.cast(c, FP64, cp, 1.0, ftz=ftz)
            r = np.array([rng.next_double() for _ in range(N)])
            u = np.array([rng.next_double() for _ in range(N)])
            alpha = 2.0 * rng.next_double()
            r2, u2 = R.update_rc(dim, n, r, u, c, cp, alpha, ftz=ftz)
            for nm, v in (("c", c), ("r", r), ("u", u), ("r_out", r2), ("u_out", u2)):
                out[f"urc_{j}_{nm}"] = v
            out[f"urc_{j}_meta"] = np.array([dim, n, cp, ftz, alpha])
            j += 1
    out["urc_count"] = np.array(j)
    # scaled casts (cast_vector): tiny residual, scale = its norm
    rng = SplitMix64(13)
    x = np.array([(2.0 * rng.next_double() - 1.0) * 1e-7 for _ in range(50)])
    nx = R.norm2(x)
    out["cast_x"] = x
    out["cast_norm"] = np.array(nx)
    for ftz in (0, 1):
        for tgt in (FP16, FP32):
            out[f"cast_{tgt}_{ftz}_scaled"] = R.cast(x, FP64, tgt, nx, ftz=ftz)
            out[f"cast_{tgt}_{ftz}_unscaled"] = R.cast(x, FP64, tgt, 1.0, ftz=ftz)
    return out


def hierarchy(R):
    out = {}
    for dim, n, L in ((2, 17, 4), (3, 9, 3), (2, 65, 6), (3, 33, 5)):
        for variant in VARIANTS:
            for ftz in (0, 1):
                h = R.hierarchy(dim, n, L, variant, ftz=ftz)
                key = f"{dim}_{n}_{variant}_{ftz}"
                out[f"{key}_prec"] = np.array([h.prec(l) for l in range(L)])
                out[f"{key}_rows"] = np.array([h.rows(l) for l in range(L)])
                for l in range(L):
                    cols, vals = h.matrix(l, 0)
                    # centre row's taps (the per-level stencil) + all-rows check
                    out[f"{key}_l{l}_invdiag"] = h.invdiag(l)
                    if n <= 17:
                        out[f"{key}_l{l}_A_cols"] = cols
                        out[f"{key}_l{l}_A_vals"] = vals
                        if l < L - 1:  # coarse level holds the transfers to the finer one
                            for w, nm in ((1, "P"), (2, "R")):
                                c2, v2 = h.matrix(l, w)
                                out[f"{key}_l{l}_{nm}_cols"] = c2
                                out[f"{key}_l{l}_{nm}_vals"] = v2
                    else:
                        m = (n - 1) >> (L - 1 - l)
                        c = (m - 2) // 2  # interior centre node
                        row = c + (m - 1) * c + ((m - 1) ** 2 * c if dim == 3 else 0)
                        out[f"{key}_l{l}_A_row"] = vals[row]
    for dim, n in ((2, 5), (2, 9), (2, 33), (2, 257), (3, 5), (3, 9), (3, 17), (3, 65), (3, 129), (3, 257)):
        out[f"stencil_{dim}_{n}"] = R.stencil(dim, n)
    for dim, n in ((2, 33), (3, 17)):
        b, ue = R.rhs(dim, n)
        out[f"rhs_{dim}_{n}"] = b
        out[f"exact_{dim}_{n}"] = ue
    return out


def cycles(R):
    out = {}
    for dim, n, L in ((2, 33, 5), (3, 17, 4), (3, 33, 5)):
        b, _ = R.rhs(dim, n)
        for variant in VARIANTS:
            for ftz in (0, 1):
                for acc32 in (0, 1):
                    if n > 17 and dim == 3 and (acc32 or variant not in ("h_mg", "hsd_mg")):
                        continue  # keep the fixture small
                    h = R.hierarchy(dim, n, L, variant, ftz=ftz)
                    fp = h.prec(L - 1)
                    scale = R.norm2(b) if variant != "d_mg" else 1.0
                    rl = R.cast(b, FP64, fp, scale, ftz=ftz)
                    key = f"{dim}_{n}_{variant}_{ftz}_{acc32}"
                    out[f"vc_{key}_in"] = rl
                    out[f"vc_{key}_out"] = h.v_cycle(rl, acc32=bool(acc32))
    # CG base solves on 15^2 / 7^3 level-0 grids
    rng = SplitMix64(5)
    for dim, n in ((2, 65), (3, 33)):
        for variant in ("d_mg", "h_mg", "hsd_mg"):
            h = R.hierarchy(dim, n, 3, variant, ftz=1)
            N0 = h.rows(0)
            x = np.array([2.0 * rng.next_double() - 1.0 for _ in range(N0)])
            bb = R.cast(x, FP64, h.prec(0), 1.0, ftz=1)
            u, it, conv, res = h.cg(0, bb)
            key = f"cg_{dim}_{n}_{variant}"
            out[f"{key}_b"] = bb
            out[f"{key}_u"] = u
            out[f"{key}_meta"] = np.array([it, int(conv), res])
    return out


def solves(R):
    out = {}
    cases = [
        # BASELINE.json configs[0]: 65^3, FP64 V(2,2) Jacobi-MG preconditioned IR
        ("cfg0", 3, 65, 6, "d_mg", 2, 2, 1),
        ("3_65_h_mg_ftz0", 3, 65, 6, "h_mg", 3, 3, 0),
        ("3_65_h_mg_ftz1", 3, 65, 6, "h_mg", 3, 3, 1),
        ("3_65_hsd_mg_ftz0", 3, 65, 6, "hsd_mg", 3, 3, 0),
        ("3_65_dsh_mg_ftz0", 3, 65, 6, "dsh_mg", 3, 3, 0),
        ("3_65_d_mg_ftz0", 3, 65, 6, "d_mg", 3, 3, 0),
        ("2_257_h_mg_ftz0", 2, 257, 8, "h_mg", 3, 3, 0),
        ("2_257_hsd_mg_ftz1", 2, 257, 8, "hsd_mg", 3, 3, 1),
        ("3_33_h_mg_ftz0", 3, 33, 5, "h_mg", 3, 3, 0),
    ]
    for name, dim, n, L, variant, pre, post, ftz in cases:
        h = R.hierarchy(dim, n, L, variant, pre=pre, post=post, ftz=ftz)
        s = h.ir_solve(rel_tol=1e-10, want_u=(n <= 33))
        out[f"{name}_meta"] = np.array([dim, n, L, ["d_mg", "h_mg", "dsh_mg", "hsd_mg"].index(variant), pre, post,
                                        ftz, s["iterations"], int(s["converged"])])
        out[f"{name}_history"] = s["history"]
        out[f"{name}_final"] = np.array(s["final_residual"])
        if n <= 33:
            out[f"{name}_u"] = s["u"]
        print(name, s["iterations"], s["history"][-1], flush=True)
    return out


def main():
    R = Reference()
    for name, fn in (("kernels", kernels), ("hierarchy", hierarchy), ("cycles", cycles), ("solves", solves)):
        d = fn(R)
        path = os.path.join(HERE, f"{name}.npz")
        np.savez_compressed(path, **d)
        print(f"wrote {path}: {len(d)} arrays, {os.path.getsize(path) / 1024:.0f} KiB", flush=True)


if __name__ == "__main__":
    main()
