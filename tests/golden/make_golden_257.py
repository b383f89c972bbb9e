"""Generates tests/golden/solves257_<variant>.npz: the UNMODIFIED reference's ir_solve at
the headline configuration (BASELINE.json configs[1]/[2]: 3D Poisson 257^3,
L = 8, V(3,3), damped Jacobi w = 2/3, u0 = 0, ||r|| <= 1e-10 ||b||, FTZ off,
FMA on) for D_MG, H_MG and HSD_MG.

Test infrastructure only. Needs oracle/_ref/libmpmg_ref.so (make -C oracle,
in the build container where /root/reference exists). Each solve takes
2-11 minutes on one core (the reference is single-threaded), so this is a
separate script from make_golden.py:

    python tests/golden/make_golden_257.py [variant ...]

Stored per variant (the full 133 MB solution cannot be committed):
  meta      [iterations, converged, wall_s, build_s]
  history   ||r|| per outer iteration (ir_solver.cpp:96-104)
  final     SolveReport.final_residual (ir_solver.cpp:120-123)
  u_norm    ||u||_2 (sequential fma, kernels.cpp:384-395 order)
  u_sum     sum of u in index order
  u_sample  u[::STRIDE] (compact interior order, every STRIDE-th unknown)
  err_l2    nodal_l2_error against the manufactured exact solution
"""
from __future__ import annotations

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import Reference  # noqa: E402

STRIDE = 997  # prime: the sample walks through every x/y/z residue class


def main(variants):
    R = Reference()
    for spec in variants:  # "h_mg" (FTZ off), "h_mg:1" (FTZ on, the reference default), "2d:h_mg" (8193^2)
        dim, n, L = 3, 257, 8
        if spec.startswith("2d:"):
            dim, n, L, spec = 2, 8193, 13, spec[3:]
        variant, _, f = spec.partition(":")
        ftz = int(f or 0)
        tag = "257" if dim == 3 else "8193_2d"
        path = os.path.join(HERE, f"solves{tag}_{variant}" + ("_ftz1" if ftz else "") + ".npz")
        out = {"stride": np.array(STRIDE)}
        t0 = time.perf_counter()
        h = R.hierarchy(dim, n, L, variant, pre=3, post=3, ftz=ftz)
        build_s = time.perf_counter() - t0
        s = h.ir_solve(rel_tol=1e-10, want_u=True)
        u = s["u"]
        key = f"{variant}_ftz{ftz}"
        out[f"{key}_meta"] = np.array([s["iterations"], int(s["converged"]), s["wall_s"], build_s])
        out[f"{key}_history"] = s["history"]
        out[f"{key}_final"] = np.array(s["final_residual"])
        out[f"{key}_u_norm"] = np.array(R.norm2(u))
        out[f"{key}_u_sum"] = np.array(float(np.sum(u)))
        out[f"{key}_u_sample"] = u[::STRIDE].copy()
        out[f"{key}_err_l2"] = np.array(s["err_l2"])
        np.savez_compressed(path, **out)
        print(f"{spec}: {s['iterations']} its, final {s['final_residual']:.6e}, solve {s['wall_s']:.1f} s, "
              f"build {build_s:.1f} s", flush=True)
        del h, u


if __name__ == "__main__":
    main(sys.argv[1:] or ["d_mg", "h_mg", "hsd_mg"])
