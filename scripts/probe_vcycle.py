"""Bisect a V-cycle mismatch at large grids: level ops of every streaming
level and one whole V-cycle of a (dim, n, L, variant) hierarchy against the
implicit oracle (full vectors; minutes at 513^3).
    python scripts/probe_vcycle.py 513 9 d_mg"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import paper_2007_07539_b200 as mg
    from oracle import Oracle
    O = Oracle()
    n, L, variant = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3]
    ctx = O.ctx(False, True, False)
    h = mg.Hierarchy(3, n, L, variant, ftz=False)
    ho = O.hierarchy(3, n, L, variant, ftz=False, implicit=True)
    rng = np.random.default_rng(5)
    for l in range(L - 1, max(L - 5, 0), -1):
        prec = ho.prec(l)
        Nl = ho.rows(l)
        b = O.cast((rng.random(Nl) * 2 - 1), prec, 1.0, ctx)
        u = O.cast((rng.random(Nl) * 2 - 1) * 1e-3, prec, 1.0, ctx)
        t0 = time.time()
        res = {}
        res["jacobi2"] = (h.jacobi(l, b, u, 2), ho.jacobi(l, b, u, 2, ctx=ctx))
        res["jacobi_z3"] = (h.jacobi(l, b, None, 3), ho.jacobi(l, b, np.zeros(Nl), 3, ctx=ctx))
        res["restrict"] = (h.restrict(l, b), ho.restrict(l, b, False, ctx=ctx)[0])
        c = O.cast((rng.random(ho.rows(l - 1)) * 2 - 1) * 0.5, ho.prec(l - 1), 1.0, ctx)
        res["prolong"] = (h.prolong_correct(l, c, u), O.axpy(prec, 1.0, ho.prolong(l, c, 1.0, ctx=ctx), u, ctx))
        for k, (g, o) in res.items():
            bad = np.count_nonzero(g != o)
            print(f"level {l} (P={(n - 1) >> (L - 1 - l)}) {k}: {'OK' if bad == 0 else f'{bad} MISMATCHES'}", flush=True)
        print(f"  ({time.time() - t0:.1f} s)", flush=True)
    b = O.rhs(3, n)
    fp = ho.prec(L - 1)
    rl = O.cast(b, fp, O.norm2(b) if variant != "d_mg" else 1.0, ctx)
    cg = h.v_cycle(rl)
    co = ho.v_cycle(rl, ctx)
    bad = np.count_nonzero(cg != co)
    print("v_cycle:", "OK" if bad == 0 else f"{bad} MISMATCHES, rel diff {np.linalg.norm(cg - co) / np.linalg.norm(co):.3e}",
          flush=True)


if __name__ == "__main__":
    main()
