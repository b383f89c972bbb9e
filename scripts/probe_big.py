"""Large-grid probe: one solve per (variant, nodes) with its residual history
(stagnation / scaling behaviour of the pure binary16 cycle at 513^3 and
1025^3).  python scripts/probe_big.py 513:h_mg 1025:d_mg ..."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    import paper_2007_07539_b200 as mg
    lib = mg.lib()
    for spec in sys.argv[1:]:
        n, variant = spec.split(":")
        n = int(n)
        L = {129: 7, 257: 8, 513: 9, 1025: 10}[n]
        t0 = time.perf_counter()
        b = mg.problem_rhs(3, n)
        tol = 1e-10 * float(np.sqrt(np.dot(b, b)))
        print(spec, "rhs", round(time.perf_counter() - t0, 1), "s", flush=True)
        h = mg.Hierarchy(3, n, L, variant, ftz=False)
        print(spec, "created", flush=True)
        u, rep = h.ir_solve(b, mg.IrConfig(outer_tolerance=tol, max_outer_iterations=40))
        print(spec, "its", rep.iterations, "conv", rep.converged, "dev_s", round(rep.device_seconds, 4), "wall_s",
              round(rep.wall_seconds, 2), "final", rep.final_residual, flush=True)
        print(spec, "history", " ".join(f"{x:.3e}" for x in rep.residual_history), flush=True)
        h.close()
        del u, b
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
