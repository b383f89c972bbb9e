"""BASELINE configs[4] on ONE B200: 3D Poisson 1025^3 (1,070,599,167
unknowns), L = 10, V(3,3), FP64 IR to 1e-10 ||b||, u0 = 0, FTZ off -- H_MG
and D_MG (device-resident, L2 irrelevant at this size), plus the checks the
reference cannot run at this size (its ELL would be ~700 GB):
  * both variants converge and their solutions agree within 1e-9 relative L2
    (any correct solver at this tolerance lands ~1e-11 apart);
  * the final TRUE residual ||b - A u|| (a fresh FP64 defect) is below the
    tolerance for D_MG (H_MG converges on the incrementally updated r, like
    the reference, ir_solver.cpp:96-104).
    python scripts/run_1025.py [out.json]
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import paper_2007_07539_b200 as mg
    lib = mg.lib()
    dim, n, L = 3, 1025, 10
    N = mg.unknowns(dim, n)
    t0 = time.perf_counter()
    b = mg.problem_rhs(dim, n)
    rhs_s = time.perf_counter() - t0
    nb = float(np.sqrt(np.dot(b, b)))
    tol = 1e-10 * nb
    bt = torch.from_numpy(b)
    del b
    out = {"config": "3D Poisson 1025^3 (1,070,599,167 unknowns), L=10, V(3,3), FP64 IR to 1e-10*||b||, u0 = 0, "
                     "FTZ off, one B200", "rhs_assembly_s": rhs_s, "tolerance": tol}
    sols = {}
    for variant in ("h_mg", "d_mg"):
        t0 = time.perf_counter()
        h = mg.Hierarchy(dim, n, L, variant, ftz=False)
        create_s = time.perf_counter() - t0
        bd, ud = h.device_buffers()
        btd = bt.cuda()
        mg._check(lib.mpmg_gpu_pack(dim, n, mg.FP64, btd.data_ptr(), bd, None), "pack")
        del btd
        torch.cuda.synchronize()
        cfg = mg.IrConfig(outer_tolerance=tol)
        reps = []
        for k in range(3):  # first = warm-up (graph capture)
            rep = h.ir_solve_ptr(bd, ud, cfg, device=True)
            reps.append(rep)
        rep = reps[-1]
        times = [r.device_seconds for r in reps[1:]]
        # solution back to the host (compact order)
        comp = torch.empty(N, dtype=torch.float64, device="cuda")
        mg._check(lib.mpmg_gpu_unpack(dim, n, mg.FP64, ud, comp.data_ptr(), None), "unpack")
        torch.cuda.synchronize()
        sols[variant] = comp.cpu()
        del comp
        free, total = torch.cuda.mem_get_info()
        out[variant] = {"seconds": float(np.mean(times)), "seconds_each": times, "iterations": rep.iterations,
                        "converged": rep.converged, "final_residual": rep.final_residual,
                        "final_true_residual_below_tol": rep.final_residual < tol, "cuda_graph": rep.used_graph,
                        "hierarchy_create_s": create_s, "device_mem_used_gb": (total - free) / 1e9}
        h.close()
        torch.cuda.empty_cache()
        print(variant, json.dumps(out[variant]), flush=True)
    du = (sols["h_mg"] - sols["d_mg"]).double()
    out["rel_l2_h_vs_d"] = float(torch.linalg.vector_norm(du) / torch.linalg.vector_norm(sols["d_mg"]))
    out["speedup_h_vs_d"] = out["d_mg"]["seconds"] / out["h_mg"]["seconds"]
    print(json.dumps(out))
    if len(sys.argv) > 1:
        with open(sys.argv[1], "w") as f:
            json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
