"""Multi-GPU solver overhead on ONE B200 (no multi-GPU box in this run):
W z-slab ranks of csrc/mpmg_dist.cu (one thread + one stream each, raw peer
pointers) solve the problem concurrently on the same GPU. Together they do
the single-GPU solve's work plus the multi-GPU extras (halo handshakes, the
replicated agglomerated coarse cycle, the norm slot exchange), so

    overhead(W) = t_dist(W ranks sharing one GPU) / t_single - 1

bounds what the decomposition costs per solve; it says nothing about NVLink
bandwidth (the halos move through the same HBM here).
    python scripts/dist_proxy.py [nodes] [levels] [variant] [worlds...] [--out f.json]
"""
import json
import os
import sys
import threading

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    args = [x for x in sys.argv[1:] if not x.startswith("--")]
    out_path = sys.argv[sys.argv.index("--out") + 1] if "--out" in sys.argv else None
    if out_path in args:
        args.remove(out_path)
    n = int(args[0]) if args else 513
    L = int(args[1]) if len(args) > 1 else 9
    variant = args[2] if len(args) > 2 else "h_mg"
    worlds = [int(w) for w in args[3:]] or [1, 2, 4]
    import ctypes as C

    import torch

    import paper_2007_07539_b200 as mg
    from paper_2007_07539_b200.dist import DistSolver
    lib = mg.lib()
    lib.mpmg_dev_h2d.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t]
    b = mg.problem_rhs(3, n)
    tol = 1e-10 * float(np.sqrt(np.dot(b, b)))
    P, m = n - 1, n - 2
    res = {"nodes": n, "levels": L, "variant": variant}
    # single-GPU solver, device-resident
    h = mg.Hierarchy(3, n, L, variant, ftz=False)
    bd, ud = h.device_buffers()
    bt = torch.from_numpy(b).cuda()
    mg._check(lib.mpmg_gpu_pack(3, n, mg.FP64, bt.data_ptr(), bd, None), "pack")
    del bt
    cfg = mg.IrConfig(outer_tolerance=tol)
    ts = []
    for k in range(4):
        rep = h.ir_solve_ptr(bd, ud, cfg, device=True)
        if k:
            ts.append(rep.device_seconds)
    res["single"] = {"seconds": float(np.min(ts)), "iterations": rep.iterations}
    h.close()
    torch.cuda.empty_cache()
    print("single", res["single"], flush=True)
    bc = b.reshape(m, m, m)
    for W in worlds:
        for fuse in ("1", "0") if W > 1 else ("1",):
            os.environ["MPMG_DIST_FUSE_HALOS"] = fuse
            ranks = [DistSolver(n, L, variant, r, W, ftz=False) for r in range(W)]
            blobs = [r.blob for r in ranks]
            for r in ranks:
                r.connect(blobs)
            for r in ranks:
                bptr, _ = r.buffers()
                slab = np.zeros((r.nz + 2, P, P))
                slab[1:1 + r.nz, 1:P, 1:P] = bc[r.z_lo - 1:r.z_lo - 1 + r.nz]
                mg._check(lib.mpmg_dev_h2d(bptr, slab.ctypes.data, slab.nbytes), "h2d")
                del slab
            for r in ranks:
                r.prepare(tol)
            stats = [r.exchange_stats() for r in ranks]
            times, its = [], None
            for k in range(4):
                out = [None] * W
                th = [threading.Thread(target=lambda i=i: out.__setitem__(i, ranks[i].solve(tol))) for i in range(W)]
                for t in th:
                    t.start()
                for t in th:
                    t.join()
                its = out[0][0].iterations
                if k:
                    times.append(max(o[0].device_seconds for o in out))
            key = f"W{W}" + ("" if W == 1 else ("_fused" if fuse == "1" else "_copy"))
            res[key] = {"seconds": float(np.min(times)), "iterations": its,
                        "overhead_vs_single": float(np.min(times)) / res["single"]["seconds"] - 1.0,
                        "exchanges_fused_copied_rank0": stats[0]}
            print(key, res[key], flush=True)
            for r in ranks:
                r.close()
            torch.cuda.empty_cache()
    print(json.dumps(res))
    if out_path:
        with open(out_path, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
