"""Per-level kernel timing inside a CUDA graph (warm L2, back-to-back
launches of the same op), H_MG binary16 levels of the 257^3 hierarchy:
the in-graph cost of each V-cycle operation at each level, launch gaps
included. Usage: python scripts/level_probe.py [reps]"""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2007_07539_b200 as mg


def main():
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
    lib = mg.lib()
    dev = torch.device("cuda:0")
    pol = mg.policy_word(False, True, False)
    print(f"{'nodes':>6} {'op':>10} {'us/launch':>10}")
    for n in (257, 129, 65, 33):
        plen = lib.mpmg_padded_len(3, n)
        nc = (n - 1) // 2 + 1
        pc = lib.mpmg_padded_len(3, nc)
        A = mg.level_stencil(3, n, mg.FP16, False)
        N = mg.unknowns(3, n)
        comp = ((torch.rand(N, device=dev, dtype=torch.float64) * 2 - 1) / N ** 0.5).to(torch.float16)
        b = torch.zeros(plen, dtype=torch.float16, device=dev)
        mg._check(lib.mpmg_gpu_pack(3, n, mg.FP16, comp.data_ptr(), b.data_ptr(), None), "pack")
        u = b.clone()
        u2 = torch.zeros_like(b)
        cc = torch.zeros(pc, dtype=torch.float16, device=dev)
        ops = {
            "jacobi": lambda sp: lib.mpmg_gpu_jacobi(C.byref(A), b.data_ptr(), u.data_ptr(), u2.data_ptr(),
                                                     2.0 / 3.0, pol, sp),
            "jacobi0": lambda sp: lib.mpmg_gpu_jacobi(C.byref(A), b.data_ptr(), None, u2.data_ptr(), 2.0 / 3.0,
                                                      pol, sp),
            "defect": lambda sp: lib.mpmg_gpu_defect(C.byref(A), b.data_ptr(), u.data_ptr(), u2.data_ptr(), pol, sp),
            "restrict": lambda sp: lib.mpmg_gpu_restrict(3, n, mg.FP16, mg.FP16, u.data_ptr(), cc.data_ptr(), None,
                                                         pol, sp),
            "prolong": lambda sp: lib.mpmg_gpu_prolong_correct(3, n, mg.FP16, mg.FP16, cc.data_ptr(),
                                                               u2.data_ptr(), None, pol, sp),
        }
        for name, fn in ops.items():
            s = torch.cuda.Stream(dev)
            with torch.cuda.stream(s):
                mg._check(fn(s.cuda_stream), name)  # warm-up / attributes
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s):
                for _ in range(reps):
                    fn(s.cuda_stream)
            with torch.cuda.stream(s):
                g.replay()
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            best = 1e9
            with torch.cuda.stream(s):
                for _ in range(5):
                    e0.record(s)
                    g.replay()
                    e1.record(s)
                    e1.synchronize()
                    best = min(best, e0.elapsed_time(e1) * 1e3 / reps)
            print(f"{n:>6} {name:>10} {best:>10.2f}", flush=True)


if __name__ == "__main__":
    main()
