"""Benchmark of the B200 hot path (BASELINE.json metric):

  "IR-MG time to 1e-10 rel. residual (s), FP16/mixed vs FP64; kernel HBM GB/s"

Workload (BASELINE.json configs[1]): 3D Poisson on the unit cube, 257^3 nodes
(255^3 = 16,581,375 unknowns), L = 8 levels, V(3,3) damped Jacobi (omega 2/3),
FP64 iterative refinement preconditioned by one pure-binary16 V-cycle with
residuum scaling (H_MG), u0 = 0, stopping at ||r||_2 <= 1e-10 ||b||_2. The
same solver in all-binary64 (D_MG, the same fused kernels at 8 bytes/value) is
timed beside it. Arithmetic policy: flush_subnormals_to_zero = false,
fused_multiply_add = true (SURVEY §7 hard part 2; the reference default
flushes, `--ftz 1` selects it).

One "step" = one complete ir_solve (device-resident inputs for `value`; host
buffers through the C ABI for `e2e`). Every FP64 level vector of the finest
grid is 133 MB and the three of them exceed the 126 MB L2; the L2 is
additionally flushed (a 512 MiB write) before every timed solve.

`--impl reference` times the reference's own CPU implementation (the
unmodified library compiled from /root/reference into oracle/_ref/) on the
same workload: one complete 257^3 solve (~10 minutes on one core), see
run_reference(). The B200 arm's `cpu_baseline` is a bounded, measured sample
(one complete reference solve at 65^3): see cpu_reference().
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "IR-MG time to 1e-10 rel. residual (s), FP16/mixed vs FP64; kernel HBM GB/s"
UNIT = "s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--dim", type=int, default=3)
    ap.add_argument("--nodes", type=int, default=257)
    ap.add_argument("--levels", type=int, default=0, help="0 = max depth (base 3 nodes/dim)")
    ap.add_argument("--variant", default="h_mg", choices=["h_mg", "hsd_mg", "dsh_mg", "d_mg"])
    ap.add_argument("--ftz", type=int, default=0)
    ap.add_argument("--pre", type=int, default=3)
    ap.add_argument("--post", type=int, default=3)
    ap.add_argument("--rel-tol", type=float, default=1e-10)
    ap.add_argument("--no-fp64", action="store_true", help="skip the all-FP64 comparison solve")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-kernels", action="store_true", help="skip the per-kernel roofline timing")
    ap.add_argument("--kernel-reps", type=int, default=20)
    ap.add_argument("--only-kernels", action="store_true", help="per-kernel timing only (for ncu captures)")
    ap.add_argument("--no-graph", action="store_true",
                    help="host-driven IR loop instead of the graph WHILE node (ncu cannot profile conditional graphs)")
    ap.add_argument("--no-extra", action="store_true",
                    help="skip the secondary BASELINE configs (HSD_MG 257^3, FTZ-on 257^3, 2D 8193^2)")
    return ap.parse_args()


def max_depth(n):
    L = 1
    while ((n - 1) >> L) >= 2 and ((n - 1) % (1 << L)) == 0:
        L += 1
    return L


def dist_info():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


# ---------------------------------------------------------------------------
# clocks: nvidia-smi sampled during the timed region
# ---------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,utilization.gpu,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.idx = gpu_index
        self.p = None
        self.path = os.path.join("/tmp", f"mpmg_clocks_{os.getpid()}.csv")

    def start(self):
        try:
            self.f = open(self.path, "w")
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.FIELDS}",
                                       "--format=csv,noheader,nounits", "-lms", "50"], stdout=self.f,
                                      stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.12)
        self.p.terminate()
        try:
            self.p.wait(timeout=5)
        except Exception:
            self.p.kill()
        self.f.close()
        rows = []
        with open(self.path) as f:
            for line in f:
                parts = [x.strip() for x in line.split(",")]
                if len(parts) < 10:
                    continue
                try:
                    rows.append(parts)
                except Exception:
                    pass
        os.unlink(self.path)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"], "samples": 0}

        def num(x):
            try:
                return float(x)
            except ValueError:
                return None
        load = [r for r in rows if (num(r[3]) or 0) >= 50] or rows
        sm = sorted(num(r[1]) for r in load if num(r[1]) is not None)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[6 + i].lower() == "active"})
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": num(rows[0][2]), "reasons": reasons,
                "samples": len(rows), "samples_under_load": len(load),
                "power_w_max": max((num(r[4]) or 0) for r in rows)}


# ---------------------------------------------------------------------------
# B200 arm
# ---------------------------------------------------------------------------
def run_b200(a):
    import numpy as np
    import torch

    import paper_2007_07539_b200 as mg

    ws, rank, local = dist_info()
    torch.cuda.set_device(local)
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    L = a.levels or max_depth(a.nodes)
    dim, n = a.dim, a.nodes
    N = mg.unknowns(dim, n)
    ftz = bool(a.ftz)
    lib = mg.lib()

    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)

    def flush_l2():
        flush.fill_(1.0)
        torch.cuda.synchronize()

    # host problem setup (assemble_rhs on the host, once)
    b = mg.problem_rhs(dim, n)
    tol = a.rel_tol * float(np.sqrt(np.dot(b, b)))
    cfgs = [(a.variant, "mixed")] + ([] if (a.no_fp64 or a.variant == "d_mg") else [("d_mg", "fp64")])
    if a.only_kernels:
        print(json.dumps(kernel_roofline(a, dim, n, L, ftz, dev, flush_l2)))
        return
    results = {}
    sampler = ClockSampler(local)
    launches_per_solve = {}
    for variant, tag in cfgs:
        h = mg.Hierarchy(dim, n, L, variant, pre=a.pre, post=a.post, ftz=ftz, device=local)
        bd, ud = h.device_buffers()
        # upload the rhs into the solver's padded FP64 buffer
        bt = torch.from_numpy(b).to(dev)
        torch.cuda.synchronize()
        mg._check(lib.mpmg_gpu_pack(dim, n, mg.FP64, bt.data_ptr(), bd, None), "pack")
        torch.cuda.synchronize()
        cfg = mg.IrConfig(outer_tolerance=tol, use_graph=not a.no_graph)
        for _ in range(a.warmup):
            flush_l2()
            rep = h.ir_solve_ptr(bd, ud, cfg, device=True)
        if tag == "mixed":
            sampler.start()
        if ws > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        times, its = [], []
        for _ in range(a.steps):
            flush_l2()
            rep = h.ir_solve_ptr(bd, ud, cfg, device=True)  # CUDA events on the solver stream
            times.append(rep.device_seconds)
            its.append(rep.iterations)
            graph_used = rep.used_graph
            assert rep.converged, f"{variant} did not converge"
        torch.cuda.synchronize()
        if ws > 1:
            torch.distributed.barrier()
        t = float(np.mean(times))
        if ws > 1:
            tt = torch.tensor([t], device=dev, dtype=torch.float64)
            torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
            t = float(tt.item())
        results[tag] = dict(variant=variant, seconds=t, iterations=int(its[-1]), min_s=float(np.min(times)),
                            final_residual=rep.final_residual, graph=bool(graph_used))
        launches_per_solve[tag] = solve_launches(h, its[-1], a, variant)
        if tag == "mixed":
            # e2e through the public C ABI with pinned HOST buffers: H2D of b,
            # pack, solve, unpack, D2H of u inside the timed region
            bh = torch.from_numpy(b).pin_memory()
            uh = torch.empty(N, dtype=torch.float64).pin_memory()
            for _ in range(max(1, a.warmup)):
                flush_l2()
                h.ir_solve_ptr(bh.data_ptr(), uh.data_ptr(), cfg, device=False)
            e2e = []
            for _ in range(a.steps):
                flush_l2()
                t0 = time.perf_counter()
                rep = h.ir_solve_ptr(bh.data_ptr(), uh.data_ptr(), cfg, device=False)
                e2e.append(time.perf_counter() - t0)
            e2e_t = float(np.mean(e2e))
            if ws > 1:
                tt = torch.tensor([e2e_t], device=dev, dtype=torch.float64)
                torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
                e2e_t = float(tt.item())
            results["e2e"] = e2e_t
        h.close()
        del bt
        torch.cuda.empty_cache()

    kernels = {} if a.no_kernels else kernel_roofline(a, dim, n, L, ftz, dev, flush_l2)
    clocks = sampler.stop()
    extra = None
    if not a.no_extra and ws == 1 and dim == 3 and n == 257 and a.variant == "h_mg" and not ftz:
        extra = extra_configs(a, dev, flush_l2)

    if rank != 0:
        if ws > 1:
            torch.distributed.destroy_process_group()
        return
    mix = results["mixed"]
    peaks = load_peaks()
    out = {
        "metric": METRIC, "value": mix["seconds"], "unit": UNIT, "n_gpus": ws, "steps": a.steps, "warmup": a.warmup,
        "ms_per_step": mix["seconds"] * 1e3, "higher_is_better": False, "scaling": "weak",
        "vs_baseline": None, "dtype": "fp16" if a.variant == "h_mg" else "mixed fp16/fp32/fp64",
        "data": "synthetic: the reference's own manufactured Poisson problem (assemble_rhs k=1), u0 = 0",
        "config": {"workload": f"{dim}D Poisson {n}^{dim} ({N} unknowns), L={L}, V({a.pre},{a.post}) Jacobi "
                               f"w=2/3, {a.variant.upper()} preconditioned FP64 IR to {a.rel_tol:g}*||b||",
                   "variant": a.variant, "policy": {"flush_subnormals_to_zero": ftz, "fused_multiply_add": True,
                                                    "fp16_accumulation": "fp16"},
                   "l2": "flushed (512 MiB write) before every timed solve; finest FP64 vectors 3x133 MB > L2",
                   "parallelism": "replicas only (one independent solve per GPU)" if ws > 1 else "1 GPU"},
        "iterations": mix["iterations"],
        "cuda_graph": mix["graph"],
        "final_residual": mix["final_residual"],
        "tolerance": tol,
    }
    if "fp64" in results:
        d = results["fp64"]
        out["fp64_baseline"] = {"variant": "d_mg", "seconds": d["seconds"], "iterations": d["iterations"],
                                "speedup_mixed_vs_fp64": d["seconds"] / mix["seconds"]}
    out["e2e"] = {"value": results["e2e"], "unit": UNIT, "h2d_bytes_per_step": 8 * N,
                  "d2h_bytes_per_step": 8 * N + 32 + 8,  # solution + IR state + final norm
                  "path": "mpmg_solver_solve (C ABI, pinned host b/u)"}
    out["gpu_launches"] = launches_per_solve["mixed"] * a.steps
    out["gpu_launches_per_solve"] = launches_per_solve
    if kernels:
        dom = kernels[kernels["dominant"]]
        traffic = None
        try:
            with open(os.path.join(ROOT, "profiles", "round2_roofline_traffic.json")) as f:
                traffic = json.load(f).get(kernels["dominant"], {}).get("traffic")
        except Exception:
            pass
        out["roofline"] = {"bound": "hbm", "achieved": dom["achieved_gbs"], "peak": peaks["hbm_gbs"],
                           "unit": "GB/s", "frac": dom["achieved_gbs"] / peaks["hbm_gbs"],
                           "traffic": traffic, "kernel": kernels["dominant"],
                           "algorithmic_bytes": dom["bytes"], "avg_us": dom["avg_us"],
                           "peak_source": peaks["source"]}
        if kernels["dominant"] == "jacobi_fine" and a.variant in ("h_mg", "hsd_mg") and dim == 3:
            # the binary16 27-point step is FMA-pipe bound on sm_100a: HFMA2 issues
            # at 0.5 warp-instructions / clock / SM sub-partition (measured,
            # profiles/round2_probe_hfma2_rate.txt); 21 live taps + the 3-op
            # epilogue = 12 HFMA2-class thread-instructions per unknown
            sms = torch.cuda.get_device_properties(dev).multi_processor_count
            mhz = float(clocks.get("sm_mhz") or 1965.0)
            floor_us = (12.0 * N / 32.0) * 2.0 / (sms * 4) / (mhz * 1e6) * 1e6  # warp-instructions x 2 clk
            out["roofline"]["fma_pipe"] = {"floor_us": floor_us, "frac": floor_us / dom["avg_us"],
                                           "model": "12 HFMA2-class thread-instructions per unknown at 0.5 warp-inst/clk/SMSP"}
        out["kernels"] = {k: v for k, v in kernels.items() if k != "dominant"}
    if extra:
        out["configs"] = extra
    out["clocks"] = clocks
    if not a.no_cpu and ws == 1:
        try:
            out["cpu_baseline"] = cpu_reference(a, dim, n, L, ftz)
        except Exception as ex:  # reported, not fatal
            out["cpu_baseline"] = {"error": str(ex)[:200]}
    print(json.dumps(out), flush=True)
    if ws > 1:
        torch.distributed.destroy_process_group()


def extra_configs(a, dev, flush_l2):
    """The other BASELINE.json configs on one B200 (device time per solve,
    L2 flushed before each, CUDA events on the solver stream):
      configs[2]  3D 257^3 HSD_MG (FP16 fine / FP32 / FP64 coarse) vs D_MG;
      the reference-default policy (FTZ on) at 257^3: H_MG and D_MG;
      configs[3]  2D 8193^2 (L = 13) H_MG vs D_MG, plus the finest 2D
                  Jacobi kernel (k_row2d) against the HBM roofline;
      configs[4]  its 1025^3 grid on one GPU, H_MG vs D_MG."""
    import numpy as np
    import torch

    import paper_2007_07539_b200 as mg
    lib = mg.lib()
    steps = max(2, min(a.steps, 5))

    def solve(dim, n, variant, ftz):
        big = n > 513
        L = max_depth(n)
        b = mg.problem_rhs(dim, n)
        tol = a.rel_tol * float(np.sqrt(np.dot(b, b)))
        h = mg.Hierarchy(dim, n, L, variant, ftz=ftz)
        bd, ud = h.device_buffers()
        bt = torch.from_numpy(b).to(dev)
        mg._check(lib.mpmg_gpu_pack(dim, n, mg.FP64, bt.data_ptr(), bd, None), "pack")
        torch.cuda.synchronize()
        cfg = mg.IrConfig(outer_tolerance=tol)
        for _ in range(1 if big else 2):
            flush_l2()
            rep = h.ir_solve_ptr(bd, ud, cfg, device=True)
        times = []
        for _ in range(2 if big else steps):
            flush_l2()
            rep = h.ir_solve_ptr(bd, ud, cfg, device=True)
            times.append(rep.device_seconds)
        h.close()
        del bt
        torch.cuda.empty_cache()
        return {"seconds": float(np.mean(times)), "iterations": rep.iterations, "converged": rep.converged,
                "final_residual": rep.final_residual, "tolerance": tol, "steps": steps}

    out = {}
    d0 = solve(3, 257, "d_mg", False)
    hsd = solve(3, 257, "hsd_mg", False)
    out["hsd_mg_257"] = {"config": "BASELINE configs[2]: 3D 257^3, L=8, HSD_MG (binary16 levels 3-7, binary32 "
                                   "level 2, binary64 levels 0-1), FTZ off", **hsd,
                         "d_mg_seconds": d0["seconds"], "d_mg_iterations": d0["iterations"],
                         "speedup_vs_fp64": d0["seconds"] / hsd["seconds"]}
    hf = solve(3, 257, "h_mg", True)
    df = solve(3, 257, "d_mg", True)
    out["ftz_on_257"] = {"config": "3D 257^3, L=8, the reference's default policy (binary16 subnormals flushed "
                                   "after rounding); H_MG stagnates like the reference (100 its, unconverged)",
                         "h_mg": hf, "d_mg": df}
    h2 = solve(2, 8193, "h_mg", False)
    d2 = solve(2, 8193, "d_mg", False)
    n2 = 8193
    N2 = mg.unknowns(2, n2)
    # finest 2D binary16 Jacobi: 3 x 2 bytes x N, operands rotated over 3 sets (> L2)
    plen = lib.mpmg_padded_len(2, n2)
    A = mg.level_stencil(2, n2, mg.FP16, False)
    sets = [(torch.zeros(plen, dtype=torch.float16, device=dev), torch.zeros(plen, dtype=torch.float16, device=dev),
             torch.zeros(plen, dtype=torch.float16, device=dev)) for _ in range(3)]
    stream = torch.cuda.current_stream(dev)
    sp = stream.cuda_stream
    pol = mg.policy_word(False, True, False)
    for bb, uu, oo in sets:
        mg._check(lib.mpmg_gpu_jacobi(C.byref(A), bb.data_ptr(), uu.data_ptr(), oo.data_ptr(), 2.0 / 3.0, pol, sp), "j")
    flush_l2()
    reps = 21
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for k in range(reps):
        bb, uu, oo = sets[k % 3]
        lib.mpmg_gpu_jacobi(C.byref(A), bb.data_ptr(), uu.data_ptr(), oo.data_ptr(), 2.0 / 3.0, pol, sp)
    e1.record(stream)
    e1.synchronize()
    avg = e0.elapsed_time(e1) * 1e-3 / reps
    peaks = load_peaks()
    jb = 3 * 2 * N2
    out["2d_8193"] = {"config": "BASELINE configs[3]: 2D 8193^2 (67,092,481 unknowns), L=13, V(3,3), FTZ off",
                      "h_mg": h2, "d_mg": d2, "speedup_vs_fp64": d2["seconds"] / h2["seconds"],
                      "jacobi_fine": {"bytes": jb, "avg_us": avg * 1e6, "achieved_gbs": jb / avg / 1e9,
                                      "frac": jb / avg / 1e9 / peaks["hbm_gbs"], "kernel": "k_row2d (binary16, 9-pt)"}}
    del sets
    torch.cuda.empty_cache()
    # configs[4]'s grid on ONE B200 (the slab-decomposed multi-GPU run needs a
    # multi-GPU node): 1025^3, L = 10
    h4 = solve(3, 1025, "h_mg", False)
    d4 = solve(3, 1025, "d_mg", False)
    out["1025_one_gpu"] = {"config": "BASELINE configs[4]'s grid on one B200: 3D 1025^3 (1,070,599,167 unknowns), "
                                     "L=10, V(3,3), FTZ off (L2 irrelevant at this size)",
                           "h_mg": h4, "d_mg": d4, "speedup_vs_fp64": d4["seconds"] / h4["seconds"]}
    return out


def solve_launches(h, iterations, a, variant):
    """Kernels launched by one graph-captured solve (see mpmg_solver.cu):
    init = state reset + r = b (or the FP64 defect) + control; per iteration =
    downcast (not for D_MG, whose scale-1 cast is an alias) + per streaming
    level (pre-smoothing with the first two steps fused, post-smoothing,
    defect, restriction, prolongation) + one coarse kernel + outer update
    (+ the gated fold of parked corrections for binary16/32 finest levels) +
    gated refresh defect + control; final = (fold) + residual-norm defect +
    finalize."""
    big = sum(1 for l in range(h.levels) if (h.level_nodes(l) - 1) >= 64)
    deferred = variant in ("h_mg", "hsd_mg")
    pre = a.pre - 1 if a.pre >= 2 else a.pre
    per_level = pre + a.post + 3
    per_it = (0 if variant == "d_mg" else 1) + big * per_level + 1 + 1 + (1 if deferred else 0) + 1 + 1
    return 3 + iterations * per_it + (1 if deferred else 0) + 2


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return {"hbm_gbs": float(d["hbm_gbs"]), "source": "measured (MEASURED_PEAKS.json hbm_gbs)"}
    except Exception:
        return {"hbm_gbs": 6650.0, "source": "fallback (B200_PROFILING.md)"}


def kernel_roofline(a, dim, n, L, ftz, dev, flush_l2):
    """CUDA-event timing of the finest-level kernels on the stream they are
    launched on: `kernel_reps` back-to-back launches rotating over enough
    independent buffer sets that every launch's operands were evicted from
    L2 (> 126 MB of other traffic in between), averaged. Algorithmic bytes
    per launch (each operand read/written once, N = interior
    unknowns of the finest level):
      jacobi (binary16, 27-pt)      3 * 2 * N   (read u, b; write u')
      update_rc (FP64 r,u; fp16 c)  (32 + 2) N  (read c, r, u; write r, u)
      downcast (FP64 -> binary16)   (8 + 2) N
      defect64 (FP64)               24 N        (read u, b; write r)
    """
    import torch

    import paper_2007_07539_b200 as mg
    lib = mg.lib()
    N = mg.unknowns(dim, n)
    plen = lib.mpmg_padded_len(dim, n)
    prec = {"h_mg": mg.FP16, "hsd_mg": mg.FP16, "dsh_mg": mg.FP64, "d_mg": mg.FP64}[a.variant]
    pol = mg.policy_word(ftz, True, False)
    A = mg.level_stencil(dim, n, prec, ftz)
    A64 = mg.level_stencil(dim, n, mg.FP64, ftz)
    tdt = torch.float16 if prec == mg.FP16 else torch.float64
    g = torch.Generator(device=dev).manual_seed(1)
    scale = 1.0 / (N ** 0.5)

    def padded(dt, p):
        comp = ((torch.rand(N, device=dev, generator=g, dtype=torch.float64) * 2 - 1) * scale).to(dt)
        out = torch.zeros(plen, dtype=dt, device=dev)
        mg._check(lib.mpmg_gpu_pack(dim, n, p, comp.data_ptr(), out.data_ptr(), None), "pack")
        return out

    stream = torch.cuda.current_stream(dev)
    sp = stream.cuda_stream
    bp = 2 if prec == mg.FP16 else 8
    nsets = 3
    sets = []
    for _ in range(nsets):
        sets.append(dict(u=padded(tdt, prec), b=padded(tdt, prec), u2=torch.zeros(plen, dtype=tdt, device=dev),
                         r64=padded(torch.float64, mg.FP64), u64=padded(torch.float64, mg.FP64),
                         b64=padded(torch.float64, mg.FP64)))
    alpha = torch.tensor([1e-3], dtype=torch.float64, device=dev)
    npart = lib.mpmg_gpu_partials_len(dim, n)
    if prec != mg.FP64:
        npart = max(npart, lib.mpmg_gpu_update_r_partials(dim, n, prec))
    part = torch.zeros(npart, dtype=torch.float64, device=dev)
    # deferred-correction ring (the solver's binary16 outer update): one slot
    ring_len = (plen + 63) // 64 * 64
    ring = torch.zeros(ring_len, dtype=tdt, device=dev)
    slot = torch.zeros(1, dtype=torch.int32, device=dev)
    rscale = torch.zeros(1, dtype=torch.float64, device=dev)
    specs = {
        "jacobi_fine": (3 * bp * N, lambda s: lib.mpmg_gpu_jacobi(C.byref(A), s["b"].data_ptr(), s["u"].data_ptr(),
                                                                  s["u2"].data_ptr(), 2.0 / 3.0, pol, sp)),
        "update_rc": ((32 + bp) * N, lambda s: lib.mpmg_gpu_update_rc(C.byref(A64), s["u"].data_ptr(), prec,
                                                                      s["r64"].data_ptr(), s["u64"].data_ptr(),
                                                                      alpha.data_ptr(), part.data_ptr(), pol, sp)),
        "update_r": ((16 + 2 * bp) * N, lambda s: lib.mpmg_gpu_update_r(C.byref(A64), s["u"].data_ptr(), prec,
                                                                        s["r64"].data_ptr(), alpha.data_ptr(),
                                                                        part.data_ptr(), ring.data_ptr(), ring_len,
                                                                        slot.data_ptr(), rscale.data_ptr(), pol, sp)),
        "downcast": ((8 + bp) * N, lambda s: lib.mpmg_gpu_scale_downcast(dim, n, s["r64"].data_ptr(),
                                                                         s["u2"].data_ptr(), prec, alpha.data_ptr(),
                                                                         1, pol, sp)),
        "defect64": (24 * N, lambda s: lib.mpmg_gpu_defect_f64(C.byref(A64), s["b64"].data_ptr(),
                                                                s["u64"].data_ptr(), s["r64"].data_ptr(),
                                                                part.data_ptr(), sp)),
    }
    if prec == mg.FP64 or lib.mpmg_gpu_update_r_partials(dim, n, prec) <= 0:
        specs.pop("update_r")  # FP64 finest levels (and 2D) keep the fused update
    res = {}
    reps = max(a.kernel_reps, nsets)
    for name, (nbytes, fn) in specs.items():
        for k in range(nsets):
            mg._check(fn(sets[k]), name)
        flush_l2()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for k in range(reps):
            fn(sets[k % nsets])
        e1.record(stream)
        e1.synchronize()
        avg = e0.elapsed_time(e1) * 1e-3 / reps
        res[name] = {"bytes": nbytes, "avg_us": avg * 1e6, "achieved_gbs": nbytes / avg / 1e9,
                     "timing": f"{reps} launches rotating over {nsets} buffer sets (operands evicted from L2)"}
    # per iteration: the finest Jacobi kernel runs pre + post - 2 times (the
    # first two pre-smoothing steps are one fused JACOBI_Z pass)
    # the outer update the solve runs: r-only + ring for binary16/32 finest
    # levels (u folded once per refresh), the fused update for FP64
    upd = "update_r" if "update_r" in res else "update_rc"
    share = {"jacobi_fine": res["jacobi_fine"]["avg_us"] * max(1, a.pre + a.post - 2),
             upd: res[upd]["avg_us"], "downcast": res["downcast"]["avg_us"],
             "defect64": res["defect64"]["avg_us"] / 10.0}
    res["dominant"] = max(share, key=share.get)
    for k in share:
        res[k]["us_per_iteration"] = share[k]
    del sets
    torch.cuda.empty_cache()
    return res


# ---------------------------------------------------------------------------
# CPU reference (oracle/_ref: the unmodified reference library)
# ---------------------------------------------------------------------------
CPU_SAMPLE_NODES = 65  # the my-arm cpu_baseline sample: a complete solve at 65^3


def host_info():
    model = ""
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"cpu_model": model, "nproc": os.cpu_count()}


def reference_solve(a, dim, n, L, ftz):
    """One complete reference ir_solve (ir_solver.cpp:51-127) of the variant /
    policy / smoother in `a` on a dim-D n-node grid: the unmodified library
    (oracle/_ref), single-threaded (1 core). The time is the reference's own
    SolveReport.wall_time_s (steady_clock around the solve, ir_solver.cpp:61,
    124-125); the hierarchy build is reported separately."""
    from oracle import Reference
    R = Reference()
    hr = R.hierarchy(dim, n, L, a.variant, pre=a.pre, post=a.post, ftz=ftz)
    res = hr.ir_solve(rel_tol=a.rel_tol, want_u=False)
    return res, hr.build_seconds


def cpu_reference(a, dim, n, L, ftz):
    """cpu_baseline of the B200 arm: a bounded sample -- one COMPLETE reference
    solve of the same variant, policy and smoother on the 65^3 grid (about
    10 s on one core; not scaled to 257^3). The full-size reference solve is
    the --impl reference arm."""
    sn = min(n, CPU_SAMPLE_NODES)
    sL = max_depth(sn)
    t0 = time.perf_counter()
    res, build_s = reference_solve(a, dim, sn, sL, ftz)
    return {"value": res["wall_s"], "unit": UNIT, "cores": 1, "kind": "reference",
            "sample": f"one complete reference ir_solve (oracle/_ref, unmodified library, 1 thread) at {sn}^{dim} "
                      f"L={sL}, {a.variant.upper()}, same policy and smoother: {res['iterations']} outer its; "
                      f"measured, not scaled to {n}^{dim} (the --impl reference arm runs {n}^{dim})",
            "measured_config": f"{sn}^{dim}", "iterations": res["iterations"], "converged": res["converged"],
            "build_s": build_s, "sample_wall_s": time.perf_counter() - t0, **host_info()}


def run_reference(a):
    """--impl reference: the reference's own CPU solver at the SAME workload
    as the B200 arm (3D 257^3, L = 8, V(3,3), the same variant and policy),
    one complete solve. The reference is single-threaded and one solve takes
    ~10 minutes on one core, so exactly one timed solve runs regardless of
    --steps/--warmup (reported as steps = 1, warmup = 0)."""
    ws, rank, _ = dist_info()
    if ws > 1 and rank != 0:
        return  # rank 0 alone runs the CPU reference
    L = a.levels or max_depth(a.nodes)
    ftz = bool(a.ftz)
    try:
        from oracle import Reference
        Reference()
    except Exception as ex:
        print(json.dumps({"impl": "reference", "unavailable": f"oracle/_ref not built: {ex}"[:200]}))
        return
    t0 = time.perf_counter()
    res, build_s = reference_solve(a, a.dim, a.nodes, L, ftz)
    v = res["wall_s"]
    N = (a.nodes - 2) ** a.dim
    cb = {"value": v, "unit": UNIT, "cores": 1, "kind": "reference",
          "sample": f"one complete reference ir_solve at the stated config ({a.nodes}^{a.dim}, L={L}); "
                    f"SolveReport.wall_time_s, hierarchy build excluded", "build_s": build_s, **host_info()}
    out = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": ws, "steps": 1,
           "warmup": 0, "requested": {"steps": a.steps, "warmup": a.warmup}, "ms_per_step": v * 1e3,
           "higher_is_better": False, "scaling": "weak", "vs_baseline": None,
           "dtype": "fp16 (software-emulated)" if a.variant == "h_mg" else ("fp64" if a.variant == "d_mg" else "mixed"),
           "data": "synthetic: the reference's manufactured Poisson problem (assemble_rhs k=1), u0 = 0",
           "config": {"workload": f"{a.dim}D Poisson {a.nodes}^{a.dim} ({N} unknowns), L={L}, V({a.pre},{a.post}),"
                                  f" {a.variant.upper()} IR to {a.rel_tol:g}*||b||", "variant": a.variant,
                      "policy": {"flush_subnormals_to_zero": ftz, "fused_multiply_add": True}},
           "iterations": res["iterations"], "converged": res["converged"], "final_residual": res["final_residual"],
           "cpu_baseline": cb,
           "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
           "wall_s": time.perf_counter() - t0}
    print(json.dumps(out), flush=True)


def run_dist(a):
    """N > 1 (torchrun, one process per GPU): BASELINE configs[4], 3D 1025^3
    (L = 10) -- strong scaling of the C++ z-slab solver (csrc/mpmg_dist.cu:
    peer-memory halos over NVLink through CUDA IPC, replicated agglomerated
    coarse cycle, one CUDA graph per solve). torch.distributed (NCCL) only
    moves the connection blobs and provides the barriers; the time is the max
    over ranks of each rank's CUDA-event time of one solve."""
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2007_07539_b200 as mg
    from paper_2007_07539_b200.dist import DistSolver

    ws, rank, local = dist_info()
    # MPMG_DIST_BACKEND=gloo + fewer GPUs than ranks: the ranks share GPUs
    # (a functional run of the multi-process path on a one-GPU box; NCCL
    # refuses two ranks per GPU -- the data path does not use it anyway)
    backend = os.environ.get("MPMG_DIST_BACKEND", "nccl")
    local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    if backend == "nccl":
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        dist.init_process_group(backend)
    tdev = "cuda" if backend == "nccl" else "cpu"
    dim, n = 3, (a.nodes if a.nodes != 257 else 1025)
    L = a.levels or max_depth(n)
    ftz = bool(a.ftz)
    t0 = time.perf_counter()
    b = mg.problem_rhs(dim, n)
    rhs_s = time.perf_counter() - t0
    tol = a.rel_tol * float(np.sqrt(np.dot(b, b)))
    d = DistSolver(n, L, a.variant, rank, ws, ftz=ftz, pre=a.pre, post=a.post, device=local)
    blobs = [None] * ws
    dist.all_gather_object(blobs, d.blob)
    d.connect(blobs)
    P, m = n - 1, n - 2
    lib = mg.lib()
    lib.mpmg_dev_h2d.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t]
    lib.mpmg_dev_d2h.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t]
    slab = np.zeros((d.nz + 2, P, P))
    slab[1:1 + d.nz, 1:P, 1:P] = b.reshape(m, m, m)[d.z_lo - 1:d.z_lo - 1 + d.nz]
    del b
    bptr, uptr = d.buffers()
    mg._check(lib.mpmg_dev_h2d(bptr, slab.ctypes.data, slab.nbytes), "h2d")
    d.prepare(tol)
    sampler = ClockSampler(local)
    times, rep = [], None
    for k in range(a.warmup + a.steps):
        dist.barrier()
        torch.cuda.synchronize()
        if k == a.warmup:
            sampler.start()
        rep, hist = d.solve(tol)
        if k >= a.warmup:
            times.append(rep.device_seconds)
    clocks = sampler.stop()
    t = torch.tensor([float(np.mean(times))], dtype=torch.float64, device=tdev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    # end to end: this rank's host rhs slab in (pinned), solve, host solution slab out
    bh = torch.from_numpy(slab).pin_memory()
    uh = torch.empty_like(bh).pin_memory()
    dist.barrier()
    t0 = time.perf_counter()
    mg._check(lib.mpmg_dev_h2d(bptr, bh.data_ptr(), bh.numel() * 8), "h2d")
    rep2, _ = d.solve(tol)
    mg._check(lib.mpmg_dev_d2h(uh.data_ptr(), uptr, uh.numel() * 8), "d2h")
    te = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=tdev)
    dist.all_reduce(te, op=dist.ReduceOp.MAX)
    # kernels this rank launched in the timed solves: the captured graph's
    # kernel nodes (init + final, and one IR iteration per WHILE pass)
    gk = d.graph_kernels()
    per_solve = gk[0] + rep.iterations * gk[1] if gk else None
    launches = per_solve * a.steps if per_solve is not None else None
    if rank == 0:
        N = mg.unknowns(dim, n)
        out = {"metric": METRIC, "value": float(t.item()), "unit": UNIT, "n_gpus": ws, "steps": a.steps,
               "warmup": a.warmup, "ms_per_step": float(t.item()) * 1e3, "higher_is_better": False,
               "scaling": "strong", "vs_baseline": None,
               "dtype": "fp16" if a.variant == "h_mg" else ("fp64" if a.variant == "d_mg" else "mixed"),
               "data": "synthetic: the reference's manufactured Poisson problem (assemble_rhs k=1), u0 = 0",
               "config": {"workload": f"BASELINE configs[4]: {dim}D Poisson {n}^{dim} ({N} unknowns), L={L}, "
                                      f"V({a.pre},{a.post}), {a.variant.upper()} IR to {a.rel_tol:g}*||b||, "
                                      f"z-slabs over {ws} GPUs",
                          "variant": a.variant, "policy": {"flush_subnormals_to_zero": ftz, "fused_multiply_add": True},
                          "parallelism": f"z-slab decomposition x{ws}: peer-memory halos (CUDA IPC over NVLink), "
                                         f"levels <= level {d.agg} agglomerated (replicated coarse cycle)",
                          "l2": "not flushed (the finest FP64 slabs exceed L2 at every N <= 8)"},
               "iterations": rep.iterations, "converged": bool(rep.converged), "final_residual": rep.final_residual,
               "tolerance": tol, "rhs_assembly_s": rhs_s, "clocks": clocks,
               "e2e": {"value": float(te.item()), "unit": UNIT, "h2d_bytes_per_step": int(slab.nbytes * ws),
                       "d2h_bytes_per_step": int(slab.nbytes * ws), "path": "mpmg_dist_solve_device (C ABI), slabs"},
               "gpu_launches": launches,
               "gpu_launches_per_solve": {"rank0": per_solve, "graph_kernels_outer_per_iteration": gk}}
        print(json.dumps(out), flush=True)
    dist.barrier()
    d.close()
    dist.destroy_process_group()


def main():
    a = parse()
    ws = dist_info()[0]
    if a.impl == "reference":
        run_reference(a)
    elif ws > 1:
        run_dist(a)
    else:
        run_b200(a)


if __name__ == "__main__":
    main()
