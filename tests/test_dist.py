"""Multi-GPU z-slab decomposition (paper_2007_07539_b200.dist).

CPU (gloo, world_size 2): the partition invariants, the halo exchange, the
agglomeration gather/scatter and the whole distributed IR solve driven by a
NumPy model of the slab kernels (tests/dist_numpy_ops.py) -- a V-cycle on two
ranks must equal the one-rank V-cycle bitwise, the solve must converge in
the same number of iterations.

GPU (one B200): the same driver over the sm_100a slab kernels, one rank
against the monolithic single-GPU solver, and two ranks sharing the GPU
(gloo, device tensors staged through the host) against one rank.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2007_07539_b200.dist import Comm, SlabPlan, SlabSolver, compact_of_slabs, slab_of_compact


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("nodes,levels,world", [(65, 6, 2), (257, 8, 8), (1025, 10, 8), (129, 7, 4), (33, 5, 1)])
def test_plan_invariants(nodes, levels, world):
    plan = SlabPlan(nodes, levels, world)
    assert plan.check()
    assert plan.dist[-1] and plan.agg >= 0
    for l in range(plan.agg + 1, levels):
        assert plan.P[l] // world >= 4


def test_plan_rejects_unsplittable():
    with pytest.raises(ValueError):
        SlabPlan(65, 6, 3)  # 64 planes do not split over 3 ranks


def _worker(rank, world, port, nodes, levels, q, mode):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from dist_numpy_ops import NumpyOps

        from oracle import Oracle
        plan = SlabPlan(nodes, levels, world, min_planes=2, min_pitch=4)
        ops = NumpyOps(plan)
        comm = Comm(dist, rank, world, device_tensors=False)
        S = SlabSolver(plan, ops, comm)
        b = Oracle().rhs(3, nodes)
        bs = slab_of_compact(b, plan, rank, torch, "cpu")
        F = levels - 1
        s = plan.slab(F, rank)
        if mode == "exchange":
            # owned planes carry the global plane index; halos must receive the neighbours'
            P = plan.P[F]
            t = torch.zeros(plan.slab_len(F, rank), dtype=torch.float64)
            for k in range(1, s.nz + 1):
                t[k * P * P:(k + 1) * P * P] = s.z_lo + k - 1
            comm.exchange(t, P * P, s.nz)
            q.put((rank, float(t[0]), float(t[(s.nz + 1) * P * P])))
            return
        if mode == "cycle":
            S.lv[F]["b"].copy_(bs / float(np.linalg.norm(b)))
            c = S.cycle(F)
            q.put((rank, c.numpy().copy()))
            return
        tol = 1e-10 * float(np.linalg.norm(b))
        u, its, hist, conv, final = S.solve(bs, tol, max_it=60)
        q.put((rank, u.numpy().copy(), its, hist, conv, final))
    except Exception:  # surface worker failures in the parent
        import traceback
        q.put((rank, "ERROR " + traceback.format_exc()))
    finally:
        dist.destroy_process_group()


def _run(world, nodes, levels, mode):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, nodes, levels, q, mode)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=300) for _ in range(world)]
    for o in out:
        assert not (isinstance(o[1], str) and o[1].startswith("ERROR")), o[1]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    return sorted(out, key=lambda t: t[0])


def test_halo_exchange_gloo():
    nodes, levels = 33, 5
    out = _run(2, nodes, levels, "exchange")
    plan = SlabPlan(nodes, levels, 2, min_planes=2, min_pitch=4)
    s0, s1 = plan.slab(levels - 1, 0), plan.slab(levels - 1, 1)
    # rank 0: lower halo is the boundary (untouched 0), upper halo = rank 1's first plane
    assert out[0][1] == 0.0 and out[0][2] == s1.z_lo
    # rank 1: lower halo = rank 0's last owned plane
    assert out[1][1] == s0.z_lo + s0.nz - 1


def test_vcycle_two_ranks_equals_one_rank():
    nodes, levels = 33, 5
    one = _run(1, nodes, levels, "cycle")
    two = _run(2, nodes, levels, "cycle")
    p1 = SlabPlan(nodes, levels, 1, min_planes=2, min_pitch=4)
    p2 = SlabPlan(nodes, levels, 2, min_planes=2, min_pitch=4)
    assert p1.agg == p2.agg
    c1 = compact_of_slabs([t[1] for t in one], p1, torch)
    c2 = compact_of_slabs([t[1] for t in two], p2, torch)
    assert np.array_equal(c1.view(np.uint64), c2.view(np.uint64))
    assert np.abs(c1).max() > 0


def test_ir_solve_two_ranks():
    nodes, levels = 33, 5
    one = _run(1, nodes, levels, "solve")
    two = _run(2, nodes, levels, "solve")
    assert one[0][4] and two[0][4]  # converged
    assert one[0][2] == two[0][2] == two[1][2]  # iterations
    p1 = SlabPlan(nodes, levels, 1, min_planes=2, min_pitch=4)
    p2 = SlabPlan(nodes, levels, 2, min_planes=2, min_pitch=4)
    u1 = compact_of_slabs([t[1] for t in one], p1, torch)
    u2 = compact_of_slabs([t[1] for t in two], p2, torch)
    assert np.linalg.norm(u1 - u2) <= 1e-12 * np.linalg.norm(u1)
    assert np.allclose(one[0][3], two[0][3], rtol=1e-12)


# ---------------------------------------------------------------------------
# GPU: the sm_100a slab kernels
# ---------------------------------------------------------------------------
def _gpu_worker(rank, world, port, nodes, levels, variant, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2007_07539_b200 as mg
        from paper_2007_07539_b200.dist import CudaOps
        plan = SlabPlan(nodes, levels, world)
        ops = CudaOps(plan, variant, ftz=False)
        comm = Comm(dist, rank, world, device_tensors=True)
        S = SlabSolver(plan, ops, comm)
        b = mg.problem_rhs(3, nodes)
        bs = slab_of_compact(b, plan, rank, torch, "cuda")
        F = levels - 1
        S.lv[F]["b"].copy_((bs / float(np.linalg.norm(b))).to(S.lv[F]["b"].dtype))
        c = S.cycle(F).clone()
        tol = 1e-10 * float(np.linalg.norm(b))
        u, its, hist, conv, final = S.solve(bs, tol)
        torch.cuda.synchronize()
        q.put((rank, c.double().cpu().numpy(), u.cpu().numpy(), its, hist, conv, final))
    finally:
        dist.destroy_process_group()


def _run_gpu(world, nodes, levels, variant):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_gpu_worker, args=(r, world, port, nodes, levels, variant, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=900) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    return sorted(out, key=lambda t: t[0])


@pytest.mark.gpu
@pytest.mark.parametrize("variant", ["h_mg", "d_mg", "hsd_mg"])
def test_gpu_slabs_match_single_gpu(variant):
    import paper_2007_07539_b200 as mg
    nodes, levels = 129, 7
    b = mg.problem_rhs(3, nodes)
    tol = 1e-10 * float(np.linalg.norm(b))
    h = mg.Hierarchy(3, nodes, levels, variant, ftz=False)
    u_ref, rep = h.ir_solve(b, mg.IrConfig(outer_tolerance=tol))
    one = _run_gpu(1, nodes, levels, variant)
    two = _run_gpu(2, nodes, levels, variant)
    p1, p2 = SlabPlan(nodes, levels, 1), SlabPlan(nodes, levels, 2)
    # a V-cycle is bitwise independent of the rank count
    c1 = compact_of_slabs([t[1] for t in one], p1, torch)
    c2 = compact_of_slabs([t[1] for t in two], p2, torch)
    assert np.array_equal(c1, c2)
    for res, plan in ((one, p1), (two, p2)):
        u = compact_of_slabs([t[2] for t in res], plan, torch)
        assert res[0][5], f"not converged: its {res[0][3]} hist {res[0][4][:6]} ... {res[0][4][-3:]} ref {rep.residual_history[:4]}"
        assert abs(res[0][3] - rep.iterations) <= 1
        assert np.linalg.norm(u - u_ref) <= 1e-9 * np.linalg.norm(u_ref)
        assert res[0][6] < tol


@pytest.mark.gpu
@pytest.mark.parametrize("variant", ["h_mg", "d_mg"])
def test_gpu_slab_ops_match_whole_level(variant):
    """Each sm_100a slab kernel on two slabs (halos copied by hand, one
    process) equals the same kernel on the whole level, value for value."""
    import paper_2007_07539_b200 as mg
    from paper_2007_07539_b200.dist import CudaOps
    nodes, levels = 129, 7
    p1, p2 = SlabPlan(nodes, levels, 1), SlabPlan(nodes, levels, 2)
    o1, o2 = CudaOps(p1, variant, ftz=False), CudaOps(p2, variant, ftz=False)
    F = levels - 1
    P = p1.P[F]
    pl = P * P
    rng = np.random.default_rng(3)
    dt = o1.dt[o1.prec[F]]

    def whole(vals):
        t = torch.zeros(p1.slab_len(F, 0), dtype=torch.float64)
        v = t[: P * pl].view(P, P, P)
        v[1:P, 1:P, 1:P] = torch.from_numpy(vals.reshape(P - 1, P - 1, P - 1))
        return t

    def split(t_whole, plan, l):
        Pl = plan.P[l]
        out = []
        for r in range(2):
            s = plan.slab(l, r)
            loc = torch.zeros(plan.slab_len(l, r), dtype=t_whole.dtype, device=t_whole.device)
            loc[: (s.nz + 2) * Pl * Pl] = t_whole[(s.z_lo - 1) * Pl * Pl:(s.z_lo + s.nz + 1) * Pl * Pl]
            out.append(loc)
        return out

    def owned(parts, plan, l):
        Pl = plan.P[l]
        res = []
        for r, t in enumerate(parts):
            s = plan.slab(l, r)
            res.append(t[Pl * Pl:(1 + s.nz) * Pl * Pl].double().cpu())
        return torch.cat(res)

    vals = rng.uniform(-1, 1, (P - 1) ** 3) * 1e-2
    u = whole(vals).to(dt).cuda()
    b = whole(rng.uniform(-1, 1, (P - 1) ** 3)).to(dt).cuda()
    s1 = p1.slab(F, 0)
    out1 = torch.zeros_like(u)
    o1.jacobi(F, s1, b, u, out1)
    us, bs = split(u, p2, F), split(b, p2, F)
    outs = [torch.zeros_like(x) for x in us]
    for r in range(2):
        o2.jacobi(F, p2.slab(F, r), bs[r], us[r], outs[r])
    torch.cuda.synchronize()
    ref = out1[pl:P * pl].double().cpu()
    assert torch.equal(owned(outs, p2, F), ref), "slab jacobi"
    # defect + restriction (the fine lower halo comes from the whole array)
    r1 = torch.zeros_like(u)
    o1.defect(F, s1, b, u, r1)
    rs = [torch.zeros_like(x) for x in us]
    for r in range(2):
        o2.defect(F, p2.slab(F, r), bs[r], us[r], rs[r])
    assert torch.equal(owned(rs, p2, F), r1[pl:P * pl].double().cpu()), "slab defect"
    rsplit = split(r1, p2, F)
    Pc = p1.P[F - 1]
    c1 = torch.zeros(p1.slab_len(F - 1, 0), dtype=o1.dt[o1.prec[F - 1]], device="cuda")
    o1.restrict(F, s1, p1.slab(F - 1, 0), r1, c1)
    cs = [torch.zeros(p2.slab_len(F - 1, r), dtype=c1.dtype, device="cuda") for r in range(2)]
    for r in range(2):
        o2.restrict(F, p2.slab(F, r), p2.slab(F - 1, r), rsplit[r], cs[r])
    assert torch.equal(owned(cs, p2, F - 1), c1[Pc * Pc:Pc * Pc * Pc].double().cpu()), "slab restrict"
    # prolongation (coarse upper halo from the whole array)
    csplit = split(c1, p2, F - 1)
    u1 = u.clone()
    o1.prolong(F, s1, p1.slab(F - 1, 0), c1, u1)
    u2 = [x.clone() for x in us]
    for r in range(2):
        o2.prolong(F, p2.slab(F, r), p2.slab(F - 1, r), csplit[r], u2[r])
    assert torch.equal(owned(u2, p2, F), u1[pl:P * pl].double().cpu()), "slab prolong"
