"""The C++ multi-GPU z-slab solver (csrc/mpmg_dist.cu) on ONE GPU: world = 2
and 4 ranks in one process (one thread and one stream per rank; raw peer
pointers instead of IPC handles, the same copies, flags and graphs), against
the single-GPU solver: the same outer iteration count and the same solution
(per-point arithmetic is rank-count independent; only the norm's summation
grouping differs, ~1e-16 in alpha)."""
import ctypes as C
import threading

import numpy as np
import pytest

import paper_2007_07539_b200 as mg
from paper_2007_07539_b200.dist import DistSolver

pytestmark = pytest.mark.gpu


def run_ranks(nodes, levels, variant, world, ftz=False, pre=3, post=3):
    ranks = [DistSolver(nodes, levels, variant, r, world, ftz=ftz, pre=pre, post=post) for r in range(world)]
    blobs = [r.blob for r in ranks]
    for r in ranks:
        r.connect(blobs)
    b = mg.problem_rhs(3, nodes)
    tol = 1e-10 * float(np.sqrt(np.dot(b, b)))
    P = nodes - 1
    m = P - 1
    bc = b.reshape(m, m, m)
    L = mg.lib()
    L.mpmg_dev_h2d.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t]
    L.mpmg_dev_d2h.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t]
    for r in ranks:  # this rank's owned planes of b into its FP64 slab (local planes 1..nz)
        bptr, _ = r.buffers()
        slab = np.zeros((r.nz + 2, P, P))
        slab[1:1 + r.nz, 1:P, 1:P] = bc[r.z_lo - 1:r.z_lo - 1 + r.nz]
        assert L.mpmg_dev_h2d(bptr, slab.ctypes.data, slab.nbytes) == 0
    for r in ranks:  # graphs captured up front: capture may synchronize the (shared) device
        r.prepare(tol)
    out = [None] * world
    stats = [r.exchange_stats() for r in ranks]

    def go(i):
        out[i] = ranks[i].solve(tol)

    th = [threading.Thread(target=go, args=(i,)) for i in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    # gather u (owned planes) in compact order
    u = np.zeros((m, m, m))
    for r in ranks:
        _, uptr = r.buffers()
        v = np.zeros((r.nz + 2, P, P))
        assert L.mpmg_dev_d2h(v.ctypes.data, uptr, v.nbytes) == 0
        u[r.z_lo - 1:r.z_lo - 1 + r.nz] = v[1:1 + r.nz, 1:P, 1:P]
    for r in ranks:
        r.close()
    run_ranks.stats = stats
    return out, u.reshape(-1), b, tol


@pytest.mark.parametrize("variant", ["h_mg", "d_mg", "hsd_mg"])
@pytest.mark.parametrize("world", [2, 4])
def test_dist_matches_single_gpu(variant, world):
    nodes, levels = 257, 8
    out, u, b, tol = run_ranks(nodes, levels, variant, world)
    reps = [o[0] for o in out]
    hists = [o[1] for o in out]
    # identical control flow on every rank
    assert len({r.iterations for r in reps}) == 1 and all(np.array_equal(hists[0], h) for h in hists)
    h = mg.Hierarchy(3, nodes, levels, variant, ftz=False)
    u1, rep1 = h.ir_solve(b, mg.IrConfig(outer_tolerance=tol))
    h.close()
    assert reps[0].converged and rep1.converged
    assert reps[0].iterations == rep1.iterations, (reps[0].iterations, rep1.iterations)
    # the trajectory agrees to the rounding level of each entry (the norm's
    # summation grouping differs; FP16 scaled casts may round 1 ulp apart)
    np.testing.assert_allclose(hists[0], rep1.residual_history, rtol=1e-3)
    assert np.linalg.norm(u - u1) / np.linalg.norm(u1) <= 1e-9
    assert reps[0].final_residual < tol


@pytest.mark.parametrize("variant", ["h_mg", "d_mg"])
def test_dist_fused_halos_match_copy_exchange(variant, monkeypatch):
    """the halo planes stored into the neighbours' memory by the producing
    Jacobi / defect kernel and the fused JACOBI_Z pre-smoothing sweep (both
    default) against the kernel + peer-copy exchange and pointwise step 1 +
    stencil step 2 (MPMG_DIST_FUSE_HALOS=0, MPMG_DIST_JZ=0): the identical
    solve, bit for bit"""
    nodes, levels, world = 257, 8, 4
    monkeypatch.setenv("MPMG_DIST_FUSE_HALOS", "0")
    monkeypatch.setenv("MPMG_DIST_JZ", "0")
    out0, u0, _, _ = run_ranks(nodes, levels, variant, world)
    assert all(f == 0 and c > 0 for f, c in run_ranks.stats)
    monkeypatch.setenv("MPMG_DIST_FUSE_HALOS", "1")
    monkeypatch.setenv("MPMG_DIST_JZ", "1")
    out1, u1, _, _ = run_ranks(nodes, levels, variant, world)
    # the slab Jacobi sweeps and defects of pitch 256 and 128 fused
    assert all(f > 0 for f, _ in run_ranks.stats), run_ranks.stats
    assert out0[0][0].iterations == out1[0][0].iterations
    assert np.array_equal(out0[0][1], out1[0][1])
    assert np.array_equal(u0, u1)


def _proc(rank, world, port, nodes, levels, variant, q):
    """one rank per PROCESS (the deployment shape): CUDA IPC handles for the
    peer arenas, gloo (torch.distributed) only to move the connection blobs"""
    import os
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    import torch.distributed as dist
    try:
        dist.init_process_group("gloo", rank=rank, world_size=world)
        d = DistSolver(nodes, levels, variant, rank, world)
        blobs = [None] * world
        dist.all_gather_object(blobs, d.blob)
        d.connect(blobs)
        b = mg.problem_rhs(3, nodes)
        tol = 1e-10 * float(np.sqrt(np.dot(b, b)))
        P, m = nodes - 1, nodes - 2
        slab = np.zeros((d.nz + 2, P, P))
        slab[1:1 + d.nz, 1:P, 1:P] = b.reshape(m, m, m)[d.z_lo - 1:d.z_lo - 1 + d.nz]
        L = mg.lib()
        L.mpmg_dev_h2d.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t]
        L.mpmg_dev_d2h.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t]
        bptr, uptr = d.buffers()
        assert L.mpmg_dev_h2d(bptr, slab.ctypes.data, slab.nbytes) == 0
        d.prepare(tol)
        dist.barrier()
        rep, hist = d.solve(tol)
        v = np.zeros((d.nz + 2, P, P))
        assert L.mpmg_dev_d2h(v.ctypes.data, uptr, v.nbytes) == 0
        q.put((rank, rep.iterations, bool(rep.converged), hist.tolist(), d.z_lo, d.nz, v[1:1 + d.nz, 1:P, 1:P].copy()))
        dist.barrier()
        d.close()
        dist.destroy_process_group()
    except Exception as ex:  # reported to the parent
        q.put((rank, "ERROR " + repr(ex)))


def test_dist_two_processes_ipc():
    import multiprocessing as mp
    import socket
    nodes, levels, world = 65, 6, 2
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_proc, args=(r, world, port, nodes, levels, "h_mg", q)) for r in range(world)]
    for p in ps:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in ps:
        p.join(timeout=60)
    errs = [r for r in res if isinstance(r[1], str)]
    assert not errs, errs
    res.sort(key=lambda r: r[0])
    m = nodes - 2
    u = np.zeros((m, m, m))
    for _, its, conv, hist, z_lo, nz, own in res:
        u[z_lo - 1:z_lo - 1 + nz] = own
    assert res[0][1] == res[1][1] and res[0][3] == res[1][3]  # identical control flow
    b = mg.problem_rhs(3, nodes)
    tol = 1e-10 * float(np.sqrt(np.dot(b, b)))
    h = mg.Hierarchy(3, nodes, levels, "h_mg", ftz=False)
    u1, rep1 = h.ir_solve(b, mg.IrConfig(outer_tolerance=tol))
    h.close()
    assert res[0][2] and res[0][1] == rep1.iterations
    assert np.linalg.norm(u.reshape(-1) - u1) / np.linalg.norm(u1) <= 1e-9
