"""Direct C-ABI kernel checks on device pointers (torch only allocates):
the scaled downcast (cast_vector, kernels.cpp:343-360) and the generic
ELLPACK kernels (spmv / transfer / update, kernels.cpp:137-341,
multigrid.cpp:155-232) against the oracle, bitwise."""
import ctypes as C

import numpy as np
import pytest

import paper_2007_07539_b200 as mg
from oracle import FP16, FP32, FP64, Oracle

pytestmark = pytest.mark.gpu
O = Oracle()


def same(a, b):
    return np.array_equal(np.asarray(a), np.asarray(b), equal_nan=True)


def dev(arr):
    import torch
    return torch.from_numpy(np.ascontiguousarray(arr)).cuda()


@pytest.mark.parametrize("prec", [FP16, FP32])
@pytest.mark.parametrize("ftz", [True, False])
def test_scaled_downcast_bitwise(prec, ftz):
    import torch
    L = mg.lib()
    dim, n = 3, 65
    plen = L.mpmg_padded_len(dim, n)
    rng = np.random.default_rng(11)
    for trial in range(4):
        x = rng.standard_normal(plen) * 10.0 ** rng.integers(-12, 3, plen)
        x[rng.random(plen) < 0.01] = 0.0
        alpha = float(np.sqrt(np.dot(x, x))) * (1.0 + trial * 0.37)
        xd = dev(x)
        out = torch.zeros(plen, dtype=torch.float16 if prec == FP16 else torch.float32, device="cuda")
        ad = dev(np.array([alpha]))
        rc = L.mpmg_gpu_scale_downcast(dim, n, xd.data_ptr(), out.data_ptr(), prec, ad.data_ptr(), 1,
                                       mg.policy_word(ftz), None)
        assert rc == 0
        torch.cuda.synchronize()
        got = out.double().cpu().numpy()
        ref = O.cast(x, prec, alpha, O.ctx(ftz))
        assert same(got, ref), np.count_nonzero(got != ref)


def random_ell(rng, rows, cols, rw):
    c = np.zeros((rows, rw), dtype=np.int32)
    v = np.zeros((rows, rw))
    for i in range(rows):
        k = rng.integers(1, rw + 1)
        cs = np.sort(rng.choice(cols, size=k, replace=False))
        c[i, :k] = cs
        v[i, :k] = rng.uniform(-1, 1, k)
        c[i, k:] = min(i, cols - 1)
    return c, v


@pytest.mark.parametrize("prec", [FP16, FP32, FP64])
@pytest.mark.parametrize("ftz,fma,acc32", [(True, True, False), (False, True, False), (True, False, False),
                                           (False, True, True)])
def test_generic_ell_spmv(prec, ftz, fma, acc32):
    import torch
    if acc32 and prec != FP16:
        pytest.skip("acc32 only changes binary16")
    L = mg.lib()
    rng = np.random.default_rng(5)
    rows, rw = 3000, 7
    cols, vals = random_ell(rng, rows, rows, rw)
    vals = np.array([O.round_vec(r, prec, ftz) for r in vals])
    x = O.round_vec(rng.uniform(-1, 1, rows) * 1e-3, prec, ftz)
    tdt = {FP16: torch.float16, FP32: torch.float32, FP64: torch.float64}[prec]
    cd = dev(cols.T.copy())  # slot-major
    vd = torch.from_numpy(vals.T.copy()).to(tdt).cuda()
    xd = torch.from_numpy(x).to(tdt).cuda()
    yd = torch.zeros(rows, dtype=tdt, device="cuda")
    pol = mg.policy_word(ftz, fma, acc32)
    assert L.mpmg_gpu_ell_spmv(rows, rw, cd.data_ptr(), vd.data_ptr(), prec, xd.data_ptr(), yd.data_ptr(), pol,
                               None) == 0
    torch.cuda.synchronize()
    ref = O.spmv(cols, vals, prec, x, O.ctx(ftz, fma, acc32))
    assert same(yd.double().cpu().numpy(), ref)


@pytest.mark.parametrize("fma", [True, False])
def test_update_r_and_fold_equal_fused_update(fma):
    """mpmg_gpu_update_r (r half + ring slot) followed by mpmg_gpu_fold (u half)
    equals the fused mpmg_gpu_update_rc (kernels.cpp:300-341) bitwise, over two
    iterations with different scales."""
    import torch
    L = mg.lib()
    dim, n = 3, 65
    plen = L.mpmg_padded_len(dim, n)
    pol = mg.policy_word(False, fma, False)
    A64 = mg.level_stencil(dim, n, mg.FP64, False)
    rng = np.random.default_rng(5)

    def padded(prec, scale):
        comp = (rng.random(mg.unknowns(dim, n)) * 2 - 1) * scale
        comp = O.round_vec(comp, prec, False)
        out = torch.zeros(plen, dtype=torch.float16 if prec == FP16 else torch.float64, device="cuda")
        src = torch.from_numpy(comp.astype(np.float16 if prec == FP16 else np.float64)).cuda()
        mg._check(L.mpmg_gpu_pack(dim, n, prec, src.data_ptr(), out.data_ptr(), None), "pack")
        return out

    r0, u0 = padded(FP64, 1.0), padded(FP64, 1.0)
    cs = [padded(FP16, 1.0), padded(FP16, 1e-3)]
    alphas = [dev(np.array([0.37])), dev(np.array([2.5e-4]))]
    npart = L.mpmg_gpu_partials_len(dim, n)
    p1 = torch.zeros(npart, dtype=torch.float64, device="cuda")
    r1, u1 = r0.clone(), u0.clone()
    for c, a in zip(cs, alphas):
        assert L.mpmg_gpu_update_rc(C.byref(A64), c.data_ptr(), FP16, r1.data_ptr(), u1.data_ptr(), a.data_ptr(),
                                    p1.data_ptr(), pol, None) == 0
    ring_len = (plen + 63) // 64 * 64
    ring = torch.zeros(2 * ring_len, dtype=torch.float16, device="cuda")
    scales = torch.zeros(2, dtype=torch.float64, device="cuda")
    assert L.mpmg_gpu_update_r_partials(dim, n, FP16) > 0
    p2 = torch.zeros(max(npart, L.mpmg_gpu_update_r_partials(dim, n, FP16)), dtype=torch.float64, device="cuda")
    r2, u2 = r0.clone(), u0.clone()
    for k, (c, a) in enumerate(zip(cs, alphas)):
        slot = torch.tensor([k], dtype=torch.int32, device="cuda")
        assert L.mpmg_gpu_update_r(C.byref(A64), c.data_ptr(), FP16, r2.data_ptr(), a.data_ptr(), p2.data_ptr(),
                                   ring.data_ptr(), ring_len, slot.data_ptr(), scales.data_ptr(), pol, None) == 0
    cnt = torch.tensor([2], dtype=torch.int32, device="cuda")
    assert L.mpmg_gpu_fold(plen, u2.data_ptr(), ring.data_ptr(), ring_len, FP16, scales.data_ptr(), cnt.data_ptr(),
                           pol, None) == 0
    torch.cuda.synchronize()
    assert same(r1.cpu().numpy().view(np.uint64), r2.cpu().numpy().view(np.uint64))
    assert same(u1.cpu().numpy().view(np.uint64), u2.cpu().numpy().view(np.uint64))
    assert same(scales.cpu().numpy(), np.array([0.37, 2.5e-4]))
