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
