"""TEST INFRASTRUCTURE: a NumPy model of the z-slab kernel interface of
paper_2007_07539_b200.dist (CudaOps), binary64 only (the D_MG arithmetic,
products and sums rounded separately). It lets the CPU tests run the
distributed solver's decomposition, halo-exchange and agglomeration logic
with world_size 2 on gloo and compare it with world_size 1 -- the per-point
arithmetic is identical whatever the slab boundaries, so V-cycles must agree
bitwise. It checks orchestration, not the sm_100a kernels (those are pinned
by the GPU parity tests)."""
import numpy as np
import torch

from oracle import Oracle

_O = Oracle()


class NumpyOps:
    def __init__(self, plan, pre=3, post=3, omega=2.0 / 3.0, coarse_sweeps=30):
        self.plan, self.pre, self.post, self.omega = plan, pre, post, omega
        self.variant = "d_mg"
        self.prec = [2] * plan.levels
        self.taps = [_O.stencil(3, plan.nodes_at(l)) for l in range(plan.levels)]
        self.invd = [1.0 / t[13] for t in self.taps]
        self.coarse_sweeps = coarse_sweeps

    def zeros(self, n, prec):
        return torch.zeros(n, dtype=torch.float64)

    # views -------------------------------------------------------------
    @staticmethod
    def _grid(t, P, nz):
        """(nz+2, P+1, P+1) copy with the aliased y = P / x = P ghosts as zeros"""
        v = np.zeros((nz + 2, P + 1, P + 1))
        v[:, :P, :P] = t.numpy()[: (nz + 2) * P * P].reshape(nz + 2, P, P)
        return v

    @staticmethod
    def _put(t, P, nz, vals, planes):
        """write owned interior values of `planes` (local indices) back"""
        a = t.numpy()[: (nz + 2) * P * P].reshape(nz + 2, P, P)
        for j, q in enumerate(planes):
            a[q, 1:P, 1:P] = vals[j]

    def _apply(self, taps, v, P, nz):
        acc = np.zeros((nz, P - 1, P - 1))
        t = 0
        for dz in (-1, 0, 1):
            for dy in (-1, 0, 1):
                for dx in (-1, 0, 1):
                    acc = acc + taps[t] * v[1 + dz:1 + nz + dz, 1 + dy:P + dy, 1 + dx:P + dx]
                    t += 1
        return acc

    # slab ops ----------------------------------------------------------
    def jacobi(self, l, s, b, u_in, u_out):
        P = self.plan.P[l]
        if u_in is None:
            u_out.copy_(b * self.invd[l] * self.omega)
            return
        vu = self._grid(u_in, P, s.nz)
        vb = self._grid(b, P, s.nz)
        t = self._apply(self.taps[l], vu, P, s.nz)
        r = vb[1:1 + s.nz, 1:P, 1:P] - t
        un = vu[1:1 + s.nz, 1:P, 1:P] + self.omega * (self.invd[l] * r)
        self._put(u_out, P, s.nz, un, range(1, 1 + s.nz))

    def defect(self, l, s, b, u, r):
        P = self.plan.P[l]
        vu, vb = self._grid(u, P, s.nz), self._grid(b, P, s.nz)
        self._put(r, P, s.nz, vb[1:1 + s.nz, 1:P, 1:P] - self._apply(self.taps[l], vu, P, s.nz), range(1, 1 + s.nz))

    def restrict(self, l, sf, sc, r_f, b_c):
        Pf, Pc = self.plan.P[l], self.plan.P[l - 1]
        vf = self._grid(r_f, Pf, sf.nz)
        zoff = 2 * sc.z_lo - sf.z_lo - 1
        out = []
        for k in range(1, sc.nz + 1):
            cz = 2 * k + zoff
            acc = np.zeros((Pc - 1, Pc - 1))
            for dz in (-1, 0, 1):
                for dy in (-1, 0, 1):
                    for dx in (-1, 0, 1):
                        w = (1.0 if dx == 0 else 0.5) * (1.0 if dy == 0 else 0.5) * (1.0 if dz == 0 else 0.5)
                        acc = acc + w * vf[cz + dz, 2 + dy:2 * Pc - 1 + dy:2, 2 + dx:2 * Pc - 1 + dx:2]
            out.append(acc)
        self._put(b_c, Pc, sc.nz, out, range(1, 1 + sc.nz))

    def prolong(self, l, sf, sc, c_c, u_f):
        Pf, Pc = self.plan.P[l], self.plan.P[l - 1]
        vc = self._grid(c_c, Pc, sc.nz)
        vf = self._grid(u_f, Pf, sf.nz)
        out = []
        for f in range(1, sf.nz + 1):
            gz = f + sf.z_lo - 1
            pz = [gz // 2] if gz % 2 == 0 else [(gz - 1) // 2, (gz + 1) // 2]
            wz = 1.0 if gz % 2 == 0 else 0.5
            acc = np.zeros((Pf - 1, Pf - 1))
            fy = np.arange(1, Pf)
            for zc in pz:
                q = zc - sc.z_lo + 1
                for yp in (0, 1):
                    for xp in (0, 1):
                        py = np.where(fy % 2 == 0, fy // 2, (fy - 1) // 2 + yp)
                        wy = np.where(fy % 2 == 0, 1.0 if yp == 0 else 0.0, 0.5)
                        px, wx = py, wy
                        acc = acc + wz * np.outer(wy, wx) * vc[q][np.ix_(py, px)]
            out.append(vf[f, 1:Pf, 1:Pf] + acc)
        self._put(u_f, Pf, sf.nz, out, range(1, 1 + sf.nz))

    def partials(self, s, update):
        return torch.zeros(s.nz, dtype=torch.float64), s.nz

    def local_sumsq(self, part, n):
        return float(part[:n].sum().item())

    def defect64(self, s, b, u, r, part, resnorm=False):
        l = self.plan.levels - 1
        P = self.plan.P[l]
        vu, vb = self._grid(u, P, s.nz), self._grid(b, P, s.nz)
        res = vb[1:1 + s.nz, 1:P, 1:P] - self._apply(self.taps[l], vu, P, s.nz)
        if r is not None:
            self._put(r, P, s.nz, res, range(1, 1 + s.nz))
        part[: s.nz] = torch.from_numpy((res * res).sum(axis=(1, 2)))

    def update(self, s, c, r, u, alpha_dev, part):
        l = self.plan.levels - 1
        P = self.plan.P[l]
        al = float(alpha_dev[0])
        vc, vr, vu = self._grid(c, P, s.nz), self._grid(r, P, s.nz), self._grid(u, P, s.nz)
        un = vu[1:1 + s.nz, 1:P, 1:P] + al * vc[1:1 + s.nz, 1:P, 1:P]
        rn = vr[1:1 + s.nz, 1:P, 1:P] - al * self._apply(self.taps[l], vc, P, s.nz)
        self._put(u, P, s.nz, un, range(1, 1 + s.nz))
        self._put(r, P, s.nz, rn, range(1, 1 + s.nz))
        part[: s.nz] = torch.from_numpy((rn * rn).sum(axis=(1, 2)))

    def downcast(self, s, r, out, alpha_dev, scale_enabled):
        out.copy_(r / float(alpha_dev[0]) if scale_enabled else r)

    def coarse_solver(self):
        return None

    def coarse_cycle(self, b_full, c_full):
        """a fixed number of Jacobi sweeps on the whole agglomerated level"""
        a = self.plan.agg
        P = self.plan.P[a]
        s = type("S", (), {"nz": P - 1})()
        u = torch.zeros_like(b_full)
        u2 = torch.zeros_like(b_full)
        self.jacobi(a, s, b_full, None, u)
        for _ in range(self.coarse_sweeps):
            self.jacobi(a, s, b_full, u, u2)
            u, u2 = u2, u
        c_full.copy_(u)
