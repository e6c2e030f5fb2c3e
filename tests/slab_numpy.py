"""CPU stand-in for parallel.CudaSlab (test double, numpy on CPU torch buffers).

Same method surface and buffer layout ([halo | own | halo], global voxel p at
local index p - offset + halo) as the CUDA slab, with the arithmetic of
csrc/slab.cuh / fgp.cuh restated in numpy in the oracle's operation order, so
the multi-rank choreography of parallel.SlabProx (halo exchange, pairwise
combine of the per-slab sums) can be checked over gloo against the oracle.
"""

import numpy as np
import torch


class NumpySlab:
    def __init__(self, dims, offset, count):
        self.dims = tuple(int(v) for v in dims)
        depth, height, width = self.dims
        self.dim = 3 if depth > 1 else 2
        self.nvox = depth * height * width
        self.offset, self.count = int(offset), int(count)
        self.halo = height * width if self.dim == 3 else width
        length = count + 2 * self.halo
        z = lambda: torch.zeros(length, dtype=torch.float64)  # noqa: E731
        self._b, self._u = z(), z()
        self._f = [[z() for _ in range(self.dim)] for _ in range(2)]
        self._q = [z() for _ in range(self.dim)]
        self.parity = 0
        self.w = 0.0
        # global voxel index of every local slot, and its coordinates
        p = np.arange(offset - self.halo, offset + count + self.halo)
        self._p = p
        hw = height * width
        pc = np.clip(p, 0, self.nvox - 1)
        self._z, self._s, self._t = pc // hw, (pc % hw) // width, pc % width
        self._own = slice(self.halo, self.halo + count)

    # --- buffers ------------------------------------------------------------
    def set_weight(self, w):
        self.w = float(w)

    def fields(self, name):
        if name == "b":
            return [self._b]
        if name == "u":
            return [self._u]
        if name == "q":
            return list(self._q)
        return list(self._f[self.parity if name == "p" else 1 - self.parity])

    def _np(self, bufs):
        return [b.numpy() for b in bufs]

    # --- stencils on local index arrays --------------------------------------
    def _shift(self, arr, idx, off):
        j = np.clip(idx + off, 0, arr.size - 1)
        return arr[j]

    def _div(self, fields, idx):
        """div at local indices idx, in div_at's order (zero outside the volume)."""
        depth, height, width = self.dims
        hw = height * width
        z, s, t = self._z[idx], self._s[idx], self._t[idx]
        pv, ph = fields[-2], fields[-1]
        a = np.where(s + 1 < height, self._shift(pv, idx, width), 0.0)
        b = np.where(s > 0, pv[idx], 0.0)
        c = np.where(t + 1 < width, self._shift(ph, idx, 1), 0.0)
        d = np.where(t > 0, ph[idx], 0.0)
        if self.dim == 2:
            return ((a - b) + c) - d
        pz = fields[0]
        az = np.where(z + 1 < depth, self._shift(pz, idx, hw), 0.0)
        bz = np.where(z > 0, pz[idx], 0.0)
        return ((((az - bz) + a) - b) + c) - d

    def _tv_terms(self, u, idx):
        height, width = self.dims[1], self.dims[2]
        z, s, t = self._z[idx], self._s[idx], self._t[idx]
        dv = np.where(s > 0, u[idx] - self._shift(u, idx, -width), 0.0)
        dh = np.where(t > 0, u[idx] - self._shift(u, idx, -1), 0.0)
        if self.dim == 2:
            return np.sqrt(dv * dv + dh * dh)
        dz = np.where(z > 0, u[idx] - self._shift(u, idx, -height * width), 0.0)
        return np.sqrt((dz * dz + dv * dv) + dh * dh)

    def _own_idx(self):
        return np.arange(self.halo, self.halo + self.count)

    # --- passes ---------------------------------------------------------------
    interleaved = False   # step / output vectors: this rank's slices, interleaved (slice ownership)

    def _vec_index(self):
        p = np.arange(self.offset, self.offset + self.count)
        if not self.interleaved:
            return p
        hw = self.dims[1] * self.dims[2]
        return (p % hw) * (self.count // hw) + (p // hw - self.offset // hw)

    def step(self, x_k, g, mu):
        o = self._vec_index()
        self._b.numpy()[self._own] = x_k.numpy()[o] + mu * g.numpy()[o]

    def init(self):
        for grp in self._f:
            for f in grp:
                f.zero_()
        for f in self._q:
            f.zero_()
        b = self._b.numpy()
        idx = self._own_idx()
        bo = b[idx]
        return torch.tensor([np.sum(bo * bo), np.sum(self._tv_terms(b, idx))], dtype=torch.float64)

    def candidate(self, from_p):
        src = self._np(self.fields("p") if from_p else self.fields("q"))
        cdst = self._np(self.fields("c"))
        b = self._b.numpy()
        idx = self._own_idx()
        height, width = self.dims[1], self.dims[2]
        hw = height * width
        # u = b + w div src where the candidate reads it: own voxels and one plane below
        lo = max(0, self.halo - (hw if self.dim == 3 else width))
        uidx = np.arange(lo, self.halo + self.count)
        u = np.zeros(b.size)
        valid = self._p[uidx] >= 0
        uu = b[uidx] + self.w * self._div(src, uidx)
        u[uidx] = np.where(valid, uu, 0.0)
        z, s, t = self._z[idx], self._s[idx], self._t[idx]
        uc = u[idx]
        g = []
        if self.dim == 3:
            g.append(np.where(z > 0, uc - self._shift(u, idx, -hw), 0.0))
        g.append(np.where(s > 0, uc - self._shift(u, idx, -width), 0.0))
        g.append(np.where(t > 0, uc - self._shift(u, idx, -1), 0.0))
        step = 1.0 / ((12.0 if self.dim == 3 else 8.0) * self.w)
        c = [src[k][idx] + step * g[k] for k in range(self.dim)]
        m2 = c[0] * c[0] + c[1] * c[1]
        if self.dim == 3:
            m2 = m2 + c[2] * c[2]
        mag = np.sqrt(m2)
        mag = np.where(mag < 1.0, 1.0, mag)
        for k in range(self.dim):
            cdst[k][idx] = c[k] / mag

    def dual(self, beta):
        c = self._np(self.fields("c"))
        p = self._np(self.fields("p"))
        q = self._np(self.fields("q"))
        b = self._b.numpy()
        idx = self._own_idx()
        res = b[idx] + self.w * self._div(c, idx)
        out = [np.sum(res * res)]
        sk = [c[k][idx] - p[k][idx] for k in range(self.dim)]
        for k in range(self.dim):
            q[k][idx] = c[k][idx] + beta * sk[k]
        out += [np.sum(v * v) for v in sk]
        out += [np.sum(c[k][idx] * c[k][idx]) for k in range(self.dim)]
        return torch.tensor(out, dtype=torch.float64)

    def finalize(self):
        p = self._np(self.fields("p"))
        idx = self._own_idx()
        self._u.numpy()[idx] = self._b.numpy()[idx] + self.w * self._div(p, idx)

    def energy(self):
        u, b = self._u.numpy(), self._b.numpy()
        idx = self._own_idx()
        d = u[idx] - b[idx]
        return torch.tensor([np.sum(d * d), np.sum(self._tv_terms(u, idx))], dtype=torch.float64)

    def output(self, fell, x_next, x_k, g, x_true):
        o = self._vec_index()
        src = self._b if fell else self._u
        xv = src.numpy()[self._own].copy()
        x_next.numpy()[o] = xv
        d = xv - x_k.numpy()[o]
        xe = float(np.sum((xv - x_true.numpy()[o]) ** 2)) if x_true is not None else 0.0
        return torch.tensor([float(xv @ xv), xe, float(d @ g.numpy()[o]), float(d @ d)], dtype=torch.float64)


class NumpySlabDevice(NumpySlab):
    """NumpySlab with the device-decision interface of CudaSlab (control block,
    `when`-predicated passes, `decide`): the Python restatement of
    slab.cuh's fgp_decide, so the fixed-sequence choreography of
    parallel.SlabProx.run_device is checked over gloo."""

    def __init__(self, dims, offset, count):
        super().__init__(dims, offset, count)
        self.device = False
        self.ctl = {}

    def fields(self, name):
        if name in ("d0", "d1"):
            return list(self._f[int(name[1])])
        if self.device and name in ("p", "c"):
            par = self.ctl.get("parity", 0)
            return list(self._f[par if name == "p" else 1 - par])
        return super().fields(name)

    def _skip(self, when):
        if not self.device or when == 0:
            return False
        if when == 1:
            return bool(self.ctl["done"])
        return bool(self.ctl["done"]) or not self.ctl["restart"]

    def candidate(self, from_p, when=0):
        if self._skip(when):
            return
        super().candidate(from_p)

    def dual(self, beta, when=0):
        if self._skip(when):
            return torch.zeros(1 + 2 * self.dim, dtype=torch.float64)
        return super().dual(self.ctl["beta"] if self.device else beta)

    def output(self, fell, x_next, x_k, g, x_true):
        return super().output(self.ctl["fell"] if self.device else fell, x_next, x_k, g, x_true)

    @staticmethod
    def _next_beta(c):
        import math
        c["t_next"] = 0.5 * (1.0 + math.sqrt(1.0 + (4.0 * c["t_mom"]) * c["t_mom"]))
        c["beta"] = (c["t_mom"] - 1.0) / c["t_next"]

    def decide(self, stage, it, gathered, program, world, tol):
        import math
        when = stage if stage in (1, 2) else 0
        if self._skip(when):
            return
        k = gathered.numel() // world
        g = gathered.numpy().reshape(world, k)
        stk = []
        for op in program:
            if op >= 0:
                stk.append([float(v) for v in g[op]])
            else:
                b, a = stk.pop(), stk.pop()
                stk.append([x + y for x, y in zip(a, b)])
        v = stk[0]
        c = self.ctl
        if stage == 0:
            c.update(phi_prev=v[0], tv_b=v[1], t_mom=1.0, tv_out=0.0, iters=0, restarts=0, done=0, parity=0,
                     restart=0, fell=0)
            self._next_beta(c)
            return
        if stage == 3:
            two_w = 2.0 * self.w
            c["fell"] = 1 if (v[0] + two_w * v[1]) > (0.0 + two_w * c["tv_b"]) else 0
            c["tv_out"] = v[1]
            return
        phi = v[0]
        if stage == 1 and phi > c["phi_prev"]:
            c["restart"] = 1
            c["restarts"] += 1
            c["t_mom"] = 1.0
            self._next_beta(c)
            return
        c["restart"] = 0
        c["parity"] ^= 1
        c["phi_prev"] = c["phi_prev"] if c["phi_prev"] < phi else phi
        c["t_mom"] = c["t_next"]
        c["iters"] = it + 1
        d = self.dim
        ch2, sc2 = v[1] + v[2], v[1 + d] + v[2 + d]
        if d == 3:
            ch2, sc2 = ch2 + v[3], sc2 + v[6]
        change, scale = math.sqrt(ch2), math.sqrt(sc2)
        if change <= tol * (1e-30 if 1e-30 > scale else scale):
            c["done"] = 1
        else:
            self._next_beta(c)

    def info(self):
        c = self.ctl
        return {"iterations": c["iters"], "converged": c["done"], "restarts": c["restarts"], "fell_back": c["fell"],
                "tv": c["tv_b"] if c["fell"] else c["tv_out"]}
