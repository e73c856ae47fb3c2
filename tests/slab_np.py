"""tests/slab_np.py -- TEST INFRASTRUCTURE: numpy mirror of the x1-slab protocol.

Restates, per rank, the data movement the slab path of libveloreg_gpu performs
 so the N > 1 decomposition can be checked on CPU with
torch.distributed over gloo (world_size 2 and 4), against the global numpy
oracle (oracle/veloreg_np.py):

  * geometry            -- taken from the library itself (vr_slab_layout)
  * halo exchange       -- Transport::halo: H planes from each x1 neighbour
  * FFT transposes      -- Transport::alltoall: slab [L][n2][nh] <-> x1 layout
                           [n1][n2s][nh] (spectral.cu transpose_to_x1/from_x1)
  * tricubic gathers    -- sl.cu make_stencil/gather: x1 base unwrapped to the
                           image nearest the point's own plane, then made
                           slab-relative and read from the halo-padded slab
  * reductions          -- per-rank partials gathered and summed in rank order
  * grid transfer       -- the coarse-band exchange of the two-level preconditioner
                           (twolevel.cu resample_scalar_slabs)

The compute itself is numpy (the oracle's arithmetic); only the decomposition
is under test here. The CUDA slab path is checked on the GPU
(tests/test_gpu_dist.py).
"""
from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

from oracle import veloreg_np as O
import paper_1808_04487_b200.veloreg as V


def _t(a):
    return torch.from_numpy(np.ascontiguousarray(a))


class Slab:
    """Rank `rank` of `P`: planes [off1, off1 + L) of an (n1, n2, n3) grid."""

    def __init__(self, shape, rank, P, halo):
        self.shape = tuple(shape)
        self.rank, self.P = rank, P
        lay = V.slab_layout(self.shape, rank, P, halo)
        self.L, self.off1, self.H = lay["planes"], lay["first_plane"], lay["halo"]
        self.n2s, self.k2_off = lay["n2s"], lay["k2_off"]
        n1, n2, n3 = self.shape
        self.nh = n3 // 2 + 1
        assert lay["points"] == self.L * n2 * n3 and lay["spectrum"] == self.L * n2 * self.nh
        assert lay["padded_stride"] == (self.L + 2 * self.H) * n2 * n3
        self.h = O.spacing(self.shape)

    # ---- communication ---------------------------------------------------------
    def _exchange(self, sends, recv_shapes, peers_send, peers_recv, tag0):
        reqs, outs = [], []
        for i, (a, p) in enumerate(zip(sends, peers_send)):
            if p == self.rank:
                continue
            reqs.append(dist.isend(_t(a), p, tag=tag0 + i))
        for i, (shp, p) in enumerate(zip(recv_shapes, peers_recv)):
            outs.append(torch.empty(shp, dtype=torch.float64))
            if p != self.rank:
                reqs.append(dist.irecv(outs[-1], p, tag=tag0 + i))
        for r in reqs:
            r.wait()
        return outs

    def halo_pad(self, f):
        """(L, n2, n3) -> (L + 2H, n2, n3): lower halo = left neighbour's last H
        planes, upper halo = right neighbour's first H (periodic in x1)."""
        H, left, right = self.H, (self.rank - 1) % self.P, (self.rank + 1) % self.P
        lo, hi = self._exchange([f[-H:], f[:H]], [f[:H].shape, f[:H].shape], [right, left], [left, right], 10)
        return np.concatenate([lo.numpy(), f, hi.numpy()])

    def alltoall(self, chunks):
        """chunks[r] goes to rank r; returns the chunk received from each rank."""
        P, me = self.P, self.rank
        sends = [c for c in chunks]
        out = [None] * P
        reqs = []
        recv = [torch.empty(c.shape, dtype=torch.float64) for c in chunks]
        for r in range(P):
            if r == me:
                out[r] = np.array(chunks[r])
                continue
            reqs.append(dist.isend(_t(sends[r]), r, tag=100 + me))
            reqs.append(dist.irecv(recv[r], r, tag=100 + r))
        for q in reqs:
            q.wait()
        for r in range(P):
            if r != me:
                out[r] = recv[r].numpy()
        return out

    def allsum(self, x):
        """Rank-ordered sum of per-rank partials (blas1.cu finalize_sums)."""
        parts = [torch.zeros(1, dtype=torch.float64) for _ in range(self.P)]
        dist.all_gather(parts, torch.tensor([float(x)], dtype=torch.float64))
        s = 0.0
        for p in parts:
            s += float(p.item())
        return s

    def allmax(self, x):
        t = torch.tensor([float(x)], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # ---- distributed FFT (spectral.cu fft_r2c / fft_c2r) -----------------------
    def rfft(self, f):
        """slab real (L, n2, n3) -> x1-layout spectrum (n1, n2s, nh) of the global rfftn."""
        a = np.fft.fft(np.fft.rfft(f, axis=2), axis=1)
        re = self.alltoall([np.stack([a[:, r * self.n2s:(r + 1) * self.n2s].real,
                                      a[:, r * self.n2s:(r + 1) * self.n2s].imag]) for r in range(self.P)])
        b = np.concatenate([c[0] + 1j * c[1] for c in re], axis=0)
        return np.fft.fft(b, axis=0)

    def irfft(self, s):
        """x1-layout spectrum (n1, n2s, nh) -> slab real (L, n2, n3), 1/Ng normalised."""
        b = np.fft.ifft(s, axis=0)
        L = self.L
        re = self.alltoall([np.stack([b[r * L:(r + 1) * L].real, b[r * L:(r + 1) * L].imag])
                            for r in range(self.P)])
        a = np.concatenate([c[0] + 1j * c[1] for c in re], axis=1)
        return np.fft.irfft(np.fft.ifft(a, axis=1), n=self.shape[2], axis=2)

    # ---- two-level grid transfer (twolevel.cu resample_scalar_slabs) ----------------
    # The x1-layout spectra hold the k2 rows [k2_off, k2_off + n2s) of every rank. Coarse row
    # j2 (of m2 = n2 / 2) is fine row j2 (j2 < m2 / 2) or j2 + m2 (j2 > m2 / 2), the Nyquist
    # row m2 / 2 folds the fine rows m2 / 2 and 3 m2 / 2: the band a coarse rank needs lives on
    # the lowest / highest quarter of the fine ranks. Restriction: per destination rank the
    # partial alias sums of the rows this rank holds, one all-to-all, blocks added in rank
    # order. Prolongation: all-gathered coarse slabs, every rank fills its own fine rows.
    # (x3 Nyquist-plane images are left to the GPU tests; inputs here stay below them.)
    @staticmethod
    def _fine_rows(j, m):
        """fine indices (axis length 2 m) aliasing onto coarse index j (axis length m)"""
        if 2 * j < m:
            return [j]
        if 2 * j == m:
            return [m // 2, 2 * m - m // 2]
        return [j + m]

    def restrict_to(self, spec, coarse: "Slab"):
        """fine x1-layout spectrum (n1, n2s, nh) of this slab -> coarse (m1, m2s, mh)."""
        (n1, n2, n3), (m1, m2, m3) = self.shape, coarse.shape
        assert (n1, n2, n3) == (2 * m1, 2 * m2, 2 * m3) and coarse.P == self.P
        scale = (m1 * m2 * m3) / (n1 * n2 * n3)
        mh = coarse.nh
        blocks = []
        for q in range(self.P):
            blk = np.zeros((m1, coarse.n2s, mh), dtype=complex)
            for jl in range(coarse.n2s):
                for i2 in self._fine_rows(q * coarse.n2s + jl, m2):
                    l2 = i2 - self.k2_off
                    if not 0 <= l2 < self.n2s:
                        continue  # another rank's row
                    for j1 in range(m1):
                        for i1 in self._fine_rows(j1, m1):
                            blk[j1, jl, :] += spec[i1, l2, :mh]
            blocks.append(np.stack([blk.real, blk.imag]) * scale)
        got = self.alltoall(blocks)
        out = np.zeros((m1, coarse.n2s, mh), dtype=complex)
        for c in got:  # rank order
            out = out + (c[0] + 1j * c[1])
        return out

    def prolong_to(self, spec_c, fine: "Slab"):
        """coarse x1-layout spectrum (m1, m2s, mh) of this slab -> fine (n1, n2s, nh)."""
        (m1, m2, m3), (n1, n2, n3) = self.shape, fine.shape
        assert (n1, n2, n3) == (2 * m1, 2 * m2, 2 * m3)
        scale = (n1 * n2 * n3) / (m1 * m2 * m3)
        own = np.stack([spec_c.real, spec_c.imag])
        allc = self.alltoall([own for _ in range(self.P)])  # all-gather of the coarse slabs
        full = np.concatenate([c[0] + 1j * c[1] for c in allc], axis=1)  # (m1, m2, mh)
        out = np.zeros((n1, fine.n2s, fine.nh), dtype=complex)
        mh = self.nh
        for j2 in range(m2):
            rows2 = self._fine_rows(j2, m2)
            for i2 in rows2:
                l2 = i2 - fine.k2_off
                if not 0 <= l2 < fine.n2s:
                    continue
                for j1 in range(m1):
                    rows1 = self._fine_rows(j1, m1)
                    for i1 in rows1:
                        out[i1, l2, :mh] = full[j1, j2, :] * (scale / (len(rows1) * len(rows2)))
        out[:, :, mh - 1] *= 0.5  # the coarse x3 Nyquist bin folds onto +-m3/2
        return out

    def kgrids(self, deriv=False):
        f = O.deriv_freq if deriv else O.fft_freq
        n1, n2, n3 = self.shape
        k1 = f(n1)[:, None, None]
        k2 = f(n2)[self.k2_off:self.k2_off + self.n2s][None, :, None]
        k3 = (O.deriv_freq(n3) if deriv else O.fft_freq(n3))[: self.nh][None, None, :]
        return k1, k2, k3

    def gradient(self, f):
        c = self.rfft(f)
        k = self.kgrids(deriv=True)
        return np.stack([self.irfft(1j * k[a] * c) for a in range(3)])

    def divergence(self, v):
        k = self.kgrids(deriv=True)
        acc = 0
        for a in range(3):
            acc = acc + 1j * k[a] * self.rfft(v[a])
        return self.irfft(acc)

    def reg(self, v, beta):
        """H2 regularization operator beta (|k|^2)^2 (spectral.cpp:166-184)."""
        k1, k2, k3 = self.kgrids()
        k2f = k1 * k1 + k2 * k2 + k3 * k3
        return np.stack([self.irfft(self.rfft(v[c]) * (beta * k2f * k2f)) for c in range(3)])

    def inner_product(self, a, b):
        vol = O.cell_volume(self.shape)
        if a.ndim == 4:
            return sum(self.allsum(np.sum(a[c] * b[c])) * vol for c in range(3))
        return self.allsum(np.sum(a * b)) * vol

    # ---- semi-Lagrangian on the slab (sl.cu) ----------------------------------
    def coords(self):
        x1, x2, x3 = O.coords(self.shape)
        x1 = x1[self.off1:self.off1 + self.L]
        return np.meshgrid(x1, x2, x3, indexing="ij")

    def tricubic(self, fpad, pts):
        """Interpolate the halo-padded slab fpad at global points pts (3, L, n2, n3)."""
        n1, n2, n3 = self.shape
        (i2, w2) = O._axis_stencil(pts[1], self.h[1], n2)
        (i3, w3) = O._axis_stencil(pts[2], self.h[2], n3)
        u = pts[0] / self.h[0]
        r = np.rint(u)
        u = np.where(np.abs(u - r) < 1e-12, r, u)
        fl = np.floor(u)
        w1 = O.cubic_weights(u - fl)
        b1 = fl.astype(np.int64) - 1
        own = (self.off1 + np.arange(self.L))[:, None, None]
        d = b1 - own
        b1 = np.where(d > n1 // 2, b1 - n1, np.where(d < -(n1 // 2), b1 + n1, b1))
        reach = int(np.max(np.abs(b1 - own)))  # planes between a point and its stencil base
        b1 = b1 - self.off1
        if np.any(b1 < -self.H) or np.any(b1 + 3 >= self.L + self.H):
            raise RuntimeError("departure point beyond the x1 halo")
        flat = fpad.reshape(-1)
        acc = np.zeros(pts.shape[1:])
        for a in range(4):
            o1 = (b1 + a + self.H) * n2
            acc1 = np.zeros_like(acc)
            for b in range(4):
                o2 = (o1 + i2[b]) * n3
                acc2 = np.zeros_like(acc)
                for c in range(4):
                    acc2 = acc2 + w3[c] * flat[o2 + i3[c]]
                acc1 = acc1 + w2[b] * acc2
            acc = acc + w1[a] * acc1
        return acc, reach

    def trace(self, v, nt, direction):
        dt = 1.0 / nt
        sign = -1.0 if direction == "backward" else 1.0
        x = self.coords()
        mid = np.stack([O.wrap_coord(x[c] + sign * 0.5 * dt * v[c]) for c in range(3)])
        vi = [self.tricubic(self.halo_pad(v[c]), mid)[0] for c in range(3)]
        return np.stack([O.wrap_coord(x[c] + sign * dt * vi[c]) for c in range(3)])

    def interp(self, f, pts):
        return self.tricubic(self.halo_pad(f), pts)[0]

    def solve_state(self, m_T, bwd, nt):
        hist = [m_T.copy()]
        for _ in range(nt):
            hist.append(self.interp(hist[-1], bwd))
        return np.stack(hist)

    def gradient_dot(self, f, w):
        g = self.gradient(f)
        out = np.zeros_like(f)
        for a in range(3):
            out = out + g[a] * w[a]
        return out

    def hessian_matvec(self, m_R, m_T, v, vt, nt, beta_v):
        """GN Hessian matvec on the slab, the oracle's sequence (objective.cpp:114-156)."""
        dt, hdt = 1.0 / nt, 0.5 / nt
        bwd = self.trace(v, nt, "backward")
        fwd = self.trace(v, nt, "forward")
        hist = self.solve_state(m_T, bwd, nt)
        dv = self.divergence(v)
        factor = np.exp(0.5 * dt * (dv + self.interp(dv, fwd)))
        # incremental state
        mt = np.zeros_like(m_T)
        q_prev = self.gradient_dot(hist[0], vt)
        for j in range(nt):
            q_next = self.gradient_dot(hist[j + 1], vt)
            tmp = 1.0 * mt + (-hdt) * q_prev
            mt = self.interp(tmp, bwd) + (-hdt) * q_next
            q_prev = q_next
        # incremental adjoint sweep with the body-force accumulation
        b = np.zeros((3,) + m_T.shape)
        cur = -mt
        for j in range(nt, -1, -1):
            if j < nt:
                cur = self.interp(cur, fwd) * factor
            w = 0.5 * dt if (j == 0 or j == nt) else dt
            g = self.gradient(hist[j])
            for a in range(3):
                b[a] = b[a] + w * cur * g[a]
        return b + 1.0 * self.reg(vt, beta_v), hist
