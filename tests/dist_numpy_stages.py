"""TEST DOUBLE: numpy implementations of the per-rank slab stages
(vsr_slab_* in include/vsr.h) on CPU torch tensors, so the distributed host
orchestration (paper_2010_15491_b200/dist.py) and its exchange layouts can be
tested over gloo on CPU.  Never used by the product path."""
import contextlib
import math

import numpy as np
import torch

import volsr_oracle as O


def _c(t, shape):
    return t.numpy().view(np.complex128).reshape(shape)


def _r(t, shape):
    return t.numpy().reshape(shape)


def _dnorm(length):
    return O.diff_norm_table(length)


class NumpyStages:
    def zeros(self, rank, n, dtype=torch.float64):
        return torch.zeros(n, dtype=dtype)

    def stream(self, rank):
        return contextlib.nullcontext()

    def synchronize(self, rank):
        pass

    def fft3_full(self, rank, dims, x, real, out, scale):
        m, n, s = dims
        a = _r(x, (s, n, m)) if real else _c(x, (s, n, m))
        _c(out, (s, n, m))[...] = np.fft.fftn(a) * scale

    def fwd_xy_pack(self, rank, g, x, real, work, send):
        shp = (g.sz, g.n, g.m)
        a = _r(x, shp) if real else _c(x, shp)
        F = np.fft.fft(np.fft.fft(a, axis=2), axis=1)
        _c(work, shp)[...] = F
        sv = _c(send, (g.P, g.sz, g.nP, g.m))
        for q in range(g.P):
            sv[q] = F[:, g.rows(q), :]

    def axis3(self, rank, g, W, inverse, scale):
        A = _c(W, (g.s, g.nP, g.m))
        A[...] = (np.fft.ifft(A, axis=0) * g.s if inverse else np.fft.fft(A, axis=0)) * scale

    def lr_slice(self, rank, g, Yl, Yl_loc):
        _c(Yl_loc, (g.sl, g.nlP, g.ml))[...] = _c(Yl, (g.sl, g.nl, g.ml))[:, rank * g.nlP:(rank + 1) * g.nlP, :]

    def _local(self, g):
        return O.DecimationSpec((g.m, g.nP, g.s), g.rates)

    def tik_fold(self, rank, g, Yl_loc, lam, xbh, reg, W):
        sp = self._local(g)
        L = _c(lam, (g.s, g.nP, g.m))
        X = _c(xbh, (g.s, g.nP, g.m))
        Y = _c(Yl_loc, (g.sl, g.nlP, g.ml))
        d = sp.rate()
        k = np.conj(L) * (O.alias_expand(Y, sp) / math.sqrt(d)) + 2.0 * reg * X
        f = O.FoldedSpectrum(L, sp)
        w = f.apply(k) / (O.gram_diag(f) + 2.0 * reg * d)
        xh = (k - f.apply_adjoint(w)) * (1.0 / (2.0 * reg))
        _c(W, (g.s, g.nP, g.m))[...] = np.fft.ifft(xh, axis=0) * g.s

    def tv_prepare(self, rank, g, lam):
        pass  # the numpy fold has no cached tables

    def tv_fold(self, rank, g, Yl_loc, lam, W, mu, tau, fwd_scale, fit):
        sp = self._local(g)
        L = _c(lam, (g.s, g.nP, g.m))
        Y = _c(Yl_loc, (g.sl, g.nlP, g.ml))
        A = np.fft.fft(_c(W, (g.s, g.nP, g.m)), axis=0) * fwd_scale
        nr, ns = _dnorm(g.m), _dnorm(g.s)
        nc = _dnorm(g.n)[g.rows(rank)]
        gam = 1.0 / (((nr[None, None, :] + nc[None, :, None]) + ns[:, None, None]) + tau)
        d = sp.rate()
        k = np.conj(L) * (O.alias_expand(Y, sp) / math.sqrt(d)) + mu * A
        f = O.FoldedSpectrum(L, sp)
        ghat = gam * k
        w = f.apply(ghat) / (O.gram_diag_weighted(f, gam) + mu * d)
        xh = (ghat - f.apply_adjoint_weighted(w, gam)) * (1.0 / mu)
        r = Y - f.apply(xh) / math.sqrt(d)
        fit[0] = float(np.sum(np.abs(r) ** 2))
        _c(W, (g.s, g.nP, g.m))[...] = np.fft.ifft(xh, axis=0) * g.s

    def unpack_inv_xy(self, rank, g, recv, work, out, scale, sums, bad):
        R = _c(recv, (g.P, g.sz, g.nP, g.m))
        F = _c(work, (g.sz, g.n, g.m))
        for q in range(g.P):
            F[:, g.rows(q), :] = R[q]
        z = np.fft.ifft(np.fft.ifft(F, axis=1), axis=2) * (g.n * g.m) * scale
        _r(out, (g.sz, g.n, g.m))[...] = z.real
        sums[0] = float(np.sum(z.imag ** 2))
        sums[1] = float(np.sum(np.abs(z) ** 2))
        badm = ~np.isfinite(z.real.reshape(-1))
        bad[0] = int(np.argmax(badm)) if badm.any() else -1

    def stencil(self, rank, g, init, x_ext, dual_in_ext, dual_out_ext, theta, thr, sums):
        x = _r(x_ext, (g.sz + 2, g.n, g.m))
        nxt = lambda a, ax: np.roll(a, -1, axis=ax)
        # rho on ext planes 0..sz (needs x planes 0..sz+1)
        xs, xn = x[:-1], x[1:]
        l0 = nxt(xs, 2) - xs
        l1 = nxt(xs, 1) - xs
        l2 = xn - xs
        if init:
            rho = [l0, l1, l2]
            u = [l0, l1, l2]
            dn = [np.zeros_like(l0)] * 3
        else:
            din = _r(dual_in_ext, (3, g.sz + 1, g.n, g.m))
            nu = [l0 + din[0], l1 + din[1], l2 + din[2]]
            u = list(O.tv_shrink(nu[0], nu[1], nu[2], thr))
            dn = [nu[a] - u[a] for a in range(3)]
            rho = [u[a] - dn[a] for a in range(3)]
        dout = _r(dual_out_ext, (3, g.sz + 1, g.n, g.m))
        for a in range(3):
            dout[a, 1:] = dn[a][1:]
        prev = lambda a, ax: np.roll(a, 1, axis=ax)
        th = ((prev(rho[0], 2) - rho[0])[1:] + (prev(rho[1], 1) - rho[1])[1:]) + (rho[2][:-1] - rho[2][1:])
        _r(theta, (g.sz, g.n, g.m))[...] = th
        lx = [l0[1:], l1[1:], l2[1:]]
        res = 0.0 if init else sum(float(np.sum((lx[a] - u[a][1:]) ** 2)) for a in range(3))
        sums[0] = res
        sums[1] = float(np.sum(np.sqrt(lx[0] ** 2 + lx[1] ** 2 + lx[2] ** 2)))
        sums[2] = 0.0
        sums[3] = 0.0

    def fit(self, rank, g, Yl_loc, lam, xh, out):
        sp = self._local(g)
        L = _c(lam, (g.s, g.nP, g.m))
        Y = _c(Yl_loc, (g.sl, g.nlP, g.ml))
        f = O.FoldedSpectrum(L, sp)
        r = Y - f.apply(_c(xh, (g.s, g.nP, g.m))) / math.sqrt(sp.rate())
        out[0] = float(np.sum(np.abs(r) ** 2))
