"""Memory-lean restatement of the reference solve path for very large volumes
-- TEST INFRASTRUCTURE ONLY (the checker for BASELINE config 4, 1024^3).

The reference itself (oracle/_ref) needs about 300 bytes of host memory per
HR voxel for admm_tv (measured: 5.0 GB peak RSS at 256^3, 297 B/voxel), i.e.
~320 GB at 1024^3, more than the GPU box's 196 GB host.  This module restates
the same arithmetic as `volsr_oracle` (which follows the reference line by
line) with the large temporaries removed, so the 1024^3 ADMM-TV iterations can
be checked on the box's host in ~100 GB:

  * Lambda is the only HR spectrum kept resident (16 N bytes); FoldedSpectrum's
    block-major copy and hr_index_ (spectral.cpp:37-57) are replaced by strided
    block VIEWS of Lambda in b_lin order (br fastest, spectral.cpp:44-56,63);
  * Gamma (solvers.cpp:191-205) and the difference spectra (operators.cpp:
    225-243) are evaluated per block from their three 1-D tables
    |e^{2 pi i f/len} - 1|^2, in the reference's summation order
    ((rows + cols) + slices) + tau;
  * data_hat = conj(Lambda) * fft3(D^H y) (solvers.cpp:346-348) uses the
    unitary identity fft3_HR(D^H y)[g + b*lr] = fft3_LR(y)[g] / sqrt(d), so
    only the LR spectrum of y is held;
  * every transform runs in place (scipy.fft, all host threads), and the
    elementwise updates are chunked over z planes.

Every formula keeps the reference's operation order except where noted; the
results agree with `volsr_oracle` and with the reference binary to rounding
(pinned in tests/test_oracle_pins.py at sizes both finish in seconds).
Reference: /root/reference/proj/src/solvers.cpp:36-67 (TikhonovOperator),
:219-241 (tv_x_core, tv_denominator), :286-319 (tv_shrink, objective_tv),
:321-411 (admm_tv); src/fft.cpp:66-97 (unitary transforms, residue check).
"""
from __future__ import annotations

import math
import os
import time
from typing import Optional

import numpy as np
import scipy.fft as sfft

from volsr_oracle import (INIT_PROVIDED, INIT_UPSAMPLED, INIT_ZERO, DecimationSpec, NumericError,
                          SolveReport, diff_norm_table, require_positive, shape_of)

WORKERS = os.cpu_count() or 1
ZC = 32  # z planes per elementwise chunk


def _fftn(a: np.ndarray, inverse: bool, norm: Optional[str]) -> np.ndarray:
    f = sfft.ifftn if inverse else sfft.fftn
    return f(a, norm=norm, workers=WORKERS, overwrite_x=True)


def _to_complex(x: np.ndarray) -> np.ndarray:
    out = np.empty(x.shape, np.complex128)
    for z in range(0, x.shape[0], ZC):
        out[z:z + ZC].real = x[z:z + ZC]
        out[z:z + ZC].imag = 0.0
    return out


def psf_to_spectrum(psf: np.ndarray) -> np.ndarray:
    """operators.cpp:121-123: unnormalised DFT of the origin-wrapped PSF."""
    return _fftn(_to_complex(psf), False, None)


def _b6(a: np.ndarray, spec: DecimationSpec) -> np.ndarray:
    dr, dc, ds = spec.rates
    ml, nl, sl = spec.lr
    return a.reshape(ds, sl, dc, nl, dr, ml)


def _blocks(spec: DecimationSpec):
    """(br, bc, bs) in b_lin = br + dr*bc + dr*dc*bs ascending (spectral.cpp:63)."""
    dr, dc, ds = spec.rates
    for bs in range(ds):
        for bc in range(dc):
            for br in range(dr):
                yield br, bc, bs


def _blk(v6: np.ndarray, br: int, bc: int, bs: int) -> np.ndarray:
    return v6[bs, :, bc, :, br, :]


class _GammaTables:
    """make_gamma (solvers.cpp:191-205) per alias block from 1-D tables."""

    def __init__(self, spec: DecimationSpec, tau: float):
        if tau < 0.0:
            raise ValueError("make_gamma: tau must be nonnegative")
        m, n, s = spec.hr
        self.nr, self.nc, self.ns = diff_norm_table(m), diff_norm_table(n), diff_norm_table(s)
        self.spec, self.tau = spec, tau
        if not (tau > 0.0):
            raise NumericError(
                "make_gamma: difference-operator gram is singular at the zero frequency (DC); "
                "a positive tau floor is required")

    def block(self, br, bc, bs):
        ml, nl, sl = self.spec.lr
        a = self.nr[br * ml:(br + 1) * ml][None, None, :]
        b = self.nc[bc * nl:(bc + 1) * nl][None, :, None]
        c = self.ns[bs * sl:(bs + 1) * sl][:, None, None]
        return 1.0 / (((a + b) + c) + self.tau)


def ifft3_real_inplace(xh: np.ndarray, max_rel_imag: float = 1e-8) -> np.ndarray:
    """fft.cpp:82-97 on a complex HR array that is consumed (transformed in place)."""
    full = _fftn(xh, True, "ortho")
    im2 = tot2 = 0.0
    out = np.empty(full.shape, np.float64)
    for z in range(0, full.shape[0], ZC):
        c = full[z:z + ZC]
        re, im = c.real, c.imag
        im2 += float(np.sum(im * im))
        tot2 += float(np.sum(re * re + im * im))
        out[z:z + ZC] = re
    del full
    if tot2 > 0.0 and math.sqrt(im2 / tot2) > max_rel_imag:
        raise NumericError(f"ifft3_real: imaginary residue {math.sqrt(im2 / tot2)} exceeds {max_rel_imag} "
                           "(spectral bookkeeping bug?)")
    return out


def _require_finite(x: np.ndarray, where: str):
    for z in range(0, x.shape[0], ZC):
        bad = ~np.isfinite(x[z:z + ZC])
        if bad.any():
            p = int(np.argmax(bad.reshape(-1))) + z * x.shape[1] * x.shape[2]
            raise NumericError(f"{where}: non-finite value at flat index {p}")


def tikhonov_fast(y, psf_or_lam, spec: DecimationSpec, reg: float, xbar: np.ndarray) -> np.ndarray:
    """solvers.cpp:36-67 (ctor + solve): x = ifft3_real((k - apply_adjoint(
    apply(k) / (gram + 2 reg d))) / (2 reg)), k = conj(L) fft3(D^H y) + 2 reg fft3(xbar)."""
    require_positive(reg, "lambda")
    lam = psf_or_lam if np.iscomplexobj(psf_or_lam) else psf_to_spectrum(psf_or_lam)
    d = spec.rate()
    k = _fftn(_to_complex(xbar), False, "ortho")            # xbar_hat_ (:45)
    yl = _fftn(y.astype(np.complex128), False, "ortho") / math.sqrt(d)
    L6, K6 = _b6(lam, spec), _b6(k, spec)
    ml, nl, sl = spec.lr
    gram = np.zeros((sl, nl, ml))
    w = np.zeros((sl, nl, ml), np.complex128)
    for br, bc, bs in _blocks(spec):
        Lb, kb = _blk(L6, br, bc, bs), _blk(K6, br, bc, bs)
        kb[...] = np.conj(Lb) * yl + 2.0 * reg * kb          # (:53-54)
        gram += Lb.real * Lb.real + Lb.imag * Lb.imag       # gram_diag (spectral.cpp:125-131)
        w += Lb * kb                                        # apply (spectral.cpp:67-75)
    w /= gram + 2.0 * reg * float(d)                        # (:42-44, :56-57)
    inv = 1.0 / (2.0 * reg)
    for br, bc, bs in _blocks(spec):
        Lb, kb = _blk(L6, br, bc, bs), _blk(K6, br, bc, bs)
        kb[...] = (kb - np.conj(Lb) * w) * inv              # (:58-62)
    x = ifft3_real_inplace(k)
    _require_finite(x, "tikhonov_fast")
    return x


def _roll_diff(x: np.ndarray, axis: int, forward: bool) -> np.ndarray:
    """operators.cpp:191-223: forward x[next] - x[p]; adjoint x[prev] - x[p]."""
    npax = {0: 2, 1: 1, 2: 0}[axis]
    return np.roll(x, -1 if forward else 1, axis=npax) - x


def _objective(x, y, lam, spec, lam_tv, lx=None):
    """objective_tv (solvers.cpp:303-319): 0.5 ||y - D H x||^2 + w sum_j ||(Lx)_j||."""
    tv = 0.0
    if lx is None:
        lx = [_roll_diff(x, a, True) for a in range(3)]
    for z in range(0, x.shape[0], ZC):
        g = [l[z:z + ZC] for l in lx]
        tv += float(np.sum(np.sqrt(g[0] * g[0] + g[1] * g[1] + g[2] * g[2])))
    del lx
    xh = _fftn(_to_complex(x), False, "ortho")
    for z in range(0, x.shape[0], ZC):
        xh[z:z + ZC] *= lam[z:z + ZC]
    hx = _fftn(xh, True, "ortho")
    dr, dc, ds = spec.rates
    zv = np.ascontiguousarray(hx[::ds, ::dc, ::dr].real)
    del hx, xh
    r = y - zv
    fit = float(np.sum(r * r))
    return 0.5 * fit + lam_tv * tv


def admm_tv(y, psf, spec: DecimationSpec, lam_tv: float, mu: float, max_iters: int, tau: Optional[float] = None,
            init: int = INIT_ZERO, init_volume=None, log=None):
    """solvers.cpp:321-411 with rel_tol = 0 (fixed iteration count)."""
    require_positive(lam_tv, "lambda")
    require_positive(mu, "mu")
    if max_iters < 1:
        raise ValueError("admm_tv: max_iters must be >= 1")
    t0 = time.perf_counter()
    hr = spec.hr
    d = spec.rate()
    tau = 1e-8 * mu if tau is None else tau
    lam = psf_to_spectrum(psf)
    gam = _GammaTables(spec, tau)
    L6 = _b6(lam, spec)
    ml, nl, sl = spec.lr
    denom = np.zeros((sl, nl, ml))
    for br, bc, bs in _blocks(spec):                        # tv_denominator (:235-241)
        Lb = _blk(L6, br, bc, bs)
        denom += gam.block(br, bc, bs) * (Lb.real * Lb.real + Lb.imag * Lb.imag)
    denom += mu * float(d)
    yl = _fftn(y.astype(np.complex128), False, "ortho") / math.sqrt(d)  # fft3(D^H y) in LR form
    if init == INIT_ZERO:
        x = np.zeros(shape_of(hr))
    elif init == INIT_UPSAMPLED:
        dr, dc, ds = spec.rates
        x = np.repeat(np.repeat(np.repeat(y, ds, 0), dc, 1), dr, 2)  # nn_upsample (operators.cpp:155-164)
    else:
        x = np.array(init_volume, dtype=np.float64, copy=True)
    u = [_roll_diff(x, a, True) for a in range(3)]
    dual = [np.zeros(shape_of(hr)) for _ in range(3)]
    rep = SolveReport()
    rep.initial_objective = _objective(x, y, lam, spec, lam_tv)
    thr = lam_tv / mu
    for it in range(1, max_iters + 1):
        theta = np.zeros(shape_of(hr))
        for a in range(3):                                  # (:367-373)
            rho = u[a] - dual[a]
            theta += _roll_diff(rho, a, False)
            del rho
        del u
        k = _fftn(_to_complex(theta), False, "ortho")
        del theta
        K6 = _b6(k, spec)
        w = np.zeros((sl, nl, ml), np.complex128)
        for br, bc, bs in _blocks(spec):
            Lb, kb = _blk(L6, br, bc, bs), _blk(K6, br, bc, bs)
            kb[...] = np.conj(Lb) * yl + mu * kb            # k_hat = data_hat + mu fft3(theta) (:374-375)
            kb *= gam.block(br, bc, bs)                      # g_hat = Gamma k_hat (:223)
            w += Lb * kb                                     # apply (spectral.cpp:71-73)
        w /= denom                                           # (:226)
        inv = 1.0 / mu
        for br, bc, bs in _blocks(spec):
            Lb, kb = _blk(L6, br, bc, bs), _blk(K6, br, bc, bs)
            kb[...] = (kb - (gam.block(br, bc, bs) * np.conj(Lb)) * w) * inv  # (:228-231, spectral.cpp:110)
        del K6
        x = ifft3_real_inplace(k)
        del k
        lx = [_roll_diff(x, a, True) for a in range(3)]
        for a in range(3):
            dual[a] += lx[a]                                 # nu = Lx + dual (:380-382)
        u = [np.empty(shape_of(hr)) for _ in range(3)]
        residual = 0.0
        for z in range(0, x.shape[0], ZC):                   # tv_shrink (:286-301) + dual (:384-392)
            n1, n2, n3 = (dual[a][z:z + ZC] for a in range(3))
            mag = np.sqrt(n1 * n1 + n2 * n2 + n3 * n3)
            with np.errstate(divide="ignore", invalid="ignore"):
                f = np.where(mag > thr, 1.0 - thr / mag, 0.0)
            for a, na in enumerate((n1, n2, n3)):
                ua = f * na
                u[a][z:z + ZC] = ua
                r = lx[a][z:z + ZC] - ua
                residual += float(np.sum(r * r))
                na -= ua                                     # dual = nu - u
        obj = _objective(x, y, lam, spec, lam_tv, lx)
        del lx
        rep.objective.append(obj)
        rep.primal_residual.append(math.sqrt(residual))
        rep.iterations = it
        if log:
            log(f"lean admm_tv iteration {it}: objective {obj!r}, residual {math.sqrt(residual)!r}, "
                f"{time.perf_counter() - t0:.1f} s")
    _require_finite(x, "admm_tv")
    rep.seconds = time.perf_counter() - t0
    return x, rep
