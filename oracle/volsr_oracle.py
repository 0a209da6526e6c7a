"""CPU oracle for the 3D-FSR reconstruction hot path — TEST INFRASTRUCTURE ONLY.

This module is a numpy restatement of the reference `volsr` C++ solver path
(`/root/reference/proj/src/*.cpp`).  It is the *checker*: only `tests/`,
`__graft_entry__.smoke()` and `bench.py`'s CPU-baseline leg may import it.
The product path (`paper_2010_15491_b200`) never calls into this file and
fails loudly when its CUDA library is missing.

Pinning: this restatement is checked (tests/test_oracle_pins.py) against
  * the reference's own known-answer tests restated (DC = c*sqrt(N), Parseval,
    dense unitary DFT agreement, identity-operator Tikhonov formula, huge-lambda
    limit, dense normal-equation oracles, shrink closed forms), and
  * the reference itself compiled here from its sources (oracle/_ref, built by
    oracle/Makefile with a FFTW3-API shim and an Eigen-subset shim) through
    committed golden vectors under tests/golden/ (tools/make_golden.py).

Conventions (reference `include/volsr/volume.hpp:26-45`): a volume with dims
(m, n, s) is stored lexicographically with axis 1 (m) fastest; here it is a
numpy array of shape (s, n, m) in C order, so the flat index is i + m*j + m*n*k.
The third-party FFT (FFTW3, version unpinned in the reference,
`proj/CMakeLists.txt:16-17`) is restated by numpy's pocketfft: unitary
(`norm="ortho"`) for fft3/ifft3 (`src/fft.cpp:66-80`), unnormalised for
dft3_unnormalized (`src/fft.cpp:99-101`); sign -1 forward.
"""
from __future__ import annotations

import math
import time
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np


class ShapeError(ValueError):
    """reference `volume.hpp:12-15` shape_error (derives std::invalid_argument)."""


class NumericError(RuntimeError):
    """reference `volume.hpp:18-20` numeric_error."""


def dims_of(v: np.ndarray) -> tuple:
    """(m, n, s) of a volume stored as shape (s, n, m)."""
    s, n, m = v.shape
    return (m, n, s)


def shape_of(dims: Sequence[int]) -> tuple:
    m, n, s = dims
    return (s, n, m)


def require_same_dims(a, b, where: str):
    """reference `src/volume.cpp:25-29`."""
    if tuple(a) != tuple(b):
        raise ShapeError(f"{where}: dims mismatch, {a} vs {b}")


def require_finite(v: np.ndarray, where: str):
    """reference `src/volume.cpp:31-36`: first non-finite flat index."""
    bad = ~np.isfinite(v.reshape(-1))
    if bad.any():
        p = int(np.argmax(bad))
        raise NumericError(f"{where}: non-finite value at flat index {p}")


def require_positive(v: float, name: str):
    """reference `src/solvers.cpp:18-22`."""
    if not (v > 0.0):
        raise ValueError(f"{name} must be positive, got {v}")


# --------------------------------------------------------------------------
# Decimation spec (reference src/operators.cpp:8-21)
# --------------------------------------------------------------------------
class DecimationSpec:
    def __init__(self, hr_dims: Sequence[int], rates: Sequence[int]):
        names = ("1 (rows)", "2 (cols)", "3 (slices)")
        for a in range(3):
            if rates[a] == 0:
                raise ShapeError(f"DecimationSpec: zero rate on axis {names[a]}")
            if hr_dims[a] % rates[a] != 0:
                raise ShapeError(
                    f"DecimationSpec: rate {rates[a]} does not divide axis {names[a]} "
                    f"of length {hr_dims[a]}")
        self.hr = tuple(int(x) for x in hr_dims)
        self.rates = tuple(int(r) for r in rates)
        self.lr = tuple(self.hr[a] // self.rates[a] for a in range(3))

    def rate(self) -> int:
        return self.rates[0] * self.rates[1] * self.rates[2]


# --------------------------------------------------------------------------
# FFT contract (reference src/fft.cpp)
# --------------------------------------------------------------------------
_counters = {"forward": 0, "inverse": 0}


def reset_fft_counters():
    """reference src/fft.cpp:108-111."""
    _counters["forward"] = 0
    _counters["inverse"] = 0


def fft_counters():
    return dict(_counters)


def fft3(v: np.ndarray) -> np.ndarray:
    """Unitary forward 3D DFT (reference src/fft.cpp:66-73)."""
    if v.size == 0:
        raise ShapeError("fft3: empty volume")
    _counters["forward"] += 1
    return np.fft.fftn(v.astype(np.complex128, copy=False), norm="ortho")


def ifft3(v: np.ndarray) -> np.ndarray:
    """Unitary inverse 3D DFT (reference src/fft.cpp:75-80)."""
    if v.size == 0:
        raise ShapeError("fft3: empty volume")
    _counters["inverse"] += 1
    return np.fft.ifftn(v, norm="ortho")


def ifft3_real(v: np.ndarray, max_rel_imag: float = 1e-8) -> np.ndarray:
    """reference src/fft.cpp:82-97: L2 imaginary-residue check then real part."""
    full = ifft3(v)
    imag_sq = float(np.sum(full.imag * full.imag))
    total_sq = float(np.sum(full.real * full.real + full.imag * full.imag))
    if total_sq > 0.0 and math.sqrt(imag_sq / total_sq) > max_rel_imag:
        raise NumericError(
            f"ifft3_real: imaginary residue {math.sqrt(imag_sq / total_sq)} exceeds "
            f"{max_rel_imag} (spectral bookkeeping bug?)")
    return np.ascontiguousarray(full.real)


def dft3_unnormalized(v: np.ndarray) -> np.ndarray:
    """reference src/fft.cpp:99-101."""
    _counters["forward"] += 1
    return np.fft.fftn(v.astype(np.complex128, copy=False))


# --------------------------------------------------------------------------
# Forward-model operators (reference src/operators.cpp)
# --------------------------------------------------------------------------
def _sample_gaussian_1d(size: int, sigma: float) -> np.ndarray:
    """reference src/operators.cpp:48-60."""
    half = size // 2
    t = np.arange(-half, half + 1, dtype=np.float64)
    if sigma <= 0.0:
        return (t == 0).astype(np.float64)
    return np.exp(-0.5 * (t / sigma) * (t / sigma))


def make_gaussian_psf(size: Sequence[int], sigma: Sequence[float], hr_dims: Sequence[int],
                      weights: Optional[np.ndarray] = None) -> np.ndarray:
    """reference src/operators.cpp:64-119: sampled separable Gaussian (or explicit
    weights, normalised by PsfSpec::explicit_kernel :30-44), normalised to unit
    sum, centre wrapped to voxel (0,0,0)."""
    for a in range(3):
        if size[a] % 2 == 0:
            raise ValueError(f"make_gaussian_psf: kernel size must be odd on axis {a + 1}")
    for a in range(3):
        if size[a] > hr_dims[a]:
            raise ValueError(
                f"make_gaussian_psf: kernel size {size[a]} exceeds volume axis {a + 1} "
                f"of length {hr_dims[a]}")
    kr, kc, ks = size
    if weights is not None:
        w = np.asarray(weights, dtype=np.float64).reshape(-1)
        if w.size != kr * kc * ks:
            raise ValueError("PsfSpec: weight count does not match kernel size")
        if not np.all(w >= 0.0):
            raise ValueError("PsfSpec: weights must be nonnegative")
        tot = 0.0
        for x in w:
            tot += x
        if tot <= 0.0:
            raise ValueError("PsfSpec: weights must not all be zero")
        kernel = (w / tot).reshape(ks, kc, kr)
    else:
        wr = _sample_gaussian_1d(kr, sigma[0])
        wc = _sample_gaussian_1d(kc, sigma[1])
        ws = _sample_gaussian_1d(ks, sigma[2])
        kernel = (wr[None, None, :] * wc[None, :, None]) * ws[:, None, None]
        tot = 0.0
        for x in kernel.reshape(-1):  # sequential sum, reference :86-93
            tot += x
        kernel = kernel / tot
    psf = np.zeros(shape_of(hr_dims), dtype=np.float64)
    m, n, s = hr_dims
    ii = (np.arange(kr) - kr // 2) % m
    jj = (np.arange(kc) - kc // 2) % n
    kk = (np.arange(ks) - ks // 2) % s
    for c in range(ks):
        for b in range(kc):
            np.add.at(psf[kk[c], jj[b]], ii, kernel[c, b])
    return psf


def psf_to_spectrum(psf: np.ndarray) -> np.ndarray:
    """reference src/operators.cpp:121-123 (Lambda = unnormalised DFT)."""
    return dft3_unnormalized(psf)


def blur_apply(x: np.ndarray, lam: np.ndarray, conjugate: bool = False) -> np.ndarray:
    """reference src/operators.cpp:125-131."""
    require_same_dims(dims_of(x), dims_of(lam), "blur_apply")
    xh = fft3(x)
    xh = xh * (np.conj(lam) if conjugate else lam)
    return ifft3_real(xh)


def decimate(x: np.ndarray, spec: DecimationSpec) -> np.ndarray:
    """reference src/operators.cpp:133-142: y[i,j,k] = x[i*dr, j*dc, k*ds]."""
    require_same_dims(dims_of(x), spec.hr, "decimate")
    dr, dc, ds = spec.rates
    return np.ascontiguousarray(x[::ds, ::dc, ::dr])


def decimate_adjoint(y: np.ndarray, spec: DecimationSpec) -> np.ndarray:
    """reference src/operators.cpp:144-153 (zero interpolation)."""
    require_same_dims(dims_of(y), spec.lr, "decimate_adjoint")
    dr, dc, ds = spec.rates
    x = np.zeros(shape_of(spec.hr), dtype=np.float64)
    x[::ds, ::dc, ::dr] = y
    return x


def nn_upsample(y: np.ndarray, spec: DecimationSpec) -> np.ndarray:
    """reference src/operators.cpp:155-164."""
    require_same_dims(dims_of(y), spec.lr, "nn_upsample")
    dr, dc, ds = spec.rates
    return np.ascontiguousarray(np.repeat(np.repeat(np.repeat(y, ds, 0), dc, 1), dr, 2))


def zero_fill_upsample(y: np.ndarray, spec: DecimationSpec) -> np.ndarray:
    """reference src/operators.cpp:166-171."""
    return decimate_adjoint(y, spec) * float(spec.rate())


_AXIS_NP = {0: 2, 1: 1, 2: 0}  # reference Axis (Rows, Cols, Slices) -> numpy axis


def diff_forward(x: np.ndarray, axis: int) -> np.ndarray:
    """reference src/operators.cpp:191-206: out[p] = x[next] - x[p], periodic."""
    return np.roll(x, -1, axis=_AXIS_NP[axis]) - x


def diff_adjoint(x: np.ndarray, axis: int) -> np.ndarray:
    """reference src/operators.cpp:208-223: out[p] = x[prev] - x[p], periodic."""
    return np.roll(x, 1, axis=_AXIS_NP[axis]) - x


def diff_norm_table(length: int) -> np.ndarray:
    """|e^{2 pi i f/len} - 1|^2 per frequency, evaluated exactly as
    std::norm({cos(ang) - 1, sin(ang)}) (reference src/operators.cpp:233-240)."""
    f = np.arange(length, dtype=np.float64)
    ang = 2.0 * math.pi * f / float(length)
    re = np.cos(ang) - 1.0
    im = np.sin(ang)
    out = re * re + im * im
    out[0] = 0.0  # exact zero at DC
    return out


def finite_diff_spectra(hr_dims: Sequence[int]):
    """reference src/operators.cpp:225-243 (rows, cols, slices spectra)."""
    m, n, s = hr_dims

    def ev(length):
        f = np.arange(length, dtype=np.float64)
        ang = 2.0 * math.pi * f / float(length)
        z = (np.cos(ang) - 1.0) + 1j * np.sin(ang)
        z[0] = 0.0
        return z

    shape = shape_of(hr_dims)
    rows = np.broadcast_to(ev(m)[None, None, :], shape).astype(np.complex128)
    cols = np.broadcast_to(ev(n)[None, :, None], shape).astype(np.complex128)
    slices = np.broadcast_to(ev(s)[:, None, None], shape).astype(np.complex128)
    return rows, cols, slices


def make_gamma_from_spectra(diffs, tau: float) -> np.ndarray:
    """reference src/solvers.cpp:191-205."""
    if tau < 0.0:
        raise ValueError("make_gamma: tau must be nonnegative")
    r, c, s = diffs
    nr = r.real * r.real + r.imag * r.imag
    nc = c.real * c.real + c.imag * c.imag
    ns = s.real * s.real + s.imag * s.imag
    g = ((nr + nc) + ns) + tau
    if not np.all(g > 0.0):
        raise NumericError(
            "make_gamma: difference-operator gram is singular at the zero frequency (DC); "
            "a positive tau floor is required")
    return 1.0 / g


def make_gamma(hr_dims: Sequence[int], tau: float) -> np.ndarray:
    return make_gamma_from_spectra(finite_diff_spectra(hr_dims), tau)


# --------------------------------------------------------------------------
# Spectral fold (reference src/spectral.cpp)
# --------------------------------------------------------------------------
def _blocks(v: np.ndarray, spec: DecimationSpec) -> np.ndarray:
    """View of an HR spectrum as [b_lin, g3, g2, g1] with b_lin = br + dr*bc + dr*dc*bs
    (contiguous frequency blocks, reference spectral.cpp:37-57,63)."""
    dr, dc, ds = spec.rates
    ml, nl, sl = spec.lr
    t = v.reshape(ds, sl, dc, nl, dr, ml)
    t = t.transpose(0, 2, 4, 1, 3, 5)  # bs, bc, br, g3, g2, g1
    return t.reshape(ds * dc * dr, sl, nl, ml)


def _unblocks(b: np.ndarray, spec: DecimationSpec) -> np.ndarray:
    dr, dc, ds = spec.rates
    ml, nl, sl = spec.lr
    t = b.reshape(ds, dc, dr, sl, nl, ml).transpose(0, 3, 1, 4, 2, 5)
    return np.ascontiguousarray(t.reshape(shape_of(spec.hr)))


def alias_fold(hr_spectrum: np.ndarray, spec: DecimationSpec) -> np.ndarray:
    """reference src/spectral.cpp:7-20 (sum over blocks, b_lin ascending)."""
    require_same_dims(dims_of(hr_spectrum), spec.hr, "alias_fold")
    b = _blocks(hr_spectrum, spec)
    out = np.zeros(b.shape[1:], dtype=np.complex128)
    for i in range(b.shape[0]):
        out = out + b[i]
    return out


def alias_expand(lr_spectrum: np.ndarray, spec: DecimationSpec) -> np.ndarray:
    """reference src/spectral.cpp:22-35."""
    require_same_dims(dims_of(lr_spectrum), spec.lr, "alias_expand")
    b = np.broadcast_to(lr_spectrum[None], (spec.rate(),) + lr_spectrum.shape)
    return _unblocks(b, spec)


class FoldedSpectrum:
    """reference src/spectral.cpp:37-113 (block-major Lambda, b_lin order)."""

    def __init__(self, lam: np.ndarray, spec: DecimationSpec):
        require_same_dims(dims_of(lam), spec.hr, "FoldedSpectrum")
        self.spec = spec
        self.blocks = np.ascontiguousarray(_blocks(lam, spec))

    def block_value(self, br, bc, bs, g_flat):
        sp = self.spec
        if br >= sp.rates[0] or bc >= sp.rates[1] or bs >= sp.rates[2]:
            raise IndexError("FoldedSpectrum::block_value: block offset out of range")
        b = br + sp.rates[0] * bc + sp.rates[0] * sp.rates[1] * bs
        return self.blocks[b].reshape(-1)[g_flat]

    def apply(self, hr_spectrum):
        """w[g] = sum_b blocks[b,g] * v[hr(b,g)], b ascending (spectral.cpp:67-75)."""
        require_same_dims(dims_of(hr_spectrum), self.spec.hr, "FoldedSpectrum::apply")
        v = _blocks(hr_spectrum, self.spec)
        out = np.zeros(v.shape[1:], dtype=np.complex128)
        for b in range(v.shape[0]):
            out = out + self.blocks[b] * v[b]
        return out

    def apply_adjoint(self, lr_spectrum):
        """spectral.cpp:77-85."""
        require_same_dims(dims_of(lr_spectrum), self.spec.lr, "FoldedSpectrum::apply_adjoint")
        return _unblocks(np.conj(self.blocks) * lr_spectrum[None], self.spec)

    def apply_weighted(self, hr_spectrum, hr_weights):
        """spectral.cpp:87-99."""
        v = _blocks(hr_spectrum, self.spec)
        w = _blocks(hr_weights, self.spec)
        out = np.zeros(v.shape[1:], dtype=np.complex128)
        for b in range(v.shape[0]):
            out = out + (self.blocks[b] * w[b]) * v[b]
        return out

    def apply_adjoint_weighted(self, lr_spectrum, hr_weights):
        """spectral.cpp:101-113: out = w * conj(block) * lr."""
        w = _blocks(hr_weights, self.spec)
        return _unblocks((w * np.conj(self.blocks)) * lr_spectrum[None], self.spec)

    def swap_blocks_for_fault_injection(self):
        """spectral.cpp:115-119."""
        if self.spec.rate() < 2:
            return
        self.blocks[[0, 1]] = self.blocks[[1, 0]]


def gram_diag(folded: FoldedSpectrum) -> np.ndarray:
    """spectral.cpp:125-131."""
    out = np.zeros(folded.blocks.shape[1:], dtype=np.float64)
    for b in range(folded.blocks.shape[0]):
        z = folded.blocks[b]
        out = out + (z.real * z.real + z.imag * z.imag)
    return out


def gram_diag_weighted(folded: FoldedSpectrum, hr_weights: np.ndarray) -> np.ndarray:
    """spectral.cpp:133-142."""
    w = _blocks(hr_weights, folded.spec)
    out = np.zeros(folded.blocks.shape[1:], dtype=np.float64)
    for b in range(folded.blocks.shape[0]):
        z = folded.blocks[b]
        out = out + w[b] * (z.real * z.real + z.imag * z.imag)
    return out


# --------------------------------------------------------------------------
# Solvers (reference src/solvers.cpp)
# --------------------------------------------------------------------------
@dataclass
class SolveReport:
    """reference include/volsr/solvers.hpp:15-21."""
    iterations: int = 0
    initial_objective: float = 0.0
    objective: list = field(default_factory=list)
    primal_residual: list = field(default_factory=list)
    seconds: float = 0.0


def rel_change(nxt: np.ndarray, prev: np.ndarray) -> float:
    """reference src/solvers.cpp:24-32."""
    d = nxt - prev
    return math.sqrt(float(np.sum(d * d))) / max(math.sqrt(float(np.sum(prev * prev))), 1e-300)


class TikhonovOperator:
    """reference src/solvers.cpp:36-67."""

    def __init__(self, lam: np.ndarray, spec: DecimationSpec, reg: float, xbar: np.ndarray):
        require_positive(reg, "lambda")
        require_same_dims(dims_of(lam), spec.hr, "TikhonovOperator")
        require_same_dims(dims_of(xbar), spec.hr, "TikhonovOperator: xbar")
        self.spec = spec
        self.lam = lam
        self.reg = reg
        self.folded = FoldedSpectrum(lam, spec)
        self.denom = gram_diag(self.folded) + 2.0 * reg * float(spec.rate())
        self.xbar_hat = fft3(xbar)

    def solve(self, y: np.ndarray) -> np.ndarray:
        require_same_dims(dims_of(y), self.spec.lr, "TikhonovOperator::solve")
        k_hat = fft3(decimate_adjoint(y, self.spec))
        k_hat = np.conj(self.lam) * k_hat + 2.0 * self.reg * self.xbar_hat
        w = self.folded.apply(k_hat) / self.denom
        corr = self.folded.apply_adjoint(w)
        x_hat = (k_hat - corr) * (1.0 / (2.0 * self.reg))
        x = ifft3_real(x_hat)
        require_finite(x, "tikhonov_fast")
        return x


def tikhonov_fast(y, lam, spec, reg, xbar):
    """reference src/solvers.cpp:69-72."""
    return TikhonovOperator(lam, spec, reg, xbar).solve(y)


def _tv_x_core(k_hat, folded, spec, mu, gamma, denom):
    """reference src/solvers.cpp:219-233."""
    g_hat = gamma * k_hat
    w = folded.apply(g_hat) / denom
    corr = folded.apply_adjoint_weighted(w, gamma)
    x_hat = (g_hat - corr) * (1.0 / mu)
    return ifft3_real(x_hat), x_hat


def tv_denominator(folded, spec, mu, gamma):
    """reference src/solvers.cpp:235-241."""
    return gram_diag_weighted(folded, gamma) + mu * float(spec.rate())


def require_gamma_valid(gamma):
    """reference src/solvers.cpp:209-216."""
    bad = ~((gamma > 0.0) & np.isfinite(gamma))
    if bad.any():
        p = int(np.argmax(bad.reshape(-1)))
        raise NumericError(
            "tv_x_update: gamma must be strictly positive and finite everywhere; entry "
            f"{p} is not (unfloored DC singularity of the difference gram?)")


def tv_x_update(y, folded, lam, spec, mu, theta_hat, gamma):
    """reference src/solvers.cpp:245-259."""
    require_positive(mu, "mu")
    require_same_dims(dims_of(y), spec.lr, "tv_x_update")
    require_same_dims(dims_of(theta_hat), spec.hr, "tv_x_update: theta_hat")
    require_same_dims(dims_of(gamma), spec.hr, "tv_x_update: gamma")
    require_gamma_valid(gamma)
    k_hat = fft3(decimate_adjoint(y, spec))
    k_hat = np.conj(lam) * k_hat + mu * theta_hat
    x, _ = _tv_x_core(k_hat, folded, spec, mu, gamma, tv_denominator(folded, spec, mu, gamma))
    return x


def tv_shrink(nu1, nu2, nu3, threshold):
    """reference src/solvers.cpp:286-301 (strict '>' at the threshold)."""
    if threshold < 0.0:
        raise ValueError("tv_shrink: threshold must be >= 0")
    mag = np.sqrt(nu1 * nu1 + nu2 * nu2 + nu3 * nu3)
    with np.errstate(divide="ignore", invalid="ignore"):
        factor = np.where(mag > threshold, 1.0 - threshold / mag, 0.0)
    return factor * nu1, factor * nu2, factor * nu3


def objective_tv(x, y, lam, spec, tv_weight):
    """reference src/solvers.cpp:303-319."""
    require_same_dims(dims_of(x), spec.hr, "objective_tv")
    require_same_dims(dims_of(y), spec.lr, "objective_tv")
    z = decimate(blur_apply(x, lam), spec)
    fit = float(np.sum((y - z) * (y - z)))
    g = [diff_forward(x, a) for a in range(3)]
    tv = float(np.sum(np.sqrt(g[0] * g[0] + g[1] * g[1] + g[2] * g[2])))
    return 0.5 * fit + tv_weight * tv


INIT_ZERO, INIT_UPSAMPLED, INIT_PROVIDED = 0, 1, 2


def admm_tv(y, psf, spec, lam_tv=0.06, mu=0.1, max_iters=30, rel_tol=1e-6, tau=None,
            init=INIT_ZERO, init_volume=None, return_state=False):
    """reference src/solvers.cpp:321-411 (ADMM-TV, Algorithm 1)."""
    require_positive(lam_tv, "lambda")
    require_positive(mu, "mu")
    if max_iters < 1:
        raise ValueError("admm_tv: max_iters must be >= 1")
    require_same_dims(dims_of(y), spec.lr, "admm_tv")
    require_same_dims(dims_of(psf), spec.hr, "admm_tv: psf")
    t0 = time.perf_counter()
    hr = spec.hr
    tau = 1e-8 * mu if tau is None else tau
    lam = psf_to_spectrum(psf)
    folded = FoldedSpectrum(lam, spec)
    gamma = make_gamma(hr, tau)
    denom = tv_denominator(folded, spec, mu, gamma)
    data_hat = fft3(decimate_adjoint(y, spec)) * np.conj(lam)

    if init == INIT_ZERO:
        x = np.zeros(shape_of(hr))
    elif init == INIT_UPSAMPLED:
        x = nn_upsample(y, spec)
    else:
        require_same_dims(dims_of(init_volume), hr, "admm_tv: init volume")
        x = np.array(init_volume, dtype=np.float64, copy=True)
    u = [diff_forward(x, a) for a in range(3)]
    dual = [np.zeros(shape_of(hr)) for _ in range(3)]
    report = SolveReport()
    report.initial_objective = objective_tv(x, y, lam, spec, lam_tv)
    for it in range(1, max_iters + 1):
        x_prev = x
        theta = np.zeros(shape_of(hr))
        for a in range(3):
            theta = theta + diff_adjoint(u[a] - dual[a], a)
        k_hat = data_hat + mu * fft3(theta)
        x, _ = _tv_x_core(k_hat, folded, spec, mu, gamma, denom)
        lx = [diff_forward(x, a) for a in range(3)]
        nu = [lx[a] + dual[a] for a in range(3)]
        u = list(tv_shrink(nu[0], nu[1], nu[2], lam_tv / mu))
        residual = 0.0
        for a in range(3):
            dual[a] = nu[a] - u[a]
            r = lx[a] - u[a]
            residual += float(np.sum(r * r))
        z = decimate(blur_apply(x, lam), spec)
        fit = float(np.sum((y - z) * (y - z)))
        tv = float(np.sum(np.sqrt(lx[0] * lx[0] + lx[1] * lx[1] + lx[2] * lx[2])))
        report.objective.append(0.5 * fit + lam_tv * tv)
        report.primal_residual.append(math.sqrt(residual))
        report.iterations = it
        if rel_tol > 0.0 and rel_change(x, x_prev) < rel_tol:
            break
    require_finite(x, "admm_tv")
    report.seconds = time.perf_counter() - t0
    if return_state:
        return x, report, {"u": u, "dual": dual}
    return x, report


def admm_l2l2(y, lam, spec, reg, xbar, max_iters, mu=0.1, rel_tol=1e-10, warm_start=None):
    """reference src/solvers.cpp:95-189 (iterative l2-l2 comparator)."""
    require_positive(reg, "lambda")
    require_positive(mu, "mu")
    require_same_dims(dims_of(y), spec.lr, "admm_l2l2")
    require_same_dims(dims_of(xbar), spec.hr, "admm_l2l2: xbar")
    if max_iters < 1:
        raise ValueError("admm_l2l2: max_iters must be >= 1")
    t0 = time.perf_counter()
    hr = spec.hr
    xbar_hat = fft3(xbar)
    denom = mu * (lam.real * lam.real + lam.imag * lam.imag) + 2.0 * reg
    if warm_start is not None:
        x, v, dual = (np.array(a, dtype=np.float64) for a in warm_start)
    else:
        x, v, dual = (np.zeros(shape_of(hr)) for _ in range(3))

    def objective(xx):
        z = decimate(ifft3_real(fft3(xx) * lam), spec)
        return 0.5 * float(np.sum((y - z) ** 2)) + reg * float(np.sum((xx - xbar) ** 2))

    report = SolveReport()
    report.initial_objective = objective(x)
    dr, dc, ds = spec.rates
    for it in range(1, max_iters + 1):
        x_prev = x
        t_hat = fft3(v - dual)
        x_hat = (mu * np.conj(lam) * t_hat + 2.0 * reg * xbar_hat) / denom
        x = ifft3_real(x_hat)
        hx = ifft3_real(lam * x_hat)
        work = hx + dual
        v = work.copy()
        v[::ds, ::dc, ::dr] = (y + mu * work[::ds, ::dc, ::dr]) / (1.0 + mu)
        r = hx - v
        dual = dual + r
        z = decimate(hx, spec)
        report.objective.append(0.5 * float(np.sum((y - z) ** 2)) +
                                reg * float(np.sum((x - xbar) ** 2)))
        report.primal_residual.append(math.sqrt(float(np.sum(r * r))))
        report.iterations = it
        if rel_tol > 0.0 and rel_change(x, x_prev) < rel_tol:
            break
    require_finite(x, "admm_l2l2")
    report.seconds = time.perf_counter() - t0
    return x, report


# --------------------------------------------------------------------------
# Dense oracles (reference src/dense.cpp, src/solvers.cpp:74-93,261-284)
# --------------------------------------------------------------------------
DENSE_MAX_VOXELS = 4096


def _require_dense(n, where):
    if n > DENSE_MAX_VOXELS:
        raise ValueError(f"{where}: dense size guard exceeded ({n} > {DENSE_MAX_VOXELS} voxels)")


def build_dense_decimation(spec):
    """reference src/dense.cpp:14-30."""
    _require_dense(int(np.prod(spec.hr)), "build_dense_decimation")
    nl, nh = int(np.prod(spec.lr)), int(np.prod(spec.hr))
    idx = np.arange(nh).reshape(shape_of(spec.hr))
    dr, dc, ds = spec.rates
    cols = idx[::ds, ::dc, ::dr].reshape(-1)
    D = np.zeros((nl, nh))
    D[np.arange(nl), cols] = 1.0
    return D


def build_dense_blur(psf):
    """reference src/dense.cpp:32-55: column q = PSF cyclically shifted to q."""
    m, n, s = dims_of(psf)
    N = m * n * s
    _require_dense(N, "build_dense_blur")
    H = np.zeros((N, N))
    for q in range(N):
        kq, rem = divmod(q, m * n)
        jq, iq = divmod(rem, m)
        H[:, q] = np.roll(np.roll(np.roll(psf, kq, 0), jq, 1), iq, 2).reshape(-1)
    return H


def build_dense_dft(dims):
    """reference src/dense.cpp:57-79 (unitary, sign -1)."""
    m, n, s = dims
    N = m * n * s
    _require_dense(N, "build_dense_dft")
    k, j, i = np.meshgrid(np.arange(s), np.arange(n), np.arange(m), indexing="ij")
    i, j, k = i.reshape(-1), j.reshape(-1), k.reshape(-1)
    ang = 2 * np.pi * (np.outer(i, i) / m + np.outer(j, j) / n + np.outer(k, k) / s)
    return (np.cos(ang) - 1j * np.sin(ang)) / math.sqrt(N)


def build_dense_diff(dims, axis):
    """reference src/dense.cpp:81-98."""
    N = int(np.prod(dims))
    _require_dense(N, "build_dense_diff")
    I = np.eye(N)
    out = np.zeros((N, N))
    for p in range(N):
        e = I[p].reshape(shape_of(dims))
        out[:, p] = diff_forward(e, axis).reshape(-1)
    return out


def dense_tikhonov(y, psf, spec, reg, xbar):
    """reference src/solvers.cpp:74-93."""
    require_positive(reg, "lambda")
    H = build_dense_blur(psf)
    D = build_dense_decimation(spec)
    DH = D @ H
    N = H.shape[0]
    A = DH.T @ DH + 2.0 * reg * np.eye(N)
    rhs = DH.T @ y.reshape(-1) + 2.0 * reg * xbar.reshape(-1)
    L = np.linalg.cholesky(A)
    return np.linalg.solve(L.T, np.linalg.solve(L, rhs)).reshape(shape_of(spec.hr))


def dense_tv_x_update(y, psf, spec, mu, theta, tau):
    """reference src/solvers.cpp:261-284."""
    require_positive(mu, "mu")
    H = build_dense_blur(psf)
    D = build_dense_decimation(spec)
    DH = D @ H
    N = H.shape[0]
    LtL = np.zeros((N, N))
    for a in range(3):
        L = build_dense_diff(spec.hr, a)
        LtL += L.T @ L
    A = DH.T @ DH + mu * LtL + mu * tau * np.eye(N)
    rhs = DH.T @ y.reshape(-1) + mu * theta.reshape(-1)
    L = np.linalg.cholesky(A)
    return np.linalg.solve(L.T, np.linalg.solve(L, rhs)).reshape(shape_of(spec.hr))


def mse(ref, x):
    """reference src/metrics.cpp:9-17."""
    return float(np.mean((ref - x) ** 2))


def psnr(ref, x, peak=None):
    """reference src/metrics.cpp:19-26."""
    e = mse(ref, x)
    pk = float(np.max(ref)) if peak is None else peak
    if e == 0.0:
        return math.inf
    return 10.0 * math.log10(pk * pk / e)


# ---------------------------------------------------------------- input synthesis
class _MT19937_64:
    """std::mt19937_64 (the reference's noise generator, sim.cpp:88-104);
    pure Python, for the small oracle cases only."""

    def __init__(self, seed):
        self.mt = [0] * 312
        self.mt[0] = seed & 0xFFFFFFFFFFFFFFFF
        for i in range(1, 312):
            self.mt[i] = (6364136223846793005 * (self.mt[i - 1] ^ (self.mt[i - 1] >> 62)) + i) & 0xFFFFFFFFFFFFFFFF
        self.i = 312

    def __call__(self):
        if self.i >= 312:
            mt, um, lm = self.mt, 0xFFFFFFFF80000000, 0x7FFFFFFF
            for k in range(312):
                x = (mt[k] & um) | (mt[(k + 1) % 312] & lm)
                xa = x >> 1
                if x & 1:
                    xa ^= 0xB5026F5AA96619E9
                mt[k] = mt[(k + 156) % 312] ^ xa
            self.i = 0
        y = self.mt[self.i]
        self.i += 1
        y ^= (y >> 29) & 0x5555555555555555
        y ^= (y << 17) & 0x71D67FFFEDA60000
        y ^= (y << 37) & 0xFFF7EEE000000000
        y ^= y >> 43
        return y & 0xFFFFFFFFFFFFFFFF


def gaussian_noise(dims, seed):
    """reference src/sim.cpp:88-104 (mt19937_64 + Box-Muller, (r >> 11 + 1) 2^-53)."""
    import math
    m, n, s = dims
    N = m * n * s
    rng = _MT19937_64(seed)
    out = np.empty(N)
    for p in range(0, N, 2):
        u1 = ((rng() >> 11) + 1.0) * 2.0 ** -53
        u2 = ((rng() >> 11) + 1.0) * 2.0 ** -53
        r = math.sqrt(-2.0 * math.log(u1))
        out[p] = r * math.cos(2.0 * math.pi * u2)
        if p + 1 < N:
            out[p + 1] = r * math.sin(2.0 * math.pi * u2)
    return out.reshape(s, n, m)


def degrade(x, psf, spec, bsnr_db=None, seed=0):
    """reference src/sim.cpp:106-127: y = D H x (+ noise at bsnr_db); returns (y, sigma)."""
    y = decimate(blur_apply(x, psf_to_spectrum(psf)), spec)
    sigma = 0.0
    if bsnr_db is not None:
        mean = float(np.sum(y)) / y.size
        var = float(np.sum((y - mean) ** 2)) / y.size
        sigma = float(np.sqrt(var / 10.0 ** (bsnr_db / 10.0)))
        y = y + sigma * gaussian_noise(spec.lr, seed)
    require_finite(y, "degrade")
    return y, sigma
