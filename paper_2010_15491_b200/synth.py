"""Seeded synthetic inputs for the five BASELINE configurations (host side).

The reference's benchmark volumes (paper's uCT/CBCT teeth) are proprietary and
absent; BASELINE.json's configs are fully synthetic and restated here
(SURVEY.md §8(d)).  Input preparation is OUT of the timed hot path; it uses
numpy (pocketfft for the blur, seeded PCG64 for every random draw):

  phantom  : sum of 20 random ellipsoids, centres uniform in the volume,
             semi-axes uniform in 5-30% of the edge per axis, intensities
             uniform in [0.1, 1], overlaps add;
  texture  : uniform [0,1) noise -> circular Gaussian smoothing (sigma 3,
             separable support 25) -> min-max to [0,1] -> x 0.1, added;
  PSF      : reference make_gaussian_psf (operators.cpp:64-119) restated;
  noise    : reference BSNR convention (sim.cpp:106-127): sigma^2 =
             var(mean-removed D H x) / 10^(bsnr/10), Gaussian draws.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Optional, Sequence, Tuple

import numpy as np


def shape_of(dims) -> tuple:
    m, n, s = dims
    return (s, n, m)


def _sample_gaussian_1d(size: int, sigma: float) -> np.ndarray:
    half = size // 2
    t = np.arange(-half, half + 1, dtype=np.float64)
    if sigma <= 0.0:
        return (t == 0).astype(np.float64)
    return np.exp(-0.5 * (t / sigma) * (t / sigma))


def make_gaussian_psf(size, sigma, hr_dims, weights=None) -> np.ndarray:
    """Padded, normalised, origin-wrapped PSF (reference operators.cpp:64-119,
    explicit weights normalised as PsfSpec::explicit_kernel :30-44)."""
    for a in range(3):
        if size[a] % 2 == 0:
            raise ValueError(f"make_gaussian_psf: kernel size must be odd on axis {a + 1}")
    for a in range(3):
        if size[a] > hr_dims[a]:
            raise ValueError(f"make_gaussian_psf: kernel size {size[a]} exceeds volume axis "
                             f"{a + 1} of length {hr_dims[a]}")
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
        wr, wc, ws = (_sample_gaussian_1d(size[a], sigma[a]) for a in range(3))
        kernel = (wr[None, None, :] * wc[None, :, None]) * ws[:, None, None]
        tot = 0.0
        for x in kernel.reshape(-1):  # sequential, as the reference (:86-93)
            tot += x
        kernel = kernel / tot
    psf = np.zeros(shape_of(hr_dims))
    m, n, s = hr_dims
    ii = (np.arange(kr) - kr // 2) % m
    jj = (np.arange(kc) - kc // 2) % n
    kk = (np.arange(ks) - ks // 2) % s
    for c in range(ks):
        for b in range(kc):
            np.add.at(psf[kk[c], jj[b]], ii, kernel[c, b])
    return psf


def ellipsoid_phantom(dims, seed: int, count: int = 20) -> np.ndarray:
    rng = np.random.default_rng(seed)
    m, n, s = dims
    vol = np.zeros(shape_of(dims))
    ext = np.array([m, n, s], dtype=np.float64)
    for _ in range(count):
        c = rng.uniform(0.0, 1.0, 3) * ext
        ax = rng.uniform(0.05, 0.30, 3) * ext
        val = rng.uniform(0.1, 1.0)
        lo = np.maximum(np.floor(c - ax).astype(int), 0)
        hi = np.minimum(np.ceil(c + ax).astype(int) + 1, [m, n, s])
        if np.any(hi <= lo):
            continue
        i = (np.arange(lo[0], hi[0]) + 0.5 - c[0]) / ax[0]
        j = (np.arange(lo[1], hi[1]) + 0.5 - c[1]) / ax[1]
        k = (np.arange(lo[2], hi[2]) + 0.5 - c[2]) / ax[2]
        r2 = (k * k)[:, None, None] + (j * j)[None, :, None] + (i * i)[None, None, :]
        vol[lo[2]:hi[2], lo[1]:hi[1], lo[0]:hi[0]] += np.where(r2 <= 1.0, val, 0.0)
    return vol


def _circular_smooth(v: np.ndarray, sigma: float, support: int) -> np.ndarray:
    w = _sample_gaussian_1d(support, sigma)
    w = w / w.sum()
    out = v
    for ax in range(3):
        L = out.shape[ax]
        k = np.zeros(L)
        for t, wt in zip(range(-(support // 2), support // 2 + 1), w):
            k[t % L] += wt
        K = np.fft.rfft(k)
        out = np.fft.irfft(np.fft.rfft(out, axis=ax) * K.reshape([-1 if a == ax else 1 for a in range(3)]),
                           n=L, axis=ax)
    return out


def texture(dims, seed: int, sigma: float = 3.0, amplitude: float = 0.1) -> np.ndarray:
    rng = np.random.default_rng(seed)
    noise = rng.uniform(0.0, 1.0, shape_of(dims))
    sm = _circular_smooth(noise, sigma, int(round(4 * sigma)) * 2 + 1)
    lo, hi = sm.min(), sm.max()
    sm = (sm - lo) / (hi - lo if hi > lo else 1.0)
    return amplitude * sm


def decimate(x: np.ndarray, rates) -> np.ndarray:
    dr, dc, ds = rates
    return np.ascontiguousarray(x[::ds, ::dc, ::dr])


def degrade(x: np.ndarray, psf: np.ndarray, rates, bsnr_db: Optional[float], seed: int):
    """y = D H x + n (reference sim.cpp:106-127 conventions, numpy host side)."""
    lam = np.fft.rfftn(psf)
    hx = np.fft.irfftn(np.fft.rfftn(x) * lam, s=x.shape, axes=(0, 1, 2))
    y = decimate(hx, rates)
    sigma = 0.0
    if bsnr_db is not None:
        mean = y.mean()
        var = float(np.mean((y - mean) ** 2))
        sigma = math.sqrt(var / 10.0 ** (bsnr_db / 10.0))
        y = y + sigma * np.random.default_rng(seed).standard_normal(y.shape)
    return np.ascontiguousarray(y), sigma


def zero_fill_upsample(y: np.ndarray, rates) -> np.ndarray:
    """d * D^H y (reference operators.cpp:166-171) — the CLI's default x̄."""
    dr, dc, ds = rates
    s, n, m = y.shape
    x = np.zeros((s * ds, n * dc, m * dr))
    x[::ds, ::dc, ::dr] = y * float(dr * dc * ds)
    return x


def spectral_upsample(y: np.ndarray, rates) -> np.ndarray:
    """Zero-padded spectral upsampling of y (config 2's x0): the LR spectrum
    placed at the HR low frequencies, scaled by d to keep intensities."""
    dr, dc, ds = rates
    Y = np.fft.fftn(y)
    S, Nn, M = y.shape
    H = (S * ds, Nn * dc, M * dr)
    X = np.zeros(H, np.complex128)

    def split(l, Lh):
        pos = np.arange(0, (l + 1) // 2)
        neg = np.arange(l - l // 2, l)
        return np.concatenate([pos, neg]), np.concatenate([pos, neg - l + Lh])

    (ks, kS), (kn, kN), (km, kM) = split(S, H[0]), split(Nn, H[1]), split(M, H[2])
    X[np.ix_(kS, kN, kM)] = Y[np.ix_(ks, kn, km)]
    return np.ascontiguousarray(np.real(np.fft.ifftn(X)) * float(dr * dc * ds))


@dataclass
class Config:
    idx: int
    hr: Tuple[int, int, int]
    rates: Tuple[int, int, int]
    psf_size: Tuple[int, int, int]
    psf_sigma: Tuple[float, float, float]
    bsnr: float
    solver: str               # "tikhonov" | "tv" | "tikhonov+tv"
    texture: bool
    seeds: Tuple[int, ...]
    reg: float = 1e-3         # Tikhonov tau (TikhonovConfig::lambda)
    tv_lambda: float = 2e-3
    tv_mu: float = 0.05
    tv_iters: int = 0
    init: str = "zero"        # "zero" | "spectral"

    @property
    def lr(self):
        return tuple(self.hr[a] // self.rates[a] for a in range(3))

    @property
    def d(self):
        return self.rates[0] * self.rates[1] * self.rates[2]

    @property
    def voxels(self):
        return self.hr[0] * self.hr[1] * self.hr[2]

    def name(self):
        return f"config{self.idx}"


CONFIGS = {
    0: Config(0, (64, 64, 64), (2, 2, 2), (9, 9, 9), (1.0, 1.0, 1.0), 40.0, "tikhonov", False, (0, 1)),
    1: Config(1, (256, 256, 256), (2, 2, 2), (13, 13, 13), (1.5, 1.5, 1.5), 30.0, "tikhonov", True,
              (0, 1, 2)),
    2: Config(2, (256, 256, 256), (4, 4, 4), (13, 13, 13), (1.5, 1.5, 1.5), 30.0, "tv", True, (0, 1, 2),
              tv_lambda=2e-3, tv_mu=0.05, tv_iters=100, init="spectral"),
    3: Config(3, (512, 512, 256), (2, 2, 4), (15, 15, 21), (1.2, 1.2, 2.0), 35.0, "tv", True, (3, 4, 5),
              tv_lambda=1e-3, tv_mu=0.05, tv_iters=50),
    4: Config(4, (1024, 1024, 1024), (2, 2, 2), (13, 13, 13), (1.5, 1.5, 1.5), 30.0, "tikhonov+tv", True,
              (6, 7, 8), tv_lambda=2e-3, tv_mu=0.05, tv_iters=20),
}


def scaled(cfg: Config, hr) -> Config:
    """Same recipe at a smaller HR grid (parity cases the oracle finishes in seconds)."""
    psf = tuple(min(cfg.psf_size[a], hr[a] - (1 - hr[a] % 2)) for a in range(3))
    psf = tuple(p if p % 2 == 1 else p - 1 for p in psf)
    return Config(cfg.idx, tuple(hr), cfg.rates, psf, cfg.psf_sigma, cfg.bsnr, cfg.solver,
                  cfg.texture, cfg.seeds, cfg.reg, cfg.tv_lambda, cfg.tv_mu, cfg.tv_iters, cfg.init)


@dataclass
class Inputs:
    cfg: Config
    truth: np.ndarray
    psf: np.ndarray
    y: np.ndarray
    noise_sigma: float
    xbar: Optional[np.ndarray] = None
    x0: Optional[np.ndarray] = None


def make_inputs(cfg: Config, with_truth: bool = True) -> Inputs:
    truth = ellipsoid_phantom(cfg.hr, cfg.seeds[0])
    if cfg.texture:
        truth = truth + texture(cfg.hr, cfg.seeds[1])
    psf = make_gaussian_psf(cfg.psf_size, cfg.psf_sigma, cfg.hr)
    y, sigma = degrade(truth, psf, cfg.rates, cfg.bsnr, cfg.seeds[-1])
    inp = Inputs(cfg, truth if with_truth else None, psf, y, sigma)
    if "tikhonov" in cfg.solver:
        inp.xbar = zero_fill_upsample(y, cfg.rates)
    if cfg.init == "spectral":
        inp.x0 = spectral_upsample(y, cfg.rates)
    return inp
