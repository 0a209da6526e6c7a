"""ctypes binding over oracle/_ref/libvolsr_ref.so — the REFERENCE volsr C++
library compiled from its own sources (oracle/Makefile) — TEST
INFRASTRUCTURE.  Used to generate golden vectors (tools/make_golden.py), to
pin the numpy oracle, and as bench.py's CPU baseline / reference arm."""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

_PATH = Path(__file__).resolve().parent / "_ref" / "libvolsr_ref.so"
_lib = None


def available() -> bool:
    global _lib
    if _lib is not None:
        return True
    if not _PATH.exists():
        return False
    try:
        _lib = C.CDLL(str(_PATH))
    except OSError:
        return False
    _setup()
    return True


_dp = C.POINTER(C.c_double)
_sz = C.POINTER(C.c_size_t)


def _setup():
    L = _lib
    L.ref_last_error.restype = C.c_char_p
    for n in ("ref_fft3", "ref_fft3_real", "ref_ifft3", "ref_psf_to_spectrum"):
        getattr(L, n).argtypes = [_sz, _dp, _dp]
    L.ref_ifft3_real.argtypes = [_sz, _dp, _dp, C.c_double]
    L.ref_make_gaussian_psf.argtypes = [_sz, _dp, _sz, _dp]
    L.ref_tikhonov_create.argtypes = [_sz, _sz, _dp, C.c_double, _dp]
    L.ref_tikhonov_create.restype = C.c_void_p
    L.ref_tikhonov_solve.argtypes = [C.c_void_p, _dp, _dp]
    L.ref_tikhonov_destroy.argtypes = [C.c_void_p]
    L.ref_make_gamma.argtypes = [_sz, C.c_double, _dp]
    L.ref_tv_x_update.argtypes = [_sz, _sz, _dp, _dp, C.c_double, _dp, _dp, _dp]
    L.ref_objective_tv.argtypes = [_sz, _sz, _dp, _dp, _dp, C.c_double, _dp]
    L.ref_admm_tv.argtypes = [_sz, _sz, _dp, _dp, C.c_double, C.c_double, C.c_size_t, C.c_double,
                              C.c_int, C.c_double, C.c_int, _dp, _dp, _dp, _dp, _sz, _dp, _dp]
    L.ref_admm_l2l2.argtypes = [_sz, _sz, _dp, _dp, C.c_double, _dp, C.c_size_t, C.c_double, C.c_double,
                                _dp, _dp, _dp, _sz, _dp]
    L.ref_save_volume.argtypes = [C.c_char_p, _sz, _dp, C.c_int]
    L.ref_degrade.argtypes = [_sz, _sz, _dp, _sz, _dp, C.c_int, C.c_double, C.c_ulonglong, _dp, _dp]
    L.ref_load_volume.argtypes = [C.c_char_p, _sz, _dp, C.c_size_t]
    L.ref_make_phantom.argtypes = [_sz, C.c_int, C.c_ulonglong, _dp]


class RefError(RuntimeError):
    pass


def _chk(rc):
    if rc != 0:
        raise RefError(f"[code {rc}] " + _lib.ref_last_error().decode())


def _d(dims):
    return (C.c_size_t * 3)(*[int(v) for v in dims])


def _p(a):
    return a.ctypes.data_as(_dp)


def _dims(v):
    s, n, m = v.shape
    return (m, n, s)


def fft3(x):
    x = np.ascontiguousarray(x)
    out = np.empty(x.shape, np.complex128)
    if np.iscomplexobj(x):
        _chk(_lib.ref_fft3(_d(_dims(x)), _p(x.view(np.float64)), _p(out.view(np.float64))))
    else:
        x = x.astype(np.float64)
        _chk(_lib.ref_fft3_real(_d(_dims(x)), _p(x), _p(out.view(np.float64))))
    return out


def ifft3_real(xh, tol=1e-8):
    xh = np.ascontiguousarray(xh, dtype=np.complex128)
    out = np.empty(xh.shape)
    _chk(_lib.ref_ifft3_real(_d(_dims(xh)), _p(xh.view(np.float64)), _p(out), float(tol)))
    return out


def psf_to_spectrum(psf):
    psf = np.ascontiguousarray(psf, dtype=np.float64)
    out = np.empty(psf.shape, np.complex128)
    _chk(_lib.ref_psf_to_spectrum(_d(_dims(psf)), _p(psf), _p(out.view(np.float64))))
    return out


def make_gaussian_psf(size, sigma, hr):
    m, n, s = hr
    out = np.empty((s, n, m))
    sig = (C.c_double * 3)(*sigma)
    _chk(_lib.ref_make_gaussian_psf(_d(size), sig, _d(hr), _p(out)))
    return out


def make_gamma(hr, tau):
    m, n, s = hr
    out = np.empty((s, n, m))
    _chk(_lib.ref_make_gamma(_d(hr), float(tau), _p(out)))
    return out


class TikhonovOperator:
    """Reference TikhonovOperator(psf_to_spectrum(psf), spec, {reg, xbar})."""

    def __init__(self, psf_or_lambda, hr, rates, reg, xbar):
        lam = psf_or_lambda if np.iscomplexobj(psf_or_lambda) else psf_to_spectrum(psf_or_lambda)
        lam = np.ascontiguousarray(lam)
        xbar = np.ascontiguousarray(xbar, dtype=np.float64)
        self.hr, self.rates = tuple(hr), tuple(rates)
        self.h = _lib.ref_tikhonov_create(_d(hr), _d(rates), _p(lam.view(np.float64)), float(reg), _p(xbar))
        if not self.h:
            raise RefError(_lib.ref_last_error().decode())

    def solve(self, y):
        y = np.ascontiguousarray(y, dtype=np.float64)
        m, n, s = self.hr
        out = np.empty((s, n, m))
        _chk(_lib.ref_tikhonov_solve(self.h, _p(y), _p(out)))
        return out

    def __del__(self):
        try:
            if self.h:
                _lib.ref_tikhonov_destroy(self.h)
        except Exception:
            pass


def tv_x_update(y, lam, hr, rates, mu, theta_hat, gamma):
    y = np.ascontiguousarray(y, dtype=np.float64)
    lam = np.ascontiguousarray(lam, dtype=np.complex128)
    th = np.ascontiguousarray(theta_hat, dtype=np.complex128)
    g = np.ascontiguousarray(gamma, dtype=np.float64)
    m, n, s = hr
    out = np.empty((s, n, m))
    _chk(_lib.ref_tv_x_update(_d(hr), _d(rates), _p(y), _p(lam.view(np.float64)), float(mu),
                              _p(th.view(np.float64)), _p(g), _p(out)))
    return out


def objective_tv(x, y, lam, hr, rates, w):
    out = C.c_double()
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.ascontiguousarray(y, dtype=np.float64)
    lam = np.ascontiguousarray(lam, dtype=np.complex128)
    _chk(_lib.ref_objective_tv(_d(hr), _d(rates), _p(x), _p(y), _p(lam.view(np.float64)), float(w),
                               C.byref(out)))
    return out.value


def admm_tv(y, psf, hr, rates, lam_tv, mu, max_iters, rel_tol, tau=None, init=0, init_volume=None):
    y = np.ascontiguousarray(y, dtype=np.float64)
    psf = np.ascontiguousarray(psf, dtype=np.float64)
    m, n, s = hr
    x = np.empty((s, n, m))
    obj = np.zeros(max_iters)
    res = np.zeros(max_iters)
    iters = C.c_size_t()
    init_obj = C.c_double()
    secs = C.c_double()
    iv = np.ascontiguousarray(init_volume, dtype=np.float64) if init_volume is not None else None
    _chk(_lib.ref_admm_tv(_d(hr), _d(rates), _p(y), _p(psf), float(lam_tv), float(mu), int(max_iters),
                          float(rel_tol), 0 if tau is None else 1, 0.0 if tau is None else float(tau),
                          int(init), _p(iv) if iv is not None else None, _p(x), _p(obj), _p(res),
                          C.byref(iters), C.byref(init_obj), C.byref(secs)))
    k = iters.value
    return x, {"iterations": k, "initial_objective": init_obj.value, "objective": obj[:k],
               "primal_residual": res[:k], "seconds": secs.value}


def admm_l2l2(y, lam, hr, rates, reg, xbar, max_iters, mu=0.1, rel_tol=1e-10):
    y = np.ascontiguousarray(y, dtype=np.float64)
    lam = np.ascontiguousarray(lam, dtype=np.complex128)
    xbar = np.ascontiguousarray(xbar, dtype=np.float64)
    m, n, s = hr
    x = np.empty((s, n, m))
    obj = np.zeros(max_iters)
    res = np.zeros(max_iters)
    iters = C.c_size_t()
    init_obj = C.c_double()
    _chk(_lib.ref_admm_l2l2(_d(hr), _d(rates), _p(y), _p(lam.view(np.float64)), float(reg), _p(xbar),
                            C.c_size_t(max_iters), float(mu), float(rel_tol), _p(x), _p(obj), _p(res),
                            C.byref(iters), C.byref(init_obj)))
    k = iters.value
    return x, {"iterations": k, "initial_objective": init_obj.value, "objective": obj[:k],
               "primal_residual": res[:k]}


def save_volume(base, v, f32=False):
    """reference volsr::save_volume (volume_io.cpp:34-57)."""
    v = np.ascontiguousarray(v, dtype=np.float64)
    _chk(_lib.ref_save_volume(str(base).encode(), _d(_dims(v)), _p(v), int(bool(f32))))


def load_volume(base, cap=1 << 20):
    """reference volsr::load_volume (volume_io.cpp:61-131); returns (s, n, m) array."""
    d = (C.c_size_t * 3)()
    out = np.empty(cap)
    _chk(_lib.ref_load_volume(str(base).encode(), d, _p(out), cap))
    m, n, s = int(d[0]), int(d[1]), int(d[2])
    return out[:m * n * s].reshape(s, n, m).copy()


def degrade(x, psf_size, psf_sigma, rates, bsnr_db, seed):
    """reference volsr::degrade (sim.cpp:106-127) with a Gaussian PsfSpec; returns (y, sigma)."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    m, n, s = _dims(x)
    y = np.empty((s // rates[2], n // rates[1], m // rates[0]))
    sig = C.c_double()
    _chk(_lib.ref_degrade(_d((m, n, s)), _d(rates), _p(x), _d(psf_size), (C.c_double * 3)(*psf_sigma),
                          int(bsnr_db is not None), float(bsnr_db or 0.0), int(seed), _p(y), C.byref(sig)))
    return y, sig.value


def make_phantom(hr, kind=0, seed=0):
    """Reference make_phantom (sim.cpp:23-73); kind 0 NestedEllipsoids, 1 RandomSmooth, 2 Constant."""
    out = np.empty((hr[2], hr[1], hr[0]))
    _chk(_lib.ref_make_phantom(_d(hr), kind, seed, _p(out)))
    return out
