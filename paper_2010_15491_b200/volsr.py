"""Python mirror of the reference `volsr` solver API over the C ABI (include/vsr.h).

Names, argument meaning and error behaviour follow the reference C++ API
(/root/reference/proj/include/volsr/*.hpp) so the parity tests read like the
reference's own tests:

  reference                                   here
  ------------------------------------------  ----------------------------------
  TikhonovOperator(lambda, spec, cfg).solve   TikhonovOperator(lam, spec, cfg).solve
  tikhonov_fast(y, lambda, spec, cfg)         tikhonov_fast(y, lam, spec, cfg)
  tv_x_update(y, folded, lambda, spec, ...)   tv_x_update(y, folded, lam, spec, mu, theta_hat, gamma)
  tv_shrink / make_gamma / objective_tv       same names
  admm_tv(y, psf, spec, TvAdmmConfig)         admm_tv(y, psf, spec, cfg) -> (x, SolveReport)
  fft3 / ifft3 / ifft3_real / dft3_unnorm.    same names (GPU engine)
  FoldedSpectrum / alias_fold / gram_diag     same names
  shape_error / numeric_error                 ShapeError / NumericError

Volumes are numpy arrays of shape (s, n, m) in C order (axis 1 = m fastest,
reference include/volsr/volume.hpp:26-45); spectra are complex128.  Every
numeric step runs in libvsr_b200.so on the GPU; there is no CPU fallback and
importing this module without the built library raises.
"""
from __future__ import annotations

import ctypes as C
import math
import os
from dataclasses import dataclass, field
from pathlib import Path
from typing import Optional, Sequence

import numpy as np

_LIB_PATH = Path(__file__).resolve().parent / "_lib" / "libvsr_b200.so"

VSR_OK, VSR_ERR_SHAPE, VSR_ERR_INVALID, VSR_ERR_NUMERIC, VSR_ERR_OUT_OF_RANGE, VSR_ERR_CUDA = range(6)
VSR_ERR_IO = 7
VSR_DTYPE_F64, VSR_DTYPE_F32 = 0, 1
INIT_ZERO, INIT_UPSAMPLED, INIT_PROVIDED = 0, 1, 2


class ShapeError(ValueError):
    """volsr::shape_error (derives std::invalid_argument), volume.hpp:12-15."""


class NumericError(RuntimeError):
    """volsr::numeric_error, volume.hpp:18-20."""


class DeviceError(RuntimeError):
    """CUDA/runtime failure inside the library."""


class VolumeIOError(OSError):
    """volsr::io_error (volume files), volume.hpp:22-24."""


def load_library() -> C.CDLL:
    if not _LIB_PATH.exists():
        raise ImportError(
            f"volsr B200 library not built: {_LIB_PATH} is missing "
            "(run `python -c 'import __graft_entry__ as g; g.build()'`)")
    return C.CDLL(str(_LIB_PATH))


_lib = load_library()
_dp = C.POINTER(C.c_double)
_szp = C.POINTER(C.c_size_t)
_vp = C.c_void_p


class _TvConfig(C.Structure):
    _fields_ = [("lambda_", C.c_double), ("mu", C.c_double), ("max_iters", C.c_size_t),
                ("rel_tol", C.c_double), ("has_tau", C.c_int), ("tau", C.c_double),
                ("init", C.c_int), ("init_volume", _dp), ("precision", C.c_int)]


class _Report(C.Structure):
    _fields_ = [("iterations", C.c_size_t), ("initial_objective", C.c_double),
                ("seconds", C.c_double), ("objective", _dp), ("primal_residual", _dp)]


def _sig(name, args, res=C.c_int):
    f = getattr(_lib, name)
    f.argtypes = args
    f.restype = res
    return f


_sig("vsr_last_error_message", [], C.c_char_p)
_sig("vsr_ctx_create", [C.c_int, C.POINTER(_vp)])
_sig("vsr_ctx_destroy", [_vp])
_sig("vsr_ctx_synchronize", [_vp])
_sig("vsr_ctx_stream", [_vp], _vp)
_sig("vsr_host_alloc", [C.c_size_t, C.POINTER(_vp)])
_sig("vsr_host_free", [_vp])
_sig("vsr_device_alloc", [_vp, C.c_size_t, C.POINTER(_vp)])
_sig("vsr_device_free", [_vp, _vp])
_sig("vsr_memcpy_h2d", [_vp, _vp, _vp, C.c_size_t])
_sig("vsr_memcpy_d2h", [_vp, _vp, _vp, C.c_size_t])
for _n in ("vsr_fft3", "vsr_fft3_real", "vsr_ifft3", "vsr_dft3_unnormalized", "vsr_psf_to_spectrum"):
    _sig(_n, [_vp, _szp, _dp, _dp])
_sig("vsr_ifft3_real", [_vp, _szp, _dp, _dp, C.c_double])
_sig("vsr_fft_counters", [C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)])
_sig("vsr_reset_fft_counters", [])
_sig("vsr_decimate", [_vp, _szp, _szp, _dp, _dp])
_sig("vsr_decimate_adjoint", [_vp, _szp, _szp, _dp, _dp])
_sig("vsr_diff_forward", [_vp, _szp, C.c_int, _dp, _dp])
_sig("vsr_diff_adjoint", [_vp, _szp, C.c_int, _dp, _dp])
_sig("vsr_blur_apply", [_vp, _szp, _dp, _dp, C.c_int, _dp])
_sig("vsr_alias_fold", [_vp, _szp, _szp, _dp, _dp])
_sig("vsr_alias_expand", [_vp, _szp, _szp, _dp, _dp])
_sig("vsr_folded_create", [_vp, _szp, _szp, _dp, C.POINTER(_vp)])
_sig("vsr_folded_destroy", [_vp])
_sig("vsr_folded_block_value", [_vp, C.c_size_t, C.c_size_t, C.c_size_t, C.c_size_t, _dp])
_sig("vsr_folded_apply", [_vp, _dp, _dp])
_sig("vsr_folded_apply_adjoint", [_vp, _dp, _dp])
_sig("vsr_folded_apply_weighted", [_vp, _dp, _dp, _dp])
_sig("vsr_folded_apply_adjoint_weighted", [_vp, _dp, _dp, _dp])
_sig("vsr_folded_gram_diag", [_vp, _dp])
_sig("vsr_folded_gram_diag_weighted", [_vp, _dp, _dp])
_sig("vsr_folded_swap_blocks_for_fault_injection", [_vp])
_sig("vsr_tikhonov_create", [_vp, _szp, _szp, _dp, C.c_double, _dp, C.POINTER(_vp)])
_sig("vsr_tikhonov_create_d", [_vp, _szp, _szp, _vp, C.c_double, _vp, C.POINTER(_vp)])
_sig("vsr_tikhonov_destroy", [_vp])
_sig("vsr_tikhonov_solve", [_vp, _dp, _dp])
_sig("vsr_tikhonov_solve_d", [_vp, _vp, _vp])
_sig("vsr_tikhonov_solve_f32", [_vp, _vp, _vp])
_sig("vsr_tikhonov_solve_f32_d", [_vp, _vp, _vp])
_sig("vsr_tikhonov_fp32_ok", [_vp])
_sig("vsr_tv_x_f32_d", [_vp, C.POINTER(C.c_void_p)])
_sig("vsr_tikhonov_check", [_vp])
_sig("vsr_tikhonov_algorithmic_bytes", [_szp, _szp], C.c_double)
_sig("vsr_make_gamma", [_vp, _szp, C.c_double, _dp])
_sig("vsr_tv_x_update", [_vp, _szp, _szp, _dp, _dp, C.c_double, _dp, _dp, _dp])
_sig("vsr_tv_shrink", [_vp, C.c_size_t, _dp, _dp, _dp, C.c_double, _dp, _dp, _dp])
_sig("vsr_objective_tv", [_vp, _szp, _szp, _dp, _dp, _dp, C.c_double, _dp])
_sig("vsr_admm_tv", [_vp, _szp, _szp, _dp, _dp, C.POINTER(_TvConfig), _dp, C.POINTER(_Report)])
_sig("vsr_tv_create_d", [_vp, _szp, _szp, _vp, _vp, C.POINTER(_TvConfig), C.POINTER(_vp)])
_sig("vsr_tv_iterate_d", [_vp, C.c_size_t])
_sig("vsr_tv_x_d", [_vp, C.POINTER(_vp)])
_sig("vsr_tv_report", [_vp, C.POINTER(_Report)])
_sig("vsr_tv_destroy", [_vp])
_sig("vsr_tv_algorithmic_bytes", [_szp, _szp], C.c_double)


def check(rc: int):
    if rc == VSR_OK:
        return
    msg = _lib.vsr_last_error_message().decode(errors="replace")
    if rc == VSR_ERR_SHAPE:
        raise ShapeError(msg)
    if rc == VSR_ERR_INVALID:
        raise ValueError(msg)
    if rc == VSR_ERR_NUMERIC:
        raise NumericError(msg)
    if rc == VSR_ERR_OUT_OF_RANGE:
        raise IndexError(msg)
    if rc == VSR_ERR_IO:
        raise VolumeIOError(msg)
    raise DeviceError(msg)


# ---------------------------------------------------------------- context
class Context:
    """One device + one stream (vsr_ctx)."""

    def __init__(self, device: int = 0):
        h = _vp()
        check(_lib.vsr_ctx_create(int(device), C.byref(h)))
        self.handle = h
        self.device = int(device)

    def stream(self) -> int:
        return int(_lib.vsr_ctx_stream(self.handle) or 0)

    def synchronize(self):
        check(_lib.vsr_ctx_synchronize(self.handle))

    def close(self):
        if self.handle:
            _lib.vsr_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_default_ctx: Optional[Context] = None


def default_context() -> Context:
    global _default_ctx
    if _default_ctx is None:
        _default_ctx = Context(int(os.environ.get("VSR_DEVICE", "0")))
    return _default_ctx


def _ctx(ctx):
    return (ctx or default_context()).handle


# ---------------------------------------------------------------- helpers
def dims_of(v: np.ndarray) -> tuple:
    s, n, m = v.shape
    return (m, n, s)


def shape_of(dims) -> tuple:
    m, n, s = dims
    return (s, n, m)


def _dims_arr(dims):
    return (C.c_size_t * 3)(*[int(x) for x in dims])


def _real(v) -> np.ndarray:
    a = np.ascontiguousarray(v, dtype=np.float64)
    if a.ndim != 3:
        raise ShapeError(f"expected a 3D volume, got shape {a.shape}")
    return a


def _cplx(v) -> np.ndarray:
    a = np.ascontiguousarray(v, dtype=np.complex128)
    if a.ndim != 3:
        raise ShapeError(f"expected a 3D spectrum, got shape {a.shape}")
    return a


def _p(a: np.ndarray):
    return a.ctypes.data_as(_dp)


def require_same_dims(a, b, where):
    """reference src/volume.cpp:25-29."""
    if tuple(a) != tuple(b):
        raise ShapeError(f"{where}: dims mismatch, {a[0]}x{a[1]}x{a[2]} vs {b[0]}x{b[1]}x{b[2]}")


def require_positive(v, name):
    if not (v > 0.0):
        raise ValueError(f"{name} must be positive, got {v:f}")


# ---------------------------------------------------------------- spec
class DecimationSpec:
    """reference include/volsr/operators.hpp:12-27 (validated on the host)."""

    def __init__(self, hr_dims: Sequence[int], rates: Sequence[int]):
        names = ("1 (rows)", "2 (cols)", "3 (slices)")
        for a in range(3):
            if rates[a] == 0:
                raise ShapeError(f"DecimationSpec: zero rate on axis {names[a]}")
            if hr_dims[a] % rates[a] != 0:
                raise ShapeError(f"DecimationSpec: rate {rates[a]} does not divide axis {names[a]} "
                                 f"of length {hr_dims[a]}")
        self.hr = tuple(int(x) for x in hr_dims)
        self.rates = tuple(int(r) for r in rates)
        self.lr = tuple(self.hr[a] // self.rates[a] for a in range(3))

    def rate(self) -> int:
        return self.rates[0] * self.rates[1] * self.rates[2]

    def dr(self):
        return self.rates[0]

    def dc(self):
        return self.rates[1]

    def ds(self):
        return self.rates[2]


# ---------------------------------------------------------------- FFT contract
def fft3(v: np.ndarray, ctx=None) -> np.ndarray:
    """Unitary forward 3D FFT (fft.hpp:12-14).  Real or complex input."""
    if np.iscomplexobj(v):
        a = _cplx(v)
        out = np.empty_like(a)
        check(_lib.vsr_fft3(_ctx(ctx), _dims_arr(dims_of(a)), _p(a.view(np.float64)),
                            _p(out.view(np.float64))))
        return out
    a = _real(v)
    out = np.empty(a.shape, np.complex128)
    check(_lib.vsr_fft3_real(_ctx(ctx), _dims_arr(dims_of(a)), _p(a), _p(out.view(np.float64))))
    return out


def ifft3(v: np.ndarray, ctx=None) -> np.ndarray:
    a = _cplx(v)
    out = np.empty_like(a)
    check(_lib.vsr_ifft3(_ctx(ctx), _dims_arr(dims_of(a)), _p(a.view(np.float64)),
                         _p(out.view(np.float64))))
    return out


def ifft3_real(v: np.ndarray, max_rel_imag: float = 1e-8, ctx=None) -> np.ndarray:
    """fft.hpp:19-23: residue check then real part."""
    a = _cplx(v)
    out = np.empty(a.shape, np.float64)
    check(_lib.vsr_ifft3_real(_ctx(ctx), _dims_arr(dims_of(a)), _p(a.view(np.float64)), _p(out),
                              float(max_rel_imag)))
    return out


def dft3_unnormalized(v: np.ndarray, ctx=None) -> np.ndarray:
    a = _real(v)
    out = np.empty(a.shape, np.complex128)
    check(_lib.vsr_dft3_unnormalized(_ctx(ctx), _dims_arr(dims_of(a)), _p(a),
                                     _p(out.view(np.float64))))
    return out


def fft_counters() -> dict:
    f, i = C.c_uint64(), C.c_uint64()
    check(_lib.vsr_fft_counters(C.byref(f), C.byref(i)))
    return {"forward": f.value, "inverse": i.value}


def reset_fft_counters():
    check(_lib.vsr_reset_fft_counters())


# ---------------------------------------------------------------- operators
def make_gaussian_psf(size, sigma, hr_dims, weights=None) -> np.ndarray:
    """Host-side PSF construction (operators.cpp:64-119; setup, out of the hot path)."""
    from .synth import make_gaussian_psf as _mk
    return _mk(size, sigma, hr_dims, weights)


def psf_to_spectrum(psf: np.ndarray, ctx=None) -> np.ndarray:
    """operators.cpp:121-123 on the GPU engine."""
    return dft3_unnormalized(psf, ctx)


def blur_apply(x, lam, conjugate=False, ctx=None):
    a = _real(x)
    L = _cplx(lam)
    require_same_dims(dims_of(a), dims_of(L), "blur_apply")
    out = np.empty_like(a)
    check(_lib.vsr_blur_apply(_ctx(ctx), _dims_arr(dims_of(a)), _p(a), _p(L.view(np.float64)),
                              int(bool(conjugate)), _p(out)))
    return out


def decimate(x, spec: DecimationSpec, ctx=None):
    a = _real(x)
    require_same_dims(dims_of(a), spec.hr, "decimate")
    out = np.empty(shape_of(spec.lr))
    check(_lib.vsr_decimate(_ctx(ctx), _dims_arr(spec.hr), _dims_arr(spec.rates), _p(a), _p(out)))
    return out


def decimate_adjoint(y, spec: DecimationSpec, ctx=None):
    a = _real(y)
    require_same_dims(dims_of(a), spec.lr, "decimate_adjoint")
    out = np.empty(shape_of(spec.hr))
    check(_lib.vsr_decimate_adjoint(_ctx(ctx), _dims_arr(spec.hr), _dims_arr(spec.rates), _p(a),
                                    _p(out)))
    return out


def zero_fill_upsample(y, spec, ctx=None):
    return decimate_adjoint(y, spec, ctx) * float(spec.rate())


def diff_forward(x, axis: int, ctx=None):
    a = _real(x)
    out = np.empty_like(a)
    check(_lib.vsr_diff_forward(_ctx(ctx), _dims_arr(dims_of(a)), int(axis), _p(a), _p(out)))
    return out


def diff_adjoint(x, axis: int, ctx=None):
    a = _real(x)
    out = np.empty_like(a)
    check(_lib.vsr_diff_adjoint(_ctx(ctx), _dims_arr(dims_of(a)), int(axis), _p(a), _p(out)))
    return out


# ---------------------------------------------------------------- spectral fold
def alias_fold(hr_spectrum, spec, ctx=None):
    a = _cplx(hr_spectrum)
    require_same_dims(dims_of(a), spec.hr, "alias_fold")
    out = np.empty(shape_of(spec.lr), np.complex128)
    check(_lib.vsr_alias_fold(_ctx(ctx), _dims_arr(spec.hr), _dims_arr(spec.rates),
                              _p(a.view(np.float64)), _p(out.view(np.float64))))
    return out


def alias_expand(lr_spectrum, spec, ctx=None):
    a = _cplx(lr_spectrum)
    require_same_dims(dims_of(a), spec.lr, "alias_expand")
    out = np.empty(shape_of(spec.hr), np.complex128)
    check(_lib.vsr_alias_expand(_ctx(ctx), _dims_arr(spec.hr), _dims_arr(spec.rates),
                                _p(a.view(np.float64)), _p(out.view(np.float64))))
    return out


class FoldedSpectrum:
    """spectral.hpp:21-63 — Lambda held on the device in natural HR layout."""

    def __init__(self, lam, spec: DecimationSpec, ctx=None):
        L = _cplx(lam)
        require_same_dims(dims_of(L), spec.hr, "FoldedSpectrum")
        self.spec = spec
        self.lam = L
        self._ctx = ctx or default_context()
        h = _vp()
        check(_lib.vsr_folded_create(self._ctx.handle, _dims_arr(spec.hr), _dims_arr(spec.rates),
                                     _p(L.view(np.float64)), C.byref(h)))
        self.handle = h

    def __del__(self):
        try:
            if self.handle:
                _lib.vsr_folded_destroy(self.handle)
        except Exception:
            pass

    def block_value(self, br, bc, bs, g):
        out = np.zeros(2)
        check(_lib.vsr_folded_block_value(self.handle, br, bc, bs, g, _p(out)))
        return complex(out[0], out[1])

    def apply(self, hr_spectrum):
        a = _cplx(hr_spectrum)
        require_same_dims(dims_of(a), self.spec.hr, "FoldedSpectrum::apply")
        out = np.empty(shape_of(self.spec.lr), np.complex128)
        check(_lib.vsr_folded_apply(self.handle, _p(a.view(np.float64)), _p(out.view(np.float64))))
        return out

    def apply_adjoint(self, lr_spectrum):
        a = _cplx(lr_spectrum)
        require_same_dims(dims_of(a), self.spec.lr, "FoldedSpectrum::apply_adjoint")
        out = np.empty(shape_of(self.spec.hr), np.complex128)
        check(_lib.vsr_folded_apply_adjoint(self.handle, _p(a.view(np.float64)),
                                            _p(out.view(np.float64))))
        return out

    def apply_weighted(self, hr_spectrum, hr_weights):
        a = _cplx(hr_spectrum)
        w = _real(hr_weights)
        require_same_dims(dims_of(a), self.spec.hr, "FoldedSpectrum::apply_weighted")
        require_same_dims(dims_of(w), self.spec.hr, "FoldedSpectrum::apply_weighted")
        out = np.empty(shape_of(self.spec.lr), np.complex128)
        check(_lib.vsr_folded_apply_weighted(self.handle, _p(a.view(np.float64)), _p(w),
                                             _p(out.view(np.float64))))
        return out

    def apply_adjoint_weighted(self, lr_spectrum, hr_weights):
        a = _cplx(lr_spectrum)
        w = _real(hr_weights)
        require_same_dims(dims_of(a), self.spec.lr, "FoldedSpectrum::apply_adjoint_weighted")
        require_same_dims(dims_of(w), self.spec.hr, "FoldedSpectrum::apply_adjoint_weighted")
        out = np.empty(shape_of(self.spec.hr), np.complex128)
        check(_lib.vsr_folded_apply_adjoint_weighted(self.handle, _p(a.view(np.float64)), _p(w),
                                                     _p(out.view(np.float64))))
        return out

    def swap_blocks_for_fault_injection(self):
        check(_lib.vsr_folded_swap_blocks_for_fault_injection(self.handle))


def fold_lambda(lam, spec, ctx=None):
    return FoldedSpectrum(lam, spec, ctx)


def gram_diag(folded: FoldedSpectrum):
    out = np.empty(shape_of(folded.spec.lr))
    check(_lib.vsr_folded_gram_diag(folded.handle, _p(out)))
    return out


def gram_diag_weighted(folded: FoldedSpectrum, hr_weights):
    w = _real(hr_weights)
    require_same_dims(dims_of(w), folded.spec.hr, "gram_diag_weighted")
    out = np.empty(shape_of(folded.spec.lr))
    check(_lib.vsr_folded_gram_diag_weighted(folded.handle, _p(w), _p(out)))
    return out


# ---------------------------------------------------------------- Tikhonov
@dataclass
class TikhonovConfig:
    """solvers.hpp:10-13."""
    lambda_: float = 0.01
    xbar: Optional[np.ndarray] = None


class TikhonovOperator:
    """solvers.hpp:27-43: precompute at construction, solve() = 1 fwd + 1 inv FFT."""

    def __init__(self, lam, spec: DecimationSpec, cfg: TikhonovConfig, ctx=None):
        require_positive(cfg.lambda_, "lambda")
        L = _cplx(lam)
        require_same_dims(dims_of(L), spec.hr, "TikhonovOperator")
        if cfg.xbar is None:
            raise ShapeError(f"TikhonovOperator: xbar: dims mismatch, 0x0x0 vs "
                             f"{spec.hr[0]}x{spec.hr[1]}x{spec.hr[2]}")
        xb = _real(cfg.xbar)
        require_same_dims(dims_of(xb), spec.hr, "TikhonovOperator: xbar")
        self.spec = spec
        self._ctx = ctx or default_context()
        h = _vp()
        check(_lib.vsr_tikhonov_create(self._ctx.handle, _dims_arr(spec.hr), _dims_arr(spec.rates),
                                       _p(L.view(np.float64)), float(cfg.lambda_), _p(xb),
                                       C.byref(h)))
        self.handle = h

    def solve(self, y) -> np.ndarray:
        a = _real(y)
        require_same_dims(dims_of(a), self.spec.lr, "TikhonovOperator::solve")
        out = np.empty(shape_of(self.spec.hr))
        check(_lib.vsr_tikhonov_solve(self.handle, _p(a), _p(out)))
        return out

    def solve_f32(self, y) -> np.ndarray:
        """fp32 mode (not a reference entry point): y and x in fp32, the LR
        stage in fp64, the expansion in fp32; spatial path only (fp32_ok())."""
        a = np.ascontiguousarray(y, dtype=np.float32)
        require_same_dims(dims_of(a), self.spec.lr, "TikhonovOperator::solve")
        out = np.empty(shape_of(self.spec.hr), dtype=np.float32)
        check(_lib.vsr_tikhonov_solve_f32(self.handle, a.ctypes.data, out.ctypes.data))
        return out

    def fp32_ok(self) -> bool:
        return bool(_lib.vsr_tikhonov_fp32_ok(self.handle))

    def path(self) -> dict:
        """Which specialisations the device solve uses (vsr_tikhonov_separable /
        _lattice_prior / _spatial)."""
        return {"separable": bool(_lib.vsr_tikhonov_separable(self.handle)),
                "lattice_prior": bool(_lib.vsr_tikhonov_lattice_prior(self.handle)),
                "spatial": bool(_lib.vsr_tikhonov_spatial(self.handle))}

    def close(self):
        if getattr(self, "handle", None):
            _lib.vsr_tikhonov_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def tikhonov_fast(y, lam, spec, cfg: TikhonovConfig, ctx=None):
    """solvers.cpp:69-72."""
    op = TikhonovOperator(lam, spec, cfg, ctx)
    try:
        return op.solve(y)
    finally:
        op.close()


# ---------------------------------------------------------------- TV
def make_gamma(hr_dims, tau: float, ctx=None) -> np.ndarray:
    """solvers.hpp:117 (from the analytic difference spectra)."""
    out = np.empty(shape_of(hr_dims))
    check(_lib.vsr_make_gamma(_ctx(ctx), _dims_arr(hr_dims), float(tau), _p(out)))
    return out


def tv_x_update(y, folded: FoldedSpectrum, lam, spec, mu, theta_hat, gamma, ctx=None):
    """solvers.hpp:89-91 (folded carries Lambda; lam must be the same spectrum)."""
    require_positive(mu, "mu")
    a = _real(y)
    require_same_dims(dims_of(a), spec.lr, "tv_x_update")
    th = _cplx(theta_hat)
    require_same_dims(dims_of(th), spec.hr, "tv_x_update: theta_hat")
    g = _real(gamma)
    require_same_dims(dims_of(g), spec.hr, "tv_x_update: gamma")
    L = _cplx(lam)
    out = np.empty(shape_of(spec.hr))
    check(_lib.vsr_tv_x_update(_ctx(ctx), _dims_arr(spec.hr), _dims_arr(spec.rates), _p(a),
                               _p(L.view(np.float64)), float(mu), _p(th.view(np.float64)), _p(g),
                               _p(out)))
    return out


def tv_shrink(nu1, nu2, nu3, threshold, ctx=None):
    """solvers.hpp:100-101."""
    a, b, c = _real(nu1), _real(nu2), _real(nu3)
    require_same_dims(dims_of(a), dims_of(b), "tv_shrink")
    require_same_dims(dims_of(a), dims_of(c), "tv_shrink")
    o = [np.empty_like(a) for _ in range(3)]
    check(_lib.vsr_tv_shrink(_ctx(ctx), a.size, _p(a), _p(b), _p(c), float(threshold), _p(o[0]),
                             _p(o[1]), _p(o[2])))
    return tuple(o)


def objective_tv(x, y, lam, spec, tv_weight, ctx=None) -> float:
    """solvers.hpp:111-112."""
    a, b, L = _real(x), _real(y), _cplx(lam)
    require_same_dims(dims_of(a), spec.hr, "objective_tv")
    require_same_dims(dims_of(b), spec.lr, "objective_tv")
    out = C.c_double()
    check(_lib.vsr_objective_tv(_ctx(ctx), _dims_arr(spec.hr), _dims_arr(spec.rates), _p(a), _p(b),
                                _p(L.view(np.float64)), float(tv_weight), C.byref(out)))
    return out.value


@dataclass
class TvAdmmConfig:
    """solvers.hpp:72-83."""
    lambda_: float = 0.06
    mu: float = 0.1
    max_iters: int = 30
    rel_tol: float = 1e-6
    tau: Optional[float] = None
    init: int = INIT_ZERO
    init_volume: Optional[np.ndarray] = None
    # "f64" (reference precision) or "f32": fp32 iteration state and fp32
    # transforms / fold (LR frequency 0 in fp64); not a reference field
    precision: str = "f64"


@dataclass
class SolveReport:
    """solvers.hpp:15-21."""
    iterations: int = 0
    initial_objective: float = 0.0
    objective: list = field(default_factory=list)
    primal_residual: list = field(default_factory=list)
    seconds: float = 0.0


def _tv_cfg(cfg: TvAdmmConfig, init_ptr=None) -> _TvConfig:
    c = _TvConfig()
    c.lambda_ = float(cfg.lambda_)
    c.mu = float(cfg.mu)
    c.max_iters = int(cfg.max_iters) if cfg.max_iters > 0 else 0
    c.rel_tol = float(cfg.rel_tol)
    c.has_tau = 0 if cfg.tau is None else 1
    c.tau = 0.0 if cfg.tau is None else float(cfg.tau)
    c.init = int(cfg.init)
    c.init_volume = init_ptr
    if cfg.precision not in ("f64", "f32"):
        raise ValueError("admm_tv: unknown precision")
    c.precision = 1 if cfg.precision == "f32" else 0
    return c


def admm_tv(y, psf, spec: DecimationSpec, cfg: TvAdmmConfig, ctx=None):
    """solvers.hpp:106-107 -> (x, SolveReport)."""
    require_positive(cfg.lambda_, "lambda")
    require_positive(cfg.mu, "mu")
    if cfg.max_iters < 1:
        raise ValueError("admm_tv: max_iters must be >= 1")
    a, p = _real(y), _real(psf)
    require_same_dims(dims_of(a), spec.lr, "admm_tv")
    require_same_dims(dims_of(p), spec.hr, "admm_tv: psf")
    init = None
    if cfg.init == INIT_PROVIDED:
        if cfg.init_volume is None:
            raise ShapeError("admm_tv: init volume: dims mismatch")
        init = _real(cfg.init_volume)
        require_same_dims(dims_of(init), spec.hr, "admm_tv: init volume")
    c = _tv_cfg(cfg, _p(init) if init is not None else None)
    obj = np.zeros(max(cfg.max_iters, 1))
    res = np.zeros(max(cfg.max_iters, 1))
    rep = _Report()
    rep.objective = _p(obj)
    rep.primal_residual = _p(res)
    out = np.empty(shape_of(spec.hr))
    check(_lib.vsr_admm_tv(_ctx(ctx), _dims_arr(spec.hr), _dims_arr(spec.rates), _p(a), _p(p),
                           C.byref(c), _p(out), C.byref(rep)))
    it = int(rep.iterations)
    report = SolveReport(iterations=it, initial_objective=float(rep.initial_objective),
                         objective=obj[:it].tolist(), primal_residual=res[:it].tolist(),
                         seconds=float(rep.seconds))
    return out, report


@dataclass
class AdmmL2Options:
    """solvers.hpp:58-62; warm_start = (x, v, dual) HR volumes or None."""
    mu: float = 0.1
    rel_tol: float = 1e-10
    warm_start: Optional[tuple] = None


class _L2Config(C.Structure):
    _fields_ = [("mu", C.c_double), ("rel_tol", C.c_double), ("warm_x", C.c_void_p),
                ("warm_v", C.c_void_p), ("warm_dual", C.c_void_p)]


_sig("vsr_admm_l2l2", [_vp, _szp, _szp, _dp, _dp, C.c_double, _dp, C.c_size_t, C.POINTER(_L2Config), _dp,
                       C.POINTER(_Report)])


def admm_l2l2(y, lam, spec, cfg: TikhonovConfig, max_iters: int, opts: Optional[AdmmL2Options] = None, ctx=None):
    """solvers.hpp:67-70 / solvers.cpp:95-189 -> (x, SolveReport)."""
    opts = opts or AdmmL2Options()
    require_positive(cfg.lambda_, "lambda")
    require_positive(opts.mu, "mu")
    a = _real(y)
    require_same_dims(dims_of(a), spec.lr, "admm_l2l2")
    if cfg.xbar is None:
        raise ShapeError("admm_l2l2: xbar: dims mismatch")
    xb = _real(cfg.xbar)
    require_same_dims(dims_of(xb), spec.hr, "admm_l2l2: xbar")
    if max_iters < 1:
        raise ValueError("admm_l2l2: max_iters must be >= 1")
    L = _cplx(lam)
    require_same_dims(dims_of(L), spec.hr, "admm_l2l2: lambda")
    c = _L2Config(float(opts.mu), float(opts.rel_tol), None, None, None)
    keep = []
    if opts.warm_start is not None:
        ws = [_real(w) for w in opts.warm_start]
        for w in ws:
            require_same_dims(dims_of(w), spec.hr, "admm_l2l2: warm start")
        keep = ws
        c.warm_x, c.warm_v, c.warm_dual = (w.ctypes.data for w in ws)
    obj = np.zeros(max_iters)
    res = np.zeros(max_iters)
    rep = _Report()
    rep.objective = _p(obj)
    rep.primal_residual = _p(res)
    out = np.empty(shape_of(spec.hr))
    check(_lib.vsr_admm_l2l2(_ctx(ctx), _dims_arr(spec.hr), _dims_arr(spec.rates), _p(a),
                             _p(L.view(np.float64)), float(cfg.lambda_), _p(xb), C.c_size_t(max_iters),
                             C.byref(c), _p(out), C.byref(rep)))
    del keep
    it = int(rep.iterations)
    report = SolveReport(iterations=it, initial_objective=float(rep.initial_objective),
                         objective=obj[:it].tolist(), primal_residual=res[:it].tolist(),
                         seconds=float(rep.seconds))
    return out, report


def tikhonov_algorithmic_bytes(hr_dims, rates) -> float:
    return float(_lib.vsr_tikhonov_algorithmic_bytes(_dims_arr(hr_dims), _dims_arr(rates)))


def tv_algorithmic_bytes(hr_dims, rates) -> float:
    return float(_lib.vsr_tv_algorithmic_bytes(_dims_arr(hr_dims), _dims_arr(rates)))


# ---------------------------------------------------------------- slab stages (dist.py)
_sig("vsr_fft3_d", [_vp, _szp, _vp, C.c_int, _vp, C.c_double])


# ---------------------------------------------------------------- instrumentation
_sig("vsr_launch_count", [C.POINTER(C.c_uint64)])
_sig("vsr_tikhonov_separable", [_vp])
_sig("vsr_tikhonov_lattice_prior", [_vp])
_sig("vsr_tikhonov_spatial", [_vp])
_sig("vsr_tv_separable", [_vp])
_sig("vsr_profile_enable", [_vp, C.c_int])
_sig("vsr_profile_read", [_vp, C.c_int, C.c_char_p, C.c_size_t, _dp, C.POINTER(C.c_uint64),
                          C.POINTER(C.c_int)])


def launch_count() -> int:
    v = C.c_uint64()
    check(_lib.vsr_launch_count(C.byref(v)))
    return v.value


def profile_enable(ctx: Context, on: bool):
    check(_lib.vsr_profile_enable(ctx.handle, int(bool(on))))


def profile_read(ctx: Context, max_stages: int = 64) -> dict:
    """{stage: (total_ms, launches)} recorded since the last read."""
    L = 48
    names = C.create_string_buffer(max_stages * L)
    ms = (C.c_double * max_stages)()
    cnt = (C.c_uint64 * max_stages)()
    n = C.c_int()
    check(_lib.vsr_profile_read(ctx.handle, max_stages, names, L, ms, cnt, C.byref(n)))
    out = {}
    for i in range(n.value):
        nm = names.raw[i * L:(i + 1) * L].split(b"\0", 1)[0].decode()
        out[nm] = (ms[i], cnt[i])
    return out


class DeviceBuffer:
    """Raw device allocation on a context (bench / device-resident API)."""

    def __init__(self, ctx: Context, nbytes: int):
        self.ctx = ctx
        self.nbytes = int(nbytes)
        p = _vp()
        check(_lib.vsr_device_alloc(ctx.handle, self.nbytes, C.byref(p)))
        self.ptr = p

    def upload(self, a: np.ndarray):
        a = np.ascontiguousarray(a)
        assert a.nbytes == self.nbytes
        check(_lib.vsr_memcpy_h2d(self.ctx.handle, self.ptr, a.ctypes.data_as(_vp), a.nbytes))

    def download(self, a: np.ndarray):
        assert a.nbytes == self.nbytes and a.flags.c_contiguous
        check(_lib.vsr_memcpy_d2h(self.ctx.handle, a.ctypes.data_as(_vp), self.ptr, a.nbytes))

    def free(self):
        if self.ptr:
            _lib.vsr_device_free(self.ctx.handle, self.ptr)
            self.ptr = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


class PinnedBuffer:
    """Page-locked host buffer viewed as a numpy array."""

    def __init__(self, shape, dtype=np.float64):
        self.dtype = np.dtype(dtype)
        self.shape = tuple(shape)
        nbytes = int(np.prod(self.shape)) * self.dtype.itemsize
        p = _vp()
        check(_lib.vsr_host_alloc(max(nbytes, 1), C.byref(p)))
        self.ptr = p
        buf = (C.c_char * max(nbytes, 1)).from_address(p.value)
        self.array = np.frombuffer(buf, dtype=self.dtype, count=int(np.prod(self.shape))).reshape(self.shape)

    def free(self):
        if self.ptr:
            self.array = None
            _lib.vsr_host_free(self.ptr)
            self.ptr = None


class TikhonovDevice:
    """Device-resident TikhonovOperator (vsr_tikhonov_*_d) for streaming/bench use."""

    def __init__(self, ctx: Context, spec: DecimationSpec, lam_dev: DeviceBuffer, reg: float,
                 xbar_dev: DeviceBuffer):
        h = _vp()
        check(_lib.vsr_tikhonov_create_d(ctx.handle, _dims_arr(spec.hr), _dims_arr(spec.rates),
                                         lam_dev.ptr, float(reg), xbar_dev.ptr, C.byref(h)))
        self.handle = h
        self.spec = spec

    def solve_d(self, y_dev, x_dev):
        check(_lib.vsr_tikhonov_solve_d(self.handle, y_dev.ptr, x_dev.ptr))

    def solve_host(self, y: np.ndarray, x_out: np.ndarray):
        check(_lib.vsr_tikhonov_solve(self.handle, _p(y), _p(x_out)))

    def solve_f32_d(self, y_dev, x_dev):
        check(_lib.vsr_tikhonov_solve_f32_d(self.handle, y_dev.ptr, x_dev.ptr))

    def solve_f32_host(self, y: np.ndarray, x_out: np.ndarray):
        check(_lib.vsr_tikhonov_solve_f32(self.handle, y.ctypes.data, x_out.ctypes.data))

    def check(self):
        check(_lib.vsr_tikhonov_check(self.handle))

    def separable(self) -> bool:
        return bool(_lib.vsr_tikhonov_separable(self.handle))

    def lattice_prior(self) -> bool:
        return bool(_lib.vsr_tikhonov_lattice_prior(self.handle))

    def spatial(self) -> bool:
        return bool(_lib.vsr_tikhonov_spatial(self.handle))

    def close(self):
        if self.handle:
            _lib.vsr_tikhonov_destroy(self.handle)
            self.handle = None


class TvDevice:
    """Device-resident ADMM-TV stepper (vsr_tv_*_d)."""

    def __init__(self, ctx: Context, spec: DecimationSpec, y_dev: DeviceBuffer, psf_dev: DeviceBuffer,
                 cfg: TvAdmmConfig, init_dev: Optional[DeviceBuffer] = None):
        c = _tv_cfg(cfg, C.cast(init_dev.ptr, _dp) if init_dev is not None else None)
        h = _vp()
        check(_lib.vsr_tv_create_d(ctx.handle, _dims_arr(spec.hr), _dims_arr(spec.rates), y_dev.ptr,
                                   psf_dev.ptr, C.byref(c), C.byref(h)))
        self.handle = h
        self.spec = spec
        self.max_iters = cfg.max_iters

    def iterate(self, k: int):
        check(_lib.vsr_tv_iterate_d(self.handle, int(k)))

    def report(self) -> SolveReport:
        obj = np.zeros(max(self.max_iters, 1))
        res = np.zeros(max(self.max_iters, 1))
        rep = _Report()
        rep.objective = _p(obj)
        rep.primal_residual = _p(res)
        check(_lib.vsr_tv_report(self.handle, C.byref(rep)))
        it = int(rep.iterations)
        return SolveReport(it, float(rep.initial_objective), obj[:it].tolist(), res[:it].tolist(),
                           float(rep.seconds))

    def separable(self) -> bool:
        return bool(_lib.vsr_tv_separable(self.handle))

    def x_ptr(self) -> int:
        p = _vp()
        check(_lib.vsr_tv_x_d(self.handle, C.byref(p)))
        return p.value

    def close(self):
        if self.handle:
            _lib.vsr_tv_destroy(self.handle)
            self.handle = None


# ---------------------------------------------------------------- volume files
_sig("vsr_volume_header", [C.c_char_p, _szp, C.POINTER(C.c_int)])
_sig("vsr_load_volume", [C.c_char_p, _vp, C.c_size_t])
_sig("vsr_save_volume", [C.c_char_p, _szp, _vp, C.c_int])
_sig("vsr_load_volume_d", [_vp, C.c_char_p, _vp, C.c_size_t])
_sig("vsr_save_volume_d", [_vp, C.c_char_p, _szp, _vp, C.c_int])


def strip_volume_extension(path: str) -> str:
    """volume_io.cpp:27-31."""
    for ext in (".volhdr", ".vol"):
        if path.endswith(ext):
            return path[: -len(ext)]
    return path


def volume_header(path: str):
    """(dims (m, n, s), dtype "f32" | "f64") of <base>.volhdr."""
    d = (C.c_size_t * 3)()
    t = C.c_int()
    check(_lib.vsr_volume_header(str(path).encode(), d, C.byref(t)))
    return (int(d[0]), int(d[1]), int(d[2])), ("f32" if t.value == VSR_DTYPE_F32 else "f64")


def load_volume(path: str) -> np.ndarray:
    """volsr::load_volume (volume_io.cpp:61-131): array of shape (s, n, m)."""
    dims, _ = volume_header(path)
    out = np.empty(shape_of(dims))
    check(_lib.vsr_load_volume(str(path).encode(), _p(out), out.size))
    return out


def save_volume(v: np.ndarray, path: str, dtype: str = "f64"):
    """volsr::save_volume (volume_io.cpp:34-57); v has shape (s, n, m)."""
    a = _real(v)
    check(_lib.vsr_save_volume(str(path).encode(), _dims_arr(dims_of(a)), _p(a),
                               VSR_DTYPE_F32 if dtype == "f32" else VSR_DTYPE_F64))


def load_volume_device(path: str, out_dev, ctx=None):
    """Streams <base>.vol into a device buffer (object with .ptr) of dims.count() doubles."""
    dims, _ = volume_header(path)
    check(_lib.vsr_load_volume_d(_ctx(ctx), str(path).encode(), out_dev.ptr, dims[0] * dims[1] * dims[2]))
    return dims


def save_volume_device(in_dev, dims, path: str, dtype: str = "f64", ctx=None):
    """Streams a device volume (object with .ptr) to <base>.volhdr/.vol."""
    check(_lib.vsr_save_volume_d(_ctx(ctx), str(path).encode(), _dims_arr(tuple(dims)), in_dev.ptr,
                                 VSR_DTYPE_F32 if dtype == "f32" else VSR_DTYPE_F64))


# ---------------------------------------------------------------- degrade
_sig("vsr_degrade", [_vp, _szp, _szp, _vp, _vp, C.c_int, C.c_double, C.c_uint64, _vp, C.POINTER(C.c_double)])


def degrade(x, psf, spec: DecimationSpec, bsnr_db: Optional[float] = None, seed: int = 0, ctx=None):
    """volsr::degrade (sim.cpp:106-127) on the GPU: y = D H x + sigma n with the
    reference's mt19937_64 + Box-Muller noise stream.  psf: HR volume as
    make_gaussian_psf builds it.  Returns (y, noise_sigma)."""
    a, p = _real(x), _real(psf)
    require_same_dims(dims_of(a), spec.hr, "degrade")
    require_same_dims(dims_of(p), spec.hr, "degrade")
    y = np.empty(shape_of(spec.lr))
    sig = C.c_double()
    check(_lib.vsr_degrade(_ctx(ctx), _dims_arr(spec.hr), _dims_arr(spec.rates), _p(a), _p(p),
                           int(bsnr_db is not None), float(bsnr_db or 0.0), int(seed), _p(y), C.byref(sig)))
    return y, sig.value
