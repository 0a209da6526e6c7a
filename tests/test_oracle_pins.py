"""Pins the CPU oracle (oracle/volsr_oracle.py) to the reference's own
known-answer and dense-oracle tests (restated; the reference keeps no golden
files).  Each test cites the reference test it restates.  CPU only."""
import math

import numpy as np
import pytest

from conftest import random_psf, random_spectrum, random_volume, rel_err


# ------------------------------------------------------------------ FFT contract
def test_fft3_constant_dc(O):
    """test_volume.cpp:44-50: DC = c*sqrt(N), zero elsewhere."""
    d = (4, 3, 5)
    c = 0.75
    sp = O.fft3(np.full(O.shape_of(d), c))
    assert abs(sp.reshape(-1)[0] - c * math.sqrt(60)) < 1e-12
    assert np.all(np.abs(sp.reshape(-1)[1:]) < 1e-12)


@pytest.mark.parametrize("d", [(5, 3, 7), (4, 6, 2), (8, 8, 8), (1, 9, 4)])
def test_fft3_roundtrip_parseval(O, d):
    """test_volume.cpp:52-69."""
    rng = np.random.default_rng(7)
    x = random_volume(d, rng)
    xh = O.fft3(x)
    back = O.ifft3(xh)
    assert rel_err(back, x) < 1e-12
    assert abs(np.sum(np.abs(xh) ** 2) - np.sum(x * x)) / np.sum(x * x) < 1e-12


def test_fft3_matches_dense_dft(O):
    """test_volume.cpp:71-81: pins sign, scale and axis order."""
    rng = np.random.default_rng(11)
    d = (4, 3, 2)
    x = random_volume(d, rng)
    want = O.build_dense_dft(d) @ x.reshape(-1)
    assert np.max(np.abs(O.fft3(x).reshape(-1) - want)) < 1e-12


def test_ifft3_real_rejects_nonhermitian(O):
    """test_volume.cpp:83-87."""
    rng = np.random.default_rng(3)
    with pytest.raises(O.NumericError):
        O.ifft3_real(random_spectrum((4, 4, 4), rng), 1e-8)


# ------------------------------------------------------------------ operators
def test_psf_normalised_and_symmetric(O):
    """test_operators.cpp (PSF normalisation / symmetry)."""
    psf = O.make_gaussian_psf((5, 5, 3), (1.5, 1.2, 1.0), (8, 8, 8))
    assert abs(psf.sum() - 1.0) < 1e-14
    assert np.allclose(psf, np.roll(np.flip(psf), 1, axis=(0, 1, 2)))


def test_blur_equals_dense_circulant(O):
    rng = np.random.default_rng(4)
    d = (4, 3, 5)
    psf = random_psf(d, 3, rng)
    x = random_volume(d, rng)
    want = O.build_dense_blur(psf) @ x.reshape(-1)
    got = O.blur_apply(x, O.psf_to_spectrum(psf))
    assert rel_err(got.reshape(-1), want) < 1e-12


@pytest.mark.parametrize("axis", [0, 1, 2])
def test_diff_spectra_match_stencils(O, axis):
    """test_operators.cpp: difference spectra diagonalise the periodic stencil."""
    rng = np.random.default_rng(5)
    d = (5, 4, 3)
    x = random_volume(d, rng)
    spec = O.finite_diff_spectra(d)[axis]
    got = O.ifft3_real(spec * O.fft3(x))
    assert rel_err(got, O.diff_forward(x, axis)) < 1e-12
    # adjointness <Lx, y> = <x, L^T y>
    y = random_volume(d, rng)
    assert abs(np.sum(O.diff_forward(x, axis) * y) - np.sum(x * O.diff_adjoint(y, axis))) < 1e-12


def test_decimation_adjoint(O):
    rng = np.random.default_rng(6)
    spec = O.DecimationSpec((6, 4, 8), (3, 2, 4))
    x = random_volume(spec.hr, rng)
    y = random_volume(spec.lr, rng)
    assert abs(np.sum(O.decimate(x, spec) * y) - np.sum(x * O.decimate_adjoint(y, spec))) < 1e-12
    assert np.array_equal(O.decimate(O.decimate_adjoint(y, spec), spec), y)  # D D^H = I


def test_decimation_spec_errors(O):
    with pytest.raises(O.ShapeError, match="does not divide axis 2"):
        O.DecimationSpec((4, 5, 4), (2, 2, 2))
    with pytest.raises(O.ShapeError, match="zero rate"):
        O.DecimationSpec((4, 4, 4), (0, 1, 1))


# ------------------------------------------------------------------ spectral fold
def test_alias_fold_single_axis(O):
    """test_spectral.cpp:35-49."""
    spec = O.DecimationSpec((4, 1, 1), (2, 1, 1))
    v = np.array([1 + 2j, 3 - 1j, 0.5 + 0.25j, -2 + 1j]).reshape(1, 1, 4)
    out = O.alias_fold(v, spec).reshape(-1)
    assert out[0] == v.reshape(-1)[0] + v.reshape(-1)[2]
    assert out[1] == v.reshape(-1)[1] + v.reshape(-1)[3]


def test_alias_fold_rate1_identity(O):
    rng = np.random.default_rng(1)
    spec = O.DecimationSpec((3, 4, 5), (1, 1, 1))
    v = random_spectrum(spec.hr, rng)
    assert rel_err(O.alias_fold(v, spec), v) == 0.0


def _structural(O, spec):
    def kron(a, b):
        return np.kron(a, b)

    def factor(d, ln):
        return kron(np.ones((1, d)), np.eye(ln))

    return kron(factor(spec.rates[2], spec.lr[2]),
                kron(factor(spec.rates[1], spec.lr[1]), factor(spec.rates[0], spec.lr[0])))


@pytest.mark.parametrize("hr,rates", [((4, 4, 2), (2, 2, 1)), ((6, 4, 4), (3, 2, 2)), ((8, 4, 4), (2, 1, 2))])
def test_fold_matches_dense(O, hr, rates):
    """test_spectral.cpp: fold == structural matrix; apply/adjoint/gram vs dense."""
    rng = np.random.default_rng(2)
    spec = O.DecimationSpec(hr, rates)
    v = random_spectrum(hr, rng)
    S = _structural(O, spec)
    assert np.max(np.abs(O.alias_fold(v, spec).reshape(-1) - S @ v.reshape(-1))) < 1e-12
    lam = random_spectrum(hr, rng)
    f = O.FoldedSpectrum(lam, spec)
    A = S @ np.diag(lam.reshape(-1))
    assert np.max(np.abs(f.apply(v).reshape(-1) - A @ v.reshape(-1))) < 1e-12
    w = random_spectrum(spec.lr, rng)
    assert np.max(np.abs(f.apply_adjoint(w).reshape(-1) - A.conj().T @ w.reshape(-1))) < 1e-12
    assert np.max(np.abs(O.gram_diag(f).reshape(-1) - np.real(np.diag(A @ A.conj().T)))) < 1e-12
    gw = rng.uniform(0.1, 1.0, O.shape_of(hr))
    Aw = A @ np.diag(gw.reshape(-1))
    assert np.max(np.abs(O.gram_diag_weighted(f, gw).reshape(-1) - np.real(np.diag(Aw @ A.conj().T)))) < 1e-12


@pytest.mark.parametrize("hr,rates", [((4, 4, 4), (2, 2, 2)), ((6, 4, 2), (3, 2, 1)), ((4, 6, 4), (2, 3, 2)),
                                      ((8, 2, 4), (4, 1, 2)), ((3, 3, 3), (3, 3, 3))])
def test_eq8_decomposition(O, hr, rates):
    """spectral.cpp:163-178 / acceptance c1: F D^H D F^H equals the Kronecker form."""
    spec = O.DecimationSpec(hr, rates)
    D = O.build_dense_decimation(spec)
    F = O.build_dense_dft(spec.hr)
    lhs = F @ (D.T @ D) @ F.conj().T

    def oki(d, ln):
        return np.kron(np.ones((d, d)), np.eye(ln)) / d

    rhs = np.kron(oki(rates[2], spec.lr[2]), np.kron(oki(rates[1], spec.lr[1]), oki(rates[0], spec.lr[0])))
    assert np.max(np.abs(lhs - rhs)) < 1e-10


def test_fault_injection_changes_fold(O):
    rng = np.random.default_rng(3)
    spec = O.DecimationSpec((4, 4, 4), (2, 2, 2))
    lam = random_spectrum(spec.hr, rng)
    f = O.FoldedSpectrum(lam, spec)
    v = random_spectrum(spec.hr, rng)
    a = f.apply(v)
    f.swap_blocks_for_fault_injection()
    assert rel_err(f.apply(v), a) > 1e-3


# ------------------------------------------------------------------ Tikhonov
def test_tikhonov_identity_scalar_formula(O):
    """test_solvers.cpp:55-69."""
    rng = np.random.default_rng(1)
    d = (4, 4, 4)
    spec = O.DecimationSpec(d, (1, 1, 1))
    ones = np.ones(O.shape_of(d), np.complex128)
    xbar = random_volume(d, rng)
    y = random_volume(d, rng)
    x = O.tikhonov_fast(y, ones, spec, 0.35, xbar)
    want = (y + 2 * 0.35 * xbar) / (1 + 2 * 0.35)
    assert np.max(np.abs(x - want) / np.maximum(np.abs(want), 1e-300)) < 1e-12


def test_tikhonov_huge_lambda_returns_prior(O):
    """test_solvers.cpp:71-82."""
    rng = np.random.default_rng(2)
    d = (8, 8, 8)
    spec = O.DecimationSpec(d, (2, 2, 2))
    psf = random_psf(d, 3, rng)
    xbar = random_volume(d, rng)
    y = random_volume(spec.lr, rng)
    x = O.tikhonov_fast(y, O.psf_to_spectrum(psf), spec, 1e6, xbar)
    assert rel_err(x, xbar) < 1e-4


def test_tikhonov_rejects_bad_lambda(O):
    d = (4, 4, 4)
    with pytest.raises(ValueError):
        O.tikhonov_fast(np.zeros(O.shape_of(d)), np.ones(O.shape_of(d), complex),
                        O.DecimationSpec(d, (1, 1, 1)), 0.0, np.zeros(O.shape_of(d)))


@pytest.mark.parametrize("dims,rates", [((8, 8, 8), (2, 2, 2)), ((6, 4, 4), (3, 2, 1)),
                                        ((4, 6, 4), (2, 3, 2)), ((8, 4, 4), (2, 1, 2))])
def test_tikhonov_matches_dense(O, dims, rates):
    """test_solvers.cpp:94-111 (fast vs dense normal equations at 1e-8)."""
    rng = np.random.default_rng(3)
    spec = O.DecimationSpec(dims, rates)
    psf = random_psf(dims, 3, rng)
    lam = 0.02 + 0.2 * rng.uniform()
    xbar = random_volume(dims, rng)
    y = random_volume(spec.lr, rng)
    fast = O.tikhonov_fast(y, O.psf_to_spectrum(psf), spec, lam, xbar)
    dense = O.dense_tikhonov(y, psf, spec, lam, xbar)
    assert rel_err(fast, dense) < 1e-8


def test_tikhonov_normal_equations(O):
    """test_solvers.cpp:113-139."""
    rng = np.random.default_rng(4)
    d = (12, 10, 8)
    spec = O.DecimationSpec(d, (2, 2, 2))
    psf = O.make_gaussian_psf((5, 5, 5), (1.5, 1.2, 1.0), d)
    lam = O.psf_to_spectrum(psf)
    xbar = random_volume(d, rng)
    y = random_volume(spec.lr, rng)
    x = O.tikhonov_fast(y, lam, spec, 0.05, xbar)
    hx = O.blur_apply(x, lam)
    lhs = O.blur_apply(O.decimate_adjoint(O.decimate(hx, spec), spec), lam, True) + 0.1 * x
    rhs = O.blur_apply(O.decimate_adjoint(y, spec), lam, True) + 0.1 * xbar
    assert rel_err(lhs, rhs) < 1e-8


def test_tikhonov_fft_budget(O):
    """test_solvers.cpp:141-157: exactly one forward and one inverse FFT per solve."""
    rng = np.random.default_rng(5)
    d = (8, 8, 8)
    spec = O.DecimationSpec(d, (2, 2, 2))
    op = O.TikhonovOperator(O.psf_to_spectrum(random_psf(d, 3, rng)), spec, 0.1, random_volume(d, rng))
    O.reset_fft_counters()
    op.solve(random_volume(spec.lr, rng))
    assert O.fft_counters() == {"forward": 1, "inverse": 1}


# ------------------------------------------------------------------ TV pieces
def test_tv_shrink_closed_forms(O):
    """test_solvers.cpp:261-287."""
    one = lambda v: np.full((1, 1, 1), v)
    out = O.tv_shrink(one(3.0), one(0.0), one(0.0), 1.0)
    assert abs(out[0][0, 0, 0] - 2.0) < 1e-12 and out[1][0, 0, 0] == 0 and out[2][0, 0, 0] == 0
    out = O.tv_shrink(one(0.3), one(0.2), one(0.1), 1.0)
    assert all(o[0, 0, 0] == 0 for o in out)
    out = O.tv_shrink(one(0.0), one(0.0), one(0.0), 0.0)
    assert out[0][0, 0, 0] == 0
    with pytest.raises(ValueError):
        O.tv_shrink(one(1.0), one(0.0), one(0.0), -0.5)


def test_tv_shrink_is_prox(O):
    """test_solvers.cpp:289-303: agrees with a brute-force prox minimiser."""
    from scipy.optimize import minimize
    rng = np.random.default_rng(9)
    for _ in range(10):
        nu = rng.uniform(-2, 2, 3)
        t = rng.uniform(0, 1.5)
        f = lambda z: t * np.linalg.norm(z) + 0.5 * np.sum((z - nu) ** 2)
        best = min((minimize(f, x0, method="Nelder-Mead", options={"xatol": 1e-10, "fatol": 1e-14, "maxiter": 4000})
                    for x0 in (nu, np.zeros(3) + 1e-3)), key=lambda r: r.fun)
        got = O.tv_shrink(*(np.full((1, 1, 1), v) for v in nu), t)
        assert np.max(np.abs(np.array([g[0, 0, 0] for g in got]) - best.x)) < 1e-3


def test_tv_shrink_nonexpansive(O):
    """test_solvers.cpp:305-321."""
    rng = np.random.default_rng(10)
    d = (6, 6, 6)
    a = [random_volume(d, rng) for _ in range(3)]
    b = [random_volume(d, rng) for _ in range(3)]
    sa, sb = O.tv_shrink(*a, 0.4), O.tv_shrink(*b, 0.4)
    num = sum(np.sum((x - y) ** 2) for x, y in zip(sa, sb))
    den = sum(np.sum((x - y) ** 2) for x, y in zip(a, b))
    assert num <= den * (1 + 1e-12)


def test_tv_x_update_zero(O):
    """test_solvers.cpp:323-333."""
    d = (8, 8, 8)
    spec = O.DecimationSpec(d, (2, 2, 2))
    lam = O.psf_to_spectrum(O.make_gaussian_psf((3, 3, 3), (1, 1, 1), d))
    f = O.FoldedSpectrum(lam, spec)
    g = O.make_gamma(d, 1e-8)
    x = O.tv_x_update(np.zeros(O.shape_of(spec.lr)), f, lam, spec, 0.5,
                      np.zeros(O.shape_of(d), complex), g)
    assert np.sqrt(np.sum(x * x)) < 1e-12


def _random_theta(O, d, rng):
    th = np.zeros(O.shape_of(d))
    for a in range(3):
        th = th + O.diff_adjoint(random_volume(d, rng), a)
    return th


def test_tv_x_update_matches_dense(O):
    """test_solvers.cpp:335-367."""
    rng = np.random.default_rng(11)
    d = (8, 8, 8)
    spec = O.DecimationSpec(d, (2, 2, 2))
    psf = random_psf(d, 3, rng)
    lam = O.psf_to_spectrum(psf)
    f = O.FoldedSpectrum(lam, spec)
    mu, tau = 0.7, 1e-6
    g = O.make_gamma(d, tau)
    for _ in range(3):
        y = random_volume(spec.lr, rng)
        th = _random_theta(O, d, rng)
        fast = O.tv_x_update(y, f, lam, spec, mu, O.fft3(th), g)
        dense = O.dense_tv_x_update(y, psf, spec, mu, th, tau)
        assert rel_err(fast, dense) < 1e-8
    d = (6, 4, 4)
    spec = O.DecimationSpec(d, (1, 1, 1))
    psf = O.make_gaussian_psf((1, 1, 1), (0, 0, 0), d)
    lam = O.psf_to_spectrum(psf)
    f = O.FoldedSpectrum(lam, spec)
    g = O.make_gamma(d, 1e-8)
    y = random_volume(d, rng)
    th = _random_theta(O, d, rng)
    assert rel_err(O.tv_x_update(y, f, lam, spec, 1.0, O.fft3(th), g),
                   O.dense_tv_x_update(y, psf, spec, 1.0, th, 1e-8)) < 1e-6


def test_unfloored_gamma_rejected(O):
    """test_solvers.cpp:369-384."""
    with pytest.raises(O.NumericError, match="zero frequency"):
        O.make_gamma((4, 4, 4), 0.0)
    d = (4, 4, 4)
    spec = O.DecimationSpec(d, (2, 2, 2))
    lam = O.psf_to_spectrum(O.make_gaussian_psf((3, 3, 3), (1, 1, 1), d))
    f = O.FoldedSpectrum(lam, spec)
    g = O.make_gamma(d, 1e-8)
    g[0, 0, 0] = 0.0
    with pytest.raises(O.NumericError):
        O.tv_x_update(np.zeros(O.shape_of(spec.lr)), f, lam, spec, 1.0, np.zeros(O.shape_of(d), complex), g)


def test_admm_tv_near_identity(O):
    """test_solvers.cpp:386-401."""
    rng = np.random.default_rng(12)
    d = (12, 12, 12)
    spec = O.DecimationSpec(d, (1, 1, 1))
    psf = O.make_gaussian_psf((1, 1, 1), (0, 0, 0), d)
    y = random_volume(d, rng, 0.0, 1.0)
    x, rep = O.admm_tv(y, psf, spec, lam_tv=1e-6, mu=0.1, max_iters=60, rel_tol=1e-9)
    assert rel_err(x, y) < 1e-3
    assert rep.objective[-1] <= rep.initial_objective


def test_admm_tv_validates(O):
    """test_solvers.cpp:426-452."""
    d = (8, 8, 8)
    spec = O.DecimationSpec(d, (2, 2, 2))
    psf = O.make_gaussian_psf((3, 3, 3), (1, 1, 1), d)
    y = np.full(O.shape_of(spec.lr), 0.5)
    O.admm_tv(y, psf, spec, max_iters=2, init=O.INIT_UPSAMPLED)
    O.admm_tv(y, psf, spec, max_iters=2, init=O.INIT_PROVIDED, init_volume=np.full(O.shape_of(d), 0.25))
    with pytest.raises(O.ShapeError):
        O.admm_tv(y, psf, spec, max_iters=2, init=O.INIT_PROVIDED, init_volume=np.zeros((4, 4, 4)))
    with pytest.raises(ValueError):
        O.admm_tv(y, psf, spec, lam_tv=-1.0)
    with pytest.raises(ValueError):
        O.admm_tv(y, psf, spec, mu=0.0)
    with pytest.raises(ValueError):
        O.admm_tv(y, psf, spec, max_iters=0)


def test_objective_tv_examples(O):
    """test_solvers.cpp:454-492."""
    rng = np.random.default_rng(13)
    d = (6, 4, 4)
    spec = O.DecimationSpec(d, (2, 2, 2))
    psf = random_psf(d, 3, rng)
    lam = O.psf_to_spectrum(psf)
    x = np.full(O.shape_of(d), 0.8)
    y = O.decimate(O.blur_apply(x, lam), spec)
    assert O.objective_tv(x, y, lam, spec, 0.25) < 1e-20
    x = random_volume(d, rng)
    y = random_volume(spec.lr, rng)
    got = O.objective_tv(x, y, lam, spec, 0.3)
    H = O.build_dense_blur(psf)
    D = O.build_dense_decimation(spec)
    z = D @ H @ x.reshape(-1)
    want = 0.5 * np.sum((y.reshape(-1) - z) ** 2)
    g = [O.build_dense_diff(d, a) @ x.reshape(-1) for a in range(3)]
    want += 0.3 * np.sum(np.sqrt(g[0] ** 2 + g[1] ** 2 + g[2] ** 2))
    assert abs(got - want) / want < 1e-10


def test_admm_l2l2_fixed_point(O):
    """test_solvers.cpp:200-225."""
    rng = np.random.default_rng(7)
    d = (8, 8, 8)
    spec = O.DecimationSpec(d, (2, 2, 2))
    psf = random_psf(d, 3, rng)
    lam = O.psf_to_spectrum(psf)
    xbar = random_volume(d, rng)
    y = random_volume(spec.lr, rng)
    xs = O.tikhonov_fast(y, lam, spec, 0.05, xbar)
    v = O.blur_apply(xs, lam)
    r = O.decimate(v, spec) - y
    dual = O.decimate_adjoint(r, spec) / 0.3
    x1, rep = O.admm_l2l2(y, lam, spec, 0.05, xbar, 1, mu=0.3, rel_tol=0.0, warm_start=(xs, v, dual))
    assert rep.iterations == 1
    assert rel_err(x1, xs) < 1e-10


# ------------------------------------------------------------------ lean oracle
# oracle/lean_oracle.py (the config-4 checker, memory-lean) pinned to the
# line-by-line oracle and to the reference binary (oracle/_ref) where built.
@pytest.mark.parametrize("dims,rates", [((32, 32, 32), (2, 2, 2)), ((32, 16, 24), (2, 2, 4)),
                                        ((16, 16, 16), (4, 4, 4)), ((20, 12, 6), (5, 3, 2))])
def test_lean_oracle_pinned(O, dims, rates):
    import lean_oracle as LO
    import ref_binding as R
    rng = np.random.default_rng(77)
    spec = O.DecimationSpec(dims, rates)
    psf = O.make_gaussian_psf((5, 5, 3), (1.2, 1.0, 0.8), dims)
    y = random_volume(spec.lr, rng, 0.0, 1.0)
    xbar = O.zero_fill_upsample(y, spec)
    want = O.tikhonov_fast(y, O.psf_to_spectrum(psf), spec, 1e-3, xbar)
    assert rel_err(LO.tikhonov_fast(y, psf, spec, 1e-3, xbar), want) < 1e-13
    for init in (O.INIT_ZERO, O.INIT_UPSAMPLED):
        xa, ra = O.admm_tv(y, psf, spec, lam_tv=2e-3, mu=0.05, max_iters=3, rel_tol=0.0, tau=5e-5, init=init)
        xb, rb = LO.admm_tv(y, psf, spec, 2e-3, 0.05, 3, tau=5e-5, init=init)
        assert rel_err(xb, xa) < 1e-10
        assert abs(rb.initial_objective - ra.initial_objective) <= 1e-13 * abs(ra.initial_objective)
        np.testing.assert_allclose(rb.objective, ra.objective, rtol=1e-13)
        np.testing.assert_allclose(rb.primal_residual, ra.primal_residual, rtol=1e-13)
        if R.available():
            xr, rr = R.admm_tv(y, psf, dims, rates, 2e-3, 0.05, 3, 0.0, tau=5e-5, init=init)
            assert rel_err(xb, xr) < 1e-10
            np.testing.assert_allclose(rb.objective, rr["objective"], rtol=1e-12)
            np.testing.assert_allclose(rb.primal_residual, rr["primal_residual"], rtol=1e-12)
