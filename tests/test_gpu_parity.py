"""GPU parity: the CUDA path (through the C ABI, include/vsr.h) against the CPU
oracle on identical seeded inputs.  fp64 tolerance: relative L2 <= 1e-10
(BASELINE.json north_star), unless a reference test states a looser bound."""
import math

import numpy as np
import pytest

from conftest import random_psf, random_spectrum, random_volume, rel_err

pytestmark = pytest.mark.gpu
TOL = 1e-10

ODD_EVEN = [(5, 3, 7), (4, 6, 2), (8, 8, 8), (1, 9, 4), (1, 1, 1), (3, 1, 1), (12, 10, 8), (6, 4, 4)]
POW2 = [(2, 2, 2), (4, 4, 4), (16, 8, 4), (32, 32, 32), (64, 64, 64), (128, 8, 16), (2048, 2, 4),
        (1024, 4, 2), (8, 1024, 2), (4, 2, 2048), (512, 16, 4), (256, 256, 4), (64, 32, 128)]


# ------------------------------------------------------------------ FFT engine
@pytest.mark.parametrize("d", ODD_EVEN + POW2)
def test_fft3_complex_vs_numpy(V, O, d):
    rng = np.random.default_rng(hash(d) % 2 ** 32)
    x = random_spectrum(d, rng)
    assert rel_err(V.fft3(x), O.fft3(x)) < 1e-13
    assert rel_err(V.ifft3(x), O.ifft3(x)) < 1e-13


@pytest.mark.parametrize("d", ODD_EVEN + POW2)
def test_fft3_real_and_ifft3_real(V, O, d):
    rng = np.random.default_rng(1 + hash(d) % 2 ** 31)
    x = random_volume(d, rng)
    xh = V.fft3(x)
    assert rel_err(xh, O.fft3(x)) < 1e-13
    back = V.ifft3_real(xh)
    assert rel_err(back, x) < 1e-13
    assert rel_err(V.dft3_unnormalized(x), O.dft3_unnormalized(x)) < 1e-13


def test_fft3_constant_dc(V):
    """test_volume.cpp:44-50."""
    d = (4, 3, 5)
    sp = V.fft3(np.full((5, 3, 4), 0.75))
    assert abs(sp.reshape(-1)[0] - 0.75 * math.sqrt(60)) < 1e-12
    assert np.all(np.abs(sp.reshape(-1)[1:]) < 1e-12)


def test_fft3_dense_dft(V, O):
    """test_volume.cpp:71-81 (sign, scale, axis order)."""
    rng = np.random.default_rng(11)
    d = (4, 3, 2)
    x = random_volume(d, rng)
    assert np.max(np.abs(V.fft3(x).reshape(-1) - O.build_dense_dft(d) @ x.reshape(-1))) < 1e-12


def test_ifft3_real_rejects_nonhermitian(V):
    """test_volume.cpp:83-87."""
    rng = np.random.default_rng(3)
    with pytest.raises(V.NumericError, match="imaginary residue"):
        V.ifft3_real(random_spectrum((4, 4, 4), rng), 1e-8)
    with pytest.raises(V.NumericError):
        V.ifft3_real(random_spectrum((64, 32, 16), rng), 1e-8)


def test_fft_empty_volume_rejected(V):
    with pytest.raises(V.ShapeError):
        V.fft3(np.zeros((0, 4, 4)))


# ------------------------------------------------------------------ operators
@pytest.mark.parametrize("hr,rates", [((8, 8, 8), (2, 2, 2)), ((6, 4, 8), (3, 2, 4)), ((5, 3, 7), (5, 1, 7))])
def test_decimate_ops(V, O, hr, rates):
    rng = np.random.default_rng(6)
    spec = V.DecimationSpec(hr, rates)
    ospec = O.DecimationSpec(hr, rates)
    x = random_volume(hr, rng)
    y = random_volume(spec.lr, rng)
    assert np.array_equal(V.decimate(x, spec), O.decimate(x, ospec))
    assert np.array_equal(V.decimate_adjoint(y, spec), O.decimate_adjoint(y, ospec))


@pytest.mark.parametrize("d", [(5, 4, 3), (32, 8, 16), (1, 7, 2)])
@pytest.mark.parametrize("axis", [0, 1, 2])
def test_diff_ops_bit_exact(V, O, d, axis):
    rng = np.random.default_rng(8)
    x = random_volume(d, rng)
    assert np.array_equal(V.diff_forward(x, axis), O.diff_forward(x, axis))
    assert np.array_equal(V.diff_adjoint(x, axis), O.diff_adjoint(x, axis))


def test_blur_apply(V, O):
    rng = np.random.default_rng(9)
    d = (16, 12, 8)
    psf = random_psf(d, 3, rng)
    x = random_volume(d, rng)
    lam = O.psf_to_spectrum(psf)
    assert rel_err(V.psf_to_spectrum(psf), lam) < 1e-13
    assert rel_err(V.blur_apply(x, lam), O.blur_apply(x, lam)) < TOL
    assert rel_err(V.blur_apply(x, lam, True), O.blur_apply(x, lam, True)) < TOL


# ------------------------------------------------------------------ spectral fold
@pytest.mark.parametrize("hr,rates", [((4, 4, 2), (2, 2, 1)), ((6, 4, 4), (3, 2, 2)), ((16, 16, 16), (4, 4, 4)),
                                      ((32, 16, 8), (2, 2, 4)), ((3, 4, 5), (1, 1, 1))])
def test_fold_primitives(V, O, hr, rates):
    rng = np.random.default_rng(12)
    spec, ospec = V.DecimationSpec(hr, rates), O.DecimationSpec(hr, rates)
    v = random_spectrum(hr, rng)
    lam = random_spectrum(hr, rng)
    w = random_spectrum(spec.lr, rng)
    gw = rng.uniform(0.1, 1.0, V.shape_of(hr))
    assert rel_err(V.alias_fold(v, spec), O.alias_fold(v, ospec)) < 1e-15
    assert np.array_equal(V.alias_expand(w, spec), O.alias_expand(w, ospec))
    f, of = V.FoldedSpectrum(lam, spec), O.FoldedSpectrum(lam, ospec)
    assert rel_err(f.apply(v), of.apply(v)) < 1e-14
    assert rel_err(f.apply_adjoint(w), of.apply_adjoint(w)) < 1e-15
    assert rel_err(f.apply_weighted(v, gw), of.apply_weighted(v, gw)) < 1e-14
    assert rel_err(f.apply_adjoint_weighted(w, gw), of.apply_adjoint_weighted(w, gw)) < 1e-15
    assert rel_err(V.gram_diag(f), O.gram_diag(of)) < 1e-14
    assert rel_err(V.gram_diag_weighted(f, gw), O.gram_diag_weighted(of, gw)) < 1e-14
    if spec.rate() >= 2:
        assert f.block_value(1, 0, 0, 0) == of.block_value(1, 0, 0, 0) or rates[0] == 1
        a = f.apply(v)
        f.swap_blocks_for_fault_injection()
        assert rel_err(f.apply(v), a) > 1e-3
    with pytest.raises(IndexError):
        f.block_value(rates[0], 0, 0, 0)


# ------------------------------------------------------------------ Tikhonov
TIK_CASES = [((8, 8, 8), (2, 2, 2)), ((6, 4, 4), (3, 2, 1)), ((4, 6, 4), (2, 3, 2)), ((8, 4, 4), (2, 1, 2)),
             ((12, 10, 8), (2, 2, 2)), ((32, 32, 32), (4, 4, 4)), ((64, 32, 16), (2, 2, 4)),
             ((16, 16, 16), (1, 1, 1)), ((64, 64, 64), (8, 8, 8)), ((20, 12, 6), (5, 3, 2)),
             # geometries served by the fused fold + axis-3 FFT kernel
             ((128, 64, 256), (2, 2, 2)), ((64, 32, 128), (2, 2, 4)), ((32, 64, 64), (4, 4, 4)),
             ((64, 64, 1024), (2, 2, 2)), ((16, 16, 32), (1, 1, 1))]


@pytest.mark.parametrize("dims,rates", TIK_CASES)
def test_tikhonov_vs_oracle(V, O, dims, rates):
    rng = np.random.default_rng(3)
    spec, ospec = V.DecimationSpec(dims, rates), O.DecimationSpec(dims, rates)
    psf = random_psf(dims, 3, rng)
    lam = O.psf_to_spectrum(psf)
    reg = 0.02 + 0.2 * rng.uniform()
    xbar = random_volume(dims, rng)
    y = random_volume(spec.lr, rng)
    got = V.tikhonov_fast(y, lam, spec, V.TikhonovConfig(reg, xbar))
    want = O.tikhonov_fast(y, lam, ospec, reg, xbar)
    assert rel_err(got, want) < TOL


# Gaussian (separable, compact) PSF + lattice prior xbar = zero_fill_upsample(y):
# the spatial-expansion solve (vsr_tikhonov_spatial).  Tiles wider than the
# volume, non-multiple-of-32 rows, rate 1 axes and anisotropic supports.
SPATIAL_CASES = [((64, 64, 64), (2, 2, 2), (9, 9, 9), (1.0, 1.0, 1.0)),
                 ((32, 48, 64), (2, 2, 4), (5, 7, 9), (1.0, 1.2, 2.0)),
                 ((64, 64, 64), (4, 4, 4), (13, 13, 13), (1.5, 1.5, 1.5)),
                 ((20, 12, 6), (5, 3, 2), (5, 5, 3), (1.0, 0.8, 0.7)),
                 ((8, 8, 8), (2, 2, 2), (3, 3, 3), (1.0, 1.0, 1.0)),
                 ((40, 24, 16), (2, 2, 2), (7, 5, 5), (1.3, 1.1, 0.9)),
                 ((6, 4, 4), (3, 2, 1), (3, 3, 3), (1.0, 1.0, 1.0)),
                 ((128, 32, 64), (2, 1, 2), (15, 15, 9), (1.2, 1.2, 2.0)),
                 ((96, 16, 8), (3, 2, 2), (9, 7, 7), (1.4, 1.0, 1.0)),
                 # z-march expand kernel: 13-tap (DM 7) at rate 2, config-3-like (DM 8, r3 = 4)
                 ((64, 32, 48), (2, 2, 2), (13, 13, 13), (1.5, 1.5, 1.5)),
                 ((32, 16, 40), (2, 2, 4), (15, 15, 21), (1.2, 1.2, 2.0)),
                 # z march with three distinct tap sets (the isotropic cases above share one)
                 ((64, 32, 32), (2, 2, 2), (13, 11, 9), (1.5, 1.3, 1.1)),
                 ((64, 32, 32), (2, 2, 2), (13, 13, 13), (1.5, 1.5, 1.4))]


@pytest.mark.parametrize("dims,rates,ksz,sigma", SPATIAL_CASES)
def test_tikhonov_spatial_vs_oracle(V, O, dims, rates, ksz, sigma):
    rng = np.random.default_rng(11)
    spec, ospec = V.DecimationSpec(dims, rates), O.DecimationSpec(dims, rates)
    lam = O.psf_to_spectrum(O.make_gaussian_psf(ksz, sigma, dims))
    y = random_volume(spec.lr, rng)
    xbar = O.zero_fill_upsample(y, ospec)
    for reg in (1e-3, 0.3):
        op = V.TikhonovOperator(lam, spec, V.TikhonovConfig(reg, xbar))
        assert op.path()["spatial"]
        got = op.solve(y)
        want = O.tikhonov_fast(y, lam, ospec, reg, xbar)
        assert rel_err(got, want) < TOL, (reg, rel_err(got, want))


def test_tikhonov_spatial_only_when_structured(V, O):
    rng = np.random.default_rng(12)
    dims, rates = (16, 16, 16), (2, 2, 2)
    spec, ospec = V.DecimationSpec(dims, rates), O.DecimationSpec(dims, rates)
    y = random_volume(spec.lr, rng)
    gauss = O.psf_to_spectrum(O.make_gaussian_psf((5, 5, 5), (1.0, 1.0, 1.0), dims))
    dense = O.psf_to_spectrum(random_psf(dims, 3, rng))
    lat, full = O.zero_fill_upsample(y, ospec), random_volume(dims, rng)
    cases = {(0, 0): (gauss, lat, True), (0, 1): (gauss, full, False), (1, 0): (dense, lat, False)}
    for (i, j), (lam, xbar, spatial) in cases.items():
        op = V.TikhonovOperator(lam, spec, V.TikhonovConfig(0.05, xbar))
        assert op.path()["spatial"] == spatial, (i, j)
        assert rel_err(op.solve(y), O.tikhonov_fast(y, lam, ospec, 0.05, xbar)) < TOL


def test_tikhonov_spatial_budget_and_determinism(V, O):
    """test_solvers.cpp:141-157 and test_cli.cpp:237-268 on the spatial path."""
    rng = np.random.default_rng(13)
    dims = (64, 64, 64)
    spec, ospec = V.DecimationSpec(dims, (2, 2, 2)), O.DecimationSpec(dims, (2, 2, 2))
    y = random_volume(spec.lr, rng)
    lam = O.psf_to_spectrum(O.make_gaussian_psf((9, 9, 9), (1.0, 1.0, 1.0), dims))
    op = V.TikhonovOperator(lam, spec, V.TikhonovConfig(1e-3, O.zero_fill_upsample(y, ospec)))
    assert op.path()["spatial"]
    V.reset_fft_counters()
    a = op.solve(y)
    assert V.fft_counters() == {"forward": 1, "inverse": 1}
    assert a.tobytes() == op.solve(y).tobytes()
    y2 = y.copy()
    y2[1, 2, 3] = np.inf
    with pytest.raises(V.NumericError, match="non-finite"):
        op.solve(y2)
    assert a.tobytes() == op.solve(y).tobytes()


def test_tikhonov_spatial_new_y_through_graph_replay(V, O):
    """The prior is built from y1 once; y2, y3, y1, y2 are then solved by the
    same operator.  The host API copies each y into the handle's staging
    buffer, so from the second solve on the captured graph replays with new
    contents; the device API is driven with one y buffer rewritten between
    solves (replay) and with a fresh buffer (re-capture).  Every solve must
    match the oracle for ITS y (a cached y-dependent term or a stale graph
    input would fail here)."""
    rng = np.random.default_rng(41)
    dims, rates = (64, 64, 32), (2, 2, 2)
    spec, ospec = V.DecimationSpec(dims, rates), O.DecimationSpec(dims, rates)
    lam = O.psf_to_spectrum(O.make_gaussian_psf((9, 9, 9), (1.0, 1.0, 1.0), dims))
    ys = [random_volume(spec.lr, rng, 0.0, 1.0) for _ in range(3)]
    xbar = O.zero_fill_upsample(ys[0], ospec)
    want = [O.tikhonov_fast(y, lam, ospec, 1e-3, xbar) for y in ys]
    op = V.TikhonovOperator(lam, spec, V.TikhonovConfig(1e-3, xbar))
    assert op.path()["spatial"]
    for i in (1, 2, 0, 1, 1, 2):
        assert rel_err(op.solve(ys[i]), want[i]) < TOL, i
    ctx = V.default_context()
    Nl, N = int(np.prod(spec.lr)), int(np.prod(dims))
    lam_d, xb_d = V.DeviceBuffer(ctx, 16 * N), V.DeviceBuffer(ctx, 8 * N)
    lam_d.upload(np.ascontiguousarray(lam))
    xb_d.upload(xbar)
    dop = V.TikhonovDevice(ctx, spec, lam_d, 1e-3, xb_d)
    assert dop.spatial()
    yb, yb2, xb = V.DeviceBuffer(ctx, 8 * Nl), V.DeviceBuffer(ctx, 8 * Nl), V.DeviceBuffer(ctx, 8 * N)
    out = np.empty(V.shape_of(dims))
    for buf, i in ((yb, 1), (yb, 2), (yb, 0), (yb2, 2), (yb, 1), (yb2, 0)):
        buf.upload(ys[i])
        dop.solve_d(buf, xb)
        dop.check()
        xb.download(out)
        ctx.synchronize()
        assert rel_err(out, want[i]) < TOL, i


def _perturbed_gaussian(O, dims, ksz, sigma, eps, rng):
    """Gaussian kernel times (1 + eps * u), u uniform [-1, 1] per tap: not
    separable once eps exceeds the detector's 1e-13 relative deviation."""
    w = O.make_gaussian_psf(ksz, sigma, ksz)  # origin-wrapped on its own support
    w = np.fft.fftshift(w).reshape(-1)
    w = w * (1.0 + eps * rng.uniform(-1.0, 1.0, w.size))
    return O.make_gaussian_psf(ksz, (0, 0, 0), dims, weights=w)


@pytest.mark.parametrize("eps,spatial", [(1e-12, False), (1e-9, False), (0.0, True)])
def test_tikhonov_near_separable_psf(V, O, eps, spatial):
    """Separability is accepted at a relative deviation <= 1e-13 of Lambda
    from a[f1] b[f2] c[f3].  A Gaussian perturbed tap-wise by 1e-12 or 1e-9
    must fall back to the general (dense Lambda) path; either way the solve
    matches the oracle run on the PERTURBED PSF."""
    rng = np.random.default_rng(42)
    dims, rates = (32, 32, 32), (2, 2, 2)
    spec, ospec = V.DecimationSpec(dims, rates), O.DecimationSpec(dims, rates)
    psf = _perturbed_gaussian(O, dims, (9, 9, 9), (1.2, 1.2, 1.2), eps, rng)
    lam = O.psf_to_spectrum(psf)
    y = random_volume(spec.lr, rng, 0.0, 1.0)
    xbar = O.zero_fill_upsample(y, ospec)
    op = V.TikhonovOperator(lam, spec, V.TikhonovConfig(1e-3, xbar))
    assert op.path()["separable"] == spatial and op.path()["spatial"] == spatial
    assert rel_err(op.solve(y), O.tikhonov_fast(y, lam, ospec, 1e-3, xbar)) < TOL
    cfg = V.TvAdmmConfig(lambda_=2e-3, mu=0.05, max_iters=3, rel_tol=0.0, tau=5e-5)
    xt, _ = V.admm_tv(y, psf, spec, cfg)
    xo, _ = O.admm_tv(y, psf, ospec, lam_tv=2e-3, mu=0.05, max_iters=3, rel_tol=0.0, tau=5e-5)
    assert rel_err(xt, xo) < TOL


@pytest.mark.parametrize("kind", ["cauchy", "wide_gauss", "exp"])
def test_tikhonov_long_tailed_separable_psf(V, O, kind):
    """Separable PSFs whose 1-D factors are long-tailed and fill (almost) the
    whole axis: the spatial expansion keeps every tap above 1e-14 of the
    largest, so it must stay within the parity bound whether it runs or
    falls back."""
    rng = np.random.default_rng(43)
    dims, rates = (48, 32, 40), (2, 2, 2)
    spec, ospec = V.DecimationSpec(dims, rates), O.DecimationSpec(dims, rates)
    ksz = (47, 31, 39)
    prof = []
    for a in range(3):
        t = np.arange(ksz[a]) - ksz[a] // 2
        if kind == "cauchy":
            prof.append(1.0 / (1.0 + (t / 1.5) ** 2))
        elif kind == "wide_gauss":
            prof.append(np.exp(-0.5 * (t / 6.0) ** 2))  # falls below 1e-14 only past the support edge
        else:
            prof.append(np.exp(-np.abs(t) / 0.35))     # crosses 1e-14 at |t| ~ 11: dropped tail taps
    w = (prof[2][:, None, None] * prof[1][None, :, None] * prof[0][None, None, :]).reshape(-1)
    psf = O.make_gaussian_psf(ksz, (0, 0, 0), dims, weights=w)
    lam = O.psf_to_spectrum(psf)
    y = random_volume(spec.lr, rng, 0.0, 1.0)
    xbar = O.zero_fill_upsample(y, ospec)
    for reg in (1e-3, 0.1):
        op = V.TikhonovOperator(lam, spec, V.TikhonovConfig(reg, xbar))
        assert op.path()["separable"]
        assert rel_err(op.solve(y), O.tikhonov_fast(y, lam, ospec, reg, xbar)) < TOL, (kind, reg, op.path())


def test_tikhonov_identity_formula(V):
    """test_solvers.cpp:55-69."""
    rng = np.random.default_rng(1)
    d = (4, 4, 4)
    spec = V.DecimationSpec(d, (1, 1, 1))
    xbar = random_volume(d, rng)
    y = random_volume(d, rng)
    x = V.tikhonov_fast(y, np.ones((4, 4, 4), complex), spec, V.TikhonovConfig(0.35, xbar))
    want = (y + 0.7 * xbar) / 1.7
    assert np.max(np.abs(x - want) / np.abs(want)) < 1e-12


def test_tikhonov_huge_lambda(V, O):
    rng = np.random.default_rng(2)
    d = (8, 8, 8)
    spec = V.DecimationSpec(d, (2, 2, 2))
    lam = O.psf_to_spectrum(random_psf(d, 3, rng))
    xbar = random_volume(d, rng)
    x = V.tikhonov_fast(random_volume(spec.lr, rng), lam, spec, V.TikhonovConfig(1e6, xbar))
    assert rel_err(x, xbar) < 1e-4


def test_tikhonov_errors(V):
    d = (4, 4, 4)
    spec = V.DecimationSpec(d, (1, 1, 1))
    with pytest.raises(ValueError, match="lambda must be positive"):
        V.TikhonovOperator(np.ones((4, 4, 4), complex), spec, V.TikhonovConfig(0.0, np.zeros((4, 4, 4))))
    op = V.TikhonovOperator(np.ones((4, 4, 4), complex), spec, V.TikhonovConfig(0.1, np.zeros((4, 4, 4))))
    with pytest.raises(V.ShapeError):
        op.solve(np.zeros((2, 4, 4)))
    with pytest.raises(V.ShapeError, match="does not divide"):
        V.DecimationSpec((4, 5, 4), (2, 2, 2))


def test_tikhonov_nonfinite_detected(V):
    d = (8, 8, 8)
    spec = V.DecimationSpec(d, (2, 2, 2))
    op = V.TikhonovOperator(np.ones((8, 8, 8), complex), spec, V.TikhonovConfig(0.1, np.zeros((8, 8, 8))))
    y = np.zeros((4, 4, 4))
    y[1, 2, 3] = np.nan
    with pytest.raises(V.NumericError, match="non-finite"):
        op.solve(y)
    # operator stays usable after an error
    assert np.all(np.isfinite(op.solve(np.ones((4, 4, 4)))))


def test_tikhonov_fft_budget(V, O):
    """test_solvers.cpp:141-157: 1 forward + 1 inverse transform per solve."""
    rng = np.random.default_rng(5)
    d = (8, 8, 8)
    spec = V.DecimationSpec(d, (2, 2, 2))
    op = V.TikhonovOperator(O.psf_to_spectrum(random_psf(d, 3, rng)), spec,
                            V.TikhonovConfig(0.1, random_volume(d, rng)))
    V.reset_fft_counters()
    op.solve(random_volume(spec.lr, rng))
    assert V.fft_counters() == {"forward": 1, "inverse": 1}


def test_tikhonov_deterministic(V, O):
    """test_cli.cpp:237-268: byte-identical outputs run to run."""
    rng = np.random.default_rng(6)
    d = (64, 64, 64)
    spec = V.DecimationSpec(d, (2, 2, 2))
    op = V.TikhonovOperator(O.psf_to_spectrum(random_psf(d, 5, rng)), spec,
                            V.TikhonovConfig(1e-3, random_volume(d, rng)))
    y = random_volume(spec.lr, rng)
    a, b = op.solve(y), op.solve(y)
    assert a.tobytes() == b.tobytes()


# ------------------------------------------------------------------ TV pieces
@pytest.mark.parametrize("d", [(4, 4, 4), (16, 8, 32), (5, 3, 7)])
def test_make_gamma(V, O, d):
    assert np.array_equal(V.make_gamma(d, 1e-3), O.make_gamma(d, 1e-3))


def test_make_gamma_errors(V):
    with pytest.raises(V.NumericError, match="zero frequency"):
        V.make_gamma((4, 4, 4), 0.0)
    with pytest.raises(ValueError):
        V.make_gamma((4, 4, 4), -1.0)


def test_tv_shrink(V, O):
    rng = np.random.default_rng(9)
    d = (16, 8, 4)
    nu = [random_volume(d, rng) for _ in range(3)]
    nu[0][0, 0, 0] = nu[1][0, 0, 0] = nu[2][0, 0, 0] = 0.0
    got, want = V.tv_shrink(*nu, 0.4), O.tv_shrink(*nu, 0.4)
    for g, w in zip(got, want):
        assert np.max(np.abs(g - w)) < 1e-15
    one = lambda v: np.full((1, 1, 1), v)
    out = V.tv_shrink(one(3.0), one(0.0), one(0.0), 1.0)
    assert abs(out[0][0, 0, 0] - 2.0) < 1e-12
    with pytest.raises(ValueError):
        V.tv_shrink(one(1.0), one(0.0), one(0.0), -0.5)


@pytest.mark.parametrize("dims,rates,tau", [((8, 8, 8), (2, 2, 2), 1e-6), ((16, 16, 16), (4, 4, 4), 1e-3),
                                            ((32, 16, 8), (2, 2, 4), 1e-3), ((6, 4, 4), (1, 1, 1), 1e-2),
                                            ((12, 10, 8), (2, 2, 2), 1e-3)])
def test_tv_x_update_vs_oracle(V, O, dims, rates, tau):
    rng = np.random.default_rng(11)
    spec, ospec = V.DecimationSpec(dims, rates), O.DecimationSpec(dims, rates)
    lam = O.psf_to_spectrum(random_psf(dims, 3, rng))
    mu = 0.7
    g = O.make_gamma(dims, tau)
    y = random_volume(spec.lr, rng)
    th = O.fft3(_theta(O, dims, rng))
    got = V.tv_x_update(y, V.FoldedSpectrum(lam, spec), lam, spec, mu, th, g)
    want = O.tv_x_update(y, O.FoldedSpectrum(lam, ospec), lam, ospec, mu, th, g)
    assert rel_err(got, want) < TOL


def test_tv_x_update_rejects_bad_gamma(V, O):
    d = (4, 4, 4)
    spec = V.DecimationSpec(d, (2, 2, 2))
    lam = O.psf_to_spectrum(O.make_gaussian_psf((3, 3, 3), (1, 1, 1), d))
    g = O.make_gamma(d, 1e-8)
    g[0, 0, 0] = 0.0
    with pytest.raises(V.NumericError, match="gamma must be strictly positive"):
        V.tv_x_update(np.zeros((2, 2, 2)), V.FoldedSpectrum(lam, spec), lam, spec, 1.0,
                      np.zeros((4, 4, 4), complex), g)


def _theta(O, d, rng):
    th = np.zeros(O.shape_of(d))
    for a in range(3):
        th = th + O.diff_adjoint(random_volume(d, rng), a)
    return th


def test_objective_tv(V, O):
    rng = np.random.default_rng(13)
    for d, rates in [((6, 4, 4), (2, 2, 2)), ((32, 16, 8), (4, 2, 2))]:
        spec, ospec = V.DecimationSpec(d, rates), O.DecimationSpec(d, rates)
        lam = O.psf_to_spectrum(random_psf(d, 3, rng))
        x = random_volume(d, rng)
        y = random_volume(spec.lr, rng)
        got = V.objective_tv(x, y, lam, spec, 0.3)
        want = O.objective_tv(x, y, lam, ospec, 0.3)
        assert abs(got - want) / abs(want) < 1e-12


# ------------------------------------------------------------------ ADMM-TV
TV_CASES = [((8, 8, 8), (2, 2, 2), 6), ((16, 16, 16), (4, 4, 4), 10), ((32, 32, 16), (2, 2, 4), 8),
            ((12, 10, 8), (2, 2, 2), 5), ((64, 64, 64), (4, 4, 4), 12), ((40, 24, 16), (2, 2, 2), 5),
            ((32, 32, 64), (2, 2, 4), 6), ((64, 32, 128), (2, 2, 2), 4), ((32, 32, 32), (1, 1, 1), 4),
            # half-spectrum mirror pairing: nl not a power of two, and sl = 4 (self-mirror planes 0, 2)
            ((64, 48, 32), (4, 4, 4), 5), ((64, 64, 16), (4, 4, 4), 5), ((128, 64, 32), (4, 4, 2), 4),
            # 1024-point axis-3 lines (paired real passes with 16-column tiles, as at config 4)
            ((64, 8, 1024), (2, 2, 2), 3),
            # 1024-point axis-2 lines (the wide strided pass, as at config 4)
            ((16, 1024, 8), (2, 2, 2), 3),
            # the pipelined half-spectrum sandwich (sandwich.cu) at the configs' row geometries:
            # (m, dc*ds, dr) = (256, 16, 4) config 2, (512, 8, 2) config 3, (1024, 4, 2) config 4
            ((256, 32, 32), (4, 4, 4), 3), ((512, 16, 32), (2, 2, 4), 3), ((1024, 16, 8), (2, 2, 2), 3),
            ((128, 32, 32), (2, 2, 2), 3)]


@pytest.mark.parametrize("dims,rates,iters", TV_CASES)
def test_admm_tv_vs_oracle(V, O, dims, rates, iters):
    """Parity protocol: explicit tau = 1e-3 * mu, rel_tol = 0."""
    rng = np.random.default_rng(21)
    spec, ospec = V.DecimationSpec(dims, rates), O.DecimationSpec(dims, rates)
    psf = O.make_gaussian_psf(tuple(min(5, x - (1 - x % 2)) for x in dims), (1.5, 1.5, 1.5), dims)
    y = random_volume(spec.lr, rng, 0.0, 1.0)
    mu, lam_tv = 0.05, 2e-3
    for init, x0 in [(V.INIT_ZERO, None), (V.INIT_UPSAMPLED, None),
                     (V.INIT_PROVIDED, random_volume(dims, rng, 0.0, 1.0))]:
        cfg = V.TvAdmmConfig(lambda_=lam_tv, mu=mu, max_iters=iters, rel_tol=0.0, tau=1e-3 * mu,
                             init=init, init_volume=x0)
        got, rep = V.admm_tv(y, psf, spec, cfg)
        want, orep = O.admm_tv(y, psf, ospec, lam_tv=lam_tv, mu=mu, max_iters=iters, rel_tol=0.0,
                               tau=1e-3 * mu, init=init, init_volume=x0)
        assert rel_err(got, want) < TOL
        assert rep.iterations == orep.iterations == iters
        assert abs(rep.initial_objective - orep.initial_objective) <= 1e-10 * abs(orep.initial_objective)
        assert rel_err(rep.objective, orep.objective) < 1e-10
        assert rel_err(rep.primal_residual, orep.primal_residual) < 1e-9


def test_admm_tv_rel_tol_stop(V, O):
    rng = np.random.default_rng(22)
    d = (16, 16, 16)
    spec, ospec = V.DecimationSpec(d, (2, 2, 2)), O.DecimationSpec(d, (2, 2, 2))
    psf = O.make_gaussian_psf((5, 5, 5), (1.0, 1.0, 1.0), d)
    y = random_volume(spec.lr, rng, 0.0, 1.0)
    cfg = V.TvAdmmConfig(lambda_=2e-3, mu=0.05, max_iters=200, rel_tol=1e-3, tau=5e-5)
    got, rep = V.admm_tv(y, psf, spec, cfg)
    want, orep = O.admm_tv(y, psf, ospec, lam_tv=2e-3, mu=0.05, max_iters=200, rel_tol=1e-3, tau=5e-5)
    assert rep.iterations == orep.iterations < 200
    assert rel_err(got, want) < TOL


def test_admm_tv_default_tau_dc_split(V, O):
    """At the reference default tau = 1e-8 mu the DC bin is ill-conditioned
    (SURVEY Appendix B): the mean-free part must still match to 1e-10; the
    mean is reported against the eps/(tau mu d) amplification bound."""
    rng = np.random.default_rng(23)
    d = (32, 32, 32)
    spec, ospec = V.DecimationSpec(d, (4, 4, 4)), O.DecimationSpec(d, (4, 4, 4))
    psf = O.make_gaussian_psf((5, 5, 5), (1.5, 1.5, 1.5), d)
    y = random_volume(spec.lr, rng, 0.0, 1.0)
    got, _ = V.admm_tv(y, psf, spec, V.TvAdmmConfig(lambda_=2e-3, mu=0.05, max_iters=5, rel_tol=0.0))
    want, _ = O.admm_tv(y, psf, ospec, lam_tv=2e-3, mu=0.05, max_iters=5, rel_tol=0.0)
    assert rel_err(got - got.mean(), want - want.mean()) < TOL
    bound = 1e-16 / (1e-8 * 0.05 * 0.05 * 64) * 100
    assert abs(got.mean() - want.mean()) / abs(want.mean()) < bound


def test_admm_tv_validates(V):
    d = (8, 8, 8)
    spec = V.DecimationSpec(d, (2, 2, 2))
    psf = V.make_gaussian_psf((3, 3, 3), (1, 1, 1), d)
    y = np.full((4, 4, 4), 0.5)
    V.admm_tv(y, psf, spec, V.TvAdmmConfig(max_iters=2, init=V.INIT_UPSAMPLED))
    with pytest.raises(V.ShapeError):
        V.admm_tv(y, psf, spec, V.TvAdmmConfig(max_iters=2, init=V.INIT_PROVIDED, init_volume=np.zeros((4, 4, 4))))
    for bad in (V.TvAdmmConfig(lambda_=-1.0), V.TvAdmmConfig(mu=0.0), V.TvAdmmConfig(max_iters=0)):
        with pytest.raises(ValueError):
            V.admm_tv(y, psf, spec, bad)
    with pytest.raises(V.NumericError, match="zero frequency"):
        V.admm_tv(y, psf, spec, V.TvAdmmConfig(max_iters=2, tau=0.0))


def test_admm_tv_deterministic(V):
    rng = np.random.default_rng(24)
    d = (32, 32, 32)
    spec = V.DecimationSpec(d, (2, 2, 2))
    psf = V.make_gaussian_psf((5, 5, 5), (1.5, 1.5, 1.5), d)
    y = random_volume(spec.lr, rng, 0.0, 1.0)
    cfg = V.TvAdmmConfig(lambda_=2e-3, mu=0.05, max_iters=6, rel_tol=0.0)
    a, ra = V.admm_tv(y, psf, spec, cfg)
    b, rb = V.admm_tv(y, psf, spec, cfg)
    assert a.tobytes() == b.tobytes()
    assert ra.objective == rb.objective and ra.primal_residual == rb.primal_residual


# ------------------------------------------------------------------ opt-in variants
# Every env-selected kernel variant (read once per process) runs in a fresh
# interpreter against the oracle: Tikhonov spatial path with the full-spectrum
# LR stage / the general FFT path / no graphs, and the TV iteration on the full
# spectrum; the fold fusion choices (none, axis 1, axis 3), the dense-Lambda
# fold (no separable tables) and the full-spectrum prior (no lattice form).
_VARIANT_SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, {root!r}); sys.path.insert(0, {root!r} + '/oracle'); sys.path.insert(0, {root!r} + '/tests')
from paper_2010_15491_b200 import volsr as V
import volsr_oracle as O
from conftest import rel_err
rng = np.random.default_rng(21)
dims, rates = {dims}, {rates}
spec, ospec = V.DecimationSpec(dims, rates), O.DecimationSpec(dims, rates)
psf = O.make_gaussian_psf((5, 5, 5), (1.2, 1.2, 1.2), dims)
lam = O.psf_to_spectrum(psf)
y = rng.uniform(0, 1, V.shape_of(spec.lr))
xbar = O.zero_fill_upsample(y, ospec)
op = V.TikhonovOperator(lam, spec, V.TikhonovConfig(0.01, xbar))
want = O.tikhonov_fast(y, lam, ospec, 0.01, xbar)
for _ in range(3):  # eager, captured, replayed
    e = rel_err(op.solve(y), want)
    assert e < 1e-10, ("tikhonov", e)
cfg = V.TvAdmmConfig(lambda_=2e-3, mu=0.05, max_iters=3, rel_tol=0.0, tau=5e-5)
xt, _ = V.admm_tv(y, psf, spec, cfg)
xo, _ = O.admm_tv(y, psf, ospec, lam_tv=2e-3, mu=0.05, max_iters=3, rel_tol=0.0, tau=5e-5)
e2 = rel_err(xt, xo)
assert e2 < 1e-10, ("admm_tv", e2)
print("ok", op.path())
"""


@pytest.mark.parametrize("env,dims,rates", [
    ({"VSR_NO_HALF": "1"}, (64, 64, 32), (2, 2, 2)),
    ({"VSR_TV_FULL": "1"}, (64, 64, 64), (4, 4, 4)),
    ({"VSR_NO_SPATIAL": "1"}, (64, 64, 32), (2, 2, 2)),
    ({"VSR_NO_GRAPH": "1"}, (64, 64, 32), (2, 2, 2)),
    ({"VSR_NO_FUSE": "1"}, (64, 64, 64), (4, 4, 4)),
    ({"VSR_FUSE_AXIS": "1"}, (64, 64, 32), (2, 2, 2)),
    ({"VSR_FUSE_AXIS": "3"}, (64, 64, 64), (4, 4, 4)),
    ({"VSR_FUSE_AXIS": "0"}, (64, 64, 32), (2, 2, 2)),
    ({"VSR_NO_SEP": "1"}, (64, 64, 64), (4, 4, 4)),
    ({"VSR_NO_LATTICE": "1"}, (64, 64, 32), (2, 2, 2)),
    ({"VSR_NO_MARCH": "1"}, (64, 64, 32), (2, 2, 2)),
    ({"VSR_MARCH_ZC": "5"}, (64, 64, 32), (2, 2, 2)),
    ({"VSR_MARCH_ZC": "1"}, (64, 64, 32), (2, 2, 2)),
    ({"VSR_MARCH_CY": "4"}, (64, 64, 32), (2, 2, 2)),
    ({"VSR_MARCH_ISO": "0"}, (64, 64, 32), (2, 2, 2)),
    ({"VSR_NO_PIPE": "1"}, (256, 32, 32), (4, 4, 4)),
    ({"VSR_NO_PIPE": "1"}, (512, 16, 32), (2, 2, 4)),
    # 1024-point axis-2 / axis-3 lines on the narrow one-tile-per-CTA passes (default: the wide persistent ones)
    ({"VSR_NO_WIDE": "1"}, (64, 8, 1024), (2, 2, 2)),
    ({"VSR_NO_WIDE": "1"}, (16, 1024, 8), (2, 2, 2)),
])
def test_env_variants(env, dims, rates):
    import os
    import subprocess
    import sys
    from pathlib import Path
    root = str(Path(__file__).resolve().parent.parent)
    code = _VARIANT_SCRIPT.format(root=root, dims=dims, rates=rates)
    r = subprocess.run([sys.executable, "-c", code], env={**os.environ, **env}, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr


# ------------------------------------------------------------------ admm_l2l2
L2_CASES = [((8, 8, 8), (2, 2, 2), 6), ((12, 10, 8), (2, 2, 2), 5), ((16, 16, 16), (4, 4, 4), 8),
            ((32, 16, 8), (2, 1, 2), 5), ((64, 64, 32), (2, 2, 2), 4)]


@pytest.mark.parametrize("dims,rates,iters", L2_CASES)
def test_admm_l2l2_vs_oracle(V, O, dims, rates, iters):
    """solvers.cpp:95-189, fixed iteration count (rel_tol = 0)."""
    rng = np.random.default_rng(31)
    spec, ospec = V.DecimationSpec(dims, rates), O.DecimationSpec(dims, rates)
    lam = O.psf_to_spectrum(random_psf(dims, 3, rng))
    xbar = random_volume(dims, rng)
    y = random_volume(spec.lr, rng)
    x, rep = V.admm_l2l2(y, lam, spec, V.TikhonovConfig(0.05, xbar), iters, V.AdmmL2Options(mu=0.3, rel_tol=0.0))
    xo, orep = O.admm_l2l2(y, lam, ospec, 0.05, xbar, iters, mu=0.3, rel_tol=0.0)
    assert rep.iterations == orep.iterations == iters
    assert rel_err(x, xo) < TOL
    assert abs(rep.initial_objective - orep.initial_objective) <= 1e-12 * abs(orep.initial_objective)
    np.testing.assert_allclose(rep.objective, orep.objective, rtol=1e-10)
    np.testing.assert_allclose(rep.primal_residual, orep.primal_residual, rtol=1e-9)


def test_admm_l2l2_fixed_point(V, O):
    """test_solvers.cpp:194-222: warm start at the exact minimizer stays there."""
    rng = np.random.default_rng(7)
    d = (8, 8, 8)
    spec, ospec = V.DecimationSpec(d, (2, 2, 2)), O.DecimationSpec(d, (2, 2, 2))
    lam = O.psf_to_spectrum(random_psf(d, 3, rng))
    xbar = random_volume(d, rng)
    y = random_volume(spec.lr, rng)
    xstar = O.tikhonov_fast(y, lam, ospec, 0.05, xbar)
    v = O.blur_apply(xstar, lam)
    r = O.decimate(v, ospec) - y
    dual = O.decimate_adjoint(r, ospec) / 0.3
    x1, rep = V.admm_l2l2(y, lam, spec, V.TikhonovConfig(0.05, xbar), 1,
                          V.AdmmL2Options(mu=0.3, rel_tol=0.0, warm_start=(xstar, v, dual)))
    assert rep.iterations == 1
    assert rel_err(x1, xstar) < TOL


def test_admm_l2l2_converges_to_closed_form(V, O):
    """test_solvers.cpp:224-260: converges (rel_tol stop) to the tikhonov_fast minimizer."""
    rng = np.random.default_rng(8)
    d = (16, 16, 16)
    spec, ospec = V.DecimationSpec(d, (2, 2, 2)), O.DecimationSpec(d, (2, 2, 2))
    lam = O.psf_to_spectrum(O.make_gaussian_psf((5, 5, 5), (1.5, 1.5, 1.5), d))
    y = random_volume(spec.lr, rng, 0.0, 1.0)
    xbar = O.zero_fill_upsample(y, ospec)
    cfg = V.TikhonovConfig(0.01, xbar)
    fast = V.tikhonov_fast(y, lam, spec, cfg)
    it, rep = V.admm_l2l2(y, lam, spec, cfg, 4000, V.AdmmL2Options(mu=0.1, rel_tol=1e-11))
    assert rep.iterations < 4000

    def objective(x):
        z = O.decimate(O.blur_apply(x, lam), ospec)
        return 0.5 * float(np.sum((y - z) ** 2)) + 0.01 * float(np.sum((x - xbar) ** 2))

    assert abs(rep.objective[-1] - objective(fast)) <= 1e-8 * objective(fast)
    assert rel_err(it, fast) < 1e-5


def test_admm_l2l2_errors_and_determinism(V):
    d = (8, 8, 8)
    spec = V.DecimationSpec(d, (2, 2, 2))
    lam = np.ones(V.shape_of(d), complex)
    xbar = np.zeros(V.shape_of(d))
    y = np.ones(V.shape_of(spec.lr))
    with pytest.raises(ValueError, match="mu must be positive"):
        V.admm_l2l2(y, lam, spec, V.TikhonovConfig(0.1, xbar), 3, V.AdmmL2Options(mu=0.0))
    with pytest.raises(ValueError, match="max_iters"):
        V.admm_l2l2(y, lam, spec, V.TikhonovConfig(0.1, xbar), 0)
    with pytest.raises(V.ShapeError):
        V.admm_l2l2(np.ones((2, 2, 2)), lam, spec, V.TikhonovConfig(0.1, xbar), 3)
    with pytest.raises(V.ShapeError, match="warm start"):
        V.admm_l2l2(y, lam, spec, V.TikhonovConfig(0.1, xbar), 3,
                    V.AdmmL2Options(warm_start=(xbar, xbar, np.zeros((2, 2, 2)))))
    a, _ = V.admm_l2l2(y, lam, spec, V.TikhonovConfig(0.1, xbar), 5, V.AdmmL2Options(rel_tol=0.0))
    b, _ = V.admm_l2l2(y, lam, spec, V.TikhonovConfig(0.1, xbar), 5, V.AdmmL2Options(rel_tol=0.0))
    assert a.tobytes() == b.tobytes()
