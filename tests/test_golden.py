"""Golden vectors produced by the REFERENCE itself (oracle/_ref: the reference
volsr sources compiled with the FFTW3/Eigen shims; tools/make_golden.py).

CPU tests pin the numpy oracle to them; GPU tests check the CUDA path
through the C ABI against the same vectors."""
from pathlib import Path

import numpy as np
import pytest

from conftest import rel_err

G = Path(__file__).resolve().parent / "golden"


def load(name):
    return dict(np.load(G / f"{name}.npz"))


def tup(a):
    return tuple(int(v) for v in a)


# ------------------------------------------------------------------ oracle pins
def test_oracle_fft_golden(O):
    g = load("fft")
    assert rel_err(O.fft3(g["xr"]), g["fr"]) < 1e-14
    assert rel_err(O.fft3(g["xc"]), g["fc"]) < 1e-14
    assert rel_err(O.fft3(g["xr2"]), g["fr2"]) < 1e-14
    assert rel_err(g["back2"], g["xr2"]) < 1e-14


def test_oracle_config0_golden(O):
    g = load("config0_tikhonov")
    hr, rates = tup(g["hr"]), tup(g["rates"])
    spec = O.DecimationSpec(hr, rates)
    psf = O.make_gaussian_psf(tup(g["psf_size"]), tuple(g["psf_sigma"]), hr)
    xbar = O.zero_fill_upsample(g["y"], spec)
    x = O.tikhonov_fast(g["y"], O.psf_to_spectrum(psf), spec, float(g["reg"]), xbar)
    assert rel_err(x, g["x"]) < 1e-13


def test_oracle_tikhonov_shapes_golden(O):
    g = load("tikhonov_shapes")
    for i in range(3):
        hr, rates = tup(g[f"c{i}_hr"]), tup(g[f"c{i}_rates"])
        spec = O.DecimationSpec(hr, rates)
        x = O.tikhonov_fast(g[f"c{i}_y"], O.psf_to_spectrum(g[f"c{i}_psf"]), spec, float(g[f"c{i}_reg"]),
                            g[f"c{i}_xbar"])
        assert rel_err(x, g[f"c{i}_x"]) < 1e-13


def test_oracle_tv_x_update_golden(O):
    g = load("tv_x_update")
    hr, rates = tup(g["hr"]), tup(g["rates"])
    spec = O.DecimationSpec(hr, rates)
    lam = O.psf_to_spectrum(g["psf"])
    gam = O.make_gamma(hr, float(g["tau"]))
    assert np.array_equal(gam, g["gamma"])
    x = O.tv_x_update(g["y"], O.FoldedSpectrum(lam, spec), lam, spec, float(g["mu"]), g["theta_hat"], gam)
    assert rel_err(x, g["x"]) < 1e-12


@pytest.mark.parametrize("name", ["config2_tv_32", "config3_tv_32"])
def test_oracle_admm_tv_golden(O, name):
    g = load(name)
    hr, rates = tup(g["hr"]), tup(g["rates"])
    spec = O.DecimationSpec(hr, rates)
    x0 = g.get("x0")
    x, rep = O.admm_tv(g["y"], g["psf"], spec, lam_tv=float(g["lam_tv"]), mu=float(g["mu"]),
                       max_iters=int(g["iters"]), rel_tol=0.0, tau=float(g["tau"]),
                       init=O.INIT_PROVIDED if x0 is not None else O.INIT_ZERO, init_volume=x0)
    assert rel_err(x, g["x"]) < 1e-11
    assert rel_err(rep.objective, g["objective"]) < 1e-12
    assert rel_err(rep.primal_residual, g["primal_residual"]) < 1e-11
    assert abs(rep.initial_objective - float(g["initial_objective"])) < 1e-12 * abs(float(g["initial_objective"]))


def test_oracle_objective_golden(O):
    g = load("objective_tv")
    hr, rates = tup(g["hr"]), tup(g["rates"])
    v = O.objective_tv(g["x"], g["y"], O.psf_to_spectrum(g["psf"]), O.DecimationSpec(hr, rates), float(g["w"]))
    assert abs(v - float(g["value"])) < 1e-12 * abs(float(g["value"]))


# ------------------------------------------------------------------ GPU vs golden
@pytest.mark.gpu
def test_gpu_fft_golden(V):
    g = load("fft")
    assert rel_err(V.fft3(g["xr"]), g["fr"]) < 1e-13
    assert rel_err(V.fft3(g["xc"]), g["fc"]) < 1e-13
    assert rel_err(V.fft3(g["xr2"]), g["fr2"]) < 1e-13
    assert rel_err(V.ifft3_real(g["fr2"]), g["back2"]) < 1e-13


@pytest.mark.gpu
def test_gpu_config0_golden(V):
    """BASELINE configs[0] at full size against the reference's own output."""
    g = load("config0_tikhonov")
    hr, rates = tup(g["hr"]), tup(g["rates"])
    spec = V.DecimationSpec(hr, rates)
    psf = V.make_gaussian_psf(tup(g["psf_size"]), tuple(g["psf_sigma"]), hr)
    xbar = V.zero_fill_upsample(g["y"], spec)
    x = V.tikhonov_fast(g["y"], V.psf_to_spectrum(psf), spec, V.TikhonovConfig(float(g["reg"]), xbar))
    assert rel_err(x, g["x"]) < 1e-10


@pytest.mark.gpu
def test_gpu_tikhonov_shapes_golden(V):
    g = load("tikhonov_shapes")
    for i in range(3):
        hr, rates = tup(g[f"c{i}_hr"]), tup(g[f"c{i}_rates"])
        spec = V.DecimationSpec(hr, rates)
        x = V.tikhonov_fast(g[f"c{i}_y"], V.psf_to_spectrum(g[f"c{i}_psf"]), spec,
                            V.TikhonovConfig(float(g[f"c{i}_reg"]), g[f"c{i}_xbar"]))
        assert rel_err(x, g[f"c{i}_x"]) < 1e-10


@pytest.mark.gpu
def test_gpu_tv_x_update_golden(V):
    g = load("tv_x_update")
    hr, rates = tup(g["hr"]), tup(g["rates"])
    spec = V.DecimationSpec(hr, rates)
    lam = V.psf_to_spectrum(g["psf"])
    gam = V.make_gamma(hr, float(g["tau"]))
    assert np.array_equal(gam, g["gamma"])
    x = V.tv_x_update(g["y"], V.FoldedSpectrum(lam, spec), lam, spec, float(g["mu"]), g["theta_hat"], gam)
    assert rel_err(x, g["x"]) < 1e-10


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["config2_tv_32", "config3_tv_32"])
def test_gpu_admm_tv_golden(V, name):
    g = load(name)
    hr, rates = tup(g["hr"]), tup(g["rates"])
    spec = V.DecimationSpec(hr, rates)
    x0 = g.get("x0")
    cfg = V.TvAdmmConfig(lambda_=float(g["lam_tv"]), mu=float(g["mu"]), max_iters=int(g["iters"]), rel_tol=0.0,
                         tau=float(g["tau"]), init=V.INIT_PROVIDED if x0 is not None else V.INIT_ZERO,
                         init_volume=x0)
    x, rep = V.admm_tv(g["y"], g["psf"], spec, cfg)
    assert rel_err(x, g["x"]) < 1e-10
    assert rel_err(rep.objective, g["objective"]) < 1e-10
    assert rel_err(rep.primal_residual, g["primal_residual"]) < 1e-9
    assert abs(rep.initial_objective - float(g["initial_objective"])) < 1e-10 * abs(float(g["initial_objective"]))


@pytest.mark.gpu
def test_gpu_objective_golden(V):
    g = load("objective_tv")
    hr, rates = tup(g["hr"]), tup(g["rates"])
    v = V.objective_tv(g["x"], g["y"], V.psf_to_spectrum(g["psf"]), V.DecimationSpec(hr, rates), float(g["w"]))
    assert abs(v - float(g["value"])) < 1e-12 * abs(float(g["value"]))


# ------------------------------------------------------------------ admm_l2l2
def _l2_cases():
    g = load("admm_l2l2")
    for i in range(2):
        yield (tup(g[f"c{i}_hr"]), tup(g[f"c{i}_rates"]), int(g[f"c{i}_iters"]), g[f"c{i}_lam"], g[f"c{i}_xbar"],
               g[f"c{i}_y"], g[f"c{i}_x"], g[f"c{i}_objective"], g[f"c{i}_residual"], float(g[f"c{i}_init_obj"]))


def test_oracle_admm_l2l2_golden(O):
    for hr, rates, it, lam, xbar, y, x, obj, res, init in _l2_cases():
        xo, rep = O.admm_l2l2(y, lam, O.DecimationSpec(hr, rates), 0.05, xbar, it, mu=0.3, rel_tol=0.0)
        assert rel_err(xo, x) < 1e-13
        np.testing.assert_allclose(rep.objective, obj, rtol=1e-13)
        np.testing.assert_allclose(rep.primal_residual, res, rtol=1e-12)
        assert abs(rep.initial_objective - init) <= 1e-13 * abs(init)


@pytest.mark.gpu
def test_gpu_admm_l2l2_golden(V):
    for hr, rates, it, lam, xbar, y, x, obj, res, init in _l2_cases():
        xg, rep = V.admm_l2l2(y, lam, V.DecimationSpec(hr, rates), V.TikhonovConfig(0.05, xbar), it,
                              V.AdmmL2Options(mu=0.3, rel_tol=0.0))
        assert rep.iterations == it
        assert rel_err(xg, x) < 1e-10
        np.testing.assert_allclose(rep.objective, obj, rtol=1e-10)
        np.testing.assert_allclose(rep.primal_residual, res, rtol=1e-9)
        assert abs(rep.initial_objective - init) <= 1e-10 * abs(init)
