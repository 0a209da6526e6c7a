"""fp32 mode (BASELINE north_star: relative L2 <= 1e-5 and PSNR within 0.01 dB
of the fp64 result, which is itself pinned to the reference at <= 1e-10).

ADMM-TV with TvAdmmConfig.precision = "f32": the iteration state in fp32 and
the half-spectrum transforms in fp32 arithmetic; the fold stays fp64 because
its Woodbury form cancels g_b against Gamma_b conj(Lambda_b) w, amplifying
rounding by ~Gamma_b |Lambda_b|^2 / (mu d) (1/tau at DC).  The
cases are the BASELINE configs' recipes (synth.py) on grids with the configs'
row geometries (m, dc*ds, dr) = (256, 16, 4), (512, 8, 2), (1024, 4, 2).

Tikhonov: TikhonovOperator.solve_f32 on the spatial path (fp64 LR stage,
fp32 expansion and x).  The default-tau TV cases exercise the DC bin."""
import numpy as np
import pytest

from conftest import rel_err
from paper_2010_15491_b200 import synth

pytestmark = pytest.mark.gpu

FP32_TOL = 1e-5
PSNR_TOL = 0.01


def _psnr(truth, x):
    peak = float(np.max(truth))
    return 10.0 * np.log10(peak * peak / float(np.mean((truth - x) ** 2)))


CASES = [(2, (256, 64, 64), 20), (3, (512, 64, 64), 20), (4, (1024, 32, 16), 10)]


@pytest.mark.parametrize("cfg_idx,hr,iters", CASES)
@pytest.mark.parametrize("tau", ["parity", "default"])
def test_admm_tv_fp32_vs_fp64(V, cfg_idx, hr, iters, tau):
    cfg = synth.scaled(synth.CONFIGS[cfg_idx], hr)
    inp = synth.make_inputs(cfg)
    spec = V.DecimationSpec(cfg.hr, cfg.rates)
    t = 1e-3 * cfg.tv_mu if tau == "parity" else None  # default: 1e-8 mu (solvers.cpp:332)
    out = {}
    for prec in ("f64", "f32"):
        c = V.TvAdmmConfig(lambda_=cfg.tv_lambda, mu=cfg.tv_mu, max_iters=iters, rel_tol=0.0, tau=t,
                           init=V.INIT_UPSAMPLED, precision=prec)
        out[prec] = V.admm_tv(inp.y, inp.psf, spec, c)
    (x64, r64), (x32, r32) = out["f64"], out["f32"]
    assert x32.dtype == np.float64 and r32.iterations == r64.iterations == iters
    e = rel_err(x32, x64)
    dp = abs(_psnr(inp.truth, x32) - _psnr(inp.truth, x64))
    print(f"config {cfg_idx} {hr} tau={tau}: rel L2 {e:.2e}, PSNR gap {dp:.2e} dB")
    assert e <= FP32_TOL
    assert dp < PSNR_TOL
    assert rel_err(r32.objective, r64.objective) <= FP32_TOL
    assert abs(r32.initial_objective - r64.initial_objective) <= 1e-6 * abs(r64.initial_objective)


def test_admm_tv_fp32_vs_oracle(V, O):
    """The fp32 result against the CPU oracle directly (the fp64 GPU path pins the rest)."""
    rng = np.random.default_rng(5)
    hr, rates = (256, 32, 32), (4, 4, 4)
    spec, ospec = V.DecimationSpec(hr, rates), O.DecimationSpec(hr, rates)
    psf = O.make_gaussian_psf((5, 5, 5), (1.5, 1.5, 1.5), hr)
    y = rng.uniform(0, 1, (hr[2] // 4, hr[1] // 4, hr[0] // 4))
    c = V.TvAdmmConfig(lambda_=2e-3, mu=0.05, max_iters=6, rel_tol=0.0, tau=5e-5, precision="f32")
    x, rep = V.admm_tv(y, psf, spec, c)
    want, wrep = O.admm_tv(y, psf, ospec, lam_tv=2e-3, mu=0.05, max_iters=6, rel_tol=0.0, tau=5e-5)
    assert rel_err(x, want) <= FP32_TOL
    assert rel_err(rep.objective, wrep.objective) <= FP32_TOL


def test_admm_tv_fp32_rel_tol_and_device_handle(V):
    cfg = synth.scaled(synth.CONFIGS[2], (256, 64, 64))
    inp = synth.make_inputs(cfg)
    spec = V.DecimationSpec(cfg.hr, cfg.rates)
    c64 = V.TvAdmmConfig(lambda_=2e-3, mu=0.05, max_iters=60, rel_tol=2e-2, tau=5e-5)
    c32 = V.TvAdmmConfig(lambda_=2e-3, mu=0.05, max_iters=60, rel_tol=2e-2, tau=5e-5, precision="f32")
    x64, r64 = V.admm_tv(inp.y, inp.psf, spec, c64)
    x32, r32 = V.admm_tv(inp.y, inp.psf, spec, c32)
    assert r32.iterations == r64.iterations < 60  # the same stop iteration (solvers.cpp:405)
    assert rel_err(x32, x64) <= FP32_TOL


def test_fp32_mode_rejections(V, O):
    hr, rates = (256, 32, 32), (4, 4, 4)
    spec = V.DecimationSpec(hr, rates)
    rng = np.random.default_rng(1)
    y = rng.uniform(0, 1, (8, 8, 64))
    # a non-separable PSF spectrum: no fp32 route
    w = rng.uniform(0.0, 1.0, 27)
    psf = O.make_gaussian_psf((3, 3, 3), (0, 0, 0), hr, weights=w)
    c = V.TvAdmmConfig(lambda_=2e-3, mu=0.05, max_iters=2, rel_tol=0.0, precision="f32")
    with pytest.raises(ValueError, match="fp32 mode"):
        V.admm_tv(y, psf, spec, c)
    with pytest.raises(ValueError, match="precision"):
        V.admm_tv(y, O.make_gaussian_psf((5, 5, 5), (1, 1, 1), hr), spec,
                  V.TvAdmmConfig(lambda_=2e-3, mu=0.05, max_iters=2, precision="f16"))


# ------------------------------------------------------------------ Tikhonov
TIK_CASES = [(0, (64, 64, 64)), (1, (256, 256, 256)), (1, (256, 128, 64)), (3, (128, 128, 64))]


@pytest.mark.parametrize("cfg_idx,hr", TIK_CASES)
def test_tikhonov_fp32_vs_fp64(V, cfg_idx, hr):
    """TikhonovOperator::solve_f32 (spatial path: fp64 LR stage, fp32 expansion)
    against the fp64 solve, on the configs' recipes; config 3's rates (2, 2, 4)
    exercise the R3 = 4 expansion."""
    cfg = synth.scaled(synth.CONFIGS[cfg_idx], hr)
    inp = synth.make_inputs(cfg)
    spec = V.DecimationSpec(cfg.hr, cfg.rates)
    lam = V.psf_to_spectrum(inp.psf)
    op = V.TikhonovOperator(lam, spec, V.TikhonovConfig(cfg.reg, V.zero_fill_upsample(inp.y, spec)))
    assert op.fp32_ok()
    x64 = op.solve(inp.y)
    x32 = op.solve_f32(inp.y)
    assert x32.dtype == np.float32
    e = rel_err(x32.astype(np.float64), x64)
    dp = abs(_psnr(inp.truth, x32.astype(np.float64)) - _psnr(inp.truth, x64))
    print(f"tikhonov config {cfg_idx} {hr}: rel L2 {e:.2e}, PSNR gap {dp:.2e} dB")
    assert e <= FP32_TOL and dp < PSNR_TOL
    # graph replay of fp32 solves on new y, interleaved with fp64 solves
    rng = np.random.default_rng(3)
    for _ in range(3):
        y2 = inp.y * rng.uniform(0.5, 1.5)
        assert rel_err(op.solve_f32(y2).astype(np.float64), op.solve(y2)) <= FP32_TOL
    op.close()


def test_tikhonov_fp32_rejects_general_path(V):
    rng = np.random.default_rng(2)
    hr, rates = (64, 64, 32), (2, 2, 2)
    spec = V.DecimationSpec(hr, rates)
    psf = V.make_gaussian_psf((5, 5, 5), (1.2, 1.2, 1.2), hr)
    xbar = rng.uniform(0, 1, V.shape_of(hr))  # not on the decimation lattice: no spatial path
    op = V.TikhonovOperator(V.psf_to_spectrum(psf), spec, V.TikhonovConfig(1e-3, xbar))
    assert not op.fp32_ok()
    with pytest.raises(ValueError, match="fp32 mode"):
        op.solve_f32(rng.uniform(0, 1, V.shape_of(spec.lr)))
    op.close()


# ------------------------------------------------------------------ full size
@pytest.mark.parametrize("cfg_idx", [1, 2, 3])
def test_fp32_full_size_configs(V, cfg_idx):
    """The BASELINE configs at full size and full iteration counts: fp32 mode
    against the fp64 path (itself pinned to the reference binary at full size,
    profiles/r02_fullsize_parity.md)."""
    cfg = synth.CONFIGS[cfg_idx]
    inp = synth.make_inputs(cfg)
    spec = V.DecimationSpec(cfg.hr, cfg.rates)
    if cfg.solver == "tikhonov":
        op = V.TikhonovOperator(V.psf_to_spectrum(inp.psf), spec, V.TikhonovConfig(cfg.reg, inp.xbar))
        x64, x32 = op.solve(inp.y), op.solve_f32(inp.y).astype(np.float64)
        op.close()
    else:
        x = {}
        for prec in ("f64", "f32"):
            init = V.INIT_PROVIDED if inp.x0 is not None else V.INIT_ZERO
            c = V.TvAdmmConfig(lambda_=cfg.tv_lambda, mu=cfg.tv_mu, max_iters=cfg.tv_iters, rel_tol=0.0,
                               tau=1e-3 * cfg.tv_mu, init=init, init_volume=inp.x0, precision=prec)
            x[prec] = V.admm_tv(inp.y, inp.psf, spec, c)[0]
        x64, x32 = x["f64"], x["f32"]
    e = rel_err(x32, x64)
    dp = abs(_psnr(inp.truth, x32) - _psnr(inp.truth, x64))
    print(f"full-size config {cfg_idx}: rel L2 {e:.2e}, PSNR gap {dp:.2e} dB")
    assert e <= FP32_TOL and dp < PSNR_TOL
