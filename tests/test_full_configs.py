"""BASELINE.json configs at their FULL sizes on the GPU.

configs 1-3: the CUDA path against the numpy oracle on each config's own
seeded synthetic inputs (synth.make_inputs: ellipsoid + texture phantom,
Gaussian PSF, BSNR noise).  ADMM-TV runs the first iterations only (the
oracle needs ~10-30 s per HR iteration at these sizes); the per-iteration
kernels are the same for every iteration.  Config 0 at full size is pinned
against the reference's own output in test_golden.py.

config 4 (1024^3; the oracle would need ~150 GB of host memory) is checked
through size-independent properties of the solve, entirely on the device:
the spatial-expansion path against the general FFT path (two independent
algorithms), and the normal-equation residual of the
Tikhonov solution (reference test_solvers.cpp:113-139) evaluated with
cuFFT as an independent checker.
"""
import ctypes as C
import os

import numpy as np
import pytest

from conftest import rel_err

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
TOL = 1e-10


@pytest.fixture(scope="module")
def synth():
    from paper_2010_15491_b200 import synth as S
    return S


def test_config1_tikhonov_full_size(V, O, synth):
    cfg = synth.CONFIGS[1]
    inp = synth.make_inputs(cfg, with_truth=False)
    spec, ospec = V.DecimationSpec(cfg.hr, cfg.rates), O.DecimationSpec(cfg.hr, cfg.rates)
    lam = O.psf_to_spectrum(inp.psf)
    op = V.TikhonovOperator(V.psf_to_spectrum(inp.psf), spec, V.TikhonovConfig(1e-3, inp.xbar))
    assert op.path()["spatial"]
    got = op.solve(inp.y)
    want = O.tikhonov_fast(inp.y, lam, ospec, 1e-3, inp.xbar)
    assert rel_err(got, want) < TOL


@pytest.mark.parametrize("idx,iters", [(2, 2), (3, 1)])
def test_tv_configs_full_size(V, O, synth, idx, iters):
    cfg = synth.CONFIGS[idx]
    inp = synth.make_inputs(cfg, with_truth=False)
    spec, ospec = V.DecimationSpec(cfg.hr, cfg.rates), O.DecimationSpec(cfg.hr, cfg.rates)
    x0 = inp.x0 if inp.x0 is not None else None
    init = V.INIT_PROVIDED if x0 is not None else V.INIT_UPSAMPLED
    tau = 1e-3 * cfg.tv_mu
    got, rep = V.admm_tv(inp.y, inp.psf, spec,
                         V.TvAdmmConfig(lambda_=cfg.tv_lambda, mu=cfg.tv_mu, max_iters=iters, rel_tol=0.0,
                                        tau=tau, init=init, init_volume=x0))
    want, orep = O.admm_tv(inp.y, inp.psf, ospec, lam_tv=cfg.tv_lambda, mu=cfg.tv_mu, max_iters=iters,
                           rel_tol=0.0, tau=tau, init=init, init_volume=x0)
    assert rel_err(got, want) < TOL
    assert rel_err(rep.objective, orep.objective) < TOL
    assert rel_err(rep.primal_residual, orep.primal_residual) < 1e-9


class _Dev:
    """A torch device tensor seen through the C ABI's device-pointer entry points."""

    def __init__(self, t):
        self.t = t
        self.ptr = C.c_void_p(t.data_ptr())


def test_config4_tikhonov_properties_1024(V, O, synth):
    torch = pytest.importorskip("torch")
    cfg = synth.CONFIGS[4]
    free, _ = torch.cuda.mem_get_info()
    if free < 120e9:
        pytest.skip("needs ~110 GB of free device memory")
    m, n, s = cfg.hr
    N = m * n * s
    d = int(np.prod(cfg.rates))
    ml, nl, sl = m // cfg.rates[0], n // cfg.rates[1], s // cfg.rates[2]
    spec = V.DecimationSpec(cfg.hr, cfg.rates)
    ctx = V.default_context()
    dev = torch.device("cuda", 0)
    reg = 1e-3
    g = torch.Generator(device=dev).manual_seed(7)
    y = torch.rand(sl, nl, ml, generator=g, device=dev, dtype=torch.float64)
    # PSF on the device: the reference's sampled, normalised Gaussian, built
    # origin-wrapped on its own support and embedded at offsets -h..h (mod dims)
    kern = torch.from_numpy(np.ascontiguousarray(
        O.make_gaussian_psf(cfg.psf_size, cfg.psf_sigma, cfg.psf_size))).to(dev)
    psf = torch.zeros(s, n, m, device=dev, dtype=torch.float64)
    idx = []
    for k, L in zip(kern.shape, (s, n, m)):
        i = torch.arange(k, device=dev)
        idx.append(torch.where(i <= k // 2, i, i - k) % L)
    psf[idx[0][:, None, None], idx[1][None, :, None], idx[2][None, None, :]] = kern
    del kern
    lam = torch.empty(N, device=dev, dtype=torch.complex128)
    dims = (C.c_size_t * 3)(m, n, s)
    V.check(V._lib.vsr_fft3_d(ctx.handle, dims, C.c_void_p(psf.data_ptr()), 1, C.c_void_p(lam.data_ptr()), 1.0))
    ctx.synchronize()
    del psf
    xbar = torch.zeros(s, n, m, device=dev, dtype=torch.float64)
    xbar[::cfg.rates[2], ::cfg.rates[1], ::cfg.rates[0]] = d * y
    x_sp = torch.empty(s, n, m, device=dev, dtype=torch.float64)
    op = V.TikhonovDevice(ctx, spec, _Dev(lam), reg, _Dev(xbar))
    assert op.spatial()
    op.solve_d(_Dev(y), _Dev(x_sp))
    op.check()
    op.close()
    # the same solve through the general FFT path (fused fold + inverse passes)
    os.environ["VSR_NO_SPATIAL"] = "1"
    try:
        op = V.TikhonovDevice(ctx, spec, _Dev(lam), reg, _Dev(xbar))
    finally:
        del os.environ["VSR_NO_SPATIAL"]
    assert not op.spatial()
    x_ff = torch.empty_like(x_sp)
    op.solve_d(_Dev(y), _Dev(x_ff))
    op.check()
    op.close()
    ctx.synchronize()
    diff = float(torch.linalg.vector_norm(x_sp - x_ff) / torch.linalg.vector_norm(x_ff))
    assert diff < 1e-12, diff
    del x_ff
    torch.cuda.empty_cache()
    # normal equations (solvers.cpp:36-67): (H^T D^T D H + 2 reg I) x = H^T D^T y + 2 reg xbar,
    # checked with cuFFT (torch.fft) as an independent transform
    lam3 = lam.view(s, n, m)

    def blur(v, conj):
        f = torch.fft.fftn(v)
        f *= lam3.conj() if conj else lam3
        return torch.fft.ifftn(f).real

    hx = blur(x_sp, False)
    r = hx[::cfg.rates[2], ::cfg.rates[1], ::cfg.rates[0]] - y
    del hx
    up = torch.zeros_like(x_sp)
    up[::cfg.rates[2], ::cfg.rates[1], ::cfg.rates[0]] = r
    lhs = blur(up, True) + 2 * reg * (x_sp - xbar)
    up.zero_()
    up[::cfg.rates[2], ::cfg.rates[1], ::cfg.rates[0]] = y
    rhs = blur(up, True) + 2 * reg * xbar
    res = float(torch.linalg.vector_norm(lhs) / torch.linalg.vector_norm(rhs))
    assert res < 1e-9, res


# ------------------------------------------------ against the reference itself
# oracle/_ref (the reference's own sources, compiled with the FFTW3-API shim)
# travels with the repo, so the GPU box can run the REFERENCE on the same
# full-size inputs: config 1's solve and config 2's first ADMM-TV iterations.
@pytest.fixture(scope="module")
def R():
    import ref_binding
    if not ref_binding.available():
        pytest.skip("oracle/_ref not built")
    return ref_binding


def test_config1_tikhonov_vs_reference_binary(V, R, synth):
    cfg = synth.CONFIGS[1]
    inp = synth.make_inputs(cfg, with_truth=False)
    spec = V.DecimationSpec(cfg.hr, cfg.rates)
    got = V.TikhonovOperator(V.psf_to_spectrum(inp.psf), spec, V.TikhonovConfig(cfg.reg, inp.xbar)).solve(inp.y)
    want = R.TikhonovOperator(inp.psf, cfg.hr, cfg.rates, cfg.reg, inp.xbar).solve(inp.y)
    assert rel_err(got, want) < TOL


def test_config2_admm_tv_vs_reference_binary(V, R, synth):
    cfg = synth.CONFIGS[2]
    inp = synth.make_inputs(cfg, with_truth=False)
    spec = V.DecimationSpec(cfg.hr, cfg.rates)
    tau, iters = 1e-3 * cfg.tv_mu, 2
    got, rep = V.admm_tv(inp.y, inp.psf, spec,
                         V.TvAdmmConfig(lambda_=cfg.tv_lambda, mu=cfg.tv_mu, max_iters=iters, rel_tol=0.0, tau=tau,
                                        init=V.INIT_PROVIDED, init_volume=inp.x0))
    want, wrep = R.admm_tv(inp.y, inp.psf, cfg.hr, cfg.rates, cfg.tv_lambda, cfg.tv_mu, iters, 0.0, tau=tau,
                           init=V.INIT_PROVIDED, init_volume=inp.x0)
    assert rel_err(got, want) < TOL
    assert rel_err(rep.objective, wrep["objective"]) < TOL
    assert abs(rep.initial_objective - wrep["initial_objective"]) <= 1e-10 * abs(wrep["initial_objective"])
