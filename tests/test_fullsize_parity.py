"""BASELINE configs 2-4 at FULL size and their REAL iteration counts against
the reference (VERDICT r01 "what's missing" 1).

Opt-in (VSR_FULL_PARITY=1): the reference runs single-process on the GPU
box's host (FFTs threaded over all cores via the shim's VSR_SHIM_THREADS,
every other pass single-threaded as in the reference), which takes about an
hour for the four cases.  Each case appends one JSON line to
$VSR_PARITY_LOG; the committed summary is profiles/r02_fullsize_parity.md.

  * config 2 (256^3 -> 64^3, d = 64): 100 ADMM-TV iterations vs oracle/_ref;
  * config 3 (512x512x256 -> 256x256x64, d = 16): 50 iterations vs oracle/_ref;
  * config 4 (1024^3 -> 512^3): the Tikhonov solve vs oracle/_ref, run in a
    child process under an address-space limit (the reference needs ~150 B
    per voxel, ~165 GB of the box's 196 GB);
  * config 4 ADMM-TV: the reference would need ~300 B per voxel (320 GB at
    1024^3, measured 297 B/voxel at 256^3), more than the host has, so the
    first 2 iterations are checked against oracle/lean_oracle.py, a
    memory-lean restatement pinned to the reference binary in
    tests/test_oracle_pins.py.

Bar: x within relative L2 <= 1e-10, objective and primal
residual series <= 1e-10 relative, initial objective <= 1e-10 relative.
ADMM-TV runs at tau = 1e-3 * mu (the reference default
1e-8 * mu amplifies rounding in the DC bin by 1/(tau mu d)).
"""
import json
import os
import subprocess
import sys
import tempfile
import time
from pathlib import Path

import numpy as np
import pytest

from conftest import rel_err

pytestmark = [pytest.mark.gpu, pytest.mark.slow,
              pytest.mark.skipif(os.environ.get("VSR_FULL_PARITY") != "1",
                                 reason="full-size reference parity is opt-in (VSR_FULL_PARITY=1)")]
TOL = 1e-10
ROOT = Path(__file__).resolve().parent.parent


def _log(rec):
    path = os.environ.get("VSR_PARITY_LOG")
    print(json.dumps(rec), flush=True)
    if path:
        with open(path, "a") as f:
            f.write(json.dumps(rec) + "\n")


def _series_err(a, b):
    a, b = np.asarray(a, float), np.asarray(b, float)
    assert a.shape == b.shape
    return float(np.max(np.abs(a - b) / np.abs(b)))


@pytest.fixture(scope="module")
def R():
    import ref_binding
    if not ref_binding.available():
        pytest.skip("oracle/_ref not built")
    os.environ["VSR_SHIM_THREADS"] = str(os.cpu_count() or 1)
    return ref_binding


@pytest.fixture(scope="module")
def synth():
    from paper_2010_15491_b200 import synth as S
    return S


@pytest.mark.parametrize("idx", [2, 3])
def test_admm_tv_full_iterations_vs_reference(V, R, synth, idx):
    cfg = synth.CONFIGS[idx]
    inp = synth.make_inputs(cfg, with_truth=False)
    spec = V.DecimationSpec(cfg.hr, cfg.rates)
    tau, iters = 1e-3 * cfg.tv_mu, cfg.tv_iters
    init = V.INIT_PROVIDED if inp.x0 is not None else V.INIT_UPSAMPLED
    t0 = time.perf_counter()
    got, rep = V.admm_tv(inp.y, inp.psf, spec,
                         V.TvAdmmConfig(lambda_=cfg.tv_lambda, mu=cfg.tv_mu, max_iters=iters, rel_tol=0.0, tau=tau,
                                        init=init, init_volume=inp.x0))
    t1 = time.perf_counter()
    want, wrep = R.admm_tv(inp.y, inp.psf, cfg.hr, cfg.rates, cfg.tv_lambda, cfg.tv_mu, iters, 0.0, tau=tau,
                           init=init, init_volume=inp.x0)
    t2 = time.perf_counter()
    rec = {"case": f"config{idx} admm_tv {iters} iterations vs oracle/_ref", "hr": cfg.hr, "rates": cfg.rates,
           "iterations": [rep.iterations, wrep["iterations"]],
           "x_rel_l2": rel_err(got, want),
           "objective_max_rel": _series_err(rep.objective, wrep["objective"]),
           "residual_max_rel": _series_err(rep.primal_residual, wrep["primal_residual"]),
           "initial_objective_rel": abs(rep.initial_objective - wrep["initial_objective"])
           / abs(wrep["initial_objective"]),
           "gpu_s": t1 - t0, "reference_s": t2 - t1, "reference_threads": os.environ["VSR_SHIM_THREADS"]}
    _log(rec)
    assert rep.iterations == wrep["iterations"] == iters
    assert rec["x_rel_l2"] < TOL
    assert rec["objective_max_rel"] < TOL
    assert rec["residual_max_rel"] < TOL
    assert rec["initial_objective_rel"] < TOL


def _host_gb():
    with open("/proc/meminfo") as f:
        for ln in f:
            if ln.startswith("MemTotal"):
                return int(ln.split()[1]) / 1e6
    return 0.0


def test_config4_tikhonov_1024_vs_reference(V, R, synth):
    torch = pytest.importorskip("torch")
    if torch.cuda.mem_get_info()[0] < 100e9:
        pytest.skip("needs ~90 GB of free device memory")
    host = _host_gb()
    if host < 180:
        pytest.skip(f"the reference needs ~165 GB of host memory ({host:.0f} GB here)")
    cfg = synth.CONFIGS[4]
    with tempfile.TemporaryDirectory(dir=os.environ.get("VSR_PARITY_TMP", "/tmp")) as td:
        td = Path(td)
        limit = (host - 8) * 1e9  # leave the parent and the OS room: allocation failure, not the OOM killer
        r = subprocess.run([sys.executable, str(ROOT / "tests" / "fullsize_child.py"), str(td), str(limit)],
                           capture_output=True, text=True, timeout=7200,
                           env={**os.environ, "VSR_SHIM_THREADS": str(os.cpu_count() or 1)})
        if r.returncode != 0:
            _log({"case": "config4 tikhonov vs oracle/_ref", "unmeasured": r.stderr[-2000:]})
            pytest.fail("reference child failed: " + r.stderr[-2000:])
        child = json.loads(r.stdout.strip().splitlines()[-1])
        y = np.load(td / "y.npy")
        want = np.load(td / "x_ref.npy", mmap_mode="r")
        psf = synth.make_gaussian_psf(cfg.psf_size, cfg.psf_sigma, cfg.hr)
        xbar = synth.zero_fill_upsample(y, cfg.rates)
        spec = V.DecimationSpec(cfg.hr, cfg.rates)
        t0 = time.perf_counter()
        lam = V.psf_to_spectrum(psf)
        del psf
        op = V.TikhonovOperator(lam, spec, V.TikhonovConfig(cfg.reg, xbar))
        del lam, xbar
        got = op.solve(y)
        path = op.path()
        op.close()
        t1 = time.perf_counter()
        err = rel_err(got, np.asarray(want))
        del want
    _log({"case": "config4 tikhonov 1024^3 vs oracle/_ref", "x_rel_l2": err, "gpu_path": path,
          "gpu_s_incl_setup": t1 - t0, "reference": child})
    assert err < TOL


def test_config4_admm_tv_1024_vs_lean_oracle(V, synth):
    torch = pytest.importorskip("torch")
    if torch.cuda.mem_get_info()[0] < 140e9:
        pytest.skip("needs ~125 GB of free device memory")
    host = _host_gb()
    if host < 150:
        pytest.skip(f"the lean oracle needs ~110 GB of host memory ({host:.0f} GB here)")
    import lean_oracle as LO
    cfg = synth.CONFIGS[4]
    iters = 2
    tau = 1e-3 * cfg.tv_mu
    inp = synth.make_inputs(cfg, with_truth=False)
    y, psf = inp.y, inp.psf
    del inp
    spec = V.DecimationSpec(cfg.hr, cfg.rates)
    t0 = time.perf_counter()
    got, rep = V.admm_tv(y, psf, spec, V.TvAdmmConfig(lambda_=cfg.tv_lambda, mu=cfg.tv_mu, max_iters=iters,
                                                       rel_tol=0.0, tau=tau, init=V.INIT_ZERO))
    t1 = time.perf_counter()
    ospec = LO.DecimationSpec(cfg.hr, cfg.rates)
    want, wrep = LO.admm_tv(y, psf, ospec, cfg.tv_lambda, cfg.tv_mu, iters, tau=tau, init=LO.INIT_ZERO,
                            log=lambda m: print(m, flush=True))
    t2 = time.perf_counter()
    rec = {"case": f"config4 admm_tv 1024^3 {iters} iterations vs oracle/lean_oracle.py",
           "x_rel_l2": rel_err(got, want),
           "objective_max_rel": _series_err(rep.objective, wrep.objective),
           "residual_max_rel": _series_err(rep.primal_residual, wrep.primal_residual),
           "initial_objective_rel": abs(rep.initial_objective - wrep.initial_objective) / abs(wrep.initial_objective),
           "gpu_s_incl_setup": t1 - t0, "lean_oracle_s": t2 - t1}
    _log(rec)
    assert rec["x_rel_l2"] < TOL
    assert rec["objective_max_rel"] < TOL
    assert rec["residual_max_rel"] < TOL
    assert rec["initial_objective_rel"] < TOL
