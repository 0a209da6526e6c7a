"""Generates tests/golden/*.npz from the REFERENCE itself (oracle/_ref, the
reference volsr sources compiled with the FFTW3/Eigen shims).  Run here,
where /root/reference exists:  make -C oracle && python tools/make_golden.py

Each fixture stores its inputs, so the GPU box (no /root/reference) checks
against the committed vectors without regenerating anything."""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))
import ref_binding as R  # noqa: E402
from paper_2010_15491_b200 import synth  # noqa: E402

OUT = ROOT / "tests" / "golden"


def save(name, **kw):
    OUT.mkdir(parents=True, exist_ok=True)
    np.savez_compressed(OUT / f"{name}.npz", **kw)
    print("wrote", name, sum(np.asarray(v).nbytes for v in kw.values()) // 1024, "KiB")


def main():
    assert R.available(), "build oracle/_ref first (make -C oracle)"
    rng = np.random.default_rng(2010_15491)

    # FFT contract (reference fft3 / ifft3_real through the FFTW3-API shim)
    xr = rng.uniform(-1, 1, (7, 3, 5))
    xc = rng.uniform(-1, 1, (6, 4, 8)) + 1j * rng.uniform(-1, 1, (6, 4, 8))
    xr2 = rng.uniform(-1, 1, (16, 32, 8))
    save("fft", xr=xr, fr=R.fft3(xr), xc=xc, fc=R.fft3(xc), xr2=xr2, fr2=R.fft3(xr2),
         back2=R.ifft3_real(R.fft3(xr2)))

    # Config 0 at full size: 64^3 -> 32^3, PSF sigma 1 / 9^3, 40 dB, tau 1e-3
    cfg = synth.CONFIGS[0]
    inp = synth.make_inputs(cfg, with_truth=False)
    psf = R.make_gaussian_psf(cfg.psf_size, cfg.psf_sigma, cfg.hr)
    assert np.array_equal(psf, inp.psf) or np.max(np.abs(psf - inp.psf)) < 1e-16
    lam = R.psf_to_spectrum(psf)
    op = R.TikhonovOperator(lam, cfg.hr, cfg.rates, cfg.reg, inp.xbar)
    x = op.solve(inp.y)
    save("config0_tikhonov", hr=np.array(cfg.hr), rates=np.array(cfg.rates), reg=cfg.reg,
         psf_size=np.array(cfg.psf_size), psf_sigma=np.array(cfg.psf_sigma), y=inp.y, x=x)

    # Tikhonov, non-cubic / non-power-of-two shapes
    cases = []
    for hr, rates, ksz in [((12, 10, 8), (2, 2, 2), 5), ((20, 12, 6), (5, 3, 2), 3), ((16, 8, 32), (4, 2, 4), 5)]:
        psf = R.make_gaussian_psf((ksz, ksz, ksz), (1.5, 1.2, 1.0), hr)
        y = rng.uniform(0, 1, tuple(hr[a] // rates[a] for a in (2, 1, 0)))
        xbar = rng.uniform(0, 1, (hr[2], hr[1], hr[0]))
        reg = float(rng.uniform(0.01, 0.2))
        op = R.TikhonovOperator(R.psf_to_spectrum(psf), hr, rates, reg, xbar)
        cases.append(dict(hr=np.array(hr), rates=np.array(rates), psf=psf, y=y, xbar=xbar, reg=reg,
                          x=op.solve(y)))
    save("tikhonov_shapes", **{f"c{i}_{k}": v for i, c in enumerate(cases) for k, v in c.items()})

    # tv_x_update at 16^3, d = 4^3, tau = 1e-3
    hr, rates, mu, tau = (16, 16, 16), (4, 4, 4), 0.7, 1e-3
    psf = R.make_gaussian_psf((5, 5, 5), (1.5, 1.5, 1.5), hr)
    lam = R.psf_to_spectrum(psf)
    theta = rng.uniform(-1, 1, (16, 16, 16))
    theta -= theta.mean()
    th = R.fft3(theta)
    y = rng.uniform(0, 1, (4, 4, 4))
    g = R.make_gamma(hr, tau)
    save("tv_x_update", hr=np.array(hr), rates=np.array(rates), mu=mu, tau=tau, psf=psf, y=y, theta_hat=th,
         x=R.tv_x_update(y, lam, hr, rates, mu, th, g), gamma=g)

    # ADMM-TV: config-2 recipe at 32^3 (d = 4^3, spectral-upsampled x0) and the
    # anisotropic config-3 recipe at 32x32x16 (d = 2,2,4).  Parity protocol:
    # tau = 1e-3 * mu explicit, rel_tol = 0.
    for name, base, hr, iters in [("config2_tv_32", 2, (32, 32, 32), 12), ("config3_tv_32", 3, (32, 32, 16), 8)]:
        c = synth.scaled(synth.CONFIGS[base], hr)
        c.psf_size = tuple(min(p, 7) | 1 for p in c.psf_size)
        inp = synth.make_inputs(c, with_truth=False)
        psf = R.make_gaussian_psf(c.psf_size, c.psf_sigma, c.hr)
        init = 2 if inp.x0 is not None else 0
        x, rep = R.admm_tv(inp.y, psf, c.hr, c.rates, c.tv_lambda, c.tv_mu, iters, 0.0, tau=1e-3 * c.tv_mu,
                           init=init, init_volume=inp.x0)
        kw = dict(hr=np.array(c.hr), rates=np.array(c.rates), psf=psf, y=inp.y, lam_tv=c.tv_lambda, mu=c.tv_mu,
                  tau=1e-3 * c.tv_mu, iters=iters, x=x, objective=rep["objective"],
                  primal_residual=rep["primal_residual"], initial_objective=rep["initial_objective"])
        if inp.x0 is not None:
            kw["x0"] = inp.x0
        save(name, **kw)

    # objective_tv
    hr, rates = (12, 8, 8), (2, 2, 2)
    psf = R.make_gaussian_psf((3, 3, 3), (1.0, 1.0, 1.0), hr)
    x = rng.uniform(0, 1, (8, 8, 12))
    y = rng.uniform(0, 1, (4, 4, 6))
    save("objective_tv", hr=np.array(hr), rates=np.array(rates), psf=psf, x=x, y=y, w=0.3,
         value=R.objective_tv(x, y, R.psf_to_spectrum(psf), hr, rates, 0.3))



def admm_l2l2_golden():
    """admm_l2l2 (solvers.cpp:95-189) on two small problems, fixed iteration
    counts, from the reference itself."""
    assert R.available(), "build oracle/_ref first (make -C oracle)"
    rng = np.random.default_rng(95189)
    out = {}
    for i, (hr, rates, iters) in enumerate([((8, 8, 8), (2, 2, 2), 6), ((12, 10, 8), (2, 1, 2), 5)]):
        m, n, s = hr
        w = rng.uniform(0.0, 1.0, 27)
        psf = np.zeros((s, n, m))
        k = 0
        for dz in (-1, 0, 1):
            for dy in (-1, 0, 1):
                for dx in (-1, 0, 1):
                    psf[dz % s, dy % n, dx % m] = w[k]
                    k += 1
        psf /= psf.sum()
        lam = R.fft3(psf) * np.sqrt(m * n * s)  # unnormalised DFT of the wrapped PSF
        xbar = rng.uniform(-1, 1, (s, n, m))
        lr = (m // rates[0], n // rates[1], s // rates[2])
        y = rng.uniform(-1, 1, (lr[2], lr[1], lr[0]))
        x, rep = R.admm_l2l2(y, lam, hr, rates, 0.05, xbar, iters, mu=0.3, rel_tol=0.0)
        out.update({f"c{i}_hr": np.array(hr), f"c{i}_rates": np.array(rates), f"c{i}_iters": iters,
                    f"c{i}_lam": lam, f"c{i}_xbar": xbar, f"c{i}_y": y, f"c{i}_x": x,
                    f"c{i}_objective": rep["objective"], f"c{i}_residual": rep["primal_residual"],
                    f"c{i}_init_obj": rep["initial_objective"]})
    save("admm_l2l2", **out)


def volio_golden():
    """Volume files (volume_io.cpp:34-131) written and read by the reference:
    its f64 / f32 files byte for byte, and its error text for the malformed
    cases of tests/volio_cases.py."""
    import tempfile
    sys.path.insert(0, str(ROOT / "tests"))
    import volio_cases as VC
    assert R.available(), "build oracle/_ref first (make -C oracle)"
    out = {}
    with tempfile.TemporaryDirectory() as td:
        d = Path(td)
        for f32 in (False, True):
            tag = "f32" if f32 else "f64"
            R.save_volume(d / f"w_{tag}", VC.VALS, f32=f32)
            out[f"{tag}_hdr"] = np.frombuffer((d / f"w_{tag}.volhdr").read_bytes(), dtype=np.uint8)
            out[f"{tag}_raw"] = np.frombuffer((d / f"w_{tag}.vol").read_bytes(), dtype=np.uint8)
        for name, base in VC.cases(d).items():
            try:
                v = R.load_volume(base)
                out[f"case_{name}"] = np.array("OK")
                out[f"case_{name}_vals"] = v
            except R.RefError as e:
                msg = str(e).split("] ", 1)[1]
                out[f"case_{name}"] = np.array(VC.norm(msg, d))
        bad = VC.VALS.copy()
        bad[2, 0, 1] = np.inf
        try:
            R.save_volume(d / "save_bad", bad)
            out["save_non_finite"] = np.array("OK")
        except R.RefError as e:
            out["save_non_finite"] = np.array(str(e).split("] ", 1)[1])
    save("volio", vals=VC.VALS, **out)


def degrade_golden():
    """degrade (sim.cpp:106-127) from the reference: Gaussian PsfSpec, BSNR
    noise from its mt19937_64 + Box-Muller stream, and a noiseless case."""
    assert R.available(), "build oracle/_ref first (make -C oracle)"
    rng = np.random.default_rng(106127)
    out = {}
    cases = [((16, 12, 8), (2, 2, 2), (5, 5, 5), (1.0, 1.0, 1.0), 30.0, 7),
             ((24, 16, 8), (2, 1, 2), (7, 5, 3), (1.3, 0.9, 0.7), 20.0, 123456789),
             ((12, 12, 12), (3, 2, 4), (5, 5, 5), (1.0, 1.0, 1.0), None, 0)]
    for i, (hr, rates, ksz, sig, bsnr, seed) in enumerate(cases):
        x = rng.uniform(0, 1, (hr[2], hr[1], hr[0]))
        y, sigma = R.degrade(x, ksz, sig, rates, bsnr, seed)
        out.update({f"c{i}_hr": np.array(hr), f"c{i}_rates": np.array(rates), f"c{i}_ksz": np.array(ksz),
                    f"c{i}_sigma_psf": np.array(sig), f"c{i}_bsnr": np.array(-1.0 if bsnr is None else bsnr),
                    f"c{i}_seed": np.array(seed, dtype=np.uint64), f"c{i}_x": x, f"c{i}_y": y,
                    f"c{i}_noise_sigma": np.array(sigma)})
    save("degrade", n=np.array(len(cases)), **out)


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "admm_l2l2":
        admm_l2l2_golden()
    elif len(sys.argv) > 1 and sys.argv[1] == "volio":
        volio_golden()
    elif len(sys.argv) > 1 and sys.argv[1] == "degrade":
        degrade_golden()
    else:
        main()
        admm_l2l2_golden()
        volio_golden()
        degrade_golden()
