"""degrade (reference src/sim.cpp:88-127).

tests/golden/degrade.npz is written by the REFERENCE's degrade (Gaussian
PsfSpec, mt19937_64 + Box-Muller noise, BSNR calibration) through
oracle/_ref (tools/make_golden.py degrade).  The numpy oracle restates it
(including a pure-Python mt19937_64) and is pinned to the golden on the CPU;
the GPU path (vsr_degrade: one HR forward transform, the alias fold of
Lambda X, one LR inverse; the serial noise stream on a host thread) is
checked against the same golden and, at a larger size, against the oracle."""
from pathlib import Path

import numpy as np
import pytest

from conftest import rel_err

G = Path(__file__).resolve().parent / "golden" / "degrade.npz"


def cases():
    g = dict(np.load(G))
    out = []
    for i in range(int(g["n"])):
        b = float(g[f"c{i}_bsnr"])
        out.append(dict(hr=tuple(int(v) for v in g[f"c{i}_hr"]), rates=tuple(int(v) for v in g[f"c{i}_rates"]),
                        ksz=tuple(int(v) for v in g[f"c{i}_ksz"]), sig=tuple(float(v) for v in g[f"c{i}_sigma_psf"]),
                        bsnr=None if b < 0 else b, seed=int(g[f"c{i}_seed"]), x=g[f"c{i}_x"], y=g[f"c{i}_y"],
                        noise_sigma=float(g[f"c{i}_noise_sigma"])))
    return out


@pytest.mark.parametrize("i", range(3))
def test_oracle_degrade_golden(O, i):
    c = cases()[i]
    spec = O.DecimationSpec(c["hr"], c["rates"])
    y, s = O.degrade(c["x"], O.make_gaussian_psf(c["ksz"], c["sig"], c["hr"]), spec, c["bsnr"], c["seed"])
    assert rel_err(y, c["y"]) < 1e-14
    assert abs(s - c["noise_sigma"]) <= 1e-14 * max(c["noise_sigma"], 1e-300)


def test_oracle_noise_stream_is_mt19937_64(O):
    # std::mt19937_64 default seed 5489: the 10000th draw is 9981545732273789042 (C++ [rand.predef])
    rng = O._MT19937_64(5489)
    for _ in range(9999):
        rng()
    assert rng() == 9981545732273789042


@pytest.mark.gpu
@pytest.mark.parametrize("i", range(3))
def test_gpu_degrade_golden(V, O, i):
    c = cases()[i]
    spec = V.DecimationSpec(c["hr"], c["rates"])
    y, s = V.degrade(c["x"], O.make_gaussian_psf(c["ksz"], c["sig"], c["hr"]), spec, c["bsnr"], c["seed"])
    assert rel_err(y, c["y"]) < 1e-12
    assert abs(s - c["noise_sigma"]) <= 1e-12 * max(c["noise_sigma"], 1e-300)


@pytest.mark.gpu
def test_gpu_degrade_vs_oracle_64(V, O):
    rng = np.random.default_rng(5)
    hr, rates = (64, 48, 32), (2, 2, 4)
    x = rng.uniform(0, 1, (hr[2], hr[1], hr[0]))
    psf = O.make_gaussian_psf((9, 9, 9), (1.5, 1.5, 2.0), hr)
    y, s = V.degrade(x, psf, V.DecimationSpec(hr, rates), 35.0, 2024)
    yo, so = O.degrade(x, psf, O.DecimationSpec(hr, rates), 35.0, 2024)
    assert rel_err(y, yo) < 1e-12 and abs(s - so) <= 1e-12 * so


@pytest.mark.gpu
def test_gpu_degrade_rejects_non_finite(V, O):
    hr, rates = (16, 16, 16), (2, 2, 2)
    x = np.zeros((16, 16, 16))
    x[3, 4, 5] = np.nan
    with pytest.raises(V.NumericError):
        V.degrade(x, O.make_gaussian_psf((5, 5, 5), (1.0, 1.0, 1.0), hr), V.DecimationSpec(hr, rates), 30.0, 1)


# ------------------------------------------------ reference test_sim.cpp:59-130, restated
@pytest.mark.gpu
def test_gpu_degrade_trivial_operators(V, O):
    """test_sim.cpp:59-68: 1x1x1 PSF, unit rates, no noise -> y = x (bit-exact there; here the
    unitary transform pair leaves rounding, so <= 1e-15)."""
    rng = np.random.default_rng(1)
    d = (8, 8, 8)
    x = rng.uniform(0, 1, d)
    y, s = V.degrade(x, O.make_gaussian_psf((1, 1, 1), (0, 0, 0), d), V.DecimationSpec(d, (1, 1, 1)))
    assert s == 0.0 and rel_err(y, x) < 1e-15


@pytest.mark.gpu
def test_gpu_degrade_noiseless_is_decimated_blur(V, O):
    """test_sim.cpp:70-79."""
    rng = np.random.default_rng(2)
    d = (16, 16, 16)
    psf = O.make_gaussian_psf((5, 5, 5), (1.5, 1.5, 1.5), d)
    x = rng.uniform(0, 1, d)
    y, s = V.degrade(x, psf, V.DecimationSpec(d, (2, 2, 2)))
    want = O.decimate(O.blur_apply(x, O.psf_to_spectrum(psf)), O.DecimationSpec(d, (2, 2, 2)))
    assert s == 0.0 and rel_err(y, want) < 1e-13


@pytest.mark.gpu
def test_gpu_degrade_bsnr_band(V, O):
    """test_sim.cpp:81-118: the measured BSNR lands within 0.5 dB, noise zero-mean."""
    from paper_2010_15491_b200 import synth
    d = (64, 64, 64)
    spec = V.DecimationSpec(d, (2, 2, 2))
    psf = O.make_gaussian_psf((9, 9, 9), (3, 3, 3), d)
    x = synth.ellipsoid_phantom(d, 0)
    noisy, sig = V.degrade(x, psf, spec, 30.0, 11)
    clean, _ = V.degrade(x, psf, spec, None, 11)
    n = noisy - clean
    bsnr = 10 * np.log10(np.mean((clean - clean.mean()) ** 2) / np.mean(n ** 2))
    assert 29.5 < bsnr < 30.5
    assert abs(n.mean()) < 4 * sig / np.sqrt(n.size)


@pytest.mark.gpu
def test_gpu_degrade_deterministic_per_seed(V, O):
    """test_sim.cpp:120-130."""
    rng = np.random.default_rng(5)
    d = (16, 16, 16)
    spec = V.DecimationSpec(d, (2, 2, 2))
    psf = O.make_gaussian_psf((5, 5, 5), (1.2, 1.2, 1.2), d)
    x = rng.uniform(0, 1, d)
    a, _ = V.degrade(x, psf, spec, 25.0, 123)
    b, _ = V.degrade(x, psf, spec, 25.0, 123)
    c, _ = V.degrade(x, psf, spec, 25.0, 124)
    assert a.tobytes() == b.tobytes() and np.abs(a - c).max() > 0
