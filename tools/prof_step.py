"""Short driver for ncu: config-1 Tikhonov solves and config-2 ADMM-TV
iterations on seeded random data of the benchmark shapes (values do not
affect the kernels' memory behaviour)."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2010_15491_b200 import volsr as V  # noqa: E402


def main(mode="all", reps=2):
    ctx = V.default_context()
    rng = np.random.default_rng(0)
    if mode in ("all", "tik", "tiklat", "bench"):
        hr, rates = (256, 256, 256), (2, 2, 2)
        spec = V.DecimationSpec(hr, rates)
        psf = V.make_gaussian_psf((13, 13, 13), (1.5, 1.5, 1.5), hr)
        lam = V.psf_to_spectrum(psf)
        y = rng.uniform(0, 1, V.shape_of(spec.lr))
        # tiklat: the CLI-default lattice prior (spatial-expansion solve)
        lat = mode in ("tiklat", "bench")
        xbar = V.zero_fill_upsample(y, spec) if lat else rng.uniform(0, 1, V.shape_of(hr))
        op = V.TikhonovOperator(lam, spec, V.TikhonovConfig(1e-3, xbar))
        for _ in range(reps):
            op.solve(y)
        op.close()
    if mode in ("all", "tv", "bench", "tv32"):
        hr, rates = (256, 256, 256), (4, 4, 4)
        spec = V.DecimationSpec(hr, rates)
        psf = V.make_gaussian_psf((13, 13, 13), (1.5, 1.5, 1.5), hr)
        y = rng.uniform(0, 1, V.shape_of(spec.lr))
        cfg = V.TvAdmmConfig(lambda_=2e-3, mu=0.05, max_iters=reps, rel_tol=0.0, tau=5e-5,
                             precision="f32" if mode == "tv32" else "f64")
        V.admm_tv(y, psf, spec, cfg)
    ctx.synchronize()
    print("prof_step ok", V.launch_count())


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "all", int(sys.argv[2]) if len(sys.argv) > 2 else 2)
