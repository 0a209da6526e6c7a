"""Short driver for ncu: the slab-sharded config-3 ADMM-TV (csrc/slab.cu) at
P = 1 (local comm) for a few iterations, seeded random data."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2010_15491_b200 import dist as D  # noqa: E402
from paper_2010_15491_b200 import synth  # noqa: E402
from paper_2010_15491_b200 import volsr as V  # noqa: E402


def main(iters=3, P=1):
    cfg = synth.CONFIGS[3]
    hr, rates = cfg.hr, cfg.rates
    psf = synth.make_gaussian_psf(cfg.psf_size, cfg.psf_sigma, hr)
    y = np.random.default_rng(0).uniform(0, 1, V.shape_of(cfg.lr))
    tcfg = V.TvAdmmConfig(lambda_=cfg.tv_lambda, mu=cfg.tv_mu, max_iters=iters, rel_tol=0.0,
                          tau=1e-3 * cfg.tv_mu, init=V.INIT_UPSAMPLED)
    D.admm_tv(D.SlabComm.local(P), y, psf, V.DecimationSpec(hr, rates), tcfg)
    print("prof_sharded ok")


if __name__ == "__main__":
    main(*(int(a) for a in sys.argv[1:3]))
