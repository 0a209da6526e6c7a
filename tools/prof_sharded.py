"""Short driver for ncu: the slab-sharded config-3 ADMM-TV at P = 1 (one
LocalExchange rank) for a few iterations, seeded random data."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2010_15491_b200 import dist as D  # noqa: E402
from paper_2010_15491_b200 import synth  # noqa: E402
from paper_2010_15491_b200 import volsr as V  # noqa: E402


def main(iters=3):
    cfg = synth.CONFIGS[3]
    hr, rates = cfg.hr, cfg.rates
    ctx = V.default_context()
    dev = torch.device("cuda", 0)
    g = D.SlabGeometry(hr, rates, 1)
    psf = torch.from_numpy(np.ascontiguousarray(synth.make_gaussian_psf(cfg.psf_size, cfg.psf_sigma, hr)))
    y = torch.rand(g.sl * g.nl * g.ml, device=dev, dtype=torch.float64)
    x0 = torch.rand(g.slab_elems, device=dev, dtype=torch.float64)
    tv = D.SlabADMMTV(D.GpuStages({0: ctx}), D.LocalExchange(1), hr, rates, {0: psf.reshape(-1).to(dev)},
                      {0: y}, {0: x0}, cfg.tv_lambda, cfg.tv_mu, tau=1e-3 * cfg.tv_mu)
    tv.iterate(iters)
    torch.cuda.synchronize()
    print("prof_sharded ok")


if __name__ == "__main__":
    main(*(int(a) for a in sys.argv[1:2]))
