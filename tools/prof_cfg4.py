"""Short driver for ncu: ADMM-TV iterations at configs[4]'s size (1024^3,
d = 2^3) on one GPU, seeded random LR data (values do not change the work)."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa: E402
from paper_2010_15491_b200 import synth  # noqa: E402
from paper_2010_15491_b200 import volsr as V  # noqa: E402


def main(iters=2):
    cfg = synth.CONFIGS[4]
    m, n, s = cfg.hr
    r1, r2, r3 = cfg.rates
    dev = torch.device("cuda", 0)
    ctx = V.default_context()
    y = torch.rand(s // r3, n // r2, m // r1, device=dev, dtype=torch.float64)
    kern = torch.from_numpy(np.ascontiguousarray(V.make_gaussian_psf(cfg.psf_size, cfg.psf_sigma, cfg.psf_size)))
    psf = torch.zeros(s, n, m, device=dev, dtype=torch.float64)
    idx = []
    for k, L in zip(kern.shape, (s, n, m)):
        i = torch.arange(k, device=dev)
        idx.append(torch.where(i <= k // 2, i, i - k) % L)
    psf[idx[0][:, None, None], idx[1][None, :, None], idx[2][None, None, :]] = kern.to(dev)
    tcfg = V.TvAdmmConfig(lambda_=cfg.tv_lambda, mu=cfg.tv_mu, max_iters=iters, rel_tol=0.0,
                          tau=1e-3 * cfg.tv_mu, init=V.INIT_UPSAMPLED)
    tv = V.TvDevice(ctx, V.DecimationSpec(cfg.hr, cfg.rates), bench._Dev(y), bench._Dev(psf), tcfg)
    tv.iterate(iters)
    ctx.synchronize()
    tv.close()
    print("prof_cfg4 ok")


if __name__ == "__main__":
    main(*(int(a) for a in sys.argv[1:2]))
