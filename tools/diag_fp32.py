import sys; sys.path[:0]=['.','tests','oracle']
import numpy as np
from paper_2010_15491_b200 import volsr as V, synth
cfg = synth.scaled(synth.CONFIGS[2], (256, 64, 64))
inp = synth.make_inputs(cfg)
spec = V.DecimationSpec(cfg.hr, cfg.rates)
for tau in (5e-5, None):
  for it in (1, 2, 5):
    out = {}
    for prec in ("f64", "f32"):
        c = V.TvAdmmConfig(lambda_=cfg.tv_lambda, mu=cfg.tv_mu, max_iters=it, rel_tol=0.0, tau=tau, init=V.INIT_UPSAMPLED, precision=prec)
        out[prec] = V.admm_tv(inp.y, inp.psf, spec, c)
    a, b = out["f64"][0], out["f32"][0]
    d = b - a
    D = np.fft.fftn(d, norm="ortho"); A = np.fft.fftn(a, norm="ortho")
    print(f"tau={tau} it={it} rel={np.linalg.norm(d)/np.linalg.norm(a):.3e} mean_a={a.mean():.6e} mean_d={d.mean():.3e} "
          f"nonDC rel={np.sqrt((np.abs(D)**2).sum()-abs(D[0,0,0])**2)/np.linalg.norm(a):.3e} obj64={out['f64'][1].objective[-1]:.8e} obj32={out['f32'][1].objective[-1]:.8e}")
    # error concentration in low frequencies
    s,n,m = d.shape
    f = np.sqrt(np.add.outer(np.add.outer(np.minimum(np.arange(s),s-np.arange(s))**2/ (s*s), np.minimum(np.arange(n),n-np.arange(n))**2/(n*n)), np.minimum(np.arange(m),m-np.arange(m))**2/(m*m)))
    lo = f < 0.05
    print("   low-freq err frac", np.sqrt((np.abs(D[lo])**2).sum())/np.linalg.norm(d))
