"""Child process for tests/test_fullsize_parity.py: builds BASELINE config 4's
seeded inputs (1024^3) and runs the REFERENCE TikhonovOperator (oracle/_ref)
on them under an address-space limit, so an allocation failure is a clean
error instead of the host's OOM killer.  Writes y.npy and x_ref.npy into the
given directory and prints one JSON line (timings, peak RSS).
TEST INFRASTRUCTURE."""
import json
import os
import resource
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))


def main():
    out = Path(sys.argv[1])
    limit = int(float(sys.argv[2]))
    resource.setrlimit(resource.RLIMIT_AS, (limit, limit))
    import numpy as np

    from paper_2010_15491_b200 import synth as S
    import ref_binding as R
    assert R.available(), "oracle/_ref not built"
    cfg = S.CONFIGS[4]
    t0 = time.perf_counter()
    inp = S.make_inputs(cfg, with_truth=False)
    y, psf, xbar = inp.y, inp.psf, inp.xbar
    del inp
    np.save(out / "y.npy", y)
    t1 = time.perf_counter()
    lam = R.psf_to_spectrum(psf)
    del psf
    op = R.TikhonovOperator(lam, cfg.hr, cfg.rates, cfg.reg, xbar)
    del lam, xbar
    t2 = time.perf_counter()
    x = op.solve(y)
    t3 = time.perf_counter()
    del op
    np.save(out / "x_ref.npy", x)
    print(json.dumps({"inputs_s": t1 - t0, "ctor_s": t2 - t1, "solve_s": t3 - t2,
                      "peak_rss_gb": resource.getrusage(resource.RUSAGE_SELF).ru_maxrss / 1e6,
                      "threads": os.environ.get("VSR_SHIM_THREADS")}))


if __name__ == "__main__":
    main()
