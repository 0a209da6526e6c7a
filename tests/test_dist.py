"""Slab-decomposed multi-rank path.

CPU: the host orchestration (paper_2010_15491_b200/dist.py) with the numpy
stage double, in-process virtual ranks and a real 2-process gloo group,
against the single-volume oracle.  GPU: the same programs with the CUDA
stages (C ABI vsr_slab_*) and P virtual ranks on one device."""
import math
import os
import socket

import numpy as np
import pytest
import torch

from conftest import rel_err

import volsr_oracle as O
from paper_2010_15491_b200 import dist as D
from paper_2010_15491_b200 import synth


def _case(hr, rates, seed=0):
    rng = np.random.default_rng(seed)
    m, n, s = hr
    psf = O.make_gaussian_psf((5, 5, 5), (1.2, 1.2, 1.5), hr)
    y = rng.uniform(0, 1, (s // rates[2], n // rates[1], m // rates[0]))
    xbar = synth.zero_fill_upsample(y, rates)
    x0 = rng.uniform(0, 1, (s, n, m))
    return psf, y, xbar, x0


def _slabs(vol, P, to=lambda t: t):
    sz = vol.shape[0] // P
    return {p: to(torch.from_numpy(np.ascontiguousarray(vol[p * sz:(p + 1) * sz])).reshape(-1)) for p in range(P)}


def _run_tik(stages, ex, hr, rates, psf, y, xbar, reg, to=lambda t: t, ranks=None):
    P = ex.world
    ranks = ex.ranks
    ps, xs = _slabs(psf, P, to), _slabs(xbar, P, to)
    op = D.SlabTikhonov(stages, ex, hr, rates, {r: ps[r] for r in ranks}, reg, {r: xs[r] for r in ranks})
    yt = {r: to(torch.from_numpy(np.ascontiguousarray(y)).reshape(-1)) for r in ranks}
    g = op.g
    out = {r: stages.zeros(r, g.slab_elems) for r in ranks}
    op.solve(yt, out)
    return {r: out[r].cpu().numpy().reshape(g.sz, g.n, g.m) for r in ranks}


def _run_tv(stages, ex, hr, rates, psf, y, x0, iters, to=lambda t: t):
    P = ex.world
    ranks = ex.ranks
    ps, xs = _slabs(psf, P, to), _slabs(x0, P, to)
    yt = {r: to(torch.from_numpy(np.ascontiguousarray(y)).reshape(-1)) for r in ranks}
    tv = D.SlabADMMTV(stages, ex, hr, rates, {r: ps[r] for r in ranks}, yt, {r: xs[r] for r in ranks},
                      2e-3, 0.05, tau=5e-5)
    tv.iterate(iters)
    g = tv.g
    xs_out = {r: tv.x_slab(r).cpu().numpy().reshape(g.sz, g.n, g.m) for r in ranks}
    return xs_out, tv


CASES = [((16, 16, 16), (2, 2, 2), 2), ((16, 16, 32), (2, 2, 4), 2), ((32, 16, 16), (2, 2, 2), 4),
         ((16, 32, 16), (4, 4, 4), 2)]


@pytest.mark.parametrize("hr,rates,P", CASES)
def test_slab_tikhonov_local_numpy(hr, rates, P):
    from dist_numpy_stages import NumpyStages
    psf, y, xbar, _ = _case(hr, rates)
    out = _run_tik(NumpyStages(), D.LocalExchange(P), hr, rates, psf, y, xbar, 1e-2)
    x = np.concatenate([out[p] for p in range(P)], axis=0)
    want = O.tikhonov_fast(y, O.psf_to_spectrum(psf), O.DecimationSpec(hr, rates), 1e-2, xbar)
    assert rel_err(x, want) < 1e-10


@pytest.mark.parametrize("hr,rates,P", CASES)
def test_slab_admm_tv_local_numpy(hr, rates, P):
    from dist_numpy_stages import NumpyStages
    psf, y, _, x0 = _case(hr, rates, 1)
    out, tv = _run_tv(NumpyStages(), D.LocalExchange(P), hr, rates, psf, y, x0, 4)
    x = np.concatenate([out[p] for p in range(P)], axis=0)
    want, rep = O.admm_tv(y, psf, O.DecimationSpec(hr, rates), lam_tv=2e-3, mu=0.05, max_iters=4, rel_tol=0.0,
                          tau=5e-5, init=O.INIT_PROVIDED, init_volume=x0)
    assert rel_err(x, want) < 1e-10
    assert abs(tv.initial_objective - rep.initial_objective) < 1e-10 * abs(rep.initial_objective)
    assert rel_err(tv.objective, rep.objective) < 1e-10
    assert rel_err(tv.primal_residual, rep.primal_residual) < 1e-9


def test_slab_geometry_errors():
    with pytest.raises(ValueError, match="must divide axis 3"):
        D.SlabGeometry((16, 16, 12), (2, 2, 2), 8)
    with pytest.raises(ValueError, match="LR axis 2"):
        D.SlabGeometry((16, 8, 16), (2, 2, 2), 8)
    g = D.SlabGeometry((16, 16, 16), (2, 2, 2), 2)
    # the row sets partition [0, n) and are closed under the bc aliases
    rows = np.concatenate([g.rows(p) for p in range(2)])
    assert sorted(rows.tolist()) == list(range(16))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _gloo_worker(rank, world, port, q):
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parent.parent
    sys.path.insert(0, str(root))
    sys.path.insert(0, str(root / "oracle"))
    sys.path.insert(0, str(root / "tests"))
    import torch.distributed as dist
    from dist_numpy_stages import NumpyStages
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        hr, rates = (16, 16, 16), (2, 2, 2)
        psf, y, xbar, x0 = _case(hr, rates)
        ex = D.TorchExchange()
        xt = _run_tik(NumpyStages(), ex, hr, rates, psf, y, xbar, 1e-2)[rank]
        xv, tv = _run_tv(NumpyStages(), ex, hr, rates, psf, y, x0, 3)
        q.put((rank, xt, xv[rank], tv.objective, tv.primal_residual, tv.initial_objective))
    finally:
        dist.destroy_process_group()


def test_slab_gloo_world2():
    """Two processes over gloo: all-to-all transposes, ring halos, scalar gathers."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=240) for _ in range(2)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    hr, rates = (16, 16, 16), (2, 2, 2)
    psf, y, xbar, x0 = _case(hr, rates)
    xt = np.concatenate([r[1] for r in res], axis=0)
    want = O.tikhonov_fast(y, O.psf_to_spectrum(psf), O.DecimationSpec(hr, rates), 1e-2, xbar)
    assert rel_err(xt, want) < 1e-10
    xv = np.concatenate([r[2] for r in res], axis=0)
    wtv, rep = O.admm_tv(y, psf, O.DecimationSpec(hr, rates), lam_tv=2e-3, mu=0.05, max_iters=3, rel_tol=0.0,
                         tau=5e-5, init=O.INIT_PROVIDED, init_volume=x0)
    assert rel_err(xv, wtv) < 1e-10
    for r in res:  # every rank reports the same scalars
        assert rel_err(r[3], rep.objective) < 1e-10
        assert rel_err(r[4], rep.primal_residual) < 1e-9


# ------------------------------------------------------------------ GPU
GPU_CASES = [((64, 64, 64), (2, 2, 2), 2), ((64, 64, 64), (2, 2, 2), 4), ((32, 32, 64), (2, 2, 4), 2),
             ((64, 64, 32), (4, 4, 4), 2), ((32, 32, 32), (2, 2, 2), 1)]


@pytest.mark.gpu
@pytest.mark.parametrize("hr,rates,P", GPU_CASES)
def test_slab_tikhonov_gpu(V, hr, rates, P):
    ctx = V.default_context()
    st = D.GpuStages({p: ctx for p in range(P)})
    psf, y, xbar, _ = _case(hr, rates)
    cuda = lambda t: t.to("cuda:0")
    out = _run_tik(st, D.LocalExchange(P), hr, rates, psf, y, xbar, 1e-2, to=cuda)
    x = np.concatenate([out[p] for p in range(P)], axis=0)
    want = O.tikhonov_fast(y, O.psf_to_spectrum(psf), O.DecimationSpec(hr, rates), 1e-2, xbar)
    assert rel_err(x, want) < 1e-10


@pytest.mark.gpu
@pytest.mark.parametrize("hr,rates,P", GPU_CASES)
def test_slab_admm_tv_gpu(V, hr, rates, P):
    ctx = V.default_context()
    st = D.GpuStages({p: ctx for p in range(P)})
    psf, y, _, x0 = _case(hr, rates, 1)
    cuda = lambda t: t.to("cuda:0")
    out, tv = _run_tv(st, D.LocalExchange(P), hr, rates, psf, y, x0, 4, to=cuda)
    x = np.concatenate([out[p] for p in range(P)], axis=0)
    want, rep = O.admm_tv(y, psf, O.DecimationSpec(hr, rates), lam_tv=2e-3, mu=0.05, max_iters=4, rel_tol=0.0,
                          tau=5e-5, init=O.INIT_PROVIDED, init_volume=x0)
    assert rel_err(x, want) < 1e-10
    assert rel_err(tv.objective, rep.objective) < 1e-10
    assert rel_err(tv.primal_residual, rep.primal_residual) < 1e-9
