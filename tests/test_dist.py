"""Slab-sharded multi-rank path (csrc/slab.cu, dist.py).

CPU (no GPU): the plane partition (vsr_slab_plan, host code of the library)
and a real 2-process gloo run of the decomposition restated in numpy: each
process keeps its y-slab, the axis-3 half spectrum goes plane by plane to
the plane owners, the fold runs only on owned planes (conjugate mirrors of
class -g3 are local by construction), the result comes back and the stencil
exchanges its y halos.  Checked against the single-volume oracle.

GPU: the C++ slab solvers through the C ABI on one B200 - P virtual ranks
(local comm: the same kernels, peer pointers and stage order as the
multi-GPU run), a 1-rank NCCL comm, and TWO PROCESSES sharing the GPU over a
gloo host comm (CUDA IPC peer buffers; barriers on the host, so no kernel
waits on another).  Checked against the oracle and bitwise against the
single-GPU path."""
import os
import socket
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

from conftest import rel_err

import volsr_oracle as O
from paper_2010_15491_b200 import dist as D
from paper_2010_15491_b200 import synth

ROOT = Path(__file__).resolve().parent.parent
TOL = 1e-10


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _case(hr, rates, seed=0, ksz=(5, 5, 5), sigma=(1.2, 1.2, 1.5)):
    rng = np.random.default_rng(seed)
    m, n, s = hr
    psf = O.make_gaussian_psf(ksz, sigma, hr)
    y = rng.uniform(0, 1, (s // rates[2], n // rates[1], m // rates[0]))
    x0 = rng.uniform(0, 1, (s, n, m))
    return psf, y, x0


# ------------------------------------------------------------------ plan (CPU)
@pytest.mark.parametrize("hr,rates", [((512, 512, 256), (2, 2, 4)), ((1024, 1024, 1024), (2, 2, 2)),
                                      ((64, 64, 64), (4, 4, 4)), ((64, 32, 32), (2, 2, 2))])
@pytest.mark.parametrize("P", [1, 2, 4, 8])
def test_plane_partition(hr, rates, P):
    m, n, s = hr
    if n % P:
        pytest.skip("P does not divide n")
    own = D.plane_owners(hr, rates, P)
    sl = s // rates[2]
    assert own.shape == (s // 2 + 1,) and set(own.tolist()) == set(range(P))
    # every LR class and its conjugate class live on one rank (fold alias sets are local)
    cls_owner = {}
    for f, r in enumerate(own):
        cls_owner.setdefault(f % sl, set()).add(int(r))
    for g, rs in cls_owner.items():
        assert len(rs) == 1
        if (sl - g) % sl in cls_owner:
            assert cls_owner[(sl - g) % sl] == rs
    counts = np.bincount(own, minlength=P)
    assert counts.max() <= 1.35 * (s // 2 + 1) / P + 4


def test_plane_partition_errors():
    from paper_2010_15491_b200 import volsr as V
    with pytest.raises(V.ShapeError, match="must divide axis 2"):
        D.plane_owners((64, 48, 64), (2, 2, 2), 5)
    with pytest.raises(V.ShapeError, match="conjugate LR plane classes"):
        D.plane_owners((64, 64, 16), (2, 2, 2), 8)


# ------------------------------------------------------------------ numpy decomposition on 2 gloo processes (CPU)
_NUMPY_WORKER = r'''
import os, sys, numpy as np
sys.path.insert(0, {root!r}); sys.path.insert(0, {root!r} + "/oracle")
import torch, torch.distributed as dist
import volsr_oracle as O
from paper_2010_15491_b200 import dist as D
rank, P = int(sys.argv[1]), int(sys.argv[2])
dist.init_process_group("gloo", init_method="tcp://127.0.0.1:{port}", rank=rank, world_size=P)
hr, rates = {hr}, {rates}
m, n, s = hr; dr, dc, ds = rates; ml, nl, sl = m // dr, n // dc, s // ds; nP = n // P
rng = np.random.default_rng(0)
psf = O.make_gaussian_psf((5, 5, 5), (1.2, 1.2, 1.5), hr)
y = rng.uniform(0, 1, (sl, nl, ml)); x0 = rng.uniform(0, 1, (s, n, m))
mu, lam_tv, tau, iters = 0.05, 2e-3, 5e-5, 2
own = D.plane_owners(hr, rates, P)
mine = [f for f in range(s // 2 + 1) if own[f] == rank]
lam = O.psf_to_spectrum(psf); N = m * n * s; d = dr * dc * ds
yl = np.fft.fftn(y, norm="ortho") / np.sqrt(d)
gam = O.make_gamma(hr, tau)
def allg(a):
    t = torch.from_numpy(np.ascontiguousarray(a)); out = [torch.empty_like(t) for _ in range(P)]
    dist.all_gather(out, t); return [o.numpy() for o in out]
def x_update(theta_slab):
    # axis-3 half spectrum of this rank's rows -> plane owners
    h = np.fft.rfft(theta_slab, axis=0) / np.sqrt(N)
    rows = allg(h)                                     # every rank's rows of every half plane
    W = {{f: np.concatenate([rows[q][f] for q in range(P)], axis=0) for f in mine}}
    W = {{f: np.fft.fft(np.fft.fft(W[f], axis=0), axis=1) for f in mine}}  # axes 2, 1: full (f2, f1)
    def row(f3):                                       # plane f3 of the full spectrum, from owned planes only
        if f3 <= s // 2: return W[f3]
        src = W[s - f3]                                # conj(X(-f1, -f2, s - f3)): class -g3, owned here
        return np.conj(np.roll(src[::-1, ::-1], (1, 1), axis=(0, 1)))
    out = {{}}
    for g3 in sorted({{f % sl for f in mine}}):
        fs = [g3 + bs * sl for bs in range(ds)]
        K = np.stack([row(f) for f in fs]); L = np.stack([lam[f] for f in fs]); G = np.stack([gam[f] for f in fs])
        Kb = K.reshape(ds, dc, nl, dr, ml); Lb = L.reshape(ds, dc, nl, dr, ml); Gb = G.reshape(ds, dc, nl, dr, ml)
        Yb = yl[g3][None, None, :, None, :]
        kh = np.conj(Lb) * Yb + mu * Kb; gh = Gb * kh
        den = (Gb * np.abs(Lb) ** 2).sum(axis=(0, 1, 3)) + mu * d
        w = (Lb * gh).sum(axis=(0, 1, 3)) / den
        xh = (gh - Gb * np.conj(Lb) * w[None, None, :, None, :]) / mu
        xh = xh.reshape(ds, n, m)
        for bs, f in enumerate(fs):
            if f <= s // 2: out[f] = xh[bs]
    # inverse axes 1, 2 on owned planes, rows back to their y-slab ranks, inverse axis 3
    back = {{f: np.fft.ifft(np.fft.ifft(out[f], axis=1), axis=0) for f in mine}}
    send = np.zeros((s // 2 + 1, n, m), complex)
    for f in mine: send[f] = back[f]
    allp = allg(send)
    half = sum(allp)[:, rank * nP:(rank + 1) * nP, :]
    return np.fft.irfft(half, n=s, axis=0) * np.sqrt(N)
def halo(x):                                           # rows -1 and nP from the ring neighbours
    lo, hi = allg(x[:, -1, :]), allg(x[:, 0, :])
    return lo[(rank - 1) % P], hi[(rank + 1) % P]
xs = np.ascontiguousarray(x0[:, rank * nP:(rank + 1) * nP, :])
ext = lambda a, lo, hi: np.concatenate([lo[:, None], a, hi[:, None]], axis=1)
lo, hi = halo(xs); xe = ext(xs, lo, hi)
fwd = lambda e: (np.roll(e, -1, 2)[:, 1:-1] - e[:, 1:-1], e[:, 2:] - e[:, 1:-1], np.roll(e, -1, 0)[:, 1:-1] - e[:, 1:-1])
u = list(fwd(xe)); dual = [np.zeros_like(xs) for _ in range(3)]
for it in range(iters):
    rho = [u[a] - dual[a] for a in range(3)]
    rl = [allg(r[:, -1, :]) for r in rho]
    theta = (np.roll(rho[0], 1, 2) - rho[0]) + (np.concatenate([rl[1][(rank - 1) % P][:, None], rho[1][:, :-1]], 1) - rho[1]) \
        + (np.roll(rho[2], 1, 0) - rho[2])
    xs = x_update(theta)
    lo, hi = halo(xs); lx = fwd(ext(xs, lo, hi))
    nu = [lx[a] + dual[a] for a in range(3)]
    u = list(O.tv_shrink(nu[0], nu[1], nu[2], lam_tv / mu)); dual = [nu[a] - u[a] for a in range(3)]
full = allg(xs)
if rank == 0:
    x = np.concatenate(full, axis=1)
    spec = O.DecimationSpec(hr, rates)
    want, _ = O.admm_tv(y, psf, spec, lam_tv=lam_tv, mu=mu, max_iters=iters, rel_tol=0.0, tau=tau, init=2, init_volume=x0)
    err = float(np.linalg.norm(x - want) / np.linalg.norm(want))
    print("ERR", err)
    assert err < 1e-10, err
dist.destroy_process_group()
'''


@pytest.mark.parametrize("hr,rates", [((64, 16, 16), (2, 2, 2)), ((64, 16, 32), (2, 2, 4))])
def test_numpy_decomposition_two_gloo_processes(tmp_path, hr, rates):
    port = _free_port()
    code = _NUMPY_WORKER.format(root=str(ROOT), port=port, hr=hr, rates=rates)
    script = tmp_path / "worker.py"
    script.write_text(code)
    env = {**os.environ, "CUDA_VISIBLE_DEVICES": ""}
    procs = [subprocess.Popen([sys.executable, str(script), str(r), "2"], stdout=subprocess.PIPE,
                              stderr=subprocess.PIPE, text=True, env=env) for r in range(2)]
    outs = [p.communicate(timeout=600) for p in procs]
    for p, (o, e) in zip(procs, outs):
        assert p.returncode == 0, o + e
    assert "ERR" in outs[0][0]


# ------------------------------------------------------------------ GPU: local comm (P virtual ranks)
GPU_CASES = [((64, 32, 32), (2, 2, 2)), ((64, 64, 64), (4, 4, 4)), ((64, 32, 64), (2, 2, 4)),
             # 1024-point axis-3 lines: the wide forward paired pass storing into the owners' buffers
             ((64, 16, 1024), (2, 2, 2))]


@pytest.mark.gpu
@pytest.mark.parametrize("hr,rates", GPU_CASES)
@pytest.mark.parametrize("P", [1, 2, 4])
def test_slab_admm_tv_local_ranks(V, hr, rates, P):
    psf, y, x0 = _case(hr, rates)
    spec, ospec = V.DecimationSpec(hr, rates), O.DecimationSpec(hr, rates)
    cfg = V.TvAdmmConfig(lambda_=2e-3, mu=0.05, max_iters=3, rel_tol=0.0, tau=5e-5, init=V.INIT_PROVIDED,
                         init_volume=x0)
    comm = D.SlabComm.local(P)
    xs, rep = D.admm_tv(comm, y, psf, spec, cfg, init_slabs=D.split_slabs(x0, P))
    x = D.join_slabs(xs)
    want, wrep = O.admm_tv(y, psf, ospec, lam_tv=2e-3, mu=0.05, max_iters=3, rel_tol=0.0, tau=5e-5,
                           init=O.INIT_PROVIDED, init_volume=x0)
    assert rel_err(x, want) < TOL
    assert rep.iterations == 3
    np.testing.assert_allclose(rep.objective, wrep.objective, rtol=TOL)
    np.testing.assert_allclose(rep.primal_residual, wrep.primal_residual, rtol=1e-9)
    assert abs(rep.initial_objective - wrep.initial_objective) <= TOL * abs(wrep.initial_objective)
    # the per-voxel work is the single-GPU path's kernels on the same tiles: x is bit-identical
    # (when the slab height is not a multiple of the stencil's 8-row tile, the rows whose
    # lower neighbour is computed by the tile-halo code differ between the two paths, and
    # that code rounds its shrink differently in the last bit)
    one, _ = V.admm_tv(y, psf, spec, cfg)
    if (hr[1] // P) % 8 == 0:
        assert x.tobytes() == one.tobytes()
    else:
        assert rel_err(x, one) < 1e-13


@pytest.mark.gpu
@pytest.mark.parametrize("init", ["zero", "upsampled"])
def test_slab_admm_tv_inits_and_rel_tol(V, init):
    hr, rates = (64, 64, 32), (2, 2, 2)
    psf, y, _ = _case(hr, rates, seed=3)
    spec, ospec = V.DecimationSpec(hr, rates), O.DecimationSpec(hr, rates)
    mode = V.INIT_ZERO if init == "zero" else V.INIT_UPSAMPLED
    cfg = V.TvAdmmConfig(lambda_=2e-3, mu=0.05, max_iters=40, rel_tol=1e-2, tau=5e-5, init=mode)
    xs, rep = D.admm_tv(D.SlabComm.local(2), y, psf, spec, cfg)
    want, wrep = O.admm_tv(y, psf, ospec, lam_tv=2e-3, mu=0.05, max_iters=40, rel_tol=1e-2, tau=5e-5, init=mode)
    assert rep.iterations == wrep.iterations < 40  # the same stop iteration (solvers.cpp:405)
    assert rel_err(D.join_slabs(xs), want) < TOL
    np.testing.assert_allclose(rep.objective, wrep.objective, rtol=TOL)


@pytest.mark.gpu
@pytest.mark.parametrize("hr,rates", GPU_CASES)
@pytest.mark.parametrize("P", [1, 2, 4])
def test_slab_tikhonov_local_ranks(V, hr, rates, P):
    psf, y, x0 = _case(hr, rates, seed=5)
    lam = O.psf_to_spectrum(psf)
    spec, ospec = V.DecimationSpec(hr, rates), O.DecimationSpec(hr, rates)
    comm = D.SlabComm.local(P)
    for xbar in (O.zero_fill_upsample(y, ospec), x0):  # lattice prior and a general one
        op = D.SlabTikhonov(comm, lam, spec, 1e-3, D.split_slabs(xbar, P))
        V.reset_fft_counters()
        x = D.join_slabs(op.solve(y))
        assert V.fft_counters() == {"forward": 1, "inverse": 1}
        assert rel_err(x, O.tikhonov_fast(y, lam, ospec, 1e-3, xbar)) < TOL
        y2 = np.random.default_rng(9).uniform(0, 1, y.shape)  # a second y through the same operator
        assert rel_err(D.join_slabs(op.solve(y2)), O.tikhonov_fast(y2, lam, ospec, 1e-3, xbar)) < TOL
        op.close()


@pytest.mark.gpu
def test_slab_dense_lambda_and_errors(V):
    """A non-separable (random) PSF: the dense Lambda planes of each rank's classes."""
    hr, rates = (64, 32, 32), (2, 2, 2)
    rng = np.random.default_rng(4)
    w = rng.uniform(0, 1, 27)
    psf = O.make_gaussian_psf((3, 3, 3), (0, 0, 0), hr, weights=w)
    y = rng.uniform(0, 1, (16, 16, 32))
    spec, ospec = V.DecimationSpec(hr, rates), O.DecimationSpec(hr, rates)
    cfg = V.TvAdmmConfig(lambda_=2e-3, mu=0.05, max_iters=2, rel_tol=0.0, tau=5e-5, init=V.INIT_UPSAMPLED)
    xs, _ = D.admm_tv(D.SlabComm.local(4), y, psf, spec, cfg)
    want, _ = O.admm_tv(y, psf, ospec, lam_tv=2e-3, mu=0.05, max_iters=2, rel_tol=0.0, tau=5e-5, init=1)
    assert rel_err(D.join_slabs(xs), want) < TOL
    y_bad = y.copy()
    y_bad[3, 4, 5] = np.nan
    with pytest.raises(V.NumericError, match="admm_tv: non-finite value at flat index"):
        D.admm_tv(D.SlabComm.local(2), y_bad, psf, spec, cfg)
    with pytest.raises(ValueError, match="mu must be positive"):
        D.admm_tv(D.SlabComm.local(2), y, psf, spec, V.TvAdmmConfig(lambda_=2e-3, mu=0.0, max_iters=2))
    with pytest.raises(V.ShapeError):
        D.admm_tv(D.SlabComm.local(3), y, psf, spec, cfg)


@pytest.mark.gpu
def test_slab_nccl_comm_single_rank(V):
    import torch.distributed as dist
    if not dist.is_initialized():
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{_free_port()}", rank=0, world_size=1)
    hr, rates = (64, 64, 64), (4, 4, 4)
    psf, y, x0 = _case(hr, rates, seed=6)
    spec, ospec = V.DecimationSpec(hr, rates), O.DecimationSpec(hr, rates)
    comm = D.SlabComm.nccl()
    assert (comm.world, comm.rank, comm.local) == (1, 0, 1)
    cfg = V.TvAdmmConfig(lambda_=2e-3, mu=0.05, max_iters=3, rel_tol=0.0, tau=5e-5, init=V.INIT_PROVIDED,
                         init_volume=x0)
    xs, rep = D.admm_tv(comm, y, psf, spec, cfg, init_slabs=[x0])
    want, _ = O.admm_tv(y, psf, ospec, lam_tv=2e-3, mu=0.05, max_iters=3, rel_tol=0.0, tau=5e-5, init=2,
                        init_volume=x0)
    assert rel_err(xs[0], want) < TOL
    comm.close()
    dist.destroy_process_group()


_GPU_WORKER = r'''
import os, sys, numpy as np
sys.path.insert(0, {root!r}); sys.path.insert(0, {root!r} + "/oracle"); sys.path.insert(0, {root!r} + "/tests")
import torch.distributed as dist
rank, P = int(sys.argv[1]), int(sys.argv[2])
dist.init_process_group("gloo", init_method="tcp://127.0.0.1:{port}", rank=rank, world_size=P)
import volsr_oracle as O
from conftest import rel_err
from paper_2010_15491_b200 import volsr as V, dist as D
hr, rates = {hr}, {rates}
rng = np.random.default_rng(0)
m, n, s = hr
psf = O.make_gaussian_psf((5, 5, 5), (1.2, 1.2, 1.5), hr)
y = rng.uniform(0, 1, (s // rates[2], n // rates[1], m // rates[0])); x0 = rng.uniform(0, 1, (s, n, m))
spec = V.DecimationSpec(hr, rates)
comm = D.SlabComm.host()
cfg = V.TvAdmmConfig(lambda_=2e-3, mu=0.05, max_iters=3, rel_tol=0.0, tau=5e-5, init=V.INIT_PROVIDED, init_volume=x0)
xs, rep = D.admm_tv(comm, y, psf, spec, cfg, init_slabs=[D.split_slabs(x0, P)[rank]])
lam = O.psf_to_spectrum(psf)
op = D.SlabTikhonov(comm, lam, spec, 1e-3, [D.split_slabs(O.zero_fill_upsample(y, O.DecimationSpec(hr, rates)), P)[rank]])
xt = op.solve(y)[0]
op.close()
import torch
allx = [torch.empty(xs[0].size, dtype=torch.float64) for _ in range(P)]
dist.all_gather(allx, torch.from_numpy(xs[0].reshape(-1)))
allt = [torch.empty(xt.size, dtype=torch.float64) for _ in range(P)]
dist.all_gather(allt, torch.from_numpy(xt.reshape(-1)))
if rank == 0:
    ospec = O.DecimationSpec(hr, rates)
    x = D.join_slabs([a.numpy().reshape(xs[0].shape) for a in allx])
    want, wrep = O.admm_tv(y, psf, ospec, lam_tv=2e-3, mu=0.05, max_iters=3, rel_tol=0.0, tau=5e-5, init=2, init_volume=x0)
    e1 = rel_err(x, want)
    e2 = rel_err(D.join_slabs([a.numpy().reshape(xt.shape) for a in allt]), O.tikhonov_fast(y, lam, ospec, 1e-3, O.zero_fill_upsample(y, ospec)))
    e3 = max(abs(a - b) / abs(b) for a, b in zip(rep.objective, wrep.objective))
    print("ERR", e1, e2, e3)
    assert e1 < 1e-10 and e2 < 1e-10 and e3 < 1e-10
comm.close()
dist.destroy_process_group()
'''


@pytest.mark.gpu
@pytest.mark.parametrize("hr,rates", [((64, 32, 32), (2, 2, 2)), ((64, 64, 64), (4, 4, 4))])
def test_slab_two_processes_one_gpu_host_comm(tmp_path, hr, rates):
    """Two ranks as two processes on one GPU: buffers shared by CUDA IPC, the
    kernels' peer stores/loads cross process boundaries, barriers on the host
    (gloo) - no kernel ever waits on the other process."""
    port = _free_port()
    script = tmp_path / "gpu_worker.py"
    script.write_text(_GPU_WORKER.format(root=str(ROOT), port=port, hr=hr, rates=rates))
    procs = [subprocess.Popen([sys.executable, str(script), str(r), "2"], stdout=subprocess.PIPE,
                              stderr=subprocess.PIPE, text=True) for r in range(2)]
    try:
        outs = [p.communicate(timeout=600) for p in procs]
    finally:
        for p in procs:
            if p.poll() is None:
                p.kill()
    for p, (o, e) in zip(procs, outs):
        assert p.returncode == 0, o + e[-3000:]
    assert "ERR" in outs[0][0]
