"""Slab-decomposed multi-GPU path: host orchestration.

Volumes are split along axis 3 into P z-slabs, one per rank (one process per
GPU, NCCL through torch.distributed).  A 3D transform is

  local axes 1,2 on the slab -> pack -> all-to-all -> local axis 3

where the all-to-all moves every rank's slab rows into the owner of their
alias-closed row set {g2 + bc*nl : g2 in [p nl/P, (p+1) nl/P)}; the spectral
fold is then purely local (it runs the single-GPU fused kernels on a local
geometry (m, n/P, s)).  The inverse sends whole planes back (no packing) and
unpacks into the inverse axis-2 pass.  ADMM-TV stencil halos (x planes z0-1
and z1, dual plane z0-1) travel peer-to-peer; per-rank scalar partials are
all-gathered and summed in rank order (deterministic for a given P).

The per-rank device work is `GpuStages` (C ABI, include/vsr.h `vsr_slab_*`).
Exchanges are pluggable: `TorchExchange` (torch.distributed; NCCL for CUDA
tensors, gloo for CPU) and `LocalExchange` (P virtual ranks in one process,
plain device copies — exercises the decomposition on a single GPU).
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Dict, List, Optional, Sequence

import numpy as np
import torch


# ---------------------------------------------------------------- geometry
@dataclass
class SlabGeometry:
    hr: tuple
    rates: tuple
    P: int

    def __post_init__(self):
        m, n, s = self.hr
        dr, dc, ds = self.rates
        for a in range(3):
            if self.rates[a] == 0 or self.hr[a] % self.rates[a]:
                raise ValueError("slab: rates must divide the HR dims")
        self.ml, self.nl, self.sl = m // dr, n // dc, s // ds
        if s % self.P:
            raise ValueError(f"slab: P={self.P} must divide axis 3 ({s})")
        if self.nl % self.P:
            raise ValueError(f"slab: P={self.P} must divide the LR axis 2 ({self.nl})")
        self.sz, self.nP, self.nlP = s // self.P, n // self.P, self.nl // self.P
        self.m, self.n, self.s = m, n, s

    @property
    def N(self):
        return self.m * self.n * self.s

    @property
    def slab_elems(self):
        return self.m * self.n * self.sz

    @property
    def plane(self):
        return self.m * self.n

    @property
    def lr(self):
        return (self.ml, self.nl, self.sl)

    def row_of(self, jl, p):
        """global row f2 of local spectral row jl on rank p."""
        return (p * self.nlP + jl % self.nlP) + (jl // self.nlP) * self.nl

    def rows(self, p):
        return np.array([self.row_of(j, p) for j in range(self.nP)])


# ---------------------------------------------------------------- exchanges
class LocalExchange:
    """P virtual ranks in one process: the exchange is a set of copies."""

    def __init__(self, P: int):
        self.world = P
        self.ranks = list(range(P))
        # several virtual ranks own different streams: exchanges synchronise
        # them on the host; a single one keeps everything on its stream
        self.ordered = P == 1

    def all_to_all(self, send: Dict[int, torch.Tensor], recv: Dict[int, torch.Tensor]):
        P = self.world
        for p in self.ranks:
            s = send[p].view(P, -1)
            for q in self.ranks:
                recv[q].view(P, -1)[p].copy_(s[q])

    def ring_shift(self, to_next: Dict[int, torch.Tensor], from_prev: Dict[int, torch.Tensor],
                   to_prev: Optional[Dict[int, torch.Tensor]] = None,
                   from_next: Optional[Dict[int, torch.Tensor]] = None):
        P = self.world
        for p in self.ranks:
            from_prev[(p + 1) % P].copy_(to_next[p])
            if to_prev is not None:
                from_next[(p - 1) % P].copy_(to_prev[p])

    def gather(self, vals: Dict[int, torch.Tensor]) -> List[torch.Tensor]:
        return [vals[p].detach().cpu() for p in range(self.world)]


class TorchExchange:
    """One rank per process over torch.distributed (NCCL for CUDA, gloo for CPU).

    `ordered`: the rank's device work, copies and collectives are all issued on
    the rank's library stream (NCCL orders itself against the current stream),
    so a TV iteration needs no host synchronisation."""

    ordered = True

    def __init__(self):
        import torch.distributed as dist
        self.dist = dist
        self.world = dist.get_world_size()
        self.rank = dist.get_rank()
        self.ranks = [self.rank]

    def all_to_all(self, send, recv):
        r = self.rank
        if self.world == 1:
            recv[r].copy_(send[r])
            return
        self.dist.all_to_all_single(recv[r].view(-1), send[r].view(-1))

    def ring_shift(self, to_next, from_prev, to_prev=None, from_next=None):
        r, P = self.rank, self.world
        if P == 1:
            from_prev[r].copy_(to_next[r])
            if to_prev is not None:
                from_next[r].copy_(to_prev[r])
            return
        d = self.dist
        ops = [d.P2POp(d.isend, to_next[r].contiguous(), (r + 1) % P),
               d.P2POp(d.irecv, from_prev[r], (r - 1) % P)]
        if to_prev is not None:
            ops += [d.P2POp(d.isend, to_prev[r].contiguous(), (r - 1) % P),
                    d.P2POp(d.irecv, from_next[r], (r + 1) % P)]
        for w in d.batch_isend_irecv(ops):
            w.wait()

    def gather(self, vals):
        v = vals[self.rank]
        out = [torch.empty_like(v) for _ in range(self.world)]
        self.dist.all_gather(out, v)
        return [o.detach().cpu() for o in out]


# ---------------------------------------------------------------- GPU stages
class GpuStages:
    """Per-rank device stages through the C ABI (vsr_slab_*); buffers are
    torch CUDA tensors on the rank's device, work is ordered on the vsr
    context stream (torch work in the exchanges is put on the same stream)."""

    def __init__(self, ctx_by_rank: Dict[int, object]):
        from . import volsr as V
        self.V = V
        self.ctx = ctx_by_rank
        self.device = {r: torch.device("cuda", c.device) for r, c in ctx_by_rank.items()}
        self.streams = {r: torch.cuda.ExternalStream(c.stream(), device=self.device[r])
                        for r, c in ctx_by_rank.items()}

    # buffers
    def zeros(self, rank, n, dtype=torch.float64):
        # zero-filled on the rank's library stream, so the fill is ordered
        # before every library kernel that later writes or reads the buffer
        with self.stream(rank):
            return torch.zeros(n, dtype=dtype, device=self.device[rank])

    def stream(self, rank):
        return torch.cuda.stream(self.streams[rank])

    def _d(self, t):
        import ctypes as C
        return C.c_void_p(t.data_ptr())

    def _call(self, name, *args):
        self.V.check(getattr(self.V._lib, name)(*args))

    def _geo(self, g):
        V = self.V
        return V._dims_arr(g.hr), V._dims_arr(g.rates)

    def fft3_full(self, rank, dims, x, real, out, scale):
        self._call("vsr_fft3_d", self.ctx[rank].handle, self.V._dims_arr(dims), self._d(x), int(real),
                   self._d(out), float(scale))

    def fwd_xy_pack(self, rank, g, x, real, work, send):
        hr, rt = self._geo(g)
        self._call("vsr_slab_fwd_xy_pack_d", self.ctx[rank].handle, hr, rt, g.P, self._d(x), int(real),
                   self._d(work), self._d(send))

    def axis3(self, rank, g, W, inverse, scale):
        hr, rt = self._geo(g)
        self._call("vsr_slab_axis3_d", self.ctx[rank].handle, hr, rt, g.P, self._d(W), int(inverse),
                   float(scale))

    def lr_slice(self, rank, g, Yl, Yl_loc):
        hr, rt = self._geo(g)
        self._call("vsr_slab_lr_slice_d", self.ctx[rank].handle, hr, rt, g.P, rank, self._d(Yl),
                   self._d(Yl_loc))

    def tik_fold(self, rank, g, Yl_loc, lam, xbh, reg, W):
        hr, rt = self._geo(g)
        self._call("vsr_slab_tik_fold_d", self.ctx[rank].handle, hr, rt, g.P, self._d(Yl_loc), self._d(lam),
                   self._d(xbh), float(reg), self._d(W))

    def tv_prepare(self, rank, g, lam):
        hr, rt = self._geo(g)
        self._call("vsr_slab_tv_prepare_d", self.ctx[rank].handle, hr, rt, g.P, rank, self._d(lam))

    def tv_release(self, rank, lam):
        self._call("vsr_slab_tv_release_d", self.ctx[rank].handle, self._d(lam))

    def tv_fold(self, rank, g, Yl_loc, lam, W, mu, tau, fwd_scale, fit):
        hr, rt = self._geo(g)
        self._call("vsr_slab_tv_fold_d", self.ctx[rank].handle, hr, rt, g.P, rank, self._d(Yl_loc),
                   self._d(lam), self._d(W), float(mu), float(tau), float(fwd_scale), self._d(fit))

    def unpack_inv_xy(self, rank, g, recv, work, out, scale, sums, bad):
        hr, rt = self._geo(g)
        self._call("vsr_slab_unpack_inv_xy_d", self.ctx[rank].handle, hr, rt, g.P, self._d(recv),
                   self._d(work), self._d(out), float(scale), self._d(sums), self._d(bad))

    def stencil(self, rank, g, init, x_ext, dual_in_ext, dual_out_ext, theta, thr, sums):
        hr, rt = self._geo(g)
        din = self._d(dual_in_ext) if dual_in_ext is not None else None
        self._call("vsr_slab_tv_stencil_d", self.ctx[rank].handle, hr, rt, g.P, int(init), self._d(x_ext),
                   din, self._d(dual_out_ext), self._d(theta), float(thr), self._d(sums))

    def fit(self, rank, g, Yl_loc, lam, xh, out):
        hr, rt = self._geo(g)
        self._call("vsr_slab_fit_d", self.ctx[rank].handle, hr, rt, g.P, self._d(Yl_loc), self._d(lam),
                   self._d(xh), self._d(out))

    def synchronize(self, rank):
        self.ctx[rank].synchronize()


def _ulong_max_tensor(st, rank):
    t = st.zeros(rank, 1, dtype=torch.int64)
    with st.stream(rank):
        t.fill_(-1)  # all ones == ULLONG_MAX
    return t


# ---------------------------------------------------------------- programs
class _Base:
    def __init__(self, stages, exchange, hr, rates):
        self.st = stages
        self.ex = exchange
        self.g = SlabGeometry(tuple(hr), tuple(rates), exchange.world)
        self.ranks = exchange.ranks
        g = self.g
        self.work = {r: stages.zeros(r, 2 * g.slab_elems) for r in self.ranks}
        # one rank: the all-to-all is the identity, so the xy stage packs straight
        # into the spectral buffer and the inverse unpacks straight from it
        self.solo = exchange.world == 1
        self.send = {} if self.solo else {r: stages.zeros(r, 2 * g.slab_elems) for r in self.ranks}
        self.recv = {} if self.solo else {r: stages.zeros(r, 2 * g.slab_elems) for r in self.ranks}

    def _each(self, fn):
        for r in self.ranks:
            with self.st.stream(r):
                fn(r)

    def _sync_all(self):
        for r in self.ranks:
            self.st.synchronize(r)

    def _gather(self, vals):
        """All-gather of per-rank device scalars, issued on the rank's library
        stream (NCCL orders itself against the current stream) so it reads the
        values the rank's kernels wrote."""
        if self._ordered():
            with self.st.stream(self.ranks[0]):
                return self.ex.gather(vals)
        self._sync_all()
        return self.ex.gather(vals)

    def forward3(self, slabs: Dict[int, torch.Tensor], real: bool, scale: float,
                 out: Dict[int, torch.Tensor]):
        """Distributed forward 3D FFT: z-slabs -> local spectral layout (m, n/P, s)."""
        dst = out if self.solo else self.send
        self._each(lambda r: self.st.fwd_xy_pack(r, self.g, slabs[r], real, self.work[r], dst[r]))
        if not self.solo:
            self._exchange(self.send, out)
        self._each(lambda r: self.st.axis3(r, self.g, out[r], False, scale))

    def _ordered(self):
        return getattr(self.ex, "ordered", False) and len(self.ranks) == 1

    def _exchange(self, send, recv):
        if self._ordered():
            r = self.ranks[0]
            with self.st.stream(r):
                self.ex.all_to_all(send, recv)
            return
        for r in self.ranks:
            self.st.synchronize(r)
        self.ex.all_to_all(send, recv)
        for r in self.ranks:
            if recv[r].is_cuda:
                torch.cuda.synchronize(recv[r].device)

    def _lr_spectrum(self, y_full: Dict[int, torch.Tensor]):
        g = self.g
        Nl = g.ml * g.nl * g.sl
        self.Yl_full = {r: self.st.zeros(r, 2 * Nl) for r in self.ranks}
        self.Yl = {r: self.st.zeros(r, 2 * g.ml * g.nlP * g.sl) for r in self.ranks}

        def f(r):
            self.st.fft3_full(r, g.lr, y_full[r], True, self.Yl_full[r], 1.0 / math.sqrt(Nl))
            self.st.lr_slice(r, g, self.Yl_full[r], self.Yl[r])
        self._each(f)

    def _inverse_to_slabs(self, W, out_slabs, scale, sums, bad):
        src = W if self.solo else self.recv
        if not self.solo:
            self._exchange(W, self.recv)
        self._each(lambda r: self.st.unpack_inv_xy(r, self.g, src[r], self.work[r], out_slabs[r], scale,
                                                   sums[r], bad[r]))

    def _check_status(self, sums_by_rank, where):
        """Imaginary-residue ratio (fft.cpp:89-93) and first non-finite index
        (volume.cpp:31-36) of the last inverse, summed over ranks in rank order.
        Every rank's work is complete when this returns (x is safe to read on
        any stream)."""
        g = self.g
        self._sync_all()
        sums = self._gather(sums_by_rank)
        im2 = sum(float(s[0]) for s in sums)
        tot2 = sum(float(s[1]) for s in sums)
        from .volsr import NumericError
        if tot2 > 0.0 and math.sqrt(im2 / tot2) > 1e-8:
            raise NumericError(f"ifft3_real: imaginary residue {math.sqrt(im2 / tot2):f} exceeds 0.000000 "
                               "(spectral bookkeeping bug?)")
        bads = [int(b[0]) for b in self._gather(self.bad)]
        for p, b in enumerate(bads):
            if b != -1:
                raise NumericError(f"{where}: non-finite value at flat index {p * g.slab_elems + b}")


class SlabTikhonov(_Base):
    """Distributed TikhonovOperator (solvers.cpp:36-67): Lambda and fft3(xbar)
    live in the local spectral layout; solve(y) returns the rank's x slab."""

    def __init__(self, stages, exchange, hr, rates, psf_slabs, reg, xbar_slabs):
        super().__init__(stages, exchange, hr, rates)
        if not (reg > 0.0):
            raise ValueError(f"lambda must be positive, got {reg}")
        g = self.g
        self.reg = reg
        self.lam = {r: stages.zeros(r, 2 * g.slab_elems) for r in self.ranks}
        self.xbh = {r: stages.zeros(r, 2 * g.slab_elems) for r in self.ranks}
        self.forward3(psf_slabs, True, 1.0, self.lam)                    # Lambda = DFT(psf)
        self.forward3(xbar_slabs, True, 1.0 / math.sqrt(g.N), self.xbh)  # fft3(xbar)
        self.W = {r: stages.zeros(r, 2 * g.slab_elems) for r in self.ranks}
        self.sums = {r: stages.zeros(r, 2) for r in self.ranks}
        self.bad = {r: _ulong_max_tensor(stages, r) for r in self.ranks}

    def solve(self, y_full: Dict[int, torch.Tensor], x_slabs: Dict[int, torch.Tensor]):
        g = self.g
        self._lr_spectrum(y_full)
        self._each(lambda r: self.st.tik_fold(r, g, self.Yl[r], self.lam[r], self.xbh[r], self.reg, self.W[r]))
        self._each(lambda r: self.bad[r].fill_(-1))  # on the rank stream, ahead of the unpack that sets it
        self._inverse_to_slabs(self.W, x_slabs, 1.0 / math.sqrt(g.N), self.sums, self.bad)
        self._check_status(self.sums, "tikhonov_fast")

class SlabADMMTV(_Base):
    """Distributed admm_tv (solvers.cpp:321-411) with rel_tol = 0 semantics
    (fixed iteration count); report holds objective and primal residual per
    iteration, summed over ranks in rank order."""

    def __init__(self, stages, exchange, hr, rates, psf_slabs, y_full, x0_slabs, lam_tv, mu, tau=None):
        super().__init__(stages, exchange, hr, rates)
        if not (lam_tv > 0.0):
            raise ValueError(f"lambda must be positive, got {lam_tv}")
        if not (mu > 0.0):
            raise ValueError(f"mu must be positive, got {mu}")
        g = self.g
        self.lam_tv, self.mu = lam_tv, mu
        self.tau = 1e-8 * mu if tau is None else tau
        pl = g.plane
        self.lam = {r: stages.zeros(r, 2 * g.slab_elems) for r in self.ranks}
        self.forward3(psf_slabs, True, 1.0, self.lam)
        self._each(lambda r: self.st.tv_prepare(r, g, self.lam[r]))  # fold tables for this Lambda
        self._lr_spectrum(y_full)
        self.x_ext = {r: stages.zeros(r, pl * (g.sz + 2)) for r in self.ranks}
        self.dual = [{r: stages.zeros(r, 3 * pl * (g.sz + 1)) for r in self.ranks} for _ in range(2)]
        self.cur = 0
        self.theta = {r: stages.zeros(r, g.slab_elems) for r in self.ranks}
        self.W = {r: stages.zeros(r, 2 * g.slab_elems) for r in self.ranks}
        self.s_fit = {r: stages.zeros(r, 1) for r in self.ranks}
        self.s_res = {r: stages.zeros(r, 2) for r in self.ranks}
        self.s_st = {r: stages.zeros(r, 4) for r in self.ranks}
        self.bad = {r: _ulong_max_tensor(stages, r) for r in self.ranks}
        self.halo_lo = {r: stages.zeros(r, pl) for r in self.ranks}
        self.halo_hi = {r: stages.zeros(r, pl) for r in self.ranks}
        self.dhalo_out = {r: stages.zeros(r, 3 * pl) for r in self.ranks}
        self.dhalo_in = {r: stages.zeros(r, 3 * pl) for r in self.ranks}
        # buffers above were zeroed on torch's current stream: order the rank
        # stream after them before any library kernel touches them
        self._torch_sync()
        self._each(lambda r: self.x_ext[r][pl:pl * (g.sz + 1)].copy_(x0_slabs[r].reshape(-1)))
        # initial objective: data term from fft3(x0), TV from the init stencil
        self.forward3({r: self.x_ext[r][pl:pl * (g.sz + 1)] for r in self.ranks}, True, 1.0 / math.sqrt(g.N),
                      self.W)
        self._each(lambda r: self.st.fit(r, g, self.Yl[r], self.lam[r], self.W[r], self.s_fit[r]))
        self._halo_x()
        self._each(lambda r: self.st.stencil(r, g, True, self.x_ext[r], None, self.dual[0][r], self.theta[r],
                                             lam_tv / mu, self.s_st[r]))
        fit = sum(float(v[0]) for v in self._gather(self.s_fit))
        tv = sum(float(v[1]) for v in self._gather(self.s_st))
        self.initial_objective = 0.5 * fit + lam_tv * tv
        self.objective, self.primal_residual = [], []

    def _torch_sync(self):
        for r in self.ranks:
            if self.x_ext[r].is_cuda:
                torch.cuda.synchronize(self.x_ext[r].device)

    def _halo_x(self):
        g, pl = self.g, self.g.plane
        ordered = self._ordered()
        if not ordered:
            self._sync_all()
        lo_src = {r: self.x_ext[r][pl:2 * pl] for r in self.ranks}                    # first slab plane
        hi_src = {r: self.x_ext[r][g.sz * pl:(g.sz + 1) * pl] for r in self.ranks}     # last slab plane

        def body():
            self.ex.ring_shift(hi_src, self.halo_lo, lo_src, self.halo_hi)
            for r in self.ranks:
                self.x_ext[r][0:pl].copy_(self.halo_lo[r])
                self.x_ext[r][(g.sz + 1) * pl:(g.sz + 2) * pl].copy_(self.halo_hi[r])
        if ordered:
            with self.st.stream(self.ranks[0]):
                body()
        else:
            body()
            self._torch_sync()

    def _halo_dual(self, d):
        g, pl = self.g, self.g.plane
        ext = (g.sz + 1) * pl
        ordered = self._ordered()
        if not ordered:
            self._sync_all()

        def body():
            for r in self.ranks:
                for c in range(3):
                    self.dhalo_out[r][c * pl:(c + 1) * pl].copy_(
                        d[r][c * ext + g.sz * pl:c * ext + (g.sz + 1) * pl])
            self.ex.ring_shift(self.dhalo_out, self.dhalo_in)
            for r in self.ranks:
                for c in range(3):
                    d[r][c * ext:c * ext + pl].copy_(self.dhalo_in[r][c * pl:(c + 1) * pl])
        if ordered:
            with self.st.stream(self.ranks[0]):
                body()
        else:
            body()
            self._torch_sync()

    def iterate(self, k: int = 1):
        g, pl = self.g, self.g.plane
        s = 1.0 / math.sqrt(g.N)
        # per-iteration scalars stay on the device (fit, residual^2, TV); gathered once after the loop
        hist = {}
        self._each(lambda r: hist.__setitem__(r, self.st.zeros(r, 3 * k)))
        for it in range(k):
            self.forward3_theta()
            self._each(lambda r: self.st.tv_fold(r, g, self.Yl[r], self.lam[r], self.W[r], self.mu, self.tau, s,
                                                 self.s_fit[r]))
            self._each(lambda r: self.bad[r].fill_(-1))
            self._inverse_to_slabs(self.W, {r: self.x_ext[r][pl:pl * (g.sz + 1)] for r in self.ranks}, s,
                                   self.s_res, self.bad)
            self._halo_x()
            din, dout = self.dual[self.cur], self.dual[1 - self.cur]
            self._halo_dual(din)
            self._each(lambda r: self.st.stencil(r, g, False, self.x_ext[r], din[r], dout[r], self.theta[r],
                                                 self.lam_tv / self.mu, self.s_st[r]))
            self.cur = 1 - self.cur

            def keep(r, it=it):
                hist[r][3 * it:3 * it + 1].copy_(self.s_fit[r][0:1])
                hist[r][3 * it + 1:3 * it + 3].copy_(self.s_st[r][0:2])
            self._each(keep)
        h = self._gather(hist)  # rank order: deterministic sums for a given P
        # solvers.cpp:408 require_finite(x, "admm_tv"), plus the residue check of
        # the last inverse (fft.cpp:89-93), as the single-GPU path does
        self._check_status(self.s_res, "admm_tv")
        for it in range(k):
            fit = sum(float(v[3 * it]) for v in h)
            res2 = sum(float(v[3 * it + 1]) for v in h)
            tv = sum(float(v[3 * it + 2]) for v in h)
            self.objective.append(0.5 * fit + self.lam_tv * tv)
            self.primal_residual.append(math.sqrt(res2))

    def close(self):
        """Frees the rank's cached fold tables (vsr_slab_tv_prepare_d)."""
        lam, self.lam = getattr(self, "lam", None), None
        if lam:
            for r in self.ranks:
                self.st.tv_release(r, lam[r])

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def forward3_theta(self):
        g = self.g
        dst = self.W if self.solo else self.send
        self._each(lambda r: self.st.fwd_xy_pack(r, g, self.theta[r], True, self.work[r], dst[r]))
        if not self.solo:
            self._exchange(self.send, self.W)

    def x_slab(self, r):
        pl = self.g.plane
        return self.x_ext[r][pl:pl * (self.g.sz + 1)]
