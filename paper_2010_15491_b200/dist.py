"""Slab-sharded multi-GPU path — Python mirror of the C ABI
(include/vsr.h `vsr_comm_*`, `vsr_slab_*`; implementation csrc/slab.cu).

Rank p owns the HR rows y in [p n/P, (p+1) n/P) of every plane, i.e. an
(s, n/P, m) array ("slab").  The half spectrum along axis 3 is split by plane
over conjugate LR class pairs so every fold alias set is rank-local; the
exchanges are the CUDA kernels' own NVLink peer stores/loads between
stream-ordered barriers (no packing, no staging copies).  One process per
GPU; the host-side orchestration lives in C++.

Communicators:
  SlabComm.local(P)        P virtual ranks on this process's device (stage by
                           stage in stream order; tests and P = 1 timing)
  SlabComm.nccl()          one rank per process over NCCL (torch.distributed
                           initialised; rank 0's NCCL unique id is broadcast)
  SlabComm.host(group)     one rank per process, barriers / all-gathers through
                           a torch.distributed process group (e.g. gloo): the
                           multi-process tests on a single GPU

Entry points mirror the reference solver API (solvers.hpp): `admm_tv(comm, y,
psf, spec, cfg)` -> (x slabs, SolveReport) and `SlabTikhonov(comm, lam, spec,
reg, xbar slabs).solve(y)` -> x slabs.  y, psf and Lambda are full volumes on
every rank; slab arguments/results are lists with one entry per LOCAL rank.
"""
from __future__ import annotations

import ctypes as C
from typing import List, Optional, Sequence

import numpy as np

from . import volsr as V

_lib, _vp, _dp, _szp = V._lib, V._vp, V._dp, V._szp

_BARRIER_FN = C.CFUNCTYPE(C.c_int, C.c_void_p)
_GATHER_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t)


class _HostExchange(C.Structure):
    _fields_ = [("barrier", _BARRIER_FN), ("all_gather", _GATHER_FN)]


def _sig(name, args, res=C.c_int):
    f = getattr(_lib, name)
    f.argtypes = args
    f.restype = res


_pp = C.POINTER(_dp)
_sig("vsr_comm_local", [_vp, C.c_int, C.POINTER(_vp)])
_sig("vsr_nccl_unique_id", [C.c_char_p])
_sig("vsr_comm_nccl", [_vp, C.c_int, C.c_int, C.c_char_p, C.POINTER(_vp)])
_sig("vsr_comm_host", [_vp, C.c_int, C.c_int, C.POINTER(_HostExchange), _vp, C.POINTER(_vp)])
_sig("vsr_comm_destroy", [_vp])
_sig("vsr_comm_info", [_vp, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int)])
_sig("vsr_slab_plan", [_szp, _szp, C.c_int, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int)])
_sig("vsr_slab_tv_create", [_vp, _szp, _szp, _dp, _dp, C.POINTER(V._TvConfig), _pp, C.POINTER(_vp)])
_sig("vsr_slab_tv_iterate", [_vp, C.c_size_t])
_sig("vsr_slab_tv_x_d", [_vp, C.c_int, C.POINTER(_dp)])
_sig("vsr_slab_tv_finish", [_vp, _pp, C.POINTER(V._Report)])
_sig("vsr_slab_tv_destroy", [_vp])
_sig("vsr_slab_tikhonov_create", [_vp, _szp, _szp, _dp, C.c_double, _pp, C.POINTER(_vp)])
_sig("vsr_slab_tikhonov_solve", [_vp, _dp, _pp])
_sig("vsr_slab_tikhonov_solve_d", [_vp, _vp])
_sig("vsr_slab_tikhonov_check", [_vp])
_sig("vsr_slab_tikhonov_x_d", [_vp, C.c_int, C.POINTER(_dp)])
_sig("vsr_slab_tikhonov_destroy", [_vp])


# ---------------------------------------------------------------- slabs
def split_slabs(vol: np.ndarray, P: int) -> List[np.ndarray]:
    """(s, n, m) volume -> P contiguous (s, n/P, m) y-slabs."""
    s, n, m = vol.shape
    if n % P:
        raise V.ShapeError(f"slab: P={P} must divide axis 2 ({n})")
    k = n // P
    return [np.ascontiguousarray(vol[:, p * k:(p + 1) * k, :]) for p in range(P)]


def join_slabs(slabs: Sequence[np.ndarray]) -> np.ndarray:
    return np.ascontiguousarray(np.concatenate(list(slabs), axis=1))


def plane_owners(hr, rates, P: int) -> np.ndarray:
    """Owner rank of every half-spectrum plane f3 = 0..s/2 (vsr_slab_plan; host only)."""
    out = (C.c_int * (hr[2] // 2 + 1))()
    npl = C.c_int()
    V.check(_lib.vsr_slab_plan(V._dims_arr(hr), V._dims_arr(rates), int(P), 0, out, C.byref(npl)))
    return np.array(list(out), dtype=np.int64)


def _ptrs(arrays):
    return (_dp * len(arrays))(*[V._p(a) for a in arrays])


# ---------------------------------------------------------------- comms
class SlabComm:
    def __init__(self, handle, ctx, keep=None):
        self.handle = handle
        self.ctx = ctx
        self._keep = keep  # ctypes callbacks must outlive the comm
        n, r, loc = C.c_int(), C.c_int(), C.c_int()
        V.check(_lib.vsr_comm_info(handle, C.byref(n), C.byref(r), C.byref(loc)))
        self.world, self.rank, self.local = n.value, r.value, loc.value

    @property
    def local_ranks(self) -> List[int]:
        return list(range(self.world)) if self.rank < 0 else [self.rank]

    @classmethod
    def local(cls, P: int, ctx=None):
        ctx = ctx or V.default_context()
        h = _vp()
        V.check(_lib.vsr_comm_local(ctx.handle, int(P), C.byref(h)))
        return cls(h, ctx)

    @classmethod
    def nccl(cls, ctx=None, group=None):
        """torch.distributed must be initialised (any backend); one rank per process."""
        import torch.distributed as dist
        ctx = ctx or V.default_context()
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        uid = C.create_string_buffer(128)
        if rank == 0:
            V.check(_lib.vsr_nccl_unique_id(uid))
        obj = [bytes(uid.raw)]
        dist.broadcast_object_list(obj, src=0, group=group)
        h = _vp()
        V.check(_lib.vsr_comm_nccl(ctx.handle, world, rank, obj[0], C.byref(h)))
        return cls(h, ctx)

    @classmethod
    def host(cls, group=None, ctx=None):
        """Barriers and all-gathers through a torch.distributed group (host memory)."""
        import torch
        import torch.distributed as dist
        ctx = ctx or V.default_context()
        rank, world = dist.get_rank(group), dist.get_world_size(group)

        def barrier(_user):
            try:
                dist.barrier(group=group)
                return 0
            except Exception:
                return 1

        def all_gather(_user, send, recv, nbytes):
            try:
                src = torch.frombuffer(bytearray(C.string_at(send, nbytes)), dtype=torch.uint8)
                outs = [torch.empty(nbytes, dtype=torch.uint8) for _ in range(world)]
                dist.all_gather(outs, src, group=group)
                C.memmove(recv, torch.cat(outs).numpy().tobytes(), nbytes * world)
                return 0
            except Exception:
                return 1

        keep = (_BARRIER_FN(barrier), _GATHER_FN(all_gather))
        ops = _HostExchange(keep[0], keep[1])
        h = _vp()
        V.check(_lib.vsr_comm_host(ctx.handle, world, rank, C.byref(ops), None, C.byref(h)))
        return cls(h, ctx, keep=(keep, ops))

    def close(self):
        if getattr(self, "handle", None):
            _lib.vsr_comm_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ---------------------------------------------------------------- solvers
class SlabADMMTV:
    """admm_tv (solvers.cpp:321-411) on a slab communicator; stepwise."""

    def __init__(self, comm: SlabComm, y, psf, spec: V.DecimationSpec, cfg: V.TvAdmmConfig,
                 init_slabs: Optional[Sequence[np.ndarray]] = None):
        V.require_positive(cfg.lambda_, "lambda")
        V.require_positive(cfg.mu, "mu")
        if cfg.max_iters < 1:
            raise ValueError("admm_tv: max_iters must be >= 1")
        a, p = V._real(y), V._real(psf)
        V.require_same_dims(V.dims_of(a), spec.lr, "admm_tv")
        V.require_same_dims(V.dims_of(p), spec.hr, "admm_tv: psf")
        self.comm, self.spec, self.cfg = comm, spec, cfg
        m, n, s = spec.hr
        self.slab_shape = (s, n // comm.world, m)
        init = None
        if cfg.init == V.INIT_PROVIDED:
            if init_slabs is None or len(init_slabs) != comm.local:
                raise V.ShapeError("admm_tv: init volume: dims mismatch")
            self._init = [V._real(v) for v in init_slabs]
            for v in self._init:
                if v.shape != self.slab_shape:
                    raise V.ShapeError("admm_tv: init volume: dims mismatch")
            init = _ptrs(self._init)
        c = V._tv_cfg(cfg)
        h = _vp()
        V.check(_lib.vsr_slab_tv_create(comm.handle, V._dims_arr(spec.hr), V._dims_arr(spec.rates), V._p(a), V._p(p),
                                        C.byref(c), init, C.byref(h)))
        self.handle = h

    def iterate(self, k: int):
        V.check(_lib.vsr_slab_tv_iterate(self.handle, int(k)))

    def x_dev(self, local: int = 0) -> int:
        ptr = _dp()
        V.check(_lib.vsr_slab_tv_x_d(self.handle, int(local), C.byref(ptr)))
        return C.cast(ptr, C.c_void_p).value

    def finish(self):
        """-> (x slabs of the local ranks, SolveReport); collective."""
        xs = [np.empty(self.slab_shape) for _ in range(self.comm.local)]
        obj = np.zeros(max(self.cfg.max_iters, 1))
        res = np.zeros(max(self.cfg.max_iters, 1))
        rep = V._Report()
        rep.objective = V._p(obj)
        rep.primal_residual = V._p(res)
        V.check(_lib.vsr_slab_tv_finish(self.handle, _ptrs(xs), C.byref(rep)))
        it = int(rep.iterations)
        return xs, V.SolveReport(iterations=it, initial_objective=float(rep.initial_objective),
                                 objective=obj[:it].tolist(), primal_residual=res[:it].tolist(),
                                 seconds=float(rep.seconds))

    def close(self):
        if getattr(self, "handle", None):
            _lib.vsr_slab_tv_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def admm_tv(comm: SlabComm, y, psf, spec: V.DecimationSpec, cfg: V.TvAdmmConfig, init_slabs=None):
    """solvers.hpp:106-107 on slabs -> (x slabs, SolveReport)."""
    tv = SlabADMMTV(comm, y, psf, spec, cfg, init_slabs)
    try:
        tv.iterate(cfg.max_iters)
        return tv.finish()
    finally:
        tv.close()


class SlabTikhonov:
    """TikhonovOperator (solvers.cpp:36-67) on a slab communicator."""

    def __init__(self, comm: SlabComm, lam, spec: V.DecimationSpec, reg: float, xbar_slabs: Sequence[np.ndarray]):
        V.require_positive(reg, "lambda")
        L = V._cplx(lam)
        V.require_same_dims(V.dims_of(L), spec.hr, "TikhonovOperator")
        m, n, s = spec.hr
        self.slab_shape = (s, n // comm.world, m)
        if len(xbar_slabs) != comm.local:
            raise V.ShapeError("TikhonovOperator: xbar: one slab per local rank")
        xb = [V._real(v) for v in xbar_slabs]
        for v in xb:
            if v.shape != self.slab_shape:
                raise V.ShapeError("TikhonovOperator: xbar: dims mismatch")
        self.comm, self.spec = comm, spec
        h = _vp()
        V.check(_lib.vsr_slab_tikhonov_create(comm.handle, V._dims_arr(spec.hr), V._dims_arr(spec.rates),
                                              V._p(L.view(np.float64)), float(reg), _ptrs(xb), C.byref(h)))
        self.handle = h

    def solve(self, y) -> List[np.ndarray]:
        a = V._real(y)
        V.require_same_dims(V.dims_of(a), self.spec.lr, "TikhonovOperator::solve")
        xs = [np.empty(self.slab_shape) for _ in range(self.comm.local)]
        V.check(_lib.vsr_slab_tikhonov_solve(self.handle, V._p(a), _ptrs(xs)))
        return xs

    def solve_d(self, y_dev_ptr):
        V.check(_lib.vsr_slab_tikhonov_solve_d(self.handle, C.c_void_p(y_dev_ptr)))

    def check(self):
        V.check(_lib.vsr_slab_tikhonov_check(self.handle))

    def x_dev(self, local: int = 0) -> int:
        ptr = _dp()
        V.check(_lib.vsr_slab_tikhonov_x_d(self.handle, int(local), C.byref(ptr)))
        return C.cast(ptr, C.c_void_p).value

    def close(self):
        if getattr(self, "handle", None):
            _lib.vsr_slab_tikhonov_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
