"""Row-slab decomposition of ONE large image across ranks (the
C5 config: 8192^2, 20 D-Landweber iterations over 2/4/8 GPUs).

Rank p owns rows [p*R, (p+1)*R) of x, r, g, f (R = n/P >= q+1).  One
preconditioned iteration (solver.hpp:101-125) is

    A' r       halo exchange of q rows with the slab neighbours (NCCL
               send/recv; the first/last slab synthesise the global AR rows),
               then the FFT-correlation blur on the extended slab (dbx_slab_blur)
    T~ rows    local (dbx_slab_rows)
    -> cols    all-to-all transpose: rank p receives columns [p*C, (p+1)*C)
               of every slab (C = n/P) and holds them as rows
    T~ cols, x d^T, T cols   local on the transposed slab (d^T block built
               per rank by dbx_precond_block)
    -> rows    all-to-all back
    T rows + x_k = x_{k-1} + tau (.) with ||x||^2, ||x - f||^2 partials
    A x_k      halo exchange, blur, r = g - A x_k with ||r||^2
    norms      one all-reduce of three doubles; the bookkeeping (divergence
               guard, histories, strict-'<' best iterate, residual rule) is
               then identical on every rank.

Two drivers of the same decomposition:

* `SlabRun` (the product path): the whole loop in C++ behind the C-ABI
  (`dbx_slab_create` / `dbx_slab_run`): grouped ncclSend/ncclRecv halos and
  all-to-alls, the separable direct blur on halo-extended slabs, a device-side
  ncclAllReduce of the three norms and device bookkeeping — no host
  synchronisation inside the loop.  The NCCL communicator is built by the
  library (`NcclComm`: the unique id travels over torch.distributed once).
* `SlabLandweber`: the original Python orchestration of the C-ABI building
  blocks (kept as an independent second implementation of the exchange
  schedule; its exchange layer is what the gloo world-size-2 tests drive).

Every compute step is a CUDA kernel of the C-ABI; torch is used for device
buffers and torch.distributed for the exchanges only.  `LocalWorld` runs the
P ranks of the decomposition inside one process (single-GPU parity tests:
the exchanges become device copies); `DistWorld` is one rank per process
over NCCL (or gloo for the CPU tests of the exchange layer).
"""
from __future__ import annotations

import ctypes as C
import math
from typing import Dict, List, Optional

from . import SolverDivergence, _check, _ptr, lib

SLAB_STORE, SLAB_HADAMARD, SLAB_AXPY = 0, 1, 2
KIND_AR, KIND_ARINV = 3, 4
BC_AR = 3


def slab_rows_of(n: int, world: int, q: int) -> int:
    if n % world:
        raise ValueError("row slabs: image rows must divide evenly across ranks")
    rows = n // world
    if rows < q + 1:
        raise ValueError("row slabs: every slab needs at least q + 1 rows (the global AR extension is local)")
    return rows


class LocalWorld:
    """All P ranks of the decomposition in this process (exchanges = copies)."""

    def __init__(self, size: int):
        self.size = size
        self.ranks = list(range(size))

    def halo(self, firsts: Dict[int, "object"], lasts: Dict[int, "object"]):
        tops = {p: (lasts[p - 1].clone() if p > 0 else None) for p in self.ranks}
        bots = {p: (firsts[p + 1].clone() if p + 1 < self.size else None) for p in self.ranks}
        return tops, bots

    def alltoall(self, sends: Dict[int, "object"], recvs: Dict[int, "object"]):
        P = self.size
        for p in self.ranks:
            chunk = sends[p].numel() // P
            for s in self.ranks:
                recvs[s][p * chunk:(p + 1) * chunk].copy_(sends[p][s * chunk:(s + 1) * chunk])

    def allreduce(self, vals: Dict[int, List[float]]) -> List[float]:
        tot = [0.0] * len(next(iter(vals.values())))
        for p in self.ranks:  # fixed rank order
            tot = [a + b for a, b in zip(tot, vals[p])]
        return tot


class DistWorld:
    """One rank per process over torch.distributed (NCCL between GPUs)."""

    def __init__(self):
        import torch.distributed as dist
        self.dist = dist
        self.size = dist.get_world_size()
        self.rank = dist.get_rank()
        self.ranks = [self.rank]

    def halo(self, firsts, lasts):
        import torch
        dist, p, P = self.dist, self.rank, self.size
        first, last = firsts[p], lasts[p]
        top = torch.empty_like(last) if p > 0 else None
        bot = torch.empty_like(first) if p + 1 < P else None
        ops = []
        if p > 0:
            ops += [dist.P2POp(dist.isend, first, p - 1), dist.P2POp(dist.irecv, top, p - 1)]
        if p + 1 < P:
            ops += [dist.P2POp(dist.isend, last, p + 1), dist.P2POp(dist.irecv, bot, p + 1)]
        if ops:
            for w in dist.batch_isend_irecv(ops):
                w.wait()
        return {p: top}, {p: bot}

    def alltoall(self, sends, recvs):
        self.dist.all_to_all_single(recvs[self.rank], sends[self.rank])

    def allreduce(self, vals):
        import torch
        t = torch.tensor(vals[self.rank], dtype=torch.float64,
                         device="cuda" if torch.cuda.is_available() else "cpu")
        self.dist.all_reduce(t)
        return [float(v) for v in t.tolist()]


class _Slab:
    def __init__(self, p: int, P: int, n: int, rows: int, q: int, taps, alpha: float, device: int):
        import torch
        L = lib()
        self.p, self.rows, self.cb = p, rows, n // P
        self.dev = torch.device("cuda", device)
        h = C.c_void_p()
        _check(L.dbx_plan_create(rows, n, 1, _ptr(taps), q, q, BC_AR, device, C.byref(h)))
        self.plan = h
        _check(L.dbx_plan_set_conv(h, 2))  # FFT correlation (slab blur)
        z = lambda r, c: torch.zeros((r, c), dtype=torch.float64, device=self.dev)
        self.x, self.r, self.s, self.u, self.best = (z(rows, n) for _ in range(5))
        self.ext = z(rows + 2 * q, n)
        self.send = torch.zeros(rows * n, dtype=torch.float64, device=self.dev)
        self.recv = torch.zeros(rows * n, dtype=torch.float64, device=self.dev)
        self.tA, self.tB = z(self.cb, n), z(self.cb, n)
        self.dT = z(self.cb, n)  # d^T rows c in [p C, (p+1) C): d[:, c]
        # the zero fills above are queued on torch's stream; dbx_precond_block
        # writes dT on the plan's stream, so they must have landed first
        torch.cuda.current_stream(self.dev).synchronize()
        _check(L.dbx_precond_block(h, n, n, float(alpha), 0, n, p * self.cb, self.cb, 1, _ptr(self.dT)))

    def close(self):
        if self.plan:
            lib().dbx_plan_destroy(self.plan)
            self.plan = None


class SlabLandweber:
    """D-Landweber on one n x n image split into row slabs (see module doc)."""

    def __init__(self, world, n: int, taps, q: int, alpha: float, device: int = 0):
        self.world, self.n, self.q = world, n, q
        P = world.size
        # square image, equal row and column blocks: the transposed column
        # blocks have the slab's shape, so one plan serves both passes
        self.rows = slab_rows_of(n, P, q)
        if n % P:
            raise ValueError("row slabs: columns must divide evenly across ranks")
        self.slabs = {p: _Slab(p, P, n, self.rows, q, taps, alpha, device) for p in world.ranks}

    def close(self):
        for s in self.slabs.values():
            s.close()

    # ---- exchange helpers -------------------------------------------------
    # The C-ABI calls run on each plan's own stream and synchronise it before
    # returning; torch-side copies and NCCL transfers complete on torch's
    # current stream, so that stream is synchronised before a kernel of the
    # C-ABI reads what they produced (_fence).
    @staticmethod
    def _fence():
        import torch
        torch.cuda.current_stream().synchronize()

    def _extend(self, bufs: Dict[int, "object"]):
        q = self.q
        firsts = {p: bufs[p][:q].contiguous() for p in bufs}
        lasts = {p: bufs[p][-q:].contiguous() for p in bufs}
        tops, bots = self.world.halo(firsts, lasts)
        self._fence()
        L = lib()
        for p, s in self.slabs.items():
            _check(L.dbx_slab_extend(s.plan, _ptr(bufs[p]), _ptr(tops[p]), _ptr(bots[p]), _ptr(s.ext)))

    def _to_cols(self, src: Dict[int, "object"], dst_attr: str):
        """Row slabs -> transposed column blocks (rank p: columns of block p as rows)."""
        L, P = lib(), self.world.size
        for p, s in self.slabs.items():
            _check(L.dbx_slab_pack(s.plan, _ptr(src[p]), _ptr(s.send), P, 0))
        self.world.alltoall({p: s.send for p, s in self.slabs.items()}, {p: s.recv for p, s in self.slabs.items()})
        self._fence()
        for p, s in self.slabs.items():  # recv = (n x C) rows stacked by source rank -> (C x n)
            _check(L.dbx_transpose(s.plan, _ptr(s.recv), _ptr(getattr(s, dst_attr)), self.n, s.cb))

    def _to_rows(self, src_attr: str, dst: Dict[int, "object"]):
        L, P = lib(), self.world.size
        for p, s in self.slabs.items():
            _check(L.dbx_transpose(s.plan, _ptr(getattr(s, src_attr)), _ptr(s.send), s.cb, self.n))
        self.world.alltoall({p: s.send for p, s in self.slabs.items()}, {p: s.recv for p, s in self.slabs.items()})
        self._fence()
        for p, s in self.slabs.items():
            _check(L.dbx_slab_pack(s.plan, _ptr(dst[p]), _ptr(s.recv), P, 1))

    # ---- the loop ---------------------------------------------------------
    def run(self, g: Dict[int, "object"], f: Optional[Dict[int, "object"]], iters: int, tau: float = 1.0,
            resid_eps: Optional[float] = None, on_iterate=None):
        """g, f: this process's slabs (device tensors rows x n).  Returns the
        restored slabs (best-RRE iterate when f is given, solver.hpp:127-131)
        and the global histories (identical on every rank)."""
        import torch
        L = lib()
        S = self.slabs
        gn2 = self.world.allreduce({p: [float(torch.sum(g[p] * g[p]))] for p in S})[0]
        fn2 = self.world.allreduce({p: [float(torch.sum(f[p] * f[p]))] for p in S})[0] if f else 0.0
        gnorm, fnorm = math.sqrt(gn2), math.sqrt(fn2)
        if f and not fnorm > 0.0:
            raise ValueError("rre: zero true image")  # image.hpp:89
        for p, s in S.items():
            s.x.zero_()
            s.r.copy_(g[p])
        self._fence()
        rre, res = [], []
        best_rre, best_iter, done = math.inf, 0, 0
        for k in range(1, iters + 1):
            # A' r, then T~ along the rows
            self._extend({p: s.r for p, s in S.items()})
            for s in S.values():
                _check(L.dbx_slab_blur(s.plan, _ptr(s.ext), _ptr(s.s), 1, None, None))
                _check(L.dbx_slab_rows(s.plan, KIND_ARINV, _ptr(s.s), _ptr(s.u), SLAB_STORE, None, None, 0.0, None))
            # column half of D on the transposed blocks: T~, x d^T, T
            self._to_cols({p: s.u for p, s in S.items()}, "tA")
            for s in S.values():
                _check(L.dbx_slab_rows(s.plan, KIND_ARINV, _ptr(s.tA), _ptr(s.tB), SLAB_HADAMARD, _ptr(s.dT), None,
                                       0.0, None))
                _check(L.dbx_slab_rows(s.plan, KIND_AR, _ptr(s.tB), _ptr(s.tA), SLAB_STORE, None, None, 0.0, None))
            self._to_rows("tA", {p: s.s for p, s in S.items()})
            # T along the rows + x update (+ norms)
            part = {}
            for p, s in S.items():
                nrm = (C.c_double * 2)()
                _check(L.dbx_slab_rows(s.plan, KIND_AR, _ptr(s.s), _ptr(s.u), SLAB_AXPY, _ptr(s.x),
                                       _ptr(f[p]) if f else None, float(tau), nrm))
                s.x, s.u = s.u, s.x  # x_k now in s.x
                part[p] = [nrm[0], nrm[1]]
            # r = g - A x_k
            self._extend({p: s.x for p, s in S.items()})
            for p, s in S.items():
                rr = C.c_double()
                _check(L.dbx_slab_blur(s.plan, _ptr(s.ext), _ptr(s.r), 0, _ptr(g[p]), C.byref(rr)))
                part[p].append(rr.value)
            xx, xf, rr = self.world.allreduce(part)
            # bookkeeping (solver.hpp:107-124)
            if gnorm > 0.0 and math.sqrt(xx) > 1e8 * gnorm:
                raise SolverDivergence(f"landweber diverged at iteration {k}")
            res.append(math.sqrt(rr))
            if f:
                e = math.sqrt(xf) / fnorm
                rre.append(e)
                if e < best_rre:
                    best_rre, best_iter = e, k
                    for s in S.values():
                        s.best.copy_(s.x)
                    self._fence()
            done = k
            if on_iterate is not None:  # tests: every iterate x_k, this process's slabs
                on_iterate(k, {p: s.x for p, s in S.items()})
            if resid_eps is not None and gnorm > 0.0 and math.sqrt(rr) / gnorm < resid_eps:
                break
        restored = {p: (s.best if (f and best_iter > 0) else s.x).clone() for p, s in S.items()}
        self._fence()
        return {"restored": restored, "iterations_executed": done, "best_iteration": best_iter,
                "rre_history": rre, "residual_history": res}


class NcclComm:
    """An NCCL communicator owned by libdbx (ncclCommInitRank); the unique id
    is broadcast from rank 0 over the default torch.distributed group."""

    def __init__(self, device: int):
        import torch
        import torch.distributed as dist
        L = lib()
        self.rank, self.size = dist.get_rank(), dist.get_world_size()
        buf = (C.c_ubyte * 128)()
        if self.rank == 0:
            _check(L.dbx_comm_unique_id(buf))
        t = torch.tensor(list(bytes(buf)), dtype=torch.uint8,
                         device="cuda" if dist.get_backend() == "nccl" else "cpu")
        dist.broadcast(t, 0)
        raw = (C.c_ubyte * 128)(*t.cpu().tolist())
        h = C.c_void_p()
        _check(L.dbx_comm_init(self.size, raw, self.rank, device, C.byref(h)))
        self.handle = h

    def close(self):
        if self.handle:
            lib().dbx_comm_destroy(self.handle)
            self.handle = None


class SlabRun:
    """D-Landweber on an n x n image in `parts` row slabs, driven in C++.

    rank = -1: this process holds all slabs (in-process ranks: exchanges are
    device copies); else it holds slab `rank` and `comm` (NcclComm) carries
    the exchanges (required for parts > 1)."""

    def __init__(self, n: int, parts: int, taps, q: int, alpha: float, rank: int = -1, comm=None,
                 device: int = 0):
        L = lib()
        h = C.c_void_p()
        _check(L.dbx_slab_create(n, parts, rank, _ptr(taps), q, q, float(alpha),
                                 comm.handle if comm is not None else None, device, C.byref(h)))
        self.handle, self.n, self.parts, self.rank = h, n, parts, rank
        rows, loc, sep = C.c_int(), C.c_int(), C.c_int()
        _check(L.dbx_slab_info(h, C.byref(rows), C.byref(loc), C.byref(sep), None))
        self.rows, self.local_slabs, self.separable = rows.value, loc.value, bool(sep.value)

    def stream(self):
        return lib().dbx_slab_stream(self.handle)

    def launch_count(self) -> int:
        n = C.c_int64()
        _check(lib().dbx_slab_info(self.handle, None, None, None, C.byref(n)))
        return n.value

    def run(self, g, f=None, iters: int = 20, tau: float = 1.0, resid_eps: Optional[float] = None, out=None,
            keep_iterates: bool = False):
        """g, f, out: device tensors of the rows held here (local_slabs * rows x n).
        Returns (restored, history dict); keep_iterates adds "iterates" (a
        device tensor iters x rows x n of every x_k, for the parity tests)."""
        import numpy as np
        import torch
        out = torch.empty_like(g) if out is None else out
        keep = None
        if keep_iterates:
            keep = torch.empty((iters,) + tuple(g.shape), dtype=g.dtype, device=g.device)
            _check(lib().dbx_slab_set_iterates(self.handle, _ptr(keep), iters))
        rre, res = np.zeros(iters), np.zeros(iters)
        best, done = C.c_int(), C.c_int()
        stop = 2 if resid_eps is not None else (1 if f is not None else 0)
        try:
            _check(lib().dbx_slab_run(self.handle, _ptr(g), _ptr(f) if f is not None else None, float(tau), iters,
                                      stop, float(resid_eps or 0.0), _ptr(out), _ptr(rre), _ptr(res), C.byref(best),
                                      C.byref(done)))
        finally:
            if keep is not None:
                _check(lib().dbx_slab_set_iterates(self.handle, None, 0))
        k = done.value
        return out, {"iterates": keep, "iterations_executed": k, "best_iteration": best.value,
                     "rre_history": list(rre[:k]) if f is not None else [], "residual_history": list(res[:k])}

    def close(self):
        if self.handle:
            lib().dbx_slab_destroy(self.handle)
            self.handle = None
