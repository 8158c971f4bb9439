"""z-slab domain decomposition (include/wbfbt.h "z-slab"): plumbing only.

`SlabContext` is a `Context` created by `wb_slab_create`: rank r of R owns the r-th of R cubes
of N^3 elements stacked along z, and the same calls (`set_viscosity`, `apply_A`, `apply_B`,
`apply_BT`, `apply_K`, `poisson_pcg`, `apply_wbfbt`, `hotpath`) compute the GLOBAL operators on
the rank's local vectors.  All arithmetic (the cube kernels, the plane sums, the masks, the PCG
scalars) runs in libwbfbt.so; this module only moves the bytes the library asks it to move:

* `DistComm`   -- torch.distributed: NCCL send/recv + all_reduce on the context's stream (one
                  process per GPU), or gloo with host staging (CPU tests, and two processes
                  sharing one GPU in the GPU test);
* `ThreadComm` -- R slab contexts in ONE process on one GPU, each driven by its own host thread
                  (tests on the 1-GPU box: the host threads meet at barriers; no kernel ever
                  waits for another).
"""
from __future__ import annotations

import ctypes as C
import threading

from . import _abi
from ._abi import Context, WBError

_EXCH = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int64)
_ALLR = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int, C.c_int, C.c_int)
_dp = C.c_void_p


class _CommStruct(C.Structure):  # wb_slab_comm
    _fields_ = [("user", C.c_void_p), ("exchange", _EXCH), ("allreduce", _ALLR), ("send_lo", _dp),
                ("recv_lo", _dp), ("send_hi", _dp), ("recv_hi", _dp), ("cap", C.c_int64), ("scal", _dp)]


class SlabComm:
    """Owns the exchange buffers of one rank; subclasses move them."""

    def __init__(self, rank: int, nranks: int, cap: int, device):
        import torch
        self.rank, self.nranks, self.cap, self.device = rank, nranks, int(cap), device
        z = lambda n: torch.zeros(n, dtype=torch.float64, device=device)  # noqa: E731
        self.send_lo, self.recv_lo, self.send_hi, self.recv_hi = z(cap), z(cap), z(cap), z(cap)
        self.scal = z(8)
        self.n_exchange = self.n_allreduce = 0
        self.error = None

    @property
    def has_lo(self):
        return self.rank > 0

    @property
    def has_hi(self):
        return self.rank < self.nranks - 1

    def exchange(self, n: int):  # pragma: no cover - interface
        raise NotImplementedError

    def allreduce(self, offset: int, n: int, op: int):  # pragma: no cover - interface
        raise NotImplementedError

    # ctypes callbacks (kept alive by self)
    def _struct(self) -> _CommStruct:
        def ex(_user, n):
            try:
                self.n_exchange += 1
                self.exchange(int(n))
                return 0
            except BaseException as e:  # never unwind through C
                self.error = e
                return 1

        def ar(_user, offset, n, op):
            try:
                self.n_allreduce += 1
                self.allreduce(int(offset), int(n), int(op))
                return 0
            except BaseException as e:
                self.error = e
                return 1

        self._cb = (_EXCH(ex), _ALLR(ar))
        return _CommStruct(None, self._cb[0], self._cb[1], self.send_lo.data_ptr(), self.recv_lo.data_ptr(),
                           self.send_hi.data_ptr(), self.recv_hi.data_ptr(), self.cap, self.scal.data_ptr())


class DistComm(SlabComm):
    """torch.distributed neighbours rank-1 / rank+1 of `group` (default: the world).

    NCCL: the transfers are enqueued on torch's current stream, which is the stream the
    context was created on.  gloo: buffers on a GPU are staged through the host after a
    stream synchronise (the transfer is complete on return).
    """

    def __init__(self, cap: int, device, group=None):
        import torch.distributed as dist
        self.dist, self.group = dist, group
        super().__init__(dist.get_rank(group), dist.get_world_size(group), cap, device)
        self.staged = dist.get_backend(group) != "nccl" and str(device).startswith("cuda")

    def _peer(self, r):
        return r if self.group is None else self.dist.get_global_rank(self.group, r)

    def exchange(self, n: int):
        import torch
        dist = self.dist
        if self.staged:
            torch.cuda.current_stream().synchronize()
            sl, sh = self.send_lo[:n].cpu(), self.send_hi[:n].cpu()
            rl, rh = torch.empty_like(sl), torch.empty_like(sh)
        else:
            sl, sh, rl, rh = self.send_lo[:n], self.send_hi[:n], self.recv_lo[:n], self.recv_hi[:n]
        ops = []
        if self.has_lo:
            ops += [dist.P2POp(dist.isend, sl, self._peer(self.rank - 1), self.group),
                    dist.P2POp(dist.irecv, rl, self._peer(self.rank - 1), self.group)]
        if self.has_hi:
            ops += [dist.P2POp(dist.isend, sh, self._peer(self.rank + 1), self.group),
                    dist.P2POp(dist.irecv, rh, self._peer(self.rank + 1), self.group)]
        if ops:
            for w in dist.batch_isend_irecv(ops):
                w.wait()  # NCCL: orders the current stream after the transfer; gloo: completes it
        if self.staged:
            if self.has_lo:
                self.recv_lo[:n].copy_(rl)
            if self.has_hi:
                self.recv_hi[:n].copy_(rh)
            torch.cuda.current_stream().synchronize()

    def allreduce(self, offset: int, n: int, op: int):
        import torch
        dist = self.dist
        rop = dist.ReduceOp.MAX if op == 1 else dist.ReduceOp.SUM
        v = self.scal[offset:offset + n]
        if self.staged:
            torch.cuda.current_stream().synchronize()
            h = v.cpu()
            dist.all_reduce(h, op=rop, group=self.group)
            v.copy_(h)
            torch.cuda.current_stream().synchronize()
        else:
            dist.all_reduce(v, op=rop, group=self.group)


class ThreadComm(SlabComm):
    """R ranks as R host threads of one process (see the module docstring).  Build them with
    `ThreadComm.group(R, cap, device)`; every collective call must be made by all R threads."""

    def __init__(self, rank, nranks, cap, device, shared):
        super().__init__(rank, nranks, cap, device)
        self.sh = shared
        shared["comms"][rank] = self

    @classmethod
    def group(cls, nranks: int, cap: int, device):
        shared = {"comms": [None] * nranks, "barrier": threading.Barrier(nranks)}
        return [cls(r, nranks, cap, device, shared) for r in range(nranks)]

    def _sync(self):
        import torch
        torch.cuda.synchronize(self.device)

    def exchange(self, n: int):
        comms, bar = self.sh["comms"], self.sh["barrier"]
        self._sync()
        bar.wait()
        if self.has_lo:
            self.recv_lo[:n].copy_(comms[self.rank - 1].send_hi[:n])
        if self.has_hi:
            self.recv_hi[:n].copy_(comms[self.rank + 1].send_lo[:n])
        self._sync()
        bar.wait()

    def allreduce(self, offset: int, n: int, op: int):
        import torch
        comms, bar = self.sh["comms"], self.sh["barrier"]
        self._sync()
        bar.wait()
        parts = torch.stack([c.scal[offset:offset + n] for c in comms])  # rank order on every rank
        red = parts.max(dim=0).values if op == 1 else _ordered_sum(parts)
        self._sync()
        bar.wait()
        self.scal[offset:offset + n].copy_(red)
        self._sync()


def _ordered_sum(parts):
    acc = parts[0].clone()
    for i in range(1, parts.shape[0]):
        acc += parts[i]
    return acc


class SlabContext(Context):
    """Rank `comm.rank` of `comm.nranks` z-stacked cubes (wb_slab_create + wb_slab_set_comm)."""

    def __init__(self, N: int, k: int, comm: SlabComm, flags: int = 0, stream=None):
        import torch
        self._L = _abi.lib()
        if stream is None:
            stream = torch.cuda.current_stream().cuda_stream
        if comm.cap < 3 * (k * N + 1) ** 2:
            raise ValueError("communicator buffers too small: cap >= 3 (kN+1)^2")
        h = C.c_void_p()
        st = self._L.wb_slab_create(C.byref(h), int(N), int(k), int(comm.rank), int(comm.nranks), int(flags),
                                    C.c_void_p(int(stream)))
        if st != 0:
            raise WBError(st, f"wb_slab_create(N={N}, k={k}, rank={comm.rank}/{comm.nranks}) failed")
        self._h = h
        self.N, self.k, self.flags, self.comm = N, k, flags, comm
        self.rank, self.nranks = comm.rank, comm.nranks
        v = [C.c_int64() for _ in range(5)]
        self._check(self._L.wb_sizes(h, *[C.byref(x) for x in v]))
        self.n_el, self.n_nodes, self.n_v, self.n_p, self.n_q = (int(x.value) for x in v)
        self._cs = comm._struct()
        self._check(self._L.wb_slab_set_comm(h, C.byref(self._cs)))

    def _check(self, st: int):
        if st != 0 and getattr(self, "comm", None) is not None and self.comm.error is not None:
            e, self.comm.error = self.comm.error, None
            raise WBError(st, f"communicator callback raised: {e!r}") from e
        super()._check(st)

    @staticmethod
    def plane_cap(N: int, k: int) -> int:
        return 3 * (k * N + 1) ** 2
