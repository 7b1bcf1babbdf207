"""Multi-GPU layer: outer-point sharding + all-gather of the inner field state.

One process per GPU (torch.distributed, backend "nccl"; "gloo" on CPU for
the host-logic tests).  Each rank owns a contiguous, cell-aligned block of
quadrature points (`synthetic.shard_bounds`): it samples / receives the
fields of its own points, packs them into inner records on its device
(`lb_pack_records_dev`), and one all-gather per operator evaluation
replicates the packed records of every point to every rank -- the paper's
per-point field state (w f, w grad f) plus coordinates, 10 doubles per point
at S = 2, 5.2 MB at N = 2^16.  Then, either
 * symmetric path (outer set == inner set, the default here): every rank
   Morton-orders all records identically and evaluates its share of the
   unordered tile pairs (each pair once, feeding both points): whole row
   groups of the fixed 8-group split (`lb_sym_groups`), one sum per group and
   point.  One all-gather replicates the group sums (2.6 MB per group at
   N = 2^16), and each rank adds, for its own points only, all eight in group
   order and applies the coupling -- so K and D are bitwise the same for any
   GPU count <= 8 (the reference promises bitwise invariance to `workers`,
   kernel.py:508-511).  In peer-memory mode the owner reads the peers' group
   sums directly over NVLink instead of the all-gather; or
 * general path: each rank sweeps its own outer points against all inner
   points (`lb_sweep_dev`); no collective follows.  Because the inner
   chunking depends only on the global inner count, every rank's K/D rows
   are bitwise identical to the single-GPU result.

The reference has no distributed code; the paper ran
redundant MPI replicas.  This layer is the B200 design
from BASELINE.json's north_star.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Callable

import numpy as np

from . import _lib
from .kernel import coupling
from .synthetic import shard_bounds

__all__ = ["ShardPlan", "ShardedSweep", "SYM_GROUPS", "sym_rank_groups"]

SYM_GROUPS = 8  # kSymGroups of landau_sym.cuh (lb_sym_groups)


def sym_rank_groups(rank: int, world: int):
    """Row groups [g0, g1) of `rank` among `world` (lb_sym_groups)."""
    return SYM_GROUPS * rank // world, SYM_GROUPS * (rank + 1) // world


@dataclass(frozen=True)
class ShardPlan:
    """Contiguous cell-aligned partition of n points over `world` ranks."""

    n: int
    world: int
    align: int = 9

    def bounds(self, rank: int):
        return shard_bounds(self.n, self.world, rank, self.align)

    @property
    def counts(self):
        return [hi - lo for lo, hi in (self.bounds(r) for r in range(self.world))]

    @property
    def max_count(self) -> int:
        return max(self.counts) if self.world else 0

    @property
    def even(self) -> bool:
        return len(set(self.counts)) == 1


def _device_index(device) -> int:
    """CUDA ordinal of a torch device; torch.device("cuda") means the current
    device (under torchrun: the rank's own GPU), not GPU 0."""
    import torch

    if device.index is not None:
        return int(device.index)
    return int(torch.cuda.current_device()) if torch.cuda.is_available() else 0


def _dist():
    import torch.distributed as dist

    return dist


class ShardedSweep:
    """Per-rank driver of one distributed D/K evaluation.

    Parameters
    ----------
    n, S : global inner point count and species count
    params : object with nu_hat / mass_ratio_o (CollisionParams-like)
    eps_d : exclusion radius
    device : torch device of this rank ("cuda:k", or "cpu" with injected
             pack/sweep functions for the CPU tests)
    align : shard alignment in points (9 = whole Q2 cells; 1 for point clouds)
    pack_fn, sweep_fn : injectable for CPU testing; default to the CUDA
             library (lb_pack_records_dev / lb_sweep_dev on torch tensors)
    p2p : symmetric path only -- replace the all-gather of the group sums
             by one kernel that reads every rank's group sums for this
             rank's own points through CUDA IPC peer mappings (NVLink),
             ordered by stream-level barriers
    sym_fns : injectable (prepare(rec), partial(tot), combine(groups, q0, q1,
             K, D)) for CPU testing of the symmetric host logic; `groups` is
             the list of the eight group-sum arrays in group order
    """

    def __init__(self, n: int, S: int, params, eps_d: float, device, align: int = 9,
                 group=None, pack_fn: Callable | None = None,
                 sweep_fn: Callable | None = None, symmetric: bool | None = None,
                 sym_fns: tuple | None = None, p2p: bool = False):
        import torch

        dist = _dist()
        self.group = group
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.n, self.S = int(n), int(S)
        self.plan = ShardPlan(self.n, self.world, align)
        self.lo, self.hi = self.plan.bounds(self.rank)
        self.device = torch.device(device)
        self.eps_d = float(eps_d)
        self.coK, self.coD = coupling(params)
        if pack_fn is None or sweep_fn is None:
            lib = _lib.load()
            self._lib = lib
            # a context of its own: its stream-ordered scratch (sorted records,
            # partial sums) is used on torch's stream, so it must not be shared
            # with the host entry points' cached context and its stream
            self._ctx = _lib.Context(_device_index(self.device))
            p = _lib.dptr
            self.RS = lib.lb_record_stride(self.S, p(self.coK), p(self.coD))
            self.nacc = lib.lb_accumulator_sets(self.S, p(self.coK), p(self.coD))
            if self.RS < 0:
                _lib.check(1)
        else:
            base = ((4 + 3 * self.S) + 1) & ~1  # rec_stride() of landau_common.cuh
            self.RS = base + (2 if (base // 2) % 2 == 0 else 0)
            self.nacc = self.S
        self._pack = pack_fn or self._pack_cuda
        self._sweep = sweep_fn or self._sweep_cuda
        # symmetric all-points path (each unordered pair once, tile pairs split
        # over ranks, one all-reduce of the 5S partial sums per point)
        if sym_fns is not None:
            self._sym_prepare, self._sym_partial, self._sym_combine = sym_fns
            sym_ok = True
        else:
            self._sym_prepare, self._sym_partial = self._sym_prepare_cuda, self._sym_partial_cuda
            self._sym_combine = self._sym_combine_cuda
            sym_ok = (pack_fn is None and sweep_fn is None and self.n >= 128 and bool(
                self._lib.lb_sym_supported(self.S, _lib.dptr(self.coK), _lib.dptr(self.coD))))
        self.symmetric = sym_ok if symmetric is None else (bool(symmetric) and sym_ok)
        self.p2p = bool(p2p) and self.symmetric and sym_fns is None
        self._p2p_pending = False
        self._opened = []
        self._ipc_ptr = None
        if self.symmetric:
            # group sums: 5 per accumulator set (1 set when collapsed) and point,
            # one slot per row group this rank owns (lb_sym_groups)
            self.npad = -(-self.n // 128) * 128
            self.g0, self.g1 = sym_rank_groups(self.rank, self.world)
            self.ngmax = max(b - a for a, b in (sym_rank_groups(r, self.world)
                                                 for r in range(self.world)))
            shape = (max(self.ngmax, 1), 5 * max(self.nacc, 1), self.npad)
            if self.p2p:
                self.tot = self._init_p2p(shape)
            else:
                self.tot = torch.zeros(shape, dtype=torch.float64, device=self.device)
            self.gathered = (self.tot if self.world == 1 or self.p2p else torch.zeros(
                (self.world * shape[0],) + shape[1:], dtype=torch.float64, device=self.device))
        mc = self.plan.max_count
        f64 = torch.float64
        self.send = torch.zeros((mc, self.RS), dtype=f64, device=self.device)
        self.recv = (self.send if self.world == 1 else
                     torch.zeros((self.world * mc, self.RS), dtype=f64, device=self.device))
        self.rec = (self.recv if self.plan.even else
                    torch.zeros((self.n, self.RS), dtype=f64, device=self.device))
        nl = self.hi - self.lo
        self.K = torch.empty((nl, self.S, 2), dtype=f64, device=self.device)
        self.D = torch.empty((nl, self.S, 2, 2), dtype=f64, device=self.device)
        self.launches = 0

    # ---------------------------------------------------------------- peer memory
    def _init_p2p(self, shape):
        """Partial-sum buffer in CUDA IPC memory; map every peer's buffer."""
        import ctypes as C

        import torch

        lib, ctx = self._lib, self._ctx.handle
        nbytes = 8 * shape[0] * shape[1]
        ptr = C.c_void_p()
        handle = C.create_string_buffer(64)
        _lib.check(lib.lb_ipc_alloc(ctx, nbytes, C.byref(ptr), handle))
        self._ipc_ptr = ptr.value
        handles = [bytes(handle.raw)]
        if self.world > 1:
            handles = [None] * self.world
            _dist().all_gather_object(handles, bytes(handle.raw), group=self.group)
        peers = []
        for g, h in enumerate(handles):
            if g == self.rank:
                peers.append(ptr.value)
                continue
            q = C.c_void_p()
            _lib.check(lib.lb_ipc_open(ctx, h, C.byref(q)))
            self._opened.append(q.value)
            peers.append(q.value)
        self._peers = peers
        self._flag = torch.zeros(1, dtype=torch.float64, device=self.device)

        class _View:  # torch view of the IPC allocation (__cuda_array_interface__)
            __cuda_array_interface__ = {"shape": tuple(shape), "typestr": "<f8",
                                        "data": (ptr.value, False), "version": 3,
                                        "strides": None}

        tot = torch.as_tensor(_View(), device=self.device)
        tot.zero_()
        return tot

    def _barrier(self):
        """Every rank's prior work on its stream is done before any rank's
        later work: a stream-ordered one-element NCCL all-reduce (no host
        sync), or host synchronisation + barrier on gloo."""
        if self.world == 1:
            return
        dist = _dist()
        if dist.get_backend(self.group) == "nccl":
            dist.all_reduce(self._flag, group=self.group)
        else:
            import torch

            torch.cuda.synchronize(self.device)
            dist.barrier(group=self.group)

    def close(self):
        if getattr(self, "_ipc_ptr", None) is None:
            return
        import torch

        torch.cuda.synchronize(self.device)
        self._barrier()  # no peer still reads our buffer
        for q in self._opened:
            self._lib.lb_ipc_close(self._ctx.handle, q)
        self._opened = []
        self.tot = None
        self._lib.lb_ipc_free(self._ctx.handle, self._ipc_ptr)
        self._ipc_ptr = None

    # ---------------------------------------------------------------- CUDA
    def _stream(self):
        import torch

        return torch.cuda.current_stream(self.device).cuda_stream

    def _pack_cuda(self, r, z, w, f, dfr, dfz, out):
        n = r.shape[0]
        p = _lib.dptr
        _lib.check(self._lib.lb_pack_records_dev(
            self._ctx.handle, n, self.S, r.data_ptr(), z.data_ptr(), w.data_ptr(), f.data_ptr(),
            dfr.data_ptr(), dfz.data_ptr(), p(self.coK), p(self.coD), out.data_ptr(),
            self._stream()))
        self.launches += self._lib.lb_last_launch_count(self._ctx.handle)

    def _sweep_cuda(self, ro, zo, rec, K, D):
        p = _lib.dptr
        _lib.check(self._lib.lb_sweep_dev(
            self._ctx.handle, ro.shape[0], ro.data_ptr(), zo.data_ptr(), self.n, self.S,
            rec.data_ptr(), p(self.coK), p(self.coD), self.eps_d, K.data_ptr(), D.data_ptr(),
            self._stream()))
        self.launches += self._lib.lb_last_launch_count(self._ctx.handle)

    def _sym_prepare_cuda(self, rec):
        p = _lib.dptr
        _lib.check(self._lib.lb_sym_prepare_dev(self._ctx.handle, self.n, self.S, p(self.coK),
                                                p(self.coD), rec.data_ptr(), self._stream()))
        self.launches += self._lib.lb_last_launch_count(self._ctx.handle)

    def _sym_partial_cuda(self, tot):
        _lib.check(self._lib.lb_sym_partial_dev(self._ctx.handle, self.S, self.eps_d, self.rank,
                                                self.world, tot.data_ptr(), self._stream()))
        self.launches += self._lib.lb_last_launch_count(self._ctx.handle)

    def _group_owner(self, g: int):
        """(rank, slot) holding row group g's sums."""
        for r in range(self.world):
            a, b = sym_rank_groups(r, self.world)
            if a <= g < b:
                return r, g - a
        raise AssertionError(g)

    def _group_ptrs(self):
        """Device pointers of the eight group sums in group order: the local
        buffer (one rank), the all-gathered copy, or the peers' buffers."""
        slot = 8 * 5 * max(self.nacc, 1) * self.npad
        out = []
        for g in range(SYM_GROUPS):
            r, k = self._group_owner(g)
            if self.p2p:
                base = self._peers[r]
            else:
                base = self.gathered.data_ptr() + r * self.tot.shape[0] * slot
            out.append(base + k * slot)
        return out

    def _group_views(self):
        """The eight group-sum arrays in group order (non-peer modes)."""
        views = []
        for g in range(SYM_GROUPS):
            r, k = self._group_owner(g)
            views.append(self.gathered[r * self.tot.shape[0] + k])
        return views

    def _sym_combine_cuda(self, groups, q0, q1, K, D):
        import ctypes as C

        p = _lib.dptr
        arr = (C.c_void_p * SYM_GROUPS)(*self._group_ptrs())
        _lib.check(self._lib.lb_sym_combine_groups_dev(
            self._ctx.handle, self.S, arr, p(self.coK), p(self.coD), q0, q1, K.data_ptr(),
            D.data_ptr(), self._stream()))
        self.launches += self._lib.lb_last_launch_count(self._ctx.handle)

    # ---------------------------------------------------------------- steps
    def pack_local(self, r, z, w, f, dfr, dfz):
        """Pack this rank's points (device tensors: r,z,w (nl,), f.. (S,nl))."""
        nl = self.hi - self.lo
        if r.shape[0] != nl:
            raise ValueError(f"rank {self.rank} owns {nl} points, got {r.shape[0]}")
        self._pack(r, z, w, f, dfr, dfz, self.send[:nl])

    def all_gather(self):
        """Replicate every rank's packed records (one collective)."""
        if self.world > 1:
            _dist().all_gather_into_tensor(self.recv, self.send, group=self.group)
        if not self.plan.even:  # compact the padded slots into global order
            mc = self.plan.max_count
            for k in range(self.world):
                lo, hi = self.plan.bounds(k)
                self.rec[lo:hi].copy_(self.recv[k * mc:k * mc + (hi - lo)])

    def sweep_local(self, ro, zo):
        """K, D for this rank's outer points (device tensors ro, zo)."""
        self._sweep(ro, zo, self.rec, self.K, self.D)
        return self.K, self.D

    def sym_prepare(self):
        """Symmetric path, step 1: order all n gathered records (same on
        every rank)."""
        self._sym_prepare(self.rec[:self.n])

    def sym_partial(self):
        """Step 2: this rank's row groups of the unordered tile pairs -> its
        group sums (tot)."""
        if self.p2p and self._p2p_pending:  # peers may still read our last sums
            self._barrier()
            self._p2p_pending = False
        self._sym_partial(self.tot)

    def sym_reduce(self):
        """Step 3: replicate every rank's group sums (one all-gather, 2.6 MB
        per group at N = 2^16, S = 2); peer-memory mode: only order every
        rank's group sums before the fused combine."""
        if self.p2p:
            self._barrier()
        elif self.world > 1:
            _dist().all_gather_into_tensor(self.gathered, self.tot, group=self.group)

    def sym_finish(self):
        """Step 4: the eight group sums of this rank's own points, added in
        group order, and the coupling -> K, D (peer-memory mode: read from
        the peers' buffers)."""
        if self.p2p:
            self._sym_combine(None, self.lo, self.hi, self.K, self.D)
            self._p2p_pending = True
            return self.K, self.D
        self._sym_combine(self._group_views(), self.lo, self.hi, self.K, self.D)
        return self.K, self.D

    def step(self, r, z, w, f, dfr, dfz):
        """One distributed evaluation from this rank's local fields; the local
        points are also the outer points (assemble_collision's all-points
        sweep, assembly.py:148)."""
        self.pack_local(r, z, w, f, dfr, dfz)
        self.all_gather()
        if self.symmetric:
            self.sym_prepare()
            self.sym_partial()
            self.sym_reduce()
            return self.sym_finish()
        return self.sweep_local(r, z)


def local_fields(wl, lo: int, hi: int):
    """Slice a host workload (QuadPointData-like) to points [lo, hi)."""
    sl = slice(lo, hi)
    return (np.ascontiguousarray(wl.r[sl]), np.ascontiguousarray(wl.z[sl]),
            np.ascontiguousarray(wl.w[sl]), np.ascontiguousarray(wl.f[:, sl]),
            np.ascontiguousarray(wl.df_r[:, sl]), np.ascontiguousarray(wl.df_z[:, sl]))


class ShardedOperator:
    """Multi-GPU state-level operator: `solver._assemble_at` (solver.py:81-84)
    with cells sharded over ranks, the paper's data flow (BASELINE north_star):

      1. every rank holds the state coefficients (S, n_free) -- the solver's
         small replicated vector -- and samples ITS cells on the device
         (`lb_sample_state_dev`, K4);
      2. packs its points and all-gathers the packed field state (NCCL);
      3. evaluates its row groups of the unordered tile pairs (symmetric
         sweep), one all-gather of the per-group sums, the group-ordered sum
         and the coupling for its own points (K, D of its cells);
      4. one all-gather of every point's (w, K, D) -- 1 + 6S doubles per
         point, 14.7 MB at config 4 -- and every rank contracts all cells'
         element matrices and gathers them into the CSR values
         (`lb_operator_partial_dev` over all cells, K2 + K3: ~0.3 ms at config
         4).  Every rank thus holds C, bitwise the single-GPU operator for
         any GPU count (an all-reduce of per-rank partial CSR values would
         re-associate the sums with G).
    """

    def __init__(self, mesh, ref, params, device, eps_d: float | None = None, group=None):
        import torch

        from .assembly import default_eps_d, device_mesh

        self.device = torch.device(device)
        self.group = group
        self.S = int(np.asarray(params.mass_ratio_o).shape[0])
        self.dm = device_mesh(mesh, ref, _device_index(self.device))
        if not self.dm.has_geometry:
            raise ValueError("mesh/ref lack origins/qpts/qwts needed for device sampling")
        self.ncell = self.dm.ncell
        n = 9 * self.ncell
        eps = default_eps_d(mesh) if eps_d is None else float(eps_d)
        self.sweep = ShardedSweep(n, self.S, params, eps, self.device, align=9, group=group)
        self.c0, self.c1 = self.sweep.lo // 9, self.sweep.hi // 9
        nl = self.sweep.hi - self.sweep.lo
        f64 = torch.float64
        self.coeffs = torch.empty((self.S, self.dm.n_free), dtype=f64, device=self.device)
        self.fields = torch.empty((3 + 3 * self.S, max(nl, 1)), dtype=f64, device=self.device)
        self.csr = torch.empty((self.S, self.dm.map.nnz), dtype=f64, device=self.device)
        # all-gather buffers of (w, K, D) per point: 1 + 6S doubles
        W = self.sweep.world
        self._wkd_w = 1 + 6 * self.S
        mc = self.sweep.plan.max_count
        self._wkd_send = torch.zeros((mc, self._wkd_w), dtype=f64, device=self.device)
        self._wkd_recv = (self._wkd_send if W == 1 else
                          torch.zeros((W * mc, self._wkd_w), dtype=f64, device=self.device))
        self._w_all = torch.empty(n, dtype=f64, device=self.device)
        self._K_all = torch.empty((n, self.S, 2), dtype=f64, device=self.device)
        self._D_all = torch.empty((n, self.S, 2, 2), dtype=f64, device=self.device)
        self._lib = _lib.load()
        self._ctx = self.sweep._ctx  # the sweep's own context (not the cached one)

    def _stream(self):
        import torch

        return torch.cuda.current_stream(self.device).cuda_stream

    def local_fields(self):
        """Views (r, z, w, f, df_r, df_z) of this rank's sampled points."""
        S, F = self.S, self.fields
        nl = self.sweep.hi - self.sweep.lo
        return (F[0, :nl], F[1, :nl], F[2, :nl], F[3:3 + S, :nl], F[3 + S:3 + 2 * S, :nl],
                F[3 + 2 * S:3 + 3 * S, :nl])

    def step(self, coeffs):
        """C blocks (list of S scipy CSR) for the state `coeffs` (S, n_free):
        host array or device tensor; identical on every rank."""
        import scipy.sparse as sp
        import torch

        c = coeffs if isinstance(coeffs, torch.Tensor) else torch.from_numpy(
            np.ascontiguousarray(np.atleast_2d(coeffs), dtype=np.float64))
        self.coeffs.copy_(c)
        st = self._stream()
        lib, h = self._lib, self._ctx.handle
        row = self.fields.stride(0) * 8
        o = self.fields.data_ptr()
        _lib.check(lib.lb_sample_state_dev(
            h, self.dm.handle, self.S, self.c0, self.c1, self.coeffs.data_ptr(), o, o + row,
            o + 2 * row, o + 3 * row, o + (3 + self.S) * row, o + (3 + 2 * self.S) * row, st))
        r, z, w, f, dfr, dfz = (t.contiguous() for t in self.local_fields())
        K, D = self.sweep.step(r, z, w, f, dfr, dfz)
        sw, S = self.sweep, self.S
        if sw.world == 1:
            w_all, K_all, D_all = w, K, D
        else:  # replicate (w, K, D) of every point: one all-gather
            nl = sw.hi - sw.lo
            snd = self._wkd_send
            snd[:nl, 0] = w
            snd[:nl, 1:1 + 2 * S] = K.reshape(nl, 2 * S)
            snd[:nl, 1 + 2 * S:] = D.reshape(nl, 4 * S)
            _dist().all_gather_into_tensor(self._wkd_recv, snd, group=self.group)
            mc = sw.plan.max_count
            for k in range(sw.world):
                lo, hi = sw.plan.bounds(k)
                blk = self._wkd_recv[k * mc:k * mc + (hi - lo)]
                self._w_all[lo:hi] = blk[:, 0]
                self._K_all[lo:hi] = blk[:, 1:1 + 2 * S].reshape(hi - lo, S, 2)
                self._D_all[lo:hi] = blk[:, 1 + 2 * S:].reshape(hi - lo, S, 2, 2)
            w_all, K_all, D_all = self._w_all, self._K_all, self._D_all
        _lib.check(lib.lb_operator_partial_dev(
            h, self.dm.handle, S, 0, self.ncell, w_all.data_ptr(), K_all.data_ptr(),
            D_all.data_ptr(), self.csr.data_ptr(), st))
        vals = self.csr.cpu().numpy()
        gm = self.dm.map
        return [gm.csr_block(vals[a])
                for a in range(self.S)]
