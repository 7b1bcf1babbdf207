"""Drop-in mirror of `axlandau.assembly.assemble_collision` on the B200.

`assemble_collision` (assembly.py:132-175) runs entirely on the device in one
C-ABI call (`lb_assemble_csr`): pair sweep (K1, symmetric all-points path),
outer-point transform and 9x9 element contraction (K2), and the CSR scatter
with hanging-node condensation P^T C P (K3, a per-slot gather-sum through a
map built once per mesh by `scatter.build_gather_map`).  Only the CSR values
come back; the host wraps them in scipy CSR matrices with the mesh's fixed
pattern.

`mesh` is duck-typed on the attributes the reference reads: n_cells, sizes,
cell_nodes, n_nodes, prolongation (scipy CSR), domain.L.  `ref` needs Nq, B,
dB (fem.py:50-63).  `data` must come from sampling on the same mesh
(point n = 9*cell + q).
"""

from __future__ import annotations

import sys
import time
from collections import OrderedDict
from dataclasses import dataclass, field

import numpy as np
import scipy.sparse as sp

from . import _lib
from .kernel import _f64, _host_out, _inner_fields, _n_species, coupling
from .scatter import build_gather_map

__all__ = ["CollisionMatrix", "DeviceMesh", "assemble_at", "assemble_collision",
           "assemble_species_meshes", "default_eps_d", "device_mesh", "element_matrices",
           "sample_state", "union_point_data"]


def default_eps_d(mesh) -> float:
    """Coincident-pair exclusion radius 1e-14 L (assembly.py:57-59)."""
    return 1e-14 * mesh.domain.L


@dataclass
class CollisionMatrix:
    """Per-species CSR blocks over the free dofs + phase timings
    (assembly.py:62-83); timings keys kernel / fe_transform / scatter."""

    blocks: list
    timings: dict = field(default_factory=dict)

    @property
    def n_species(self) -> int:
        return len(self.blocks)

    def apply(self, state) -> np.ndarray:
        coeffs = np.atleast_2d(np.asarray(getattr(state, "coeffs", state), dtype=float))
        return np.stack([self.blocks[a] @ coeffs[a] for a in range(self.n_species)])


def element_matrices(mesh, ref, data, params, eps_d: float | None = None,
                     return_kd: bool = False):
    """Device K1 + K2: element matrices (S, ncell, 9, 9) (assembly.py:148-165),
    plus the phase times in seconds [upload+pack, sweep, contraction+download]
    and optionally the point accumulators K (N,S,2), D (N,S,2,2)."""
    if eps_d is None:
        eps_d = default_eps_d(mesh)
    S = _n_species(params)
    if np.asarray(data.f).shape[0] != S:
        raise ValueError("species count mismatch between data and params")
    if int(ref.Nq) != 9:
        raise ValueError("the B200 path implements the Q2 / 3x3 Gauss element (Nq = 9)")
    ncell = int(mesh.n_cells)
    r, z, w, f, dfr, dfz = _inner_fields(data, S)
    if r.shape[0] != 9 * ncell:
        raise ValueError(f"data has {r.shape[0]} points, mesh has {9 * ncell} quadrature points")
    sizes = _f64(mesh.sizes)
    B = _f64(ref.B)
    dB = _f64(ref.dB)
    coK, coD = coupling(params)
    elem = np.empty((S, ncell, 9, 9))
    K = np.empty((9 * ncell, S, 2)) if return_kd else None
    D = np.empty((9 * ncell, S, 2, 2)) if return_kd else None
    phase = np.zeros(3)
    if ncell:
        ctx = _lib.context()
        p = _lib.dptr
        _lib.check(_lib.load().lb_assemble_elements(
            ctx.handle, ncell, p(sizes), S, p(r), p(z), p(w), p(f), p(dfr), p(dfz),
            p(coK), p(coD), float(eps_d), p(B), p(dB),
            p(K) if return_kd else None, p(D) if return_kd else None, p(elem), p(phase)))
    if return_kd:
        return elem, phase * 1e-3, K, D
    return elem, phase * 1e-3


class DeviceMesh:
    """A mesh resident on one device: cell sizes, Q2 basis tables and the
    CSR gather map (`lb_mesh_create`)."""

    def __init__(self, mesh, ref, device: int):
        self.map = build_gather_map(mesh.cell_nodes, int(mesh.n_nodes), mesh.prolongation)
        ctx = _lib.context(device)
        lib = _lib.load()
        self._lib = lib
        self.ncell = int(mesh.n_cells)
        sizes, B, dB = _f64(mesh.sizes), _f64(ref.B), _f64(ref.dB)
        gm = self.map
        h = _lib.C.c_void_p()
        _lib.check(lib.lb_mesh_create(
            ctx.handle, self.ncell, _lib.dptr(sizes), _lib.dptr(B), _lib.dptr(dB), gm.nnz,
            _lib.iptr(gm.slot_ptr), int(gm.gather_idx.shape[0]), _lib.iptr(gm.gather_idx),
            _lib.dptr(gm.gather_w), _lib.C.byref(h)))
        self.handle = h
        _lib.register_native(self, 1)
        self.n_free = gm.n_free
        self.has_geometry = all(hasattr(mesh, a) for a in ("origins",)) and all(
            hasattr(ref, a) for a in ("qpts", "qwts"))
        if self.has_geometry:  # enables device sampling (sample_state / assemble_at)
            P = sp.csr_matrix(mesh.prolongation)
            P.sum_duplicates()
            ptr = np.ascontiguousarray(P.indptr, dtype=np.int32)
            idx = np.ascontiguousarray(P.indices, dtype=np.int32)
            pw = _f64(P.data)
            cn = np.ascontiguousarray(mesh.cell_nodes, dtype=np.int32)
            _lib.check(lib.lb_mesh_set_geometry(
                h, _lib.dptr(_f64(mesh.origins)), _lib.dptr(_f64(ref.qpts)),
                _lib.dptr(_f64(ref.qwts)), _lib.iptr(cn), int(mesh.n_nodes), P.shape[1],
                _lib.iptr(ptr), _lib.iptr(idx), _lib.dptr(pw)))

    def close(self):
        if getattr(self, "handle", None):
            self._lib.lb_mesh_destroy(self.handle)
            self.handle = None

    def __del__(self, _finalizing=sys.is_finalizing):  # pragma: no cover
        if _finalizing():  # bound at definition: module globals may be gone at shutdown
            return
        try:
            self.close()
        except Exception:
            pass


_MESH_CACHE: "OrderedDict[tuple, tuple]" = OrderedDict()
_MESH_CACHE_SIZE = 8


def device_mesh(mesh, ref, device: int | None = None) -> DeviceMesh:
    """Cached DeviceMesh for (mesh, ref, device).  Meshes are immutable in the
    reference (mesh.py:54-56); the cache holds a reference to the mesh so its
    id cannot be reused while cached."""
    dev = _lib.current_device() if device is None else int(device)
    key = (id(mesh), id(ref), dev)
    hit = _MESH_CACHE.get(key)
    if hit is not None and hit[0] is mesh and hit[1] is ref:
        _MESH_CACHE.move_to_end(key)
        return hit[2]
    dm = DeviceMesh(mesh, ref, dev)
    _MESH_CACHE[key] = (mesh, ref, dm)
    while len(_MESH_CACHE) > _MESH_CACHE_SIZE:
        _MESH_CACHE.popitem(last=False)
    return dm


def assemble_collision(mesh, ref, data, params, eps_d: float | None = None,
                       workers: int = 1) -> CollisionMatrix:
    """C[f] per species (assembly.py:132-175), every phase on the B200.

    `workers` is accepted for signature compatibility; results are bitwise
    deterministic regardless (test_assembly.py:100-111).  `timings` holds the
    device-event times of kernel (upload + pair sweep) and fe_transform
    (contraction + scatter + download); the host CSR wrap goes to scatter.
    """
    if eps_d is None:
        eps_d = default_eps_d(mesh)
    S = _n_species(params)
    if np.asarray(data.f).shape[0] != S:
        raise ValueError("species count mismatch between data and params")
    if int(ref.Nq) != 9:
        raise ValueError("the B200 path implements the Q2 / 3x3 Gauss element (Nq = 9)")
    ncell = int(mesh.n_cells)
    r, z, w, f, dfr, dfz = _inner_fields(data, S)
    if r.shape[0] != 9 * ncell:
        raise ValueError(f"data has {r.shape[0]} points, mesh has {9 * ncell} quadrature points")
    t0 = time.perf_counter()
    dm = device_mesh(mesh, ref)
    gm = dm.map
    coK, coD = coupling(params)
    csr = _host_out((S, gm.nnz))
    phase = np.zeros(3)
    t1 = time.perf_counter()
    if ncell:
        ctx = _lib.context()
        p = _lib.dptr
        _lib.check(_lib.load().lb_assemble_csr(
            ctx.handle, dm.handle, S, p(r), p(z), p(w), p(f), p(dfr), p(dfz), p(coK), p(coD),
            float(eps_d), p(csr), None, None, p(phase)))
    t2 = time.perf_counter()
    n_free = gm.n_free
    blocks = [gm.csr_block(csr[a])
              for a in range(S)]
    t3 = time.perf_counter()
    host = max(t2 - t1 - float(phase.sum()) * 1e-3, 0.0)
    return CollisionMatrix(
        blocks=blocks,
        timings={"kernel": float(phase[0] + phase[1]) * 1e-3 + host,
                 "fe_transform": float(phase[2]) * 1e-3,
                 "scatter": (t1 - t0) + (t3 - t2)},
    )


def _coeffs(state, S_expected: int | None, n_free: int) -> np.ndarray:
    c = np.atleast_2d(np.ascontiguousarray(getattr(state, "coeffs", state), dtype=np.float64))
    if c.shape[1] != n_free:
        raise ValueError(f"state has {c.shape[1]} dofs, mesh has {n_free} free nodes")
    if S_expected is not None and c.shape[0] != S_expected:
        raise ValueError("species count mismatch between state and params")
    return c


def assemble_at(mesh, ref, state, params, eps_d: float | None = None,
                return_data: bool = False):
    """State-level operator: `solver._assemble_at` (solver.py:81-84) =
    `sample_state` + `assemble_collision`, in one device call
    (`lb_assemble_state`): nodal coefficients in, CSR blocks out."""
    if eps_d is None:
        eps_d = default_eps_d(mesh)
    S = _n_species(params)
    dm = device_mesh(mesh, ref)
    if not dm.has_geometry:
        raise ValueError("mesh/ref lack origins/qpts/qwts needed for device sampling")
    c = _coeffs(state, S, dm.n_free)
    gm = dm.map
    coK, coD = coupling(params)
    csr = _host_out((S, gm.nnz))
    n = 9 * dm.ncell
    data = np.empty((3 + 3 * S, n)) if return_data else None
    phase = np.zeros(3)
    t0 = time.perf_counter()
    if dm.ncell:
        ctx = _lib.context()
        p = _lib.dptr
        _lib.check(_lib.load().lb_assemble_state(
            ctx.handle, dm.handle, S, p(c), p(coK), p(coD), float(eps_d), p(csr),
            p(data) if return_data else None, p(phase)))
    t1 = time.perf_counter()
    blocks = [gm.csr_block(csr[a])
              for a in range(S)]
    t2 = time.perf_counter()
    host = max(t1 - t0 - float(phase.sum()) * 1e-3, 0.0)
    cm = CollisionMatrix(blocks=blocks, timings={
        "kernel": float(phase[0] + phase[1]) * 1e-3 + host,
        "fe_transform": float(phase[2]) * 1e-3, "scatter": t2 - t1})
    if return_data:
        from .kernel import QuadPointData

        qd = QuadPointData(N=n, r=data[0], z=data[1], w=data[2], f=data[3:3 + S],
                           df_r=data[3 + S:3 + 2 * S], df_z=data[3 + 2 * S:3 + 3 * S])
        return cm, qd
    return cm


def sample_state(mesh, ref, state):
    """Device `sample_state` (fem.py:170-199): QuadPointData of the state at
    all quadrature points, bitwise the reference's (`lb_sample_state`, host
    pointers in and out)."""
    dm = device_mesh(mesh, ref)
    if not dm.has_geometry:
        raise ValueError("mesh/ref lack origins/qpts/qwts needed for device sampling")
    c = _coeffs(state, None, dm.n_free)
    S = c.shape[0]
    n = 9 * dm.ncell
    out = np.empty((3 + 3 * S, n))
    if n:
        ctx = _lib.context()
        _lib.check(_lib.load().lb_sample_state(ctx.handle, dm.handle, S, _lib.dptr(c),
                                               _lib.dptr(out)))
    from .kernel import QuadPointData

    return QuadPointData(N=n, r=out[0], z=out[1], w=out[2], f=out[3:3 + S],
                         df_r=out[3 + S:3 + 2 * S], df_z=out[3 + 2 * S:3 + 3 * S])


def union_point_data(datas):
    """Species-tagged union of per-species point sets:
    datas[a] is species a's QuadPointData on its own mesh (one species row,
    or S rows of which row a is used); the union carries species a's fields
    on its own points and exact zeros elsewhere, so one all-points sweep over
    the union is the exact multi-mesh D/K.  Returns (QuadPointData, offsets)."""
    from .kernel import QuadPointData

    S = len(datas)
    ns = [int(np.asarray(d.r).shape[0]) for d in datas]
    off = np.concatenate([[0], np.cumsum(ns)]).astype(np.int64)
    n = int(off[-1])
    f = np.zeros((S, n))
    dfr = np.zeros((S, n))
    dfz = np.zeros((S, n))
    for a, d in enumerate(datas):
        row = 0 if np.atleast_2d(d.f).shape[0] == 1 else a
        sl = slice(off[a], off[a + 1])
        f[a, sl] = np.atleast_2d(d.f)[row]
        dfr[a, sl] = np.atleast_2d(d.df_r)[row]
        dfz[a, sl] = np.atleast_2d(d.df_z)[row]
    def cat(k):
        return np.ascontiguousarray(np.concatenate([np.asarray(getattr(d, k)) for d in datas]))

    return QuadPointData(N=n, r=cat("r"), z=cat("z"), w=cat("w"), f=f, df_r=dfr, df_z=dfz), off


def assemble_species_meshes(meshes, ref, datas, params, eps_d: float | None = None):
    """C_a for species a on its OWN mesh (the paper's per-species meshes,
    PAPER.md section 3.0.2; BASELINE configs 2 and 4 as worded).  One
    all-points sweep over the species-tagged union point set (symmetric,
    species-collapsed) gives every point's K/D; species a's block is then the
    element contraction + scatter on mesh a with its points' K[:, a], D[:, a]
    (`lb_elements_csr`).  eps_d defaults to 1e-14 * min_a L_a.
    Returns (list of S CSR blocks, (K, D) of the union points)."""
    from .kernel import fused_sweep

    S = _n_species(params)
    if len(meshes) != S or len(datas) != S:
        raise ValueError("need one mesh and one QuadPointData per species")
    if eps_d is None:
        eps_d = min(default_eps_d(m) for m in meshes)
    union, off = union_point_data(datas)
    K, D = fused_sweep(union.r, union.z, union, params, eps_d=eps_d)
    blocks = []
    for a, mesh in enumerate(meshes):
        dm = device_mesh(mesh, ref)
        gm = dm.map
        sl = slice(off[a], off[a + 1])
        if off[a + 1] - off[a] != 9 * dm.ncell:
            raise ValueError(f"species {a}: data points do not match its mesh")
        w = np.ascontiguousarray(union.w[sl])
        Ka = np.ascontiguousarray(K[sl, a:a + 1])
        Da = np.ascontiguousarray(D[sl, a:a + 1])
        csr = np.empty((1, gm.nnz))
        if dm.ncell:
            ctx = _lib.context()
            p = _lib.dptr
            _lib.check(_lib.load().lb_elements_csr(ctx.handle, dm.handle, 1, p(w), p(Ka), p(Da),
                                                   p(csr)))
        blocks.append(gm.csr_block(csr[0]))
    return blocks, (K, D)
