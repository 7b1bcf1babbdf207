"""Drop-in mirror of the Crank-Nicolson Newton step of `axlandau.solver` on
the B200.

The reference (solver.py:103-150) assembles C at the Newton guess, forms the
residual R = M (g - f) - dt/2 (C[g] g + C_old f) and solves
(M - dt/2 C_a) delta = -R per species with SuperLU (`splu`, solver.py:
124-133).  Here one C-ABI call (`lb_cn_newton`) does all of it on the device:
the operator is assembled at the guess without leaving the GPU (device
sampling + symmetric pair sweep + element contraction + CSR gather), the
residual and the systems are formed there, and the systems are solved by a
block-tridiagonal LU of the banded matrix, batched over species:

  * the free nodes are permuted into a banded order once per mesh (the
    mesh's natural order or reverse Cuthill-McKee, whichever has the smaller
    bandwidth b) and cut into blocks of nb = b rows, so every system is block
    tridiagonal with nb x nb blocks;
  * block LU with partial pivoting inside each diagonal block (cuBLAS
    batched getrf/getrs/gemm over the S species), then block forward and
    back substitution.

`newton_step` and `linear_cn_step` keep the reference signatures, return
types and error behaviour (StepFailure on a singular system or a non-finite
update); `install()` routes the reference's `advance` through them.
"""

from __future__ import annotations

import sys
from collections import OrderedDict

import numpy as np
import scipy.sparse as sp
from scipy.sparse.csgraph import reverse_cuthill_mckee

from . import _lib
from .assembly import default_eps_d, device_mesh
from .kernel import _n_species, coupling

__all__ = ["CNSolver", "StepFailure", "backward_euler_step", "band_order", "linear_cn_step",
           "mass_matrix", "newton_step", "pattern_values", "species_meshes_step", "theta_step"]


class StepFailure(RuntimeError):
    """A time step could not be completed (solver.py:48-54)."""

    def __init__(self, step: int, message: str):
        super().__init__(f"step {step}: {message}")
        self.step = step


# install() points this at the reference's class so its `except StepFailure`
# (solver.py:178-181) catches failures raised here
_StepFailure = StepFailure


def band_order(indptr: np.ndarray, indices: np.ndarray, n: int):
    """(perm, bandwidth) for the block-tridiagonal solve: the natural order or
    reverse Cuthill-McKee, whichever gives the smaller bandwidth.  perm[p] is
    the free node at band position p."""
    A = sp.csr_matrix((np.ones(indices.shape[0]), indices, indptr), shape=(n, n))
    rows = np.repeat(np.arange(n), np.diff(indptr))
    best = None
    for perm in (np.arange(n), reverse_cuthill_mckee(A, symmetric_mode=True)):
        inv = np.empty(n, dtype=np.int64)
        inv[perm] = np.arange(n)
        bw = int(np.abs(inv[rows] - inv[indices]).max()) if indices.shape[0] else 0
        if best is None or bw < best[1]:
            best = (np.ascontiguousarray(perm, dtype=np.int32), bw)
    return best


def pattern_values(A, indptr: np.ndarray, indices: np.ndarray, n: int) -> np.ndarray:
    """Values of the sparse matrix A in the CSR pattern (indptr, indices);
    entries of the pattern absent from A are 0.  ValueError if A has a
    non-zero outside the pattern."""
    A = sp.csr_matrix(A)
    if A.shape != (n, n):
        raise ValueError(f"matrix shape {A.shape} does not match the mesh ({n} free nodes)")
    if (A.indptr.shape == indptr.shape and np.array_equal(A.indptr, indptr)
            and np.array_equal(A.indices, indices)):
        return np.ascontiguousarray(A.data, dtype=np.float64)
    A = A.copy()
    A.sum_duplicates()
    rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(A.indptr))
    keys = rows * n + A.indices
    prow = np.repeat(np.arange(n, dtype=np.int64), np.diff(indptr))
    pkeys = prow * n + indices
    pos = np.searchsorted(pkeys, keys)
    pos = np.minimum(pos, pkeys.shape[0] - 1)
    ok = pkeys[pos] == keys
    if not np.all(ok | (A.data == 0.0)):
        raise ValueError("matrix has entries outside the mesh's Q2 pattern")
    out = np.zeros(indices.shape[0])
    out[pos[ok]] = A.data[ok]
    return out


class CNSolver:
    """Device Crank-Nicolson solver for one pattern and species count
    (`lb_cn_*`).  With a DeviceMesh the pattern is the mesh's operator
    pattern and Newton steps assemble the operator on the device."""

    def __init__(self, indptr, indices, n: int, S: int, dm=None, device: int | None = None):
        self.n, self.S = int(n), int(S)
        self.indptr = np.ascontiguousarray(indptr, dtype=np.int64)
        self.indices = np.ascontiguousarray(indices, dtype=np.int32)
        self.perm, self.bandwidth = band_order(self.indptr, self.indices, self.n)
        self.nb = max(self.bandwidth, 1)
        self._lib = _lib.load()
        ctx = _lib.context(device)
        h = _lib.C.c_void_p()
        _lib.check(self._lib.lb_cn_create(
            ctx.handle, dm.handle if dm is not None else None, self.S, self.n,
            _lib.iptr(np.ascontiguousarray(self.indptr, dtype=np.int32)), _lib.iptr(self.indices),
            _lib.iptr(self.perm), self.nb, _lib.C.byref(h)))
        self.handle = h
        self.dm = dm
        _lib.register_native(self, 0)
        self._mass_key = None
        self._c_old_ref = None  # CollisionMatrix whose values are resident as C_old

    def set_mass(self, M=None):
        """Mass values: the caller's matrix mapped onto the pattern, or (None)
        assembled on the device (fem.py:152-167).  Re-uploaded only when M
        changes: by identity plus a content fingerprint, so in-place edits of
        M are picked up."""
        key = ("device",) if M is None else ("host", id(M), _fingerprint(M))
        if key == self._mass_key:
            return
        vals = None if M is None else pattern_values(M, self.indptr, self.indices, self.n)
        _lib.check(self._lib.lb_cn_set_mass(self.handle, _lib.dptr(vals) if vals is not None else None))
        self._mass_key = key
        self._mass_ref = M  # keep M alive so its id is not reused while cached

    def mass_values(self) -> np.ndarray:
        out = np.empty(self.indices.shape[0])
        _lib.check(self._lib.lb_cn_get_mass(self.handle, _lib.dptr(out)))
        return out

    def stats(self) -> dict:
        """Last solve's relative backward error, rejected unpivoted
        factorisations, and whether the solver pivots now (lb_cn_stats)."""
        import ctypes as C

        r, nf, pv = C.c_double(), C.c_int(), C.c_int()
        _lib.check(self._lib.lb_cn_stats(self.handle, C.byref(r), C.byref(nf), C.byref(pv)))
        return {"rel_residual": r.value, "fallbacks": nf.value, "pivoting": bool(pv.value)}

    def block_values(self, blocks) -> np.ndarray:
        return np.stack([pattern_values(b, self.indptr, self.indices, self.n) for b in blocks])

    def close(self):
        if getattr(self, "handle", None):
            self._lib.lb_cn_destroy(self.handle)
            self.handle = None

    def __del__(self, _finalizing=sys.is_finalizing):  # pragma: no cover
        if _finalizing():  # bound at definition: module globals may be gone at shutdown
            return
        try:
            self.close()
        except Exception:
            pass


def _fingerprint(M) -> tuple:
    """Cheap content key of a sparse (or dense) matrix: shape, nnz and the
    XOR of the bit patterns of its values and of its indices -- one pass
    each (any single edited entry changes the key); this runs on every
    newton_step, so it stays well under the step's device time."""
    data = np.ascontiguousarray(getattr(M, "data", M), dtype=np.float64).ravel()
    key = (getattr(M, "shape", None), data.size,
           int(np.bitwise_xor.reduce(data.view(np.int64))) if data.size else 0)
    idx = getattr(M, "indices", None)
    if idx is not None and idx.size:
        key += (int(np.bitwise_xor.reduce(np.ascontiguousarray(idx).ravel())), int(idx[0]), int(idx[-1]))
    return key


_SOLVERS: "OrderedDict[tuple, tuple]" = OrderedDict()
_SOLVERS_SIZE = 4


def _mesh_solver(mesh, ref, S: int) -> CNSolver:
    dm = device_mesh(mesh, ref)
    key = (id(dm), S)
    hit = _SOLVERS.get(key)
    if hit is not None and hit[0] is dm:
        _SOLVERS.move_to_end(key)
        return hit[1]
    gm = dm.map
    s = CNSolver(gm.indptr, gm.indices, gm.n_free, S, dm=dm)
    _SOLVERS[key] = (dm, s)
    while len(_SOLVERS) > _SOLVERS_SIZE:
        _SOLVERS.popitem(last=False)
    return s


def _coeffs_of(state) -> np.ndarray:
    return np.ascontiguousarray(np.atleast_2d(getattr(state, "coeffs", state)), dtype=np.float64)


def _with_coeffs(state, coeffs: np.ndarray):
    if hasattr(state, "coeffs"):
        out = state.copy()
        out.coeffs[...] = coeffs.reshape(out.coeffs.shape)
        return out
    return coeffs.reshape(np.shape(state))


_MASS: "OrderedDict[int, tuple]" = OrderedDict()


def mass_matrix(mesh, ref):
    """fem.mass_matrix (fem.py:150-165): the r-weighted Q2 mass matrix on the
    free dofs, by the reference's own numpy/scipy operations (so bitwise
    equal to it: newton_step(M=None) must give exactly what newton_step(M=
    mass_matrix(mesh, ref)) gives, test_solver.py:166-176).  Mesh-constant
    set-up, off the operator's hot path; cached per mesh.  The device
    assembly of the same matrix is `CNSolver.set_mass(None)`."""
    key = id(mesh)
    hit = _MASS.get(key)
    if hit is not None and hit[0] is mesh:
        return hit[1]
    sizes = np.asarray(mesh.sizes, dtype=np.float64)
    dr, dz = sizes[:, 0], sizes[:, 1]
    nq = int(ref.Nq)
    detJ = np.broadcast_to((dr * dz / 4.0)[:, None], (sizes.shape[0], nq)).copy()
    coords = (np.asarray(mesh.origins)[:, None, :]
              + (np.asarray(ref.qpts)[None, :, :] + 1.0) * 0.5 * sizes[:, None, :])
    weights = np.asarray(ref.qwts)[None, :] * detJ * coords[:, :, 0]
    elem = np.einsum("iq,jq,eq->eij", ref.B, ref.B, weights)
    cn = np.asarray(mesh.cell_nodes)
    rows = np.repeat(cn, 9, axis=1).ravel()
    cols = np.tile(cn, (1, 9)).ravel()
    nn = int(mesh.n_nodes)
    Mn = sp.csr_matrix((elem.ravel(), (rows, cols)), shape=(nn, nn))
    P = mesh.prolongation
    M = (P.T @ Mn @ P).tocsr()
    _MASS[key] = (mesh, M)
    while len(_MASS) > 8:
        _MASS.popitem(last=False)
    return M


def newton_step(f_guess, f_old, mesh, ref, params, cfg, M=None, C_old=None):
    """solver.newton_step (solver.py:103-134) on the device: returns
    (f_next, rel_residual).  M / C_old as in the reference: None assembles
    them here -- M by the reference's own operations (`mass_matrix`), C_old
    on the device at f_old (bitwise what assemble_collision(sample_state)
    gives: device sampling reproduces fem.sample_state's arithmetic)."""
    S = _n_species(params)
    g, f = _coeffs_of(f_guess), _coeffs_of(f_old)
    if g.shape != f.shape:
        raise ValueError("state shapes differ")
    if g.shape[0] != S:
        raise ValueError("species count mismatch between state and params")
    solver = _mesh_solver(mesh, ref, S)
    if g.shape[1] != solver.n:
        raise ValueError(f"state has {g.shape[1]} dofs, mesh has {solver.n} free nodes")
    solver.set_mass(mass_matrix(mesh, ref) if M is None else M)
    # C_old: advance() hands the same CollisionMatrix to every Newton
    # iteration of a step (solver.py:171-181); it is uploaded once and kept
    # resident on the device for the following iterations
    Cv, mode = None, 0
    if C_old is not None:
        if C_old is solver._c_old_ref:
            mode = 2
        else:
            Cv, mode = solver.block_values(C_old.blocks), 1
    eps = getattr(cfg, "eps_d", None)
    eps = default_eps_d(mesh) if eps is None else float(eps)
    coK, coD = coupling(params)
    out = np.empty_like(g)
    rnorm = np.zeros(1)
    phase = np.zeros(4)
    # the device C_old is overwritten (mode 0/1) before anything can fail, so
    # the resident-copy marker is cleared first and set again only on success
    solver._c_old_ref = None
    try:
        _lib.check(solver._lib.lb_cn_newton(
            solver.handle, _lib.dptr(coK), _lib.dptr(coD), eps, float(cfg.dt), _lib.dptr(g),
            _lib.dptr(f), _lib.dptr(Cv) if Cv is not None else None, mode, _lib.dptr(out), None,
            _lib.dptr(rnorm), _lib.dptr(phase)))
    except _lib.SingularSystem as err:
        raise _StepFailure(-1, f"linear solve failed: {err}") from err
    solver._c_old_ref = C_old  # held: its identity marks the resident copy
    # device phase times (ms) of the last call: assembly, residual + band
    # fill, block LU, solve + download
    LAST_PHASES_MS[:] = phase
    return _with_coeffs(f_guess, out), float(rnorm[0])


LAST_PHASES_MS = np.zeros(4)

_LINEAR: "OrderedDict[tuple, CNSolver]" = OrderedDict()


def linear_cn_step(M, C, dt: float, state):
    """solver.linear_cn_step (solver.py:137-150) on the device: solves
    (M - dt/2 C_a) f+ = (M + dt/2 C_a) f per species with C held fixed."""
    return theta_step(M, C, dt, state, 0.5)


def backward_euler_step(M, C, dt: float, state):
    """Backward-Euler step with C held fixed, (M - dt C_a) f+ = M f per
    species -- the time step BASELINE configs 1-2 name; the reference has
    Crank-Nicolson only, so this is the composition of its pieces (SURVEY
    8(c)(iii)) on the device solver."""
    return theta_step(M, C, dt, state, 1.0)


def theta_step(M, C, dt: float, state, theta: float):
    """(M - theta dt C_a) f+ = (M + (1 - theta) dt C_a) f per species with C
    held fixed (lb_cn_theta_step): theta = 1/2 Crank-Nicolson, 1 backward
    Euler."""
    f = _coeffs_of(state)
    S = f.shape[0]
    if len(C.blocks) != S:
        raise ValueError("species count mismatch between state and C")
    pat = sp.csr_matrix(M, copy=True)
    pat.data[:] = 1.0
    for b in C.blocks:
        bb = sp.csr_matrix(b, copy=True)
        bb.data[:] = 1.0
        pat = pat + bb
    pat.sum_duplicates()
    pat.sort_indices()
    n = pat.shape[0]
    key = (n, S, pat.indptr.tobytes(), pat.indices.tobytes())
    solver = _LINEAR.get(key)
    if solver is None:
        solver = CNSolver(pat.indptr, pat.indices, n, S)
        _LINEAR[key] = solver
        while len(_LINEAR) > _SOLVERS_SIZE:
            _LINEAR.popitem(last=False)
    solver.set_mass(M)
    Cv = solver.block_values(C.blocks)
    out = np.empty_like(f)
    try:
        _lib.check(solver._lib.lb_cn_theta_step(solver.handle, float(dt), float(theta), _lib.dptr(Cv),
                                                _lib.dptr(f), _lib.dptr(out)))
    except _lib.SingularSystem as err:
        raise _StepFailure(-1, f"linear solve failed: {err}") from err
    return _with_coeffs(state, out)


def species_meshes_step(meshes, ref, states, params, dt: float, masses, theta: float = 1.0,
                        eps_d: float | None = None):
    """One time step with every species on its own mesh (PAPER.md section
    3.0.2; BASELINE config 2 as worded): C_a at the current state from ONE
    device sweep over the species-tagged union point set
    (`assemble_species_meshes`; device sampling of each mesh), then per
    species the theta step on its own mesh, (M_a - theta dt C_a) f_a+ =
    (M_a + (1 - theta) dt C_a) f_a -- theta = 1 (default) is backward Euler.
    `states[a]` is species a's coefficient vector on meshes[a], `masses[a]`
    its mass matrix (CSR).  Returns the new list of coefficient vectors."""
    from types import SimpleNamespace

    from .assembly import assemble_species_meshes, sample_state

    if not (len(meshes) == len(states) == len(masses)):
        raise ValueError("need one mesh, state and mass matrix per species")
    coeffs = [np.ascontiguousarray(np.asarray(getattr(c, "coeffs", c), dtype=np.float64).reshape(-1))
              for c in states]
    datas = [sample_state(mesh, ref, c[None, :]) for mesh, c in zip(meshes, coeffs)]
    blocks, _ = assemble_species_meshes(meshes, ref, datas, params, eps_d=eps_d)
    return [theta_step(M, SimpleNamespace(blocks=[blocks[a]]), dt, coeffs[a][None, :], theta)[0]
            for a, M in enumerate(masses)]
