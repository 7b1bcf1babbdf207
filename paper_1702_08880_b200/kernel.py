"""Drop-in mirror of `axlandau.kernel` for the O(N^2) pair integral.

Same names, argument meaning and error behaviour as the reference
(`pkg/src/axlandau/kernel.py`); the arithmetic runs in the sm_100a CUDA
library through the C ABI (include/landau_b200.h).  Inputs may be the
reference's own `QuadPointData` / `CollisionParams` objects or the mirrors
defined here (duck-typed on the attribute names).

Reference -> this module
  CollisionParams      kernel.py:243-267  -> CollisionParams (same validation)
  Accumulators         kernel.py:270-282  -> Accumulators
  _coupling            kernel.py:496-501  -> coupling
  fused_sweep          kernel.py:504-536  -> fused_sweep (lb_fused_sweep)
  fused_inner_loop     kernel.py:539-557  -> fused_inner_loop
  axisym_tensor_pair   kernel.py:206-235  -> axisym_tensor_pair(s) (lb_tensor_pairs)
  flop_count           kernel.py:560-574  -> flop_count (the metric's flop model)
  QuadPointData        fem.py:133-149     -> QuadPointData
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib

__all__ = [
    "QuadPointData",
    "CollisionParams",
    "Accumulators",
    "LandauTensorPair",
    "coupling",
    "fused_sweep",
    "fused_inner_loop",
    "axisym_tensor_pair",
    "axisym_tensor_pairs",
    "flop_count",
]

_BLK = 256  # accepted for signature compatibility (kernel.py:301); no effect


@dataclass(frozen=True)
class QuadPointData:
    """Structure-of-arrays state at the quadrature points (fem.py:133-149):
    r, z, w (N,); f, df_r, df_z (S, N); point n = 9*cell + q."""

    N: int
    r: np.ndarray
    z: np.ndarray
    w: np.ndarray
    f: np.ndarray
    df_r: np.ndarray
    df_z: np.ndarray


@dataclass(frozen=True)
class CollisionParams:
    """nu_hat (S, S) and mass_ratio_o (S,), validated as kernel.py:255-263."""

    nu_hat: np.ndarray
    mass_ratio_o: np.ndarray

    def __post_init__(self):
        nu = np.asarray(self.nu_hat, dtype=float)
        mro = np.asarray(self.mass_ratio_o, dtype=float)
        if nu.ndim != 2 or nu.shape[0] != nu.shape[1] or nu.shape[0] != mro.shape[0]:
            raise ValueError("nu_hat must be SxS and mass_ratio_o length S")
        if not (nu > 0).all():
            raise ValueError("collision frequencies must be positive")
        object.__setattr__(self, "nu_hat", np.ascontiguousarray(nu))
        object.__setattr__(self, "mass_ratio_o", np.ascontiguousarray(mro))

    @property
    def n_species(self) -> int:
        return self.mass_ratio_o.shape[0]


@dataclass
class Accumulators:
    """Per-outer-point K (S, 2) and D (S, 2, 2) (kernel.py:270-282)."""

    K: np.ndarray
    D: np.ndarray
    G2: np.ndarray | None = None
    G3: np.ndarray | None = None


@dataclass(frozen=True)
class LandauTensorPair:
    UK: np.ndarray
    UD: np.ndarray


def _n_species(params) -> int:
    return int(np.asarray(params.mass_ratio_o).shape[0])


def coupling(params):
    """coK = nu (m_o/m_a)(m_o/m_b), coD = -nu (m_o/m_a)^2 (kernel.py:496-501),
    with the reference's exact numpy expression order."""
    nu = np.asarray(params.nu_hat, dtype=float)
    mro = np.asarray(params.mass_ratio_o, dtype=float)
    coK = nu * mro[:, None] * mro[None, :]
    coD = -nu * (mro**2)[:, None]
    return np.ascontiguousarray(coK), np.ascontiguousarray(coD)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


_PINNED = None  # torch module when page-locked output staging is available


def _host_out(shape) -> np.ndarray:
    """Output array for a device->host copy: page-locked memory from torch's
    caching host allocator when CUDA is up (the copy then runs at full link
    speed instead of through the driver's pageable staging), else plain
    numpy.  Either way the caller gets an ordinary float64 ndarray (a
    pinned one keeps its torch storage alive through `.base`)."""
    global _PINNED
    if _PINNED is None:
        try:
            import torch

            _PINNED = torch if torch.cuda.is_available() else False
        except Exception:  # pragma: no cover
            _PINNED = False
    if _PINNED is False:
        return np.empty(shape)
    return _PINNED.empty(shape, dtype=_PINNED.float64, pin_memory=True).numpy()


def _inner_fields(data, S: int):
    r, z, w = _f64(data.r), _f64(data.z), _f64(data.w)
    f, dfr, dfz = _f64(data.f), _f64(data.df_r), _f64(data.df_z)
    n = r.shape[0]
    for name, a, shp in (("z", z, (n,)), ("w", w, (n,)), ("f", f, (S, n)),
                         ("df_r", dfr, (S, n)), ("df_z", dfz, (S, n))):
        if a.shape != shp:
            raise ValueError(f"QuadPointData.{name} has shape {a.shape}, expected {shp}")
    return r, z, w, f, dfr, dfz


def fused_sweep(outer_r, outer_z, data, params, eps_d: float = 0.0,
                workers: int = 1, block_size: int = _BLK):
    """(K (Nout,S,2), D (Nout,S,2,2)) for arbitrary outer points against all
    inner points of `data` -- the reference `fused_sweep` (kernel.py:504-536)
    on the B200.

    `workers` and `block_size` are accepted for signature compatibility and
    do not change the result (the reference asserts bitwise invariance to
    both, test_kernel.py:197-212; here the decomposition is fixed by the
    inner count alone).  Pairs with d^2 < eps_d^2 or d^2 == 0 are excluded.
    """
    ro, zo = _f64(outer_r), _f64(outer_z)
    S = _n_species(params)
    if np.asarray(data.f).shape[0] != S:
        raise ValueError("species count mismatch between data and params")
    if ro.ndim != 1 or zo.shape != ro.shape:
        raise ValueError("outer_r and outer_z must be 1-D arrays of equal length")
    if S > _lib.MAX_SPECIES:
        raise ValueError(f"at most {_lib.MAX_SPECIES} species are supported")
    r, z, w, f, dfr, dfz = _inner_fields(data, S)
    coK, coD = coupling(params)
    nout, n = ro.shape[0], r.shape[0]
    if nout == 0:
        return np.empty((0, S, 2)), np.empty((0, S, 2, 2))
    K = _host_out((nout, S, 2))
    D = _host_out((nout, S, 2, 2))
    ctx = _lib.context()
    p = _lib.dptr
    if nout == n and (ro is r or np.array_equal(ro, r)) and (zo is z or np.array_equal(zo, z)):
        # all-points sweep (assemble_collision's call, assembly.py:148): each
        # unordered pair is evaluated once on the device (symmetric path)
        _lib.check(_lib.load().lb_fused_sweep_all(
            ctx.handle, n, S, p(r), p(z), p(w), p(f), p(dfr), p(dfz), p(coK), p(coD),
            float(eps_d), p(K), p(D)))
        return K, D
    _lib.check(_lib.load().lb_fused_sweep(
        ctx.handle, nout, p(ro), p(zo), n, S, p(r), p(z), p(w), p(f), p(dfr), p(dfz),
        p(coK), p(coD), float(eps_d), p(K), p(D)))
    return K, D


def fused_inner_loop(outer, data, params, eps_d: float = 0.0,
                     block_size: int = _BLK) -> Accumulators:
    """Accumulators at one outer point (kernel.py:539-557)."""
    ri, zi = float(outer[0]), float(outer[1])
    K, D = fused_sweep(np.array([ri]), np.array([zi]), data, params,
                       eps_d=eps_d, block_size=block_size)
    return Accumulators(K=K[0], D=D[0])


def elliptic_KE(m):
    """Complete elliptic integrals (K(m), E(m)) for m in [0, 1)
    (kernel.py:93-113) on the device: the reference's polynomial fits in
    x = 1 - m with the device table log.  Scalars in, floats out; arrays in,
    arrays out; ValueError outside [0, 1)."""
    m_arr = np.asarray(m, dtype=np.float64)
    if np.any(m_arr < 0.0) or np.any(m_arr >= 1.0) or np.any(np.isnan(m_arr)):
        raise ValueError("elliptic parameter must satisfy 0 <= m < 1")
    flat = np.ascontiguousarray(m_arr.ravel())
    K = np.empty_like(flat)
    E = np.empty_like(flat)
    if flat.size:
        ctx = _lib.context()
        _lib.check(_lib.load().lb_elliptic_ke(ctx.handle, flat.size, _lib.dptr(flat), _lib.dptr(K),
                                              _lib.dptr(E)))
    if np.isscalar(m) or np.ndim(m) == 0:
        return float(K[0]), float(E[0])
    return K.reshape(m_arr.shape), E.reshape(m_arr.shape)


def axisym_tensor_pairs(r, z, rbar, zbar):
    """Vectorized device evaluation of the azimuthally integrated tensors
    (UK, UD), each (npair, 2, 2), with the sweep's own device arithmetic.
    Coincident pairs give zeros (the sweep's mask)."""
    r, z, rb, zb = (np.atleast_1d(_f64(a)) for a in (r, z, rbar, zbar))
    r, z, rb, zb = (np.ascontiguousarray(a) for a in np.broadcast_arrays(r, z, rb, zb))
    if np.any(r < 0.0) or np.any(rb < 0.0):
        raise ValueError("radial coordinates must be non-negative")
    npair = r.shape[0]
    UK = np.empty((npair, 2, 2))
    UD = np.empty((npair, 2, 2))
    if npair:
        ctx = _lib.context()
        p = _lib.dptr
        _lib.check(_lib.load().lb_tensor_pairs(ctx.handle, npair, p(r), p(z), p(rb), p(zb),
                                               p(UK), p(UD)))
    return UK, UD


def axisym_tensor_pair(r, z, rbar, zbar) -> LandauTensorPair:
    """Scalar form of `axisym_tensor_pair` (kernel.py:206-235), same
    ValueErrors for negative radii and coincident points."""
    if r < 0.0 or rbar < 0.0:
        raise ValueError("radial coordinates must be non-negative")
    if (r - rbar) ** 2 + (z - zbar) ** 2 == 0.0:
        raise ValueError("azimuthal tensors are singular at coincident points")
    UK, UD = axisym_tensor_pairs([r], [z], [rbar], [zbar])
    return LandauTensorPair(UK=UK[0], UD=UD[0])


def flop_count(N: int, S: int, outer_evals: int, overhead_per_outer: int = 0) -> int:
    """Flop model 165 + 20 S^2 per pair (kernel.py:560-574): the reporting
    convention of the headline metric."""
    if N < 0 or S < 0 or outer_evals < 0:
        raise ValueError("counts must be non-negative")
    return outer_evals * (N * (165 + 20 * S * S) + overhead_per_outer)
