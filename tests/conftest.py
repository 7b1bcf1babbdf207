"""Shared fixtures.  `-m gpu` tests need a CUDA device (B200) and the built
liblandau_b200.so; everything else runs on CPU."""

from __future__ import annotations

import sys
from pathlib import Path
from types import SimpleNamespace

import numpy as np
import pytest
import scipy.sparse as sp

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = ROOT / "tests" / "golden"
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built library")
    config.addinivalue_line("markers", "slow: long-running (full-size) case")


def golden(name: str):
    return np.load(GOLDEN / f"{name}.npz")


class Prefixed:
    """View of a fixture with keys 'prefix' + k (per-species mesh fixtures)."""

    def __init__(self, g, prefix):
        self.g, self.p = g, prefix

    def __getitem__(self, k):
        return self.g[self.p + k]

    def __contains__(self, k):
        return (self.p + k) in self.g


def csr_from(g, prefix):
    shape = tuple(int(v) for v in g[f"{prefix}_shape"])
    return sp.csr_matrix((g[f"{prefix}_data"], g[f"{prefix}_indices"], g[f"{prefix}_indptr"]),
                         shape=shape)


def blocks_from(g, prefix="C"):
    return [csr_from(g, f"{prefix}{a}") for a in range(int(g[f"{prefix}_count"]))]


def mesh_from(g):
    """Duck-typed stand-in for axlandau's VelocityMesh with exactly the
    attributes assemble_collision reads (assembly.py:153-169)."""
    cn = g["mesh_cell_nodes"]
    return SimpleNamespace(
        n_cells=cn.shape[0], sizes=g["mesh_sizes"], cell_nodes=cn, origins=g["mesh_origins"],
        n_nodes=int(g["mesh_n_nodes"]), prolongation=csr_from(g, "mesh_P"),
        domain=SimpleNamespace(L=float(g["mesh_L"])))


def ref_from(g):
    return SimpleNamespace(Nq=9, B=g["ref_B"], dB=g["ref_dB"], qpts=g["ref_qpts"],
                           qwts=g["ref_qwts"])


def data_from(g, suffix=""):
    from paper_1702_08880_b200 import QuadPointData

    r = g["r" + suffix]
    return QuadPointData(N=r.shape[0], r=r, z=g["z" + suffix], w=g["w" + suffix],
                         f=g["f" + suffix], df_r=g["df_r" + suffix], df_z=g["df_z" + suffix])


def params_from(g, nu="nu_hat", mro="mass_ratio_o"):
    from paper_1702_08880_b200 import CollisionParams

    return CollisionParams(nu_hat=g[nu], mass_ratio_o=g[mro])


def scaled(x, ref) -> float:
    ref = np.asarray(ref)
    s = np.abs(ref).max()
    return float(np.abs(np.asarray(x) - ref).max() / (s if s > 0 else 1.0))


def worst_component(K, D, Kref, Dref) -> float:
    """Worst per-species, per-component max|dX|/max|X_ref|."""
    worst = 0.0
    for a in range(Kref.shape[1]):
        for c in range(2):
            worst = max(worst, scaled(K[:, a, c], Kref[:, a, c]))
        for c, d in ((0, 0), (0, 1), (1, 1)):
            worst = max(worst, scaled(D[:, a, c, d], Dref[:, a, c, d]))
    return worst


def cuda_ok() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:  # pragma: no cover
        return False


@pytest.fixture(scope="session")
def oracle():
    from oracle import oracle as O

    O.build()
    return O


@pytest.fixture(scope="session")
def gpu():
    """Skip cleanly without a device; on a GPU box a missing library is a
    failure (no silent fallback)."""
    if not cuda_ok():
        pytest.skip("no CUDA device")
    import paper_1702_08880_b200 as pkg
    from paper_1702_08880_b200 import _lib

    lib = _lib.load()
    assert lib.lb_device_count() >= 1
    return pkg
