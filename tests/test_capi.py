"""The C-ABI library loads and exports every symbol include/*.h declares;
without a GPU the product path fails loudly (no CPU fallback).  CPU only."""

import re

import numpy as np
import pytest

from conftest import ROOT, cuda_ok


def declared_symbols():
    syms = set()
    for h in (ROOT / "include").glob("*.h"):
        text = re.sub(r"/\*.*?\*/", "", h.read_text(), flags=re.S)
        syms |= set(re.findall(r"\b(lb_[a-z0-9_]+)\s*\(", text))
    return syms


def test_library_built_and_exports_header():
    from paper_1702_08880_b200 import _lib

    lib = _lib.load()
    syms = declared_symbols()
    assert len(syms) >= 15
    for s in sorted(syms):
        assert hasattr(lib, s), s
    # and the Python binding types every declared symbol
    assert syms == set(_lib.SIGNATURES)


def test_pure_queries():
    from paper_1702_08880_b200 import _lib

    lib = _lib.load()
    assert lib.lb_version() == 100
    # even, >= 4 + 3S, half odd (conflict-free lane-varying 16-byte loads)
    for S, rs in ((1, 10), (2, 10), (3, 14), (4, 18), (5, 22), (8, 30)):
        assert lib.lb_record_stride(S, None, None) == rs
    assert lib.lb_record_stride(0, None, None) == -1 and lib.lb_record_stride(9, None, None) == -1
    # rank-one coupling (the reference's own collision_params): species collapse
    import paper_1702_08880_b200 as pkg
    from paper_1702_08880_b200 import _lib as L

    e = np.array([-1.0, 1.0, 6.0, 10.0])
    nu = np.outer(e**2, e**2)
    p4 = pkg.CollisionParams(nu_hat=nu / nu[0, 0], mass_ratio_o=1.0 / np.array([1, 3670, 21900, 335000.0]))
    coK, coD = pkg.coupling(p4)
    assert lib.lb_record_stride(4, L.dptr(coK), L.dptr(coD)) == 10
    assert lib.lb_sym_supported(4, L.dptr(coK), L.dptr(coD)) == 1
    # a coupling that is not rank one keeps the per-species layout
    nu2 = nu.copy()
    nu2[0, 1] *= 1.5
    coK2, coD2 = pkg.coupling(pkg.CollisionParams(nu_hat=nu2, mass_ratio_o=np.ones(4)))
    assert lib.lb_record_stride(4, L.dptr(coK2), L.dptr(coD2)) == 18
    assert lib.lb_sym_supported(4, L.dptr(coK2), L.dptr(coD2)) == 0
    # inner chunking is a function of n only, whole 128-point tiles, <= 64 chunks
    for n in (1, 72, 1152, 4096, 65536, 1 << 20):
        jc = lib.lb_chunk_len(n)
        assert jc % 128 == 0 and -(-n // jc) <= 64


def test_symbols_listed_in_sass():
    """The built .so carries sm_100a SASS (not just PTX)."""
    so = ROOT / "paper_1702_08880_b200" / "liblandau_b200.so"
    data = so.read_bytes()
    assert b"sm_100a" in data or b"sm_100" in data


@pytest.mark.skipif(cuda_ok(), reason="checks the no-GPU behaviour")
def test_no_device_fails_loudly():
    import paper_1702_08880_b200 as pkg
    from paper_1702_08880_b200 import _lib

    assert _lib.load().lb_device_count() == 0
    with pytest.raises(RuntimeError, match="no CUDA device"):
        _lib.Context(0)
    data = pkg.QuadPointData(N=3, r=np.ones(3), z=np.arange(3.0), w=np.ones(3),
                             f=np.ones((1, 3)), df_r=np.ones((1, 3)), df_z=np.ones((1, 3)))
    params = pkg.CollisionParams(nu_hat=np.ones((1, 1)), mass_ratio_o=np.ones(1))
    with pytest.raises(RuntimeError):
        pkg.fused_sweep(data.r, data.z, data, params)


def test_argument_errors_precede_device():
    import paper_1702_08880_b200 as pkg

    data = pkg.QuadPointData(N=3, r=np.ones(3), z=np.arange(3.0), w=np.ones(3),
                             f=np.ones((1, 3)), df_r=np.ones((1, 3)), df_z=np.ones((1, 3)))
    params2 = pkg.CollisionParams(nu_hat=np.ones((2, 2)), mass_ratio_o=np.ones(2))
    with pytest.raises(ValueError, match="species count mismatch"):
        pkg.fused_sweep(data.r, data.z, data, params2)
    with pytest.raises(ValueError):
        pkg.CollisionParams(nu_hat=np.ones((2, 3)), mass_ratio_o=np.ones(2))
    with pytest.raises(ValueError):
        pkg.CollisionParams(nu_hat=-np.ones((1, 1)), mass_ratio_o=np.ones(1))
    with pytest.raises(ValueError):
        pkg.axisym_tensor_pair(-0.1, 0.0, 0.5, 0.0)
    with pytest.raises(ValueError):
        pkg.axisym_tensor_pair(0.5, 0.1, 0.5, 0.1)
