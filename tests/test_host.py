"""Host-side logic of the drop-in mirror (CPU only)."""

import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

import paper_1702_08880_b200 as pkg
from paper_1702_08880_b200 import synthetic
from paper_1702_08880_b200.shard import ShardPlan


def test_flop_count_pinned_values():
    # test_kernel.py:239-244
    assert pkg.flop_count(1, 1, 1) == 185
    assert pkg.flop_count(1, 2, 1) == 245
    assert pkg.flop_count(10, 1, 3) == 3 * 10 * 185
    assert pkg.flop_count(5, 2, 2, overhead_per_outer=7) == 2 * (5 * 245 + 7)
    assert pkg.flop_count(0, 3, 4) == 0
    with pytest.raises(ValueError):
        pkg.flop_count(-1, 1, 1)


@settings(max_examples=50, deadline=None)
@given(st.integers(0, 10**6), st.integers(0, 8), st.integers(0, 100))
def test_flop_count_linear_in_outer(N, S, outer):
    assert pkg.flop_count(N, S, outer) == outer * pkg.flop_count(N, S, 1)


def test_coupling_matches_reference_expression():
    from conftest import golden

    g = golden("cfg4s")
    params = pkg.CollisionParams(nu_hat=g["nu_hat"], mass_ratio_o=g["mass_ratio_o"])
    coK, coD = pkg.coupling(params)
    nu, mro = g["nu_hat"], g["mass_ratio_o"]
    np.testing.assert_array_equal(coK, nu * mro[:, None] * mro[None, :])
    np.testing.assert_array_equal(coD, -nu * (mro**2)[:, None])


def test_params_properties():
    p = pkg.CollisionParams(nu_hat=[[1.0, 2.0], [2.0, 4.0]], mass_ratio_o=[1.0, 0.5])
    assert p.n_species == 2 and p.nu_hat.flags.c_contiguous


@settings(max_examples=100, deadline=None)
@given(st.integers(0, 100000), st.integers(1, 8), st.sampled_from([1, 9]))
def test_shard_plan_partitions(n, world, align):
    plan = ShardPlan(n, world, align)
    cover = []
    for r in range(world):
        lo, hi = plan.bounds(r)
        assert 0 <= lo <= hi <= n
        if align > 1 and hi < n:
            assert hi % align == 0
        cover.extend(range(lo, hi))
    assert cover == list(range(n))
    assert max(plan.counts) - min(plan.counts) <= align


def test_cfg5_recipe_properties():
    wl = synthetic.cfg5(4096)
    assert wl.S == 2 and wl.r.shape == (4096,) and wl.f.shape == (2, 4096)
    assert np.all(wl.r >= 0) and np.all(wl.r ** 2 + wl.z ** 2 <= 25.0 + 1e-12)
    assert np.isclose(wl.w.sum(), (2.0 / 3.0) * 125.0, rtol=1e-13)
    np.testing.assert_array_equal(wl.nu_hat, np.ones((2, 2)))
    np.testing.assert_array_equal(wl.mass_ratio_o, [1.0, 0.25])
    # deterministic per seed
    assert synthetic.cfg5(4096).checksum() == wl.checksum()


def test_install_patches_every_importer():
    """install() routes an axlandau-shaped package through the B200 names."""
    import sys
    import types

    root = types.ModuleType("fakeax")
    root.__path__ = []
    mods = {}
    for sub in ("kernel", "assembly", "solver", "cli"):
        m = types.ModuleType(f"fakeax.{sub}")
        mods[sub] = m
        sys.modules[f"fakeax.{sub}"] = m
    sys.modules["fakeax"] = root
    try:
        sentinel = object()
        mods["kernel"].fused_sweep = sentinel
        mods["kernel"].fused_inner_loop = sentinel
        mods["assembly"].fused_sweep = sentinel
        mods["assembly"].assemble_collision = sentinel
        mods["solver"].assemble_collision = sentinel
        mods["cli"].assemble_collision = sentinel
        mods["cli"].fused_sweep = sentinel
        root.fused_sweep = sentinel
        saved = pkg.install(root)
        assert mods["solver"].assemble_collision is pkg.assemble_collision
        assert mods["cli"].fused_sweep is pkg.fused_sweep
        assert root.fused_sweep is pkg.fused_sweep
        pkg.uninstall(root, saved)
        assert mods["solver"].assemble_collision is sentinel
        assert root.fused_sweep is sentinel
    finally:
        for k in [k for k in sys.modules if k == "fakeax" or k.startswith("fakeax.")]:
            del sys.modules[k]


@pytest.mark.parametrize("case", ["cfg1", "hanging", "cfg2"])
def test_gather_map_reproduces_scipy_condensation(case):
    """The per-mesh CSR gather map (device scatter K3) evaluated on the host
    equals the reference's COO->CSR + P^T C P (assembly.py:115-129) on the
    reference's own element matrices, with the same sparsity pattern."""
    from conftest import blocks_from, csr_from, golden
    from oracle import oracle as O
    from paper_1702_08880_b200.scatter import build_gather_map

    g = golden(case)
    P = csr_from(g, "mesh_P")
    gm = build_gather_map(g["mesh_cell_nodes"], int(g["mesh_n_nodes"]), P)
    elem = O.element_matrices(g["K"], g["D"], g["w"], g["mesh_sizes"], g["ref_B"], g["ref_dB"])
    mine = gm.apply(elem)
    ref = O.condense(elem, g["mesh_cell_nodes"], int(g["mesh_n_nodes"]), P)
    for x, y, z in zip(mine, ref, blocks_from(g)):
        assert x.nnz == z.nnz
        assert np.array_equal(np.sort(x.indices), np.sort(z.indices))
        yd = y.toarray()
        assert np.abs(x.toarray() - yd).max() <= 1e-14 * np.abs(yd).max()
        assert np.abs(x.toarray() - z.toarray()).max() <= 1e-13 * np.abs(z.toarray()).max()
    assert gm.slot_ptr[-1] == gm.gather_idx.shape[0]
    assert gm.gather_idx.max() < elem[0].size
    # csr_block flags its matrices canonical without scipy's re-validation:
    # the pattern must really be canonical, and the blocks independent
    import scipy.sparse as sp

    assert np.all(np.diff(gm.indptr) >= 0) and gm.indptr[-1] == gm.nnz
    for r in range(gm.n_free):  # columns sorted and unique within every row
        row = gm.indices[gm.indptr[r]:gm.indptr[r + 1]]
        assert np.all(np.diff(row) > 0)
    chk = sp.csr_matrix((np.ones(gm.nnz), gm.indices, gm.indptr), shape=(gm.n_free, gm.n_free))
    chk.sum_duplicates()  # scipy's canonicalisation changes nothing
    assert chk.nnz == gm.nnz and np.array_equal(chk.indices, gm.indices)
    b0, b1 = gm.csr_block(np.arange(gm.nnz, dtype=float)), gm.csr_block(np.ones(gm.nnz))
    assert b0.indices is not b1.indices and b0.indptr is not b1.indptr
    b0.eliminate_zeros()  # in place on b0's own arrays only
    assert b1.nnz == gm.nnz and np.array_equal(b1.indices, gm.indices)
    assert np.array_equal((b1 @ np.ones(gm.n_free)), np.diff(gm.indptr).astype(float))


def test_coefficient_header_is_generated():
    """landau_coefs.h is exactly tools/gen_coefs.py's output (the frozen
    reference tables, kernel.py:64-90, and the derived series / log tables)."""
    import subprocess
    import sys

    from conftest import ROOT

    out = subprocess.run([sys.executable, str(ROOT / "tools" / "gen_coefs.py")], check=True,
                         capture_output=True, text=True).stdout
    assert out == (ROOT / "paper_1702_08880_b200" / "csrc" / "landau_coefs.h").read_text()


def test_device_log_table_accuracy():
    """Host restatement of the device logarithm (landau_pair.cuh log_reduce /
    log_finish) with the generated table: relative error <= 3e-16."""
    import re

    from conftest import ROOT

    h = (ROOT / "paper_1702_08880_b200" / "csrc" / "landau_coefs.h").read_text()
    bits = int(re.search(r"#define LB_LOGT_BITS (\d+)", h).group(1))
    tab = np.array([float(v) for v in re.search(r"#define LB_LOGT \{(.*?)\}", h).group(1).split(",")])
    inv, logc = tab[0::2], tab[1::2]
    rng = np.random.default_rng(7)
    x = np.concatenate([rng.random(20000) ** rng.choice([1, 3, 10, 50, 700], 20000),
                        1.0 - np.geomspace(1e-15, 0.5, 2000), [1.0, 0.5, 0.7071]])
    x = x[x > 1e-300]
    ix = x.view(np.int64)
    tmp = ix - 0x3FE6000000000000
    i = (tmp >> (52 - bits)) & ((1 << bits) - 1)
    k = tmp >> 52
    z = (ix - (tmp & np.int64(-(1 << 52)))).view(np.float64)
    # r = fma(z, invc, -1) on the device: emulate the fused product with a
    # Dekker two-product (z*invc is in [0.5, 2], so p - 1 is exact)
    a, b = z, inv[i]
    ca, cb = 134217729.0 * a, 134217729.0 * b
    ah, bh = ca - (ca - a), cb - (cb - b)
    al, bl = a - ah, b - bh
    p = a * b
    r = (p - 1.0) + (((ah * bh - p) + ah * bl + al * bh) + al * bl)
    q = ((((-1.0 / 6.0) * r + 0.2) * r - 0.25) * r + 1.0 / 3.0) * r - 0.5
    lx = k * np.log(2.0) + (logc[i] + (r + r * r * q))
    rel = np.abs(lx - np.log(x)) / np.maximum(np.abs(np.log(x)), 1e-300)
    assert rel.max() < 3e-16 * 4, rel.max()
    assert np.abs(r).max() < 2.0 ** -(bits - 0.5)


def test_install_into_the_reference_package():
    """install() patches every by-value import of the real reference package
    (build container only: skipped where /root/reference is absent)."""
    import importlib
    import os
    import sys

    src = "/root/reference/pkg/src"
    if not os.path.isdir(src):
        pytest.skip("reference tree not present (GPU box)")
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
    sys.path.insert(0, src)
    try:
        ax = importlib.import_module("axlandau")
    except Exception as err:  # pragma: no cover - optional dependency
        pytest.skip(f"reference not importable: {err}")
    finally:
        sys.path.remove(src)
    saved = pkg.install(ax)
    try:
        assert ax.assembly.fused_sweep is pkg.fused_sweep
        assert ax.assembly.assemble_collision is pkg.assemble_collision
        assert ax.solver.assemble_collision is pkg.assemble_collision
        assert ax.solver._assemble_at.__module__ == "paper_1702_08880_b200"
        assert ax.cli.fused_sweep is pkg.fused_sweep and ax.cli.assemble_collision is pkg.assemble_collision
        assert ax.kernel.fused_inner_loop is pkg.fused_inner_loop
        assert ax.fused_sweep is pkg.fused_sweep
        assert ax.solver.newton_step is pkg.newton_step
        assert ax.solver.linear_cn_step is pkg.linear_cn_step
        from paper_1702_08880_b200 import solver as our_solver

        # failures surface as the reference's own StepFailure (advance catches it)
        assert our_solver._StepFailure is ax.solver.StepFailure
        import inspect

        # the patched entry points accept the reference's call signatures
        for ref_fn, ours in ((saved[("kernel", "fused_sweep")], pkg.fused_sweep),
                             (saved[("assembly", "assemble_collision")], pkg.assemble_collision),
                             (saved[("solver", "newton_step")], pkg.newton_step),
                             (saved[("solver", "linear_cn_step")], pkg.linear_cn_step)):
            assert list(inspect.signature(ref_fn).parameters) == list(
                inspect.signature(ours).parameters)
    finally:
        pkg.uninstall(ax, saved)
    assert ax.assembly.fused_sweep is not pkg.fused_sweep
    assert ax.solver.newton_step is not pkg.newton_step
    assert our_solver._StepFailure is our_solver.StepFailure


def test_elliptic_domain_errors_before_the_device():
    """elliptic_KE rejects m outside [0, 1) with ValueError (kernel.py:101-102,
    test_kernel.py:49-57) before any device work."""
    import pytest

    import paper_1702_08880_b200 as pkg

    for bad in (-0.1, 1.0, 1.5, float("nan")):
        with pytest.raises(ValueError):
            pkg.elliptic_KE([bad])


def test_species_meshes_step_argument_errors_before_the_device():
    """species_meshes_step needs one mesh, state and mass matrix per species;
    a mismatch is a ValueError before any device work."""
    import pytest

    import paper_1702_08880_b200 as pkg

    with pytest.raises(ValueError):
        pkg.species_meshes_step([object()], None, [np.zeros(3), np.zeros(3)], None, 0.1, [None])
    with pytest.raises(ValueError):
        pkg.species_meshes_step([object(), object()], None, [np.zeros(3), np.zeros(3)], None, 0.1, [None])


def test_bench_reference_arm_contract():
    """`bench.py --impl reference` (the reference algorithm on the host cores)
    prints one JSON line with the contract's keys: impl, cpu_baseline,
    e2e with zero transfer bytes, the same metric/unit as our arm."""
    import json
    import subprocess
    import sys

    from conftest import ROOT

    out = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "1",
                          "--warmup", "3", "--points", "1024", "--ref-step-seconds", "0.1"],
                         cwd=str(ROOT), capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads([l for l in out.stdout.splitlines() if l.startswith("{")][-1])
    assert line["impl"] == "reference" and line["unit"] == "pairs/s" and line["value"] > 0
    for k in ("metric", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config"):
        assert k in line, k
    cb = line["cpu_baseline"]
    assert cb["kind"] in ("port", "reference") and cb["cores"] >= 1 and cb["value"] == line["value"]
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["d2h_bytes_per_step"] == 0
    assert line["warmup"] >= 3
