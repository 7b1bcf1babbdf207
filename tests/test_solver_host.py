"""Host logic of the device Crank-Nicolson solver (paper_1702_08880_b200.
solver, landau_b200.cu cn_plan/cn_factor/cn_solve): the banded ordering, the
pattern mapping of M and C, and a numpy restatement of the block cyclic
reduction checked against SuperLU on the reference's own operators."""

import numpy as np
import pytest
import scipy.linalg as sla
import scipy.sparse as sp
import scipy.sparse.linalg as spla

from conftest import blocks_from, csr_from, golden
from paper_1702_08880_b200.solver import band_order, pattern_values


def _pattern(g):
    M = csr_from(g, "M")
    C = blocks_from(g, "C")[0]
    P = (abs(M) + abs(C)).tocsr()
    P.sort_indices()
    return M, C, P


def test_band_order_is_a_permutation_with_its_bandwidth():
    for case in ("cfg1", "cfg3"):
        _, _, P = _pattern(golden(case))
        n = P.shape[0]
        perm, bw = band_order(P.indptr, P.indices, n)
        assert np.array_equal(np.sort(perm), np.arange(n))
        inv = np.empty(n, dtype=np.int64)
        inv[perm] = np.arange(n)
        Q = P.tocoo()
        assert np.abs(inv[Q.row] - inv[Q.col]).max() == bw
        # natural order is a candidate, so the chosen bandwidth never exceeds it
        assert bw <= np.abs(Q.row - Q.col).max()


def test_pattern_values_maps_and_rejects():
    g = golden("cfg3")
    M, C, P = _pattern(g)
    n = P.shape[0]
    vals = pattern_values(M, P.indptr, P.indices, n)
    back = sp.csr_matrix((vals, P.indices, P.indptr), shape=(n, n))
    assert abs(back - M).max() == 0.0
    # an entry outside the pattern is an error (ValueError, like the reference's shape checks)
    bad = M.tolil()
    i, j = 0, n - 1
    assert P[i, j] == 0
    bad[i, j] = 1.0
    try:
        pattern_values(bad.tocsr(), P.indptr, P.indices, n)
    except ValueError:
        pass
    else:
        raise AssertionError("entry outside the pattern was accepted")


def block_cyclic_solve(A, b, perm, nb):
    """numpy restatement of the device solver: permute, cut into nb blocks
    (block tridiagonal since nb >= bandwidth), block cyclic reduction with
    LU (partial pivoting) of the eliminated rows' diagonal blocks."""
    n = A.shape[0]
    N = -(-n // nb)
    npad = N * nb
    Ap = np.zeros((npad, npad))
    Ap[:n, :n] = A.toarray()[np.ix_(perm, perm)]
    Ap[np.arange(n, npad), np.arange(n, npad)] = 1.0
    bp = np.zeros(npad)
    bp[:n] = b[perm]
    blk = lambda i, j: Ap[i * nb:(i + 1) * nb, j * nb:(j + 1) * nb].copy()  # noqa: E731
    D = [blk(i, i) for i in range(N)]
    L = [[blk(i, i - 1) if i else None for i in range(N)]]
    U = [[blk(i, i + 1) if i + 1 < N else None for i in range(N)]]
    v = [bp[i * nb:(i + 1) * nb].copy() for i in range(N)]
    rows = [list(range(N))]
    lus = []
    while len(rows[-1]) > 1:
        r, l = rows[-1], len(rows) - 1
        Nl = len(r)
        lu = {}
        for k in range(1, Nl, 2):
            lu[k] = sla.lu_factor(D[r[k]])
            L[l][k] = sla.lu_solve(lu[k], L[l][k])
            if k + 1 < Nl:
                U[l][k] = sla.lu_solve(lu[k], U[l][k])
        Ln, Un = [None] * ((Nl + 1) // 2), [None] * ((Nl + 1) // 2)
        for k in range(0, Nl, 2):
            if k >= 2:
                D[r[k]] -= L[l][k] @ U[l][k - 1]
                Ln[k // 2] = -L[l][k] @ L[l][k - 1]
            if k + 1 < Nl:
                D[r[k]] -= U[l][k] @ L[l][k + 1]
            if k + 2 < Nl:
                Un[k // 2] = -U[l][k] @ U[l][k + 1]
        lus.append(lu)
        L.append(Ln)
        U.append(Un)
        rows.append(r[::2])
    # forward
    for l, r in enumerate(rows[:-1]):
        Nl = len(r)
        for k in range(1, Nl, 2):
            v[r[k]] = sla.lu_solve(lus[l][k], v[r[k]])
        for k in range(0, Nl, 2):
            if k >= 2:
                v[r[k]] -= L[l][k] @ v[r[k - 1]]
            if k + 1 < Nl:
                v[r[k]] -= U[l][k] @ v[r[k + 1]]
    v[0] = np.linalg.solve(D[0], v[0])
    # backward
    for l in range(len(rows) - 2, -1, -1):
        r = rows[l]
        Nl = len(r)
        for k in range(1, Nl, 2):
            v[r[k]] -= L[l][k] @ v[r[k - 1]]
            if k + 1 < Nl:
                v[r[k]] -= U[l][k] @ v[r[k + 1]]
    x = np.empty(n)
    x[perm] = np.concatenate(v)[:n]
    return x


def test_block_cyclic_reduction_matches_splu():
    """The device algorithm (as numpy) solves the reference's CN systems
    (M - dt/2 C) to SuperLU's answer on cfg1 and the refined cfg3 mesh."""
    for case in ("cfg1", "cfg3"):
        g = golden(case)
        M, C, P = _pattern(g)
        n = P.shape[0]
        perm, bw = band_order(P.indptr, P.indices, n)
        dt = float(g["dt"])
        A = (M - 0.5 * dt * C).tocsr()
        b = (M + 0.5 * dt * C) @ g["coeffs"][0]
        want = spla.splu(A.tocsc()).solve(b)
        got = block_cyclic_solve(A, b, perm, max(bw, 1))
        assert np.abs(got - want).max() <= 1e-12 * np.abs(want).max(), case


@pytest.mark.parametrize("case", ["cfg3", "cfg1adv", "cfg3adv"])
def test_mass_matrix_bitwise_reference(case):
    """solver.mass_matrix (the M=None default of newton_step) is the
    reference's fem.mass_matrix bitwise (fem.py:150-165), hanging nodes
    included, so newton_step(M=None) == newton_step(M=mass_matrix(...))."""
    from conftest import csr_from, golden, mesh_from, ref_from
    from paper_1702_08880_b200.solver import mass_matrix

    g = golden(case)
    M = mass_matrix(mesh_from(g), ref_from(g))
    Mr = csr_from(g, "M")
    M.sort_indices()
    assert np.array_equal(M.indptr, Mr.indptr) and np.array_equal(M.indices, Mr.indices)
    assert np.array_equal(M.data, Mr.data)
