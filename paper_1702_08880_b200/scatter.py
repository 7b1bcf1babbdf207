"""Per-mesh gather map for the device CSR scatter + hanging-node condensation.

The reference assembles each species block as

    C_free = P^T (sum_e scatter(E_e)) P            (assembly.py:115-129)

with scipy: a COO->CSR conversion that sums duplicate (row, col) entries of
the 81 element-matrix entries of every cell, then two sparse products with
the prolongation P (identity rows for free nodes, three interpolation
weights for hanging nodes, mesh.py:233-241).  Entry (p, q) of C_free is a
weighted sum of element entries:

    C_free[p, q] = sum over cells e, local (i, j) with P[n_ei, p] != 0 and
                   P[n_ej, q] != 0 of  P[n_ei, p] * P[n_ej, q] * E[e, i, j]

This module precomputes, once per mesh, the CSR pattern of C_free and for
every stored slot the list of (element-entry index, weight) pairs in a fixed
order, so the device can produce the CSR values with one gather-sum thread
per slot (`lb_assemble_csr`): no atomics, deterministic.  The pattern is
species-independent (every block has plain Q2 connectivity, assembly.py:66-70).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp


@dataclass(frozen=True)
class GatherMap:
    n_free: int
    indptr: np.ndarray      # (n_free + 1,) int64, CSR row pointers of C_free
    indices: np.ndarray     # (nnz,) int32, CSR column indices (sorted per row)
    slot_ptr: np.ndarray    # (nnz + 1,) int32, per-slot range into gather_*
    gather_idx: np.ndarray  # (ncontrib,) int32, element-entry index (e*9 + i)*9 + j
    gather_w: np.ndarray    # (ncontrib,) float64, P[n_ei, p] * P[n_ej, q]

    @property
    def nnz(self) -> int:
        return int(self.indices.shape[0])

    def csr_block(self, vals: np.ndarray) -> sp.csr_matrix:
        """A scipy CSR block with this pattern and values `vals` (nnz,).
        The pattern is canonical (rows sorted, no duplicates), so the matrix
        is put together directly -- scipy's constructor re-validates and
        re-types the index arrays (~1.2 ms per block at config 4's 525,825
        entries, 4 blocks per operator call); each block gets its own copy
        of the index arrays, as a freshly assembled matrix would."""
        ind = self.indices
        ptr = self.indptr
        idx_t = np.int32 if max(int(ptr[-1]), self.n_free) < 2**31 - 1 else np.int64
        m = sp.csr_matrix((self.n_free, self.n_free), dtype=np.float64)
        m.data = np.ascontiguousarray(vals, dtype=np.float64)
        m.indices = ind.astype(idx_t, copy=True)
        m.indptr = ptr.astype(idx_t, copy=True)
        m.has_sorted_indices = True
        m.has_canonical_format = True
        return m

    def apply(self, elem: np.ndarray) -> list:
        """Host (numpy) evaluation of the map: elem (S, ncell, 9, 9) -> S CSR
        blocks.  Used by the CPU tests to check the map itself."""
        S = elem.shape[0]
        flat = elem.reshape(S, -1)
        seg = np.repeat(np.arange(self.nnz), np.diff(self.slot_ptr))
        out = []
        for a in range(S):
            vals = np.zeros(self.nnz)
            np.add.at(vals, seg, flat[a, self.gather_idx] * self.gather_w)
            out.append(self.csr_block(vals))
        return out


def build_gather_map(cell_nodes, n_nodes: int, prolongation) -> GatherMap:
    """Gather map for a mesh (cell_nodes (ncell, 9), prolongation (n_nodes,
    n_free) CSR).  Rows = test functions i, columns = trial functions j, as
    `_scatter_indices` (assembly.py:115-118)."""
    cn = np.asarray(cell_nodes, dtype=np.int64)
    ncell = cn.shape[0]
    P = sp.csr_matrix(prolongation)
    P.sum_duplicates()
    n_free = P.shape[1]
    # element entry t = (e*9 + i)*9 + j  ->  (row node, col node)
    t = np.arange(ncell * 81, dtype=np.int64)
    rn = np.repeat(cn, 9, axis=1).ravel()
    cl = np.tile(cn, (1, 9)).ravel()
    # expand each node through its prolongation row: (node) -> [(p, w)]
    cnt = np.diff(P.indptr)
    r_cnt, c_cnt = cnt[rn], cnt[cl]
    # contributions = sum over entries of r_cnt * c_cnt
    nrep = r_cnt * c_cnt
    te = np.repeat(t, nrep)
    # position inside the (r_cnt x c_cnt) product for each contribution
    start = np.repeat(np.cumsum(nrep) - nrep, nrep)
    k = np.arange(te.shape[0], dtype=np.int64) - start
    cc = np.repeat(c_cnt, nrep)
    kr, kc = k // cc, k % cc
    pr = P.indptr[rn[te]] + kr
    pc = P.indptr[cl[te]] + kc
    p = P.indices[pr].astype(np.int64)
    q = P.indices[pc].astype(np.int64)
    w = P.data[pr] * P.data[pc]
    keep = w != 0.0
    te, p, q, w = te[keep], p[keep], q[keep], w[keep]
    # slots: unique (p, q) in row-major order; contributions sorted by (slot, entry)
    key = p * n_free + q
    order = np.lexsort((te, key))
    key, te, w = key[order], te[order], w[order]
    uniq, first = np.unique(key, return_index=True)
    slot_ptr = np.append(first, key.shape[0]).astype(np.int32)
    rows = uniq // n_free
    cols = (uniq % n_free).astype(np.int32)
    indptr = np.zeros(n_free + 1, dtype=np.int64)
    np.add.at(indptr, rows + 1, 1)
    indptr = np.cumsum(indptr)
    if te.shape[0] >= 2**31 or ncell * 81 >= 2**31:
        raise ValueError("mesh too large for 32-bit gather indices")
    return GatherMap(n_free=n_free, indptr=indptr, indices=cols, slot_ptr=slot_ptr,
                     gather_idx=te.astype(np.int32), gather_w=np.ascontiguousarray(w))
