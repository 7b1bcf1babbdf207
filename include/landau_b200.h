/*
 * landau_b200.h -- C ABI of the B200-native Landau pair-integration path.
 *
 * This is the drop-in boundary for the hot path of the reference package
 * `axlandau` (arXiv 1702.08880): the O(N^2) FP64 pair integral that gives
 * every outer quadrature point its per-species friction vector K and
 * diffusion tensor D, and the per-element Jacobian contraction B^T[D,K]B.
 * Citations are `file:line` into the reference tree (pkg/src/axlandau/).
 *
 * Conventions
 *  - All arrays are float64, C order.  Host entry points (no `_dev` suffix)
 *    take caller-owned HOST pointers, copy in, run, copy out and block until
 *    the outputs are written (the reference's synchronous semantics).
 *    `_dev` entry points take DEVICE pointers and a cudaStream_t (passed as
 *    void*; NULL = the legacy default stream, as in the CUDA runtime) and
 *    are asynchronous with respect to the host.
 *  - Return value: LB_OK (0) or an LB_E* code; `lb_last_error()` returns a
 *    thread-local message for the most recent failure.  LB_EINVAL maps to
 *    Python ValueError, everything else to RuntimeError.  There is no CPU
 *    fallback: without a CUDA device every compute entry fails with
 *    LB_ENODEV.
 *  - Species count S: 1 <= S <= LB_MAX_SPECIES.
 *  - Output layouts match the reference exactly:
 *      K    (nout, S, 2)        friction  (kernel.py:520)
 *      D    (nout, S, 2, 2)     diffusion, D[..,0,1] == D[..,1,0] bitwise
 *                               (kernel.py:521, 437-440)
 *      elem (S, ncell, 9, 9)    element matrices, row = test i, col = trial j
 *                               (assembly.py:163-165)
 *  - Results are deterministic (bitwise run to run) and independent of how
 *    the outer points are split across calls / GPUs: the inner-point chunking
 *    depends only on n (the inner count) and every chunk is reduced in a
 *    fixed order.
 */
#ifndef LANDAU_B200_H
#define LANDAU_B200_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LB_OK 0
#define LB_EINVAL 1  /* bad argument: maps to ValueError */
#define LB_ECUDA 2   /* CUDA runtime / launch failure */
#define LB_ENODEV 3  /* no CUDA device visible */
#define LB_ENOMEM 4  /* device allocation failed */
#define LB_ESINGULAR 5 /* singular or non-finite linear solve: maps to solver.StepFailure */

#define LB_MAX_SPECIES 8

typedef struct lb_ctx lb_ctx;
typedef struct lb_mesh lb_mesh;
typedef struct lb_cn lb_cn;

/* ABI version (major*100 + minor). */
int lb_version(void);

/* Thread-local description of the last failure on this thread ("" if none). */
const char *lb_last_error(void);

/* Number of visible CUDA devices (0 when none); never fails. */
int lb_device_count(void);

/* One context per (host thread, device): owns a stream and grow-only device
 * scratch.  Replaces the numba thread pool of kernel.py:524-533. */
int lb_ctx_create(int device, lb_ctx **out);
int lb_ctx_destroy(lb_ctx *ctx);

/* Doubles per packed inner-point record for S species and the coupling
 * coK/coD (NULL: per-species layout): r, z, r^2, 1/r, then (w*df_r, w*df_z,
 * w*f) per species -- or, when coK and coD are rank one (always so for the
 * reference's collision_params, nu_ab ~ e_a^2 e_b^2, physics.py:77-94), the
 * species-collapsed triple (sum_b k_b w df_r, sum_b k_b w df_z,
 * sum_b be_b w f) -- padded to an even count. */
int lb_record_stride(int S, const double *coK, const double *coD);

/* Accumulator species sets the sweep keeps per point: 1 when coK/coD are
 * rank one (species collapse), else S (-1 for an invalid S). */
int lb_accumulator_sets(int S, const double *coK, const double *coD);

/* Inner-point chunk length the sweep uses for n inner points (a function of
 * n only; exposed so tests can check the decomposition). */
int lb_chunk_len(int n);

/* ---------------------------------------------------------------------
 * Kernel-level entry: replaces `fused_sweep` (kernel.py:504-536) and the
 * numba loops under it (_lanes 306-389, _accumulate_block 392-415,
 * _combine 418-440, _sweep_serial/_sweep_parallel 443-493).
 *   outer_r/outer_z (nout)            outer points (any points, nout != n ok)
 *   r, z, w (n); f, df_r, df_z (S, n)  QuadPointData fields (fem.py:133-149)
 *   coK, coD (S, S)                   coupling from _coupling (kernel.py:496-501)
 *   eps_d                             exclusion radius; pairs with
 *                                     d^2 < eps_d^2 or d^2 == 0 are skipped
 *   K_out (nout,S,2), D_out (nout,S,2,2)
 * --------------------------------------------------------------------- */
int lb_fused_sweep(lb_ctx *ctx, int nout, const double *outer_r, const double *outer_z,
                   int n, int S, const double *r, const double *z, const double *w,
                   const double *f, const double *df_r, const double *df_z,
                   const double *coK, const double *coD, double eps_d,
                   double *K_out, double *D_out);

/* Operator-level entry: replaces the kernel call plus the vectorized outer
 * point transform and 9x9 element contraction of `assemble_collision`
 * (assembly.py:148-165).  Points are the mesh's quadrature points in the
 * order n = 9*cell + q (fem.py:137-140), so n == 9*ncell.
 *   cell_sizes (ncell, 2)  (dr, dz) per cell (mesh.py VelocityMesh.sizes)
 *   B (9,9), dB (9,9,2)    reference basis tables (fem.py:66-81)
 *   K_out, D_out may be NULL (not copied back); elem_out (S, ncell, 9, 9).
 *   phase_ms (3) may be NULL; else device times (CUDA events) of
 *   [upload + pack, sweep + coupling, element contraction + download].
 * The CSR scatter + hanging-node condensation (assembly.py:168-169) stays
 * with the caller. */
int lb_assemble_elements(lb_ctx *ctx, int ncell, const double *cell_sizes, int S,
                         const double *r, const double *z, const double *w,
                         const double *f, const double *df_r, const double *df_z,
                         const double *coK, const double *coD, double eps_d,
                         const double *B, const double *dB,
                         double *K_out, double *D_out, double *elem_out, double *phase_ms);

/* All-points entry (outer set == inner set == the n points): the call
 * `assemble_collision` makes (assembly.py:148, fused_sweep(data.r, data.z,
 * data, ...)).  For S <= 2 it evaluates each unordered pair once (all
 * expensive terms are symmetric in i <-> j; only UD_xx differs for the
 * swapped pair) and feeds both points' accumulators; larger S uses the
 * general sweep.  K_out (n,S,2), D_out (n,S,2,2) in the input point order. */
int lb_fused_sweep_all(lb_ctx *ctx, int n, int S, const double *r, const double *z,
                       const double *w, const double *f, const double *df_r,
                       const double *df_z, const double *coK, const double *coD,
                       double eps_d, double *K_out, double *D_out);

/* Device-resident mesh for the operator path: cell sizes, the Q2 basis
 * tables and the gather map of the CSR scatter + hanging-node condensation
 * (assembly.py:115-129, mesh.py:233-241), built once per mesh on the host
 * (paper_1702_08880_b200/scatter.py): for each of the nslots stored entries
 * of C_free = P^T C P, slot_ptr[s]..slot_ptr[s+1] index (gather_idx,
 * gather_w) pairs = (element entry (e*9+i)*9+j, P[n_ei,p] * P[n_ej,q]). */
int lb_mesh_create(lb_ctx *ctx, int ncell, const double *cell_sizes, const double *B,
                   const double *dB, int nslots, const int *slot_ptr, int ncontrib,
                   const int *gather_idx, const double *gather_w, lb_mesh **out);
int lb_mesh_destroy(lb_mesh *mesh);

/* Whole operator on the device: replaces assembly.py:148-169 (kernel,
 * transform, contraction, scatter, condensation).  Writes the CSR values of
 * the S species blocks, csr_out (S, nslots), in the map's pattern; K_out /
 * D_out / phase_ms may be NULL (phase_ms as lb_assemble_elements, the last
 * phase also covering the scatter). */
int lb_assemble_csr(lb_ctx *ctx, const lb_mesh *mesh, int S, const double *r, const double *z,
                    const double *w, const double *f, const double *df_r, const double *df_z,
                    const double *coK, const double *coD, double eps_d, double *csr_out,
                    double *K_out, double *D_out, double *phase_ms);

/* Sampling geometry of a mesh (fem.py:84-113, mesh.py:54-106): cell
 * origins (ncell,2), reference quadrature points qpts (9,2) / weights qwts
 * (9), cell_nodes (ncell,9), and the prolongation P (n_nodes x n_free) as
 * CSR (P_ptr (n_nodes+1), P_idx, P_w). */
int lb_mesh_set_geometry(lb_mesh *mesh, const double *origins, const double *qpts,
                         const double *qwts, const int *cell_nodes, int n_nodes, int n_free,
                         const int *P_ptr, const int *P_idx, const double *P_w);

/* Device `sample_state` (fem.py:170-199) for cells [c0, c1): coeffs
 * (S, n_free) on the device -> r, z, w (9*(c1-c0)) and f, df_r, df_z
 * (S, 9*(c1-c0)), the QuadPointData layout of those cells' points (what
 * each rank feeds into the all-gather). */
int lb_sample_state_dev(lb_ctx *ctx, const lb_mesh *mesh, int S, int c0, int c1,
                        const double *coeffs, double *r, double *z, double *w, double *f,
                        double *df_r, double *df_z, void *stream);

/* Host-pointer `sample_state` (fem.py:170-199) for the whole mesh: coeffs
 * (S, n_free) host in, data_out ((3+3S) x 9*ncell host: r, z, w, f, df_r,
 * df_z) out -- bitwise the reference's (the kernel reproduces numpy's einsum
 * order). */
int lb_sample_state(lb_ctx *ctx, const lb_mesh *mesh, int S, const double *coeffs,
                    double *data_out);

/* State-level operator: replaces solver._assemble_at (solver.py:81-84) =
 * sample_state + assemble_collision.  Host coeffs (S, n_free) in, CSR
 * values csr_out (S, nslots) out; data_out ((3+3S) x 9*ncell: r, z, w, f,
 * df_r, df_z) and phase_ms may be NULL. */
int lb_assemble_state(lb_ctx *ctx, const lb_mesh *mesh, int S, const double *coeffs,
                      const double *coK, const double *coD, double eps_d, double *csr_out,
                      double *data_out, double *phase_ms);

/* Element contraction + CSR scatter/condensation from given accumulators:
 * w (9*ncell) outer weights, K (9*ncell,S,2), D (9*ncell,S,2,2) host arrays
 * of the mesh's points -> csr_out (S, nslots).  With per-species meshes the
 * accumulators come from one all-points sweep over the union of the
 * species' point sets; each species' block is assembled on
 * its own mesh (assembly.py:151-169). */
int lb_elements_csr(lb_ctx *ctx, const lb_mesh *mesh, int S, const double *w, const double *K,
                    const double *D, double *csr_out);

/* Multi-GPU operator piece: element contraction for this rank's cells
 * [c0, c1) (w, K, D device arrays of those cells' points) and the CSR
 * gather over ALL slots with the other cells' entries zero -> csr_out
 * (S, nslots) device partial values; summing them over ranks (all-reduce)
 * gives the operator (assembly.py:151-169). */
int lb_operator_partial_dev(lb_ctx *ctx, const lb_mesh *mesh, int S, int c0, int c1,
                            const double *w, const double *K, const double *D, double *csr_out,
                            void *stream);

/* Per-pair closed form on the device: replaces `axisym_tensor_pair`
 * (kernel.py:206-235) for npair independent (r, z, rbar, zbar) tuples, with
 * the same device arithmetic the sweep uses.  UK, UD: (npair, 2, 2).
 * Coincident pairs (d^2 == 0) return zeros (the sweep's mask). */
int lb_tensor_pairs(lb_ctx *ctx, int npair, const double *r, const double *z,
                    const double *rbar, const double *zbar, double *UK, double *UD);

/* ---------------------------------------------------------------------
 * Device-pointer pieces, used by the multi-GPU layer and the benchmark.
 * --------------------------------------------------------------------- */

/* Pack n inner points (SoA device arrays) into records of lb_record_stride(S)
 * doubles: the per-point field state that the sharded path all-gathers. */
int lb_pack_records_dev(lb_ctx *ctx, int n, int S, const double *r, const double *z,
                        const double *w, const double *f, const double *df_r,
                        const double *df_z, const double *coK, const double *coD,
                        double *rec, void *stream);

/* Pair sweep + species coupling over packed records (device pointers).
 * `n` is the total inner count (all shards), `rec` its packed records. */
int lb_sweep_dev(lb_ctx *ctx, int nout, const double *outer_r, const double *outer_z,
                 int n, int S, const double *rec, const double *coK, const double *coD,
                 double eps_d, double *K_out, double *D_out, void *stream);

/* Outer-point transform + element contraction from device K/D
 * (assembly.py:151-165).  w (9*ncell) outer weights, cell_sizes (ncell,2).
 * The 243 basis values B/dB become a by-value kernel parameter: this entry
 * reads them back from the device once (a synchronisation of `stream`);
 * the mesh entries (lb_mesh_create) keep a host copy instead. */
int lb_elements_dev(lb_ctx *ctx, int ncell, int S, const double *cell_sizes,
                    const double *w, const double *K, const double *D,
                    const double *B, const double *dB, double *elem_out, void *stream);

/* Symmetric all-points sweep in three device steps, for the multi-GPU
 * layer:
 *  1 lb_sym_prepare_dev  Morton-order the n packed records (all points, the
 *                        same on every rank) into the context;
 *  2 lb_sym_partial_dev  this rank's share of the unordered tile pairs: the
 *                        row groups [g0, g1) of lb_sym_groups(rank, world)
 *                        -> tot, (g1 - g0) group sums of [5S][lb_sym_npad(n)]
 *                        doubles each (sorted point order);
 *  3 lb_sym_combine_dev  K/D for original points [q0, q1) from all eight
 *                        group sums held in one buffer (world = 1, or after
 *                        an all-gather of every rank's group sums), or
 *    lb_sym_combine_groups_dev  the same from a HOST array of eight device
 *                        pointers, one per group in group order -- e.g.
 *                        peers' buffers mapped with lb_ipc_open, which makes
 *                        it the cross-rank reduction and the combine in one
 *                        kernel, reading only this rank's points.
 * The summation order is fixed by n alone: a point's total is the eight
 * group sums added in group order, each group summed by increasing row.  So
 * K and D are bitwise identical for every world size <= 8 (the reference
 * promises bitwise invariance to `workers`, kernel.py:508-511,
 * test_kernel.py:197-212).
 * lb_sym_supported(S, coK, coD) is 1 when this path implements the
 * coupling (any S with a rank-one coupling, else S <= 3).
 * lb_sym_groups returns the group count (8) and this rank's [g0, g1). */
int lb_sym_supported(int S, const double *coK, const double *coD);
int lb_sym_npad(int n);
int lb_sym_groups(int rank, int world, int *g0, int *g1);
int lb_sym_prepare_dev(lb_ctx *ctx, int n, int S, const double *coK, const double *coD,
                       const double *rec, void *stream);
int lb_sym_partial_dev(lb_ctx *ctx, int S, double eps_d, int rank, int world, double *tot,
                       void *stream);
int lb_sym_combine_dev(lb_ctx *ctx, int S, const double *tot, const double *coK,
                       const double *coD, int q0, int q1, double *K_out, double *D_out,
                       void *stream);
int lb_sym_combine_groups_dev(lb_ctx *ctx, int S, const double *const *group_ptrs,
                              const double *coK, const double *coD, int q0, int q1,
                              double *K_out, double *D_out, void *stream);

/* Execution counters of the species-collapsed symmetric sweep (the
 * benchmark's executed-FP64 count): out (3, may be NULL) receives the
 * counts since the last call -- off-diagonal thread-steps, diagonal
 * thread-steps, thread-steps that took the m < 0.01 series branch (each
 * thread-step evaluates 4 pairs: 2 outer points x 2 partners) -- then the
 * counters are zeroed and counting is switched on (enable != 0) or off.
 * Synchronises the device. */
int lb_sym_counters(lb_ctx *ctx, int enable, unsigned long long *out);

/* elliptic_KE (kernel.py:93-113): K(m), E(m) for n parameters in [0, 1)
 * (LB_EINVAL outside), with the device's table log and Horner chains. */
int lb_elliptic_ke(lb_ctx *ctx, int n, const double *m, double *K, double *E);

/* Peer memory for the symmetric multi-GPU path: every rank allocates its
 * group-sum buffer with lb_ipc_alloc (cudaMalloc + a 64-byte CUDA IPC
 * handle), the handles are exchanged out of band, and each rank maps its
 * peers' buffers with lb_ipc_open (peer access over NVLink); the mapped
 * pointers feed lb_sym_combine_groups_dev.  The caller orders the combine
 * after every rank's lb_sym_partial_dev and before any rank's next one
 * (e.g. a stream-ordered barrier). */
int lb_ipc_alloc(lb_ctx *ctx, size_t bytes, void **dptr, unsigned char *handle);
int lb_ipc_open(lb_ctx *ctx, const unsigned char *handle, void **dptr);
int lb_ipc_close(lb_ctx *ctx, void *dptr);
int lb_ipc_free(lb_ctx *ctx, void *dptr);

/* Number of kernels the most recent lb_sweep_dev / lb_elements_dev /
 * lb_pack_records_dev call launched (for the benchmark's launch count). */
int lb_last_launch_count(lb_ctx *ctx);

/* FP64 DFMA throughput microbenchmark on the context's device: a grid of
 * independent DFMA chains sized to fill every SM, timed with CUDA events.
 * Writes achieved TFLOP/s (2 flops per DFMA) and the kernel time in ms. */
int lb_fp64_peak(lb_ctx *ctx, double *tflops, double *ms);

/* ---- Crank-Nicolson time step on the device (solver.py:103-150) ----------
 * The reference solves (M - dt/2 C_a) delta = -R per species with SuperLU
 * (solver.py:124-133, splu).  Here the free nodes are permuted into a banded
 * order (perm[p] = free node at band position p, natural or reverse
 * Cuthill-McKee), cut into blocks of nb rows (nb >= the permuted bandwidth),
 * and the block-tridiagonal systems of all species are factorised together
 * on the device (block LU, partial pivoting inside diagonal blocks).
 *
 * lb_cn_create     solver with S species for an n x n CSR pattern indptr (n+1)
 *                  / indices (nnz); with a mesh, n = n_free and the pattern is
 *                  the mesh's (the order of lb_assemble_csr's values); mesh
 *                  NULL gives a linear-solve-only instance (lb_cn_linear_step).
 *                  perm (n), nb the block size; LB_EINVAL if nb is below the
 *                  permuted bandwidth.
 * lb_cn_set_mass   mass-matrix values in that pattern (host; fem.py:152-167
 *                  mass_matrix mapped onto the pattern), or NULL to assemble
 *                  M on the device from the mesh geometry.
 * lb_cn_get_mass   download the current mass values (nslots).
 * lb_cn_newton     newton_step (solver.py:103-134): assemble C at f_guess on
 *                  the device; C_old per c_old_mode: 0 = assemble at f_old,
 *                  1 = upload the caller's C_old, 2 = keep the device copy
 *                  of the previous call (advance() passes one C_old to every
 *                  iteration of a step, solver.py:171-181); residual
 *                  R = M(g - f) - dt/2 (C_g g + C_old f), solve, f_next =
 *                  f_guess + delta; rnorm = ||R|| / ||M f_old^T||.  States
 *                  are (S, n_free) host arrays, C_old / C_guess_out (S,
 *                  nslots).  LB_ESINGULAR: zero pivot or non-finite update.
 *                  phase_ms (4, optional): assembly, residual+fill, factor,
 *                  solve+download.
 * lb_cn_linear_step linear_cn_step (solver.py:137-150): (M - dt/2 C) f+ =
 *                  (M + dt/2 C) f with C (S, nslots) held fixed.
 * lb_cn_theta_step the theta method with C held fixed: (M - theta dt C) f+ =
 *                  (M + (1 - theta) dt C) f; theta = 1/2 is lb_cn_linear_step,
 *                  theta = 1 the backward-Euler step BASELINE configs 1-2
 *                  name (the reference has Crank-Nicolson only; SURVEY
 *                  8(c)(iii) composes backward Euler from its pieces).
 * Every solve first uses the block LU WITHOUT pivoting (cheaper) and accepts
 * it only if the relative backward error is <= 1e-12; otherwise the solver
 * refactorises with partial pivoting inside the diagonal blocks, and keeps
 * pivoting for later calls (LB_CN_PIVOT=1 in the environment: always). */
int lb_cn_create(lb_ctx *ctx, const lb_mesh *mesh, int S, int n, const int *indptr,
                 const int *indices, const int *perm, int nb, lb_cn **out);
int lb_cn_destroy(lb_cn *cn);
int lb_cn_set_mass(lb_cn *cn, const double *M_vals);
int lb_cn_get_mass(lb_cn *cn, double *M_vals);
int lb_cn_newton(lb_cn *cn, const double *coK, const double *coD, double eps_d, double dt,
                 const double *f_guess, const double *f_old, const double *C_old,
                 int c_old_mode, double *f_next, double *C_guess_out, double *rnorm,
                 double *phase_ms);
int lb_cn_linear_step(lb_cn *cn, double dt, const double *C, const double *f, double *f_out);
int lb_cn_theta_step(lb_cn *cn, double dt, double theta, const double *C, const double *f,
                     double *f_out);
/* Linear-solve diagnostics: relative backward error ||(M - dt/2 C) x - b|| /
 * ||b|| of the last solve, how often the unpivoted block LU was rejected
 * (then refactorised with pivoting), and whether the solver now pivots. */
int lb_cn_stats(lb_cn *cn, double *last_rel_residual, int *fallbacks, int *pivoting);

#ifdef __cplusplus
}
#endif
#endif /* LANDAU_B200_H */
