/*
 * libmg — B200-native Galerkin surface multigrid (arXiv 2104.13755), C ABI.
 *
 * The hot path of the paper's solver (Alg. 1, Alg. 2
 * P:527-561, stored hierarchy P:506) as hand-written sm_100a CUDA kernels
 * behind a plain C interface: no C++ types, no torch types.  Citations
 * "P:n" are lines of PAPER.md; readings A1..A22 are listed in DESIGN.md.
 *
 * Conventions for every call
 *   - Indices are int32, values IEEE binary64.
 *   - Matrices are CSR: row_ptr[n+1], col[nnz] (sorted, unique per row), val[nnz].
 *   - Multi-column vectors (k right-hand sides) are row-major [n][k]: the k
 *     values of one vertex are contiguous.
 *   - "host or device" pointers: the library inspects the pointer with
 *     cudaPointerGetAttributes and stages host buffers (pageable or pinned)
 *     through its own device memory; the copies run on the context stream.
 *   - All device work is enqueued on the context's stream (mg_create).
 *   - Return value: MG_OK (0) or one of the codes below; no exception crosses
 *     the ABI.  mg_last_error() returns a one-line message for the last
 *     failing call on that context.  MG_NOT_CONVERGED is non-fatal.
 *   - A context is not thread-safe; separate contexts are independent.
 *   - Ownership: every input array is copied; the caller keeps ownership of
 *     everything it passes.  The context owns all device memory it allocates
 *     and frees it in mg_destroy.
 */
#ifndef LIBMG_MG_H
#define LIBMG_MG_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum mg_status {
    MG_OK = 0,
    MG_ERR_INVALID_ARG = 1, /* null pointer, negative count, unsupported k       */
    MG_ERR_SHAPE = 2,       /* sizes inconsistent with the loaded hierarchy      */
    MG_ERR_INPUT = 3,       /* malformed input data (index range, P rows, CSR)   */
    MG_ERR_NOT_SPD = 4,     /* non-positive pivot in the coarsest Cholesky       */
    MG_ERR_STATE = 5,       /* call out of order (no hierarchy / no matrix)      */
    MG_ERR_CUDA = 6,        /* CUDA runtime error or no device                   */
    MG_ERR_NUMERIC = 7,     /* NaN/Inf in a residual norm                        */
    MG_NOT_CONVERGED = 8    /* max_cycles reached with some rho > rel_tol         */
};

typedef struct mg_ctx mg_ctx;

/* Create a context on CUDA `device`.  `cuda_stream` is a cudaStream_t (e.g.
 * torch.cuda.current_stream().cuda_stream) or NULL for a private stream.
 * Errors: MG_ERR_INVALID_ARG (out == NULL), MG_ERR_CUDA (no device / driver). */
int mg_create(mg_ctx** out, int device, void* cuda_stream);
void mg_destroy(mg_ctx* ctx);
const char* mg_last_error(const mg_ctx* ctx);

/* Relaxation sweeps per level: mu_pre before restriction, mu_post
 * after the correction.  Default 2 / 2 ("2 pre- and post-relaxation
 * iterations").  Errors: MG_ERR_INVALID_ARG if negative. */
int mg_set_options(mg_ctx* ctx, int mu_pre, int mu_post);

/* Load the precomputed hierarchy (Alg. 1 line 2), host arrays.
 *   n_levels        grids 0 (finest) .. n_levels-1 (coarsest, H = n_levels-1), >= 1
 *   n_verts[l]      vertices of level l
 *   n_faces[l]      faces of level l (only level 0's faces are required to be valid;
 *                   F[l] for l >= 1 may be NULL with n_faces[l] = 0)
 *   V[l]            positions [n_verts[l]][3]  (used for locality ordering; V[0]
 *                   also defines the fine mesh for mg_set_matrix_cotan)
 *   F[l]            triangles [n_faces[l]][3]
 *   P_cols[l],P_w[l] the prolongation P_l from level l+1 to level l, ELL-3:
 *                   [n_verts[l]][3] coarse column / barycentric weight per fine
 *                   vertex ("3 non-zeros ... barycentric coordinates"),
 *                   l = 0 .. n_levels-2.  Weights must be >= 0 and sum to 1
 *                   within 1e-12 per row; a weight of exactly 0.0 is padding and
 *                   contributes no structure (reading A9).
 * Validates index ranges, weights, and that F[0] is an edge-manifold triangle
 * list (every edge in <= 2 faces).  Resets any matrix state.
 * Errors: MG_ERR_INVALID_ARG, MG_ERR_SHAPE, MG_ERR_INPUT (message names the row). */
int mg_hierarchy_load(mg_ctx* ctx, int n_levels, const int32_t* n_verts, const int32_t* n_faces,
                      const double* const* V, const int32_t* const* F,
                      const int32_t* const* P_cols, const double* const* P_w);

/* Set the fine system matrix A (symmetric positive (semi-)definite) as
 * CSR in user vertex order; host or device arrays (`on_device` is a hint and
 * is cross-checked against the pointer attributes).  Requires
 * n == n_verts[0], sorted unique columns, a structurally symmetric pattern
 * and a diagonal entry present and > 0 in every row.  A new pattern
 * triggers pattern setup (symbolic P^T A P, Alg. 3 colouring and the internal
 * colour-grouped ordering of every level); a known pattern reuses it.  Then
 * computes every coarse operator A_{l+1} = P_l^T A_l P_l (Eq. gca P:277-279,
 * P:506) on the GPU and factors A_H (dense Cholesky, reading A12).
 * Errors: MG_ERR_STATE (no hierarchy), MG_ERR_SHAPE, MG_ERR_INPUT,
 * MG_ERR_NOT_SPD, MG_ERR_CUDA. */
int mg_set_matrix(mg_ctx* ctx, int32_t n, int64_t nnz, const int32_t* row_ptr, const int32_t* col,
                  const double* val, int on_device);

/* Assemble A = mass_coeff * M + lap_coeff * L on the GPU from positions V
 * ([n_verts[0]][3], host or device) over the fine faces F[0]: L the
 * cotangent Laplacian (PSD convention, reading A13), M the lumped
 * barycentric mass (reading A14).  Natural boundary conditions arise
 * from the assembly.  Then as mg_set_matrix (Galerkin + factor).
 * M is kept for mg_apply_mass.  The pattern is the 1-ring of F[0].
 * Errors: MG_ERR_STATE (no hierarchy or F[0] empty), MG_ERR_INVALID_ARG,
 * MG_ERR_NOT_SPD, MG_ERR_CUDA. */
int mg_set_matrix_cotan(mg_ctx* ctx, const double* V, double mass_coeff, double lap_coeff);

/* Row f3: the squared-Laplacian (bilaplacian) smoothing operator, E_{Delta^2}
 * of the data-smoothing application ("the Bilaplacian (2-ring sparsity)",
 * P:595), assembled on the GPU from positions V ([n_verts[0]][3], host
 * or device) over F[0]:
 *     A = mass_coeff * M + bilap_coeff * Q,   Q = L M^{-1} L
 * with L the cotan Laplacian (A13) and M the lumped mass (A14); the pattern is
 * the 2-ring of F[0].  For the data-smoothing system of App. D eq. 1 use
 * mass_coeff = 1 - alpha, bilap_coeff = alpha and B = (1 - alpha) M f
 * (mg_apply_mass).  Then as mg_set_matrix (Galerkin + factor; honours
 * mg_set_dirichlet).  M is kept for mg_apply_mass.
 * Errors: as mg_set_matrix_cotan. */
int mg_set_matrix_bilaplacian(mg_ctx* ctx, const double* V, double mass_coeff, double bilap_coeff);

/* B = M X with the lumped mass of the last mg_set_matrix_cotan / _bilaplacian; X, B are
 * [n][k], each host or device independently.  Errors: MG_ERR_STATE. */
int mg_apply_mass(mg_ctx* ctx, int32_t k, const double* X, double* B);

/* Solve A X = B by V(mu_pre, mu_post) cycles (Alg. 1).
 *   k            right-hand sides, 1 <= k <= 4
 *   B            [n][k] right-hand sides (host or device)
 *   X            [n][k] initial guess on entry (warm starts honoured), solution
 *                on exit (host or device)
 *   rel_tol      stop when every column has rho = ||b - A x||_2 / ||b||_2
 *                <= rel_tol (readings A3, A11); rel_tol <= 0 runs exactly
 *                max_cycles cycles
 *   res_hist     host array of (max_cycles+1)*k doubles or NULL; entry
 *                [c*k + j] = rho of column j after cycle c (c = 0 is the
 *                initial residual)
 *   cycles_out   number of V-cycles run (may be NULL)
 * Synchronises the stream before returning.
 * Returns MG_OK, MG_NOT_CONVERGED (X holds the last iterate, the history is
 * complete), MG_ERR_NUMERIC (NaN/Inf), MG_ERR_STATE, MG_ERR_INVALID_ARG. */
int mg_solve(mg_ctx* ctx, int32_t k, const double* B, double* X, double rel_tol, int32_t max_cycles,
             double* res_hist, int32_t* cycles_out);

/* ---- Dirichlet constraints (App. B) ------------- */

/* Prescribe the values of the fine vertices known[0..n_known) (user indices,
 * unique; host array, copied).  The solver then works on the reduced system
 *   A_uu x_u = b_u - A_uk x_k           (App. B, "reduced LHS" / "reduced RHS")
 * over the reduced hierarchy: the finest prolongation keeps the rows of the
 * unknowns, P_{u:}; at every level, coarse columns whose largest weight over
 * the kept rows is 0 are removed together with their row of the next
 * prolongation (reading A24 applies the rule level by level), and
 * the hierarchy ends at the last non-empty level.  After this call:
 *   - mg_set_matrix / mg_set_matrix_cotan take the FULL fine operator
 *     (n_verts[0] rows) and extract A_uu and A_uk on the GPU;
 *   - mg_solve / mg_solve_pcg take FULL [n_verts[0]][k] B and X: X holds the
 *     known values at known rows (read, never written) and the initial guess
 *     elsewhere; only the unknown rows of X are written; rho is the relative
 *     residual of the reduced system;
 *   - mg_apply_mass / mg_get_mass stay full-size; the level exports
 *     (mg_level_info, mg_get_level_csr, mg_get_colouring) describe the
 *     reduced levels (level 0 rows = unknowns in ascending user order);
 *   - the App. D split operators are not available (MG_ERR_STATE).
 * Every vertex known: solves return at once (0 cycles, X unchanged).
 * n_known = 0 restores the unconstrained hierarchy.  Invalidates the matrix.
 * Errors: MG_ERR_STATE (no hierarchy), MG_ERR_INVALID_ARG, MG_ERR_INPUT
 * (index out of range or repeated), MG_ERR_SHAPE (reduced coarsest > 4096). */
int mg_set_dirichlet(mg_ctx* ctx, int32_t n_known, const int32_t* known);

/* ---- smoother variants and MG-preconditioned CG ---------- */

/* Relaxation used by every level of the V-cycle.
 *   kind 0: multicolour Gauss-Seidel over the Alg. 3 colouring (default,
 *           reading A2: pre- and post-sweeps in ascending colour order);
 *   kind 1: damped Jacobi x <- x + omega D^{-1} (b - A x) ("(damped) Jacobi",
 *           App. E), omega in (0, 1] (default 0.8, SPEC reading).
 *   symmetric != 0: post-relaxation colours in DESCENDING order, so the
 *           post-smoother is the adjoint of the pre-smoother and the V-cycle
 *           is a symmetric operator (mg_solve_pcg always uses it).
 * Errors: MG_ERR_INVALID_ARG (unknown kind, omega out of range). */
int mg_set_smoother(mg_ctx* ctx, int kind, double omega, int symmetric);

/* Initial guess of mg_solve / mg_solve_pcg.  on != 0: every solve starts
 * from X0 = 0 (Alg. 2 applied to a zero iterate, as the paper's solves do)
 * and X is output only: its input values are not read, so a host X costs no
 * host-to-device copy.  on = 0 (default): X holds the initial guess on input.
 * Ignored while Dirichlet constraints are set (X supplies the known values,
 * App. B).  Errors: MG_ERR_INVALID_ARG (null ctx). */
int mg_set_zero_guess(mg_ctx* ctx, int32_t on);

/* Solve A X = B by conjugate gradients preconditioned with one symmetric
 * V-cycle from a zero guess per iteration ("use our multigrid solver as the
 * pre-conditioner for ... the conjugate gradient method").  Every
 * column independently (own alpha, beta), all columns iterated until every
 * column meets rel_tol.  Arguments and layout as mg_solve; res_hist[it*k + j]
 * = ||r_it||_2 / ||b_j||_2 of the recursively updated PCG residual, entry 0
 * the initial residual.  Requires mu_pre == mu_post (symmetric
 * preconditioner).  Returns MG_OK, MG_NOT_CONVERGED (X holds the last
 * iterate), MG_ERR_NUMERIC, MG_ERR_STATE, MG_ERR_INVALID_ARG. */
int mg_solve_pcg(mg_ctx* ctx, int32_t k, const double* B, double* X, double rel_tol, int32_t max_iters,
                 double* res_hist, int32_t* iters_out);

/* ---- fast data smoothing (App. D) -------------
 * The data-smoothing system (alpha Q + (1 - alpha) M) x = (1 - alpha) M f
 * (App. D eq. 1) has coarse operators
 *     P^T A(alpha) P = alpha (P^T Q P) + (1 - alpha) (P^T M P)
 * (App. D eq. 2), so P^T Q P and P^T M P are precomputed once per level and
 * every later alpha costs one scaled sparse addition per level plus the
 * coarsest refactorisation: no triple product runs in the alpha loop. */

/* Set Q and M on ONE fine CSR pattern (user order; an entry absent from one
 * operator is stored as 0 in it), host or device arrays, copied.  Pattern
 * requirements as mg_set_matrix.  Computes P^T Q P and P^T M P at every
 * level on the GPU.  The system matrix is NOT set until mg_set_alpha.
 * Errors: as mg_set_matrix (except MG_ERR_NOT_SPD). */
int mg_set_matrix_split(mg_ctx* ctx, int32_t n, int64_t nnz, const int32_t* row_ptr, const int32_t* col,
                        const double* q_val, const double* m_val);
/* As mg_set_matrix_split with Q = L (cotan Laplacian, reading A13) and M =
 * lumped mass (A14) assembled on the GPU from positions V [n_verts[0]][3]
 * (host or device) over F[0]; M is kept for mg_apply_mass. */
int mg_set_matrix_split_cotan(mg_ctx* ctx, const double* V);
/* A_h = alpha Q_h + (1 - alpha) M_h at every level (App. D eq. 2), then the
 * coarsest Cholesky.  Errors: MG_ERR_STATE (no split operators),
 * MG_ERR_INVALID_ARG (alpha not finite), MG_ERR_NOT_SPD, MG_ERR_CUDA. */
int mg_set_alpha(mg_ctx* ctx, double alpha);

/* ---- exports for parity checks (host arrays, USER vertex order) ---------- */

/* Level l sizes: rows, stored entries, colours of Alg. 3.  MG_ERR_STATE
 * before the first mg_set_matrix*. */
int mg_level_info(mg_ctx* ctx, int l, int32_t* n, int64_t* nnz, int32_t* n_colours);
/* Level-l matrix A_l in user vertex order: row_ptr[n+1], col[nnz], val[nnz]
 * (caller-allocated, sizes from mg_level_info); any of them may be NULL. */
int mg_get_level_csr(mg_ctx* ctx, int l, int32_t* row_ptr, int32_t* col, double* val);
/* Alg. 3 colour of every level-l vertex (user order), colour ids in creation order. */
int mg_get_colouring(mg_ctx* ctx, int l, int32_t* colour);
/* Lumped mass diagonal M[n_verts[0]] of the last mg_set_matrix_cotan. */
int mg_get_mass(mg_ctx* ctx, double* M);
/* Coarsest dense Cholesky factor, lower triangle, [n_H][n_H] row-major, user order. */
int mg_get_coarse_factor(mg_ctx* ctx, double* L);

/* ---- host-only utilities (no device needed): the library's own host
 * pattern-setup steps, exported so the CPU test suite can check them
 * bit-exactly against the oracle. ------------------------------------------ */

/* Alg. 3 greedy colouring (readings A6-A8) of the structural
 * off-diagonal graph of a square CSR pattern.  colour[n] out; *n_colours out. */
int mg_util_greedy_colouring(int32_t n, const int32_t* row_ptr, const int32_t* col, int32_t* colour,
                             int32_t* n_colours);

/* Symbolic Galerkin pattern of P^T A P (reading A9) for fine CSR pattern A
 * (n_fine) and ELL-3 prolongation (n_fine x n_coarse).  Two-call protocol:
 * call with c_col == NULL to get *c_nnz and fill c_row_ptr[n_coarse+1]; call
 * again with c_col of size *c_nnz. */
int mg_util_galerkin_pattern(int32_t n_fine, const int32_t* row_ptr, const int32_t* col, int32_t n_coarse,
                             const int32_t* P_cols, const double* P_w, int32_t* c_row_ptr, int64_t* c_nnz,
                             int32_t* c_col);

/* 1-ring CSR pattern of a triangle mesh (sorted columns, diagonal included:
 * the fixed pattern of the cotan assembly) and, per stored entry, the
 * row-local positions of the <= 2 vertices opposite the edge (i, col): low
 * nibble = position among row i's entries of the first, high nibble = of the
 * second, 15 = none (diagonal, boundary edge: natural BC) - the
 * table k_cotan_slots reads.  F: [n_faces][3] host.  Two-call protocol: call
 * with col == NULL to get *nnz and row_ptr[n+1]; then with col[*nnz] and
 * slots[*nnz] (slots may be NULL).  Errors: MG_ERR_INVALID_ARG, MG_ERR_INPUT
 * (index out of range, a vertex in no face), MG_ERR_SHAPE (slots requested
 * and a row has more than 15 entries: the library then keeps vertex indices). */
int mg_util_one_ring(int32_t n, int32_t n_faces, const int32_t* F, int32_t* row_ptr, int64_t* nnz, int32_t* col,
                     uint8_t* slots);

/* ---- execution options ----------------------------------------------------- */

/* How the same arithmetic is scheduled (results are bitwise identical except
 * MG_EXEC_COARSE_TRSV, which changes the coarsest solve's rounding only).
 * flags: OR of the bits below; 0 = defaults.  Must be followed by
 * mg_set_matrix* (the pattern setup builds the tile and cluster structures),
 * drops captured graphs.  MG_ERR_INVALID_ARG on unknown bits. */
#define MG_EXEC_NO_PDL 1          /* no programmatic dependent launch inside the V-cycle graph */
#define MG_EXEC_NO_PIPE 2         /* plain tile kernels instead of the TMA-bulk pipelined ones */
#define MG_EXEC_COARSE_TRSV 4     /* coarsest solve by two triangular solves (one CTA), not A_H^{-1} GEMV */
#define MG_EXEC_DEVICE_LOOP 8     /* Alg. 1 loop on the device (conditional WHILE graph node) */
int mg_set_execution(mg_ctx* ctx, int flags);

/* ---- instrumentation (bench.py) ----------------------------------------- */

/* Per-kernel-class timing with CUDA events on the context stream.  Bit c of
 * class_mask selects class c (classes listed at mg_get_profile); 0 turns
 * profiling off.  Bits 16..31, if any is set, restrict timing to those levels
 * (bit 16 + l = level l).  Inside mg_solve the events are event-record nodes of the
 * captured V-cycle graph, so the timings are taken in the production path. */
int mg_set_profiling(mg_ctx* ctx, int class_mask);
/* Accumulated device milliseconds and kernel launches per (kernel class, level):
 * classes 0 gs_sweep, 1 residual+restrict, 2 prolong, 3 coarse_solve,
 * 4 resnorm, 5 galerkin, 6 assembly, 7 factor, 8 permute, 9 coarse_tail (the
 * single-launch cluster kernel that runs the V-cycle on the small levels),
 * 10 alpha (the App. D per-level scaled addition of mg_set_alpha).  ms[cls*16 + l],
 * launches[cls*16 + l] (levels >= 16 fold into 15).  Resets the counters. */
int mg_get_profile(mg_ctx* ctx, double* ms, int64_t* launches);
/* Device kernel launches issued by this context since creation. */
int64_t mg_launch_count(const mg_ctx* ctx);
/* Shape of the loaded problem, for argument checking by bindings: *n_full =
 * fine vertices of the hierarchy as loaded (the row count of every user-side
 * B, X, V; Dirichlet constraints do not change it), *device = the CUDA device
 * the context enqueues on.  Either pointer may be NULL.  MG_ERR_STATE before
 * mg_hierarchy_load. */
int mg_problem_size(const mg_ctx* ctx, int32_t* n_full, int32_t* device);

#ifdef __cplusplus
}
#endif
#endif /* LIBMG_MG_H */
