/* ekcg_b200.h -- C ABI of the B200 enlarged-CG hot-loop kernels.
 *
 * Every entry point is `extern "C"`, takes plain device pointers and sizes,
 * never allocates, never synchronises, and launches on the CUDA stream passed
 * as `void* stream` (a cudaStream_t; NULL = legacy default stream).  Return
 * value: 0 = ok, -1 = invalid argument (nothing launched), -2 = launch error.
 *
 * Blocks are row-major n x m fp64 arrays with row stride `ld*` (>= m), the
 * layout the reference's C-contiguous numpy blocks use, so each sparse row
 * feeds m contiguous values.  `live` (may be NULL) is a device int: when it
 * reads 0 the kernel returns immediately; the solver's finalize kernel clears
 * it so iterations enqueued ahead of the host's status poll retire empty.
 *
 * The library is stateless: it holds no tunable or per-solve state.  Which
 * kernel a call launches, its grid and its split-K chunk count are functions
 * of the call's arguments (sizes, strides, pointer alignment) and of the
 * device it runs on; per-device launch set-up (shared-memory limits,
 * occupancy) is cached per device ordinal.  Calls are re-entrant per stream.
 *
 * The reference (`ekcg`, pure Python) has no FFI; each entry replaces the
 * numpy/scipy call cited beside it (paths relative to pkg/src/ekcg/).  The
 * Python driver binds these with ctypes (paper_2305_19013_b200/_lib.py);
 * INTEGRATION.md shows the binding.
 */
#ifndef EKCG_B200_H
#define EKCG_B200_H

#ifdef __cplusplus
extern "C" {
#endif

/* Grid stencil operator descriptor: the `_diffusion_matrix(shape, kappa)`
 * operator (generators.py:25-60) with per-axis coefficients c* (1.0 = the
 * reference) and node conductivity kappa(x,y,z) = kfield[(z/tz*fy + y/ty)*fx
 * + x/tx] (kfield == NULL: kappa = kconst).  dim = 2 (nz ignored) or 3.
 * Grid ordering is x-fastest (generators.py:9).
 * Rows [row_begin, row_end) are computed (row_end <= 0: all n rows).  Every
 * row-indexed pointer passed with a stencil descriptor is addressed by GLOBAL
 * row: element (i, c) of X is X[i*ldx + c] for the rows the stencil touches,
 * i.e. [row_begin - nx*ny, row_end + nx*ny) in 3-D -- a row shard passes a
 * base pointer shifted by its first row (halo planes included).
 * kself (optional, may be NULL): per tile, 2*k*k/(k+k) evaluated left to right
 * in IEEE fp64 (the harmonic mean of a tile with itself, bitwise what the
 * kernels would compute); faces between two nodes of one tile use it instead
 * of a division. */
typedef struct EkcgStencil {
    int dim;
    int nx, ny, nz;
    double cx, cy, cz;
    const double* kfield;
    int tx, ty, tz;
    int fx, fy;
    double kconst;
    long long row_begin, row_end;
    const double* kself;
    /* optional, tile fields only: face coefficients between tile t and its +x /
     * +y / +z neighbour tile, c_axis * (2 k_t k_u / (k_t + k_u)) evaluated on the
     * host with the operations of generators.py:45 (so cross-tile faces take a
     * load instead of a division; bitwise the same values). */
    const double* hx;
    const double* hy;
    const double* hz;
    /* optional, tile fields only: per-node coefficient rows built once per operator by
     * ekcg_stencil_coefs with the kernels' own arithmetic (bitwise the values computed on
     * the fly).  Row i holds EKCG_COEF_STRIDE(dim) doubles in slot order (2-D: y-, x-,
     * diag, x+, y+, pad; 3-D: z-, y-, x-, diag, x+, y+, z+, pad); absent neighbours hold
     * +0.0 (presence still follows from the grid position).  Rows are addressed by global
     * row index.  Costs 48 (2-D) / 64 (3-D) bytes per node and application, in exchange
     * for the tile lookups and face bookkeeping of every node in every column chunk. */
    const double* coef;
} EkcgStencil;

#define EKCG_COEF_STRIDE(dim) ((dim) == 3 ? 8 : 6)

/* ---- sparse operator and T^t split ------------------------------------ */

/* W[i, j] = (owner[i] == j) ? v[i] : +0.0 ; replaces Partition.split
 * (partition.py:48-55).  Bit-exact. */
int ekcg_split(const double* v, const int* owner, double* W, long long n, int t, int ldw,
               const int* live, void* stream);

/* W = split(v) + Wprev * diag(beta_sign * beta) ; the MSDO-CG candidate
 * (solvers.py:378-382). */
int ekcg_split_axpy(const double* v, const int* owner, const double* Wprev, int ldp,
                    const double* beta, double beta_sign, double* W, long long n, int t, int ldw,
                    const int* live, void* stream);

/* W[:, j] += Wprev[:, j] * beta_sign * beta[j] ; the preconditioned MSDO-CG
 * candidate (solvers.py:378-382) once W holds M^-1 split(r). */
int ekcg_axpy_cols(double* W, int ldw, const double* Wprev, int ldp, const double* beta, double beta_sign,
                   long long n, int t, const int* live, void* stream);

/* Y = A X for CSR A (int64 row_ptr, int32 col_idx) ; replaces spmm/spmv
 * (linalg.py:133-152).  Bit-exact with numpy's reduceat association. */
int ekcg_spmm_csr(const long long* row_ptr, const int* col_idx, const double* values,
                  const double* X, int ldx, double* Y, int ldy, long long n, int m,
                  const int* live, void* stream);

/* ekcg_spmm_csr with an explicit kernel form, for cross-checks of the forms
 * against each other (all are bit-identical): 0 = automatic (ekcg_spmm_csr),
 * 1 = software-pipelined (256-bit gathers when 32-B aligned), 2 = pipelined
 * with 128-bit accesses, 3 = 4 columns per thread, 4 = 2 columns per thread,
 * 5 = one thread per (row, column).  -1 when the form does not apply. */
int ekcg_spmm_csr_kernel(int form, const long long* row_ptr, const int* col_idx, const double* values,
                         const double* X, int ldx, double* Y, int ldy, long long n, int m,
                         const int* live, void* stream);

/* Y = A X for the grid stencil operator; bit-exact with ekcg_spmm_csr on the
 * CSR that generators.py:25-60 assembles for the same kappa. */
int ekcg_spmm_stencil(const EkcgStencil* desc, const double* X, int ldx, double* Y, int ldy,
                      int m, const int* live, void* stream);

/* Fill coef (n x EKCG_COEF_STRIDE(dim) doubles, n = nx*ny*nz, all rows regardless of
 * row_begin / row_end) with the per-node coefficient rows of a kfield descriptor (its own
 * coef pointer is ignored).  Attach the array to the descriptor's `coef` afterwards. */
int ekcg_stencil_coefs(const EkcgStencil* desc, double* coef, void* stream);

/* ekcg_spmm_stencil with an explicit kernel form: 0 = automatic, 1 = the TMA
 * plane march at any size (-1 when it does not apply: m % 4, alignment, or a
 * row range that is not whole planes), 2 = the row-parallel kernel. */
int ekcg_spmm_stencil_kernel(int form, const EkcgStencil* desc, const double* X, int ldx, double* Y, int ldy,
                             int m, const int* live, void* stream);

/* ---- tall-skinny block products (aortho.py:92-94,105,108; solvers.py:394-396) */

/* Number of row chunks (split-K partials) ekcg_gram uses for these sizes. */
int ekcg_gram_chunks(long long n, int d, int m1, int m2);

/* partials[p][i][a][b] = sum over rows r of chunk p of X_i[r,a] * Y[r,b],
 * for i < d.  Xs is a DEVICE array of d block pointers (row stride ldx,
 * width m1); Y has width m2.  partials holds chunks * d * m1 * m2 doubles,
 * chunks = ekcg_gram_chunks(n, d, m1, m2). Deterministic (no atomics). */
int ekcg_gram(const double* const* Xs, int ldx, int d, int m1, const double* Y, int ldy, int m2,
              long long n, double* partials, const int* live, void* stream);

/* out[j] = sum_{p < chunks} partials[p * len + j] in fixed order. */
int ekcg_reduce(const double* partials, int chunks, long long len, double* out,
                const int* live, void* stream);

/* Wout = beta * Win + sign * sum_i Q_i C_i  (Q_i: n x m1 via device pointer
 * array Qs; C: d*m1 x m2 row-major, block i at rows i*m1).  Wout may alias
 * Win.  Replaces `W -= q_i @ C` (aortho.py:93-94) and, with d = 1, beta = 0,
 * `trsm_right_inv` applied as W * R^{-1} (linalg.py:187-196). */
int ekcg_block_update(const double* const* Qs, int ldq, int d, int m1, const double* C,
                      const double* Win, int ldwi, double* Wout, int ldwo, int m2,
                      double beta, double sign, long long n, const int* live, void* stream);

/* out = W S for an upper-triangular m x m S (zeros below the diagonal): the
 * Pre-CholQR / A-CholQR applies W R0^-1 and W0 R^-1 that replace
 * trsm_right_inv (linalg.py:187-196, aortho.py:106,109).  Ws is a device
 * array holding the one block pointer.  At m = 64 the blocks of S below the
 * diagonal are skipped (FP64-bound width); other widths run ekcg_block_update. */
int ekcg_tri_apply(const double* const* Ws, int ldw, const double* S, double* out, int ldo, int m,
                   long long n, const int* live, void* stream);

/* x += W alpha ; r -= AW alpha ; rho2_partials[p] = partial sum of r_new^2
 * (solvers.py:394-397).  Uses ekcg_vec_chunks(n) partials. */
int ekcg_vec_chunks(long long n);
int ekcg_xr_update(const double* W, int ldw, const double* AW, int ldaw, const double* alpha, int m,
                   double* x, double* r, long long n, double* rho2_partials,
                   const int* live, void* stream);

/* partials[p] = partial sum of v^2 (ekcg_vec_chunks(n) partials). */
int ekcg_sumsq(const double* v, long long n, double* partials, const int* live, void* stream);

/* Block-diagonal dense product Y = B X (Y != X) over consecutive row blocks:
 * block b covers rows [starts[b], starts[b+1]), its dense nb x nb row-major
 * lower-triangular matrix sits at data[offs[b]]; transpose = 1 applies B_b^T.
 * row_block[i] is the block of row i.  With B = L^-1 / L this is the
 * block-Jacobi forward_solve / backward_solve / mult_l / mult_lt of
 * blockjacobi.py:145-170 (inverse factors precomputed at setup). */
int ekcg_block_diag_apply(const double* data, const long long* offs, const int* starts, const int* row_block,
                          int transpose, const double* X, int ldx, double* Y, int ldy, long long n, int m,
                          const int* live, void* stream);

/* Block-diagonal triangular solves by substitution, one thread per (block,
 * column): L_b Y_b = X_b (transpose = 0) or L_b^T Y_b = X_b (transpose = 1),
 * the solve_triangular calls of blockjacobi.py:145-152.  Y may alias X. */
int ekcg_block_trsv(const double* L, const long long* offs, const int* starts, int nblocks, int transpose,
                    const double* X, int ldx, double* Y, int ldy, int m, const int* live, void* stream);

/* dst[i, 0:w] = src[i, 0:w] for i < n (row strides lds, ldd): the s-step
 * chain seed V1 = newest t columns of the cached A W (solvers.py:338-339). */
int ekcg_copy_cols(const double* src, int lds, double* dst, int ldd, long long n, int w,
                   const int* live, void* stream);

/* out = a - b elementwise (r = b - A x, solvers.py:342). */
int ekcg_sub(const double* a, const double* b, double* out, long long n, const int* live, void* stream);

/* ---- small dense factorizations (linalg.py:164-184, aortho.py:74-79,98-110) */

/* Pre-CholQR step: from Graw = W^T W (m x m), column norms D, G0 = sym(D^-1
 * Graw D^-1), R0 = chol(G0); writes S0 = D^-1 R0^-1 (upper).  Breakdown
 * (zero column or pivot <= tol * max diag) is recorded in ctrl and clears
 * ctrl->live.  `ctrl` points at an EkcgCtrl block. */
int ekcg_prechol(const double* Graw, int m, double* S0, void* ctrl, int iteration, double tol,
                 void* stream);

/* A-CholQR step: R = chol(sym(G)); writes S = R^-1 (upper). */
int ekcg_cholinv(const double* G, int m, double* S, void* ctrl, int iteration, double tol,
                 void* stream);

/* Standalone Cholesky (no breakdown side effects): R (upper, m x m) and info
 * = {0 ok | 1 breakdown, column, pivot-as-double-bits}. Test surface for
 * cholesky_small (linalg.py:164-184). */
int ekcg_cholesky(const double* B, int m, double tol, double* R, double* info, void* stream);

/* ---- fused iteration kernels (m in {8,16,32,64}) -------------------------
 * Each reduces its split-K partials in-kernel (last CTA to arrive, fixed
 * order) and runs the m x m factor / bookkeeping there.  `partials` holds
 * ekcg_fused_partials(n, m) doubles; `counter` points to EKCG_FUSED_COUNTERS
 * device uint32 that must be 0 before the first call (the kernels leave them 0). */
#define EKCG_FUSED_COUNTERS 64
int ekcg_fused_partials(long long n, int m);

/* Wout = Win - sum_i Q_i C_i (CGS2 pass 2, aortho.py:93-94) fused with
 * Graw = Wout^T Wout and the Pre-CholQR factor S0 (aortho.py:104-106). */
int ekcg_update_prechol(const double* const* Qs, int ldq, int d, const double* C, const double* Win, int ldwi,
                        double* Wout, int ldwo, int m, long long n, double* partials, unsigned int* counter,
                        double* S0, void* ctrl, int iteration, double tol, void* stream);

/* Wout = Q_0 S (W_k = W0 R^-1, linalg.py:187-196) fused with vout = Wout^T vec
 * (alpha = W^T r, solvers.py:394). */
int ekcg_update_vec(const double* const* Qs, int ldq, const double* S, double* Wout, int ldwo, int m, long long n,
                    const double* vec, double* partials, unsigned int* counter, double* vout, void* ctrl,
                    void* stream);

/* G = X^T (A X) for the stencil operator without materialising A X, fused
 * with the A-CholQR factor S = chol(sym G)^-1 (aortho.py:107-109). ldx == m.
 * finalize = 0 writes the (local) G to `out` instead -- a row shard
 * allreduces it and calls ekcg_cholinv. */
int ekcg_stencil_cholinv(const EkcgStencil* desc, const double* X, int ldx, int m, double* partials,
                         unsigned int* counter, double* out, void* ctrl, int iteration, double tol, int finalize,
                         void* stream);

/* Y = A X (written) fused with x += X alpha, r -= Y alpha, |r|^2 and, when
 * do_finish, the end-of-iteration bookkeeping of ekcg_finish (else |r|^2 is
 * stored to *rho2_out) -- solvers.py:394-415. */
int ekcg_stencil_xr(const EkcgStencil* desc, const double* X, int ldx, double* Y, int ldy, int m,
                    const double* alpha, double* x, double* r, double* partials, unsigned int* counter, void* ctrl,
                    int k, int kmax, int stagnation_window, double* history, int do_finish, double* rho2_out,
                    void* stream);

/* ---- whole solve in one kernel (small problems) ------------------------- */

/* The complete truncated-window SRE-CG / SRE-CG2 loop of `_run_engine`
 * (solvers.py:319-428: candidate, CGS2 aortho.py:89-95, Pre-CholQR + A-CholQR
 * aortho.py:98-110, alpha / x / r update and stop test solvers.py:394-415, the
 * true-residual log every `every` iterations :401-402) as ONE kernel on one
 * thread-block cluster (up to 16 CTAs, distributed-shared-memory reductions,
 * hardware cluster barriers): for problems whose blocks live in L2, where an
 * iteration of separate launches is latency-bound.  Unpreconditioned, s = 1,
 * t <= 16, window <= 4 (t <= 8) or <= 2 (t <= 16), n t <= 2^22
 * (ekcg_cluster_solve_fits); the operator is the stencil `desc` (whole grid)
 * or, with desc == NULL, a CSR matrix whose rows hold at most 8 entries.
 * Before the call: x = x0, r = b - A x0, and ctrl / history[0] initialised by
 * ekcg_start.  `blocks` is scratch of (2 window + 3) * span + n doubles (span >=
 * n t, a multiple of 32).  On return (stream order) ctrl holds the final
 * status / k_done / breakdown record, history[1..k_done] the residual norms,
 * checks[j] the true residual after iteration (j + 1) * every.  A CSR matrix with a
 * row of more than 8 entries is refused: ctrl->status = 5, nothing else written.  phase_ticks (may
 * be NULL) is a diagnostic: 20 device int64 that CTA 0 increments by the SM cycles
 * it spent in each phase of the iteration (tools/cluster_time.py names them). */
int ekcg_cluster_solve_fits(long long n, int t, int window);
int ekcg_cluster_solve(const EkcgStencil* desc, const long long* row_ptr, const int* col_idx,
                       const double* values, long long n, int t, int window, int kmax, int every,
                       const int* owner, const double* b, double* x, double* r, double* blocks,
                       long long span, void* ctrl, double* history, double* checks, double chol_tol,
                       long long* phase_ticks, void* stream);

/* Classical unpreconditioned CG (`cg`, solvers.py:199-258) as one kernel on one thread-block
 * cluster, for small problems (n <= 2^22; rows of at most 8 entries in CSR form): one cluster
 * barrier and two scalar exchanges per iteration, no host reads inside the loop.  Before the
 * call: x = x0, r = b - A x0, ctrl / history[0] initialised by ekcg_start (tol_abs = tol * rho0).
 * `scratch` holds 2 n doubles (p, A p).  On return ctrl holds status (1 converged, 2 maxiter,
 * 3 = nonpositive curvature with brk_pivot = p^T A p and brk_iter = the iteration, 5 = a CSR
 * row of more than 8 entries: refused) and k_done. */
int ekcg_cluster_cg(const EkcgStencil* desc, const long long* row_ptr, const int* col_idx,
                    const double* values, long long n, int kmax, double* x, double* r, double* scratch,
                    void* ctrl, double* history, void* stream);

/* ---- engine bookkeeping ------------------------------------------------ */

/* Size in bytes of the control block. */
int ekcg_ctrl_bytes(void);

/* Initialise ctrl from rho0^2 = *rho2 : history[0] = rho0, tol_abs = tol*rho0,
 * converged immediately when rho0 == 0. */
int ekcg_start(void* ctrl, const double* rho2, double tol, double* history, void* stream);

/* End of iteration k: rho = sqrt(*rho2), history[k] = rho, stagnation guard
 * (window > 0), convergence (rho <= tol*rho0) and kmax checks (solvers.py:357,399,406-415).
 * Everywhere an iteration number is passed (k / iteration arguments of the
 * finish, factor and fused kernels), k <= 0 means "read it on the device as
 * ctrl->k_done + 1" -- what CUDA-graph replay of an iteration uses. */
int ekcg_finish(void* ctrl, const double* rho2, int k, int kmax, int stagnation_window,
                double* history, void* stream);

/* checks[slot] = sqrt(*rho2) when the solve is live (true residual log, solvers.py:401-402). */
int ekcg_store_norm(const double* rho2, double* checks, int slot, const int* live, void* stream);

/* Kernel launches issued through this library since load. */
unsigned long long ekcg_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* EKCG_B200_H */
