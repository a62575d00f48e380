/*
 * redhess.h -- C ABI of the B200-native batched adjoint-adjoint reduced-Hessian
 * library (arXiv 2201.00241, "Batched Second-Order Adjoint Sensitivity for
 * Reduced Space Methods").  fp64 throughout, 0-based indices, extern "C".
 *
 * Problem (section 3, Eq. powerflow, Eq. powerflowvec
 * PAPER.md:225-239, Eq. nonlinearopt): for the AC power-flow
 * balance equations g(x, p) = 0 with
 *     x = (theta_pv, theta_pq, v_pq)          (order: DESIGN.md R5)
 *     p = (Pg_pv, v_{ref u pv})               (R3, R5)
 * and the cost f = sum_gen c2 Pg^2 + c1 Pg + c0 (Pg_ref = P_ref + Pd_ref,
 * DESIGN.md R4), the library evaluates
 *   * the first-order adjoint lambda = -(grad_x g)^{-T} grad_x f^T and the reduced
 *     gradient grad_p F = grad_p f + lambda^T grad_p g   (Eq. reduced_gradient,
 *     PAPER.md:324-333);
 *   * batches of N reduced Hessian-vector products by Alg. 2:
 *     B = G_p W; J Z = -B; [Y_x; Y_p] = grad^2 l [Z; W]; J^T Psi = -Y_x;
 *     HW = Y_p + G_p^T Psi  (Eq. socadjoint, Eq. hessvecprod
 *     PAPER.md:393-399), J = grad_x g, G_p = grad_p g, l = f + lambda^T g;
 *   * the full reduced Hessian grad^2_pp F by ceil(n_p/N) Cartesian batches
 *     (R10).
 *
 * Memory / ownership
 *   - The caller owns every pointer it passes; the library keeps none after a
 *     call returns.  Host arrays (rh_grid, rh_orderings outputs, *_host calls)
 *     are read/written synchronously.
 *   - "device" pointers are CUDA device memory on the context's device; calls
 *     that take them are stream-ordered on `stream` (a cudaStream_t passed as
 *     void*; NULL = legacy default stream).  Inputs are copied into library
 *     buffers before the call's work completes in stream order.
 *   - rh_ctx owns all internal device memory (grid, maps, factors, tape,
 *     workspace).  The workspace grows with the largest N seen: about
 *     2 * n_x * roundup(N, 32) * 8 bytes.
 *   - Batched blocks are row-major with the batch index fastest ("SoA across
 *     the batch"): element (row i, direction k) of W is W[i * ldw + k].
 *
 * Errors
 *   Every call returns an rh_status; rh_last_error() gives a message for the
 *   last non-OK return on that context.  Usage errors (bad arguments, calls
 *   out of order) are detected synchronously.  Kernel errors are asynchronous
 *   and surface at the next synchronizing call (rh_set_state synchronizes once
 *   to read the refactorization pivot flag, R15).
 *
 * Threading: one context per host thread; contexts are independent.
 */
#ifndef REDHESS_H
#define REDHESS_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct rh_ctx rh_ctx;

typedef enum rh_status {
  RH_OK = 0,
  RH_E_ARG = 1,       /* invalid argument (null pointer, size, ld < N, ...)          */
  RH_E_GRID = 2,      /* grid rejected by validation (R24, R25)            */
  RH_E_ORDER = 3,     /* call out of order (e.g. rh_hvp before rh_set_state)         */
  RH_E_SINGULAR = 4,  /* refactorization pivot below threshold (static pivots, R15)  */
  RH_E_CUDA = 5,      /* CUDA runtime error (message in rh_last_error)               */
  RH_E_NOMEM = 6,     /* device allocation failed                                    */
  RH_E_NODEV = 7,     /* compute call on a host-only context (device = -1)           */
  RH_E_NOCONV = 8,    /* Newton projection did not converge within maxit steps       */
  RH_E_NOTPD = 9      /* tracking Step 2: not positive definite after 64 shifts      */
} rh_status;

/* Bus type codes (MATPOWER): PQ = 1, PV = 2, REF = 3. */
enum { RH_PQ = 1, RH_PV = 2, RH_REF = 3 };
/* Variable kinds returned by rh_orderings. */
enum { RH_KIND_THETA = 0, RH_KIND_V = 1, RH_KIND_PG = 2 };

/*
 * Grid description (graph G = {V, E}, adjacencies A(i), line
 * admittances g_ij, b_ij; R1: Ybus convention with the diagonal).
 * All arrays are HOST memory, read during rh_load_grid only.
 */
typedef struct rh_grid {
  int32_t n_bus, n_line, n_gen;
  const int32_t *bus_type;            /* [n_bus] RH_PQ / RH_PV / RH_REF; exactly one RH_REF          */
  const double *G_ii, *B_ii;          /* [n_bus] Ybus diagonal (series, shunts, charging, taps folded) */
  const double *Pd, *Qd;              /* [n_bus] loads, per unit (positive = consumption)            */
  const int32_t *line_f, *line_t;     /* [n_line] from/to bus, f != t; parallel lines add            */
  const double *G_ft, *B_ft;          /* [n_line] Ybus[f][t] = G_ft + j B_ft                         */
  const double *G_tf, *B_tf;          /* [n_line] Ybus[t][f] = G_tf + j B_tf                         */
  const int32_t *gen_bus;             /* [n_gen] PV or REF buses, at most one generator per bus      */
  const double *c2, *c1, *c0;         /* [n_gen] cost f = sum c2 Pg^2 + c1 Pg + c0 (per unit)        */
  double theta_ref;                   /* REF angle, a constant (R6)                        */
} rh_grid;

/* Sizes and statistics of the loaded grid and its symbolic analysis. */
typedef struct rh_info {
  int32_t n_bus, n_line, n_x, n_p;
  int32_t nnz_J;        /* nonzeros of J = grad_x g                                   */
  int32_t nnz_Gp;       /* nonzeros of G_p = grad_p g                                 */
  int32_t nnz_LU;       /* nonzeros of the filled factor L+U (diagonal counted once)  */
  int32_t levels_fwd;   /* dependency levels of the L and U^T sweeps                  */
  int32_t levels_bwd;   /* dependency levels of the U and L^T sweeps                  */
  int32_t max_level_rows;
  int32_t n_blocks;     /* elimination-tree blocks (segments of whole subtrees)        */
  int32_t sep_rows;     /* rows of the separator segment above the blocks              */
  int32_t seg_levels;   /* max dependency levels inside one segment (any sweep)        */
  int64_t workspace_bytes; /* current device workspace                                 */
} rh_info;

/* Create a context on CUDA device `device`; device = -1 creates a HOST-ONLY
 * context (grid validation and symbolic analysis only; every compute call
 * returns RH_E_NODEV).  *out receives the context. */
int rh_create(int device, rh_ctx **out);
int rh_destroy(rh_ctx *ctx);
/* Message for the last non-OK return on ctx (never NULL; "" if none). */
const char *rh_last_error(const rh_ctx *ctx);

/* Validate and load a grid (host arrays, copied), build the x/p index maps
 * (R3, R5), the J and G_p patterns, a minimum-degree symmetric ordering, the
 * static-pivot symbolic LU and the level sets of the four triangular sweeps
 * (the factorization is analysed on the
 * host, numeric work happens on the device).  Writes n_x, n_p (nullable). */
int rh_load_grid(rh_ctx *ctx, const rh_grid *grid, int32_t *n_x, int32_t *n_p);

int rh_get_info(const rh_ctx *ctx, rh_info *info);

/* Orderings of x and p (R5), host outputs [n_x] and [n_p]:
 * bus index and kind (RH_KIND_*) of every entry.  Any pointer may be NULL. */
int rh_orderings(const rh_ctx *ctx, int32_t *x_bus, int32_t *x_kind,
                 int32_t *p_bus, int32_t *p_kind);

/* Symbolic factor of the symmetrically permuted J (host outputs):
 * perm[n_x] (perm[new] = old x index), lu_rowptr[n_x + 1] and
 * lu_colidx[nnz_LU] (CSR of the L+U pattern in the permuted numbering, sorted
 * columns), level_fwd[n_x], level_bwd[n_x] (0-based level of every permuted
 * row in the forward / backward sweeps).  Any pointer may be NULL. */
int rh_symbolic(const rh_ctx *ctx, int32_t *perm, int32_t *lu_rowptr, int32_t *lu_colidx,
                int32_t *level_fwd, int32_t *level_bwd);

/* Segment of every permuted row (host output [n_x]): 0..n_blocks-1 = block
 * (a union of whole elimination subtrees, processed in shared memory by one
 * CTA per column chunk), n_blocks = separator. */
int rh_segments(const rh_ctx *ctx, int32_t *segment_of_row);

/* Set the operating point: x [n_x], p [n_p] DEVICE arrays.  Runs the state
 * kernels (line trig, bus injections, g, P_ref), assembles J and G_p
 * (PAPER.md:694-713 analog), refactorizes J numerically on the fixed pattern
 * and synchronizes `stream` once to read the pivot flag.
 * Invalidates the multipliers.  RH_E_SINGULAR if a pivot |u_kk| falls below
 * 1e-14 * max|row k of J|. */
int rh_set_state(rh_ctx *ctx, const double *x, const double *p, void *stream);

/* Residual g(x, p) [n_x] (DEVICE, nullable) and objective f (DEVICE scalar,
 * nullable) at the current state (Eq. powerflowvec; R2, R4). */
int rh_residual(rh_ctx *ctx, double *g, double *f, void *stream);

/* First-order adjoint and reduced gradient (Eq. reduced_gradient,
 * PAPER.md:324-333): lambda = -J^{-T} grad_x f, grad_p F = grad_p f + G_p^T lambda.
 * grad_p [n_p] and lambda_out [n_x] are DEVICE arrays (lambda_out nullable).
 * Sets lambda as the active multipliers (R16). */
int rh_reduced_gradient(rh_ctx *ctx, double *grad_p, double *lambda_out, void *stream);

/* Override the active multipliers with lambda [n_x] (DEVICE).  Subsequent
 * HVPs return S^T grad^2 l(lambda) S W with S = [-J^{-1} G_p; I] (R16). */
int rh_set_multipliers(rh_ctx *ctx, const double *lambda, void *stream);

/* Newton-Raphson projection x(p) (Sec. 3.2; SURVEY.md 8(f)
 * NEXT-1): x_{k+1} = x_k - J_k^{-1} g(x_k, p).  x [n_x] DEVICE, in: initial
 * guess x_0, out: the solution; p [n_p] DEVICE.  Each step runs the state,
 * assembly and refactorization of rh_set_state at x_k and one device solve
 * J_k dx = g_k (block L sweep, separator S^-1, block U sweep on one column).
 * Stops `extra` steps after the first step with max|dx| <= tol (the oracle's
 * rule: quadratic convergence puts those steps on the rounding floor).  On
 * return the state (g, factors) is set at the final x, so rh_residual,
 * rh_reduced_gradient and the Hessian calls follow directly (multipliers are
 * invalidated).  iters (host, nullable): steps taken; resid (host, nullable):
 * max|g| at the final x.  Synchronizes `stream` once per step.
 * Errors: RH_E_SINGULAR (as rh_set_state), RH_E_NOCONV after maxit steps. */
int rh_newton(rh_ctx *ctx, double *x, const double *p, double tol, int32_t extra, int32_t maxit,
              int32_t *iters, double *resid, void *stream);

/* Batched reduced Hessian-vector products, Alg. 2:
 * W [n_p][ldw] (DEVICE, read), HW [n_p][ldhw] (DEVICE, written), N directions,
 * N <= ldw, N <= ldhw.  W and HW must not overlap.  Requires rh_set_state
 * and multipliers (rh_reduced_gradient or rh_set_multipliers): else RH_E_ORDER. */
int rh_hvp(rh_ctx *ctx, const double *W, int64_t ldw, double *HW, int64_t ldhw,
           int32_t N, void *stream);

/* Same as rh_hvp, and also writes the Alg. 2 intermediates in the natural x
 * order (DEVICE, [n_x][ldz] each, nullable): Z = -J^{-1} G_p W,
 * Yx = grad^2_xx l Z + grad^2_xp l W and Psi = -J^{-T} Yx.  For parity tests. */
int rh_hvp_stages(rh_ctx *ctx, const double *W, int64_t ldw, double *HW, int64_t ldhw,
                  int32_t N, double *Z, double *Yx, double *Psi, int64_t ldz, void *stream);

/* Columns j0 <= j < j1 of grad^2 F (Cartesian seeds e_j), computed in
 * batches of at most N.  Output layout selected by `transposed`:
 *   transposed = 0: H[i * ldh + (j - j0)] = (grad^2 F e_j)_i   ([n_p][ldh], ldh >= j1-j0)
 *   transposed = 1: H[(j - j0) * ldh + i] = (grad^2 F e_j)_i   ([j1-j0][ldh], ldh >= n_p)
 * (transposed = 1 makes a rank's column shard contiguous, so an all-gather
 * needs no reorder -- DESIGN.md "Multi-GPU"). DEVICE output. */
int rh_hessian_columns(rh_ctx *ctx, int32_t j0, int32_t j1, int32_t N, double *H,
                       int64_t ldh, int32_t transposed, void *stream);

/* Full reduced Hessian grad^2_pp F into H [n_p][n_p] (DEVICE, row i, column j:
 * component i of the HVP with e_j), ceil(n_p / N) batches (R10). */
int rh_full_hessian(rh_ctx *ctx, int32_t N, double *H, void *stream);

/* One pass of the whole path on DEVICE buffers: the same results as
 * rh_set_state(x, p), rh_reduced_gradient(grad_p) and
 * rh_hessian_columns(j0, j1, N, H, ldh, transposed), in one call.
 * x [n_x], p [n_p] (read), grad_p [n_p] (written, required), H as for
 * rh_hessian_columns (nullable when j0 == j1).  The first block sweep of the
 * first batches (it needs only the block factors) runs on an internal stream
 * while the separator is refactorized and inverted; `stream` waits for all of
 * it.  Synchronizes `stream` once, at the end, to read the pivot flag: on
 * RH_E_SINGULAR the outputs are invalid (as rh_set_state).
 * Errors: as rh_set_state and rh_hessian_columns. */
int rh_reduced_hessian(rh_ctx *ctx, const double *x, const double *p, int32_t j0, int32_t j1, int32_t N,
                       double *grad_p, double *H, int64_t ldh, int32_t transposed, void *stream);

/* End-to-end call with HOST buffers: copies x [n_x], p [n_p] to the device,
 * runs rh_reduced_hessian over all columns (batches of N), copies every
 * finished column block of H [n_p][n_p] back to the host while the later
 * batches compute, and grad_p [n_p] (nullable).  Blocking.
 * Pinned (page-locked) host buffers give the fastest copies. */
int rh_reduced_hessian_host(rh_ctx *ctx, const double *x, const double *p, int32_t N,
                            double *grad_p, double *H);

/* ---- Real-time tracking (section 6.3) ---- */

/* Replace the loads w = (Pd, Qd): DEVICE arrays [n_bus]
 * in the grid's bus order (either may be NULL = keep).  Invalidates the state:
 * call rh_set_state / rh_newton next.  Errors: RH_E_ORDER (no grid). */
int rh_set_loads(rh_ctx *ctx, const double *Pd, const double *Qd, void *stream);

/* Step 2 of the tracking algorithm, Eq. qp_rto: solve
 * (Hs + tau I) d = -g, Hs = (H + H^T)/2 (DESIGN.md R-T1), by a dense Cholesky
 * factorization on the device (blocked, fp64 tensor cores; dense.cu).
 * tau = 0 first; while a pivot is <= 0, tau = 1e-6, 2e-6, 4e-6, ... up to 64
 * attempts (R-T4).  DEVICE arrays: H [n][ldh] row-major (either triangle
 * order: only Hs is used), g [n], d [n] out (nullable), p [n] in/out
 * (nullable): on success p += alpha d.  tau / attempts: HOST out (nullable).
 * Needs no grid.  Blocking (one host sync per attempt).
 * Errors: RH_E_ARG (n < 0, ldh < n, NULL H/g), RH_E_NOTPD (64 attempts failed;
 * d and p untouched). */
int rh_dense_spd_solve(rh_ctx *ctx, int32_t n, const double *H, int64_t ldh, const double *g, double *d,
                       double *p, double alpha, double *tau, int32_t *attempts, void *stream);

/* One tracking update on the free controls [j0, j1) of p
 * (R-T2: [0, n_p) is the literal step; d is 0 outside the range):
 *   loads <- (Pd, Qd) (device [n_bus], NULL = keep);
 *   x <- x(p; w) by rh_newton from x (tol 1e-11, 2 extra steps, maxit 40);
 *   Step 1: grad_p [n_p] and the columns j0..j1-1 of H_t, TRANSPOSED into
 *           H [j1-j0][ldh >= n_p] (row k = column j0 + k), batches of N (Alg. 2);
 *   Step 2: H_ff d = -g_f by rh_dense_spd_solve on the [j0, j1) block,
 *           d [j1-j0] out, p[j0 + k] += alpha d[k].
 * x, p, grad_p, H, d: DEVICE.  info (HOST, nullable) [7]: Newton steps,
 * max|g(x, p)| after Newton, F(p_t; w_t), tau, Cholesky attempts,
 * Step 1 ms, Step 2 ms (CUDA events on `stream`).  The context's state is left
 * at (x(p_t; w_t), p_t).  Blocking.
 * Errors: as rh_newton, rh_reduced_hessian and rh_dense_spd_solve. */
int rh_tracking_step(rh_ctx *ctx, double *x, double *p, const double *Pd, const double *Qd, int32_t j0,
                     int32_t j1, int32_t N, double alpha, double *grad_p, double *H, int64_t ldh, double *d,
                     double *info, void *stream);

/* ---- Jacobians by column coloring + forward mode (
 *      SURVEY.md 8(f) NEXT-4) ---- */

/* Jacobian modes for rh_set_state / rh_newton / rh_reduced_hessian:
 * RH_JAC_ANALYTIC (default) assembles J and G_p from the closed-form partials;
 * RH_JAC_COLORED evaluates them the paper's way: the columns of [J | G_p] are
 * colored (greedy, column order, DESIGN.md R-C1..R-C3), one forward-mode tangent
 * per color is propagated through the residual, and J, G_p are decompressed from
 * the compressed product.  Same values up to rounding.  Invalidates the state. */
enum { RH_JAC_ANALYTIC = 0, RH_JAC_COLORED = 1 };
int rh_set_jacobian_mode(rh_ctx *ctx, int32_t mode);

/* The column coloring (host outputs): colors [n_x + n_p] (x columns, then p
 * columns; nullable), ncolors (nullable).  Needs a loaded grid. */
int rh_coloring(const rh_ctx *ctx, int32_t *colors, int32_t *ncolors);

/* Compressed Jacobian at the current state: JS [n_x][ncolors] (DEVICE,
 * row-major, rows in the natural x order = residual rows, R5) = [J | G_p] S,
 * S[j][color(j)] = 1, by forward-mode tangents.  Needs rh_set_state. */
int rh_compressed_jacobian(rh_ctx *ctx, double *JS, void *stream);

/* Number of CUDA kernels this library launched on ctx since creation
 * (bench accounting of "gpu_launches"). */
int64_t rh_launch_count(const rh_ctx *ctx);

/* Smallest static-pivot ratio |u_kk| / max_j |J_kj| (J's row k before
 * elimination) over every pivot of the most recent refactorization (block
 * rows, their tops, and the separator's Gauss-Jordan pivots; R15).
 * The factorization uses static diagonal pivots and reports RH_E_SINGULAR only
 * below 1e-14; ratios far below ~1e-8 flag an operating point where static
 * pivoting loses digits (the caller may then re-solve in the oracle or move
 * the state).  Host double *min_ratio.  One device read (synchronous).
 * Errors: RH_E_ORDER before a state, RH_E_NODEV on a host-only context. */
int rh_pivot_ratio(const rh_ctx *ctx, double *min_ratio);

/* Device-time breakdown of the most recent HVP batch when stage timing is
 * enabled (rh_set_timing(ctx, 1); adds one host sync per batch): ms_out[9]
 * receives the eight kernels of one Alg. 2 batch {blocks L (+SpMul),
 * separator L+U, blocks U, tensor projection, blocks U^T, separator U^T+L^T,
 * blocks L^T, SpMulAdd} and their total. */
int rh_set_timing(rh_ctx *ctx, int enable);
int rh_stage_times(const rh_ctx *ctx, float *ms_out);

#ifdef __cplusplus
}
#endif

#endif /* REDHESS_H */
