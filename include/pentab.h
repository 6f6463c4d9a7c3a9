/*
 * pentab.h — C ABI of libpentab.so, the B200-native (sm_100a) hot path of
 * Gloster's thesis (arxiv/paper_2101_06550): factor-once/solve-many batched
 * pentadiagonal and tridiagonal solves (cuPentBatch / cuThomasConstantBatch),
 * the cuSten-style 2D stencil, and the ADI Cahn–Hilliard time step.
 *
 * Citations "P:<lines>" are /root/reference/PAPER.md line numbers with the
 * thesis section / equation they fall in.
 *
 * Conventions (all entry points):
 *  - extern "C", plain pointers and sizes; every call returns an int status
 *    (PB_OK or a negative PB_E* code).  pb_last_error() gives details.
 *  - Data buffers are CALLER-OWNED.  Unless stated otherwise a buffer may be a
 *    device pointer (cudaMalloc / torch CUDA tensor) or a host pointer
 *    (pageable or pinned); host buffers are staged through a device scratch
 *    owned by the library, copies enqueued on `stream`.
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default
 *    stream).  All device work is enqueued on it; hot-path calls
 *    (pent_solve, tri_solve, stencil_apply, ch_adi_step with device buffers)
 *    never synchronise the host.
 *  - Handles are LIBRARY-OWNED and freed by the matching *_destroy.  The
 *    factors of a handle are read-only after *_factor; the solve's scratch
 *    (carry records, counters) is allocated per (handle, stream) under a
 *    per-handle lock, so concurrent solves with one handle -- from several
 *    host threads and/or on several streams -- are safe.  Destroying a
 *    handle while solves are queued on it is not (the caller orders that).
 *  - Inputs are never modified except the documented in-place outputs.
 *  - No CPU fallback: without a usable CUDA device every compute call
 *    returns PB_ECUDA.
 */
#ifndef PENTAB_H
#define PENTAB_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define PB_API __attribute__((visibility("default")))
#else
#define PB_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* status codes */
#define PB_OK 0
#define PB_EINVAL (-1)        /* bad size, pointer, layout, dtype or window   */
#define PB_EZEROPIVOT (-2)    /* |alpha_i| (or Thomas pivot) < 1e-14  */
#define PB_ESINGULAR (-3)     /* Navon 2x2 / Sherman–Morrison 1+v.z ~ 0       */
#define PB_ECUDA (-4)         /* CUDA launch / runtime error, or no device     */
#define PB_ENOMEM (-5)
#define PB_EUNSUPPORTED (-6)

/* element types of right-hand sides / solutions / grids */
#define PB_F64 0
#define PB_F32 1

/* batch layouts (P:1775-1777 interleaved; P:1955-1956 contiguous) */
#define PB_INTERLEAVED 0 /* entry i of system s at [i*M + s] (system-fastest)   */
#define PB_CONTIGUOUS 1  /* entry i of system s at [s*N + i] (one row/system)   */

/* stencil boundaries */
#define PB_NONPERIODIC 0
#define PB_PERIODIC 1

typedef struct pb_penta_s *pb_penta_t;
typedef struct pb_tri_s *pb_tri_t;

/* ------------------------------------------------------------------------
 * pent_factor — factor once (cuPentBatch factor / cuPentConstantBatch).
 * P:1686-1708 (§4.2.3, the 14-step LR list) and, if periodic, Navon's
 * reduction P:1498-1620 (§4.2.2, eq:xhat / eq:solve / eq:first_two).
 *
 *  batch      number of systems M the handle will solve (>= 0)
 *  n          unknowns per system N (>= 5; >= 7 if periodic)
 *  a..e       fp64 diagonals, each lhs_count*n values, interleaved
 *             [i*lhs_count + s]; row i of A is
 *             a_i x_{i-2} + b_i x_{i-1} + c_i x_i + d_i x_{i+1} + e_i x_{i+2}.
 *             Non-periodic: out-of-band a_0,a_1,b_0,d_{n-1},e_{n-2},e_{n-1}
 *             are ignored.  Periodic: the same entries are the wrap
 *             coefficients (row 1: a at column N-1, b at column N; row 2: a at
 *             column N; row N-1: e at column 1; row N: d at column 1, e at
 *             column 2), i.e. the matrix of P:1446-1453 when constant.
 *             Host or device pointers; read only.
 *  lhs_count  1 = one shared LHS for every system (cuPentConstantBatch,
 *             P:2204-2222); batch = one LHS per system (cuPentBatch).
 *  periodic   0 / 1
 *  dtype      PB_F64 or PB_F32: element type of the right-hand sides the
 *             handle solves (the factorisation is always computed in fp64 and
 *             rounded to dtype).
 *  stream     work (factor + precomputes) is enqueued here; pent_factor
 *             synchronises this stream once to report pivot errors.
 *  out        receives the handle (NULL on error).
 * Errors: PB_EINVAL (sizes/pointers/dtype), PB_EZEROPIVOT (system, row in
 * pb_last_error), PB_ESINGULAR (Navon 2x2 Schur complement), PB_ECUDA,
 * PB_ENOMEM.
 */
PB_API int pent_factor(int64_t batch, int64_t n, const double *a, const double *b, const double *c,
                const double *d, const double *e, int64_t lhs_count, int periodic, int dtype,
                void *stream, pb_penta_t *out);

/* pent_solve — solve A x = f for every system, in place (x overwrites rhs).
 * P:1710-1729 (forward g, back substitution x) and P:1585-1620 (periodic).
 *  rhs     batch*n elements of the handle's dtype in `layout`
 *          (PB_INTERLEAVED or PB_CONTIGUOUS); device or host pointer.
 * No numeric checks, no host sync for device buffers.  Errors: PB_EINVAL,
 * PB_ECUDA.                                                              */
PB_API int pent_solve(pb_penta_t h, void *rhs, int layout, void *stream);

/* pent_solve_many — `count` independent right-hand-side batches laid out
 * back to back (batch k at rhs + k*batch_stride elements), one launch.     */
PB_API int pent_solve_many(pb_penta_t h, void *rhs, int layout, int64_t count, int64_t batch_stride,
                    void *stream);

/* pent_refactor — re-factor a PER-SYSTEM handle (lhs_count == batch) in place
 * with new diagonals (cuPentBatchRewrite: matrices that change
 * every step).  a..e: DEVICE fp64 arrays laid out as for pent_factor.  Hot
 * path: no allocation after the first call, no host sync, and no pivot
 * report (a zero pivot yields non-finite solutions).  Shared-LHS handles:
 * PB_EUNSUPPORTED (factor a new one).                                      */
PB_API int pent_refactor(pb_penta_t h, const double *a, const double *b, const double *c, const double *d,
                         const double *e, void *stream);

/* pent_factor_uniform — a shared LHS whose diagonals are constants (a, b, c,
 * d, e) (cuPentUniformBatch; periodic: the wrap entries take the
 * same constants, the matrix of P:1446-1453).  Same semantics and errors as
 * pent_factor with lhs_count = 1.                                          */
PB_API int pent_factor_uniform(int64_t batch, int64_t n, double a, double b, double c, double d, double e,
                               int periodic, int dtype, void *stream, pb_penta_t *out);

/* pent_solve_strided — the general batched form (systems stored
 * interleaved, one per thread, or one after another).  System s of batch b
 * occupies rhs[b*outer_stride + s*inner_stride + i*row_stride], i = 0..n-1,
 * for s < n_inner and b < n_outer, solved in place.  Examples: interleaved
 * batch = {M, 1, 1, -, M}; a pitched sub-block of systems [s0, s0+m) of a
 * wider interleaved array with row pitch P = {m, 1, 1, -, P} at rhs + s0; the
 * ADI y-sweep of S grids = {n, 1, S, n*n, n}; contiguous rows (the x-sweep) =
 * {S*n, n, 1, -, 1}.  n_inner must equal the handle's batch for a per-system
 * LHS (any count for a shared LHS); strides > 0; n_outer <= 65535.
 * Interleaved (inner_stride 1) or contiguous (row_stride 1) forms with
 * 16-byte-aligned pitches take the fused streaming solve; other strides are
 * solved one thread per system.  Errors: PB_EINVAL, PB_ECUDA.             */
typedef struct {
    int64_t n_inner;      /* systems per batch                                  */
    int64_t inner_stride; /* elements between systems s and s+1                 */
    int64_t n_outer;      /* batches                                            */
    int64_t outer_stride; /* elements between batches b and b+1                 */
    int64_t row_stride;   /* elements between unknowns i and i+1 of one system  */
} pb_layout;
PB_API int pent_solve_strided(pb_penta_t h, void *rhs, const pb_layout *L, void *stream);

/* pent_solve_info — diagnostic: the configuration of the fused streaming
 * solve for one batch of the handle in `layout`; info points to 4 ints:
 * info[0] = thread-block cluster size CS (0 = no clusters), info[1] =
 * 64-row chunks per CTA, info[2] = clusters (CTAs) launched, info[3] =
 * kernel: 3 = two-pass streaming kernels (interleaved, 8 < N/64 <= 128:
 * P1 / segmented scan / P2, f re-read partly from L2), 2 = tiles held on
 * chip between the two sweeps (f read once; interleaved N <= 512,
 * contiguous N <= 16*8*64), 1 = two-pass cluster kernel, 0 = global-scan
 * kernel (N beyond the cluster span);
 * all -1 when the handle has no fused plan: per-system LHS, or chunk maps
 * of the factored LHS that grow (max-abs entry >= 1 over a 64-row chunk,
 * e.g. kappa ~ 1e6+) -- such handles are solved one thread per system, the
 * sequential order of P:1712-1724, because the chunked carry scan would
 * amplify rounding.                                                        */
PB_API int pent_solve_info(pb_penta_t h, int layout, int *info);

PB_API int pent_destroy(pb_penta_t h);

/* ------------------------------------------------------------------------
 * tri_factor / tri_solve / tri_destroy — Thomas algorithm with a shared or
 * per-system LHS (cuThomasConstantBatch), P:2239-2280 (§5.3.1; the printed
 * back substitution is corrected to x_i = dhat_i - chat_i x_{i+1}), and for
 * periodic systems Sherman–Morrison, P:2318-2385 (§5.3.3; A'z = u once).
 *  a,b,c   fp64 sub/main/super diagonals, lhs_count*n, interleaved.
 *          Periodic corners: a_0 at (1, N), c_{n-1} at (N, 1).  n >= 3.
 * Errors as pent_*; 1 + v.z ~ 0 -> PB_ESINGULAR.                          */
PB_API int tri_factor(int64_t batch, int64_t n, const double *a, const double *b, const double *c,
               int64_t lhs_count, int periodic, int dtype, void *stream, pb_tri_t *out);
PB_API int tri_solve(pb_tri_t h, void *rhs, int layout, void *stream);
PB_API int tri_solve_strided(pb_tri_t h, void *rhs, const pb_layout *L, void *stream);
/* tri_refactor / tri_factor_uniform: as pent_refactor / pent_factor_uniform
 * (the CN diffusion matrix (-s, 1+2s, -s)).                  */
PB_API int tri_refactor(pb_tri_t h, const double *a, const double *b, const double *c, void *stream);
PB_API int tri_factor_uniform(int64_t batch, int64_t n, double a, double b, double c, int periodic, int dtype,
                              void *stream, pb_tri_t *out);
PB_API int tri_destroy(pb_tri_t h);

/* ------------------------------------------------------------------------
 * stencil_apply — cuSten Compute2D{X,Y,XY}{p,np} with linear weights,
 * P:947-983 (§3.3) and P:1091-1101.
 *  g        grid descriptor: batch of ny x nx grids, row-major [b][j][i]
 *           (i = x fastest), element type g->dtype.
 *  in, out  device or host pointers, must not alias ("the same memory
 *           cannot be used for both").
 *  w        window: `left`/`right` points in i, `top` rows above (j-top) and
 *           `bottom` rows below.  X if top = bottom = 0, Y if left = right =
 *           0, XY (corners included) otherwise.
 *  weights  HOST array of (top+bottom+1)*(left+right+1) fp64 weights,
 *           row-major from the top-left, "left to right in i, row by row in
 *           j"; at most 15 x 15.
 *  boundary PB_PERIODIC (wrap both axes) or PB_NONPERIODIC (cells whose
 *           window leaves the grid are left untouched in `out`).
 * Errors: PB_EINVAL (aliasing, extents >= grid size, > 15x15), PB_ECUDA.   */
typedef struct {
    int64_t batch, ny, nx;
    int dtype;
} pb_grid;
typedef struct {
    int left, right, top, bottom;
} pb_window;
PB_API int stencil_apply(const pb_grid *g, const void *in, void *out, const pb_window *w,
                  const double *weights, int boundary, void *stream);

/* ------------------------------------------------------------------------
 * ch_adi_step — nsteps of the ADI Cahn–Hilliard scheme, Eq 3.1
 * (§3.5.1):
 *   L_x w = -2/3 (C^n - C^{n-1}) - 2/3 dt D gamma grad^4 Cbar + 2/3 D dt grad^2 (C^3 - C)^n
 *   L_y v = w ;  C^{n+1} = Cbar + v ;  Cbar = 2 C^n - C^{n-1}
 *   L_x = I + 2/3 D gamma dt d_xxxx  (cyclic penta (s,-4s,1+6s,-4s,s), s = 2/3 D gamma dt/dx^4)
 * with the readings of DESIGN.md §3 (dx = L/n; 13-point biharmonic with the
 * Fig 3.1 cross stencil; 5-point Laplacian; D*gamma on the explicit grad^4).
 *  s->c_cur, s->c_prev : device pointers to sims*n*n elements ([sim][j][i]);
 *       the caller initialises both to C^0.  On return they point
 *       to the newest / previous level (buffers rotate by pointer swap).
 *  s->work : device scratch of ch_workspace_bytes() bytes (fp64 R -> w -> v,
 *       sims*n*n doubles for either state dtype), caller-owned.
 *  All three buffers 16-byte aligned.
 * One step = 4 launches: RHS stencil, x-sweep (fused solve, contiguous rows),
 * y-sweep (fused solve, interleaved columns, count = sims), combine.
 *  p : D, gamma, L (square periodic domain of side L).
 * L_x = L_y is factored once and cached per (n, dt, D, gamma, L, dtype).
 * Errors: PB_EINVAL (n < 8, bad pointers), PB_ECUDA.                      */
typedef struct {
    int64_t sims, n;
    int dtype;
    void *c_cur, *c_prev, *work;
} pb_ch_state;
typedef struct {
    double D, gamma, L;
} pb_ch_params;
PB_API int ch_workspace_bytes(int64_t sims, int64_t n, int dtype, size_t *bytes);
PB_API int ch_adi_step(pb_ch_state *s, double dt, const pb_ch_params *p, int64_t nsteps, void *stream);

/* ------------------------------------------------------------------------
 * Coarsening statistics (thesis §7.1-7.5, experiments on
 * batches of CH / Cahn–Hilliard–Cook simulations).
 *
 * ch_adi_step_cook — nsteps of Eq 3.1 for the Cahn–Hilliard–Cook equation
 * (P:4496-4509): as ch_adi_step, with the thermal noise
 *   eta_ij = sqrt(sigma / (dx^2 dt)) (div rho)_ij
 * added to the RHS as + 2/3 dt eta^n (reading r25).  rho = (rho_x, rho_y) is
 * a fresh N(0,1) vector field every step: one Box–Muller pair per cell from
 * two uniforms of the counter-based splitmix64 hash of (seed, step, sim,
 * cell) (reading r26; the same generator as the CPU oracle's); the
 * divergence by periodic central differences.  noise->step0 is the step
 * index of the first of the nsteps (steps step0 .. step0+nsteps-1 draw
 * distinct fields).  sigma = 0 is ch_adi_step exactly.
 * Errors: as ch_adi_step; PB_EINVAL for sigma < 0.                        */
typedef struct {
    double sigma;     /* noise intensity (P:4509 uses 1e-14) */
    uint64_t seed;
    int64_t step0;
} pb_ch_noise;
PB_API int ch_adi_step_cook(pb_ch_state *s, double dt, const pb_ch_params *p, const pb_ch_noise *noise,
                            int64_t nsteps, void *stream);

/* ch_free_energy — F of P:819-825 per simulation, on the device (reading
 * r24: bulk 1/4 (C^2-1)^2, the form the printed dF/dt belongs to):
 *   F_h = dx^2 sum_ij [ 1/4 (C_ij^2 - 1)^2
 *                       + 1/2 gamma ((C_{i+1,j}-C_ij)^2 + (C_{i,j+1}-C_ij)^2) / dx^2 ]
 * periodic forward differences, dx = L/n, accumulated in fp64 in a fixed
 * order (deterministic).  s: as ch_adi_step (reads s->c_cur only; uses no
 * workspace); F: device, s->sims doubles, written.  p->D is unused.
 * Errors: PB_EINVAL, PB_ECUDA.                                             */
PB_API int ch_free_energy(const pb_ch_state *s, const pb_ch_params *p, double *F, void *stream);

/* ch_coarsening_beta — the growth rate beta = -(t/F) dF/dt of nt
 * samples F[k][sim] taken at times t[k] (reading r27: central differences in
 * t, one-sided at the two ends).  t: device, nt doubles, increasing; F, beta:
 * device, nt*sims doubles.  The thesis then keeps 10 < t < 100, beta < 1
 * (P:3580-3581).  Errors: PB_EINVAL (nt < 2), PB_ECUDA.                   */
PB_API int ch_coarsening_beta(int64_t nt, int64_t sims, const double *t, const double *F, double *beta,
                              void *stream);

/* ------------------------------------------------------------------------
 * ch1d_step — nsteps of the batched 1D Cahn–Hilliard scheme, thesis §6.2
 * (eq6:1Dnumerical):
 *   (I + dt gamma d_xxxx) C^{n+1} = C^n + dt d_xx (C^3 - C)^n,  D = 1,
 * second-order differences on a periodic grid of n points, dx = L/n (r1):
 * the cyclic pentadiagonal (s, -4s, 1+6s, -4s, s), s = gamma dt/dx^4, and
 * f_i = C_i + alpha (N_{i-1} - 2 N_i + N_{i+1}), alpha = dt/dx^2,
 * N = C^3 - C (the +C_i^n term the printed f_i drops, reading r12).
 *  s->c     device, batch*n elements, interleaved [i*batch + s] (system
 *           fastest): C^n on entry, C^{n+nsteps} on return.
 *  s->work  device scratch of the same size; c and work swap each step
 *           (on return s->c points at the newest level).
 *  batch must be a multiple of 32; both buffers 16-byte aligned.
 * The matrix is factored once and cached per (n, dt, gamma, L, dtype).
 * One kernel launch per step; no host sync.
 * Errors: PB_EINVAL (sizes, alignment, pointers), PB_ECUDA.               */
typedef struct {
    int64_t batch, n;
    int dtype;
    void *c, *work;
} pb_ch1d_state;
typedef struct {
    double gamma, L;
} pb_ch1d_params;
PB_API int ch1d_step(pb_ch1d_state *s, double dt, const pb_ch1d_params *p, int64_t nsteps, void *stream);

/* ------------------------------------------------------------------------
 * Row-partitioned ADI step (configs[4]: one n x n grid over P ranks,
 * SURVEY §8(e)).  Rank r owns rows [r n/P, (r+1) n/P); one step of Eq 3.1
 * is, per rank (the orchestration and the two all-to-all
 * transposes live in paper_2101_06550_b200/dist.py):
 *   halo rows -> ch_dist_pass_a (RHS + x-sweep) -> ch_dist_pack ->
 *   all-to-all -> ch_dist_ysweep (y-sweep on the rank's n/P columns, interleaved)
 *   -> all-to-all -> ch_dist_combine (C^{n+1} = 2C^n - C^{n-1} + v).
 * The x-then-y order is the thesis's (reading r18); results equal the
 * single-grid ch_adi_step up to rounding.
 *
 * ch_dist_pass_a: cn_ext, cm_ext: device, (rows + 4) x n, rows 2..rows+1 the
 *   rank's rows, rows 0-1 / rows+2..rows+3 the two halo rows of the previous /
 *   next rank (periodic in j across ranks, periodic in i within the row).
 *   w: device fp64 rows x n (16-byte aligned, n even), receives L_x^{-1} R.
 *   dt, p as ch_adi_step; dtype = the element type of cn_ext / cm_ext.
 * ch_dist_pack: fp64 w (rows x n) -> packed [parts][rows][n/parts] (the send
 *   layout of the transpose: column block q contiguous).  n % parts == 0.
 * ch_dist_combine: cm_ext interior rows <- 2 cn_ext - cm_ext + v (dtype of
 *   cn_ext / cm_ext), with fp64 v in the receive layout [parts][rows][n/parts]
 *   (block q = columns of rank q).
 * All buffers are caller-owned device memory; work is enqueued on stream.
 * Errors: PB_EINVAL (sizes, pointers, dtype), PB_ECUDA.                    */
PB_API int ch_dist_pass_a(int64_t rows, int64_t n, int dtype, const void *cn_ext, const void *cm_ext, void *w,
                          double dt, const pb_ch_params *p, void *stream);
PB_API int ch_dist_pack(int64_t rows, int64_t n, int64_t parts, const void *w, void *packed, void *stream);
/* ch_dist_ysweep: the y-sweep L_y v = w of the rank's column block,
 *   in place: cols is fp64 [n][ncols] interleaved (ncols systems of length n,
 *   the receive layout of the first all-to-all), solved with the cyclic L_y
 *   of (n, dt, D, gamma, L) factored once and cached.  ncols must be even and
 *   cols 16-byte aligned (PB_EINVAL otherwise).                           */
PB_API int ch_dist_ysweep(int64_t ncols, int64_t n, void *cols, double dt, const pb_ch_params *p, void *stream);
PB_API int ch_dist_combine(int64_t rows, int64_t n, int64_t parts, int dtype, const void *cn_ext, void *cm_ext,
                           const void *v_packed, void *stream);

/* ------------------------------------------------------------------------
 * diagnostics */
/* Last error of the calling thread: code, system/row of a pivot failure,
 * message (NUL-terminated, truncated to len).  Returns the code.          */
PB_API int pb_last_error(int64_t *sys, int64_t *row, char *msg, size_t len);
/* Number of kernels this library has launched since load (for the bench's
 * gpu_launches count); resettable.                                        */
PB_API int64_t pb_launch_count(void);
PB_API void pb_reset_launch_count(void);
/* 0 if a CUDA device is usable, else PB_ECUDA. */
PB_API int pb_device_ok(void);

#ifdef __cplusplus
}
#endif
#endif /* PENTAB_H */
