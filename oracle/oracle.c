/*
 * oracle.c — plain, slow, obviously-correct CPU ORACLE for the hot path of
 * Gloster's thesis (arxiv/paper_2101_06550): batched penta/tri solves, the
 * cuSten-style stencil and the ADI Cahn–Hilliard step.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * It shares no code, header, table or constant generator with the CUDA
 * product path (paper_2101_06550_b200/), and neither includes the other.
 *
 * Everything is fp64, scalar, single-threaded, written in the paper's order
 * and notation.  Indices are 0-based in code; comments quote the paper's
 * 1-based steps.  "P:<lines>" cites /root/reference/PAPER.md line numbers.
 *
 * Readings of the paper (r1..r27 in DESIGN.md §3) used here:
 *   r4  4th-difference stencil is (1,-4,6,-4,1)/dx^4 (P:321 printed wrong)
 *   r5  the explicit grad^4 Cbar term of Eq 3.1 carries D*gamma
 *   r6  Cbar^{n+1} = 2C^n - C^{n-1}
 *   r8  Laplacian is the 5-point 2nd-order stencil
 *   r9  biharmonic = dx^4 + 2 dx^2dy^2 + dy^4 with the Fig 3.1 cross stencil
 *   r13 Thomas back-substitution x_i = dhat_i - chat_i x_{i+1} (P:2274 wrong)
 *   r14 Sherman–Morrison second solve is A'z = u (P:2378 says A'x = u)
 *   r16 |alpha_i| < 1e-14 is a zero pivot; no pivoting
 *
 * Parity status of every function: pinned (see tests/test_oracle_*.py).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_OK 0
#define ORC_EINVAL (-1)
#define ORC_EZEROPIVOT (-2)
#define ORC_ESINGULAR (-3)
#define ORC_ENOMEM (-5)

static const double ORC_PIVOT_TOL = 1e-14; /* r16 */

/* ------------------------------------------------------------------------ */
/* Pentadiagonal LR factorisation, P:1686-1708 (§4.2.3, the 14-step list).   */
/* Row i of A is  a_i x_{i-2} + b_i x_{i-1} + c_i x_i + d_i x_{i+1} + e_i x_{i+2}.
 * Out-of-band entries (a_0,a_1,b_0,d_{n-1},e_{n-2},e_{n-1}) are ignored.      */
int orc_penta_factor(int64_t n, const double *a, const double *b, const double *c,
                     const double *d, const double *e, double *alpha, double *beta,
                     double *gamma, double *delta, double *eps, int64_t *bad_row)
{
    if (n < 5) return ORC_EINVAL;
    for (int64_t i = 0; i < n; i++) { beta[i] = 0; gamma[i] = 0; delta[i] = 0; eps[i] = 0; }
#define PIV(i)                                                        \
    do {                                                              \
        if (!(fabs(alpha[i]) >= ORC_PIVOT_TOL)) {                     \
            if (bad_row) *bad_row = (i);                              \
            return ORC_EZEROPIVOT;                                    \
        }                                                             \
    } while (0)
    /* 1. alpha_1 = c_1 ; 2. gamma_1 = d_1/alpha_1 ; 3. delta_1 = e_1/alpha_1 */
    alpha[0] = c[0];
    PIV(0);
    gamma[0] = d[0] / alpha[0];
    delta[0] = e[0] / alpha[0];
    /* 4. beta_2 = b_2 ; 5. alpha_2 = c_2 - beta_2 gamma_1 ;
       6. gamma_2 = (d_2 - beta_2 delta_1)/alpha_2 ; 7. delta_2 = e_2/alpha_2 */
    beta[1] = b[1];
    alpha[1] = c[1] - beta[1] * gamma[0];
    PIV(1);
    gamma[1] = (d[1] - beta[1] * delta[0]) / alpha[1];
    delta[1] = e[1] / alpha[1];
    /* 8. for i = 3..N-2 (1-based) */
    for (int64_t i = 2; i <= n - 3; i++) {
        beta[i] = b[i] - a[i] * gamma[i - 2];
        alpha[i] = c[i] - a[i] * delta[i - 2] - beta[i] * gamma[i - 1];
        PIV(i);
        gamma[i] = (d[i] - beta[i] * delta[i - 1]) / alpha[i];
        delta[i] = e[i] / alpha[i];
    }
    /* 9-11. row N-1 */
    {
        int64_t i = n - 2;
        beta[i] = b[i] - a[i] * gamma[i - 2];
        alpha[i] = c[i] - a[i] * delta[i - 2] - beta[i] * gamma[i - 1];
        PIV(i);
        gamma[i] = (d[i] - beta[i] * delta[i - 1]) / alpha[i];
    }
    /* 12-13. row N */
    {
        int64_t i = n - 1;
        beta[i] = b[i] - a[i] * gamma[i - 2];
        alpha[i] = c[i] - a[i] * delta[i - 2] - beta[i] * gamma[i - 1];
        PIV(i);
    }
    /* 14. epsilon_i = a_i for all i */
    for (int64_t i = 0; i < n; i++) eps[i] = (i >= 2) ? a[i] : 0.0;
#undef PIV
    return ORC_OK;
}

/* Forward (g) and back substitution (x).  x may alias f. */
void orc_penta_solve(int64_t n, const double *alpha, const double *beta, const double *gamma,
                     const double *delta, const double *eps, const double *f, double *x)
{
    double *g = (double *)malloc(sizeof(double) * (size_t)n);
    /* 1. g_1 = f_1/alpha_1 ; 2. g_2 = (f_2 - beta_2 g_1)/alpha_2 */
    g[0] = f[0] / alpha[0];
    g[1] = (f[1] - beta[1] * g[0]) / alpha[1];
    /* 3. g_i = (f_i - eps_i g_{i-2} - beta_i g_{i-1})/alpha_i, i = 3..N */
    for (int64_t i = 2; i < n; i++) g[i] = (f[i] - eps[i] * g[i - 2] - beta[i] * g[i - 1]) / alpha[i];
    /* 1. x_N = g_N ; 2. x_{N-1} = g_{N-1} - gamma_{N-1} x_N */
    x[n - 1] = g[n - 1];
    x[n - 2] = g[n - 2] - gamma[n - 2] * x[n - 1];
    /* 3. x_i = g_i - gamma_i x_{i+1} - delta_i x_{i+2}, i = N-2..1 */
    for (int64_t i = n - 3; i >= 0; i--) x[i] = g[i] - gamma[i] * x[i + 1] - delta[i] * x[i + 2];
    free(g);
}

/* ------------------------------------------------------------------------ */
/* Cyclic pentadiagonal solve by Navon's reduction, P:1498-1620 (§4.2.2).     */
/* The wrap coefficients are the out-of-band entries of the same diagonals:
 *   row 1:   a_1 at column N-1, b_1 at column N
 *   row 2:   a_2 at column N
 *   row N-1: e_{N-1} at column 1
 *   row N:   d_N at column 1, e_N at column 2
 * which for constant diagonals is exactly the matrix of P:1446-1453.         */
typedef struct {
    int64_t n;   /* full size N; core size m = N-2 */
    double *alpha, *beta, *gamma, *delta, *eps; /* LR of E (m) */
    double *k;   /* m x 2, row-major: E X + k (x_{N-1},x_N) = fhat        */
    double *hT;  /* 2 x m, row-major: h^T X + B (x_{N-1},x_N) = (f_{N-1},f_N) */
    double *W;   /* m x 2 : W = E^{-T} h = (h^T E^{-1})^T         */
    double Sinv[4]; /* [B - h^T E^{-1} k]^{-1}, row-major 2x2 (eq:first_two) */
} orc_cpenta;

static void orc_cpenta_free(orc_cpenta *s)
{
    free(s->alpha); free(s->beta); free(s->gamma); free(s->delta); free(s->eps);
    free(s->k); free(s->hT); free(s->W);
    memset(s, 0, sizeof(*s));
}

static int orc_cpenta_init(orc_cpenta *s, int64_t n, const double *a, const double *b,
                           const double *c, const double *d, const double *e, int64_t *bad_row)
{
    memset(s, 0, sizeof(*s));
    if (n < 7) return ORC_EINVAL;
    int64_t m = n - 2;
    s->n = n;
    s->alpha = malloc(sizeof(double) * m); s->beta = malloc(sizeof(double) * m);
    s->gamma = malloc(sizeof(double) * m); s->delta = malloc(sizeof(double) * m);
    s->eps = malloc(sizeof(double) * m);
    s->k = calloc((size_t)(2 * m), sizeof(double));
    s->hT = calloc((size_t)(2 * m), sizeof(double));
    s->W = calloc((size_t)(2 * m), sizeof(double));
    /* E = A with the last two rows and columns removed: the same
       diagonals restricted to rows 1..N-2; its out-of-band entries are ignored
       by the factorisation. */
    int rc = orc_penta_factor(m, a, b, c, d, e, s->alpha, s->beta, s->gamma, s->delta, s->eps, bad_row);
    if (rc) { orc_cpenta_free(s); return rc; }
    /* k: columns N-1, N of rows 1..N-2. */
    s->k[0 * 2 + 0] = a[0];          /* row 1, col N-1 */
    s->k[0 * 2 + 1] = b[0];          /* row 1, col N   */
    s->k[1 * 2 + 1] = a[1];          /* row 2, col N   */
    s->k[(m - 2) * 2 + 0] = e[m - 2]; /* row N-3, col N-1 */
    s->k[(m - 1) * 2 + 0] = d[m - 1]; /* row N-2, col N-1 */
    s->k[(m - 1) * 2 + 1] = e[m - 1]; /* row N-2, col N   */
    /* h^T: rows N-1, N restricted to columns 1..N-2. */
    s->hT[0 * m + 0] = e[n - 2];      /* row N-1, col 1   */
    s->hT[0 * m + (m - 2)] = a[n - 2];/* row N-1, col N-3 */
    s->hT[0 * m + (m - 1)] = b[n - 2];/* row N-1, col N-2 */
    s->hT[1 * m + 0] = d[n - 1];      /* row N, col 1     */
    s->hT[1 * m + 1] = e[n - 1];      /* row N, col 2     */
    s->hT[1 * m + (m - 1)] = a[n - 1];/* row N, col N-2   */
    /* W = E^{-T} h: "(E^{-1})^T h = (h^T E^{-1})^T".  E^T is again
       pentadiagonal; factor it with the same 14-step algorithm. */
    {
        double *ta = calloc(m, sizeof(double)), *tb = calloc(m, sizeof(double)),
               *tc = calloc(m, sizeof(double)), *td = calloc(m, sizeof(double)),
               *te = calloc(m, sizeof(double));
        double *fa = malloc(sizeof(double) * m), *fb = malloc(sizeof(double) * m),
               *fg = malloc(sizeof(double) * m), *fd = malloc(sizeof(double) * m),
               *fe = malloc(sizeof(double) * m);
        double *rhs = malloc(sizeof(double) * m), *sol = malloc(sizeof(double) * m);
        /* (E^T)_{i,j} = E_{j,i}: row i of E^T has a'_i = e_{i-2}, b'_i = d_{i-1},
           c'_i = c_i, d'_i = b_{i+1}, e'_i = a_{i+2}. */
        for (int64_t i = 0; i < m; i++) {
            tc[i] = c[i];
            if (i >= 2) ta[i] = e[i - 2];
            if (i >= 1) tb[i] = d[i - 1];
            if (i + 1 < m) td[i] = b[i + 1];
            if (i + 2 < m) te[i] = a[i + 2];
        }
        rc = orc_penta_factor(m, ta, tb, tc, td, te, fa, fb, fg, fd, fe, bad_row);
        if (!rc) {
            for (int col = 0; col < 2; col++) {
                for (int64_t i = 0; i < m; i++) rhs[i] = s->hT[col * m + i]; /* column col of h */
                orc_penta_solve(m, fa, fb, fg, fd, fe, rhs, sol);
                for (int64_t i = 0; i < m; i++) s->W[i * 2 + col] = sol[i];
            }
        }
        free(ta); free(tb); free(tc); free(td); free(te);
        free(fa); free(fb); free(fg); free(fd); free(fe); free(rhs); free(sol);
        if (rc) { orc_cpenta_free(s); return rc; }
    }
    /* S = B - h^T E^{-1} k = B - W^T k ; B = [[c_{N-1}, d_{N-1}], [b_N, c_N]] */
    {
        double S[4] = {c[n - 2], d[n - 2], b[n - 1], c[n - 1]};
        for (int r = 0; r < 2; r++)
            for (int q = 0; q < 2; q++) {
                double acc = 0;
                for (int64_t i = 0; i < m; i++) acc += s->W[i * 2 + r] * s->k[i * 2 + q];
                S[r * 2 + q] -= acc;
            }
        double det = S[0] * S[3] - S[1] * S[2];
        if (!(fabs(det) >= ORC_PIVOT_TOL)) { orc_cpenta_free(s); return ORC_ESINGULAR; }
        s->Sinv[0] = S[3] / det;  s->Sinv[1] = -S[1] / det;
        s->Sinv[2] = -S[2] / det; s->Sinv[3] = S[0] / det;
    }
    return ORC_OK;
}

/* One cyclic solve: "we solve for the final two unknowns first (eq:first_two),
   then substitute into eq:solve and invert".  x may alias f. */
static void orc_cpenta_solve(const orc_cpenta *s, const double *f, double *x)
{
    int64_t n = s->n, m = n - 2;
    /* r = h^T E^{-1} fhat = W^T fhat */
    double r0 = 0, r1 = 0;
    for (int64_t i = 0; i < m; i++) { r0 += s->W[i * 2 + 0] * f[i]; r1 += s->W[i * 2 + 1] * f[i]; }
    double q0 = f[n - 2] - r0, q1 = f[n - 1] - r1;
    double xn1 = s->Sinv[0] * q0 + s->Sinv[1] * q1; /* x_{N-1} */
    double xn = s->Sinv[2] * q0 + s->Sinv[3] * q1;  /* x_N     */
    /* Xhat = E^{-1}[fhat - k (x_{N-1}, x_N)] */
    double *t = malloc(sizeof(double) * m);
    for (int64_t i = 0; i < m; i++) t[i] = f[i] - s->k[i * 2 + 0] * xn1 - s->k[i * 2 + 1] * xn;
    orc_penta_solve(m, s->alpha, s->beta, s->gamma, s->delta, s->eps, t, x);
    x[n - 2] = xn1;
    x[n - 1] = xn;
    free(t);
}

/* ------------------------------------------------------------------------ */
/* Thomas algorithm, P:2239-2280 (§5.3.1), back-substitution corrected (r13). */
int orc_tri_factor(int64_t n, const double *a, const double *b, const double *c, double *chat,
                   int64_t *bad_row)
{
    if (n < 3) return ORC_EINVAL;
    /* chat_1 = c_1/b_1 ; chat_i = c_i/(b_i - a_i chat_{i-1}) */
    if (!(fabs(b[0]) >= ORC_PIVOT_TOL)) { if (bad_row) *bad_row = 0; return ORC_EZEROPIVOT; }
    chat[0] = c[0] / b[0];
    for (int64_t i = 1; i < n; i++) {
        double den = b[i] - a[i] * chat[i - 1];
        if (!(fabs(den) >= ORC_PIVOT_TOL)) { if (bad_row) *bad_row = i; return ORC_EZEROPIVOT; }
        chat[i] = (i < n - 1) ? c[i] / den : 0.0;
    }
    return ORC_OK;
}

void orc_tri_solve(int64_t n, const double *a, const double *b, const double *chat, const double *d,
                   double *x)
{
    double *dh = malloc(sizeof(double) * n);
    /* dhat_1 = d_1/b_1 ; dhat_i = (d_i - a_i dhat_{i-1})/(b_i - a_i chat_{i-1}) */
    dh[0] = d[0] / b[0];
    for (int64_t i = 1; i < n; i++) dh[i] = (d[i] - a[i] * dh[i - 1]) / (b[i] - a[i] * chat[i - 1]);
    /* x_N = dhat_N ; x_i = dhat_i - chat_i x_{i+1}  (r13) */
    x[n - 1] = dh[n - 1];
    for (int64_t i = n - 2; i >= 0; i--) x[i] = dh[i] - chat[i] * x[i + 1];
    free(dh);
}

/* Cyclic tridiagonal by Sherman–Morrison, P:2318-2385 (§5.3.3).  Corners are
   the out-of-band entries: a_1 at (1, N), c_N at (N, 1).  u = (-b_1,0..,c_N),
   v = (1,0..,-a_1/b_1), A' = A - u v^T has A'_11 = 2 b_1, A'_NN = b_N + a_1 c_N/b_1. */
typedef struct {
    int64_t n;
    double *a, *bp, *c, *chat, *z;
    double v_last; /* v_N = -a_1/b_1 ; v_1 = 1 */
    double denom;  /* 1 + v.z */
} orc_ctri;

static void orc_ctri_free(orc_ctri *s)
{
    free(s->a); free(s->bp); free(s->c); free(s->chat); free(s->z);
    memset(s, 0, sizeof(*s));
}

static int orc_ctri_init(orc_ctri *s, int64_t n, const double *a, const double *b, const double *c,
                         int64_t *bad_row)
{
    memset(s, 0, sizeof(*s));
    if (n < 3) return ORC_EINVAL;
    if (!(fabs(b[0]) >= ORC_PIVOT_TOL)) { if (bad_row) *bad_row = 0; return ORC_EZEROPIVOT; }
    s->n = n;
    s->a = malloc(sizeof(double) * n); s->bp = malloc(sizeof(double) * n);
    s->c = malloc(sizeof(double) * n); s->chat = malloc(sizeof(double) * n);
    s->z = malloc(sizeof(double) * n);
    double top = a[0], bot = c[n - 1];
    for (int64_t i = 0; i < n; i++) { s->a[i] = (i > 0) ? a[i] : 0.0; s->bp[i] = b[i]; s->c[i] = (i < n - 1) ? c[i] : 0.0; }
    s->bp[0] = 2.0 * b[0];                       /* A'_11 = 2b          */
    s->bp[n - 1] = b[n - 1] + top * bot / b[0];  /* A'_NN = b + ac/b    */
    int rc = orc_tri_factor(n, s->a, s->bp, s->c, s->chat, bad_row);
    if (rc) { orc_ctri_free(s); return rc; }
    double *u = calloc(n, sizeof(double));
    u[0] = -b[0];
    u[n - 1] = bot;
    orc_tri_solve(n, s->a, s->bp, s->chat, u, s->z); /* A' z = u, once (r14) */
    free(u);
    s->v_last = -top / b[0];
    s->denom = 1.0 + (s->z[0] + s->v_last * s->z[n - 1]);
    if (!(fabs(s->denom) >= ORC_PIVOT_TOL)) { orc_ctri_free(s); return ORC_ESINGULAR; }
    return ORC_OK;
}

static void orc_ctri_solve(const orc_ctri *s, const double *d, double *x)
{
    int64_t n = s->n;
    double *y = malloc(sizeof(double) * n);
    orc_tri_solve(n, s->a, s->bp, s->chat, d, y);   /* A' y = d */
    double vy = y[0] + s->v_last * y[n - 1];
    double coef = vy / s->denom;                    /* (v.y)/(1+v.z) */
    for (int64_t i = 0; i < n; i++) x[i] = y[i] - coef * s->z[i];
    free(y);
}

/* ------------------------------------------------------------------------ */
/* Batched drivers (P:1775-1777 interleaved; P:1955-1956 contiguous).        */
/* layout 0 = interleaved x[i*M + s]; layout 1 = contiguous x[s*N + i].
 * lhs_count 1 = one shared LHS (cuPentConstantBatch), or M.
 * LHS diagonals are given interleaved ([i*lhs_count + s]), like the RHS.     */
static inline int64_t idx_of(int layout, int64_t n, int64_t m, int64_t i, int64_t s)
{
    return layout == 0 ? i * m + s : s * n + i;
}

static void gather_lhs(int64_t n, int64_t lhs_count, int64_t s, const double *src, double *dst)
{
    for (int64_t i = 0; i < n; i++) dst[i] = src[i * lhs_count + s];
}

int orc_penta_batch_solve(int64_t n, int64_t m, int layout, int64_t lhs_count, int periodic,
                          const double *a, const double *b, const double *c, const double *d,
                          const double *e, const double *rhs, double *x, int64_t *bad_sys,
                          int64_t *bad_row)
{
    if (n < (periodic ? 7 : 5) || m < 0 || (lhs_count != 1 && lhs_count != m)) return ORC_EINVAL;
    if (m == 0) return ORC_OK;
    double *la = malloc(sizeof(double) * n), *lb = malloc(sizeof(double) * n),
           *lc = malloc(sizeof(double) * n), *ld = malloc(sizeof(double) * n),
           *le = malloc(sizeof(double) * n);
    double *al = malloc(sizeof(double) * n), *be = malloc(sizeof(double) * n),
           *ga = malloc(sizeof(double) * n), *de = malloc(sizeof(double) * n),
           *ep = malloc(sizeof(double) * n);
    double *f = malloc(sizeof(double) * n), *sol = malloc(sizeof(double) * n);
    orc_cpenta cp;
    memset(&cp, 0, sizeof(cp));
    int rc = ORC_OK;
    int64_t factored_for = -1;
    for (int64_t s = 0; s < m && rc == ORC_OK; s++) {
        int64_t ls = (lhs_count == 1) ? 0 : s;
        if (ls != factored_for) {
            gather_lhs(n, lhs_count, ls, a, la); gather_lhs(n, lhs_count, ls, b, lb);
            gather_lhs(n, lhs_count, ls, c, lc); gather_lhs(n, lhs_count, ls, d, ld);
            gather_lhs(n, lhs_count, ls, e, le);
            if (periodic) {
                orc_cpenta_free(&cp);
                rc = orc_cpenta_init(&cp, n, la, lb, lc, ld, le, bad_row);
            } else {
                rc = orc_penta_factor(n, la, lb, lc, ld, le, al, be, ga, de, ep, bad_row);
            }
            if (rc) { if (bad_sys) *bad_sys = s; break; }
            factored_for = ls;
        }
        for (int64_t i = 0; i < n; i++) f[i] = rhs[idx_of(layout, n, m, i, s)];
        if (periodic) orc_cpenta_solve(&cp, f, sol);
        else orc_penta_solve(n, al, be, ga, de, ep, f, sol);
        for (int64_t i = 0; i < n; i++) x[idx_of(layout, n, m, i, s)] = sol[i];
    }
    orc_cpenta_free(&cp);
    free(la); free(lb); free(lc); free(ld); free(le);
    free(al); free(be); free(ga); free(de); free(ep); free(f); free(sol);
    return rc;
}

int orc_tri_batch_solve(int64_t n, int64_t m, int layout, int64_t lhs_count, int periodic,
                        const double *a, const double *b, const double *c, const double *rhs,
                        double *x, int64_t *bad_sys, int64_t *bad_row)
{
    if (n < 3 || m < 0 || (lhs_count != 1 && lhs_count != m)) return ORC_EINVAL;
    if (m == 0) return ORC_OK;
    double *la = malloc(sizeof(double) * n), *lb = malloc(sizeof(double) * n),
           *lc = malloc(sizeof(double) * n), *ch = malloc(sizeof(double) * n);
    double *f = malloc(sizeof(double) * n), *sol = malloc(sizeof(double) * n);
    orc_ctri ct;
    memset(&ct, 0, sizeof(ct));
    int rc = ORC_OK;
    int64_t factored_for = -1;
    for (int64_t s = 0; s < m && rc == ORC_OK; s++) {
        int64_t ls = (lhs_count == 1) ? 0 : s;
        if (ls != factored_for) {
            gather_lhs(n, lhs_count, ls, a, la); gather_lhs(n, lhs_count, ls, b, lb);
            gather_lhs(n, lhs_count, ls, c, lc);
            if (periodic) {
                orc_ctri_free(&ct);
                rc = orc_ctri_init(&ct, n, la, lb, lc, bad_row);
            } else {
                la[0] = 0.0; lc[n - 1] = 0.0;
                rc = orc_tri_factor(n, la, lb, lc, ch, bad_row);
            }
            if (rc) { if (bad_sys) *bad_sys = s; break; }
            factored_for = ls;
        }
        for (int64_t i = 0; i < n; i++) f[i] = rhs[idx_of(layout, n, m, i, s)];
        if (periodic) orc_ctri_solve(&ct, f, sol);
        else orc_tri_solve(n, la, lb, ch, f, sol);
        for (int64_t i = 0; i < n; i++) x[idx_of(layout, n, m, i, s)] = sol[i];
    }
    orc_ctri_free(&ct);
    free(la); free(lb); free(lc); free(ch); free(f); free(sol);
    return rc;
}

/* ------------------------------------------------------------------------ */
/* cuSten-style stencil, P:947-983 (§3.3).  Grid row-major g[b][j][i] (i = x).
 * Window: `top` rows above (j-top) .. `bottom` rows below, `left`..`right`
 * points in i.  Weights are row-major from the top-left, sweeping "left to
 * right in i, row by row in j".  periodic: wrap both axes.
 * Non-periodic: only cells whose whole window is inside are written; boundary
 * cells of `out` are left untouched.  out must differ from in. */
int orc_stencil_apply(int64_t batch, int64_t ny, int64_t nx, int left, int right, int top,
                      int bottom, const double *w, int periodic, const double *in, double *out)
{
    if (in == out || left < 0 || right < 0 || top < 0 || bottom < 0) return ORC_EINVAL;
    if (left + right >= nx || top + bottom >= ny) return ORC_EINVAL;
    int wx = left + right + 1;
    for (int64_t bb = 0; bb < batch; bb++) {
        const double *g = in + bb * ny * nx;
        double *o = out + bb * ny * nx;
        for (int64_t j = 0; j < ny; j++) {
            for (int64_t i = 0; i < nx; i++) {
                if (!periodic && (j - top < 0 || j + bottom >= ny || i - left < 0 || i + right >= nx))
                    continue;
                double acc = 0;
                for (int r = 0; r <= top + bottom; r++) {
                    int64_t jj = j - top + r;
                    if (periodic) jj = ((jj % ny) + ny) % ny;
                    for (int q = 0; q < wx; q++) {
                        int64_t ii = i - left + q;
                        if (periodic) ii = ((ii % nx) + nx) % nx;
                        acc += w[r * wx + q] * g[jj * nx + ii];
                    }
                }
                o[j * nx + i] = acc;
            }
        }
    }
    return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* ADI Cahn–Hilliard, Eq 3.1, with readings r1, r5-r10.         */
/* 5x5 weights of the linear biharmonic term grad^4 = dx^4 + 2 dx^2 dy^2 + dy^4
   (Fig 3.1 cross stencil, r4 fourth difference), scaled by 1/dx^4.   */
static void ch_biharmonic_weights(double dx, double w[25])
{
    memset(w, 0, sizeof(double) * 25);
    const double d4[5] = {1, -4, 6, -4, 1};
    const double cross[3][3] = {{1, -2, 1}, {-2, 4, -2}, {1, -2, 1}};
    for (int q = 0; q < 5; q++) w[2 * 5 + q] += d4[q];  /* delta_x^4: centre row */
    for (int r = 0; r < 5; r++) w[r * 5 + 2] += d4[r];  /* delta_y^4: centre col */
    for (int r = 0; r < 3; r++)
        for (int q = 0; q < 3; q++) w[(r + 1) * 5 + (q + 1)] += 2.0 * cross[r][q];
    double s = 1.0 / (dx * dx * dx * dx);
    for (int k = 0; k < 25; k++) w[k] *= s;
}

/* RHS of Eq 3.1(a): R = -2/3 (C^n - C^{n-1}) - 2/3 dt D gamma grad^4 Cbar
                         + 2/3 D dt grad^2 (C^3 - C)^n,   Cbar = 2C^n - C^{n-1}. */
int orc_ch_rhs(int64_t sims, int64_t n, double dt, double D, double gam, double L,
               const double *cn, const double *cm, double *R)
{
    if (n < 7) return ORC_EINVAL;
    double dx = L / (double)n; /* r1 */
    int64_t np = n * n;
    double *cbar = malloc(sizeof(double) * np), *nl = malloc(sizeof(double) * np),
           *bih = malloc(sizeof(double) * np), *lap = malloc(sizeof(double) * np);
    double wb[25], wl[9] = {0, 1, 0, 1, -4, 1, 0, 1, 0};
    ch_biharmonic_weights(dx, wb);
    for (int k = 0; k < 9; k++) wl[k] /= dx * dx; /* 5-point Laplacian (r8) */
    for (int64_t s = 0; s < sims; s++) {
        const double *Cn = cn + s * np, *Cm = cm + s * np;
        double *Rs = R + s * np;
        for (int64_t k = 0; k < np; k++) {
            cbar[k] = 2.0 * Cn[k] - Cm[k];
            nl[k] = Cn[k] * Cn[k] * Cn[k] - Cn[k];
        }
        orc_stencil_apply(1, n, n, 2, 2, 2, 2, wb, 1, cbar, bih);
        orc_stencil_apply(1, n, n, 1, 1, 1, 1, wl, 1, nl, lap);
        for (int64_t k = 0; k < np; k++)
            Rs[k] = -(2.0 / 3.0) * (Cn[k] - Cm[k]) - (2.0 / 3.0) * dt * D * gam * bih[k] +
                    (2.0 / 3.0) * D * dt * lap[k];
    }
    free(cbar); free(nl); free(bih); free(lap);
    return ORC_OK;
}

/* nsteps of Eq 3.1.  cn = C^n, cm = C^{n-1} (caller sets cm = cn = C^0 at the
   start); on return cn holds the newest level and cm the previous.   */
int orc_ch_adi_steps(int64_t sims, int64_t n, double dt, double D, double gam, double L,
                     int64_t nsteps, double *cn, double *cm)
{
    if (n < 7 || sims < 0 || nsteps < 0) return ORC_EINVAL;
    double dx = L / (double)n;
    double sig = (2.0 / 3.0) * D * gam * dt / (dx * dx * dx * dx); /* L_x = I + 2/3 D gamma dt d_xxxx */
    int64_t np = n * n;
    double *a = malloc(sizeof(double) * n), *b = malloc(sizeof(double) * n),
           *c = malloc(sizeof(double) * n), *d = malloc(sizeof(double) * n),
           *e = malloc(sizeof(double) * n);
    for (int64_t i = 0; i < n; i++) { a[i] = sig; b[i] = -4 * sig; c[i] = 1 + 6 * sig; d[i] = -4 * sig; e[i] = sig; }
    orc_cpenta cp;
    int rc = orc_cpenta_init(&cp, n, a, b, c, d, e, NULL);
    if (rc) { free(a); free(b); free(c); free(d); free(e); return rc; }
    double *R = malloc(sizeof(double) * np * (sims > 0 ? sims : 1));
    double *row = malloc(sizeof(double) * n), *sol = malloc(sizeof(double) * n);
    for (int64_t step = 0; step < nsteps; step++) {
        orc_ch_rhs(sims, n, dt, D, gam, L, cn, cm, R);
        for (int64_t s = 0; s < sims; s++) {
            double *Rs = R + s * np, *Cn = cn + s * np, *Cm = cm + s * np;
            /* L_x w = R : one cyclic solve per grid row j, along i */
            for (int64_t j = 0; j < n; j++) {
                orc_cpenta_solve(&cp, Rs + j * n, sol);
                memcpy(Rs + j * n, sol, sizeof(double) * n);
            }
            /* L_y v = w : one cyclic solve per column i, along j */
            for (int64_t i = 0; i < n; i++) {
                for (int64_t j = 0; j < n; j++) row[j] = Rs[j * n + i];
                orc_cpenta_solve(&cp, row, sol);
                for (int64_t j = 0; j < n; j++) Rs[j * n + i] = sol[j];
            }
            /* C^{n+1} = Cbar^{n+1} + v ; rotate levels */
            for (int64_t k = 0; k < np; k++) {
                double cnew = 2.0 * Cn[k] - Cm[k] + Rs[k];
                Cm[k] = Cn[k];
                Cn[k] = cnew;
            }
        }
    }
    orc_cpenta_free(&cp);
    free(a); free(b); free(c); free(d); free(e); free(R); free(row); free(sol);
    return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* 1D semi-implicit Cahn–Hilliard, P:2661-2737 (§6.2.1), with r12 (+C_i^n):
   (I + gamma dt d_xxxx) C^{n+1} = C^n + dt d_xx (C^3 - C)^n, D = 1,
   sigma = gamma dt/dx^4, alpha = dt/dx^2.  Batch of m systems, interleaved
   c[i*m + s].  Advances nsteps in place.                          */
int orc_ch1d_steps(int64_t n, int64_t m, double dt, double gam, double L, int64_t nsteps,
                   double *c)
{
    if (n < 7) return ORC_EINVAL;
    double dx = L / (double)n;
    double sig = gam * dt / (dx * dx * dx * dx), alp = dt / (dx * dx);
    double *a = malloc(sizeof(double) * n), *b = malloc(sizeof(double) * n),
           *cc = malloc(sizeof(double) * n), *d = malloc(sizeof(double) * n),
           *e = malloc(sizeof(double) * n);
    for (int64_t i = 0; i < n; i++) { a[i] = sig; b[i] = -4 * sig; cc[i] = 1 + 6 * sig; d[i] = -4 * sig; e[i] = sig; }
    orc_cpenta cp;
    int rc = orc_cpenta_init(&cp, n, a, b, cc, d, e, NULL);
    free(a); free(b); free(cc); free(d); free(e);
    if (rc) return rc;
    double *u = malloc(sizeof(double) * n), *nl = malloc(sizeof(double) * n),
           *f = malloc(sizeof(double) * n);
    for (int64_t step = 0; step < nsteps; step++) {
        for (int64_t s = 0; s < m; s++) {
            for (int64_t i = 0; i < n; i++) { u[i] = c[i * m + s]; nl[i] = u[i] * u[i] * u[i] - u[i]; }
            for (int64_t i = 0; i < n; i++) {
                int64_t im = (i + n - 1) % n, ip = (i + 1) % n;
                f[i] = u[i] + alp * (nl[im] - 2.0 * nl[i] + nl[ip]);
            }
            orc_cpenta_solve(&cp, f, u);
            for (int64_t i = 0; i < n; i++) c[i * m + s] = u[i];
        }
    }
    orc_cpenta_free(&cp);
    free(u); free(nl); free(f);
    return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* Coarsening statistics (thesis §7.1-7.5).                   */

/* Free energy of P:819-825 (reading r24): the bulk term is 1/4 (C^2-1)^2,
   whose derivative C^3 - C is the chemical potential of eq2:ch and whose
   decay rate is the printed dF/dt = -int |grad(C^3 - C - gamma lap C)|^2
   (the printed 1/2 (C^2-1)^2 would differentiate to 2(C^3 - C)):
   F_h = dx^2 sum_ij [ 1/4 (C_ij^2 - 1)^2
                       + 1/2 gamma ((C_{i+1,j} - C_ij)^2 + (C_{i,j+1} - C_ij)^2) / dx^2 ]
   with periodic forward differences.  One value per simulation.             */
int orc_ch_free_energy(int64_t sims, int64_t n, double L, double gam, const double *c, double *F)
{
    if (n < 2 || sims < 0) return ORC_EINVAL;
    double dx = L / (double)n; /* r1 */
    for (int64_t s = 0; s < sims; s++) {
        const double *C = c + s * n * n;
        double acc = 0.0;
        for (int64_t j = 0; j < n; j++)
            for (int64_t i = 0; i < n; i++) {
                double v = C[j * n + i];
                double gx = (C[j * n + (i + 1) % n] - v) / dx;
                double gy = (C[((j + 1) % n) * n + i] - v) / dx;
                acc += 0.25 * (v * v - 1.0) * (v * v - 1.0) + 0.5 * gam * (gx * gx + gy * gy);
            }
        F[s] = acc * dx * dx;
    }
    return ORC_OK;
}

/* The growth rate beta = -(t/F) dF/dt of P:3576 from samples F(t_k) of one
   simulation (reading r27: central differences in t at interior samples,
   one-sided at the two ends).  F, beta: [nt][sims].                         */
int orc_coarsening_beta(int64_t nt, int64_t sims, const double *t, const double *F, double *beta)
{
    if (nt < 2 || sims < 0) return ORC_EINVAL;
    for (int64_t k = 0; k < nt; k++) {
        int64_t a = k > 0 ? k - 1 : 0, b = k < nt - 1 ? k + 1 : nt - 1;
        for (int64_t s = 0; s < sims; s++) {
            double dFdt = (F[b * sims + s] - F[a * sims + s]) / (t[b] - t[a]);
            beta[k * sims + s] = -(t[k] / F[k * sims + s]) * dFdt;
        }
    }
    return ORC_OK;
}

/* Counter-based normals for the Cahn–Hilliard–Cook noise (reading r26): the
   thesis draws uniforms and applies Box–Muller; the generator
   is unspecified, so both sides use this one.  splitmix64 finaliser chained
   over (seed, step, sim, cell); two uniforms in (0,1) from two counters;
   Box–Muller gives rho_x (cos branch) and rho_y (sin branch) of one cell.  */
static uint64_t orc_mix64(uint64_t z)
{
    z += 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
void orc_cook_rho(uint64_t seed, int64_t step, int64_t sim, int64_t cell, double *rx, double *ry)
{
    uint64_t k = orc_mix64(orc_mix64(orc_mix64(seed) ^ (uint64_t)step) ^ (uint64_t)sim);
    uint64_t h1 = orc_mix64(k ^ (2 * (uint64_t)cell)), h2 = orc_mix64(k ^ (2 * (uint64_t)cell + 1));
    double u1 = ((double)(h1 >> 11) + 0.5) * (1.0 / 9007199254740992.0);
    double u2 = ((double)(h2 >> 11) + 0.5) * (1.0 / 9007199254740992.0);
    double r = sqrt(-2.0 * log(u1)), th = 2.0 * 3.14159265358979323846 * u2;
    *rx = r * cos(th);
    *ry = r * sin(th);
}

/* eta_ij = sqrt(sigma / (dx^2 dt)) (div rho)_ij, the divergence
   by periodic central differences (reading r26):
   (div rho)_ij = (rho_x[i+1,j] - rho_x[i-1,j] + rho_y[i,j+1] - rho_y[i,j-1]) / (2 dx). */
int orc_cook_noise(int64_t sims, int64_t n, double dt, double L, double sigma, uint64_t seed, int64_t step,
                   double *eta)
{
    if (n < 3 || sims < 0 || !(dt > 0)) return ORC_EINVAL;
    double dx = L / (double)n, amp = sqrt(sigma / (dx * dx * dt));
    int64_t np = n * n;
    double *rx = malloc(sizeof(double) * np), *ry = malloc(sizeof(double) * np);
    if (!rx || !ry) { free(rx); free(ry); return ORC_ENOMEM; }
    for (int64_t s = 0; s < sims; s++) {
        for (int64_t k = 0; k < np; k++) orc_cook_rho(seed, step, s, k, &rx[k], &ry[k]);
        for (int64_t j = 0; j < n; j++)
            for (int64_t i = 0; i < n; i++) {
                int64_t ip = (i + 1) % n, im = (i + n - 1) % n, jp = (j + 1) % n, jm = (j + n - 1) % n;
                double div = (rx[j * n + ip] - rx[j * n + im] + ry[jp * n + i] - ry[jm * n + i]) / (2.0 * dx);
                eta[s * np + j * n + i] = amp * div;
            }
    }
    free(rx); free(ry);
    return ORC_OK;
}

/* nsteps of Eq 3.1 for the Cahn–Hilliard–Cook equation: the
   noise of step step0 + k enters the RHS as + 2/3 dt eta^n (reading r25:
   the BDF2 weight of every explicit term of Eq 3.1(a)); otherwise as
   orc_ch_adi_steps.  sigma = 0 is orc_ch_adi_steps exactly.                 */
int orc_ch_adi_steps_cook(int64_t sims, int64_t n, double dt, double D, double gam, double L, double sigma,
                          uint64_t seed, int64_t step0, int64_t nsteps, double *cn, double *cm)
{
    if (n < 7 || sims < 0 || nsteps < 0) return ORC_EINVAL;
    int64_t np = n * n;
    double *eta = malloc(sizeof(double) * np * (sims > 0 ? sims : 1));
    double *R = malloc(sizeof(double) * np * (sims > 0 ? sims : 1));
    if (!eta || !R) { free(eta); free(R); return ORC_ENOMEM; }
    double dx = L / (double)n;
    double sig = (2.0 / 3.0) * D * gam * dt / (dx * dx * dx * dx);
    double *a = malloc(sizeof(double) * n), *b = malloc(sizeof(double) * n),
           *c = malloc(sizeof(double) * n), *d = malloc(sizeof(double) * n),
           *e = malloc(sizeof(double) * n);
    for (int64_t i = 0; i < n; i++) { a[i] = sig; b[i] = -4 * sig; c[i] = 1 + 6 * sig; d[i] = -4 * sig; e[i] = sig; }
    orc_cpenta cp;
    int rc = orc_cpenta_init(&cp, n, a, b, c, d, e, NULL);
    free(a); free(b); free(c); free(d); free(e);
    if (rc) { free(eta); free(R); return rc; }
    double *row = malloc(sizeof(double) * n), *sol = malloc(sizeof(double) * n);
    for (int64_t step = 0; step < nsteps; step++) {
        orc_ch_rhs(sims, n, dt, D, gam, L, cn, cm, R);
        orc_cook_noise(sims, n, dt, L, sigma, seed, step0 + step, eta);
        for (int64_t k = 0; k < np * sims; k++) R[k] += (2.0 / 3.0) * dt * eta[k];
        for (int64_t s = 0; s < sims; s++) {
            double *Rs = R + s * np, *Cn = cn + s * np, *Cm = cm + s * np;
            for (int64_t j = 0; j < n; j++) {
                orc_cpenta_solve(&cp, Rs + j * n, sol);
                memcpy(Rs + j * n, sol, sizeof(double) * n);
            }
            for (int64_t i = 0; i < n; i++) {
                for (int64_t j = 0; j < n; j++) row[j] = Rs[j * n + i];
                orc_cpenta_solve(&cp, row, sol);
                for (int64_t j = 0; j < n; j++) Rs[j * n + i] = sol[j];
            }
            for (int64_t k = 0; k < np; k++) {
                double cnew = 2.0 * Cn[k] - Cm[k] + Rs[k];
                Cm[k] = Cn[k];
                Cn[k] = cnew;
            }
        }
    }
    orc_cpenta_free(&cp);
    free(eta); free(R); free(row); free(sol);
    return ORC_OK;
}
