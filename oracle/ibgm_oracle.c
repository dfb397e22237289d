/*
 * oracle/ibgm_oracle.c -- TEST INFRASTRUCTURE, NOT PRODUCT CODE.
 *
 * A plain, slow, obviously-correct CPU implementation of the IB-GM time step of
 * Wiens & Stockie, "An Efficient Parallel Immersed Boundary Algorithm using a
 * Pseudo-Compressible Fluid Solver" (arXiv:1305.3976).  Every function cites the
 * PAPER.md passage it follows ("PAPER.md:L" = line L of the paper's LaTeX source).
 *
 * Rules (DESIGN.md section "Oracle"):
 *   - Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg (and its
 *     --impl reference arm) may load this library.  The product path
 *     (paper_1305_3976_b200/) never does.
 *   - It shares no code, header, table or constant generator with the CUDA path.
 *   - fp64 fields; the cyclic tridiagonal line solves run in long double
 *     (SURVEY A16 reading, R16); compiled with -ffp-contract=off.
 *   - No blocking, fusion or reordering beyond what the paper's algorithm states:
 *     Step 1a, 1b, 1c, 2a, 2b, 3a, ..., 3f in order.
 *
 * Parity status per part:
 *   pinned  : delta kernels (moments), interpolation/spreading (invariants,
 *             adjointness), fibre force (circle closed form, paper D_s form),
 *             stencils (eigenvalues / identities), skew advection (energy
 *             identity + 2nd-order convergence), cyclic solves (dense LU),
 *             viscous Douglas sweeps (Stokes Taylor-Green closed form),
 *             psi / p pipeline (per-Fourier-mode linear recurrence), start-up,
 *             time integration (Step 1c midpoint in uniform flow, Step 1b AB2 order
 *             from tracer self-convergence, eq. (nonlinear) AB2 advection from the
 *             explicit increment u* - u^n via the orc_keep_ustar test hook),
 *             minimum-image force connections (R26: through-the-boundary spring
 *             equals its nearby image), box side H (R2: the 2x2 ellipse array on
 *             [0,2]^2 equals the tiled single ellipse), and the whole method against
 *             the paper's Table 6.
 *   parity unpinned: the choice of the cosine kernel (COS4) for the BASELINE
 *             configs, the 3D edge-spring scaling (kappa=sigma, w=1) and the
 *             input sampling recipes -- these are BASELINE-defined, not paper-defined.
 */
#include <math.h>
#include <stdlib.h>
#include <string.h>
#include <stdint.h>

#define ORC_COS4 0    /* phi(r) = (1 + cos(pi r / 2)) / 4, |r| < 2  (BASELINE.json configs) */
#define ORC_PESKIN4 1 /* PAPER.md:510-520, eq. (discretedelta)                           */

/* ------------------------------------------------------------------------- */
/* Grid helpers.  Periodic box [0,H]^d, N cells per side, h = H/N (H = 1 in */
/* every BASELINE config; the P x P ellipse array of PAPER.md:1972-2003 is    */
/* H = P, R2)                                                       */
/* (PAPER.md:413-446).  Storage: idx = i + N*(j + N*k), x fastest.           */
/* ------------------------------------------------------------------------- */
typedef struct {
    int dim;
    long n;
    double h;
    double H;     /* box side */
} orc_grid;

static long wrap(long i, long n)
{
    if (i >= 0 && i < n) return i;
    long r = i % n;
    return r < 0 ? r + n : r;
}

static long idx3(const orc_grid* g, long i, long j, long k)
{
    long n = g->n;
    if (g->dim == 2) return wrap(i, n) + n * wrap(j, n);
    return wrap(i, n) + n * (wrap(j, n) + n * wrap(k, n));
}

/* value of q at (I + s*e_a) with periodic wrap; I = (i,j,k) */
static double at(const orc_grid* g, const double* q, long i, long j, long k)
{
    return q[idx3(g, i, j, k)];
}

static long ncell(const orc_grid* g) { return g->dim == 2 ? g->n * g->n : g->n * g->n * g->n; }

/* ------------------------------------------------------------------------- */
/* Spatial finite-difference operators                      */
/* ------------------------------------------------------------------------- */

/* D_aa q at (i,j,k): (q_{+e_a} - 2 q + q_{-e_a}) / h^2 */
static double op_d2(const orc_grid* g, const double* q, long i, long j, long k, int a)
{
    long di = (a == 0), dj = (a == 1), dk = (a == 2);
    return (at(g, q, i + di, j + dj, k + dk) - 2.0 * at(g, q, i, j, k) +
            at(g, q, i - di, j - dj, k - dk)) / (g->h * g->h);
}

/* G^{C->E} p, component c, at the u_c point with index (i,j,k):
 * (p_{I} - p_{I - e_c}) / h */
static double op_grad(const orc_grid* g, const double* p, long i, long j, long k, int c)
{
    long di = (c == 0), dj = (c == 1), dk = (c == 2);
    return (at(g, p, i, j, k) - at(g, p, i - di, j - dj, k - dk)) / g->h;
}

/* D^{E->C} . u at the cell centre (i,j,k): sum_c (u_c[I + e_c] - u_c[I]) / h
 * */
static double op_div(const orc_grid* g, double* const* u, long i, long j, long k)
{
    double s = 0.0;
    for (int c = 0; c < g->dim; c++) {
        long di = (c == 0), dj = (c == 1), dk = (c == 2);
        s += (at(g, u[c], i + di, j + dj, k + dk) - at(g, u[c], i, j, k)) / g->h;
    }
    return s;
}

/* Skew-symmetric advection N_c(u) = 1/2 u.grad u_c + 1/2 div(u u_c), second-order
 * centred on the staggered grid after Morinishi et al..  The
 * paper only cites the scheme; the reading (R4) is Morinishi's
 * "Skew.-S2": for each direction j, at the face of the u_c control volume
 * located at x_c(I) - h/2 e_j,
 *     T = (u_j[I] + u_j[I - e_c]) / 2      transport velocity (interpolated in c)
 *     A = (u_c[I] + u_c[I - e_j]) / 2      advected velocity (interpolated in j)
 *     g = (u_c[I] - u_c[I - e_j]) / h      d u_c / d x_j
 * divergence form   Div_c = sum_j (T A|_{I+e_j} - T A|_{I}) / h
 * advective form    Adv_c = sum_j (T g|_{I} + T g|_{I+e_j}) / 2
 * N_c = (Div_c + Adv_c) / 2. */
static void face_terms(const orc_grid* g, double* const* u, int c, int jd,
                       long i, long j, long k, double* T, double* A, double* G)
{
    long ci = (c == 0), cj = (c == 1), ck = (c == 2);
    long ji = (jd == 0), jj = (jd == 1), jk = (jd == 2);
    *T = 0.5 * (at(g, u[jd], i, j, k) + at(g, u[jd], i - ci, j - cj, k - ck));
    *A = 0.5 * (at(g, u[c], i, j, k) + at(g, u[c], i - ji, j - jj, k - jk));
    *G = (at(g, u[c], i, j, k) - at(g, u[c], i - ji, j - jj, k - jk)) / g->h;
}

static double op_adv(const orc_grid* g, double* const* u, int c, long i, long j, long k)
{
    double dv = 0.0, ad = 0.0;
    for (int jd = 0; jd < g->dim; jd++) {
        long ji = (jd == 0), jj = (jd == 1), jk = (jd == 2);
        double Tm, Am, Gm, Tp, Ap, Gp;
        face_terms(g, u, c, jd, i, j, k, &Tm, &Am, &Gm);                 /* face at -h/2 e_j */
        face_terms(g, u, c, jd, i + ji, j + jj, k + jk, &Tp, &Ap, &Gp);  /* face at +h/2 e_j */
        dv += (Tp * Ap - Tm * Am) / g->h;
        ad += 0.5 * (Tm * Gm + Tp * Gp);
    }
    return 0.5 * (dv + ad);
}

/* ------------------------------------------------------------------------- */
/* Discrete delta kernel                                    */
/* ------------------------------------------------------------------------- */
double orc_phi(int kernel, double r)
{
    double a = fabs(r);
    if (kernel == ORC_PESKIN4) {            /* eq. (discretedelta) */
        if (a < 1.0) return (3.0 - 2.0 * a + sqrt(1.0 + 4.0 * a - 4.0 * a * a)) / 8.0;
        if (a < 2.0) return (5.0 - 2.0 * a - sqrt(-7.0 + 12.0 * a - 4.0 * a * a)) / 8.0;
        return 0.0;
    }
    /* 4-point cosine kernel named by BASELINE.json configs (parity unpinned choice) */
    if (a < 2.0) return 0.25 * (1.0 + cos(M_PI * a / 2.0));
    return 0.0;
}

/* staggering offset o_{c,a}: u_c lives at ((I_a + o_{c,a}) h)_a; o = 0 on the
 * component's own axis, 1/2 elsewhere.  c = dim means the
 * cell centre (o = 1/2 everywhere). */
static double stag(int c, int a) { return (c == a) ? 0.0 : 0.5; }

/* U_c(X) = sum_I u_c[I] delta_h(x_I - X) h^d = sum_I u_c[I] prod_a phi(X_a/h - I_a - o_{c,a})
 * (Step 1a).  The sum runs over the 4^d nodes where phi != 0
 * (support |r| < 2); indices wrap periodically. */
static double interp1(const orc_grid* g, int kernel, const double* uc, int c, const double* X)
{
    long base[3] = {0, 0, 0};
    double xs[3] = {0, 0, 0};
    for (int a = 0; a < g->dim; a++) {
        xs[a] = X[a] / g->h - stag(c, a);
        base[a] = (long)floor(xs[a]) - 1;
    }
    double s = 0.0;
    int m2max = (g->dim == 3) ? 4 : 1;
    for (int m2 = 0; m2 < m2max; m2++)
        for (int m1 = 0; m1 < 4; m1++)
            for (int m0 = 0; m0 < 4; m0++) {
                long I0 = base[0] + m0, I1 = base[1] + m1, I2 = base[2] + m2;
                double w = orc_phi(kernel, xs[0] - I0) * orc_phi(kernel, xs[1] - I1);
                if (g->dim == 3) w *= orc_phi(kernel, xs[2] - I2);
                s += at(g, uc, I0, I1, I2) * w;
            }
    return s;
}

/* f_c[I] += F_c w delta_h(x_I - X) = F_c w h^{-d} prod_a phi(...)
 * (Step 2b; w = h_s for a 2D fibre, trapezoidal rule PAPER.md:567-570) */
static void spread1(const orc_grid* g, int kernel, double* fc, int c, const double* X, double Fw)
{
    long base[3] = {0, 0, 0};
    double xs[3] = {0, 0, 0};
    for (int a = 0; a < g->dim; a++) {
        xs[a] = X[a] / g->h - stag(c, a);
        base[a] = (long)floor(xs[a]) - 1;
    }
    double hd = (g->dim == 3) ? g->h * g->h * g->h : g->h * g->h;
    int m2max = (g->dim == 3) ? 4 : 1;
    for (int m2 = 0; m2 < m2max; m2++)
        for (int m1 = 0; m1 < 4; m1++)
            for (int m0 = 0; m0 < 4; m0++) {
                long I0 = base[0] + m0, I1 = base[1] + m1, I2 = base[2] + m2;
                double w = orc_phi(kernel, xs[0] - I0) * orc_phi(kernel, xs[1] - I1);
                if (g->dim == 3) w *= orc_phi(kernel, xs[2] - I2);
                fc[idx3(g, I0, I1, I2)] += Fw * w / hd;
            }
}

/* ------------------------------------------------------------------------- */
/* Cyclic (periodic) tridiagonal solve, PAPER.md:985-995 (eq. TriDiagX):      */
/*     c x_{i-1} + a x_i + b x_{i+1} = d_i,  indices mod n.                   */
/* Thomas's algorithm + Sherman-Morrison for the two corner entries, all in   */
/* long double (R16).  The paper's own serial building block is     */
/* Thomas's algorithm; the periodic corners are removed  */
/* by the rank-one Sherman-Morrison update (R16 states the formula).*/
/* ------------------------------------------------------------------------- */
static void thomas_ld(long n, long double c, const long double* diag, long double b,
                      const long double* d, long double* x, long double* cp, long double* dp)
{
    /* non-periodic tridiagonal: c x_{i-1} + diag_i x_i + b x_{i+1} = d_i */
    long double inv = 1.0L / diag[0];
    cp[0] = b * inv;
    dp[0] = d[0] * inv;
    for (long i = 1; i < n; i++) {
        inv = 1.0L / (diag[i] - c * cp[i - 1]);
        cp[i] = b * inv;
        dp[i] = (d[i] - c * dp[i - 1]) * inv;
    }
    x[n - 1] = dp[n - 1];
    for (long i = n - 2; i >= 0; i--) x[i] = dp[i] - cp[i] * x[i + 1];
}

static void cyclic_solve_ws(long n, double c_, double a_, double b_, const double* d, double* x,
                            long double* ws)
{
    long double c = c_, a = a_, b = b_;
    long double *diag = ws, *rhs = ws + n, *y = ws + 2 * n, *z = ws + 3 * n, *u = ws + 4 * n;
    long double *cp = ws + 5 * n, *dp = ws + 6 * n;
    /* A = T + u v^T, u = (gamma, 0, ..., 0, b)^T, v = (1, 0, ..., 0, c/gamma)^T,
     * A[0][n-1] = c (row 0 wraps to x_{n-1}), A[n-1][0] = b (row n-1 wraps to x_0). */
    long double gamma = -a;
    for (long i = 0; i < n; i++) { diag[i] = a; rhs[i] = d[i]; u[i] = 0.0L; }
    diag[0] = a - gamma;
    diag[n - 1] = a - b * c / gamma;
    u[0] = gamma;
    u[n - 1] = b;
    thomas_ld(n, c, diag, b, rhs, y, cp, dp);
    thomas_ld(n, c, diag, b, u, z, cp, dp);
    long double fact = (y[0] + c * y[n - 1] / gamma) / (1.0L + z[0] + c * z[n - 1] / gamma);
    for (long i = 0; i < n; i++) x[i] = (double)(y[i] - fact * z[i]);
}

void orc_cyclic_solve(long n, double c, double a, double b, const double* d, double* x)
{
    long double* ws = (long double*)malloc(sizeof(long double) * 7 * n);
    cyclic_solve_ws(n, c, a, b, d, x, ws);
    free(ws);
}

/* Solve (c, a, b) cyclic systems along axis `ax` for every grid line of q, in place. */
static void solve_axis(const orc_grid* g, double* q, int ax, double c, double a, double b)
{
    long n = g->n;
    double* line = (double*)malloc(sizeof(double) * n);
    double* sol = (double*)malloc(sizeof(double) * n);
    long double* ws = (long double*)malloc(sizeof(long double) * 7 * n);
    long kmax = (g->dim == 3) ? n : 1;
    /* the two coordinates transverse to ax */
    for (long t1 = 0; t1 < kmax; t1++)
        for (long t0 = 0; t0 < n; t0++) {
            for (long s = 0; s < n; s++) {
                long i = 0, j = 0, k = 0;
                if (ax == 0) { i = s; j = t0; k = t1; }
                else if (ax == 1) { i = t0; j = s; k = t1; }
                else { i = t0; j = t1; k = s; }
                line[s] = q[idx3(g, i, j, k)];
            }
            cyclic_solve_ws(n, c, a, b, line, sol, ws);
            for (long s = 0; s < n; s++) {
                long i = 0, j = 0, k = 0;
                if (ax == 0) { i = s; j = t0; k = t1; }
                else if (ax == 1) { i = t0; j = s; k = t1; }
                else { i = t0; j = t1; k = s; }
                q[idx3(g, i, j, k)] = sol[s];
            }
        }
    free(line); free(sol); free(ws);
}

/* Exported: solve every line of the N^dim array q along `axis`, in place. */
void orc_solve_axis(int dim, long n, int axis, double c, double a, double b, double* q)
{
    orc_grid g = {dim, n, 1.0 / (double)n, 1.0};
    solve_axis(&g, q, axis, c, a, b);
}

/* ------------------------------------------------------------------------- */
/* Exported single-operator entry points (used by the oracle's pin tests).    */
/* ------------------------------------------------------------------------- */
static orc_grid mkgrid(int dim, long n) { orc_grid g = {dim, n, 1.0 / (double)n, 1.0}; return g; }

#define LOOP_CELLS(g)                                              \
    for (long k = 0; k < ((g).dim == 3 ? (g).n : 1); k++)          \
        for (long j = 0; j < (g).n; j++)                           \
            for (long i = 0; i < (g).n; i++)

void orc_op_d2(int dim, long n, int axis, const double* q, double* out)
{
    orc_grid g = mkgrid(dim, n);
    LOOP_CELLS(g) out[idx3(&g, i, j, k)] = op_d2(&g, q, i, j, k, axis);
}

void orc_op_grad(int dim, long n, int comp, const double* p, double* out)
{
    orc_grid g = mkgrid(dim, n);
    LOOP_CELLS(g) out[idx3(&g, i, j, k)] = op_grad(&g, p, i, j, k, comp);
}

void orc_op_div(int dim, long n, const double* u, const double* v, const double* w, double* out)
{
    orc_grid g = mkgrid(dim, n);
    double* U[3] = {(double*)u, (double*)v, (double*)w};
    LOOP_CELLS(g) out[idx3(&g, i, j, k)] = op_div(&g, U, i, j, k);
}

void orc_op_adv(int dim, long n, const double* u, const double* v, const double* w,
                double* nu, double* nv, double* nw)
{
    orc_grid g = mkgrid(dim, n);
    double* U[3] = {(double*)u, (double*)v, (double*)w};
    double* O[3] = {nu, nv, nw};
    for (int c = 0; c < dim; c++)
        LOOP_CELLS(g) O[c][idx3(&g, i, j, k)] = op_adv(&g, U, c, i, j, k);
}

/* interpolate all components at npts points X[npts][dim] -> U[npts][dim] */
static void interp_grid(const orc_grid* g, int kernel, const double* u, const double* v, const double* w,
                        long npts, const double* X, double* U)
{
    const double* F[3] = {u, v, w};
    for (long p = 0; p < npts; p++)
        for (int c = 0; c < g->dim; c++) U[p * g->dim + c] = interp1(g, kernel, F[c], c, X + p * g->dim);
}

void orc_op_interp(int dim, long n, int kernel, const double* u, const double* v, const double* w,
                   long npts, const double* X, double* U)
{
    orc_grid g = mkgrid(dim, n);
    interp_grid(&g, kernel, u, v, w, npts, X, U);
}

/* spread forces F[npts][dim] with quadrature weights wgt[npts] (NULL -> 1) into
 * zeroed-or-not f arrays (accumulates) */
static void spread_grid(const orc_grid* g, int kernel, long npts, const double* X, const double* F,
                        const double* wgt, double* fu, double* fv, double* fw)
{
    double* O[3] = {fu, fv, fw};
    for (long p = 0; p < npts; p++)
        for (int c = 0; c < g->dim; c++)
            spread1(g, kernel, O[c], c, X + p * g->dim, F[p * g->dim + c] * (wgt ? wgt[p] : 1.0));
}

void orc_op_spread(int dim, long n, int kernel, long npts, const double* X, const double* F,
                   const double* wgt, double* fu, double* fv, double* fw)
{
    orc_grid g = mkgrid(dim, n);
    spread_grid(&g, kernel, npts, X, F, wgt, fu, fv, fw);
}

/* Elastic force of the force-connection network, Step 2a in the
 * FC form of PAPER.md:856-861.  Edge e = (a, b) with stiffness kappa_e and rest length
 * L_e acts as  F_a += kappa_e (X_b - X_a)(1 - L_e/|X_b - X_a|),  F_b -= the same.
 * For a closed 2D fibre with kappa = sigma/h_s^2 and L_e = L h_s this is exactly
 * sigma D_s^-( D_s^+ X (1 - L/|D_s^+ X|) )  (R9/R10).
 * X_b - X_a is the minimum-image displacement in the periodic unit box, so a fibre
 * that closes through the boundary acts on its periodic copy ("the ends of the
 * cylinder are connected to their periodic copies"; R26). */
static void force_box(int dim, long npts, const double* X, long nedges, const int64_t* edges,
                      const double* kappa, const double* rest, double* F, double H);

void orc_op_force(int dim, long npts, const double* X, long nedges, const int64_t* edges,
                  const double* kappa, const double* rest, double* F)
{
    force_box(dim, npts, X, nedges, edges, kappa, rest, F, 1.0);
}

static void force_box(int dim, long npts, const double* X, long nedges, const int64_t* edges,
                      const double* kappa, const double* rest, double* F, double H)
{
    for (long p = 0; p < npts * dim; p++) F[p] = 0.0;
    for (long e = 0; e < nedges; e++) {
        long a = (long)edges[2 * e], b = (long)edges[2 * e + 1];
        double D[3] = {0, 0, 0}, len2 = 0.0;
        for (int c = 0; c < dim; c++) {
            D[c] = X[b * dim + c] - X[a * dim + c];
            D[c] -= H * nearbyint(D[c] / H);  /* minimum image, box side H */
            len2 += D[c] * D[c];
        }
        double t = kappa[e];
        if (rest && rest[e] != 0.0) t = kappa[e] * (1.0 - rest[e] / sqrt(len2));
        for (int c = 0; c < dim; c++) { F[a * dim + c] += t * D[c]; F[b * dim + c] -= t * D[c]; }
    }
}

/* ------------------------------------------------------------------------- */
/* The IB-GM time step                                      */
/* ------------------------------------------------------------------------- */
typedef struct {
    orc_grid g;
    double mu, rho, dt, chi;
    int kernel, advection, rotate;
    long nc;
    double *u[3], *nprev[3], *nadv[3], *f[3], *ws[3];
    double *p, *psi, *r;
    long npts, nedges;
    double *X, *Xh, *Xn, *U, *Uprev, *F, *wgt;
    int64_t* edges;
    double *kappa, *rest;
    long step;
    int keep_ustar;              /* test hook: keep u* and p* of the last step */
    double *ustar[3], *pstar;
} orc_state;

void orc_destroy(orc_state* s);

orc_state* orc_create_box(int dim, long n, double H, double mu, double rho, double dt, double chi,
                          int kernel, int advection, int rotate);

orc_state* orc_create(int dim, long n, double mu, double rho, double dt, double chi,
                      int kernel, int advection, int rotate)
{
    return orc_create_box(dim, n, 1.0, mu, rho, dt, chi, kernel, advection, rotate);
}

/* the box [0,H]^d: h = H/N in every operator (D_aa = delta_aa/h^2 literally, R2) */
orc_state* orc_create_box(int dim, long n, double H, double mu, double rho, double dt, double chi,
                          int kernel, int advection, int rotate)
{
    if ((dim != 2 && dim != 3) || n < 4 || !(H > 0)) return NULL;
    orc_state* s = (orc_state*)calloc(1, sizeof(orc_state));
    s->g = mkgrid(dim, n);
    s->g.H = H;
    s->g.h = H / (double)n;
    s->mu = mu; s->rho = rho; s->dt = dt; s->chi = chi;
    s->kernel = kernel; s->advection = advection; s->rotate = rotate;
    s->nc = ncell(&s->g);
    for (int c = 0; c < dim; c++) {
        s->u[c] = (double*)calloc(s->nc, sizeof(double));
        s->nprev[c] = (double*)calloc(s->nc, sizeof(double));
        s->nadv[c] = (double*)calloc(s->nc, sizeof(double));
        s->f[c] = (double*)calloc(s->nc, sizeof(double));
        s->ws[c] = (double*)calloc(s->nc, sizeof(double));
        if (!s->u[c] || !s->nprev[c] || !s->nadv[c] || !s->f[c] || !s->ws[c]) { orc_destroy(s); return NULL; }
    }
    s->p = (double*)calloc(s->nc, sizeof(double));
    s->psi = (double*)calloc(s->nc, sizeof(double));
    s->r = (double*)calloc(s->nc, sizeof(double));
    if (!s->p || !s->psi || !s->r) { orc_destroy(s); return NULL; }
    return s;
}

void orc_destroy(orc_state* s)
{
    if (!s) return;
    for (int c = 0; c < 3; c++) { free(s->u[c]); free(s->nprev[c]); free(s->nadv[c]); free(s->f[c]); free(s->ws[c]); free(s->ustar[c]); }
    free(s->pstar);
    free(s->p); free(s->psi); free(s->r);
    free(s->X); free(s->Xh); free(s->Xn); free(s->U); free(s->Uprev); free(s->F); free(s->wgt);
    free(s->edges); free(s->kappa); free(s->rest);
    free(s);
}

/* u, v, (w): velocity u^0 on the MAC faces; p: p^{-1/2}; psi^{-1/2} = 0 (R5) */
void orc_set_fields(orc_state* s, const double* u, const double* v, const double* w, const double* p)
{
    const double* in[3] = {u, v, w};
    for (int c = 0; c < s->g.dim; c++) memcpy(s->u[c], in[c], sizeof(double) * s->nc);
    if (p) memcpy(s->p, p, sizeof(double) * s->nc); else memset(s->p, 0, sizeof(double) * s->nc);
    memset(s->psi, 0, sizeof(double) * s->nc);
    s->step = 0;
}

/* X[npts][dim]; edges[nedges][2]; kappa[nedges]; rest[nedges] or NULL; wgt[npts] or NULL */
int orc_set_boundary(orc_state* s, long npts, const double* X, long nedges, const int64_t* edges,
                     const double* kappa, const double* rest, const double* wgt)
{
    int d = s->g.dim;
    free(s->X); free(s->Xh); free(s->Xn); free(s->U); free(s->Uprev); free(s->F); free(s->wgt);
    free(s->edges); free(s->kappa); free(s->rest);
    s->npts = npts; s->nedges = nedges;
    s->X = (double*)calloc(npts * d + 1, sizeof(double));
    s->Xh = (double*)calloc(npts * d + 1, sizeof(double));
    s->Xn = (double*)calloc(npts * d + 1, sizeof(double));
    s->U = (double*)calloc(npts * d + 1, sizeof(double));
    s->Uprev = (double*)calloc(npts * d + 1, sizeof(double));
    s->F = (double*)calloc(npts * d + 1, sizeof(double));
    s->wgt = (double*)calloc(npts + 1, sizeof(double));
    s->edges = (int64_t*)calloc(2 * nedges + 1, sizeof(int64_t));
    s->kappa = (double*)calloc(nedges + 1, sizeof(double));
    s->rest = (double*)calloc(nedges + 1, sizeof(double));
    memcpy(s->X, X, sizeof(double) * npts * d);
    memcpy(s->edges, edges, sizeof(int64_t) * 2 * nedges);
    memcpy(s->kappa, kappa, sizeof(double) * nedges);
    for (long e = 0; e < nedges; e++) {
        if (edges[2 * e] < 0 || edges[2 * e] >= npts || edges[2 * e + 1] < 0 || edges[2 * e + 1] >= npts) return -1;
        s->rest[e] = rest ? rest[e] : 0.0;
    }
    for (long p = 0; p < npts; p++) s->wgt[p] = wgt ? wgt[p] : 1.0;
    s->step = 0;
    return 0;
}

static void one_step(orc_state* s)
{
    orc_grid* g = &s->g;
    const int d = g->dim;
    const long nc = s->nc;
    const long n = s->step;
    const double dt = s->dt, rho = s->rho, mu = s->mu;

    /* Step 1a: U^n = interpolate u^n at X^n */
    interp_grid(g, s->kernel, s->u[0], s->u[1], d == 3 ? s->u[2] : NULL, s->npts, s->X, s->U);

    /* Step 1b: X^{n+1} = X^n + dt (3/2 U^n - 1/2 U^{n-1}); forward Euler at n = 0
     * */
    for (long q = 0; q < s->npts * d; q++) {
        if (n == 0) s->Xn[q] = s->X[q] + dt * s->U[q];
        else s->Xn[q] = s->X[q] + dt * (1.5 * s->U[q] - 0.5 * s->Uprev[q]);
        /* Step 1c: X^{n+1/2} = (X^{n+1} + X^n)/2 */
        s->Xh[q] = 0.5 * (s->Xn[q] + s->X[q]);
    }

    /* Step 2a: F^{n+1/2} at X^{n+1/2} */
    force_box(d, s->npts, s->Xh, s->nedges, s->edges, s->kappa, s->rest, s->F, g->H);

    /* Step 2b: f^{n+1/2} = sum_k F_k delta_h(x - X^{n+1/2}_k) w_k */
    for (int c = 0; c < d; c++) memset(s->f[c], 0, sizeof(double) * nc);
    spread_grid(g, s->kernel, s->npts, s->Xh, s->F, s->wgt, s->f[0], s->f[1], d == 3 ? s->f[2] : NULL);

    /* Step 3a: p* = p^{n-1/2} + psi^{n-1/2}; p* = 0 at n = 0 */
    /* (kept in s->r temporarily) */
    for (long q = 0; q < nc; q++) s->r[q] = (n == 0) ? 0.0 : s->p[q] + s->psi[q];

    /* Step 3b: explicit momentum with the AB2 advection
     * N^{n+1/2} = 3/2 N(u^n) - 1/2 N(u^{n-1}), N^{1/2} = N(u^0) at
     * n = 0:
     *   rho ((u* - u^n)/dt + N^{n+1/2}) = mu (sum_a D_aa) u^n - G p* + f          */
    for (int c = 0; c < d; c++) {
        LOOP_CELLS(*g) {
            long q = idx3(g, i, j, k);
            s->nadv[c][q] = s->advection ? op_adv(g, s->u, c, i, j, k) : 0.0;
        }
    }
    for (int c = 0; c < d; c++) {
        LOOP_CELLS(*g) {
            long q = idx3(g, i, j, k);
            double lap = 0.0;
            for (int a = 0; a < d; a++) lap += op_d2(g, s->u[c], i, j, k, a);
            double nhalf = (n == 0) ? s->nadv[c][q] : 1.5 * s->nadv[c][q] - 0.5 * s->nprev[c][q];
            s->ws[c][q] = s->u[c][q] + dt * (-nhalf + (mu * lap - op_grad(g, s->r, i, j, k, c) + s->f[c][q]) / rho);
        }
        if (s->keep_ustar) memcpy(s->ustar[c], s->ws[c], sizeof(double) * nc);
    }
    if (s->keep_ustar) memcpy(s->pstar, s->r, sizeof(double) * nc);

    /* Steps 3c, 3d (and z in 3D): Douglas direction-split Crank-Nicolson sweeps
     *   (1 - (mu dt / 2 rho) D_aa) u^{(a)} = u^{(a-1)} - (mu dt / 2 rho) D_aa u^n
     * (eqs. umacstep1/umacstep2 PAPER.md:953-965).  The order is
     * rotated each step: x,y(,z) on even n, reversed on odd n
     * (R3). */
    int order[3];
    for (int a = 0; a < d; a++) order[a] = (s->rotate && (n % 2 == 1)) ? d - 1 - a : a;
    const double kap = mu * dt / (2.0 * rho);
    const double h2 = g->h * g->h;
    for (int oi = 0; oi < d; oi++) {
        int ax = order[oi];
        for (int c = 0; c < d; c++) {
            LOOP_CELLS(*g) {
                long q = idx3(g, i, j, k);
                s->ws[c][q] -= kap * op_d2(g, s->u[c], i, j, k, ax);
            }
            solve_axis(g, s->ws[c], ax, -kap / h2, 1.0 + 2.0 * kap / h2, -kap / h2);
        }
    }
    /* ws = u^{n+1} */

    /* Step 3e: (1 - D_xx)(1 - D_yy)[(1 - D_zz)] psi = -(rho/dt) D.u^{n+1}
     * (PAPER.md:668-675), solved as d sequential line-solve factors
     * (eqs. PenaltyStepPart1/2) in the rotated order. */
    LOOP_CELLS(*g) {
        long q = idx3(g, i, j, k);
        s->r[q] = -(rho / dt) * op_div(g, s->ws, i, j, k);
    }
    for (int oi = 0; oi < d; oi++)
        solve_axis(g, s->r, order[oi], -1.0 / h2, 1.0 + 2.0 / h2, -1.0 / h2);

    /* Step 3f: p^{n+1/2} = p^{n-1/2} + psi^{n+1/2} - chi mu D.((u^{n+1} + u^n)/2)
     * */
    LOOP_CELLS(*g) {
        long q = idx3(g, i, j, k);
        double dnew = op_div(g, s->ws, i, j, k), dold = op_div(g, s->u, i, j, k);
        s->p[q] = s->p[q] + s->r[q] - s->chi * mu * 0.5 * (dnew + dold);
    }
    memcpy(s->psi, s->r, sizeof(double) * nc);

    /* roll the state: u^n <- u^{n+1}, N(u^{n-1}) <- N(u^n), U^{n-1} <- U^n, X^n <- X^{n+1} */
    for (int c = 0; c < d; c++) {
        double* t = s->u[c]; s->u[c] = s->ws[c]; s->ws[c] = t;
        t = s->nprev[c]; s->nprev[c] = s->nadv[c]; s->nadv[c] = t;
    }
    memcpy(s->Uprev, s->U, sizeof(double) * s->npts * d);
    memcpy(s->X, s->Xn, sizeof(double) * s->npts * d);
    s->step++;
}

void orc_step(orc_state* s, long nsteps)
{
    for (long t = 0; t < nsteps; t++) one_step(s);
}

/* u^n, v^n, (w^n), p^{n-1/2}, psi^{n-1/2}, X^n, U^{n-1} (the velocity interpolated in
 * the last step).  Any pointer may be NULL. */
void orc_get_fields(const orc_state* s, double* u, double* v, double* w, double* p, double* psi,
                    double* X, double* U)
{
    double* out[3] = {u, v, w};
    for (int c = 0; c < s->g.dim; c++) if (out[c]) memcpy(out[c], s->u[c], sizeof(double) * s->nc);
    if (p) memcpy(p, s->p, sizeof(double) * s->nc);
    if (psi) memcpy(psi, s->psi, sizeof(double) * s->nc);
    if (X) memcpy(X, s->X, sizeof(double) * s->npts * s->g.dim);
    if (U) memcpy(U, s->Uprev, sizeof(double) * s->npts * s->g.dim);
}

/* Intermediate quantities of the last step: f^{n+1/2} (per component), N(u^n)
 * (the stored advection), F^{n+1/2} and X^{n+1/2}. */
void orc_get_aux(const orc_state* s, double* fu, double* fv, double* fw, double* nu, double* nv,
                 double* nw, double* F, double* Xh)
{
    double* fo[3] = {fu, fv, fw};
    double* no[3] = {nu, nv, nw};
    for (int c = 0; c < s->g.dim; c++) {
        if (fo[c]) memcpy(fo[c], s->f[c], sizeof(double) * s->nc);
        if (no[c]) memcpy(no[c], s->nprev[c], sizeof(double) * s->nc);
    }
    if (F) memcpy(F, s->F, sizeof(double) * s->npts * s->g.dim);
    if (Xh) memcpy(Xh, s->Xh, sizeof(double) * s->npts * s->g.dim);
}

long orc_steps_done(const orc_state* s) { return s->step; }

/* Test hook: from now on keep u* (the explicit momentum result of Step 3b, before
 * the Douglas sweeps) and p* (Step 3a) of each step.  Returns -1 on allocation
 * failure.  Storage only -- no arithmetic changes. */
int orc_keep_ustar(orc_state* s)
{
    if (s->keep_ustar) return 0;
    for (int c = 0; c < s->g.dim; c++) {
        s->ustar[c] = (double*)calloc(s->nc, sizeof(double));
        if (!s->ustar[c]) return -1;
    }
    s->pstar = (double*)calloc(s->nc, sizeof(double));
    if (!s->pstar) return -1;
    s->keep_ustar = 1;
    return 0;
}

/* u* (per component) and p* of the last step; requires orc_keep_ustar() first. */
int orc_get_ustar(const orc_state* s, double* us, double* vs, double* ws, double* pstar)
{
    if (!s->keep_ustar) return -1;
    double* o[3] = {us, vs, ws};
    for (int c = 0; c < s->g.dim; c++) if (o[c]) memcpy(o[c], s->ustar[c], sizeof(double) * s->nc);
    if (pstar) memcpy(pstar, s->pstar, sizeof(double) * s->nc);
    return 0;
}
