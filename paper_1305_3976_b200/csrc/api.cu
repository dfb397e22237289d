// C-ABI of libibgm.so (include/ibgm.h): context management, host-side precompute of
// the line-solver factors, the per-step schedule, host<->device copies.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <utility>
#include <vector>

#include "ibgm_internal.cuh"

using namespace ibgm;

struct ib_ctx {
    Ctx s;
};

static thread_local std::string g_err;

static int fail(int code, const char* fmt, ...)
{
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

#define CKC(call)                                                                          \
    do {                                                                                   \
        cudaError_t e_ = (call);                                                           \
        if (e_ != cudaSuccess)                                                             \
            return fail(e_ == cudaErrorMemoryAllocation ? IB_ENOMEM : IB_ECUDA, "%s: %s (%s:%d)", \
                        #call, cudaGetErrorString(e_), __FILE__, __LINE__);                \
    } while (0)

namespace ibgm {

// Long-double precompute of everything line-independent in the Schur-segmented
// cyclic solve (see LineCoef).  For part p with interface y_p and interior block
// z_p (m = L-1 unknowns, matrix B = tridiag(c, a, b)):
//   z_p = B^{-1} f_p - c y_p g - b y_{p+1} h,   g = B^{-1} e_1,  h = B^{-1} e_m,
// and the interface equations give the periodic P x P Schur matrix
//   S_pp = a - b c (h_m + g_1),  S_{p,p-1} = -c^2 g_m,  S_{p,p+1} = -b^2 h_1
// (PAPER.md:1192-1219 specialised to constant-coefficient lines).
struct SchurF {
    int m, P;
    std::vector<long double> inv, cp, g, h, sinv, colsum;
    long double gsum, hsum;
};

static void schur_factors(int64_t N, int L, long double c, long double a, long double b, SchurF* F)
{
    const int m = L - 1;
    const int P = (int)(N / L);
    F->m = m;
    F->P = P;
    F->inv.assign(m, 0.0L); F->cp.assign(m, 0.0L); F->g.assign(m, 0.0L); F->h.assign(m, 0.0L);
    std::vector<long double> den(m > 0 ? m : 1), cp(m > 0 ? m : 1);
    if (m > 0) {
        den[0] = a;
        cp[0] = b / den[0];
        for (int i = 1; i < m; ++i) {
            den[i] = a - c * cp[i - 1];
            cp[i] = b / den[i];
        }
    }
    for (int i = 0; i < m; ++i) {
        F->inv[i] = 1.0L / den[i];
        F->cp[i] = cp[i];
    }
    auto solveB = [&](const std::vector<long double>& d, std::vector<long double>& x) {
        std::vector<long double> dp(m);
        dp[0] = d[0] / den[0];
        for (int i = 1; i < m; ++i) dp[i] = (d[i] - c * dp[i - 1]) / den[i];
        x[m - 1] = dp[m - 1];
        for (int i = m - 2; i >= 0; --i) x[i] = dp[i] - cp[i] * x[i + 1];
    };
    long double g1 = 0.0L, gm = 0.0L, h1 = 0.0L, hm = 0.0L;
    F->gsum = F->hsum = 0.0L;
    if (m > 0) {
        std::vector<long double> e1(m, 0.0L), em(m, 0.0L);
        e1[0] = 1.0L;
        em[m - 1] = 1.0L;
        solveB(e1, F->g);
        solveB(em, F->h);
        for (int i = 0; i < m; ++i) { F->gsum += F->g[i]; F->hsum += F->h[i]; }
        g1 = F->g[0]; gm = F->g[m - 1]; h1 = F->h[0]; hm = F->h[m - 1];
    }
    // m = 0 (one unknown per part): the parts couple directly, S = tridiag(c, a, b)
    const long double s0 = (m > 0) ? a - b * c * (hm + g1) : a;
    const long double sm = (m > 0) ? -c * c * gm : c;
    const long double sp = (m > 0) ? -b * b * h1 : b;
    std::vector<long double> S((size_t)P * P, 0.0L), I((size_t)P * P, 0.0L);
    for (int p = 0; p < P; ++p) {
        S[(size_t)p * P + p] += s0;
        S[(size_t)p * P + (p + P - 1) % P] += sm;
        S[(size_t)p * P + (p + 1) % P] += sp;
        I[(size_t)p * P + p] = 1.0L;
    }
    // Gauss-Jordan with partial pivoting (P is small)
    for (int col = 0; col < P; ++col) {
        int piv = col;
        for (int r = col + 1; r < P; ++r)
            if (fabsl(S[(size_t)r * P + col]) > fabsl(S[(size_t)piv * P + col])) piv = r;
        if (piv != col)
            for (int q = 0; q < P; ++q) {
                std::swap(S[(size_t)col * P + q], S[(size_t)piv * P + q]);
                std::swap(I[(size_t)col * P + q], I[(size_t)piv * P + q]);
            }
        const long double d = S[(size_t)col * P + col];
        for (int q = 0; q < P; ++q) {
            S[(size_t)col * P + q] /= d;
            I[(size_t)col * P + q] /= d;
        }
        for (int r = 0; r < P; ++r) {
            if (r == col) continue;
            const long double f = S[(size_t)r * P + col];
            if (f == 0.0L) continue;
            for (int q = 0; q < P; ++q) {
                S[(size_t)r * P + q] -= f * S[(size_t)col * P + q];
                I[(size_t)r * P + q] -= f * I[(size_t)col * P + q];
            }
        }
    }
    F->sinv = I;
    F->colsum.assign(P, 0.0L);
    for (int q = 0; q < P; ++q)
        for (int p = 0; p < P; ++p) F->colsum[q] += I[(size_t)p * P + q];
}

void make_line_coef(LineCoef* C, SchurInv* SI, int64_t N, int L, double c_, double a_, double b_, int mean_fix,
                    double* ext_host)
{
    memset(C, 0, sizeof(*C));
    memset(SI, 0, sizeof(*SI));
    SchurF F;
    schur_factors(N, L, c_, a_, b_, &F);
    C->c = c_; C->a = a_; C->b = b_;
    C->L = L; C->P = F.P; C->N = (int)N; C->mean_fix = mean_fix;
    C->inv_rowsum = (double)(1.0L / ((long double)a_ + b_ + c_));
    for (int i = 0; i < F.m; ++i) {
        if (L <= kMaxL) {
            C->inv[i] = (double)F.inv[i];
            C->cp[i] = (double)F.cp[i];
            C->g[i] = (double)F.g[i];
            C->h[i] = (double)F.h[i];
        } else if (ext_host) {
            ext_host[i] = (double)F.inv[i];
            ext_host[F.m + i] = (double)F.cp[i];
            ext_host[2 * F.m + i] = (double)F.g[i];
            ext_host[3 * F.m + i] = (double)F.h[i];
        }
    }
    C->gsum = (double)F.gsum;
    C->hsum = (double)F.hsum;
    for (int i = 0; i < F.P * F.P; ++i) SI->sinv[i] = (double)F.sinv[i];
    for (int p = 0; p < F.P; ++p)
        for (int q = 0; q < F.P; ++q) SI->sinvT[q * F.P + p] = SI->sinv[p * F.P + q];
    C->inv_n = (double)(1.0L / (long double)N);
    for (int q = 0; q < F.P; ++q) SI->colsum[q] = (double)F.colsum[q];
    // banded S^{-1} (LineCoef::band): circulant to rounding, and negligible beyond the band
    // (A/B switch: IBGM_BAND=0 keeps the dense product)
    C->band = -1;
    const int P = F.P;
    const long double ref = fabsl(F.sinv[0]);
    const char* eb = getenv("IBGM_BAND");
    bool circ = P > 1 && ref > 0 && !(eb && atoi(eb) == 0);
    for (int p = 0; p < P && circ; ++p)
        for (int q = 0; q < P; ++q)
            if (fabsl(F.sinv[p * P + q] - F.sinv[(q - p + P) % P]) > 1e-14L * ref) { circ = false; break; }
    {
        // (A/B switch: IBGM_CIRC=0 stages the dense S^{-1} for the non-banded systems)
        const char* ec = getenv("IBGM_CIRC");
        C->circ = (circ && !(ec && atoi(ec) == 0)) ? 1 : 0;
        if (C->circ)
            for (int d = 0; d < P; ++d) C->wf[d] = (double)F.sinv[d];
    }
    for (int bw = 0; circ && bw <= kMaxBand && 2 * bw + 1 < P; ++bw) {
        long double out = 0;
        for (int d = bw + 1; d <= P - 1 - bw; ++d) out = std::max(out, fabsl(F.sinv[d]));
        if (out <= 1e-18L * ref) {
            C->band = bw;
            for (int d = -bw; d <= bw; ++d) C->w[kMaxBand + d] = (double)F.sinv[(d + P) % P];
            break;
        }
    }
}

// Slab coefficient block (layout in ibgm_internal.cuh): the same factors for a line of
// N = P nz unknowns cut at the slab boundaries (part = slab).
static std::vector<double> slab_coef_block(int64_t N, int nz, double c, double a, double b, int mf)
{
    SchurF F;
    schur_factors(N, nz, c, a, b, &F);
    const int m = F.m, P = F.P;
    std::vector<double> v(SC_HDR + 4 * m + P * P + P, 0.0);
    v[SC_C] = c; v[SC_A] = a; v[SC_B] = b;
    v[SC_INVROW] = (double)(1.0L / ((long double)a + b + c));
    v[SC_GSUM] = (double)F.gsum;
    v[SC_HSUM] = (double)F.hsum;
    v[SC_N] = (double)N;
    v[SC_MF] = mf;
    for (int i = 0; i < m; ++i) {
        v[SC_HDR + i] = (double)F.inv[i];
        v[SC_HDR + m + i] = (double)F.cp[i];
        v[SC_HDR + 2 * m + i] = (double)F.g[i];
        v[SC_HDR + 3 * m + i] = (double)F.h[i];
    }
    for (int i = 0; i < P * P; ++i) v[SC_HDR + 4 * m + i] = (double)F.sinv[i];
    for (int q = 0; q < P; ++q) v[SC_HDR + 4 * m + P * P + q] = (double)F.colsum[q];
    return v;
}

}  // namespace ibgm

static bool choose_segmentation(int64_t n, int* L, int* P)
{
    // N <= 1024: segments of <= 32 unknowns (registers); 2D N in {2048, 4096}: 32 segments
    // of 64 / 128 unknowns solved in shared memory
    static const int cands[] = {8, 12, 16, 24, 32, 6, 4, 3, 2, 64, 128};
    for (int c : cands) {
        if (n % c == 0 && n / c <= kMaxSeg) {
            *L = c;
            *P = (int)(n / c);
            return true;
        }
    }
    return false;
}

static void drop_graphs(Ctx* s)
{
    for (int k = 0; k < 4; ++k) {
        if (s->gvalid[k]) cudaGraphExecDestroy(s->gexec[k]);
        s->gvalid[k] = false;
    }
}

static void free_lagrangian(Ctx* s)
{
    cudaFree(s->X); cudaFree(s->Xh); cudaFree(s->Uprev); cudaFree(s->F); cudaFree(s->wgt);
    cudaFree(s->csr_ptr); cudaFree(s->csr_nbr); cudaFree(s->csr_kappa); cudaFree(s->csr_rest);
    cudaFree(s->bin_bid); cudaFree(s->bin_sorted);
    cudaFree(s->pt_user); cudaFree(s->lag_tmp);
    cudaFree(s->Xold); cudaFree(s->Uold);
    s->Xold = s->Uold = nullptr;
    s->ib_ahead = false;
    s->pt_user = nullptr;
    s->lag_tmp = nullptr;
    s->bin_bid = s->bin_sorted = nullptr;
    s->X = s->Xh = s->Uprev = s->F = s->wgt = nullptr;
    s->csr_ptr = s->csr_nbr = nullptr;
    s->csr_kappa = s->csr_rest = nullptr;
    s->npts = s->nedges = 0;
    if (s->grp) {
        cudaFree(s->grp->Upart); cudaFree(s->grp->Ured);
        s->grp->Upart = s->grp->Ured = nullptr;
        s->grp->ucap = 0;
        for (int r = 0; r < s->grp->nloc; ++r) { cudaFree(s->grp->sel[r]); s->grp->sel[r] = nullptr; }
        cudaFree(s->grp->sel_cnt);
        s->grp->sel_cnt = nullptr;
    }
}

// one field of the local extent (plus a halo plane on each side on a z-slab), zeroed;
// the pointer addresses plane 0
static cudaError_t field_alloc(Ctx* s, double** out)
{
    const int halo = s->wrap ? 0 : 1;
    const size_t bytes = (size_t)(s->nl + 2 * halo) * s->plane * sizeof(double);
    double* b = nullptr;
    cudaError_t e = cudaMalloc(&b, bytes);
    if (e != cudaSuccess) return e;
    e = cudaMemsetAsync(b, 0, bytes, s->stream);
    *out = b + s->hoff;
    return e;
}

static void field_free(Ctx* s, double*& p)
{
    if (p) cudaFree(p - s->hoff);
    p = nullptr;
}

static cudaError_t alloc_fields(Ctx* s)
{
    cudaError_t e;
    for (int q = 0; q < s->dim; ++q) {
        if ((e = field_alloc(s, &s->u[q])) != cudaSuccess) return e;
        if ((e = field_alloc(s, &s->st[q])) != cudaSuccess) return e;
        if ((e = field_alloc(s, &s->nadv[q])) != cudaSuccess) return e;
        if ((e = field_alloc(s, &s->nprev[q])) != cudaSuccess) return e;
    }
    if ((e = field_alloc(s, &s->p)) != cudaSuccess) return e;
    if ((e = field_alloc(s, &s->pstar)) != cudaSuccess) return e;
    if ((e = field_alloc(s, &s->tmp)) != cudaSuccess) return e;
    return cudaMalloc(&s->d_flag, sizeof(int));
}

static void free_fields(Ctx* s)
{
    for (int q = 0; q < 3; ++q) {
        field_free(s, s->u[q]); field_free(s, s->st[q]); field_free(s, s->nadv[q]);
        field_free(s, s->nprev[q]); field_free(s, s->f[q]);
    }
    field_free(s, s->p); field_free(s, s->pstar); field_free(s, s->tmp);
    cudaFree(s->d_flag);
    s->d_flag = nullptr;
}

// local slabs of a context: itself on a single GPU, else the group's slabs
static int nslabs(Ctx* s) { return s->grp ? s->grp->nloc : 1; }
static Ctx* slab_at(Ctx* s, int r) { return s->grp ? s->grp->slab[r] : s; }

// host-array offset (doubles) of a slab's plane 0 in the fields passed through the API
static size_t host_off(Ctx* s, Ctx* sl)
{
    return (s->grp && s->grp->transport == IB_TRANSPORT_EMULATE) ? (size_t)(sl->z0 * sl->plane) : 0;
}

static int64_t total_launches(Ctx* s)
{
    int64_t t = s->launches;
    if (s->grp)
        for (int r = 0; r < s->grp->nloc; ++r) t += s->grp->slab[r]->launches;
    return t;
}

static int upload_coef(Ctx* s, int sys, double c, double a, double b, int mf)
{
    Group* G = s->grp;
    std::vector<double> v = slab_coef_block(s->n, (int)(s->n / (G->P * G->Q)), c, a, b, mf);
    if (G->coef[sys]) cudaFree(G->coef[sys]);
    G->coef[sys] = nullptr;
    CKC(cudaMalloc(&G->coef[sys], v.size() * sizeof(double)));
    CKC(cudaMemcpyAsync(G->coef[sys], v.data(), v.size() * sizeof(double), cudaMemcpyHostToDevice, s->stream));
    CKC(cudaStreamSynchronize(s->stream));
    if (sys == SYS_VISC) {
        // is the cut-axis S^{-1} diagonal to rounding?  (A/B switch: IBGM_SLAB_LOCAL=0)
        const int PQ = G->P * G->Q, m = (int)(s->n / PQ) - 1;
        const double* S = v.data() + SC_HDR + 4 * m;
        const double ref = std::fabs(S[0]);
        bool diag = PQ > 1 && ref > 0;
        for (int p = 0; p < PQ && diag; ++p)
            for (int q = 0; q < PQ; ++q) {
                const double e = std::fabs(S[p * PQ + q]);
                if ((p == q) ? std::fabs(e - ref) > 1e-14 * ref : e > 1e-18 * ref) { diag = false; break; }
            }
        const char* el = getenv("IBGM_SLAB_LOCAL");
        G->visc_local = (diag && !(el && atoi(el) == 0)) ? 1 : 0;
        G->visc_w0 = S[0];
    }
    return IB_OK;
}

// a Lagrangian array [npts][dim] to a host buffer in the caller's point order
static cudaError_t points_out(Ctx* s, const double* dev, double* host)
{
    if (!host || s->npts == 0) return cudaSuccess;
    cudaError_t e = launch_scatter_pts(s, dev, s->lag_tmp);
    if (e != cudaSuccess) return e;
    return cudaMemcpyAsync(host, s->lag_tmp, (size_t)s->npts * s->dim * sizeof(double), cudaMemcpyDeviceToHost,
                           s->stream);
}

// default interval of the in-step state check (ib_set_check_interval)
static const int64_t kDefaultCheckEvery = 100;

// the sticky errors raised by kernels (k_force: degenerate connection; the periodic
// state check: non-finite values, a point moving more than a cell).  The words are
// mapped host memory written with plain device stores, so a flag becomes visible once
// the kernel that raised it has run; IB_OK if none is set.
static int poll_errors(Ctx* s)
{
    volatile int* e = s->err_h;
    if (!e) return IB_OK;
    if (e[ERR_DEGENERATE])
        return fail(IB_EDEGENERATE, "a force connection with rest length L != 0 has zero length |X_m - X_k| = 0 "
                                    "(singular strain, SPEC.md:140); the state is suspect from step <= %lld on",
                    (long long)s->step);
    if (e[ERR_NONFINITE]) return fail(IB_ENONFINITE, "non-finite value in u, p or X (in-step check, <= %lld steps)",
                                      (long long)s->step);
    if (e[ERR_DOMAIN])
        return fail(IB_EDOMAIN, "an immersed-boundary point moved more than one cell h in one step (<= %lld steps): "
                                "the 4-point support left its halo (SPEC.md:131); reduce dt", (long long)s->step);
    return IB_OK;
}

static void clear_errors(Ctx* s)
{
    if (s->err_h) memset((void*)s->err_h, 0, ERR_WORDS * sizeof(int));
}

// the in-step state check: every field held by the context (or its slabs) and X for
// non-finite values, X^{n+1} - X^{n+1/2} for a move of more than a cell
static cudaError_t enqueue_check(Ctx* s)
{
    const int ns = s->grp ? s->grp->nloc : 0;
    for (int r = 0; r < ns; ++r) {
        cudaError_t e = launch_check_finite(s->grp->slab[r], s->err_d + ERR_NONFINITE);
        if (e != cudaSuccess) return e;
    }
    cudaError_t e = launch_check_finite(s, s->err_d + ERR_NONFINITE);
    if (e == cudaSuccess) e = launch_check_domain(s, s->err_d + ERR_DOMAIN);
    return e;
}

// With the look-ahead the device already holds X^{n+1}, U^n (and the IB history of
// step n+1); Xold/Uold keep X^n, U^{n-1}.  Put the state of step n back before
// anything restarts the time stepping from it.
static cudaError_t undo_lookahead(Ctx* s)
{
    if (s->ib_ahead && s->npts > 0) {
        const size_t pb = (size_t)s->npts * s->dim * sizeof(double);
        cudaError_t e = cudaMemcpyAsync(s->X, s->Xold, pb, cudaMemcpyDeviceToDevice, s->stream);
        if (e == cudaSuccess) e = cudaMemcpyAsync(s->Uprev, s->Uold, pb, cudaMemcpyDeviceToDevice, s->stream);
        if (e != cudaSuccess) return e;
    }
    s->ib_ahead = false;
    return cudaSuccess;
}

extern "C" {

void ib_default_options(ib_options* o)
{
    memset(o, 0, sizeof(*o));
    o->kernel = IB_DELTA_COS4;
    o->chi = 0.6;
    o->advection = 1;
    o->device = 0;
    o->stream = nullptr;
    o->rank = 0;
    o->nranks = 1;
    o->transport = IB_TRANSPORT_NCCL;
    o->nccl_id = nullptr;
}

const char* ib_last_error(void) { return g_err.c_str(); }

int ib_slab_range(int64_t n, int32_t nranks, int32_t rank, int64_t* z0, int64_t* nz)
{
    if (nranks < 1 || nranks > kMaxRanks) return fail(IB_EINVAL, "nranks must be in [1, %d]", kMaxRanks);
    if (rank < 0 || rank >= nranks) return fail(IB_EINVAL, "rank %d out of [0, %d)", rank, nranks);
    if (n % nranks != 0) return fail(IB_EINVAL, "N = %lld is not divisible by nranks = %d", (long long)n, nranks);
    if (n / nranks < 2) return fail(IB_EINVAL, "slab depth N/nranks = %lld < 2", (long long)(n / nranks));
    if (z0) *z0 = (n / nranks) * rank;
    if (nz) *nz = n / nranks;
    return IB_OK;
}

int ib_nccl_unique_id(void* out)
{
    if (!out) return fail(IB_EINVAL, "null argument");
    const char* e = nccl_load();
    if (e) return fail(IB_ENCCL, "%s", e);
    NcclUid id;
    const int rc = nccl_unique_id(&id);
    if (rc != 0) return fail(IB_ENCCL, "ncclGetUniqueId: %s", nccl_error_string(rc));
    memcpy(out, &id, sizeof(id));
    return IB_OK;
}

int ib_create(const ib_grid* grid, double nu, double rho, double dt, const ib_options* opt, ib_ctx** out)
{
    if (!grid || !out) return fail(IB_EINVAL, "null argument");
    *out = nullptr;
    ib_options o;
    if (opt) o = *opt; else ib_default_options(&o);
    if (grid->dim != 2 && grid->dim != 3) return fail(IB_EINVAL, "dim must be 2 or 3 (got %d)", grid->dim);
    if (grid->n < 8 || grid->n > (grid->dim == 2 ? 4096 : 1024))
        return fail(IB_EINVAL, "N must be in [8, %d] (got %lld)", grid->dim == 2 ? 4096 : 1024, (long long)grid->n);
    if (!(grid->H > 0)) return fail(IB_EINVAL, "the box side H must be > 0");
    if (!(dt > 0) || !(rho > 0) || !(nu >= 0)) return fail(IB_EINVAL, "need dt > 0, rho > 0, nu >= 0");
    if (!(o.chi > 0 && o.chi <= 1)) return fail(IB_EINVAL, "chi must be in (0, 1]");
    if (o.kernel != IB_DELTA_COS4 && o.kernel != IB_DELTA_PESKIN4) return fail(IB_EINVAL, "unknown delta kernel");
    if (o.transport != IB_TRANSPORT_NCCL && o.transport != IB_TRANSPORT_EMULATE)
        return fail(IB_EINVAL, "unknown transport %d", o.transport);
    const int P = o.nranks;
    if (P < 1) return fail(IB_EINVAL, "nranks must be >= 1");
    // the slab path also runs with one slab when asked for explicitly (EMULATE, or an
    // NCCL id: a 1-rank communicator), which exercises the transports on one GPU
    const bool slab = P > 1 || o.transport == IB_TRANSPORT_EMULATE || o.nccl_id != nullptr;
    if (slab) {
        const int rc = ib_slab_range(grid->n, P, o.transport == IB_TRANSPORT_NCCL ? o.rank : 0, nullptr, nullptr);
        if (rc != IB_OK) return rc;
        if (o.transport == IB_TRANSPORT_EMULATE && o.rank != 0) return fail(IB_EINVAL, "EMULATE transport: rank must be 0");
        if (o.transport == IB_TRANSPORT_NCCL && !o.nccl_id) return fail(IB_EINVAL, "NCCL transport needs nccl_id");
    } else if (o.rank != 0) {
        return fail(IB_EINVAL, "rank must be 0 when nranks = 1");
    }
    int L, Pseg;
    if (!choose_segmentation(grid->n, &L, &Pseg))
        return fail(IB_EINVAL, "N = %lld has no divisor L in {2,...,32, 64, 128} with N/L <= 32",
                    (long long)grid->n);

    ib_ctx* c = new ib_ctx();
    Ctx* s = &c->s;
    memset(s, 0, sizeof(*s));
    s->dim = grid->dim;
    s->n = grid->n;
    s->ncell = grid->dim == 3 ? grid->n * grid->n * grid->n : grid->n * grid->n;
    s->plane = grid->dim == 3 ? grid->n * grid->n : grid->n;
    s->H = grid->H;
    s->h = grid->H / (double)grid->n;       // every operator uses h = H/N (R2)
    s->rho = rho;
    s->mu = nu * rho;
    s->dt = dt;
    s->chi = o.chi;
    s->kernel = o.kernel;
    s->advection = o.advection;
    s->device = o.device;
    s->L = L; s->P = Pseg;
    s->use_graphs = true;
    s->wrap = 1;
    s->nl = s->n;
    *out = c;

    CKC(cudaSetDevice(o.device));
    CKC(cudaHostAlloc((void**)&s->err_h, ERR_WORDS * sizeof(int), cudaHostAllocMapped));
    memset(s->err_h, 0, ERR_WORDS * sizeof(int));
    CKC(cudaHostGetDevicePointer((void**)&s->err_d, s->err_h, 0));
    s->check_every = kDefaultCheckEvery;
    if (o.stream) {
        s->stream = (cudaStream_t)o.stream;
        s->own_stream = false;
    } else {
        CKC(cudaStreamCreateWithFlags(&s->stream, cudaStreamNonBlocking));
        s->own_stream = true;
    }
    CKC(cudaMalloc(&s->sinv, sizeof(SchurInv) * SYS_COUNT));
    SchurInv hs[SYS_COUNT];
    // viscous Douglas sweeps: (1 - kap delta) with kap = mu dt / (2 rho h^2)
    const double kv = s->mu * dt / (2.0 * rho * s->h * s->h);
    // (well conditioned, cond <= 1 + 4 kv: no mean correction needed, R16)
    const double kp = 1.0 / (s->h * s->h);
    {
        // psi factors: (1 - D_aa) with D_aa = delta / h^2 (R2)
        const double cc[SYS_COUNT] = {-kv, -kp, -kv};
        const int mfx[SYS_COUNT] = {0, 1, 0};
        std::vector<double> ext((size_t)4 * (L - 1) + 1);
        for (int k = 0; k < SYS_COUNT; ++k) {
            make_line_coef(&s->hcoef[k], &hs[k], s->n, L, cc[k], 1.0 - 2.0 * cc[k], cc[k], mfx[k], ext.data());
            if (L > kMaxL) {
                CKC(cudaMalloc(&s->lcext[k], ext.size() * sizeof(double)));
                CKC(cudaMemcpy(s->lcext[k], ext.data(), ext.size() * sizeof(double), cudaMemcpyHostToDevice));
                s->hcoef[k].ext = s->lcext[k];
            }
        }
    }
    CKC(cudaMemcpyAsync(s->sinv, hs, sizeof(SchurInv) * SYS_COUNT, cudaMemcpyHostToDevice, s->stream));

    if (!slab) {
        s->nlocal = s->ncell;
        s->hoff = 0;
        CKC(alloc_fields(s));
    } else {
        // z-slab decomposition: the top context keeps the Lagrangian state; each slab
        // context holds the fields of nz planes (+ halos) and borrows the stream and the
        // line factors of the top
        s->nlocal = 0;
        CKC(cudaMalloc(&s->d_flag, sizeof(int)));
        Group* G = new Group();
        memset(G, 0, sizeof(*G));
        s->grp = G;
        G->P = P;
        G->transport = o.transport;
        G->rank = (o.transport == IB_TRANSPORT_NCCL) ? o.rank : 0;
        G->nloc = (o.transport == IB_TRANSPORT_EMULATE) ? P : 1;
        const int64_t nz = s->n / P;
        for (int r = 0; r < G->nloc; ++r) {
            Ctx* sl = new Ctx();
            memset(sl, 0, sizeof(*sl));
            sl->dim = s->dim; sl->n = s->n; sl->ncell = s->ncell; sl->plane = s->plane;
            sl->h = s->h; sl->H = s->H; sl->mu = s->mu; sl->rho = s->rho; sl->dt = s->dt; sl->chi = s->chi;
            sl->kernel = s->kernel; sl->advection = s->advection; sl->device = s->device;
            sl->stream = s->stream; sl->own_stream = false;
            sl->L = L; sl->P = Pseg;
            sl->sinv = s->sinv;
            sl->err_h = s->err_h;
            sl->err_d = s->err_d;
            memcpy(sl->hcoef, s->hcoef, sizeof(s->hcoef));
            sl->rank = (o.transport == IB_TRANSPORT_EMULATE) ? r : o.rank;
            sl->nl = nz;
            sl->z0 = nz * sl->rank;
            sl->wrap = 0;
            sl->nlocal = nz * s->plane;
            sl->hoff = s->plane;
            G->slab[r] = sl;
            CKC(alloc_fields(sl));
        }
        // Schur parts per slab: the smallest divisor Q of nz that gives >= 64k threads per
        // cut-axis pass (a slab is then Q consecutive parts of every line; R29)
        G->Q = 1;
        while (G->Q < nz && ((int64_t)s->plane * G->Q < 65536 || nz % G->Q != 0)) {
            ++G->Q;
            while (G->Q < nz && nz % G->Q != 0) ++G->Q;
            if ((int64_t)s->plane * G->Q >= 65536) break;
        }
        // (Q stays 1 when one part per slab already gives enough threads: every extra
        //  part adds one reduced-system row per line to the master exchange)
        // parts of at most 17 planes keep the forward phase's column in registers
        // (k_slab_fwd_reg: one read of d and one write of f* per cell, against the two
        // passes of k_slab_fwd), at Q + 2 more scalars per line in the exchange
        while (nz / G->Q > 17 && G->Q < nz && (G->Q + 1) * P <= kSlabMaxParts) {
            ++G->Q;
            while (G->Q < nz && nz % G->Q != 0) ++G->Q;
        }
        {
            const char* e = getenv("IBGM_SLAB_Q");   // A/B override
            if (e && atoi(e) > 0 && nz % atoi(e) == 0) G->Q = atoi(e);
        }
        if (nz / G->Q < 2) G->Q = nz / 2;
        if (G->Q * P > kSlabMaxParts) G->Q = kSlabMaxParts / P > 0 ? kSlabMaxParts / P : 1;   // reduced system <= kSlabMaxParts
        if (G->Q < 1) G->Q = 1;
        while (nz % G->Q != 0) --G->Q;
        {
            // exchange buffers (slab.cu layouts): a send and a receive buffer per rank; the
            // EMULATE context holds the P ranks' sets back to back
            const size_t NI = (size_t)(s->plane / P), nb = (size_t)G->Q + 2;
            const bool emu = (o.transport == IB_TRANSPORT_EMULATE);
            const size_t up = (size_t)P * G->Q * kSlabSlots * NI * (emu ? P : 1);
            const size_t dn = (size_t)P * 3 * nb * NI * (emu ? P : 1);
            CKC(cudaMalloc(&G->up_s, up * sizeof(double)));
            CKC(cudaMalloc(&G->dn_s, dn * sizeof(double)));
            CKC(cudaMalloc(&G->up_rv, up * sizeof(double)));
            CKC(cudaMalloc(&G->dn_rv, dn * sizeof(double)));
            CKC(cudaMemsetAsync(G->up_s, 0, up * sizeof(double), s->stream));
            CKC(cudaMemsetAsync(G->dn_s, 0, dn * sizeof(double), s->stream));
            CKC(cudaMemsetAsync(G->up_rv, 0, up * sizeof(double), s->stream));
            CKC(cudaMemsetAsync(G->dn_rv, 0, dn * sizeof(double), s->stream));
        }
        int rc;
        if ((rc = upload_coef(s, SYS_VISC, -kv, 1.0 + 2.0 * kv, -kv, 0)) != IB_OK) return rc;
        if ((rc = upload_coef(s, SYS_PSI, -kp, 1.0 + 2.0 * kp, -kp, 1)) != IB_OK) return rc;
        if (o.transport == IB_TRANSPORT_NCCL) {
            const char* e = nccl_load();
            if (e) return fail(IB_ENCCL, "%s", e);
            NcclUid id;
            memcpy(&id, o.nccl_id, sizeof(id));
            const int nr = nccl_comm_init(&G->comm, P, &id, o.rank);
            if (nr != 0) return fail(IB_ENCCL, "ncclCommInitRank: %s", nccl_error_string(nr));
            // (collective; without ncclCommSplit the slab look-ahead stays off)
            if (nccl_comm_split(G->comm, o.rank, &G->comm_side) != 0) G->comm_side = nullptr;
            if (nccl_comm_split(G->comm, o.rank, &G->comm_halo) != 0) G->comm_halo = nullptr;
        }
    }
    {
        // the look-ahead IB kernels (latency-bound, few blocks) get the higher priority so
        // that their blocks take SM slots as the psi passes' blocks retire
        int prio_lo = 0, prio_hi = 0;
        CKC(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
        // (A/B switches: IBGM_LOOKAHEAD=0 runs the IB phase in line; IBGM_SIDE_PRIO=0 gives
        //  the side stream the default priority)
        const char* ep = getenv("IBGM_SIDE_PRIO");
        const int prio = (ep && atoi(ep) == 0) ? prio_lo : prio_hi;
        CKC(cudaStreamCreateWithPriority(&s->side, cudaStreamNonBlocking, prio));
        CKC(cudaEventCreateWithFlags(&s->ev_fork, cudaEventDisableTiming));
        CKC(cudaEventCreateWithFlags(&s->ev_join, cudaEventDisableTiming));
        if (s->grp) {
            CKC(cudaStreamCreateWithFlags(&s->comm, cudaStreamNonBlocking));
            CKC(cudaEventCreateWithFlags(&s->ev_h0, cudaEventDisableTiming));
            CKC(cudaEventCreateWithFlags(&s->ev_h1, cudaEventDisableTiming));
        }
        const char* el = getenv("IBGM_LOOKAHEAD");
        s->lookahead = (el && atoi(el) == 0) ? 0 : 1;
    }
    // brick grid for the binned spread: 4^3 cells (3D) / 8^2 (2D)
    {
        const int B = (s->dim == 3) ? 4 : 8;     // kBrick3 / kBrick2 in ib.cu
        s->nb = (int)((s->n + B - 1) / B);
        s->nbricks = (s->dim == 3) ? (int64_t)s->nb * s->nb * s->nb : (int64_t)s->nb * s->nb;
        CKC(cudaMalloc(&s->bin_count, sizeof(int) * s->nbricks));
        CKC(cudaMalloc(&s->bin_start, sizeof(int) * s->nbricks));
        CKC(cudaMalloc(&s->bin_cursor, sizeof(int) * s->nbricks));
        CKC(cudaMalloc(&s->bin_list, sizeof(int) * s->nbricks));
        CKC(cudaMalloc(&s->bin_nlist, sizeof(int)));
        CKC(cudaMalloc(&s->bin_partial, sizeof(int) * ((s->nbricks + 1023) / 1024 + 1)));
    }
    CKC(cudaStreamSynchronize(s->stream));
    return IB_OK;
}

int ib_set_fields(ib_ctx* c, const double* u, const double* v, const double* w, const double* p)
{
    if (!c || !u || !v || (c->s.dim == 3 && !w)) return fail(IB_EINVAL, "null field pointer");
    Ctx* s = &c->s;
    const double* in[3] = {u, v, w};
    for (int r = 0; r < nslabs(s); ++r) {
        Ctx* sl = slab_at(s, r);
        const size_t fb = (size_t)sl->nlocal * sizeof(double);
        const size_t off = host_off(s, sl);
        const size_t full = (size_t)(sl->nl + (sl->wrap ? 0 : 2)) * sl->plane * sizeof(double);
        for (int q = 0; q < s->dim; ++q) {
            CKC(cudaMemcpyAsync(sl->u[q], in[q] + off, fb, cudaMemcpyHostToDevice, s->stream));
            CKC(cudaMemsetAsync(sl->nprev[q] - sl->hoff, 0, full, s->stream));
        }
        // p^{-1/2} = p (or 0), psi^{-1/2} = 0, so p* = p (R5)
        if (p) {
            CKC(cudaMemcpyAsync(sl->p, p + off, fb, cudaMemcpyHostToDevice, s->stream));
            CKC(cudaMemcpyAsync(sl->pstar, p + off, fb, cudaMemcpyHostToDevice, s->stream));
        } else {
            CKC(cudaMemsetAsync(sl->p, 0, fb, s->stream));
            CKC(cudaMemsetAsync(sl->pstar, 0, fb, s->stream));
        }
    }
    // X^n and U^{n-1} of the current time level (PAPER.md:686-697 restart from them)
    CKC(undo_lookahead(s));
    CKC(cudaStreamSynchronize(s->stream));
    clear_errors(s);
    s->step = 0;
    s->fields_set = true;
    s->u_halo_ready = false;
    return IB_OK;
}

int ib_set_boundary(ib_ctx* c, int64_t npts, const double* X, int64_t nedges, const int64_t* edges,
                    const double* kappa, const double* rest, const double* weight)
{
    if (!c) return fail(IB_EINVAL, "null context");
    Ctx* s = &c->s;
    if (npts < 0 || nedges < 0) return fail(IB_EINVAL, "negative count");
    if (npts > 0 && !X) return fail(IB_EINVAL, "null X");
    if (nedges > 0 && (!edges || !kappa)) return fail(IB_EINVAL, "null edges/kappa");
    if (npts >= (1LL << 31) || 2 * nedges >= (1LL << 31)) return fail(IB_EINVAL, "too many points/edges for int32 CSR");
    for (int64_t e = 0; e < nedges; ++e)
        if (edges[2 * e] < 0 || edges[2 * e] >= npts || edges[2 * e + 1] < 0 || edges[2 * e + 1] >= npts)
            return fail(IB_EINVAL, "edge %lld references a point out of range", (long long)e);
    CKC(cudaStreamSynchronize(s->stream));
    drop_graphs(s);
    free_lagrangian(s);
    clear_errors(s);
    s->step = 0;
    if (npts == 0) return IB_OK;
    const int d = s->dim;
    // internal order: Morton order of the cells holding the initial positions, so that
    // consecutive points (one CTA of the box-staged interpolation / spreading) are close
    // in space; ord[i] = caller index of internal point i, inv = its inverse
    std::vector<int32_t> ord(npts), inv(npts);
    {
        std::vector<uint64_t> key(npts);
        for (int64_t k = 0; k < npts; ++k) {
            uint64_t code = 0;
            for (int a = 0; a < d; ++a) {
                long long ci = (long long)floor(X[k * d + a] / s->h);
                ci %= s->n;
                if (ci < 0) ci += s->n;
                for (int bit = 0; bit < 11; ++bit) code |= (uint64_t)((ci >> bit) & 1) << (bit * d + a);
            }
            key[k] = code;
        }
        for (int64_t k = 0; k < npts; ++k) ord[k] = (int32_t)k;
        std::stable_sort(ord.begin(), ord.end(), [&](int32_t a, int32_t b) { return key[a] < key[b]; });
        for (int64_t i = 0; i < npts; ++i) inv[ord[i]] = (int32_t)i;
    }
    std::vector<double> Xi((size_t)npts * d);
    for (int64_t i = 0; i < npts; ++i)
        for (int a = 0; a < d; ++a) Xi[i * d + a] = X[(int64_t)ord[i] * d + a];
    // CSR adjacency in internal indices: every edge appears in the lists of both endpoints
    std::vector<int32_t> ptr(npts + 1, 0), nbr(2 * nedges);
    std::vector<double> kap(2 * nedges), rst(2 * nedges);
    for (int64_t e = 0; e < nedges; ++e) { ptr[inv[edges[2 * e]] + 1]++; ptr[inv[edges[2 * e + 1]] + 1]++; }
    for (int64_t k = 0; k < npts; ++k) ptr[k + 1] += ptr[k];
    std::vector<int32_t> fill(ptr.begin(), ptr.end() - 1);
    int has_rest = 0;
    for (int64_t e = 0; e < nedges; ++e) {
        const int64_t a = inv[edges[2 * e]], b = inv[edges[2 * e + 1]];
        const double L = rest ? rest[e] : 0.0;
        if (L != 0.0) has_rest = 1;
        int32_t ia = fill[a]++, ib = fill[b]++;
        nbr[ia] = (int32_t)b; kap[ia] = kappa[e]; rst[ia] = L;
        nbr[ib] = (int32_t)a; kap[ib] = kappa[e]; rst[ib] = L;
    }
    std::vector<double> wv(npts, 1.0);
    if (weight) for (int64_t k = 0; k < npts; ++k) wv[k] = weight[ord[k]];
    const size_t pb = (size_t)npts * d * sizeof(double);
    CKC(cudaMalloc(&s->X, pb));
    CKC(cudaMalloc(&s->Xh, pb));
    CKC(cudaMalloc(&s->Uprev, pb));
    CKC(cudaMalloc(&s->F, pb));
    CKC(cudaMalloc(&s->wgt, npts * sizeof(double)));
    CKC(cudaMalloc(&s->csr_ptr, (npts + 1) * sizeof(int32_t)));
    CKC(cudaMalloc(&s->bin_bid, npts * sizeof(int)));
    CKC(cudaMalloc(&s->bin_sorted, npts * sizeof(int)));
    const size_t ne2 = (size_t)(2 * nedges > 0 ? 2 * nedges : 1);
    CKC(cudaMalloc(&s->csr_nbr, ne2 * sizeof(int32_t)));
    CKC(cudaMalloc(&s->csr_kappa, ne2 * sizeof(double)));
    CKC(cudaMalloc(&s->csr_rest, ne2 * sizeof(double)));
    CKC(cudaMalloc(&s->Xold, pb));
    CKC(cudaMalloc(&s->Uold, pb));
    CKC(cudaMemsetAsync(s->Uold, 0, pb, s->stream));
    CKC(cudaMalloc(&s->pt_user, npts * sizeof(int32_t)));
    CKC(cudaMalloc(&s->lag_tmp, pb));
    CKC(cudaMemcpyAsync(s->pt_user, ord.data(), npts * sizeof(int32_t), cudaMemcpyHostToDevice, s->stream));
    CKC(cudaMemcpyAsync(s->X, Xi.data(), pb, cudaMemcpyHostToDevice, s->stream));
    CKC(cudaMemcpyAsync(s->Xh, Xi.data(), pb, cudaMemcpyHostToDevice, s->stream));
    CKC(cudaMemsetAsync(s->Uprev, 0, pb, s->stream));
    CKC(cudaMemsetAsync(s->F, 0, pb, s->stream));
    CKC(cudaMemcpyAsync(s->wgt, wv.data(), npts * sizeof(double), cudaMemcpyHostToDevice, s->stream));
    CKC(cudaMemcpyAsync(s->csr_ptr, ptr.data(), (npts + 1) * sizeof(int32_t), cudaMemcpyHostToDevice, s->stream));
    if (nedges > 0) {
        CKC(cudaMemcpyAsync(s->csr_nbr, nbr.data(), 2 * nedges * sizeof(int32_t), cudaMemcpyHostToDevice, s->stream));
        CKC(cudaMemcpyAsync(s->csr_kappa, kap.data(), 2 * nedges * sizeof(double), cudaMemcpyHostToDevice, s->stream));
        CKC(cudaMemcpyAsync(s->csr_rest, rst.data(), 2 * nedges * sizeof(double), cudaMemcpyHostToDevice, s->stream));
    }
    if (s->grp) {
        Group* G = s->grp;
        const int64_t cnt = npts * d;
        const int slots = (G->transport == IB_TRANSPORT_EMULATE) ? G->P : 1;
        CKC(cudaMalloc(&G->Upart, sizeof(double) * cnt * slots));
        CKC(cudaMalloc(&G->Ured, sizeof(double) * cnt));
        CKC(cudaMemsetAsync(G->Upart, 0, sizeof(double) * cnt * slots, s->stream));
        G->ucap = cnt;
        // (k_slab_select appends warp-aligned 32-slot chunks: up to npts rounded up to its 128-thread blocks)
        for (int r = 0; r < G->nloc; ++r) CKC(cudaMalloc(&G->sel[r], sizeof(int) * (size_t)((npts + 127) / 128 * 128)));
        CKC(cudaMalloc(&G->sel_cnt, sizeof(int) * G->nloc));
    }
    CKC(cudaStreamSynchronize(s->stream));
    s->npts = npts;
    s->nedges = nedges;
    s->has_rest = has_rest;
    return IB_OK;
}

int ib_set_fibers(ib_ctx* c, int32_t n_fibers, const int64_t* pts_per_fiber, const double* X, double sigma)
{
    if (!c || n_fibers < 0 || (n_fibers > 0 && (!pts_per_fiber || !X))) return fail(IB_EINVAL, "bad fibre arguments");
    if (c->s.dim != 2) return fail(IB_EINVAL, "ib_set_fibers builds closed 2D fibres");
    int64_t npts = 0;
    for (int f = 0; f < n_fibers; ++f) {
        if (pts_per_fiber[f] < 3) return fail(IB_EINVAL, "a closed fibre needs >= 3 points");
        npts += pts_per_fiber[f];
    }
    std::vector<int64_t> edges(2 * npts);
    std::vector<double> kap(npts), w(npts);
    int64_t off = 0;
    for (int f = 0; f < n_fibers; ++f) {
        const int64_t m = pts_per_fiber[f];
        const double hs = 1.0 / (double)m;
        for (int64_t k = 0; k < m; ++k) {
            edges[2 * (off + k)] = off + k;
            edges[2 * (off + k) + 1] = off + (k + 1) % m;
            kap[off + k] = sigma / (hs * hs);   // sigma D_s^- D_s^+ (L = 0)
            w[off + k] = hs;                    // trapezoidal weight
        }
        off += m;
    }
    return ib_set_boundary(c, npts, X, npts, edges.data(), kap.data(), nullptr, w.data());
}

static cudaError_t clear3(Ctx* s, double* const* f)
{
    const size_t fb = (size_t)s->nlocal * sizeof(double);
    for (int q = 0; q < s->dim; ++q) {
        cudaError_t e = cudaMemsetAsync(f[q], 0, fb, s->stream);
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

// one phase, bracketed by an event pair when profiling
#define PHASE(id, call)                                                          \
    do {                                                                         \
        if (s->profiling) CKC(cudaEventRecord(s->ev[id][0], s->stream));         \
        CKC(call);                                                               \
        if (s->profiling) {                                                      \
            CKC(cudaEventRecord(s->ev[id][1], s->stream));                       \
            s->ph_pending[id] = true;                                            \
        }                                                                        \
    } while (0)

// a transport call (returns 0 or a cudaError_t / ncclResult_t)
#define CKG(call)                                                                                   \
    do {                                                                                            \
        const int rc_ = (call);                                                                     \
        if (rc_ != 0) {                                                                             \
            if (s->grp->transport == IB_TRANSPORT_NCCL)                                             \
                return fail(IB_ENCCL, "%s: %s (%s:%d)", #call, nccl_error_string(rc_), __FILE__, __LINE__); \
            return fail(IB_ECUDA, "%s: %s (%s:%d)", #call, cudaGetErrorString((cudaError_t)rc_), __FILE__, \
                        __LINE__);                                                                  \
        }                                                                                           \
    } while (0)

// every local slab
#define FOR_SLABS(call)                                          \
    do {                                                         \
        for (int r_ = 0; r_ < s->grp->nloc; ++r_) {              \
            Ctx* sl = s->grp->slab[r_];                          \
            (void)sl;                                            \
            CKC(call);                                           \
        }                                                        \
    } while (0)

static int enqueue_step(Ctx* s, int first);
static int enqueue_step_slab(Ctx* s, int first);
static bool early_halo_on(const Ctx* s);

static void swap_state(Ctx* s)
{
    for (int r = 0; r < nslabs(s); ++r) {
        Ctx* sl = slab_at(s, r);
        for (int q = 0; q < s->dim; ++q) {
            std::swap(sl->u[q], sl->st[q]);
            std::swap(sl->nadv[q], sl->nprev[q]);
        }
    }
    s->parity ^= 1;
}

static int enqueue_any(Ctx* s, int first) { return s->grp ? enqueue_step_slab(s, first) : enqueue_step(s, first); }

static bool lookahead_on(const Ctx* s)
{
    // on z-slabs the look-ahead's all-reduce of U needs its own communicator (NCCL)
    const bool slab_ok = !s->grp || s->grp->transport == IB_TRANSPORT_EMULATE || s->grp->comm_side != nullptr;
    return s->lookahead && slab_ok && s->npts > 0 && !s->profiling && !s->debug_keep_f;
}

// A captured step keeps the stream priorities as kernel-node priorities (the look-ahead
// IB kernels were launched on the high-priority side stream), but a graph launch runs
// every node at the priority of the stream it is launched into unless instantiated
// with cudaGraphInstantiateFlagUseNodePriority.  IBGM_NODE_PRIO selects:
//   0 (default) the launch stream's priority for every node;
//   1 the captured priorities (IB look-ahead above the psi passes);
//   2 as 1, and list the kernel nodes with their priorities on stderr;
//   3 inverted (the psi passes above the IB look-ahead).
// Measured (graph ms/step, config 4 / config 3): 0: 4.643-4.672 / 0.1623-0.1638;
// 1: 4.849 / 0.1638; 3: 4.663 / 0.1711 -- the block scheduler's default interleaving wins.
static cudaError_t instantiate_step_graph(Ctx* s, cudaGraph_t g, cudaGraphExec_t* ge)
{
    (void)s;
    const char* e = getenv("IBGM_NODE_PRIO");
    const int mode = e ? atoi(e) : 0;
    if (mode == 3) {
        int lo = 0, hi = 0;
        cudaDeviceGetStreamPriorityRange(&lo, &hi);
        size_t nn = 0;
        cudaGraphGetNodes(g, nullptr, &nn);
        std::vector<cudaGraphNode_t> nodes(nn);
        cudaGraphGetNodes(g, nodes.data(), &nn);
        for (size_t i = 0; i < nn; ++i) {
            cudaGraphNodeType t;
            cudaGraphNodeGetType(nodes[i], &t);
            if (t != cudaGraphNodeTypeKernel) continue;
            cudaLaunchAttributeValue v{};
            cudaGraphKernelNodeGetAttribute(nodes[i], cudaLaunchAttributePriority, &v);
            v.priority = (v.priority == hi) ? lo : hi;
            cudaGraphKernelNodeSetAttribute(nodes[i], cudaLaunchAttributePriority, &v);
        }
    }
    if (mode == 2) {
        size_t nn = 0;
        cudaGraphGetNodes(g, nullptr, &nn);
        std::vector<cudaGraphNode_t> nodes(nn);
        cudaGraphGetNodes(g, nodes.data(), &nn);
        for (size_t i = 0; i < nn; ++i) {
            cudaGraphNodeType t;
            cudaGraphNodeGetType(nodes[i], &t);
            if (t != cudaGraphNodeTypeKernel) continue;
            cudaLaunchAttributeValue v{};
            cudaGraphKernelNodeGetAttribute(nodes[i], cudaLaunchAttributePriority, &v);
            cudaKernelNodeParams kp{};
            cudaGraphKernelNodeGetParams(nodes[i], &kp);
            const char* nm = nullptr;
            cudaFuncGetName(&nm, kp.func);
            fprintf(stderr, "[ibgm] graph kernel node %zu prio %d %s\n", i, v.priority, nm ? nm : "?");
        }
    }
    return cudaGraphInstantiateWithFlags(ge, g, mode ? cudaGraphInstantiateFlagUseNodePriority : 0);
}

// Steps 1-2 (interpolate + evolve, force, spread) on context view v
static cudaError_t enqueue_ib(Ctx* v, int first)
{
    cudaError_t e = launch_interp_evolve(v, first);
    if (e == cudaSuccess) e = launch_force(v);
    if (e == cudaSuccess) e = launch_spread(v);
    return e;
}

int ib_step(ib_ctx* c, int64_t nsteps)
{
    if (!c) return fail(IB_EINVAL, "null context");
    Ctx* s = &c->s;
    if (!s->fields_set) return fail(IB_ESTATE, "ib_step before ib_set_fields");
    if (nsteps < 0) return fail(IB_EINVAL, "nsteps < 0");
    {
        const int pe = poll_errors(s);
        if (pe != IB_OK) return pe;
    }
    for (int64_t t = 0; t < nsteps; ++t) {
        const int first = (s->step == 0);
        // (on z-slabs a captured step expects the u halos from the step before: after
        //  ib_set_fields / ib_set_state one step runs eagerly with the full exchange)
        const bool halo_ok = !s->grp || s->u_halo_ready || !early_halo_on(s);
        if (!first && !s->profiling && s->use_graphs && !s->debug_keep_f && halo_ok) {
            // replay the captured regular step for the current pointer parity and
            // look-ahead state
            const int par = s->parity * 2 + (s->ib_ahead ? 1 : 0);
            if (!s->gvalid[par]) {
                cudaGraph_t g;
                const int64_t l0 = total_launches(s);
                CKC(cudaStreamBeginCapture(s->stream, cudaStreamCaptureModeThreadLocal));
                const int rc = enqueue_any(s, 0);
                cudaError_t ce = cudaStreamEndCapture(s->stream, &g);
                if (rc != IB_OK) return rc;
                CKC(ce);
                CKC(instantiate_step_graph(s, g, &s->gexec[par]));
                cudaGraphDestroy(g);
                s->gvalid[par] = true;
                s->glaunches[par] = total_launches(s) - l0;
                s->launches -= s->glaunches[par];   // captured, not launched
            }
            CKC(cudaGraphLaunch(s->gexec[par], s->stream));
            s->launches += s->glaunches[par];
            s->ib_ahead = lookahead_on(s);   // what the captured step leaves behind
        } else {
            const int rc = enqueue_any(s, first);
            if (rc != IB_OK) return rc;
        }
        swap_state(s);
        s->step++;
        if (s->check_every > 0 && s->step % s->check_every == 0) CKC(enqueue_check(s));
        if (s->profiling) {
            CKC(cudaStreamSynchronize(s->stream));
            for (int ph = 0; ph < IB_NPHASES; ++ph) {
                if (!s->ph_pending[ph]) continue;
                float ms = 0.f;
                CKC(cudaEventElapsedTime(&ms, s->ev[ph][0], s->ev[ph][1]));
                s->ph_ms[ph] += ms;
                s->ph_cnt[ph] += 1;
                s->ph_pending[ph] = false;
            }
        }
    }
    return poll_errors(s);
}

// all device work of one time step (Steps 1a-3f), enqueued on the context's stream
static int enqueue_step(Ctx* s, int first)
{
    const int d = s->dim;
    {
        // n = 0: no N(u^{-1}); the history G starts as 0 + (2/rho) f
        if (first) PHASE(IB_PH_CLEAR, clear3(s, s->nprev));
        if (s->debug_keep_f && s->npts > 0) PHASE(IB_PH_CLEAR, clear3(s, s->f));
        if (s->npts > 0 && !s->ib_ahead) {
            // Step 1 (interpolate, evolve) and Step 2 (force, spread)
            PHASE(IB_PH_INTERP, launch_interp_evolve(s, first));
            PHASE(IB_PH_FORCE, launch_force(s));
            PHASE(IB_PH_SPREAD, launch_spread(s));
        }
        // Steps 3a-3c: p*, explicit momentum, x sweep
        PHASE(IB_PH_S1, launch_s1_x(s, first));
        // Step 3d: the remaining Douglas sweeps; the last one forms u^{n+1}
        if (d == 3) {
            PHASE(IB_PH_SWEEP_Y, launch_sweep_mid(s, 1));
            PHASE(IB_PH_SWEEP_Z, launch_sweep_last(s, 2));
        } else {
            PHASE(IB_PH_SWEEP_Y, launch_sweep_last(s, 1));
        }
        // look-ahead: Steps 1-2 of step n+1 need only u^{n+1} (now in st), X and U^n;
        // they spread into N(u^n) (nadv, the next step's history G) while the psi passes
        // below run on the main stream
        const bool look = lookahead_on(s);
        if (look) {
            Ctx v = *s;
            for (int q = 0; q < 3; ++q) { v.u[q] = s->st[q]; v.nprev[q] = s->nadv[q]; }
            v.stream = s->side;
            v.launches = 0;
            CKC(cudaEventRecord(s->ev_fork, s->stream));
            CKC(cudaStreamWaitEvent(s->side, s->ev_fork, 0));
            CKC(enqueue_ib(&v, 0));
            CKC(cudaEventRecord(s->ev_join, s->side));
            s->launches += v.launches;
        }
        // Step 3e: RHS and the psi factors (last axis first); Step 3f fused
        PHASE(IB_PH_DIVPSI, launch_div_psi_first(s, d - 1));
        if (d == 3) PHASE(IB_PH_PSI_Y, launch_psi_mid(s, 1));
        PHASE(IB_PH_PSI_X, launch_psi_last_x(s));
        if (look) CKC(cudaStreamWaitEvent(s->stream, s->ev_join, 0));
        s->ib_ahead = look;
    }
    return IB_OK;
}

static double* fld_u0(Ctx* c) { return c->u[0]; }
static double* fld_u1(Ctx* c) { return c->u[1]; }
static double* fld_u2(Ctx* c) { return c->u[2]; }
static double* fld_pstar(Ctx* c) { return c->pstar; }
static double* fld_st_last2(Ctx* c) { return c->st[1]; }
static double* fld_st0(Ctx* c) { return c->st[0]; }
static double* fld_st1(Ctx* c) { return c->st[1]; }

// the early u halos (A/B switch: IBGM_EARLY_HALO=0); NCCL needs the third communicator
static bool early_halo_on(const Ctx* s)
{
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("IBGM_EARLY_HALO");
        v = (e && atoi(e) == 0) ? 0 : 1;
    }
    const Group* G = s->grp;
    return v == 1 && G && s->comm && (G->transport == IB_TRANSPORT_EMULATE || G->comm_halo != nullptr);
}
static double* fld_st_last3(Ctx* c) { return c->st[2]; }

// The same step on a z-slab decomposition: each phase runs on every local slab, with
// the exchanges between phases (a12: halos, a13: the cut-axis line solves, and the
// sum of the partial interpolations).
// Steps 1-2 on a z-slab decomposition (top: the context holding the Lagrangian state,
// views: its slabs, all possibly re-pointed for the look-ahead; side: the all-reduce
// runs on the look-ahead communicator)
static int enqueue_ib_slab(Ctx* s, Ctx* top, Ctx* const* views, int first, bool side)
{
    Group* G = s->grp;
    const int d = s->dim;
    if (s->profiling) CKC(cudaEventRecord(s->ev[IB_PH_INTERP][0], top->stream));
    // Step 1a: each slab interpolates from the nodes it owns; U^n = sum over slabs
    const int64_t cnt = top->npts * d;
    for (int r = 0; r < G->nloc; ++r) {
        double* part = G->Upart + ((G->transport == IB_TRANSPORT_EMULATE) ? (size_t)r * cnt : 0);
        CKC(slab_interp_part(top, views[r], part, G->sel[r], G->sel_cnt + r));
    }
    CKG(group_allreduce_U(G, top, top->stream, side));
    // Steps 1b-1c on every rank (identical arithmetic on identical U^n)
    CKC(slab_evolve(top, G->Ured, first));
    if (s->profiling) {
        CKC(cudaEventRecord(s->ev[IB_PH_INTERP][1], top->stream));
        s->ph_pending[IB_PH_INTERP] = true;
    }
    if (s->profiling) CKC(cudaEventRecord(s->ev[IB_PH_FORCE][0], top->stream));
    CKC(launch_force(top));
    if (s->profiling) {
        CKC(cudaEventRecord(s->ev[IB_PH_FORCE][1], top->stream));
        s->ph_pending[IB_PH_FORCE] = true;
    }
    if (s->profiling) CKC(cudaEventRecord(s->ev[IB_PH_SPREAD][0], top->stream));
    for (int r = 0; r < G->nloc; ++r) CKC(slab_spread_part(top, views[r], G->sel[r], G->sel_cnt + r));
    if (s->profiling) {
        CKC(cudaEventRecord(s->ev[IB_PH_SPREAD][1], top->stream));
        s->ph_pending[IB_PH_SPREAD] = true;
    }
    return IB_OK;
}

// The same step on a z-slab decomposition: each phase runs on every local slab, with
// the exchanges between phases (a12: halos, a13: the cut-axis line solves, and the
// sum of the partial interpolations).
static int enqueue_step_slab(Ctx* s, int first)
{
    const int d = s->dim;
    Group* G = s->grp;
    if (first) FOR_SLABS(clear3(sl, sl->nprev));
    if (s->debug_keep_f && s->npts > 0) FOR_SLABS(clear3(sl, sl->f));
    if (s->npts > 0 && !s->ib_ahead) {
        const int rc = enqueue_ib_slab(s, s, G->slab, first, false);
        if (rc != IB_OK) return rc;
    }
    if (s->profiling) CKC(cudaEventRecord(s->ev[IB_PH_S1][0], s->stream));
    // halos for Steps 3a-3b: u (every component) on both sides, p* below -- u's already
    // arrived during the previous step's psi passes when u_halo_ready
    {
        HaloSpec h[4] = {{fld_u0, true, true}, {fld_u1, true, true}, {fld_u2, true, true}, {fld_pstar, true, false}};
        if (d == 2) h[2] = h[3];
        if (s->u_halo_ready && early_halo_on(s)) CKG(group_halo(G, 1, h + d, s->stream));
        else CKG(group_halo(G, d + 1, h, s->stream));
    }
    FOR_SLABS(launch_s1_x(sl, first));
    if (s->profiling) {
        CKC(cudaEventRecord(s->ev[IB_PH_S1][1], s->stream));
        s->ph_pending[IB_PH_S1] = true;
    }
    const int last_ph = (d == 3) ? IB_PH_SWEEP_Z : IB_PH_SWEEP_Y;
    if (d == 3) {
        if (s->profiling) CKC(cudaEventRecord(s->ev[IB_PH_SWEEP_Y][0], s->stream));
        FOR_SLABS(launch_sweep_mid(sl, 1));
        if (s->profiling) {
            CKC(cudaEventRecord(s->ev[IB_PH_SWEEP_Y][1], s->stream));
            s->ph_pending[IB_PH_SWEEP_Y] = true;
        }
    }
    // the last Douglas sweep along the cut axis (distributed Schur solve)
    if (s->profiling) CKC(cudaEventRecord(s->ev[last_ph][0], s->stream));
    FOR_SLABS(slab_sweep_last_fwd(sl, G));
    if (G->visc_local) {
        // S^{-1} diagonal: each part's y from its neighbour parts (nearest-neighbour exchange)
        CKG(group_edge(G, d, s->stream));
    } else {
        CKG(group_up(G, 2 * d, s->stream));
        CKC(slab_master(G->slab[0], G, SYS_VISC, d, 2 * d, 0));
        CKG(group_dn(G, d, s->stream));
    }
    FOR_SLABS(slab_sweep_last_corr(sl, G));
    if (s->profiling) {
        CKC(cudaEventRecord(s->ev[last_ph][1], s->stream));
        s->ph_pending[last_ph] = true;
    }
    // look-ahead (as on one GPU): Steps 1-2 of step n+1 need u^{n+1} (now in st, owned
    // planes only), X and U^n; on the side stream, spreading into N(u^n) = the next
    // step's history, while the psi passes below run
    const bool look = lookahead_on(s);
    Ctx vtop = *s;
    std::vector<Ctx> vsl(look ? G->nloc : 0);
    Ctx* vptr[kMaxRanks];
    if (look) {
        vtop.stream = s->side;
        vtop.launches = 0;
        for (int r = 0; r < G->nloc; ++r) {
            vsl[r] = *G->slab[r];
            for (int q = 0; q < 3; ++q) { vsl[r].u[q] = G->slab[r]->st[q]; vsl[r].nprev[q] = G->slab[r]->nadv[q]; }
            vsl[r].stream = s->side;
            vsl[r].launches = 0;
            vptr[r] = &vsl[r];
        }
        CKC(cudaEventRecord(s->ev_fork, s->stream));
        CKC(cudaStreamWaitEvent(s->side, s->ev_fork, 0));
        const int rc = enqueue_ib_slab(s, &vtop, vptr, 0, true);
        if (rc != IB_OK) return rc;
        CKC(cudaEventRecord(s->ev_join, s->side));
        s->launches += vtop.launches;
        for (int r = 0; r < G->nloc; ++r) s->launches += vsl[r].launches;
    }
    // Step 3e: D.u^{n+1} needs u^{n+1}_last one plane above
    if (s->profiling) CKC(cudaEventRecord(s->ev[IB_PH_DIVPSI][0], s->stream));
    {
        HaloSpec h[1] = {{d == 3 ? fld_st_last3 : fld_st_last2, false, true}};
        CKG(group_halo(G, 1, h, s->stream));
    }
    // the rest of u^{n+1}'s halos for the next step's S1, on the comm stream while the psi
    // passes run (u^{n+1} is final here; joined at the end of the step)
    const bool early = early_halo_on(s);
    if (early) {
        HaloSpec h[3] = {{fld_st0, true, true}, {fld_st1, true, true}, {d == 3 ? fld_st_last3 : fld_st_last2, true, false}};
        if (d == 2) h[1] = h[2];
        CKC(cudaEventRecord(s->ev_h0, s->stream));
        CKC(cudaStreamWaitEvent(s->comm, s->ev_h0, 0));
        CKG(group_halo(G, d, h, s->comm, G->comm_halo));
        CKC(cudaEventRecord(s->ev_h1, s->comm));
    }
    FOR_SLABS(slab_divpsi_fwd(sl, G));
    CKG(group_up(G, 4, s->stream));
    CKC(slab_master(G->slab[0], G, SYS_PSI, 1, 4, 1));
    CKG(group_dn(G, 1, s->stream));
    FOR_SLABS(slab_divpsi_corr(sl, G));
    if (s->profiling) {
        CKC(cudaEventRecord(s->ev[IB_PH_DIVPSI][1], s->stream));
        s->ph_pending[IB_PH_DIVPSI] = true;
    }
    if (d == 3) {
        if (s->profiling) CKC(cudaEventRecord(s->ev[IB_PH_PSI_Y][0], s->stream));
        FOR_SLABS(launch_psi_mid(sl, 1));
        if (s->profiling) {
            CKC(cudaEventRecord(s->ev[IB_PH_PSI_Y][1], s->stream));
            s->ph_pending[IB_PH_PSI_Y] = true;
        }
    }
    if (s->profiling) CKC(cudaEventRecord(s->ev[IB_PH_PSI_X][0], s->stream));
    FOR_SLABS(launch_psi_last_x(sl));
    if (s->profiling) {
        CKC(cudaEventRecord(s->ev[IB_PH_PSI_X][1], s->stream));
        s->ph_pending[IB_PH_PSI_X] = true;
    }
    if (look) CKC(cudaStreamWaitEvent(s->stream, s->ev_join, 0));
    s->ib_ahead = look;
    if (early) CKC(cudaStreamWaitEvent(s->stream, s->ev_h1, 0));
    s->u_halo_ready = early;
    return IB_OK;
}

int ib_set_debug(ib_ctx* c, int32_t flags)
{
    if (!c) return fail(IB_EINVAL, "null context");
    Ctx* s = &c->s;
    if (((flags >> 1) & 7) > 6 || ((flags >> 4) & 7) > 5 || (flags >> 7) != 0)
        return fail(IB_EINVAL, "debug flags 0x%x: spreading method > 6, interpolation method > 5 or unknown bits",
                    (unsigned)flags);
    const int keep = (flags & 1) != 0;
    if (keep && !s->debug_keep_f && s->ib_ahead)
        return fail(IB_ESTATE, "set debug bit 0 before stepping: the next step's IB phase has already run");
    for (int r = 0; r < nslabs(s); ++r) {
        Ctx* sl = slab_at(s, r);
        if (keep && !sl->f[0])
            for (int q = 0; q < s->dim; ++q) CKC(field_alloc(sl, &sl->f[q]));
    }
    drop_graphs(s);
    s->debug_keep_f = keep;
    s->spread_mode = (flags >> 1) & 7;   // bits 1-3: spreading method (include/ibgm.h)
    s->interp_mode = (flags >> 4) & 7;   // bits 4-6: interpolation method
    return IB_OK;
}

int ib_set_profiling(ib_ctx* c, int32_t on)
{
    if (!c) return fail(IB_EINVAL, "null context");
    Ctx* s = &c->s;
    if (on && !s->ev_made) {
        for (int ph = 0; ph < IB_NPHASES; ++ph)
            for (int k = 0; k < 2; ++k) CKC(cudaEventCreate(&s->ev[ph][k]));
        s->ev_made = true;
    }
    for (int ph = 0; ph < IB_NPHASES; ++ph) { s->ph_ms[ph] = 0; s->ph_cnt[ph] = 0; s->ph_pending[ph] = false; }
    s->profiling = on ? 1 : 0;
    return IB_OK;
}

int ib_get_phase_times(ib_ctx* c, double* ms, int64_t* count)
{
    if (!c) return fail(IB_EINVAL, "null context");
    for (int ph = 0; ph < IB_NPHASES; ++ph) {
        if (ms) ms[ph] = c->s.ph_ms[ph];
        if (count) count[ph] = c->s.ph_cnt[ph];
    }
    return IB_OK;
}

int ib_sync(ib_ctx* c)
{
    if (!c) return fail(IB_EINVAL, "null context");
    CKC(cudaStreamSynchronize(c->s.stream));
    return poll_errors(&c->s);
}

int ib_set_check_interval(ib_ctx* c, int64_t every)
{
    if (!c) return fail(IB_EINVAL, "null context");
    if (every < 0) return fail(IB_EINVAL, "check interval must be >= 0");
    c->s.check_every = every;
    return IB_OK;
}

int ib_get_fields(ib_ctx* c, double* u, double* v, double* w, double* p, double* psi, double* X, double* U)
{
    if (!c) return fail(IB_EINVAL, "null context");
    Ctx* s = &c->s;
    double* out[3] = {u, v, w};
    for (int r = 0; r < nslabs(s); ++r) {
        Ctx* sl = slab_at(s, r);
        const size_t fb = (size_t)sl->nlocal * sizeof(double);
        const size_t off = host_off(s, sl);
        for (int q = 0; q < s->dim; ++q)
            if (out[q]) CKC(cudaMemcpyAsync(out[q] + off, sl->u[q], fb, cudaMemcpyDeviceToHost, s->stream));
        if (p) CKC(cudaMemcpyAsync(p + off, sl->p, fb, cudaMemcpyDeviceToHost, s->stream));
        if (psi) {
            // the state keeps p* = p + psi; psi^{n-1/2} = p* - p
            CKC(launch_sub(sl, sl->pstar, sl->p, sl->tmp));
            CKC(cudaMemcpyAsync(psi + off, sl->tmp, fb, cudaMemcpyDeviceToHost, s->stream));
        }
    }
    // with the next step's IB phase already done, X^n and U^{n-1} are in Xold/Uold
    CKC(points_out(s, s->ib_ahead ? s->Xold : s->X, X));
    CKC(points_out(s, s->ib_ahead ? s->Uold : s->Uprev, U));
    CKC(cudaStreamSynchronize(s->stream));
    return IB_OK;
}

// ---------------------------------------------------------------------------------
// Checkpoint / resume: the complete state that the next step reads.
// Blob = StateHdr, then per local slab u[d], G[d] (the momentum history N(u^{n-1}) +
// (2/rho) f of a look-ahead), p, p* (nlocal doubles each), then the Lagrangian X, U^{n-1},
// X_old, U_old ([npts][d] each, internal order) and the internal order pt_user[npts].
// ---------------------------------------------------------------------------------
struct StateHdr {
    uint64_t magic;
    int32_t version, dim;
    int64_t n, nlocal_total, npts, step;
    int32_t ib_ahead, nslabs, rank, nranks;
    double dt, mu, rho, H;
};
static const uint64_t kStateMagic = 0x31564154534D4749ull;   // "IGMSTAV1"

static int64_t state_bytes(Ctx* s)
{
    int64_t cells = 0;
    for (int r = 0; r < nslabs(s); ++r) cells += slab_at(s, r)->nlocal;
    return (int64_t)sizeof(StateHdr) + cells * (2 * s->dim + 2) * (int64_t)sizeof(double) +
           s->npts * s->dim * 4 * (int64_t)sizeof(double) + s->npts * (int64_t)sizeof(int32_t);
}

int ib_state_size(ib_ctx* c, int64_t* bytes)
{
    if (!c || !bytes) return fail(IB_EINVAL, "null argument");
    *bytes = state_bytes(&c->s);
    return IB_OK;
}

int ib_get_state(ib_ctx* c, void* buf, int64_t bytes)
{
    if (!c || !buf) return fail(IB_EINVAL, "null argument");
    Ctx* s = &c->s;
    if (!s->fields_set) return fail(IB_ESTATE, "ib_get_state before ib_set_fields");
    if (bytes < state_bytes(s)) return fail(IB_EINVAL, "state buffer of %lld bytes < %lld", (long long)bytes,
                                            (long long)state_bytes(s));
    StateHdr h;
    memset(&h, 0, sizeof(h));
    h.magic = kStateMagic; h.version = 1; h.dim = s->dim; h.n = s->n; h.npts = s->npts; h.step = s->step;
    h.ib_ahead = s->ib_ahead ? 1 : 0; h.nslabs = nslabs(s);
    h.rank = s->grp ? s->grp->rank : 0; h.nranks = s->grp ? s->grp->P : 1;
    h.dt = s->dt; h.mu = s->mu; h.rho = s->rho; h.H = s->H;
    for (int r = 0; r < nslabs(s); ++r) h.nlocal_total += slab_at(s, r)->nlocal;
    memcpy(buf, &h, sizeof(h));
    char* q = (char*)buf + sizeof(h);
    for (int r = 0; r < nslabs(s); ++r) {
        Ctx* sl = slab_at(s, r);
        const size_t fb = (size_t)sl->nlocal * sizeof(double);
        double* flds[8] = {sl->u[0], sl->u[1], sl->u[2], sl->nprev[0], sl->nprev[1], sl->nprev[2], sl->p, sl->pstar};
        for (int k = 0; k < 8; ++k) {
            if (k % 3 >= s->dim && k < 6) continue;
            CKC(cudaMemcpyAsync(q, flds[k], fb, cudaMemcpyDeviceToHost, s->stream));
            q += fb;
        }
    }
    if (s->npts) {
        const size_t pb = (size_t)s->npts * s->dim * sizeof(double);
        double* lag[4] = {s->X, s->Uprev, s->Xold, s->Uold};
        for (int k = 0; k < 4; ++k) { CKC(cudaMemcpyAsync(q, lag[k], pb, cudaMemcpyDeviceToHost, s->stream)); q += pb; }
        CKC(cudaMemcpyAsync(q, s->pt_user, (size_t)s->npts * sizeof(int32_t), cudaMemcpyDeviceToHost, s->stream));
    }
    CKC(cudaStreamSynchronize(s->stream));
    return poll_errors(s);
}

int ib_set_state(ib_ctx* c, const void* buf, int64_t bytes)
{
    if (!c || !buf) return fail(IB_EINVAL, "null argument");
    Ctx* s = &c->s;
    StateHdr h;
    if (bytes < (int64_t)sizeof(h)) return fail(IB_EINVAL, "state buffer too small");
    memcpy(&h, buf, sizeof(h));
    int64_t cells = 0;
    for (int r = 0; r < nslabs(s); ++r) cells += slab_at(s, r)->nlocal;
    if (h.magic != kStateMagic || h.version != 1) return fail(IB_EINVAL, "not an ib_get_state blob");
    if (h.dim != s->dim || h.n != s->n || h.nlocal_total != cells || h.nslabs != nslabs(s) ||
        h.rank != (s->grp ? s->grp->rank : 0) || h.nranks != (s->grp ? s->grp->P : 1))
        return fail(IB_EINVAL, "state blob is for another grid or decomposition");
    if (h.dt != s->dt || h.mu != s->mu || h.rho != s->rho || h.H != s->H)
        return fail(IB_EINVAL, "state blob is for other parameters (dt, mu, rho or H)");
    if (h.npts != s->npts) return fail(IB_EINVAL, "state blob has %lld points, the context %lld (call ib_set_boundary "
                                              "with the same boundary first)", (long long)h.npts, (long long)s->npts);
    if (bytes < state_bytes(s)) return fail(IB_EINVAL, "state buffer truncated");
    const char* q = (const char*)buf + sizeof(h);
    if (s->npts) {
        // the internal point order must be this context's (same boundary, same Morton order)
        std::vector<int32_t> ord(s->npts);
        const char* qo = q + (size_t)cells * (2 * s->dim + 2) * sizeof(double) + (size_t)s->npts * s->dim * 4 * sizeof(double);
        CKC(cudaMemcpyAsync(ord.data(), s->pt_user, (size_t)s->npts * sizeof(int32_t), cudaMemcpyDeviceToHost, s->stream));
        CKC(cudaStreamSynchronize(s->stream));
        if (memcmp(ord.data(), qo, (size_t)s->npts * sizeof(int32_t)) != 0)
            return fail(IB_EINVAL, "state blob was taken with another immersed boundary (point order differs)");
    }
    for (int r = 0; r < nslabs(s); ++r) {
        Ctx* sl = slab_at(s, r);
        const size_t fb = (size_t)sl->nlocal * sizeof(double);
        double* flds[8] = {sl->u[0], sl->u[1], sl->u[2], sl->nprev[0], sl->nprev[1], sl->nprev[2], sl->p, sl->pstar};
        for (int k = 0; k < 8; ++k) {
            if (k % 3 >= s->dim && k < 6) continue;
            CKC(cudaMemcpyAsync(flds[k], q, fb, cudaMemcpyHostToDevice, s->stream));
            q += fb;
        }
    }
    if (s->npts) {
        const size_t pb = (size_t)s->npts * s->dim * sizeof(double);
        double* lag[4] = {s->X, s->Uprev, s->Xold, s->Uold};
        for (int k = 0; k < 4; ++k) { CKC(cudaMemcpyAsync(lag[k], q, pb, cudaMemcpyHostToDevice, s->stream)); q += pb; }
        // (X^{n+1/2} and F are intermediates of an IB phase, not state: the next step
        //  reads only G, X and U^{n-1})
    }
    // the blob may come from pinned memory the caller reuses right after the call
    CKC(cudaStreamSynchronize(s->stream));
    clear_errors(s);
    s->step = h.step;
    s->ib_ahead = h.ib_ahead != 0;
    s->fields_set = true;
    s->u_halo_ready = false;
    return IB_OK;
}

int ib_get_aux(ib_ctx* c, double* fu, double* fv, double* fw, double* nu, double* nv, double* nw, double* F,
               double* Xh)
{
    if (!c) return fail(IB_EINVAL, "null context");
    Ctx* s = &c->s;
    double* fo[3] = {fu, fv, fw};
    double* no[3] = {nu, nv, nw};
    if ((fu || fv || fw) && !s->debug_keep_f) return fail(IB_ESTATE, "f is only kept with ib_set_debug(ctx, 1)");
    for (int r = 0; r < nslabs(s); ++r) {
        Ctx* sl = slab_at(s, r);
        const size_t fb = (size_t)sl->nlocal * sizeof(double);
        const size_t off = host_off(s, sl);
        for (int q = 0; q < s->dim; ++q) {
            if (fo[q]) CKC(cudaMemcpyAsync(fo[q] + off, sl->f[q], fb, cudaMemcpyDeviceToHost, s->stream));
            if (no[q]) CKC(cudaMemcpyAsync(no[q] + off, sl->nprev[q], fb, cudaMemcpyDeviceToHost, s->stream));
        }
    }
    CKC(points_out(s, s->F, F));
    CKC(points_out(s, s->Xh, Xh));
    CKC(cudaStreamSynchronize(s->stream));
    return IB_OK;
}

int ib_line_solve(ib_ctx* c, int32_t axis, double kappa, const double* d, double* x)
{
    if (!c || !d || !x) return fail(IB_EINVAL, "null argument");
    Ctx* s = &c->s;
    if (axis < 0 || axis >= s->dim) return fail(IB_EINVAL, "axis %d out of range", axis);
    if (!(kappa >= 0)) return fail(IB_EINVAL, "kappa must be >= 0");
    // the exact mean correction is applied to the ill-conditioned systems (kappa > 1, R16)
    const int mf = kappa > 1.0 ? 1 : 0;
    if (s->grp) {
        if (axis != s->dim - 1) return fail(IB_EINVAL, "on a z-slab context ib_line_solve solves along the cut axis");
        const int rc = upload_coef(s, SYS_USER, -kappa, 1.0 + 2.0 * kappa, -kappa, mf);
        if (rc != IB_OK) return rc;
        for (int r = 0; r < nslabs(s); ++r) {
            Ctx* sl = slab_at(s, r);
            CKC(cudaMemcpyAsync(sl->tmp, d + host_off(s, sl), (size_t)sl->nlocal * sizeof(double),
                                cudaMemcpyHostToDevice, s->stream));
        }
        FOR_SLABS(slab_user_fwd(sl, s->grp, sl->tmp, mf));
        CKG(group_up(s->grp, mf ? 4 : 2, s->stream));
        CKC(slab_master(s->grp->slab[0], s->grp, SYS_USER, 1, mf ? 4 : 2, mf));
        CKG(group_dn(s->grp, 1, s->stream));
        FOR_SLABS(slab_user_corr(sl, s->grp, sl->tmp, mf));
        for (int r = 0; r < nslabs(s); ++r) {
            Ctx* sl = slab_at(s, r);
            CKC(cudaMemcpyAsync(x + host_off(s, sl), sl->tmp, (size_t)sl->nlocal * sizeof(double),
                                cudaMemcpyDeviceToHost, s->stream));
        }
        CKC(cudaStreamSynchronize(s->stream));
        return IB_OK;
    }
    static SchurInv hs;
    std::vector<double> ext((size_t)4 * (s->L - 1) + 1);
    make_line_coef(&s->hcoef[SYS_USER], &hs, s->n, s->L, -kappa, 1.0 + 2.0 * kappa, -kappa, mf, ext.data());
    if (s->L > kMaxL) {
        CKC(cudaMemcpy(s->lcext[SYS_USER], ext.data(), ext.size() * sizeof(double), cudaMemcpyHostToDevice));
        s->hcoef[SYS_USER].ext = s->lcext[SYS_USER];
    }
    const size_t fb = (size_t)s->ncell * sizeof(double);
    CKC(cudaMemcpyAsync(s->sinv + SYS_USER, &hs, sizeof(SchurInv), cudaMemcpyHostToDevice, s->stream));
    CKC(cudaMemcpyAsync(s->tmp, d, fb, cudaMemcpyHostToDevice, s->stream));
    CKC(launch_line_solve(s, axis, SYS_USER, s->tmp));
    CKC(cudaMemcpyAsync(x, s->tmp, fb, cudaMemcpyDeviceToHost, s->stream));
    CKC(cudaStreamSynchronize(s->stream));
    return IB_OK;
}

int ib_psi_solve(ib_ctx* c, const double* f, double* psi, int32_t repeats, double* device_ms)
{
    if (!c || !f || !psi) return fail(IB_EINVAL, "null argument");
    Ctx* s = &c->s;
    if (repeats < 1) return fail(IB_EINVAL, "repeats must be >= 1");
    if (s->grp) return fail(IB_EINVAL, "ib_psi_solve runs on a single-GPU context");
    const size_t fb = (size_t)s->ncell * sizeof(double);
    CKC(cudaMemcpyAsync(s->tmp, f, fb, cudaMemcpyHostToDevice, s->stream));
    cudaEvent_t e0, e1;
    CKC(cudaEventCreate(&e0));
    CKC(cudaEventCreate(&e1));
    // the applications are captured once into a CUDA graph so that the device time is
    // not bounded by host launch latency on small grids
    for (int a = s->dim - 1; a >= 0; --a) CKC(launch_line_solve(s, a, SYS_PSI, s->tmp));   // first use: attributes
    CKC(cudaMemcpyAsync(s->tmp, f, fb, cudaMemcpyHostToDevice, s->stream));
    cudaGraph_t g;
    cudaGraphExec_t ge;
    CKC(cudaStreamBeginCapture(s->stream, cudaStreamCaptureModeThreadLocal));
    for (int r = 0; r < repeats; ++r)
        for (int a = s->dim - 1; a >= 0; --a) {
            const cudaError_t le = launch_line_solve(s, a, SYS_PSI, s->tmp);
            if (le != cudaSuccess) {
                cudaStreamEndCapture(s->stream, &g);
                return fail(IB_ECUDA, "launch_line_solve: %s", cudaGetErrorString(le));
            }
        }
    CKC(cudaStreamEndCapture(s->stream, &g));
    CKC(cudaGraphInstantiate(&ge, g, 0));
    cudaGraphDestroy(g);
    CKC(cudaEventRecord(e0, s->stream));
    CKC(cudaGraphLaunch(ge, s->stream));
    CKC(cudaEventRecord(e1, s->stream));
    CKC(cudaMemcpyAsync(psi, s->tmp, fb, cudaMemcpyDeviceToHost, s->stream));
    CKC(cudaStreamSynchronize(s->stream));
    float ms = 0.f;
    CKC(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaGraphExecDestroy(ge);
    if (device_ms) *device_ms = ms / repeats;
    return IB_OK;
}

int ib_check_finite(ib_ctx* c)
{
    if (!c) return fail(IB_EINVAL, "null context");
    Ctx* s = &c->s;
    int bad = 0;
    // fields per slab; X (and, on a single GPU, the fields) on the top context, whose
    // nlocal is 0 when it holds no fields
    for (int r = 0; r <= (s->grp ? s->grp->nloc : 0); ++r) {
        Ctx* cc = (s->grp && r < s->grp->nloc) ? s->grp->slab[r] : s;
        CKC(cudaMemsetAsync(cc->d_flag, 0, sizeof(int), s->stream));
        CKC(launch_check_finite(cc, cc->d_flag));
        int flag = 0;
        CKC(cudaMemcpyAsync(&flag, cc->d_flag, sizeof(int), cudaMemcpyDeviceToHost, s->stream));
        CKC(cudaStreamSynchronize(s->stream));
        bad |= flag;
    }
    if (bad) return fail(IB_ENONFINITE, "non-finite value in u, p or X after %lld steps", (long long)s->step);
    return IB_OK;
}

int ib_get_stats(ib_ctx* c, double* ms_per_phase, int64_t* steps, int64_t* launches)
{
    if (!c) return fail(IB_EINVAL, "null context");
    const Ctx* s = &c->s;
    if (ms_per_phase)
        for (int ph = 0; ph < IB_NPHASES; ++ph) ms_per_phase[ph] = s->ph_cnt[ph] ? s->ph_ms[ph] / s->ph_cnt[ph] : 0.0;
    if (launches) *launches = total_launches(&c->s);
    if (steps) *steps = c->s.step;
    return IB_OK;
}

int ib_destroy(ib_ctx* c)
{
    if (!c) return IB_OK;
    Ctx* s = &c->s;
    if (s->stream) cudaStreamSynchronize(s->stream);
    drop_graphs(s);
    if (s->grp) {
        Group* G = s->grp;
        for (int r = 0; r < G->nloc; ++r) {
            if (!G->slab[r]) continue;
            free_fields(G->slab[r]);
            delete G->slab[r];
        }
        cudaFree(G->up_s); cudaFree(G->up_rv); cudaFree(G->dn_s); cudaFree(G->dn_rv);
        for (int k = 0; k < SYS_COUNT; ++k) cudaFree(G->coef[k]);
        free_lagrangian(s);
        nccl_comm_destroy(G->comm_side);
        nccl_comm_destroy(G->comm_halo);
        nccl_comm_destroy(G->comm);
        delete G;
        s->grp = nullptr;
        cudaFree(s->d_flag);
    } else {
        free_fields(s);
        free_lagrangian(s);
    }
    cudaFree(s->sinv);
    for (int k = 0; k < SYS_COUNT; ++k) cudaFree(s->lcext[k]);
    cudaFree(s->bin_count); cudaFree(s->bin_start); cudaFree(s->bin_cursor); cudaFree(s->bin_list);
    cudaFree(s->bin_nlist); cudaFree(s->bin_partial);
    if (s->ev_made)
        for (int ph = 0; ph < IB_NPHASES; ++ph) { cudaEventDestroy(s->ev[ph][0]); cudaEventDestroy(s->ev[ph][1]); }
    if (s->side) cudaStreamDestroy(s->side);
    if (s->comm) cudaStreamDestroy(s->comm);
    if (s->ev_h0) cudaEventDestroy(s->ev_h0);
    if (s->ev_h1) cudaEventDestroy(s->ev_h1);
    if (s->ev_fork) cudaEventDestroy(s->ev_fork);
    if (s->ev_join) cudaEventDestroy(s->ev_join);
    if (s->own_stream && s->stream) cudaStreamDestroy(s->stream);
    if (s->err_h) cudaFreeHost(s->err_h);
    delete c;
    return IB_OK;
}

}  // extern "C"
