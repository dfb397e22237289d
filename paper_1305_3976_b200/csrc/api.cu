// C-ABI of libibgm.so (include/ibgm.h): context management, host-side precompute of
// the line-solver factors, the per-step schedule, host<->device copies.
#include <cuda_runtime.h>

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
void make_line_coef(LineCoef* C, SchurInv* SI, int64_t N, int L, double c_, double a_, double b_, int mean_fix)
{
    memset(C, 0, sizeof(*C));
    memset(SI, 0, sizeof(*SI));
    const long double c = c_, a = a_, b = b_;
    const int m = L - 1;
    const int P = (int)(N / L);
    C->c = c_; C->a = a_; C->b = b_;
    C->L = L; C->P = P; C->N = (int)N; C->mean_fix = mean_fix;
    C->inv_rowsum = (double)(1.0L / (a + b + c));
    long double den[kMaxL], cp[kMaxL];
    den[0] = a;
    cp[0] = b / den[0];
    for (int i = 1; i < m; ++i) {
        den[i] = a - c * cp[i - 1];
        cp[i] = b / den[i];
    }
    for (int i = 0; i < m; ++i) {
        C->inv[i] = (double)(1.0L / den[i]);
        C->cp[i] = (double)cp[i];
    }
    auto solveB = [&](const long double* d, long double* x) {
        long double dp[kMaxL];
        dp[0] = d[0] / den[0];
        for (int i = 1; i < m; ++i) dp[i] = (d[i] - c * dp[i - 1]) / den[i];
        x[m - 1] = dp[m - 1];
        for (int i = m - 2; i >= 0; --i) x[i] = dp[i] - cp[i] * x[i + 1];
    };
    long double e1[kMaxL] = {0}, em[kMaxL] = {0}, g[kMaxL], h[kMaxL];
    e1[0] = 1.0L;
    em[m - 1] = 1.0L;
    solveB(e1, g);
    solveB(em, h);
    long double gs = 0.0L, hs = 0.0L;
    for (int i = 0; i < m; ++i) {
        C->g[i] = (double)g[i];
        C->h[i] = (double)h[i];
        gs += g[i];
        hs += h[i];
    }
    C->gsum = (double)gs;
    C->hsum = (double)hs;
    const long double s0 = a - b * c * (h[m - 1] + g[0]);
    const long double sm = -c * c * g[m - 1];
    const long double sp = -b * b * h[0];
    std::vector<long double> S((size_t)P * P, 0.0L), I((size_t)P * P, 0.0L);
    for (int p = 0; p < P; ++p) {
        S[(size_t)p * P + p] += s0;
        S[(size_t)p * P + (p + P - 1) % P] += sm;
        S[(size_t)p * P + (p + 1) % P] += sp;
        I[(size_t)p * P + p] = 1.0L;
    }
    // Gauss-Jordan with partial pivoting (P <= 32)
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
    for (int i = 0; i < P * P; ++i) SI->sinv[i] = (double)I[i];
    for (int q = 0; q < P; ++q) {
        long double cs = 0.0L;
        for (int p = 0; p < P; ++p) cs += I[(size_t)p * P + q];
        SI->colsum[q] = (double)cs;
    }
}

}  // namespace ibgm

static bool choose_segmentation(int64_t n, int* L, int* P)
{
    static const int cands[] = {8, 12, 16, 24, 32, 6, 4, 3, 2};
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
    for (int k = 0; k < 2; ++k) {
        if (s->gvalid[k]) cudaGraphExecDestroy(s->gexec[k]);
        s->gvalid[k] = false;
    }
}

static void free_lagrangian(Ctx* s)
{
    cudaFree(s->X); cudaFree(s->Xh); cudaFree(s->Uprev); cudaFree(s->F); cudaFree(s->wgt);
    cudaFree(s->csr_ptr); cudaFree(s->csr_nbr); cudaFree(s->csr_kappa); cudaFree(s->csr_rest);
    cudaFree(s->bin_bid); cudaFree(s->bin_sorted);
    s->bin_bid = s->bin_sorted = nullptr;
    s->X = s->Xh = s->Uprev = s->F = s->wgt = nullptr;
    s->csr_ptr = s->csr_nbr = nullptr;
    s->csr_kappa = s->csr_rest = nullptr;
    s->npts = s->nedges = 0;
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
}

const char* ib_last_error(void) { return g_err.c_str(); }

int ib_create(const ib_grid* grid, double nu, double rho, double dt, const ib_options* opt, ib_ctx** out)
{
    if (!grid || !out) return fail(IB_EINVAL, "null argument");
    *out = nullptr;
    ib_options o;
    if (opt) o = *opt; else ib_default_options(&o);
    if (grid->dim != 2 && grid->dim != 3) return fail(IB_EINVAL, "dim must be 2 or 3 (got %d)", grid->dim);
    if (grid->n < 8 || grid->n > 1024) return fail(IB_EINVAL, "N must be in [8, 1024] (got %lld)", (long long)grid->n);
    if (grid->H != 1.0) return fail(IB_EINVAL, "H must be 1 (the psi operator is literal, DESIGN.md R2)");
    if (!(dt > 0) || !(rho > 0) || !(nu >= 0)) return fail(IB_EINVAL, "need dt > 0, rho > 0, nu >= 0");
    if (!(o.chi > 0 && o.chi <= 1)) return fail(IB_EINVAL, "chi must be in (0, 1]");
    if (o.nranks != 1 || o.rank != 0) return fail(IB_EINVAL, "this build runs one rank per process (nranks = 1)");
    if (o.kernel != IB_DELTA_COS4 && o.kernel != IB_DELTA_PESKIN4) return fail(IB_EINVAL, "unknown delta kernel");
    int L, P;
    if (!choose_segmentation(grid->n, &L, &P))
        return fail(IB_EINVAL, "N = %lld has no divisor L in {2,3,4,6,8,12,16,24,32} with N/L <= 32",
                    (long long)grid->n);

    ib_ctx* c = new ib_ctx();
    Ctx* s = &c->s;
    memset(s, 0, sizeof(*s));
    s->dim = grid->dim;
    s->n = grid->n;
    s->ncell = grid->dim == 3 ? grid->n * grid->n * grid->n : grid->n * grid->n;
    s->h = 1.0 / (double)grid->n;
    s->rho = rho;
    s->mu = nu * rho;
    s->dt = dt;
    s->chi = o.chi;
    s->kernel = o.kernel;
    s->advection = o.advection;
    s->device = o.device;
    s->L = L; s->P = P;
    s->use_graphs = true;
    *out = c;

    CKC(cudaSetDevice(o.device));
    if (o.stream) {
        s->stream = (cudaStream_t)o.stream;
        s->own_stream = false;
    } else {
        CKC(cudaStreamCreateWithFlags(&s->stream, cudaStreamNonBlocking));
        s->own_stream = true;
    }
    const size_t fb = (size_t)s->ncell * sizeof(double);
    for (int q = 0; q < s->dim; ++q) {
        CKC(cudaMalloc(&s->u[q], fb));
        CKC(cudaMalloc(&s->st[q], fb));
        CKC(cudaMalloc(&s->nadv[q], fb));
        CKC(cudaMalloc(&s->nprev[q], fb));
        CKC(cudaMemsetAsync(s->u[q], 0, fb, s->stream));
        CKC(cudaMemsetAsync(s->st[q], 0, fb, s->stream));
        CKC(cudaMemsetAsync(s->nadv[q], 0, fb, s->stream));
        CKC(cudaMemsetAsync(s->nprev[q], 0, fb, s->stream));
    }
    CKC(cudaMalloc(&s->p, fb));
    CKC(cudaMalloc(&s->pstar, fb));
    CKC(cudaMalloc(&s->tmp, fb));
    CKC(cudaMemsetAsync(s->p, 0, fb, s->stream));
    CKC(cudaMemsetAsync(s->pstar, 0, fb, s->stream));
    CKC(cudaMalloc(&s->d_flag, sizeof(int)));
    // brick grid for the binned spread: 8^3 cells (3D) / 16^2 (2D)
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
    CKC(cudaMalloc(&s->sinv, sizeof(SchurInv) * SYS_COUNT));
    SchurInv hs[SYS_COUNT];
    // viscous Douglas sweeps: (1 - kap delta) with kap = mu dt / (2 rho h^2)
    const double kv = s->mu * dt / (2.0 * rho * s->h * s->h);
    // (well conditioned, cond <= 1 + 4 kv: no mean correction needed, R16)
    make_line_coef(&s->hcoef[SYS_VISC], &hs[SYS_VISC], s->n, L, -kv, 1.0 + 2.0 * kv, -kv, 0);
    // psi factors: (1 - D_aa) with D_aa = delta / h^2 (R2)
    const double kp = 1.0 / (s->h * s->h);
    make_line_coef(&s->hcoef[SYS_PSI], &hs[SYS_PSI], s->n, L, -kp, 1.0 + 2.0 * kp, -kp, 1);
    make_line_coef(&s->hcoef[SYS_USER], &hs[SYS_USER], s->n, L, -kv, 1.0 + 2.0 * kv, -kv, 0);
    CKC(cudaMemcpyAsync(s->sinv, hs, sizeof(SchurInv) * SYS_COUNT, cudaMemcpyHostToDevice, s->stream));
    CKC(cudaStreamSynchronize(s->stream));
    return IB_OK;
}

int ib_set_fields(ib_ctx* c, const double* u, const double* v, const double* w, const double* p)
{
    if (!c || !u || !v || (c->s.dim == 3 && !w)) return fail(IB_EINVAL, "null field pointer");
    Ctx* s = &c->s;
    const size_t fb = (size_t)s->ncell * sizeof(double);
    const double* in[3] = {u, v, w};
    for (int q = 0; q < s->dim; ++q) {
        CKC(cudaMemcpyAsync(s->u[q], in[q], fb, cudaMemcpyHostToDevice, s->stream));
        CKC(cudaMemsetAsync(s->nprev[q], 0, fb, s->stream));
    }
    // p^{-1/2} = p (or 0), psi^{-1/2} = 0, so p* = p (R5)
    if (p) {
        CKC(cudaMemcpyAsync(s->p, p, fb, cudaMemcpyHostToDevice, s->stream));
        CKC(cudaMemcpyAsync(s->pstar, p, fb, cudaMemcpyHostToDevice, s->stream));
    } else {
        CKC(cudaMemsetAsync(s->p, 0, fb, s->stream));
        CKC(cudaMemsetAsync(s->pstar, 0, fb, s->stream));
    }
    CKC(cudaStreamSynchronize(s->stream));
    s->step = 0;
    s->fields_set = true;
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
    s->step = 0;
    if (npts == 0) return IB_OK;
    const int d = s->dim;
    // CSR adjacency: every edge appears in the lists of both endpoints
    std::vector<int32_t> ptr(npts + 1, 0), nbr(2 * nedges);
    std::vector<double> kap(2 * nedges), rst(2 * nedges);
    for (int64_t e = 0; e < nedges; ++e) { ptr[edges[2 * e] + 1]++; ptr[edges[2 * e + 1] + 1]++; }
    for (int64_t k = 0; k < npts; ++k) ptr[k + 1] += ptr[k];
    std::vector<int32_t> fill(ptr.begin(), ptr.end() - 1);
    int has_rest = 0;
    for (int64_t e = 0; e < nedges; ++e) {
        const int64_t a = edges[2 * e], b = edges[2 * e + 1];
        const double L = rest ? rest[e] : 0.0;
        if (L != 0.0) has_rest = 1;
        int32_t ia = fill[a]++, ib = fill[b]++;
        nbr[ia] = (int32_t)b; kap[ia] = kappa[e]; rst[ia] = L;
        nbr[ib] = (int32_t)a; kap[ib] = kappa[e]; rst[ib] = L;
    }
    std::vector<double> wv(npts, 1.0);
    if (weight) for (int64_t k = 0; k < npts; ++k) wv[k] = weight[k];
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
    CKC(cudaMemcpyAsync(s->X, X, pb, cudaMemcpyHostToDevice, s->stream));
    CKC(cudaMemcpyAsync(s->Xh, X, pb, cudaMemcpyHostToDevice, s->stream));
    CKC(cudaMemsetAsync(s->Uprev, 0, pb, s->stream));
    CKC(cudaMemsetAsync(s->F, 0, pb, s->stream));
    CKC(cudaMemcpyAsync(s->wgt, wv.data(), npts * sizeof(double), cudaMemcpyHostToDevice, s->stream));
    CKC(cudaMemcpyAsync(s->csr_ptr, ptr.data(), (npts + 1) * sizeof(int32_t), cudaMemcpyHostToDevice, s->stream));
    if (nedges > 0) {
        CKC(cudaMemcpyAsync(s->csr_nbr, nbr.data(), 2 * nedges * sizeof(int32_t), cudaMemcpyHostToDevice, s->stream));
        CKC(cudaMemcpyAsync(s->csr_kappa, kap.data(), 2 * nedges * sizeof(double), cudaMemcpyHostToDevice, s->stream));
        CKC(cudaMemcpyAsync(s->csr_rest, rst.data(), 2 * nedges * sizeof(double), cudaMemcpyHostToDevice, s->stream));
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
    const size_t fb = (size_t)s->ncell * sizeof(double);
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

static int enqueue_step(Ctx* s, int first);

static void swap_state(Ctx* s)
{
    for (int q = 0; q < s->dim; ++q) {
        std::swap(s->u[q], s->st[q]);
        std::swap(s->nadv[q], s->nprev[q]);
    }
    s->parity ^= 1;
}

int ib_step(ib_ctx* c, int64_t nsteps)
{
    if (!c) return fail(IB_EINVAL, "null context");
    Ctx* s = &c->s;
    if (!s->fields_set) return fail(IB_ESTATE, "ib_step before ib_set_fields");
    if (nsteps < 0) return fail(IB_EINVAL, "nsteps < 0");
    for (int64_t t = 0; t < nsteps; ++t) {
        const int first = (s->step == 0);
        if (!first && !s->profiling && s->use_graphs && !s->debug_keep_f) {
            // replay the captured regular step for the current pointer parity
            const int par = s->parity;
            if (!s->gvalid[par]) {
                cudaGraph_t g;
                const int64_t l0 = s->launches;
                CKC(cudaStreamBeginCapture(s->stream, cudaStreamCaptureModeThreadLocal));
                const int rc = enqueue_step(s, 0);
                cudaError_t ce = cudaStreamEndCapture(s->stream, &g);
                if (rc != IB_OK) return rc;
                CKC(ce);
                CKC(cudaGraphInstantiate(&s->gexec[par], g, 0));
                cudaGraphDestroy(g);
                s->gvalid[par] = true;
                s->glaunches[par] = s->launches - l0;
                s->launches = l0;
            }
            CKC(cudaGraphLaunch(s->gexec[par], s->stream));
            s->launches += s->glaunches[par];
        } else {
            const int rc = enqueue_step(s, first);
            if (rc != IB_OK) return rc;
        }
        swap_state(s);
        s->step++;
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
    return IB_OK;
}

// all device work of one time step (Steps 1a-3f), enqueued on the context's stream
static int enqueue_step(Ctx* s, int first)
{
    const int d = s->dim;
    {
        // n = 0: no N(u^{-1}); the history G starts as 0 + (2/rho) f
        if (first) PHASE(IB_PH_CLEAR, clear3(s, s->nprev));
        if (s->debug_keep_f && s->npts > 0) PHASE(IB_PH_CLEAR, clear3(s, s->f));
        if (s->npts > 0) {
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
        // Step 3e: RHS and the psi factors (last axis first); Step 3f fused
        PHASE(IB_PH_DIVPSI, launch_div_psi_first(s, d - 1));
        if (d == 3) PHASE(IB_PH_PSI_Y, launch_psi_mid(s, 1));
        PHASE(IB_PH_PSI_X, launch_psi_last_x(s));
    }
    return IB_OK;
}

int ib_set_debug(ib_ctx* c, int32_t flags)
{
    if (!c) return fail(IB_EINVAL, "null context");
    Ctx* s = &c->s;
    const int keep = (flags & 1) != 0;
    if (keep && !s->f[0]) {
        const size_t fb = (size_t)s->ncell * sizeof(double);
        for (int q = 0; q < s->dim; ++q) {
            CKC(cudaMalloc(&s->f[q], fb));
            CKC(cudaMemsetAsync(s->f[q], 0, fb, s->stream));
        }
    }
    drop_graphs(s);
    s->debug_keep_f = keep;
    s->spread_mode = (flags >> 1) & 3;   // bits 1-2: spread method (0 auto, 1 direct, 2 brick)
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
    return IB_OK;
}

int ib_get_fields(ib_ctx* c, double* u, double* v, double* w, double* p, double* psi, double* X, double* U)
{
    if (!c) return fail(IB_EINVAL, "null context");
    Ctx* s = &c->s;
    const size_t fb = (size_t)s->ncell * sizeof(double);
    double* out[3] = {u, v, w};
    for (int q = 0; q < s->dim; ++q)
        if (out[q]) CKC(cudaMemcpyAsync(out[q], s->u[q], fb, cudaMemcpyDeviceToHost, s->stream));
    if (p) CKC(cudaMemcpyAsync(p, s->p, fb, cudaMemcpyDeviceToHost, s->stream));
    if (psi) {
        // the state keeps p* = p + psi; psi^{n-1/2} = p* - p
        CKC(launch_sub(s, s->pstar, s->p, s->tmp));
        CKC(cudaMemcpyAsync(psi, s->tmp, fb, cudaMemcpyDeviceToHost, s->stream));
    }
    const size_t pb = (size_t)s->npts * s->dim * sizeof(double);
    if (X && pb) CKC(cudaMemcpyAsync(X, s->X, pb, cudaMemcpyDeviceToHost, s->stream));
    if (U && pb) CKC(cudaMemcpyAsync(U, s->Uprev, pb, cudaMemcpyDeviceToHost, s->stream));
    CKC(cudaStreamSynchronize(s->stream));
    return IB_OK;
}

int ib_get_aux(ib_ctx* c, double* fu, double* fv, double* fw, double* nu, double* nv, double* nw, double* F,
               double* Xh)
{
    if (!c) return fail(IB_EINVAL, "null context");
    Ctx* s = &c->s;
    const size_t fb = (size_t)s->ncell * sizeof(double);
    double* fo[3] = {fu, fv, fw};
    double* no[3] = {nu, nv, nw};
    if ((fu || fv || fw) && !s->debug_keep_f) return fail(IB_ESTATE, "f is only kept with ib_set_debug(ctx, 1)");
    for (int q = 0; q < s->dim; ++q) {
        if (fo[q]) CKC(cudaMemcpyAsync(fo[q], s->f[q], fb, cudaMemcpyDeviceToHost, s->stream));
        if (no[q]) CKC(cudaMemcpyAsync(no[q], s->nprev[q], fb, cudaMemcpyDeviceToHost, s->stream));
    }
    const size_t pb = (size_t)s->npts * s->dim * sizeof(double);
    if (F && pb) CKC(cudaMemcpyAsync(F, s->F, pb, cudaMemcpyDeviceToHost, s->stream));
    if (Xh && pb) CKC(cudaMemcpyAsync(Xh, s->Xh, pb, cudaMemcpyDeviceToHost, s->stream));
    CKC(cudaStreamSynchronize(s->stream));
    return IB_OK;
}

int ib_line_solve(ib_ctx* c, int32_t axis, double kappa, const double* d, double* x)
{
    if (!c || !d || !x) return fail(IB_EINVAL, "null argument");
    Ctx* s = &c->s;
    if (axis < 0 || axis >= s->dim) return fail(IB_EINVAL, "axis %d out of range", axis);
    if (!(kappa >= 0)) return fail(IB_EINVAL, "kappa must be >= 0");
    static SchurInv hs;
    // the exact mean correction is applied to the ill-conditioned systems (kappa > 1, R16)
    make_line_coef(&s->hcoef[SYS_USER], &hs, s->n, s->L, -kappa, 1.0 + 2.0 * kappa, -kappa, kappa > 1.0 ? 1 : 0);
    const size_t fb = (size_t)s->ncell * sizeof(double);
    CKC(cudaMemcpyAsync(s->sinv + SYS_USER, &hs, sizeof(SchurInv), cudaMemcpyHostToDevice, s->stream));
    CKC(cudaMemcpyAsync(s->tmp, d, fb, cudaMemcpyHostToDevice, s->stream));
    CKC(launch_line_solve(s, axis, SYS_USER, s->tmp));
    CKC(cudaMemcpyAsync(x, s->tmp, fb, cudaMemcpyDeviceToHost, s->stream));
    CKC(cudaStreamSynchronize(s->stream));
    return IB_OK;
}

int ib_check_finite(ib_ctx* c)
{
    if (!c) return fail(IB_EINVAL, "null context");
    Ctx* s = &c->s;
    CKC(launch_check_finite(s));
    int flag = 0;
    CKC(cudaMemcpyAsync(&flag, s->d_flag, sizeof(int), cudaMemcpyDeviceToHost, s->stream));
    CKC(cudaStreamSynchronize(s->stream));
    if (flag) return fail(IB_ENONFINITE, "non-finite value in u, p or X after %lld steps", (long long)s->step);
    return IB_OK;
}

int ib_get_stats(ib_ctx* c, int64_t* launches, int64_t* steps)
{
    if (!c) return fail(IB_EINVAL, "null context");
    if (launches) *launches = c->s.launches;
    if (steps) *steps = c->s.step;
    return IB_OK;
}

int ib_destroy(ib_ctx* c)
{
    if (!c) return IB_OK;
    Ctx* s = &c->s;
    if (s->stream) cudaStreamSynchronize(s->stream);
    drop_graphs(s);
    for (int q = 0; q < 3; ++q) {
        cudaFree(s->u[q]); cudaFree(s->st[q]); cudaFree(s->nadv[q]); cudaFree(s->nprev[q]); cudaFree(s->f[q]);
    }
    cudaFree(s->p); cudaFree(s->pstar); cudaFree(s->tmp); cudaFree(s->sinv); cudaFree(s->d_flag);
    cudaFree(s->bin_count); cudaFree(s->bin_start); cudaFree(s->bin_cursor); cudaFree(s->bin_list);
    cudaFree(s->bin_nlist); cudaFree(s->bin_partial);
    free_lagrangian(s);
    if (s->ev_made)
        for (int ph = 0; ph < IB_NPHASES; ++ph) { cudaEventDestroy(s->ev[ph][0]); cudaEventDestroy(s->ev[ph][1]); }
    if (s->own_stream && s->stream) cudaStreamDestroy(s->stream);
    delete c;
    return IB_OK;
}

}  // extern "C"
