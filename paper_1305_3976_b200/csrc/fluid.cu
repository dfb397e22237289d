// Fluid passes of the IB-GM step on the GPU (sm_100a, fp64).
//
// Steps 3a-3f of PAPER.md:624-683 as five kinds of line passes over the periodic
// MAC grid (x fastest, flat index i + N*(j + N*k)):
//   S1   x-lines : p* (3a), explicit momentum with AB2 skew advection (3b), and the
//                  x Douglas sweep (3c) fused; also stores N(u^n) for the next step
//   VISC y/z     : remaining Douglas sweeps (3d, eqs. umacstep1/2)
//   DIV  cells   : r = -(rho/dt) D.u^{n+1} (3e right-hand side) and
//                  q = p - chi mu D.((u^{n+1}+u^n)/2) (the explicit part of 3f)
//   PSI  lines   : the factors of (1-D_xx)(1-D_yy)[(1-D_zz)] psi = r (3e, eqs.
//                  PenaltyStepPart1/2); the last (x) factor also
//                  finishes 3f: p = q + psi.
// Every line pass solves N^{d-1} independent cyclic tridiagonal systems (eq.
// TriDiagX) with the Schur-complement splitting of PAPER.md:
// 1025-1262 mapped onto one CTA: a line is cut into P parts of L unknowns, one
// thread per part runs Thomas's algorithm on its interior block in registers,
// the P x P periodic Schur system S y = g - F f* is solved with the precomputed
// dense S^{-1} through shared memory, and each thread corrects x = f* - B^{-1}E y.
// Strided (y, z) lines map 32 (or 16) neighbouring lines to the lanes of a warp so
// every global load/store is coalesced; contiguous x lines are staged through a
// padded shared-memory tile with coalesced loads and stores.
#include <cuda_runtime.h>

#include <cstdio>

#include "ibgm_internal.cuh"

namespace ibgm {

enum OpX { OPX_S1 = 0, OPX_PSI_LAST = 1, OPX_USER = 2 };
enum OpYZ { OPYZ_VISC = 0, OPYZ_PSI = 1, OPYZ_USER = 2 };

struct S1Args {
    const double* u[3];
    const double* nprev[3];
    const double* f[3];
    const double* p;
    const double* psi;
    double* nadv[3];
    double* out[3];
    double dt, rho, mu, invh, kap;   // kap = mu dt / (2 rho h^2)
    int first, advection;
};

struct XArgs {
    const double* in;
    double* out;
    double* p;   // PSI_LAST: p += x
};

struct YZArgs {
    const double* in[3];
    const double* un[3];
    double* out[3];
    double kap;
};

__device__ __forceinline__ int wrapn(int i, int n) { return i < 0 ? i + n : (i >= n ? i - n : i); }

// -------------------------------------------------------------------------------
// Schur-segmented solve of one part (L unknowns) of a cyclic line.  On entry
// x[0..L-1] holds the right-hand side of rows sL..sL+L-1 of line l; on exit the
// solution.  All threads of the block must call it (block-uniform control flow).
// -------------------------------------------------------------------------------
template <int L>
__device__ __forceinline__ void schur_solve(double (&x)[L], const LineCoef* __restrict__ C, int s, int l,
                                            int R, int P, double* sh)
{
    constexpr int M = L - 1;
    const double c = C->c, b = C->b;
    const int PR = P * R;
    double* sh_first = sh;
    double* sh_last = sh + PR;
    double* sh_r = sh + 2 * PR;
    double* sh_dsum = sh + 3 * PR;
    double* sh_xsum = sh + 4 * PR;
    const int me = s * R + l;
    const int mean_fix = C->mean_fix;

    double dsum = 0.0;
#pragma unroll
    for (int i = 0; i < L; ++i) dsum += x[i];

    // f*_p = B_p^{-1} f_p  (eq. LocalTriSystem; Thomas)
    x[1] *= C->inv[0];
#pragma unroll
    for (int i = 2; i <= M; ++i) x[i] = (x[i] - c * x[i - 1]) * C->inv[i - 1];
#pragma unroll
    for (int i = M - 1; i >= 1; --i) x[i] -= C->cp[i - 1] * x[i + 1];

    // gather the first/last entries of f*_p and g_p
    sh_first[me] = x[1];
    sh_last[me] = x[M];
    sh_dsum[me] = dsum;
    __syncthreads();
    const int sm1 = (s == 0) ? P - 1 : s - 1;
    const int sp1 = (s == P - 1) ? 0 : s + 1;
    // right-hand side of the Schur system  g - F f*  (eq. SchurSystem)
    sh_r[me] = x[0] - c * sh_last[sm1 * R + l] - b * sh_first[me];
    __syncthreads();
    // y = S^{-1}(g - F f*): this part needs y_p and y_{p+1}
    double ys = 0.0, ys1 = 0.0;
    const double* Si = C->sinv + s * P;
    const double* Si1 = C->sinv + sp1 * P;
    for (int q = 0; q < P; ++q) {
        const double r = sh_r[q * R + l];
        ys = fma(Si[q], r, ys);
        ys1 = fma(Si1[q], r, ys1);
    }
    // x_p = f*_p - B_p^{-1} E_p y; E_p y = c y_p e_1 + b y_{p+1} e_m
    x[0] = ys;
    const double cy = c * ys, by = b * ys1;
#pragma unroll
    for (int i = 1; i <= M; ++i) x[i] -= cy * C->g[i - 1] + by * C->h[i - 1];

    if (mean_fix) {
        // exact line-mean correction (R16): 1^T A = (a+b+c) 1^T for the
        // circulant A, so mean(x) must equal mean(d)/(a+b+c).
        double xs = 0.0;
#pragma unroll
        for (int i = 0; i < L; ++i) xs += x[i];
        sh_xsum[me] = xs;
        __syncthreads();
        double D = 0.0, X = 0.0;
        for (int q = 0; q < P; ++q) {
            D += sh_dsum[q * R + l];
            X += sh_xsum[q * R + l];
        }
        const double corr = (D * C->inv_rowsum - X) / (double)(P * L);
#pragma unroll
        for (int i = 0; i < L; ++i) x[i] += corr;
    }
}

// -------------------------------------------------------------------------------
// S1 right-hand side at (i,j,k) for component c: Steps 3a-3c.
// -------------------------------------------------------------------------------
template <int DIM>
__device__ __forceinline__ double s1_rhs(const S1Args& A, int c, int i, int j, int k, int n, size_t q0)
{
    const int xi[3] = {wrapn(i - 1, n), i, wrapn(i + 1, n)};
    const int yj[3] = {wrapn(j - 1, n), j, wrapn(j + 1, n)};
    const int zk[3] = {DIM == 3 ? wrapn(k - 1, n) : 0, k, DIM == 3 ? wrapn(k + 1, n) : 0};
    auto at = [&](int di, int dj, int dk) -> size_t {
        return (size_t)xi[di + 1] + (size_t)n * ((size_t)yj[dj + 1] + (size_t)n * (size_t)zk[dk + 1]);
    };
    auto E = [](int a, int ax) { return a == ax ? 1 : 0; };
    const double* uc = A.u[c];
    const double u0 = uc[q0];
    const double invh = A.invh;

    // skew-symmetric advection (Morinishi "Skew.-S2", R4)
    double Nc = 0.0;
    if (A.advection) {
        double dv = 0.0, ad = 0.0;
#pragma unroll
        for (int jd = 0; jd < DIM; ++jd) {
            const double* uj = A.u[jd];
            const int ex = E(0, jd), ey = E(1, jd), ez = E(2, jd);
            const int cx = E(0, c), cy = E(1, c), cz = E(2, c);
            const double ucm = uc[at(-ex, -ey, -ez)];
            const double ucp = uc[at(ex, ey, ez)];
            const double Tm = 0.5 * (uj[q0] + uj[at(-cx, -cy, -cz)]);
            const double Tp = 0.5 * (uj[at(ex, ey, ez)] + uj[at(ex - cx, ey - cy, ez - cz)]);
            const double Am = 0.5 * (u0 + ucm), Ap = 0.5 * (ucp + u0);
            const double Gm = (u0 - ucm) * invh, Gp = (ucp - u0) * invh;
            dv += (Tp * Ap - Tm * Am) * invh;
            ad += 0.5 * (Tm * Gm + Tp * Gp);
        }
        Nc = 0.5 * (dv + ad);
        A.nadv[c][q0] = Nc;
    }
    const double Nh = A.first ? Nc : 1.5 * Nc - 0.5 * A.nprev[c][q0];

    // mu sum_a D_aa u^n_c
    const double uxm = uc[at(-1, 0, 0)], uxp = uc[at(1, 0, 0)];
    double lap = (uxp - 2.0 * u0 + uxm);
    lap += uc[at(0, 1, 0)] - 2.0 * u0 + uc[at(0, -1, 0)];
    if (DIM == 3) lap += uc[at(0, 0, 1)] - 2.0 * u0 + uc[at(0, 0, -1)];
    lap *= invh * invh;

    // G p*, p* = p^{n-1/2} + psi^{n-1/2} (0 at n = 0)
    double gp = 0.0;
    if (!A.first) {
        const size_t qm = at(-E(0, c), -E(1, c), -E(2, c));
        gp = ((A.p[q0] + A.psi[q0]) - (A.p[qm] + A.psi[qm])) * invh;
    }
    const double ustar = u0 + A.dt * (-Nh + (A.mu * lap - gp + A.f[c][q0]) / A.rho);
    // Douglas x-sweep right-hand side: u* - (mu dt/2rho) D_xx u^n
    return ustar - A.kap * (uxp - 2.0 * u0 + uxm);
}

// -------------------------------------------------------------------------------
// x-line kernel: R consecutive rows (j0..j0+R-1 at fixed k) staged in a padded
// shared tile [R][N+1]; thread t -> row l = t % R, part s = t / R.
// -------------------------------------------------------------------------------
template <int L, int OP, int DIM>
__global__ void __launch_bounds__(512) k_line_x(const LineCoef* __restrict__ coef, int sys, int n, int R,
                                                 S1Args s1, XArgs xa, int ncomp)
{
    extern __shared__ double smem[];
    const int pitch = n + 1;
    double* tile = smem;
    double* red = smem + (size_t)R * pitch;
    const LineCoef* C = coef + sys;
    const int P = C->P;
    const int t = threadIdx.x, nthr = blockDim.x;
    const int l = t % R, s = t / R;
    const int j0 = blockIdx.x * R;
    const int k = blockIdx.y;
    const size_t plane = (size_t)n * n;

    for (int comp = 0; comp < ncomp; ++comp) {
        // fill (coalesced along x)
        for (int e = t; e < R * n; e += nthr) {
            const int row = e / n, i = e - row * n;
            const int j = j0 + row;
            double v = 0.0;
            if (j < n) {
                const size_t q = (size_t)i + (size_t)n * j + plane * k;
                if (OP == OPX_S1) v = s1_rhs<DIM>(s1, comp, i, j, k, n, q);
                else v = xa.in[q];
            }
            tile[row * pitch + i] = v;
        }
        __syncthreads();
        double x[L];
#pragma unroll
        for (int i = 0; i < L; ++i) x[i] = tile[l * pitch + s * L + i];
        schur_solve<L>(x, C, s, l, R, P, red);
#pragma unroll
        for (int i = 0; i < L; ++i) tile[l * pitch + s * L + i] = x[i];
        __syncthreads();
        // store (coalesced along x)
        for (int e = t; e < R * n; e += nthr) {
            const int row = e / n, i = e - row * n;
            const int j = j0 + row;
            if (j < n) {
                const size_t q = (size_t)i + (size_t)n * j + plane * k;
                const double v = tile[row * pitch + i];
                if (OP == OPX_S1) s1.out[comp][q] = v;
                else if (OP == OPX_PSI_LAST) { xa.out[q] = v; xa.p[q] += v; }  // Step 3f: p = q + psi
                else xa.out[q] = v;
            }
        }
        __syncthreads();
    }
}

// -------------------------------------------------------------------------------
// y/z-line kernel: R neighbouring lines (consecutive i) per block, direct coalesced
// global access; thread t -> line l = t % R, part s = t / R.  blockIdx.z = component.
// -------------------------------------------------------------------------------
template <int L, int OP>
__global__ void __launch_bounds__(512) k_line_yz(const LineCoef* __restrict__ coef, int sys, int n, int R,
                                                  int axis, YZArgs A)
{
    extern __shared__ double smem[];
    const LineCoef* C = coef + sys;
    const int P = C->P;
    const int t = threadIdx.x;
    const int l = t % R, s = t / R;
    const int i = blockIdx.x * R + l;
    const int comp = blockIdx.z;
    const bool active = i < n;
    const size_t S = (axis == 1) ? (size_t)n : (size_t)n * n;        // stride along the line
    const size_t T = (axis == 1) ? (size_t)n * n : (size_t)n;        // stride of the transverse index
    const size_t base = (size_t)(active ? i : 0) + T * blockIdx.y;
    const int pos0 = s * L;

    double x[L];
    if (OP == OPYZ_VISC) {
        const double* in = A.in[comp];
        const double* un = A.un[comp];
        double w[L + 2];
#pragma unroll
        for (int m = 0; m < L + 2; ++m) w[m] = un[base + S * (size_t)wrapn(pos0 - 1 + m, n)];
#pragma unroll
        for (int m = 0; m < L; ++m)
            x[m] = in[base + S * (size_t)(pos0 + m)] - A.kap * (w[m + 2] - 2.0 * w[m + 1] + w[m]);
    } else {
        const double* in = A.in[comp];
#pragma unroll
        for (int m = 0; m < L; ++m) x[m] = in[base + S * (size_t)(pos0 + m)];
    }
    schur_solve<L>(x, C, s, l, R, P, smem);
    if (active) {
        double* out = A.out[comp];
#pragma unroll
        for (int m = 0; m < L; ++m) out[base + S * (size_t)(pos0 + m)] = x[m];
    }
}

// -------------------------------------------------------------------------------
// DIV: r = -(rho/dt) D.u^{n+1} -> psi ; p <- p - chi mu D.((u^{n+1} + u^n)/2)
// -------------------------------------------------------------------------------
template <int DIM>
__global__ void k_div(const double* __restrict__ u0, const double* __restrict__ u1, const double* __restrict__ u2,
                      const double* __restrict__ s0, const double* __restrict__ s1, const double* __restrict__ s2,
                      double* __restrict__ psi, double* __restrict__ p, int n, double invh, double rho_dt,
                      double chimu)
{
    const size_t nc = (DIM == 3) ? (size_t)n * n * n : (size_t)n * n;
    for (size_t q = blockIdx.x * (size_t)blockDim.x + threadIdx.x; q < nc; q += (size_t)gridDim.x * blockDim.x) {
        const int i = (int)(q % n);
        const int j = (int)((q / n) % n);
        const size_t qx = (i == n - 1) ? q - (n - 1) : q + 1;
        const size_t qy = (j == n - 1) ? q - (size_t)(n - 1) * n : q + n;
        double dn = (s0[qx] - s0[q]) + (s1[qy] - s1[q]);
        double dol = (u0[qx] - u0[q]) + (u1[qy] - u1[q]);
        if (DIM == 3) {
            const int k = (int)(q / ((size_t)n * n));
            const size_t qz = (k == n - 1) ? q - (size_t)(n - 1) * n * n : q + (size_t)n * n;
            dn += s2[qz] - s2[q];
            dol += u2[qz] - u2[q];
        }
        dn *= invh;
        dol *= invh;
        psi[q] = -rho_dt * dn;                       // Step 3e right-hand side
        p[q] = p[q] - chimu * 0.5 * (dn + dol);      // Step 3f, explicit part
    }
}

// -------------------------------------------------------------------------------
// launchers
// -------------------------------------------------------------------------------
static size_t red_bytes(const Ctx* s) { return (size_t)5 * s->P * s->R * sizeof(double); }
static size_t tile_bytes(const Ctx* s) { return (size_t)s->R * (s->n + 1) * sizeof(double); }

template <int L, int OP, int DIM>
static cudaError_t go_x(Ctx* s, int sys, const S1Args& a1, const XArgs& xa, int ncomp)
{
    auto kern = k_line_x<L, OP, DIM>;
    const size_t sm = tile_bytes(s) + red_bytes(s);
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) return e;
    dim3 grid((unsigned)((s->n + s->R - 1) / s->R), (unsigned)(s->dim == 3 ? s->n : 1));
    kern<<<grid, s->R * s->P, sm, s->stream>>>(s->coef, sys, (int)s->n, s->R, a1, xa, ncomp);
    s->launches++;
    return cudaGetLastError();
}

template <int L, int OP>
static cudaError_t go_yz(Ctx* s, int sys, int axis, const YZArgs& a, int ncomp)
{
    auto kern = k_line_yz<L, OP>;
    const size_t sm = red_bytes(s);
    dim3 grid((unsigned)((s->n + s->R - 1) / s->R), (unsigned)(s->dim == 3 ? s->n : 1), (unsigned)ncomp);
    kern<<<grid, s->R * s->P, sm, s->stream>>>(s->coef, sys, (int)s->n, s->R, axis, a);
    s->launches++;
    return cudaGetLastError();
}

#define IBGM_DISPATCH_L(Lval, CALL)      \
    switch (Lval) {                      \
        case 2: { constexpr int LL = 2; return CALL; }   \
        case 3: { constexpr int LL = 3; return CALL; }   \
        case 4: { constexpr int LL = 4; return CALL; }   \
        case 6: { constexpr int LL = 6; return CALL; }   \
        case 8: { constexpr int LL = 8; return CALL; }   \
        case 12: { constexpr int LL = 12; return CALL; } \
        case 16: { constexpr int LL = 16; return CALL; } \
        case 24: { constexpr int LL = 24; return CALL; } \
        case 32: { constexpr int LL = 32; return CALL; } \
        default: return cudaErrorInvalidValue;           \
    }

template <int OP>
static cudaError_t go_x_dim(Ctx* s, int sys, const S1Args& a1, const XArgs& xa, int ncomp)
{
    if (s->dim == 3) { IBGM_DISPATCH_L(s->L, (go_x<LL, OP, 3>(s, sys, a1, xa, ncomp))) }
    IBGM_DISPATCH_L(s->L, (go_x<LL, OP, 2>(s, sys, a1, xa, ncomp)))
}

cudaError_t launch_s1_x(Ctx* s, int first_step)
{
    S1Args a{};
    for (int c = 0; c < 3; ++c) {
        a.u[c] = s->u[c]; a.nprev[c] = s->nprev[c]; a.f[c] = s->f[c];
        a.nadv[c] = s->nadv[c]; a.out[c] = s->st[c];
    }
    a.p = s->p; a.psi = s->psi;
    a.dt = s->dt; a.rho = s->rho; a.mu = s->mu; a.invh = 1.0 / s->h;
    a.kap = s->mu * s->dt / (2.0 * s->rho * s->h * s->h);
    a.first = first_step; a.advection = s->advection;
    XArgs xa{};
    return go_x_dim<OPX_S1>(s, SYS_VISC, a, xa, s->dim);
}

cudaError_t launch_visc_sweep(Ctx* s, int axis)
{
    YZArgs a{};
    for (int c = 0; c < 3; ++c) { a.in[c] = s->st[c]; a.un[c] = s->u[c]; a.out[c] = s->st[c]; }
    a.kap = s->mu * s->dt / (2.0 * s->rho * s->h * s->h);
    IBGM_DISPATCH_L(s->L, (go_yz<LL, OPYZ_VISC>(s, SYS_VISC, axis, a, s->dim)))
}

cudaError_t launch_div(Ctx* s)
{
    const int threads = 256;
    const size_t nc = (size_t)s->ncell;
    unsigned blocks = (unsigned)((nc + threads - 1) / threads);
    if (blocks > 148u * 16u) blocks = 148u * 16u;
    const double invh = 1.0 / s->h;
    if (s->dim == 3)
        k_div<3><<<blocks, threads, 0, s->stream>>>(s->u[0], s->u[1], s->u[2], s->st[0], s->st[1], s->st[2], s->psi,
                                                     s->p, (int)s->n, invh, s->rho / s->dt, s->chi * s->mu);
    else
        k_div<2><<<blocks, threads, 0, s->stream>>>(s->u[0], s->u[1], nullptr, s->st[0], s->st[1], nullptr, s->psi,
                                                     s->p, (int)s->n, invh, s->rho / s->dt, s->chi * s->mu);
    s->launches++;
    return cudaGetLastError();
}

cudaError_t launch_psi_sweep(Ctx* s, int axis, int last)
{
    if (axis == 0) {
        S1Args a1{};
        XArgs xa{};
        xa.in = s->psi; xa.out = s->psi; xa.p = s->p;
        if (last) return go_x_dim<OPX_PSI_LAST>(s, SYS_PSI, a1, xa, 1);
        return go_x_dim<OPX_USER>(s, SYS_PSI, a1, xa, 1);
    }
    YZArgs a{};
    a.in[0] = s->psi; a.out[0] = s->psi;
    IBGM_DISPATCH_L(s->L, (go_yz<LL, OPYZ_PSI>(s, SYS_PSI, axis, a, 1)))
}

cudaError_t launch_line_solve(Ctx* s, int axis, int sys, double* data)
{
    if (axis == 0) {
        S1Args a1{};
        XArgs xa{};
        xa.in = data; xa.out = data;
        return go_x_dim<OPX_USER>(s, sys, a1, xa, 1);
    }
    YZArgs a{};
    a.in[0] = data; a.out[0] = data;
    IBGM_DISPATCH_L(s->L, (go_yz<LL, OPYZ_USER>(s, sys, axis, a, 1)))
}

}  // namespace ibgm
