// Fluid passes of the IB-GM step on the GPU (sm_100a, fp64).
//
// Steps 3a-3f of PAPER.md:624-683 as line passes over the periodic MAC grid (x
// fastest, flat index i + N*(j + N*k)).  3D schedule (2D drops the z pass):
//   S1   x-lines  p* (3a), explicit momentum with AB2 skew advection (3b) and the x
//                 Douglas sweep (3c), all components at once; stores N(u^n).
//   MID  y-lines  Douglas sweep (3d) on the increments.
//   LAST z-lines  last Douglas sweep; u^{n+1} = u^n + delta.
//   DIVPSI z      r = -(rho/dt) D.u^{n+1} (3e RHS) computed on the fly, q = p -
//                 chi mu D.(u^{n+1}+u^n)/2 (explicit part of 3f), and the first psi
//                 factor (1 - D_zz)^{-1} (eqs. PenaltyStepPart1/2).
//   PSIMID y      (1 - D_yy)^{-1}.
//   PSILAST x     (1 - D_xx)^{-1}; p^{n+1/2} = q + psi (3f); p* = p + psi for 3a.
// The Douglas sweeps run in increment form: with A_a = (mu dt/2rho) D_aa,
//   (1-A_x) d1 = u* - u^n,  (1-A_y) d2 = d1,  (1-A_z) d3 = d2,  u^{n+1} = u^n + d3,
// which is algebraically identical to eqs. umacstep1/2 and needs no
// re-read of u^n per sweep (R23).  The spread force enters through the AB2
// history: G = N(u^{n-1}) + (2/rho) f, so that 3/2 N(u^n) - 1/2 G = N^{n+1/2} - f/rho.
//
// Every line pass solves independent cyclic tridiagonal systems (eq. TriDiagX,
// PAPER.md:985-995) with the paper's Schur-complement splitting
// mapped onto one CTA: a line is cut into P parts of L unknowns; one thread per part
// runs Thomas's algorithm on its interior block in registers, the P x P periodic
// Schur system is solved with the precomputed dense S^{-1} through shared memory, and
// each thread corrects x = f* - B^{-1} E y.  Strided (y, z) lines put neighbouring
// lines on neighbouring lanes so every global access is coalesced; contiguous x lines
// are staged through a padded shared-memory tile with coalesced loads and stores.
#include <cuda_runtime.h>

#include <cstdio>

#include "ibgm_internal.cuh"

namespace ibgm {

__device__ __forceinline__ int wrapn(int i, int n) { return i < 0 ? i + n : (i >= n ? i - n : i); }
__device__ __forceinline__ double ldg(const double* p) { return __ldg(p); }
// select one of three pointers without dynamic indexing of a parameter array (which
// would copy the kernel parameters to local memory)
template <typename T>
__device__ __forceinline__ T pick3(T a, T b, T c, int i) { return i == 0 ? a : (i == 1 ? b : c); }

// -------------------------------------------------------------------------------
// Schur-segmented solve of NC independent lines' parts (one part per thread and
// component).  On entry x[k][0..L-1] holds the right-hand side of rows sL..sL+L-1;
// on exit the solution.  Block-uniform control flow (2 __syncthreads).
//   sh layout: per component k: first[PR] last[PR] r[PR] e[PR]   (PR = P*R)
// -------------------------------------------------------------------------------
template <int L, int NC>
__device__ __forceinline__ void schur_solve(double (&x)[NC][L], const LineCoef& C, int s, int l, int R, int P,
                                            const double* __restrict__ sh_sinv, const double* __restrict__ sh_cs,
                                            double* sh)
{
    constexpr int M = L - 1;
    const double c = C.c, b = C.b;
    const int PR = P * R;
    const int me = s * R + l;
    const int sm1 = (s == 0) ? P - 1 : s - 1;
    const int sp1 = (s == P - 1) ? 0 : s + 1;
    const bool mf = C.mean_fix != 0;
#pragma unroll
    for (int k = 0; k < NC; ++k) {
        double dsum = 0.0;
        if (mf) {
#pragma unroll
            for (int i = 0; i < L; ++i) dsum += x[k][i];
        }
        // f*_p = B_p^{-1} f_p  (eq. LocalTriSystem; Thomas)
        x[k][1] *= C.inv[0];
#pragma unroll
        for (int i = 2; i <= M; ++i) x[k][i] = (x[k][i] - c * x[k][i - 1]) * C.inv[i - 1];
#pragma unroll
        for (int i = M - 1; i >= 1; --i) x[k][i] -= C.cp[i - 1] * x[k][i + 1];
        double* shk = sh + 4 * PR * k;
        // gather first/last entries of f*_p
        shk[me] = x[k][1];
        shk[PR + me] = x[k][M];
        if (mf) {
            double fsum = 0.0;
#pragma unroll
            for (int i = 1; i <= M; ++i) fsum += x[k][i];
            shk[3 * PR + me] = dsum * C.inv_rowsum - fsum;
        }
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < NC; ++k) {
        double* shk = sh + 4 * PR * k;
        // right-hand side of the Schur system  g - F f*  (eq. SchurSystem)
        shk[2 * PR + me] = x[k][0] - c * shk[PR + sm1 * R + l] - b * shk[me];
    }
    __syncthreads();
    const double* Si = sh_sinv + s * P;
    const double* Si1 = sh_sinv + sp1 * P;
#pragma unroll
    for (int k = 0; k < NC; ++k) {
        const double* shk = sh + 4 * PR * k;
        // y = S^{-1}(g - F f*); this part needs y_p and y_{p+1}
        double ys = 0.0, ys1 = 0.0, ysum = 0.0, E = 0.0;
        for (int q = 0; q < P; ++q) {
            const double r = shk[2 * PR + q * R + l];
            ys = fma(Si[q], r, ys);
            ys1 = fma(Si1[q], r, ys1);
            if (mf) {
                ysum = fma(sh_cs[q], r, ysum);
                E += shk[3 * PR + q * R + l];
            }
        }
        // x_p = f*_p - B_p^{-1} E_p y; E_p y = c y_p e_1 + b y_{p+1} e_m
        x[k][0] = ys;
        const double cy = c * ys, by = b * ys1;
#pragma unroll
        for (int i = 1; i <= M; ++i) x[k][i] -= cy * C.g[i - 1] + by * C.h[i - 1];
        if (mf) {
            // exact line-mean correction (R16): 1^T A = (a+b+c) 1^T, so
            // sum(x) must equal sum(d)/(a+b+c).  sum over the line of the computed x is
            // (1 - c sum g - b sum h) sum_p y_p + sum_p sum f*_p  (no third barrier).
            const double corr = (E - (1.0 - c * C.gsum - b * C.hsum) * ysum) / (double)(P * L);
#pragma unroll
            for (int i = 0; i < L; ++i) x[k][i] += corr;
        }
    }
}

__device__ __forceinline__ void load_sinv(const SchurInv* __restrict__ SI, int P, double* sh_sinv, double* sh_cs)
{
    for (int e = threadIdx.x; e < P * P; e += blockDim.x) sh_sinv[e] = SI->sinv[e];
    for (int e = threadIdx.x; e < P; e += blockDim.x) sh_cs[e] = SI->colsum[e];
}

// -------------------------------------------------------------------------------
// S1: all components of  d = u* - u^n  at one cell (Steps 3a-3b)
// -------------------------------------------------------------------------------
struct S1Args {
    const double* u[3];
    const double* G[3];     // N(u^{n-1}) + (2/rho) f^{n+1/2}
    const double* pstar;    // p^{n-1/2} + psi^{n-1/2}
    double* nadv[3];        // out: N(u^n)
    double* out[3];         // out: d1 (x-swept increment)
    double dt, inv_rho, mu, invh, a1;   // a1 = 3/2, or 1 at n = 0
    int first, advection;
};

template <int DIM>
__device__ __forceinline__ void s1_cell(const S1Args& A, int i, int j, int k, int n, double (&d)[3])
{
    const size_t N = (size_t)n;
    const int im = (i == 0) ? n - 1 : i - 1, ip = (i == n - 1) ? 0 : i + 1;
    const size_t rj = N * j, rjm = N * (size_t)((j == 0) ? n - 1 : j - 1), rjp = N * (size_t)((j == n - 1) ? 0 : j + 1);
    size_t rk = 0, rkm = 0, rkp = 0;
    if (DIM == 3) {
        rk = N * N * k;
        rkm = N * N * (size_t)((k == 0) ? n - 1 : k - 1);
        rkp = N * N * (size_t)((k == n - 1) ? 0 : k + 1);
    }
    // offsets of I, I+e_x, I-e_x, I+e_y, I-e_y, I+e_z, I-e_z  (index 0, 1+2a, 2+2a)
    size_t o[7];
    o[0] = i + rj + rk;
    o[1] = ip + rj + rk;
    o[2] = im + rj + rk;
    o[3] = i + rjp + rk;
    o[4] = i + rjm + rk;
    o[5] = i + rj + rkp;
    o[6] = i + rj + rkm;
    // I + e_m - e_c  (m != c)
    size_t mx[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
    mx[0][1] = ip + rjm + rk;
    mx[1][0] = im + rjp + rk;
    if (DIM == 3) {
        mx[0][2] = ip + rj + rkm;
        mx[1][2] = i + rjp + rkm;
        mx[2][0] = im + rj + rkp;
        mx[2][1] = i + rjm + rkp;
    }
    constexpr int NO = 1 + 2 * DIM;
    double U[DIM][NO];
    double X[DIM][DIM];
#pragma unroll
    for (int m = 0; m < DIM; ++m) {
#pragma unroll
        for (int q = 0; q < NO; ++q) U[m][q] = ldg(A.u[m] + o[q]);
#pragma unroll
        for (int c = 0; c < DIM; ++c) X[m][c] = (c == m) ? 0.0 : ldg(A.u[m] + mx[m][c]);
    }
    double ps0 = 0.0, psm[3] = {0, 0, 0};
    if (!A.first) {
        ps0 = ldg(A.pstar + o[0]);
#pragma unroll
        for (int c = 0; c < DIM; ++c) psm[c] = ldg(A.pstar + o[2 + 2 * c]);
    }
    const double invh = A.invh;
#pragma unroll
    for (int c = 0; c < DIM; ++c) {
        const double u0 = U[c][0];
        // skew-symmetric advection, Morinishi "Skew.-S2" (R4)
        double Nc = 0.0;
        if (A.advection) {
            double dv = 0.0, ad = 0.0;
#pragma unroll
            for (int jd = 0; jd < DIM; ++jd) {
                const double ucm = U[c][2 + 2 * jd], ucp = U[c][1 + 2 * jd];
                const double Tm = 0.5 * (U[jd][0] + U[jd][2 + 2 * c]);
                const double Tp = 0.5 * (U[jd][1 + 2 * jd] + ((jd == c) ? u0 : X[jd][c]));
                const double Am = 0.5 * (u0 + ucm), Ap = 0.5 * (ucp + u0);
                const double Gm = (u0 - ucm) * invh, Gp = (ucp - u0) * invh;
                dv += (Tp * Ap - Tm * Am) * invh;
                ad += 0.5 * (Tm * Gm + Tp * Gp);
            }
            Nc = 0.5 * (dv + ad);
        }
        A.nadv[c][o[0]] = Nc;
        double lap = 0.0;
#pragma unroll
        for (int a = 0; a < DIM; ++a) lap += U[c][1 + 2 * a] - 2.0 * u0 + U[c][2 + 2 * a];
        lap *= invh * invh;
        const double gp = A.first ? 0.0 : (ps0 - psm[c]) * invh;     // G^{C->E} p*
        const double Gc = ldg(A.G[c] + o[0]);
        // u* - u^n = dt ( -3/2 N + 1/2 G + (mu lap - G p*)/rho ),  G carries f
        d[c] = A.dt * (-A.a1 * Nc + 0.5 * Gc + (A.mu * lap - gp) * A.inv_rho);
    }
}

// -------------------------------------------------------------------------------
// x-line kernels: R consecutive rows (j0..j0+R-1 at fixed k) staged in padded shared
// tiles [NC][R][N+1]; thread t -> row l = t % R, part s = t / R.
// -------------------------------------------------------------------------------
enum XOp { XOP_S1 = 0, XOP_PSI_LAST = 1, XOP_USER = 2 };

struct XArgs {
    const double* in;
    double* out;     // PSI_LAST: p* ; USER: x
    double* p;       // PSI_LAST: holds q, becomes p^{n+1/2}
};

template <int L, int OP, int DIM, int NCB>
__global__ void __launch_bounds__(512) k_line_x(const LineCoef C, const SchurInv* __restrict__ SI, int n, int R,
                                                 S1Args s1, XArgs xa)
{
    constexpr int NC = (OP == XOP_S1) ? DIM : 1;   // components in the tile; NCB solved jointly
    extern __shared__ double smem[];
    const int P = C.P;
    const int pitch = n + 1;
    double* sh_sinv = smem;
    double* sh_cs = sh_sinv + P * P;
    double* tile = sh_cs + P;
    double* red = tile + (size_t)NC * R * pitch;
    const int t = threadIdx.x, nthr = blockDim.x;
    const int l = t % R, s = t / R;
    const int j0 = blockIdx.x * R;
    const int k = blockIdx.y;
    const size_t plane = (size_t)n * n;
    load_sinv(SI, P, sh_sinv, sh_cs);

    // fill (coalesced along x)
    for (int e = t; e < R * n; e += nthr) {
        const int row = e / n, i = e - row * n;
        const int j = j0 + row;
        double v[3] = {0.0, 0.0, 0.0};
        if (j < n) {
            if (OP == XOP_S1) {
                s1_cell<DIM>(s1, i, j, k, n, v);
            } else {
                v[0] = ldg(xa.in + (size_t)i + (size_t)n * j + plane * k);
            }
        }
#pragma unroll
        for (int c = 0; c < NC; ++c) tile[(size_t)c * R * pitch + row * pitch + i] = v[c];
    }
    __syncthreads();
#pragma unroll
    for (int c0 = 0; c0 < NC; c0 += NCB) {
        double x[NCB][L];
#pragma unroll
        for (int c = 0; c < NCB; ++c)
#pragma unroll
            for (int i = 0; i < L; ++i) x[c][i] = tile[(size_t)(c0 + c) * R * pitch + l * pitch + s * L + i];
        schur_solve<L, NCB>(x, C, s, l, R, P, sh_sinv, sh_cs, red);
#pragma unroll
        for (int c = 0; c < NCB; ++c)
#pragma unroll
            for (int i = 0; i < L; ++i) tile[(size_t)(c0 + c) * R * pitch + l * pitch + s * L + i] = x[c][i];
    }
    __syncthreads();
    // store (coalesced along x)
    for (int e = t; e < R * n; e += nthr) {
        const int row = e / n, i = e - row * n;
        const int j = j0 + row;
        if (j < n) {
            const size_t q = (size_t)i + (size_t)n * j + plane * k;
            if (OP == XOP_S1) {
#pragma unroll
                for (int c = 0; c < NC; ++c) s1.out[c][q] = tile[(size_t)c * R * pitch + row * pitch + i];
            } else if (OP == XOP_PSI_LAST) {
                const double psi = tile[row * pitch + i];
                const double pn = xa.p[q] + psi;        // Step 3f: p^{n+1/2} = q + psi^{n+1/2}
                xa.p[q] = pn;
                xa.out[q] = pn + psi;                   // Step 3a of the next step: p* = p + psi
            } else {
                xa.out[q] = tile[row * pitch + i];
            }
        }
    }
}

// -------------------------------------------------------------------------------
// y/z-line kernel: R neighbouring lines (consecutive i) per block, direct coalesced
// global access; thread t -> line l = t % R, part s = t / R.
// -------------------------------------------------------------------------------
enum YOp { YOP_MID = 0, YOP_LAST = 1, YOP_DIVPSI = 2 };

struct YArgs {
    double* io[3];          // MID: in/out increments; LAST: in increments, out u^{n+1}; DIVPSI: out psi
    const double* un[3];    // LAST / DIVPSI: u^n
    const double* unew[3];  // DIVPSI: u^{n+1}
    double* p;              // DIVPSI: p -> q
    double neg_rho_dt, chimu_half, invh;
};

template <int L, int NC, int OP, int DIM, int AX>
__global__ void __launch_bounds__(512) k_line_yz(const LineCoef C, const SchurInv* __restrict__ SI, int n, int R,
                                                  YArgs A)
{
    // NC components per block, starting at component blockIdx.z * NC; AX = line axis (1 or 2)
    constexpr int axis = AX;
    const int c0 = blockIdx.z * NC;
    extern __shared__ double smem[];
    const int P = C.P;
    double* sh_sinv = smem;
    double* sh_cs = sh_sinv + P * P;
    double* red = sh_cs + P;
    const int t = threadIdx.x;
    const int l = t % R, s = t / R;
    const int i = blockIdx.x * R + l;
    const bool active = i < n;
    const int ii = active ? i : 0;
    const size_t N = (size_t)n;
    const size_t S = (AX == 1) ? N : N * N;          // stride along the line
    const size_t T = (AX == 1) ? N * N : N;          // stride of the transverse index
    const size_t base = (size_t)ii + T * blockIdx.y;
    const int pos0 = s * L;
    load_sinv(SI, P, sh_sinv, sh_cs);

    double x[NC][L];
    if (OP == YOP_DIVPSI) {
        // D.u at the cells of this part for u^{n+1} and u^n; the
        // line axis component's +1 neighbour is the next position along the line.
        const size_t dxp = (ii == n - 1) ? (size_t)0 - (N - 1) : (size_t)1;               // +e_x offset
        const size_t dyp = (blockIdx.y == (unsigned)(n - 1)) ? (size_t)0 - (N - 1) * N : N; // +e_y (3D z-lines)
        double pn[L + 1];
#pragma unroll
        for (int m = 0; m <= L; ++m) pn[m] = 0.0;
        double dn[L], dol[L];
#pragma unroll
        for (int m = 0; m < L; ++m) { dn[m] = 0.0; dol[m] = 0.0; }
        // line-axis component: values at positions pos0 .. pos0+L (wrapped)
        {
            const double* a1 = A.unew[axis];
            const double* a0 = A.un[axis];
            double v1[L + 1], v0[L + 1];
#pragma unroll
            for (int m = 0; m <= L; ++m) {
                const size_t q = base + S * (size_t)wrapn(pos0 + m, n);
                v1[m] = ldg(a1 + q);
                v0[m] = ldg(a0 + q);
            }
#pragma unroll
            for (int m = 0; m < L; ++m) { dn[m] += v1[m + 1] - v1[m]; dol[m] += v0[m + 1] - v0[m]; }
        }
#pragma unroll
        for (int c = 0; c < DIM; ++c) {
            if (c == axis) continue;
            const size_t off = (c == 0) ? dxp : dyp;
            const double* a1 = A.unew[c];
            const double* a0 = A.un[c];
#pragma unroll
            for (int m = 0; m < L; ++m) {
                const size_t q = base + S * (size_t)(pos0 + m);
                dn[m] += ldg(a1 + q + off) - ldg(a1 + q);
                dol[m] += ldg(a0 + q + off) - ldg(a0 + q);
            }
        }
#pragma unroll
        for (int m = 0; m < L; ++m) {
            const size_t q = base + S * (size_t)(pos0 + m);
            const double dnew = dn[m] * A.invh, dold = dol[m] * A.invh;
            x[0][m] = A.neg_rho_dt * dnew;                             // Step 3e RHS
            if (active) A.p[q] = A.p[q] - A.chimu_half * (dnew + dold);  // Step 3f, explicit part
        }
    } else {
#pragma unroll
        for (int c = 0; c < NC; ++c) {
            const double* in = pick3<double*>(A.io[0], A.io[1], A.io[2], c0 + c);
#pragma unroll
            for (int m = 0; m < L; ++m) x[c][m] = ldg(in + base + S * (size_t)(pos0 + m));
        }
    }
    schur_solve<L, NC>(x, C, s, l, R, P, sh_sinv, sh_cs, red);
    if (active) {
#pragma unroll
        for (int c = 0; c < NC; ++c) {
            double* out = pick3<double*>(A.io[0], A.io[1], A.io[2], c0 + c);
            const double* un = pick3<const double*>(A.un[0], A.un[1], A.un[2], c0 + c);
#pragma unroll
            for (int m = 0; m < L; ++m) {
                const size_t q = base + S * (size_t)(pos0 + m);
                if (OP == YOP_LAST) out[q] = ldg(un + q) + x[c][m];   // u^{n+1} = u^n + d
                else out[q] = x[c][m];
            }
        }
    }
}

__global__ void k_sub(const double* __restrict__ a, const double* __restrict__ b, double* __restrict__ o, size_t cnt)
{
    for (size_t q = blockIdx.x * (size_t)blockDim.x + threadIdx.x; q < cnt; q += (size_t)gridDim.x * blockDim.x)
        o[q] = a[q] - b[q];
}

// -------------------------------------------------------------------------------
// launchers
// -------------------------------------------------------------------------------
static size_t smem_limit() { return 220 * 1024; }

// rows per x block: prefer 16, shrink to fit 512 threads and the shared-memory budget
static int pick_rx(const Ctx* s, int nc)
{
    for (int R = 16; R >= 1; R /= 2) {
        if (R * s->P > 512) continue;
        const size_t sm = ((size_t)s->P * s->P + s->P + (size_t)nc * R * (s->n + 1) + (size_t)4 * nc * s->P * R) * 8;
        if (sm <= smem_limit()) return R;
    }
    return 1;
}

static int pick_ryz(const Ctx* s, int nc)
{
    int R = (nc > 1 ? 256 : 512) / s->P;
    if (R > 32) R = 32;
    if (R < 1) R = 1;
    return R;
}

// components solved jointly per thread: keep the register arrays x[NCB][L] small
template <int L, int NC, int LIM>
struct Ncb { static constexpr int value = (L * NC <= LIM) ? NC : 1; };

template <int L, int OP, int DIM>
static cudaError_t go_x(Ctx* s, int sys, const S1Args& a1, const XArgs& xa)
{
    constexpr int NC = (OP == XOP_S1) ? DIM : 1;
    constexpr int NCB = Ncb<L, NC, 36>::value;
    const int R = pick_rx(s, NC);
    auto kern = k_line_x<L, OP, DIM, NCB>;
    const size_t sm = ((size_t)s->P * s->P + s->P + (size_t)NC * R * (s->n + 1) + (size_t)4 * NCB * s->P * R) * 8;
    static bool attr_set = false;   // per instantiation
    if (!attr_set) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_limit());
        if (e != cudaSuccess) return e;
        attr_set = true;
    }
    dim3 grid((unsigned)((s->n + R - 1) / R), (unsigned)(s->dim == 3 ? s->n : 1));
    kern<<<grid, R * s->P, sm, s->stream>>>(s->hcoef[sys], s->sinv + sys, (int)s->n, R, a1, xa);
    s->launches++;
    return cudaGetLastError();
}

template <int L, int NC, int OP, int DIM, int AX>
static cudaError_t go_yz(Ctx* s, int sys, const YArgs& a)
{
    constexpr int NCB = Ncb<L, NC, 24>::value;
    const int R = pick_ryz(s, NCB);
    auto kern = k_line_yz<L, NCB, OP, DIM, AX>;
    const size_t sm = ((size_t)s->P * s->P + s->P + (size_t)4 * NCB * s->P * R) * 8;
    static bool attr_set = false;
    if (!attr_set) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_limit());
        if (e != cudaSuccess) return e;
        attr_set = true;
    }
    dim3 grid((unsigned)((s->n + R - 1) / R), (unsigned)(s->dim == 3 ? s->n : 1), (unsigned)(NC / NCB));
    kern<<<grid, R * s->P, sm, s->stream>>>(s->hcoef[sys], s->sinv + sys, (int)s->n, R, a);
    s->launches++;
    return cudaGetLastError();
}

#define IBGM_DISPATCH_L(Lval, CALL)                      \
    switch (Lval) {                                      \
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
static cudaError_t go_x_dim(Ctx* s, int sys, const S1Args& a1, const XArgs& xa)
{
    if (s->dim == 3) { IBGM_DISPATCH_L(s->L, (go_x<LL, OP, 3>(s, sys, a1, xa))) }
    IBGM_DISPATCH_L(s->L, (go_x<LL, OP, 2>(s, sys, a1, xa)))
}

// NC3/NC2: components of the pass in 3D/2D; axis 1 or 2
template <int NC3, int NC2, int OP>
static cudaError_t go_yz_dim(Ctx* s, int sys, int axis, const YArgs& a)
{
    if (s->dim == 3) {
        if (axis == 2) { IBGM_DISPATCH_L(s->L, (go_yz<LL, NC3, OP, 3, 2>(s, sys, a))) }
        IBGM_DISPATCH_L(s->L, (go_yz<LL, NC3, OP, 3, 1>(s, sys, a)))
    }
    IBGM_DISPATCH_L(s->L, (go_yz<LL, NC2, OP, 2, 1>(s, sys, a)))
}

cudaError_t launch_s1_x(Ctx* s, int first_step)
{
    S1Args a{};
    for (int c = 0; c < 3; ++c) {
        a.u[c] = s->u[c]; a.G[c] = s->nprev[c]; a.nadv[c] = s->nadv[c]; a.out[c] = s->st[c];
    }
    a.pstar = s->pstar;
    a.dt = s->dt; a.inv_rho = 1.0 / s->rho; a.mu = s->mu; a.invh = 1.0 / s->h;
    a.a1 = first_step ? 1.0 : 1.5;
    a.first = first_step; a.advection = s->advection;
    XArgs xa{};
    return go_x_dim<XOP_S1>(s, SYS_VISC, a, xa);
}

cudaError_t launch_sweep_mid(Ctx* s, int axis)
{
    YArgs a{};
    for (int c = 0; c < 3; ++c) a.io[c] = s->st[c];
    return go_yz_dim<3, 2, YOP_MID>(s, SYS_VISC, axis, a);
}

cudaError_t launch_sweep_last(Ctx* s, int axis)
{
    YArgs a{};
    for (int c = 0; c < 3; ++c) { a.io[c] = s->st[c]; a.un[c] = s->u[c]; }
    return go_yz_dim<3, 2, YOP_LAST>(s, SYS_VISC, axis, a);
}

cudaError_t launch_div_psi_first(Ctx* s, int axis)
{
    YArgs a{};
    a.io[0] = s->pstar;
    for (int c = 0; c < 3; ++c) { a.un[c] = s->u[c]; a.unew[c] = s->st[c]; }
    a.p = s->p;
    a.neg_rho_dt = -s->rho / s->dt;
    a.chimu_half = 0.5 * s->chi * s->mu;
    a.invh = 1.0 / s->h;
    return go_yz_dim<1, 1, YOP_DIVPSI>(s, SYS_PSI, axis, a);
}

cudaError_t launch_psi_mid(Ctx* s, int axis)
{
    YArgs a{};
    a.io[0] = s->pstar;
    return go_yz_dim<1, 1, YOP_MID>(s, SYS_PSI, axis, a);
}

cudaError_t launch_psi_last_x(Ctx* s)
{
    S1Args a1{};
    XArgs xa{};
    xa.in = s->pstar; xa.out = s->pstar; xa.p = s->p;
    return go_x_dim<XOP_PSI_LAST>(s, SYS_PSI, a1, xa);
}

cudaError_t launch_line_solve(Ctx* s, int axis, int sys, double* data)
{
    if (axis == 0) {
        S1Args a1{};
        XArgs xa{};
        xa.in = data; xa.out = data;
        return go_x_dim<XOP_USER>(s, sys, a1, xa);
    }
    YArgs a{};
    a.io[0] = data;
    return go_yz_dim<1, 1, YOP_MID>(s, sys, axis, a);
}

cudaError_t launch_sub(Ctx* s, const double* a, const double* b, double* out)
{
    k_sub<<<592, 256, 0, s->stream>>>(a, b, out, (size_t)s->ncell);
    s->launches++;
    return cudaGetLastError();
}

}  // namespace ibgm
