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
// mapped onto one WARP: a line is cut into P parts of L unknowns and the P parts sit
// in P lanes.  Each lane runs Thomas's algorithm on its interior block in registers
// (the paper's "local tridiagonal solver"), the gather/scatter of the interface
// values become register shuffles, the P x P periodic Schur
// system is applied through the precomputed dense S^{-1}, and each lane corrects
// x = f* - B^{-1} E y -- no block barrier inside the solve.  Every pass stages its
// R lines x N positions through a segment-padded shared-memory tile, filled and
// drained with coalesced global accesses (consecutive x for every axis).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "ibgm_internal.cuh"

namespace ibgm {

__device__ __forceinline__ int wrapn(int i, int n) { return i < 0 ? i + n : (i >= n ? i - n : i); }
__device__ __forceinline__ double ldg(const double* p) { return __ldg(p); }
// select one of three pointers without dynamic indexing of a parameter array (which
// would copy the kernel parameters to local memory)
template <typename T>
__device__ __forceinline__ T pick3(T a, T b, T c, int i) { return i == 0 ? a : (i == 1 ? b : c); }


constexpr unsigned kFull = 0xffffffffu;

// cp.async (LDGSTS) of one double global -> shared, cached in L1/L2; completes at
// cp_async_wait_all().  Lets a thread keep all its tile loads in flight at once.
__device__ __forceinline__ void cp_async8(double* sdst, const double* gsrc)
{
    const unsigned sa = (unsigned)__cvta_generic_to_shared(sdst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all()
{
    asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
}

// -------------------------------------------------------------------------------
// Staged tile: R lines x N positions; segment s of a line (L positions) occupies L+1
// doubles so that lanes holding consecutive segments of a line hit distinct banks,
// and the line pitch TP is odd so that consecutive lines do too.
// -------------------------------------------------------------------------------
__host__ __device__ inline int tile_pitch(int P, int L)
{
    const int tp = P * (L + 1);
    return (tp % 2 == 0) ? tp + 1 : tp;
}

template <int L>
__device__ __forceinline__ int tile_off(int l, int m, int TP)
{
    const int s = m / L;
    return l * TP + s * (L + 1) + (m - s * L);
}

template <int P2>
__device__ __forceinline__ double group_sum(double v, int P, int gbase)
{
    if ((P & (P - 1)) == 0) {
        for (int off = P >> 1; off >= 1; off >>= 1) v += __shfl_xor_sync(kFull, v, off);
        return v;
    }
    double t = 0.0;
    for (int q = 0; q < P; ++q) t += __shfl_sync(kFull, v, gbase + q);
    return t;
}

// Which forms of y = S^{-1} r a pass compiles (MODES bit mask; the unused unrolled
// forms cost instruction-cache space): viscous passes are banded, psi passes circulant.
constexpr int kSchurBand = 1, kSchurCirc = 2;
__host__ __device__ constexpr int schur_modes(int kind)
{
    return (kind == 0 || kind == 2) ? kSchurBand : ((kind == 3 || kind == 4) ? kSchurCirc : kSchurBand | kSchurCirc);
}

// y_s = (S^{-1} r)_s with r_q held by lane gbase + q: the banded circulant form when the
// line's S^{-1} allows it (LineCoef::band), the full circulant row (LineCoef::circ), else
// the dense row s of S^{-1} (sinvT in shared memory).  All 32 lanes must call it.
template <int MODES>
__device__ __forceinline__ double schur_apply_lanes(const LineCoef& C, double r, int s, int P, int gbase,
                                                    const double* __restrict__ sinvT)
{
    const int B = C.band;
    if ((MODES & kSchurBand) && B >= 0) {
        double ys = C.w[kMaxBand] * r;
#pragma unroll
        for (int d = 1; d <= kMaxBand; ++d) {
            if (d > B) break;
            const int qp = (s + d >= P) ? s + d - P : s + d, qm = (s - d < 0) ? s - d + P : s - d;
            ys = fma(C.w[kMaxBand + d], __shfl_sync(kFull, r, gbase + qp), ys);
            ys = fma(C.w[kMaxBand - d], __shfl_sync(kFull, r, gbase + qm), ys);
        }
        return ys;
    }
    double ys = 0.0;
    if ((MODES & kSchurCirc) && C.circ) {
        // circulant: y_s = sum_d wf[d] r_{(s+d) mod P}, wf uniform across lanes
#pragma unroll
        for (int d = 0; d < kMaxSeg; ++d) {
            if (d >= P) break;
            const int q = (s + d >= P) ? s + d - P : s + d;
            ys = fma(C.wf[d], __shfl_sync(kFull, r, gbase + q), ys);
        }
        return ys;
    }
    for (int q = 0; q < P; ++q) ys = fma(sinvT[q * P + s], __shfl_sync(kFull, r, gbase + q), ys);
    return ys;
}

// -------------------------------------------------------------------------------
// Warp-synchronous Schur-segmented solve of one part (L unknowns, rows sL..sL+L-1)
// of a cyclic line whose P parts sit in lanes gbase .. gbase+P-1.  All 32 lanes of
// the warp must call it.
// -------------------------------------------------------------------------------
template <int L, int MODES>
__device__ __forceinline__ void ws_solve(double (&x)[L], const LineCoef& C, int s, int P, int gbase,
                                         const double* __restrict__ sinvT)
{
    constexpr int M = L - 1;
    const double c = C.c, b = C.b;
    const bool mf = C.mean_fix != 0;
    double dsum = 0.0;
    if (mf) {
#pragma unroll
        for (int i = 0; i < L; ++i) dsum += x[i];
    }
    // f*_p = B_p^{-1} f_p  (eq. LocalTriSystem; Thomas)
    x[1] *= C.inv[0];
#pragma unroll
    for (int i = 2; i <= M; ++i) x[i] = (x[i] - c * x[i - 1]) * C.inv[i - 1];
#pragma unroll
    for (int i = M - 1; i >= 1; --i) x[i] -= C.cp[i - 1] * x[i + 1];
    // gather: the interface row p couples to the last entry of f*_{p-1} and the first
    // of f*_p; r = g - F f*  (eq. SchurSystem)
    const int sprev = gbase + ((s == 0) ? P - 1 : s - 1);
    const int snext = gbase + ((s == P - 1) ? 0 : s + 1);
    const double fl_prev = __shfl_sync(kFull, x[M], sprev);
    const double r = x[0] - c * fl_prev - b * x[1];
    // y = S^{-1} r  (S precomputed); this part needs y_p, y_{p+1}
    const double ys = schur_apply_lanes<MODES>(C, r, s, P, gbase, sinvT);
    const double ys1 = __shfl_sync(kFull, ys, snext);
    // correction x_p = f*_p - B_p^{-1} E_p y, E_p y = c y_p e_1 + b y_{p+1} e_m
    x[0] = ys;
    const double cy = c * ys, by = b * ys1;
#pragma unroll
    for (int i = 1; i <= M; ++i) x[i] -= cy * C.g[i - 1] + by * C.h[i - 1];
    if (mf) {
        // exact line-mean correction (R16): 1^T A = (a+b+c) 1^T, so
        // sum(x) must equal sum(d)/(a+b+c)
        double xs = 0.0;
#pragma unroll
        for (int i = 0; i < L; ++i) xs += x[i];
        const double D = group_sum<0>(dsum, P, gbase);
        const double X = group_sum<0>(xs, P, gbase);
        const double corr = (D * C.inv_rowsum - X) * C.inv_n;
#pragma unroll
        for (int i = 0; i < L; ++i) x[i] += corr;
    }
}

// -------------------------------------------------------------------------------
// The same solve for long segments (L = 64, 128: 2D N = 2048, 4096), run directly on the
// lane's segment of the shared tile (no register array) with the factors in C.ext.
// -------------------------------------------------------------------------------
template <int L, int MODES>
__device__ __forceinline__ void ws_solve_smem(double* x, const LineCoef& C, int s, int P, int gbase,
                                              const double* __restrict__ sinvT)
{
    constexpr int M = L - 1;
    const double c = C.c, b = C.b;
    const bool mf = C.mean_fix != 0;
    const double* inv = C.ext;
    const double* cpv = C.ext + M;
    const double* gv = C.ext + 2 * M;
    const double* hv = C.ext + 3 * M;
    double dsum = 0.0;
    if (mf)
        for (int i = 0; i < L; ++i) dsum += x[i];
    // Thomas on the interior block
    double prev = x[1] * __ldg(inv);
    x[1] = prev;
    for (int i = 2; i <= M; ++i) {
        prev = (x[i] - c * prev) * __ldg(inv + i - 1);
        x[i] = prev;
    }
    for (int i = M - 1; i >= 1; --i) {
        prev = x[i] - __ldg(cpv + i - 1) * prev;
        x[i] = prev;
    }
    const int sprev = gbase + ((s == 0) ? P - 1 : s - 1);
    const int snext = gbase + ((s == P - 1) ? 0 : s + 1);
    const double fl_prev = __shfl_sync(kFull, x[M], sprev);
    const double r = x[0] - c * fl_prev - b * x[1];
    const double ys = schur_apply_lanes<MODES>(C, r, s, P, gbase, sinvT);
    const double ys1 = __shfl_sync(kFull, ys, snext);
    x[0] = ys;
    const double cy = c * ys, by = b * ys1;
    double xs = ys;
    for (int i = 1; i <= M; ++i) {
        const double v = x[i] - (cy * __ldg(gv + i - 1) + by * __ldg(hv + i - 1));
        x[i] = v;
        xs += v;
    }
    if (mf) {
        const double D = group_sum<0>(dsum, P, gbase);
        const double X = group_sum<0>(xs, P, gbase);
        const double corr = (D * C.inv_rowsum - X) * C.inv_n;
        for (int i = 0; i < L; ++i) x[i] += corr;
    }
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
    double* divn;           // out (if set): D.u^n at each cell, for the first psi pass (Step 3f)
    double dt, inv_rho, mu, invh, a1;   // a1 = 3/2, or 1 at n = 0
    int first, advection;
};

// Row bases of one x-row (j, k) and its y/z neighbours, signed 32-bit flat offsets.
// The last axis (z in 3D, y in 2D) has nl local planes; it wraps periodically on a
// single GPU (wrap = 1) and, on a z-slab (wrap = 0), reaches the halo planes -1 and nl
// that the halo exchange filled.
struct RowB {
    int r0, ryp, rym, rzp, rzm, rypzm, rymzp;
};

__device__ __forceinline__ int nbr_lo(int k, int nl, int wrap) { return (k == 0) ? (wrap ? nl - 1 : -1) : k - 1; }
__device__ __forceinline__ int nbr_hi(int k, int nl, int wrap) { return (k == nl - 1) ? (wrap ? 0 : nl) : k + 1; }

template <int DIM>
__device__ __forceinline__ RowB row_bases(int j, int k, int n, int nl, int wrap)
{
    const int N = n, NN = n * n;
    int jm, jp;
    if (DIM == 2) {
        jm = nbr_lo(j, nl, wrap);
        jp = nbr_hi(j, nl, wrap);
    } else {
        jm = (j == 0) ? n - 1 : j - 1;
        jp = (j == n - 1) ? 0 : j + 1;
    }
    RowB b;
    int kk = 0, km = 0, kp = 0;
    if (DIM == 3) {
        kk = NN * k;
        km = NN * nbr_lo(k, nl, wrap);
        kp = NN * nbr_hi(k, nl, wrap);
    }
    b.r0 = N * j + kk;
    b.ryp = N * jp + kk;
    b.rym = N * jm + kk;
    b.rzp = N * j + kp;
    b.rzm = N * j + km;
    b.rypzm = N * jp + km;
    b.rymzp = N * jm + kp;
    return b;
}

// Skew-symmetric advection (Morinishi "Skew.-S2", R4).  With
// T = u_j averaged in c, A = u_c averaged in j and g = d_j u_c at the faces I -/+ h/2 e_j,
// (1/2)[ sum_j (TA|+ - TA|-)/h + sum_j (Tg|- + Tg|+)/2 ] collapses exactly (the u_c(I)
// terms cancel) to
//   N_c = 1/(4h) sum_j [ (u_j(I+e_j) + u_j(I+e_j-e_c)) u_c(I+e_j) - (u_j(I) + u_j(I-e_c)) u_c(I-e_j) ]
// L2 prefetch of the operands that miss in L1/L2 for cell i of a row (its centre, its
// z-neighbour planes, the history G and p*), issued one row ahead by the fill loop
// k_xwarp S1: warps per block and blocks per SM the registers must allow (measured at
// config 4, graph ms/step: 4 warps x 4 blocks 4.90-4.95, 8 x 2 4.86-4.89, 16 x 1 4.92-4.97,
// 2 x 8 5.22, 6 x 2 5.08)
#ifndef IBGM_S1_MINB
#define IBGM_S1_MINB 2
#endif
#ifndef IBGM_XWARP_WPB
#define IBGM_XWARP_WPB 8
#endif
#ifndef IBGM_S1_PREFETCH
#define IBGM_S1_PREFETCH 1
#endif
#ifndef IBGM_PF_L1
#define IBGM_PF_L1 0
#endif
#ifndef IBGM_PF_DIST
#define IBGM_PF_DIST 2          // fill iterations ahead (rows = T / n per iteration, n < T)
#endif
#ifndef IBGM_PF_ROWS
#define IBGM_PF_ROWS 1          // rows ahead when a row spans the block (n >= T)
#endif
#ifndef IBGM_PF_DIV
#define IBGM_PF_DIV 1           // prefetch in the divergence fill of the first psi pass (N <= 128)
#endif
#ifndef IBGM_DIV_CHUNK
#define IBGM_DIV_CHUNK 1        // contiguous-chunk, two-cells-in-flight fill when S1 supplies D.u^n
#endif
__device__ __forceinline__ void pf_l2(const double* p)
{
    if (IBGM_PF_L1) asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
    else asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}

template <int DIM>
__device__ __forceinline__ void s1_prefetch(const S1Args& A, int i, const RowB& rb)
{
    if (!IBGM_S1_PREFETCH) return;
#pragma unroll
    for (int c = 0; c < DIM; ++c) {
        pf_l2(A.u[c] + i + rb.r0);
        if (DIM == 3) {
            pf_l2(A.u[c] + i + rb.rzp);
            pf_l2(A.u[c] + i + rb.rzm);
        }
        pf_l2(A.G[c] + i + rb.r0);
    }
    pf_l2(A.pstar + i + rb.r0);
}

// The arithmetic of Steps 3a-3b at one cell from its gathered operands:
//   U[m][q]  u_m at I, I+e_x, I-e_x, I+e_y, I-e_y, I+e_z, I-e_z   (q = 0, 1+2a, 2+2a)
//   X[m][c]  u_m at I + e_m - e_c (m != c), the skew form's transport neighbours
//   ps0, psm p* at I and I - e_c;  Gv the AB2 history G_c at I
// returns N_c(u^n) and d_c = u*_c - u^n_c.
template <int DIM>
__device__ __forceinline__ void s1_eval(const S1Args& A, const double (&U)[DIM][1 + 2 * DIM],
                                        const double (&X)[DIM][DIM], double ps0, const double (&psm)[3],
                                        const double (&Gv)[3], double (&d)[3], double (&Nout)[3])
{
    const double invh = A.invh;
    const double dt_rho = A.dt * A.inv_rho;
#pragma unroll
    for (int c = 0; c < DIM; ++c) {
        const double u0 = U[c][0];
        double Nc = 0.0;
        if (A.advection) {
#pragma unroll
            for (int jd = 0; jd < DIM; ++jd) {
                const double Tp = U[jd][1 + 2 * jd] + ((jd == c) ? u0 : X[jd][c]);
                const double Tm = U[jd][0] + U[jd][2 + 2 * c];
                Nc = fma(Tp, U[c][1 + 2 * jd], Nc);
                Nc = fma(-Tm, U[c][2 + 2 * jd], Nc);
            }
            Nc *= 0.25 * invh;
        }
        Nout[c] = Nc;
        double lap = 0.0;
#pragma unroll
        for (int a = 0; a < DIM; ++a) lap += U[c][1 + 2 * a] + U[c][2 + 2 * a];
        lap = (lap - 2.0 * DIM * u0) * (invh * invh);
        const double gp = A.first ? 0.0 : (ps0 - psm[c]) * invh;     // G^{C->E} p*
        // u* - u^n = dt ( -3/2 N + 1/2 G + (mu lap - G p*)/rho ),  G carries f
        d[c] = A.dt * (0.5 * Gv[c] - A.a1 * Nc) + dt_rho * (A.mu * lap - gp);
    }
}

template <int DIM>
__device__ __forceinline__ void s1_cell(const S1Args& A, int i, const RowB& rb, int n, double (&d)[3])
{
    const int im = (i == 0) ? n - 1 : i - 1, ip = (i == n - 1) ? 0 : i + 1, ii = i;
    // offsets of I, I+e_x, I-e_x, I+e_y, I-e_y, I+e_z, I-e_z  (index 0, 1+2a, 2+2a)
    int o[7];
    o[0] = ii + rb.r0;
    o[1] = ip + rb.r0;
    o[2] = im + rb.r0;
    o[3] = ii + rb.ryp;
    o[4] = ii + rb.rym;
    o[5] = ii + rb.rzp;
    o[6] = ii + rb.rzm;
    // I + e_m - e_c  (m != c)
    int mx[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
    mx[0][1] = ip + rb.rym;
    mx[1][0] = im + rb.ryp;
    if (DIM == 3) {
        mx[0][2] = ip + rb.rzm;
        mx[1][2] = ii + rb.rypzm;
        mx[2][0] = im + rb.rzp;
        mx[2][1] = ii + rb.rymzp;
    }
    constexpr int NO = 1 + 2 * DIM;
    double U[DIM][NO];
    double X[DIM][DIM];
#pragma unroll
    for (int m = 0; m < DIM; ++m) {
#pragma unroll
        for (int q = 0; q < NO; ++q) U[m][q] = ldg(A.u[m] + o[q]);
#pragma unroll
        for (int c = 0; c < DIM; ++c) X[m][c] = (c == m || !A.advection) ? 0.0 : ldg(A.u[m] + mx[m][c]);
    }
    double ps0 = 0.0, psm[3] = {0, 0, 0};
    if (!A.first) {
        ps0 = ldg(A.pstar + o[0]);
#pragma unroll
        for (int c = 0; c < DIM; ++c) psm[c] = ldg(A.pstar + o[2 + 2 * c]);
    }
    double Gv[3] = {0, 0, 0};
#pragma unroll
    for (int c = 0; c < DIM; ++c) Gv[c] = ldg(A.G[c] + o[0]);
    double Nv[3];
    s1_eval<DIM>(A, U, X, ps0, psm, Gv, d, Nv);
#pragma unroll
    for (int c = 0; c < DIM; ++c) A.nadv[c][o[0]] = Nv[c];
    if (A.divn) {
        // D.u^n from operands already in registers: the first psi pass
        // then reads one field instead of gathering u^n again for Step 3f's chi term
        double dv = 0.0;
#pragma unroll
        for (int c = 0; c < DIM; ++c) dv += U[c][1 + 2 * c] - U[c][0];
        A.divn[o[0]] = dv * A.invh;
    }
}

// -------------------------------------------------------------------------------
// The line-pass kernel.  AX: line axis (0 = x, rows of R consecutive j at fixed k;
// 1 = y / 2 = z, R consecutive i at fixed k / j).  NC tiles are staged (NC = DIM for
// S1, else 1 with the component in blockIdx.z).
// -------------------------------------------------------------------------------
enum Kind { K_S1 = 0, K_MID = 1, K_LAST = 2, K_DIVPSI = 3, K_PSI_LAST = 4, K_USER = 5 };

struct LArgs {
    S1Args s1;
    double* io[3];          // MID/USER: in-place data; LAST: increments in, u^{n+1} out; DIVPSI: psi out
    const double* un[3];    // LAST, DIVPSI: u^n
    const double* unew[3];  // DIVPSI: u^{n+1}
    const double* divn;     // DIVPSI: D.u^n written by S1 (else gathered from u^n)
    double* p;              // DIVPSI: p -> q ; PSI_LAST: q -> p^{n+1/2}
    double* pstar;          // PSI_LAST: psi in, p* out
    double neg_rho_dt, chimu_half, invh;
    int nl;                 // local planes of the last axis (N, or the slab depth)
    int wrap;               // 1: the last axis is periodic here; 0: z-slab with halo planes
    int s1flat;             // S1 fill flattened over the tile's cells when n >= threads
    int mfwarp;             // k_strided: mean-correction line sums by warp partials (IBGM_MFWARP=0: off)
};

// Visit every (line l, position m) of a tile with coalesced global offsets: consecutive
// threads take consecutive x.  t / T: this thread's index among the T threads that
// share the work.  f(l, m, q) with q the 32-bit flat index.
// nrow bounds the rows of an x-line tile (the local planes of the last axis in 2D).
template <int AX, class F>
__device__ __forceinline__ void for_tile(int n, int nrow, int R, int g0, unsigned tb, int t, int T, F&& f)
{
    const unsigned N = (unsigned)n;
    if (AX == 0) {
        if (n >= T) {
            for (int l = 0; l < R; ++l) {
                if (g0 + l >= nrow) break;
                const unsigned rb = N * (unsigned)(g0 + l) + N * N * tb;
                for (int m = t; m < n; m += T) f(l, m, rb + (unsigned)m);
            }
        } else {
            const int rows = T / n;          // rows covered per sweep of the threads
            const int l0 = t / n, m = t - l0 * n;
            if (l0 >= rows) return;
            for (int l = l0; l < R && g0 + l < nrow; l += rows) f(l, m, (unsigned)m + N * (unsigned)(g0 + l) + N * N * tb);
        }
    } else {
        const int lg = 31 - __clz(R);        // R is a power of two
        const int l = t & (R - 1);
        if (g0 + l >= n) return;
        const int mstep = T >> lg;
        const unsigned S = (AX == 1) ? N : N * N;
        const unsigned base = (unsigned)(g0 + l) + ((AX == 1) ? N * N * tb : N * tb);
        for (int m = t >> lg; m < n; m += mstep) f(l, m, base + S * (unsigned)m);
    }
}

template <int L, int KIND, int DIM, int AX, int NC>
struct LinePass {
    // fill a tile (and tile2) for lines g0 .. g0+R-1 of slice tb (component comp)
    static __device__ __forceinline__ void fill(double* tile, double* tile2, const LArgs& A, int n, int R, int TP,
                                                int g0, unsigned tb, int comp, int t, int T)
    {
        const unsigned RTP = (unsigned)R * TP;
        const int nrow = (DIM == 2) ? A.nl : n;
        if (KIND == K_S1) {
            if (n >= T && A.s1flat == 1) {
                // the tile's R x n cells flattened over the threads (n = 384 on 256 threads:
                // 12 cells each instead of two rounds per row with half the threads idle)
                const int lmax = min(R, nrow - g0);
                const int tot = lmax * n;
                for (int e = t; e < tot; e += T) {
                    const int l = e / n, m = e - l * n;
                    const int ep = e + IBGM_PF_DIST * T;
                    if (ep < tot) {
                        const int lp = ep / n;
                        s1_prefetch<DIM>(A.s1, ep - lp * n, row_bases<DIM>(g0 + lp, (int)tb, n, A.nl, A.wrap));
                    }
                    const RowB rb = row_bases<DIM>(g0 + l, (int)tb, n, A.nl, A.wrap);
                    double v[3];
                    s1_cell<DIM>(A.s1, m, rb, n, v);
                    const int off = tile_off<L>(l, m, TP);
#pragma unroll
                    for (int c = 0; c < NC; ++c) tile[c * RTP + off] = v[c];
                }
            } else if (n >= T) {
                for (int l = 0; l < R && g0 + l < nrow; ++l) {
                    const RowB rb = row_bases<DIM>(g0 + l, (int)tb, n, A.nl, A.wrap);
                    if (l + IBGM_PF_ROWS < R && g0 + l + IBGM_PF_ROWS < nrow) {
                        const RowB rn = row_bases<DIM>(g0 + l + IBGM_PF_ROWS, (int)tb, n, A.nl, A.wrap);
                        for (int m = t; m < n; m += T) s1_prefetch<DIM>(A.s1, m, rn);
                    }
                    for (int m = t; m < n; m += T) {
                        // (a warp-owned row, A.s1flat == 2: prefetch this row two steps ahead)
                        if (A.s1flat == 2 && m + IBGM_PF_DIST * T < n) s1_prefetch<DIM>(A.s1, m + IBGM_PF_DIST * T, rb);
                        double v[3];
                        s1_cell<DIM>(A.s1, m, rb, n, v);
                        const int off = tile_off<L>(l, m, TP);
#pragma unroll
                        for (int c = 0; c < NC; ++c) tile[c * RTP + off] = v[c];
                    }
                }
            } else {
                const int rows = T / n;
                const int l0 = t / n, m = t - l0 * n;
                if (l0 < rows)
                    for (int l = l0; l < R && g0 + l < nrow; l += rows) {
                        const RowB rb = row_bases<DIM>(g0 + l, (int)tb, n, A.nl, A.wrap);
                        if (l + IBGM_PF_DIST * rows < R && g0 + l + IBGM_PF_DIST * rows < nrow)
                            s1_prefetch<DIM>(A.s1, m,
                                             row_bases<DIM>(g0 + l + IBGM_PF_DIST * rows, (int)tb, n, A.nl, A.wrap));
                        double v[3];
                        s1_cell<DIM>(A.s1, m, rb, n, v);
                        const int off = tile_off<L>(l, m, TP);
#pragma unroll
                        for (int c = 0; c < NC; ++c) tile[c * RTP + off] = v[c];
                    }
            }
        } else if (KIND == K_DIVPSI && AX != 0 && IBGM_DIV_CHUNK) {
            if (A.divn) {
                div_fill_chunk(tile, A, n, R, TP, g0, tb, t, T);
                return;
            }
            div_fill_gather(tile, A, n, nrow, R, TP, g0, tb, t, T);
        } else if (KIND == K_DIVPSI) {
            div_fill_gather(tile, A, n, nrow, R, TP, g0, tb, t, T);
        } else {
            // pure copies: cp.async keeps every load of the tile in flight at once
            issue(tile, tile2, A, n, R, TP, g0, tb, comp, t, T);
            cp_async_wait_all();
        }
    }

    // The first psi pass's fill with D.u^n from S1 (A.divn): each thread walks a contiguous
    // chunk of its line, so u^{n+1}_AX(I + e_AX) of one cell is u^{n+1}_AX(I) of the next,
    // and the operands of cell m+1 are loaded before cell m is evaluated and p stored
    // (two cells in flight per thread: the fill was bound by one load latency per cell).
    static __device__ __forceinline__ void div_fill_chunk(double* tile, const LArgs& A, int n, int R, int TP, int g0,
                                                          unsigned tb, int t, int T)
    {
        const unsigned N = (unsigned)n;
        const unsigned stp[3] = {1u, N, N * N};
        const int lg = 31 - __clz(R);
        const int l = t & (R - 1);
        if (g0 + l >= n) return;
        const int nthr = T >> lg;                       // threads per line
        const int chunk = (n + nthr - 1) / nthr;
        const int mb = (t >> lg) * chunk, me = min(n, mb + chunk);
        if (mb >= me) return;
        const unsigned S = stp[AX];
        const unsigned base = (unsigned)(g0 + l) + ((AX == 1) ? N * N * tb : N * tb);
        int ijk[3];
        ijk[0] = g0 + l;
        ijk[1] = (AX == 1) ? 0 : (int)tb;
        ijk[2] = (AX == 2) ? 0 : (int)tb;
        // operands of one cell: u_c^{n+1}(I + e_c), u_c^{n+1}(I) for c != AX, u_AX^{n+1}(I + e_AX),
        // D.u^n, p
        struct Ops {
            double up[3], u0[3], dv, pp;
        };
        auto load = [&](int m, Ops& o) {
            const unsigned q = base + S * (unsigned)m;
#pragma unroll
            for (int c = 0; c < DIM; ++c) {
                const int ic = (c == AX) ? m : ijk[c];
                const unsigned qp = (ic == n - 1) ? q - (N - 1) * stp[c] : q + stp[c];
                o.up[c] = ldg(A.unew[c] + qp);
                o.u0[c] = (c == AX) ? 0.0 : ldg(A.unew[c] + q);
            }
            o.dv = ldg(A.divn + q);
            o.pp = A.p[q];
        };
        double zc = ldg(A.unew[AX] + base + S * (unsigned)mb);
        Ops cur, nxt;
        load(mb, cur);
        for (int m = mb; m < me; ++m) {
            if (m + 1 < me) load(m + 1, nxt);
            double dn = cur.up[AX] - zc;
#pragma unroll
            for (int c = 0; c < DIM; ++c)
                if (c != AX) dn += cur.up[c] - cur.u0[c];
            dn *= A.invh;
            const unsigned q = base + S * (unsigned)m;
            tile[tile_off<L>(l, m, TP)] = A.neg_rho_dt * dn;               // Step 3e RHS
            A.p[q] = cur.pp - A.chimu_half * (dn + cur.dv);                 // Step 3f, explicit part
            zc = cur.up[AX];
            cur = nxt;
        }
    }

    // The first psi pass's fill, D.u^{n+1} and D.u^n gathered at every cell
    static __device__ __forceinline__ void div_fill_gather(double* tile, const LArgs& A, int n, int nrow, int R,
                                                           int TP, int g0, unsigned tb, int t, int T)
    {
        const unsigned N = (unsigned)n;
        {
            const unsigned stp[3] = {1u, N, N * N};
            const int mstep = (AX == 0) ? 0 : (T >> (31 - __clz(R)));   // this thread's next position
            for_tile<AX>(n, nrow, R, g0, tb, t, T, [&](int l, int m, unsigned q) {
                // measured: config 3 0.1981 -> 0.1956 ms/step, config 4 5.70 -> 5.97 (so N <= 128)
                if (IBGM_PF_DIV && AX != 0 && n <= 128 && m + mstep < n) {
                    const unsigned qn = q + stp[AX] * (unsigned)mstep;
#pragma unroll
                    for (int c = 0; c < DIM; ++c) {
                        pf_l2(A.unew[c] + qn);
                        pf_l2(A.un[c] + qn);
                    }
                    pf_l2(A.p + qn);
                }
                // cell coordinates along each axis: i = g0 + l; the line axis coordinate is m
                int ijk[3];
                ijk[0] = g0 + l;
                if (AX == 1) { ijk[1] = m; ijk[2] = (int)tb; } else { ijk[1] = (int)tb; ijk[2] = m; }
                double dn = 0.0, dol = 0.0;
                if (A.divn) {
#pragma unroll
                    for (int c = 0; c < DIM; ++c) {
                        const unsigned qp = (ijk[c] == n - 1) ? q - (N - 1) * stp[c] : q + stp[c];
                        dn += ldg(A.unew[c] + qp) - ldg(A.unew[c] + q);
                    }
                    dn *= A.invh;
                    dol = ldg(A.divn + q);
                } else {
#pragma unroll
                    for (int c = 0; c < DIM; ++c) {
                        const unsigned qp = (ijk[c] == n - 1) ? q - (N - 1) * stp[c] : q + stp[c];
                        dn += ldg(A.unew[c] + qp) - ldg(A.unew[c] + q);
                        dol += ldg(A.un[c] + qp) - ldg(A.un[c] + q);
                    }
                    dn *= A.invh;
                    dol *= A.invh;
                }
                tile[tile_off<L>(l, m, TP)] = A.neg_rho_dt * dn;         // Step 3e RHS
                A.p[q] = A.p[q] - A.chimu_half * (dn + dol);             // Step 3f, explicit part
            });
        }
    }

    // copy kinds: start the cp.async loads of a tile (the caller commits and waits)
    static __device__ __forceinline__ void issue(double* tile, double* tile2, const LArgs& A, int n, int R, int TP,
                                                 int g0, unsigned tb, int comp, int t, int T)
    {
        const int nrow = (DIM == 2) ? A.nl : n;
        const double* src = (KIND == K_PSI_LAST) ? A.pstar : pick3<double*>(A.io[0], A.io[1], A.io[2], comp);
        const double* src2 = (KIND == K_LAST) ? pick3<const double*>(A.un[0], A.un[1], A.un[2], comp)
                                              : (KIND == K_PSI_LAST ? A.p : nullptr);
        for_tile<AX>(n, nrow, R, g0, tb, t, T, [&](int l, int m, unsigned q) {
            const int off = tile_off<L>(l, m, TP);
            cp_async8(tile + off, src + q);
            if (KIND == K_LAST || KIND == K_PSI_LAST) cp_async8(tile2 + off, src2 + q);
        });
    }

    // warp-synchronous solve of the tile's R lines (P lanes per line); w / nw: this
    // warp's index among the nw warps that share the work
    static __device__ __forceinline__ void solve(double* tile, const LineCoef& C, const double* sinvT, int R, int TP,
                                                 int w, int nw)
    {
        const int P = C.P;
        const unsigned RTP = (unsigned)R * TP;
        const int lane = threadIdx.x & 31;
        if constexpr (L > kMaxL) {
            // long segments: P = 32 lanes = one line per warp, solved in place in the tile
            for (int l = w; l < R; l += nw)
#pragma unroll 1
                for (int c = 0; c < NC; ++c)
                    ws_solve_smem<L, schur_modes(KIND)>(tile + c * RTP + l * TP + lane * (L + 1), C, lane, P, 0, sinvT);
            return;
        }
        const int lpw = (P <= 32) ? 32 / P : 1;          // lines per warp per round
        const int sub = lane / P;
        const int s = lane - sub * P;
        const int gbase = sub * P;
        for (int lb = w * lpw; lb < R; lb += nw * lpw) {
            const int l = lb + sub;
            const bool ok = (sub < lpw) && (l < R);
            const int lc = ok ? l : lb;
#pragma unroll
            for (int c = 0; c < NC; ++c) {
                double* tl = tile + c * RTP + lc * TP + s * (L + 1);
                double x[L];
#pragma unroll
                for (int i = 0; i < L; ++i) x[i] = tl[i];
                ws_solve<L, schur_modes(KIND)>(x, C, s, P, gbase, sinvT);
                if (ok) {
#pragma unroll
                    for (int i = 0; i < L; ++i) tl[i] = x[i];
                }
            }
        }
    }

    // coalesced store of the solved tile (with the pass's epilogue)
    static __device__ __forceinline__ void store(const double* tile, const double* tile2, const LArgs& A, int n, int R,
                                                 int TP, int g0, unsigned tb, int comp, int t, int T)
    {
        const unsigned RTP = (unsigned)R * TP;
        const int nrow = (DIM == 2) ? A.nl : n;
        if (KIND == K_S1) {
            for_tile<AX>(n, nrow, R, g0, tb, t, T, [&](int l, int m, unsigned q) {
                const int off = tile_off<L>(l, m, TP);
#pragma unroll
                for (int c = 0; c < NC; ++c) A.s1.out[c][q] = tile[c * RTP + off];
            });
        } else {
            double* dst = (KIND == K_PSI_LAST) ? A.pstar : pick3<double*>(A.io[0], A.io[1], A.io[2], comp);
            for_tile<AX>(n, nrow, R, g0, tb, t, T, [&](int l, int m, unsigned q) {
                const int off = tile_off<L>(l, m, TP);
                if (KIND == K_LAST) {
                    dst[q] = tile2[off] + tile[off];            // u^{n+1} = u^n + d
                } else if (KIND == K_PSI_LAST) {
                    const double psi = tile[off];
                    const double pn = tile2[off] + psi;        // Step 3f: p^{n+1/2} = q + psi^{n+1/2}
                    A.p[q] = pn;
                    dst[q] = pn + psi;                         // Step 3a of the next step: p* = p + psi
                } else {
                    dst[q] = tile[off];
                }
            });
        }
    }
};

// doubles of shared memory the staged S^{-1} takes: none when the pass applies the
// line's S^{-1} in banded or circulant form (the freed space admits more blocks per SM)
template <int MODES>
__host__ __device__ __forceinline__ int sinv_slots(const LineCoef& C)
{
    return (((MODES & kSchurBand) && C.band >= 0) || ((MODES & kSchurCirc) && C.circ)) ? 0 : C.P * C.P;
}

template <int MODES>
__device__ __forceinline__ void load_sinvT(double* sinvT, const SchurInv* SI, const LineCoef& C)
{
    if (sinv_slots<MODES>(C) == 0) return;
    const int P = C.P;
    for (int e = threadIdx.x; e < P * P; e += blockDim.x) sinvT[e] = SI->sinvT[e];
}

// One tile per block, all threads in every phase (short grids; ib_line_solve).
template <int L, int KIND, int DIM, int AX, int NC, int MINB>
__global__ void __launch_bounds__(256, MINB) k_lines(const LineCoef C, const SchurInv* __restrict__ SI, int n, int R,
                                                     LArgs A)
{
    using LP = LinePass<L, KIND, DIM, AX, NC>;
    extern __shared__ double smem[];
    const int P = C.P;
    const int TP = tile_pitch(P, L);
    double* sinvT = smem;
    double* tile = smem + sinv_slots<schur_modes(KIND)>(C);
    double* tile2 = tile + (size_t)NC * R * TP;   // LAST: u^n, PSI_LAST: q (prefetched with the fill)
    load_sinvT<schur_modes(KIND)>(sinvT, SI, C);                     // line factors: not written by the predecessor
    pdl_wait();
    pdl_trigger();
    const int comp = (NC == 1) ? blockIdx.z : 0;
    const int g0 = blockIdx.x * R;
    const unsigned tb = blockIdx.y;
    LP::fill(tile, tile2, A, n, R, TP, g0, tb, comp, threadIdx.x, blockDim.x);
    __syncthreads();
    LP::solve(tile, C, sinvT, R, TP, threadIdx.x >> 5, blockDim.x >> 5);
    __syncthreads();
    LP::store(tile, tile2, A, n, R, TP, g0, tb, comp, threadIdx.x, blockDim.x);
}

// -------------------------------------------------------------------------------
// Warp-independent x-line pass (S1, psi_x + Step 3f): every warp owns lpw = 32/P whole
// x-lines in its own slice of shared memory and runs fill -> solve -> store with only
// warp barriers, so the warps of an SM drift into different phases and the stencil
// gathers of some overlap the register-resident solves of others (k_lines orders the
// three phases of all its warps with block barriers: the memory system idles while
// the whole block solves).
// -------------------------------------------------------------------------------
template <int L, int KIND, int DIM, int NC, int WPB, int MINB>
__global__ void __launch_bounds__(32 * WPB, MINB) k_xwarp(const LineCoef C, const SchurInv* __restrict__ SI, int n,
                                                          LArgs A)
{
    using LP = LinePass<L, KIND, DIM, 0, NC>;
    extern __shared__ double smem[];
    const int P = C.P;
    const int TP = tile_pitch(P, L);
    const int lpw = 32 / P;
    constexpr int NT = (KIND == K_PSI_LAST) ? 2 : 1;
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double* sinvT = smem;
    double* tile = smem + sinv_slots<schur_modes(KIND)>(C) + (size_t)w * NT * NC * lpw * TP;
    double* tile2 = tile + (size_t)NC * lpw * TP;
    load_sinvT<schur_modes(KIND)>(sinvT, SI, C);
    __syncthreads();
    const int g0 = (blockIdx.x * WPB + w) * lpw;
    const int nrow = (DIM == 2) ? A.nl : n;
    if (g0 >= nrow) return;
    LP::fill(tile, tile2, A, n, lpw, TP, g0, blockIdx.y, 0, lane, 32);
    __syncwarp();
    LP::solve(tile, C, sinvT, lpw, TP, 0, 1);
    __syncwarp();
    LP::store(tile, tile2, A, n, lpw, TP, g0, blockIdx.y, 0, lane, 32);
}

// -------------------------------------------------------------------------------
// Strided-line pass (y / z lines, and y in 2D): one thread per (line, part).  A block
// holds RI neighbouring lines (consecutive i) x P parts; warp w covers RI lines of one
// part, so each of a thread's L loads is one coalesced RI-wide row.  The part stays in
// registers: Thomas on its interior, the interface values and the
// reduced right-hand side go through a small shared array (4 barriers), y = S^{-1} r,
// correction and the exact line-mean correction (R16) -- the
// arithmetic of ws_solve with shared memory in place of the lane shuffles, and no
// staged tile.
// -------------------------------------------------------------------------------
// minimum blocks of 512 threads per SM (register cap 64 / 40) for the passes whose parts
// fit; 0 leaves the choice to ptxas (the divergence pass and long parts take up to 128)
__host__ __device__ constexpr int strided_minb(int l, int kind)
{
    return (kind == K_DIVPSI && l <= 16)
               ? 1   // (all 128 registers: ptxas otherwise stops at 106 and sinks five of the fill's loads below the first store)
               : ((kind == K_MID && l <= 8) ? 3 : (((kind == K_MID && l <= 16) || (kind == K_LAST && l <= 12)) ? 2 : 0));
}

template <int L, int KIND, int DIM, int AX>
__global__ void __launch_bounds__(512, strided_minb(L, KIND)) k_strided(const LineCoef C, const SchurInv* __restrict__ SI, int n, int RI,
                                                 LArgs A)
{
    static_assert(AX != 0, "x lines use the tiled pass");
    constexpr int M = L - 1;
    extern __shared__ double smem[];
    const int P = C.P;
    double* sinvT = smem;
    double* xl = sinvT + sinv_slots<schur_modes(KIND)>(C);   // [P][RI] last interior value f*_{s,m}
    double* yb = xl + P * RI;            // [P][RI] y_s
    double* ds = yb + P * RI;            // [P][RI] line sums of d (mean correction)
    double* xs = ds + P * RI;            // [P][RI] line sums of x
    double* rr = xs + P * RI;            // [P][RI] reduced right-hand side r_s, every four parts
                                         // shifted by 8 doubles (rr_at; P RI + 2 P doubles)
    // (only the kinds that can take the tiled dense circulant form shift r; the last
    //  viscous sweep keeps the plain [P][RI] indexing and none of the warp-sum code)
    constexpr bool kTile = (schur_modes(KIND) & kSchurCirc) != 0;
    auto rr_at = [RI](int q, int l) { return kTile ? q * RI + l + ((q >> 2) << 3) : q * RI + l; };
    load_sinvT<schur_modes(KIND)>(sinvT, SI, C);
    const int il = threadIdx.x % RI, s = threadIdx.x / RI;
    const int i = blockIdx.x * RI + il;
    const int comp = (KIND == K_DIVPSI) ? 0 : blockIdx.z;
    const unsigned N = (unsigned)n;
    const unsigned S = (AX == 1) ? N : N * N;                     // stride along the line
    const unsigned base = (unsigned)i + ((AX == 1) ? ((DIM == 3) ? N * N * blockIdx.y : 0u) : N * blockIdx.y);
    const unsigned q0 = base + S * (unsigned)(s * L);
    double x[L];
    double un[L];
    if (KIND == K_DIVPSI && A.divn) {
        // D.u^{n+1} at the part's cells with D.u^n from S1: u_AX^{n+1}(I + e_AX) of one cell
        // is u_AX^{n+1}(I) of the next; every load of the part before the first p store
        const unsigned stp[3] = {1u, N, N * N};
        double pq[L];
        double zc = ldg(pick3<const double*>(A.unew[0], A.unew[1], A.unew[2], AX) + q0);
#pragma unroll
        for (int j = 0; j < L; ++j) {
            const unsigned q = q0 + S * (unsigned)j;
            int ijk[3];
            ijk[0] = i;
            if (AX == 1) { ijk[1] = s * L + j; ijk[2] = 0; } else { ijk[1] = (int)blockIdx.y; ijk[2] = s * L + j; }
            double dn = 0.0;
#pragma unroll
            for (int c = 0; c < DIM; ++c) {
                const unsigned qp = (ijk[c] == n - 1) ? q - (N - 1) * stp[c] : q + stp[c];
                const double* unw = pick3<const double*>(A.unew[0], A.unew[1], A.unew[2], c);
                const double up = ldg(unw + qp);
                if (c == AX) {
                    dn += up - zc;
                    zc = up;
                } else {
                    dn += up - ldg(unw + q);
                }
            }
            dn *= A.invh;
            x[j] = A.neg_rho_dt * dn;
            pq[j] = A.p[q] - A.chimu_half * (dn + ldg(A.divn + q));
        }
#pragma unroll
        for (int j = 0; j < L; ++j) A.p[q0 + S * (unsigned)j] = pq[j];
    } else if (KIND == K_DIVPSI) {
        // D.u^{n+1} and D.u^n at the part's cells; Step 3e RHS and the
        // explicit part of Step 3f
        const unsigned stp[3] = {1u, N, N * N};
#pragma unroll
        for (int j = 0; j < L; ++j) {
            const unsigned q = q0 + S * (unsigned)j;
            int ijk[3];
            ijk[0] = i;
            if (AX == 1) { ijk[1] = s * L + j; ijk[2] = 0; } else { ijk[1] = (int)blockIdx.y; ijk[2] = s * L + j; }
            double dn = 0.0, dol = 0.0;
#pragma unroll
            for (int c = 0; c < DIM; ++c) {
                const unsigned qp = (ijk[c] == n - 1) ? q - (N - 1) * stp[c] : q + stp[c];
                const double* unw = pick3<const double*>(A.unew[0], A.unew[1], A.unew[2], c);
                const double* uo = pick3<const double*>(A.un[0], A.un[1], A.un[2], c);
                dn += ldg(unw + qp) - ldg(unw + q);
                dol += ldg(uo + qp) - ldg(uo + q);
            }
            dn *= A.invh;
            dol *= A.invh;
            x[j] = A.neg_rho_dt * dn;
            A.p[q] = A.p[q] - A.chimu_half * (dn + dol);
        }
    } else {
        const double* src = pick3<double*>(A.io[0], A.io[1], A.io[2], comp);
#pragma unroll
        for (int j = 0; j < L; ++j) x[j] = ldg(src + q0 + S * (unsigned)j);
        if (KIND == K_LAST && L <= 16) {    // (longer parts load u^n in the epilogue)
            const double* u0 = pick3<const double*>(A.un[0], A.un[1], A.un[2], comp);
#pragma unroll
            for (int j = 0; j < L; ++j) un[j] = ldg(u0 + q0 + S * (unsigned)j);
        }
    }
    const double c = C.c, b = C.b;
    const bool mf = C.mean_fix != 0;
    double dsum = 0.0;
    if (mf) {
#pragma unroll
        for (int j = 0; j < L; ++j) dsum += x[j];
    }
    x[1] *= C.inv[0];
#pragma unroll
    for (int j = 2; j <= M; ++j) x[j] = (x[j] - c * x[j - 1]) * C.inv[j - 1];
#pragma unroll
    for (int j = M - 1; j >= 1; --j) x[j] -= C.cp[j - 1] * x[j + 1];
    const int sp = (s == 0) ? P - 1 : s - 1, sn = (s == P - 1) ? 0 : s + 1;
    xl[s * RI + il] = x[M];
    // line sums for the mean correction: a warp holds 32 / RI consecutive parts of its RI
    // lines (lane = (s mod 32/RI) RI + il), so it sums them by shuffles and stores one
    // partial per (warp, line); each thread then adds P RI / 32 partials instead of P
    // (psi_y at config 4: 64 -> 16 shared loads per thread; IBGM_MFWARP=0 for A/B)
    const bool wsum = kTile && mf && A.mfwarp && RI <= 32 && (32 % RI) == 0 && ((P * RI) & 31) == 0;
    const int wq = threadIdx.x >> 5, nwq = (P * RI) >> 5;
    const bool wlead = (threadIdx.x & 31) < RI;
    if (wsum) {
        for (int off = RI; off < 32; off <<= 1) dsum += __shfl_xor_sync(0xffffffffu, dsum, off);
        if (wlead) ds[wq * RI + il] = dsum;
    } else if (mf) {
        ds[s * RI + il] = dsum;
    }
    __syncthreads();
    rr[rr_at(s, il)] = x[0] - c * xl[sp * RI + il] - b * x[1];
    __syncthreads();
    double ys = 0.0;
    constexpr int MODES = schur_modes(KIND);
    const bool banded = (MODES & kSchurBand) && C.band >= 0;   // (takes precedence: 2 band + 1 taps)
    if (!banded && (MODES & kSchurCirc) && C.circ && P == kMaxSeg && A.mfwarp >= 2) {
        // dense circulant S^{-1} at P = 32, register-tiled: the first P/4 RI threads form
        // four consecutive outputs each from 35 loads of r (y_{s0+j} = sum_d wf[d] r_{s0+j+d},
        // d ascending as below: the same sums), instead of 32 loads per output in every thread
        if ((int)threadIdx.x < (kMaxSeg / 4) * RI) {
            const int s0 = 4 * s;                     // this thread's (il, s) as output group s
            double y0 = 0.0, y1 = 0.0, y2 = 0.0, y3 = 0.0;
#pragma unroll
            for (int k = 0; k < kMaxSeg + 3; ++k) {
                const int q = (s0 + k >= kMaxSeg) ? s0 + k - kMaxSeg : s0 + k;
                const double r = rr[rr_at(q, il)];
                if (k < kMaxSeg) y0 = fma(C.wf[k], r, y0);
                if (k >= 1 && k - 1 < kMaxSeg) y1 = fma(C.wf[k >= 1 ? k - 1 : 0], r, y1);
                if (k >= 2 && k - 2 < kMaxSeg) y2 = fma(C.wf[k >= 2 ? k - 2 : 0], r, y2);
                if (k >= 3) y3 = fma(C.wf[k >= 3 ? k - 3 : 0], r, y3);
            }
            yb[(s0 + 0) * RI + il] = y0;
            yb[(s0 + 1) * RI + il] = y1;
            yb[(s0 + 2) * RI + il] = y2;
            yb[(s0 + 3) * RI + il] = y3;
        }
        __syncthreads();
        ys = yb[s * RI + il];
    } else {
        if (banded) {
            // banded circulant S^{-1} (LineCoef::band)
            ys = C.w[kMaxBand] * rr[rr_at(s, il)];
#pragma unroll
            for (int d = 1; d <= kMaxBand; ++d) {
                if (d > C.band) break;
                const int qp = (s + d >= P) ? s + d - P : s + d, qm = (s - d < 0) ? s - d + P : s - d;
                ys = fma(C.w[kMaxBand + d], rr[rr_at(qp, il)], ys);
                ys = fma(C.w[kMaxBand - d], rr[rr_at(qm, il)], ys);
            }
        } else if ((MODES & kSchurCirc) && C.circ) {
#pragma unroll
            for (int d = 0; d < kMaxSeg; ++d) {
                if (d >= P) break;
                const int q = (s + d >= P) ? s + d - P : s + d;
                ys = fma(C.wf[d], rr[rr_at(q, il)], ys);
            }
        } else {
            for (int q = 0; q < P; ++q) ys = fma(sinvT[q * P + s], rr[rr_at(q, il)], ys);
        }
        yb[s * RI + il] = ys;
        __syncthreads();
    }
    const double ys1 = yb[sn * RI + il];
    x[0] = ys;
    const double cy = c * ys, by = b * ys1;
#pragma unroll
    for (int j = 1; j <= M; ++j) x[j] -= cy * C.g[j - 1] + by * C.h[j - 1];
    if (mf) {
        double t = 0.0;
#pragma unroll
        for (int j = 0; j < L; ++j) t += x[j];
        if (wsum) {
            for (int off = RI; off < 32; off <<= 1) t += __shfl_xor_sync(0xffffffffu, t, off);
            if (wlead) xs[wq * RI + il] = t;
        } else {
            xs[s * RI + il] = t;
        }
        __syncthreads();
        double D = 0.0, X = 0.0;
        const int nq = wsum ? nwq : P;
        for (int q = 0; q < nq; ++q) {
            D += ds[q * RI + il];
            X += xs[q * RI + il];
        }
        const double corr = (D * C.inv_rowsum - X) * C.inv_n;
#pragma unroll
        for (int j = 0; j < L; ++j) x[j] += corr;
    }
    double* dst = (KIND == K_DIVPSI) ? A.io[0] : pick3<double*>(A.io[0], A.io[1], A.io[2], comp);
#pragma unroll
    for (int j = 0; j < L; ++j) {
        const unsigned q = q0 + S * (unsigned)j;
        if (KIND == K_LAST)                                     // u^{n+1} = u^n + delta (R23)
            dst[q] = (L <= 16 ? un[j] : ldg(pick3<const double*>(A.un[0], A.un[1], A.un[2], comp) + q)) + x[j];
        else dst[q] = x[j];
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

static size_t lines_smem(int P, int L, int nc, int R) { return ((size_t)P * P + (size_t)nc * R * tile_pitch(P, L)) * 8; }
static int tiles_of(int kind, int nc) { return (kind == K_LAST || kind == K_PSI_LAST) ? 2 * nc : nc; }

// lines per block: the largest of {32, 16, 8} whose tile keeps >= 2 blocks per SM
bool pdl_enabled()
{
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("IBGM_PDL");
        v = (e && atoi(e) == 0) ? 0 : 1;
    }
    return v == 1;
}

// x-line passes by k_xwarp (IBGM_XWARP=0: the block-tiled k_lines pass, for A/B)
static bool xwarp_enabled()
{
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("IBGM_XWARP");
        v = (e && atoi(e) == 0) ? 0 : 1;
    }
    return v == 1;
}

static int sm_count()
{
    static int n = 0;
    if (!n) {
        int dev = 0;
        cudaGetDevice(&dev);
        if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n < 1) n = 148;
    }
    return n;
}

// lines per block R (a power of two): the largest whose tile fits (<= 100 KB for R >= 8,
// i.e. >= 2 blocks per SM) and that still gives the grid >= minblk blocks: one per SM in
// 2D, four per SM in 3D.  Measured (graph-mode ms/step): config 1 (256^2, 256 lines per
// pass) 0.056 -> 0.025 (R 32/16 -> 1; one block per SM beats a few large tiles), config 2
// 0.086 -> 0.076 (R 4), config 3 0.1974 -> 0.1959 (psi passes R 16), config 4 unchanged.
// y / z passes by k_strided (IBGM_STRIDED=0: the tiled k_lines pass, for A/B)
static bool strided_enabled()
{
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("IBGM_STRIDED");
        v = (e && atoi(e) == 0) ? 0 : 1;
    }
    return v == 1;
}

// the first psi pass strided when S1 supplies D.u^n: with five u^{n+1} loads per cell
// (u_z reused along the part) and every load of the part issued before the p stores, the
// register-resident layout beats the tile (config 4: 731 -> 658 us, 3.996 -> 3.927
// ms/step).  A/B switch: IBGM_DIV_STRIDED=0 (tiled, contiguous-chunk fill).
static bool div_strided_enabled()
{
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("IBGM_DIV_STRIDED");
        v = (e && atoi(e) == 0) ? 0 : 1;
    }
    return v == 1;
}

static int pick_r(const Ctx* s, int L, int nc, int64_t rows, int64_t other, int per_sm = 0)
{
    static int forced = -1, mb_env = -1;
    if (forced < 0) {
        const char* e = getenv("IBGM_R");
        forced = e ? atoi(e) : 0;
        e = getenv("IBGM_MINBLK");
        mb_env = e ? atoi(e) : 0;
    }
    if (forced >= 1 && forced <= 32 && (forced & (forced - 1)) == 0 &&
        lines_smem(s->P, L, nc, forced) <= (forced >= 8 ? 100 : 200) * 1024)
        return forced;
    const int64_t minblk = mb_env > 0 ? mb_env : (int64_t)sm_count() * (per_sm > 0 ? per_sm : (s->dim == 3 ? 4 : 1));
    int best = 0;
    for (int R = 32; R >= 1; R /= 2) {
        if (lines_smem(s->P, L, nc, R) > (R >= 8 ? 100 : 200) * 1024) continue;
        best = R;
        if ((rows + R - 1) / R * other >= minblk) return R;
    }
    return best ? best : 1;
}

template <int L, int KIND, int DIM, int AX, int NC, int MINB>
static cudaError_t go_lines_k(Ctx* s, int sys, const LArgs& la, int ncomp_grid, int64_t rows, int gy);

template <int L, int KIND, int DIM, int AX, int NC>
static cudaError_t go_lines(Ctx* s, int sys, const LArgs& a, int ncomp_grid)
{
    // a pass along the last axis needs the whole line on this GPU
    if (AX == DIM - 1 && !s->wrap) return cudaErrorInvalidValue;
    LArgs la = a;
    la.nl = (int)s->nl;
    la.wrap = s->wrap;
    {
        static int mw = -1;
        if (mw < 0) {
            const char* e = getenv("IBGM_MFWARP");
            mw = e ? atoi(e) : 2;   // 1: warp partial sums only, 2: + tiled dense circulant S^{-1}
        }
        la.mfwarp = mw;
    }
    {
        static int fl = -1;
        if (fl < 0) {
            const char* e = getenv("IBGM_S1FLAT");
            fl = (e && atoi(e) == 0) ? 0 : 1;
        }
        la.s1flat = fl;
    }
    // (the divergence pass gathering u^n stays tiled: strided it measured 35.3 -> 41.4 us
    //  at config 3, 995 -> 1335 us at config 4 -- twelve gathers per cell before the solve;
    //  with D.u^n from S1 it runs strided, see div_strided_enabled)
    if constexpr (AX != 0 && L <= 32 && (KIND == K_MID || KIND == K_LAST || KIND == K_DIVPSI)) {
        if (strided_enabled() && (KIND != K_DIVPSI || (la.divn && div_strided_enabled()))) {
            static int ri_env = -1;
            if (ri_env < 0) {
                const char* e = getenv("IBGM_RI");
                ri_env = e ? atoi(e) : 0;
            }
            // 256 threads per block: RI = 256 / P lines (measured: config 3 RI 16 0.1777 vs
            // 32 0.1818 ms/step; config 4 z sweep RI 8 771 vs 16 882 us); 512 for L = 32
            // (config 2 y sweep: RI 16 13.0 us, 8 14.8, 4 20.4; tiled 25.0)
            // round 2, banded S^{-1} (no staged S^{-1} left in shared memory): the z sweep
            // at P = 32 takes 512 threads, RI 16 (config 4: 750 -> 686 us; y passes 424 ->
            // 431, psi_y 232 -> 243 at RI 16, so they keep RI 8)
            const bool wide = ((KIND == K_LAST || KIND == K_DIVPSI) && AX == 2 && s->P >= 32);
            int RI = ri_env > 0 ? ri_env : std::max(8, std::min(32, (L > 16 || wide ? 512 : 256) / s->P));
            {
                // per-kind A/B override: IBGM_RI_K1 (y passes), IBGM_RI_K2 (last sweep), IBGM_RI_K3 (first psi pass)
                static int rk = -1;
                if (rk < 0) {
                    char nm[32];
                    snprintf(nm, sizeof(nm), "IBGM_RI_K%d", KIND);
                    const char* e = getenv(nm);
                    rk = e ? atoi(e) : 0;
                }
                if (rk > 0) RI = rk;
            }
            if (s->n % RI == 0 && s->P * RI <= 512) {
                auto kern = k_strided<L, KIND, DIM, AX>;
                const size_t sm = ((size_t)sinv_slots<schur_modes(KIND)>(s->hcoef[sys]) + 5 * (size_t)s->P * RI + 2 * (size_t)s->P) *
                                  sizeof(double);
                const int gy = (DIM == 3) ? (int)s->nl : 1;
                const dim3 grid((unsigned)(s->n / RI), (unsigned)gy, (unsigned)ncomp_grid);
                kern<<<grid, s->P * RI, sm, s->stream>>>(s->hcoef[sys], s->sinv + sys, (int)s->n, RI, la);
                s->launches++;
                return cudaGetLastError();
            }
        }
    }
    const int64_t rows = (AX == 0 && DIM == 2) ? s->nl : s->n;
    const int gy = (DIM == 3) ? (int)s->nl : 1;
    if constexpr (AX == 0 && L <= kMaxL && (KIND == K_S1 || KIND == K_PSI_LAST)) {
        // measured (graph ms/step): config 4 (384^3) 5.056 -> 4.957; config 3 (128^3) 0.1686 ->
        // 0.1724 and config 2 (1024^2) 0.066 -> 0.075 slower, so only 3D grids of N >= 256
        if (xwarp_enabled() && DIM == 3 && s->n >= 256 && s->P <= 32) {
            constexpr int WPB = (KIND == K_S1) ? IBGM_XWARP_WPB : 4;
            constexpr int MINB = (KIND == K_S1) ? IBGM_S1_MINB : 8;
            auto kern = k_xwarp<L, KIND, DIM, NC, WPB, MINB>;
            const int lpw = 32 / s->P;
            const int TP = tile_pitch(s->P, L);
            const int NT = (KIND == K_PSI_LAST) ? 2 : 1;
            const size_t sm = ((size_t)sinv_slots<schur_modes(KIND)>(s->hcoef[sys]) + (size_t)WPB * NT * NC * lpw * TP) *
                              sizeof(double);
            static unsigned long long attr_mask = 0;
            const cudaError_t ae = smem_attr_once(attr_mask, kern, (int)smem_limit());
            if (ae != cudaSuccess) return ae;
            {
                // IBGM_XFLAT=1: the flattened fill (row and cell from one index per cell)
                static int fl = -1;
                if (fl < 0) {
                    const char* e = getenv("IBGM_XFLAT");
                    fl = (e && atoi(e) == 1) ? 1 : 2;
                }
                la.s1flat = fl;
            }
            const dim3 grid((unsigned)((rows + WPB * lpw - 1) / (WPB * lpw)), (unsigned)gy, 1u);
            kern<<<grid, 32 * WPB, sm, s->stream>>>(s->hcoef[sys], s->sinv + sys, (int)s->n, la);
            s->launches++;
            return cudaGetLastError();
        }
    }
    return go_lines_k<L, KIND, DIM, AX, NC, (KIND == K_S1 || L >= 24) ? 2 : 4>(s, sys, la, ncomp_grid, rows, gy);
}

template <int L, int KIND, int DIM, int AX, int NC, int MINB>
static cudaError_t go_lines_k(Ctx* s, int sys, const LArgs& la, int ncomp_grid, int64_t rows, int gy)
{
    auto kern = k_lines<L, KIND, DIM, AX, NC, MINB>;
    // the divergence + first psi factor pass: two blocks per SM suffice in 3D (config 3:
    // R 32 31.4 us vs R 16 35.3 us, 0.1716 -> 0.1680 ms/step; config 4 keeps R 16 -- its
    // R 32 tile exceeds the 100 KB two-blocks-per-SM bound and measured 1261 vs 998 us)
    int R = pick_r(s, L, tiles_of(KIND, NC), rows, (int64_t)gy * ncomp_grid, (KIND == K_DIVPSI && DIM == 3) ? 2 : 0);
    {
        static int rk = -2;
        if (rk == -2) {
            char nm[32];
            snprintf(nm, sizeof(nm), "IBGM_R_K%d", KIND);
            const char* e = getenv(nm);
            rk = e ? atoi(e) : 0;
        }
        if (rk > 0 && lines_smem(s->P, L, tiles_of(KIND, NC), rk) <= 200 * 1024) R = rk;
    }
    // (the tiled passes keep the S^{-1} space in their allocation even when they do not
    //  stage it: trimmed, the divergence pass at config 4 runs 4 blocks per SM instead of 3
    //  and measured 723 -> 824 us; the strided and warp-owned passes gain from the trim:
    //  y sweep 416 -> 397 us, psi_x 341 -> 334 us)
    const size_t sm = lines_smem(s->P, L, tiles_of(KIND, NC), R);
    static unsigned long long attr_mask = 0;   // per instantiation, per device
    {
        const cudaError_t e = smem_attr_once(attr_mask, kern, (int)smem_limit());
        if (e != cudaSuccess) return e;
    }
    dim3 grid((unsigned)((rows + R - 1) / R), (unsigned)gy, (unsigned)ncomp_grid);
    // PDL on 2D grids only: measured config 2 0.0896 -> 0.0846 ms/step; on 3D the waiting
    // dependents hold SM slots that the look-ahead IB kernels need (config 3 +5%)
    const cudaError_t e = launch_pdl_if(DIM == 2, kern, grid, dim3(256), sm, s->stream, s->hcoef[sys], s->sinv + sys,
                                        (int)s->n, R, la);
    s->launches++;
    return e;
}

#define IBGM_DISPATCH_L2D(Lval, CALL)                    \
    switch (Lval) {                                      \
        case 64: { constexpr int LL = 64; return CALL; } \
        case 128: { constexpr int LL = 128; return CALL; } \
        default: IBGM_DISPATCH_L(Lval, CALL)              \
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

// one component per block (blockIdx.z), any axis
template <int KIND>
static cudaError_t go_axis(Ctx* s, int sys, int axis, const LArgs& a, int ncomp)
{
    if (s->dim == 3) {
        if (axis == 0) { IBGM_DISPATCH_L(s->L, (go_lines<LL, KIND, 3, 0, 1>(s, sys, a, ncomp))) }
        if (axis == 1) { IBGM_DISPATCH_L(s->L, (go_lines<LL, KIND, 3, 1, 1>(s, sys, a, ncomp))) }
        IBGM_DISPATCH_L(s->L, (go_lines<LL, KIND, 3, 2, 1>(s, sys, a, ncomp)))
    }
    if (axis == 0) { IBGM_DISPATCH_L2D(s->L, (go_lines<LL, KIND, 2, 0, 1>(s, sys, a, ncomp))) }
    IBGM_DISPATCH_L2D(s->L, (go_lines<LL, KIND, 2, 1, 1>(s, sys, a, ncomp)))
}

// S1 hands D.u^n to the first psi pass through the scratch field (on a slab: to the
// cut-axis forward phase, slab.cu).  Measured (graph ms/step, same box): config 4 4.361
// -> 4.275 (div+psi_z 1058 -> 935 us, S1 1312 -> 1373 us); config 3 0.1563 -> 0.1578,
// so 3D grids of N >= 256 only.  A/B switch: IBGM_DIVN=0 / 1 (force).
bool divn_fused(const Ctx* s)
{
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("IBGM_DIVN");
        v = e ? atoi(e) : 2;
    }
    if (v == 0 || s->tmp == nullptr) return false;
    return v == 1 || (s->dim == 3 && s->n >= 256);
}

cudaError_t launch_s1_x(Ctx* s, int first_step)
{
    LArgs a{};
    S1Args& b = a.s1;
    for (int c = 0; c < 3; ++c) {
        b.u[c] = s->u[c]; b.G[c] = s->nprev[c]; b.nadv[c] = s->nadv[c]; b.out[c] = s->st[c];
    }
    b.pstar = s->pstar;
    b.dt = s->dt; b.inv_rho = 1.0 / s->rho; b.mu = s->mu; b.invh = 1.0 / s->h;
    b.a1 = first_step ? 1.0 : 1.5;
    b.first = first_step; b.advection = s->advection;
    b.divn = divn_fused(s) ? s->tmp : nullptr;
    if (s->dim == 3) { IBGM_DISPATCH_L(s->L, (go_lines<LL, K_S1, 3, 0, 3>(s, SYS_VISC, a, 1))) }
    IBGM_DISPATCH_L2D(s->L, (go_lines<LL, K_S1, 2, 0, 2>(s, SYS_VISC, a, 1)))
}

cudaError_t launch_sweep_mid(Ctx* s, int axis)
{
    LArgs a{};
    for (int c = 0; c < 3; ++c) a.io[c] = s->st[c];
    return go_axis<K_MID>(s, SYS_VISC, axis, a, s->dim);
}

cudaError_t launch_sweep_last(Ctx* s, int axis)
{
    LArgs a{};
    for (int c = 0; c < 3; ++c) { a.io[c] = s->st[c]; a.un[c] = s->u[c]; }
    return go_axis<K_LAST>(s, SYS_VISC, axis, a, s->dim);
}

cudaError_t launch_div_psi_first(Ctx* s, int axis)
{
    LArgs a{};
    a.io[0] = a.io[1] = a.io[2] = s->pstar;
    for (int c = 0; c < 3; ++c) { a.un[c] = s->u[c]; a.unew[c] = s->st[c]; }
    a.p = s->p;
    a.divn = divn_fused(s) ? s->tmp : nullptr;
    a.neg_rho_dt = -s->rho / s->dt;
    a.chimu_half = 0.5 * s->chi * s->mu;
    a.invh = 1.0 / s->h;
    if (axis == 0) return cudaErrorInvalidValue;
    return go_axis<K_DIVPSI>(s, SYS_PSI, axis, a, 1);
}

cudaError_t launch_psi_mid(Ctx* s, int axis)
{
    LArgs a{};
    a.io[0] = a.io[1] = a.io[2] = s->pstar;
    return go_axis<K_MID>(s, SYS_PSI, axis, a, 1);
}

cudaError_t launch_psi_last_x(Ctx* s)
{
    LArgs a{};
    a.pstar = s->pstar;
    a.p = s->p;
    return go_axis<K_PSI_LAST>(s, SYS_PSI, 0, a, 1);
}

cudaError_t launch_line_solve(Ctx* s, int axis, int sys, double* data)
{
    LArgs a{};
    a.io[0] = a.io[1] = a.io[2] = data;
    return go_axis<K_USER>(s, sys, axis, a, 1);
}

cudaError_t launch_sub(Ctx* s, const double* a, const double* b, double* out)
{
    k_sub<<<592, 256, 0, s->stream>>>(a, b, out, (size_t)s->nlocal);
    s->launches++;
    return cudaGetLastError();
}

}  // namespace ibgm
