// Immersed-boundary kernels of the IB-GM step (sm_100a, fp64): Steps 1a-1c and 2a-2b
// of PAPER.md:577-621.  Lagrangian arrays are point-major [npts][dim].
#include <cuda_runtime.h>

#include <climits>
#include <cstdlib>

#include "ibgm_internal.cuh"

namespace ibgm {

// 1D weights of the 4-point kernel for the nodes base-1 .. base+2 around
// x = X/h - o (o = staggering offset), base = floor(x), r = x - base in [0,1).
//   COS4   : phi(r) = (1 + cos(pi r/2))/4 -> ((1-sin), (1+cos), (1+sin), (1-cos))/4 at pi r/2
//   PESKIN4: eq. (discretedelta) on the same four nodes, with
//            q = sqrt(1 + 4r - 4r^2): ((3-2r-q), (3-2r+q), (1+2r+q), (1+2r-q))/8
template <int KER>
__device__ __forceinline__ void weights4(double x, int n, int& i0, double w[4])
{
    const double fl = floor(x);
    const double r = x - fl;
    long long b = (long long)fl - 1;
    b %= n;
    if (b < 0) b += n;
    i0 = (int)b;
    if (KER == IB_DELTA_COS4) {
        double sn, cs;
        sincospi(0.5 * r, &sn, &cs);
        w[0] = 0.25 * (1.0 - sn);
        w[1] = 0.25 * (1.0 + cs);
        w[2] = 0.25 * (1.0 + sn);
        w[3] = 0.25 * (1.0 - cs);
    } else {
        const double q = sqrt(1.0 + 4.0 * r - 4.0 * r * r);
        w[0] = 0.125 * (3.0 - 2.0 * r - q);
        w[1] = 0.125 * (3.0 - 2.0 * r + q);
        w[2] = 0.125 * (1.0 + 2.0 * r + q);
        w[3] = 0.125 * (1.0 + 2.0 * r - q);
    }
}

__device__ __forceinline__ int wrap1(int i, int n) { return i >= n ? i - n : i; }

// Steps 1a-1c: U^n = sum u^n delta_h h^d at X^n; X^{n+1} by AB2
// (forward Euler at n = 0); X^{n+1/2} = (X^{n+1}+X^n)/2.
template <int DIM, int KER>
__global__ void k_interp_evolve(const double* __restrict__ u0, const double* __restrict__ u1,
                                const double* __restrict__ u2, double* __restrict__ X, double* __restrict__ Xh,
                                double* __restrict__ Uprev, double* __restrict__ Xold, double* __restrict__ Uold,
                                int64_t npts, int n, double invh, double dt, int first)
{
    pdl_wait();
    pdl_trigger();
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= npts) return;
    const double* uc[3] = {u0, u1, u2};
    double Xk[3];
#pragma unroll
    for (int a = 0; a < DIM; ++a) Xk[a] = X[k * DIM + a];
    const size_t nn = (size_t)n;
#pragma unroll
    for (int c = 0; c < DIM; ++c) {
        int i0[3] = {0, 0, 0};
        double w[3][4];
#pragma unroll
        for (int a = 0; a < DIM; ++a) weights4<KER>(Xk[a] * invh - (a == c ? 0.0 : 0.5), n, i0[a], w[a]);
        double acc = 0.0;
        if (DIM == 2) {
#pragma unroll
            for (int m1 = 0; m1 < 4; ++m1) {
                const size_t row = nn * (size_t)wrap1(i0[1] + m1, n);
                double r = 0.0;
#pragma unroll
                for (int m0 = 0; m0 < 4; ++m0) r += w[0][m0] * uc[c][row + wrap1(i0[0] + m0, n)];
                acc += w[1][m1] * r;
            }
        } else {
#pragma unroll
            for (int m2 = 0; m2 < 4; ++m2) {
                const size_t pl = nn * nn * (size_t)wrap1(i0[2] + m2, n);
                double pa = 0.0;
#pragma unroll
                for (int m1 = 0; m1 < 4; ++m1) {
                    const size_t row = pl + nn * (size_t)wrap1(i0[1] + m1, n);
                    double r = 0.0;
#pragma unroll
                    for (int m0 = 0; m0 < 4; ++m0) r += w[0][m0] * uc[c][row + wrap1(i0[0] + m0, n)];
                    pa += w[1][m1] * r;
                }
                acc += w[2][m2] * pa;
            }
        }
        const double up = Uprev[k * DIM + c];
        const double xn = first ? Xk[c] + dt * acc : Xk[c] + dt * (1.5 * acc - 0.5 * up);
        Xh[k * DIM + c] = 0.5 * (xn + Xk[c]);
        X[k * DIM + c] = xn;
        Uprev[k * DIM + c] = acc;   // U^n becomes U^{n-1} of the next step
        Xold[k * DIM + c] = Xk[c];  // X^n, U^{n-1}: the state before this step's IB phase
        Uold[k * DIM + c] = up;
    }
}

// The same Steps 1a-1c with one thread per (point, component): a 64 * DIM block holds
// 64 points, warp group c interpolates component c of all of them (3x the threads of
// k_interp_evolve at a third of the registers); the block barrier orders every read of
// X^n before the writes of X^{n+1}.
template <int DIM, int KER>
__global__ void __launch_bounds__(64 * DIM) k_interp_comp(const double* __restrict__ u0, const double* __restrict__ u1,
                                                        const double* __restrict__ u2, double* __restrict__ X,
                                                        double* __restrict__ Xh, double* __restrict__ Uprev,
                                                        double* __restrict__ Xold, double* __restrict__ Uold,
                                                        int64_t npts, int n, double invh, double dt, int first)
{
    const int c = threadIdx.x >> 6;
    const int64_t k = blockIdx.x * 64LL + (threadIdx.x & 63);
    const bool ok = k < npts;
    double Xk[3] = {0, 0, 0};
    if (ok) {
#pragma unroll
        for (int a = 0; a < DIM; ++a) Xk[a] = X[k * DIM + a];
    }
    __syncthreads();
    if (!ok) return;
    const double* uc = (c == 0) ? u0 : (c == 1 ? u1 : u2);
    const size_t nn = (size_t)n;
    int i0[3] = {0, 0, 0};
    double w[3][4];
#pragma unroll
    for (int a = 0; a < DIM; ++a) weights4<KER>(Xk[a] * invh - (a == c ? 0.0 : 0.5), n, i0[a], w[a]);
    double acc = 0.0;
    if (DIM == 2) {
#pragma unroll
        for (int m1 = 0; m1 < 4; ++m1) {
            const size_t row = nn * (size_t)wrap1(i0[1] + m1, n);
            double r = 0.0;
#pragma unroll
            for (int m0 = 0; m0 < 4; ++m0) r += w[0][m0] * uc[row + wrap1(i0[0] + m0, n)];
            acc += w[1][m1] * r;
        }
    } else {
#pragma unroll
        for (int m2 = 0; m2 < 4; ++m2) {
            const size_t pl = nn * nn * (size_t)wrap1(i0[2] + m2, n);
            double pa = 0.0;
#pragma unroll
            for (int m1 = 0; m1 < 4; ++m1) {
                const size_t row = pl + nn * (size_t)wrap1(i0[1] + m1, n);
                double r = 0.0;
#pragma unroll
                for (int m0 = 0; m0 < 4; ++m0) r += w[0][m0] * uc[row + wrap1(i0[0] + m0, n)];
                pa += w[1][m1] * r;
            }
            acc += w[2][m2] * pa;
        }
    }
    const double xc = (c == 0) ? Xk[0] : (c == 1 ? Xk[1] : Xk[2]);
    const double up = Uprev[k * DIM + c];
    const double xn = first ? xc + dt * acc : xc + dt * (1.5 * acc - 0.5 * up);
    Xh[k * DIM + c] = 0.5 * (xn + xc);
    X[k * DIM + c] = xn;
    Uprev[k * DIM + c] = acc;
    Xold[k * DIM + c] = xc;
    Uold[k * DIM + c] = up;
}

// Step 2a: F_k = sum_{e=(k,m)} kappa_e (X_m - X_k)(1 - L_e/|X_m - X_k|) at X^{n+1/2}
// (PAPER.md:607-614 in the force-connection form of PAPER.md:856-861), gathered per
// point from a CSR adjacency (no atomics).  X_m - X_k is the minimum-image displacement
// in the periodic unit box (a fibre closing through the boundary connects to its
// periodic copy; R26).
template <int DIM>
__global__ void k_force(const double* __restrict__ Xh, const int32_t* __restrict__ ptr,
                        const int32_t* __restrict__ nbr, const double* __restrict__ kap,
                        const double* __restrict__ rest, int has_rest, double* __restrict__ F, int64_t npts,
                        double H, double invH, int* __restrict__ err)
{
    pdl_wait();
    pdl_trigger();
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= npts) return;
    double xk[3] = {0, 0, 0}, acc[3] = {0, 0, 0};
#pragma unroll
    for (int a = 0; a < DIM; ++a) xk[a] = Xh[k * DIM + a];
    for (int e = ptr[k]; e < ptr[k + 1]; ++e) {
        const int m = nbr[e];
        double d[3] = {0, 0, 0}, l2 = 0.0;
#pragma unroll
        for (int a = 0; a < DIM; ++a) {
            d[a] = Xh[(int64_t)m * DIM + a] - xk[a];
            d[a] -= H * rint(d[a] * invH);
            l2 += d[a] * d[a];
        }
        double t = kap[e];
        if (has_rest) {
            const double L = rest[e];
            if (L != 0.0) {
                if (l2 > 0.0) {
                    t *= 1.0 - L / sqrt(l2);
                } else {
                    // |X_m - X_k| = 0 with L != 0: the strain direction is undefined
                    // (SPEC.md:140 singular strain).  Raise IB_EDEGENERATE and drop the
                    // connection's (0-length) force instead of spreading NaN.
                    *(volatile int*)(err + ERR_DEGENERATE) = 1;
                    t = 0.0;
                }
            }
        }
#pragma unroll
        for (int a = 0; a < DIM; ++a) acc[a] += t * d[a];
    }
#pragma unroll
    for (int a = 0; a < DIM; ++a) F[k * DIM + a] = acc[a];
}

// Step 2b: f_c += F_k,c w_k h^{-d} prod_a phi(X_a/h - I_a - o_{c,a}) at X^{n+1/2}
// (PAPER.md:616-621).  The force is accumulated (fp64 atomics) directly into the AB2
// history G = N(u^{n-1}) + (2/rho) f that the momentum pass reads (R24), so
// f is never cleared or re-read as a separate field; with keep_f it is also written
// to f for ib_get_aux.
template <int DIM, int KER, bool KEEP>
__global__ void __launch_bounds__(128) k_spread(const double* __restrict__ Xh, const double* __restrict__ F,
                         const double* __restrict__ wgt, double* __restrict__ g0, double* __restrict__ g1,
                         double* __restrict__ g2, double* __restrict__ f0, double* __restrict__ f1,
                         double* __restrict__ f2, int64_t npts, int n, double invh, double invhd, double two_rho)
{
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= npts) return;
    double* gc[3] = {g0, g1, g2};
    double* fc[3] = {f0, f1, f2};
    double Xk[3];
#pragma unroll
    for (int a = 0; a < DIM; ++a) Xk[a] = Xh[k * DIM + a];
    const double wk = wgt[k] * invhd;
    const size_t nn = (size_t)n;
#pragma unroll
    for (int c = 0; c < DIM; ++c) {
        int i0[3] = {0, 0, 0};
        double w[3][4];
#pragma unroll
        for (int a = 0; a < DIM; ++a) weights4<KER>(Xk[a] * invh - (a == c ? 0.0 : 0.5), n, i0[a], w[a]);
        const double Fc = F[k * DIM + c] * wk;
        if (DIM == 2) {
#pragma unroll
            for (int m1 = 0; m1 < 4; ++m1) {
                const size_t row = nn * (size_t)wrap1(i0[1] + m1, n);
                const double a1 = Fc * w[1][m1];
#pragma unroll
                for (int m0 = 0; m0 < 4; ++m0) {
                    const size_t q = row + wrap1(i0[0] + m0, n);
                    const double v = a1 * w[0][m0];
                    atomicAdd(gc[c] + q, two_rho * v);
                    if (KEEP) atomicAdd(fc[c] + q, v);
                }
            }
        } else {
#pragma unroll
            for (int m2 = 0; m2 < 4; ++m2) {
                const size_t pl = nn * nn * (size_t)wrap1(i0[2] + m2, n);
                const double a2 = Fc * w[2][m2];
#pragma unroll
                for (int m1 = 0; m1 < 4; ++m1) {
                    const size_t row = pl + nn * (size_t)wrap1(i0[1] + m1, n);
                    const double a1 = a2 * w[1][m1];
#pragma unroll
                    for (int m0 = 0; m0 < 4; ++m0) {
                        const size_t q = row + wrap1(i0[0] + m0, n);
                        const double v = a1 * w[0][m0];
                        atomicAdd(gc[c] + q, two_rho * v);
                        if (KEEP) atomicAdd(fc[c] + q, v);
                    }
                }
            }
        }
    }
}

// -------------------------------------------------------------------------------
// Brick-binned spreading (Step 2b).  Points are counting-sorted each step into bricks
// of B^d cells (by the cell containing X^{n+1/2}); one CTA per non-empty brick
// accumulates the contributions of its points into a shared tile covering the brick
// plus the 4-point support (B+4 nodes per axis), each tile column owned by one thread
// (no atomics inside the brick), then flushes the non-zero tile entries into G (and f)
// with native fp64 reductions (REDG).  This replaces 4^d d scattered atomics per point
// by ~(B+4)^d d per brick.
// -------------------------------------------------------------------------------
template <int DIM, int B>
__device__ __forceinline__ int brick_of(const double* Xk, double invh, int n, int nb)
{
    int id = 0, mul = 1;
#pragma unroll
    for (int a = 0; a < DIM; ++a) {
        long long c = (long long)floor(Xk[a] * invh);
        c %= n;
        if (c < 0) c += n;
        id += (int)(c / B) * mul;
        mul *= nb;
    }
    return id;
}

template <int DIM, int B>
__global__ void k_bin_count(const double* __restrict__ Xh, int64_t npts, int n, int nb, double invh,
                            int* __restrict__ bid, int* __restrict__ count)
{
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= npts) return;
    double Xk[3];
#pragma unroll
    for (int a = 0; a < DIM; ++a) Xk[a] = Xh[k * DIM + a];
    const int b = brick_of<DIM, B>(Xk, invh, n, nb);
    bid[k] = b;
    atomicAdd(count + b, 1);
}

// exclusive scan of the brick counts in three launches (block partial sums, scan of
// the partials, block-local scan + offset), and the list of non-empty bricks
constexpr int kScanB = 1024;

__device__ __forceinline__ int block_excl_scan(int v, int* sh)
{
    // Hillis-Steele over blockDim.x (<= 1024) entries; returns the exclusive prefix
    const int t = threadIdx.x;
    sh[t] = v;
    __syncthreads();
    for (int off = 1; off < (int)blockDim.x; off <<= 1) {
        const int a = (t >= off) ? sh[t - off] : 0;
        __syncthreads();
        sh[t] += a;
        __syncthreads();
    }
    const int incl = sh[t];
    __syncthreads();
    return incl - v;
}

__global__ void k_scan_partial(const int* __restrict__ count, int nbricks, int* __restrict__ partial)
{
    __shared__ int sh[kScanB];
    const int b = blockIdx.x * kScanB + threadIdx.x;
    const int v = (b < nbricks) ? count[b] : 0;
    sh[threadIdx.x] = v;
    __syncthreads();
    for (int off = kScanB / 2; off > 0; off >>= 1) {
        if ((int)threadIdx.x < off) sh[threadIdx.x] += sh[threadIdx.x + off];
        __syncthreads();
    }
    if (threadIdx.x == 0) partial[blockIdx.x] = sh[0];
}

__global__ void k_scan_top(int* __restrict__ partial, int nparts, int* __restrict__ nlist)
{
    __shared__ int sh[kScanB];
    // nparts <= kScanB * per; each thread owns a contiguous range
    const int per = (nparts + kScanB - 1) / kScanB;
    const int lo = threadIdx.x * per, hi = min(nparts, lo + per);
    int sum = 0;
    for (int i = lo; i < hi; ++i) sum += partial[i];
    int run = block_excl_scan(sum, sh);
    for (int i = lo; i < hi; ++i) {
        const int v = partial[i];
        partial[i] = run;
        run += v;
    }
    if (threadIdx.x == 0) *nlist = 0;
}

__global__ void k_scan_final(const int* __restrict__ count, int nbricks, const int* __restrict__ partial,
                             int* __restrict__ start, int* __restrict__ cursor, int* __restrict__ list,
                             int* __restrict__ nlist)
{
    __shared__ int sh[kScanB];
    const int b = blockIdx.x * kScanB + threadIdx.x;
    const int v = (b < nbricks) ? count[b] : 0;
    const int ex = block_excl_scan(v, sh) + partial[blockIdx.x];
    if (b < nbricks) {
        start[b] = ex;
        cursor[b] = 0;
        if (v > 0) list[atomicAdd(nlist, 1)] = b;
    }
}

__global__ void k_bin_fill(const int* __restrict__ bid, int64_t npts, const int* __restrict__ start,
                           int* __restrict__ cursor, int* __restrict__ sorted)
{
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= npts) return;
    const int b = bid[k];
    sorted[start[b] + atomicAdd(cursor + b, 1)] = (int)k;
}

template <int DIM, int KER, int B, bool KEEP>
__global__ void __launch_bounds__(256) k_brick_spread(
    const double* __restrict__ Xh, const double* __restrict__ F, const double* __restrict__ wgt,
    const int* __restrict__ sorted, const int* __restrict__ start, const int* __restrict__ count,
    const int* __restrict__ list, const int* __restrict__ nlist, double* __restrict__ g0, double* __restrict__ g1,
    double* __restrict__ g2, double* __restrict__ f0, double* __restrict__ f1, double* __restrict__ f2, int n, int nb,
    double invh, double invhd, double two_rho)
{
    constexpr int T = B + 4;                    // tile nodes per axis
    constexpr int TV = (DIM == 3) ? T * T * T : T * T;
    constexpr int CH = 128;                     // points per chunk
    extern __shared__ double sm[];
    double* tile = sm;                          // [DIM][TV]
    double* W = tile + DIM * TV;                // [CH][DIM comps][DIM axes][4]
    double* coef = W + CH * DIM * DIM * 4;      // [CH][DIM]
    int* base = (int*)(coef + CH * DIM);        // [CH][DIM][DIM] tile-relative base node
    const int t = threadIdx.x, NT = blockDim.x;
    const int nl = *nlist;
    for (int li = blockIdx.x; li < nl; li += gridDim.x) {
        const int b = list[li];
        int bo[3] = {0, 0, 0};                  // tile origin (node index of tile entry 0)
        {
            int r = b;
#pragma unroll
            for (int a = 0; a < DIM; ++a) { bo[a] = (r % nb) * B - 2; r /= nb; }
        }
        for (int e = t; e < DIM * TV; e += NT) tile[e] = 0.0;
        const int p0 = start[b], np = count[b];
        for (int c0 = 0; c0 < np; c0 += CH) {
            const int nc = min(CH, np - c0);
            __syncthreads();
            // per (point, component): tile-relative base node and 1D weights per axis
            for (int e = t; e < nc * DIM; e += NT) {
                const int pi = e / DIM, c = e - pi * DIM;
                const int k = sorted[p0 + c0 + pi];
                double Xk[3];
#pragma unroll
                for (int a = 0; a < DIM; ++a) Xk[a] = Xh[(int64_t)k * DIM + a];
#pragma unroll
                for (int a = 0; a < DIM; ++a) {
                    const double x = Xk[a] * invh - (a == c ? 0.0 : 0.5);
                    const double fl = floor(x);
                    const double r = x - fl;
                    // base node i0 = fl - 1, relative to the tile origin (same periodic image as the brick)
                    long long i0 = (long long)fl - 1;
                    long long rel = i0 - bo[a];
                    rel = ((rel % n) + n) % n;
                    if (rel > (long long)T) rel -= n;   // keep in the tile's image
                    base[(pi * DIM + c) * DIM + a] = (int)rel;
                    double* w = W + ((pi * DIM + c) * DIM + a) * 4;
                    if (KER == IB_DELTA_COS4) {
                        double sn, cs;
                        sincospi(0.5 * r, &sn, &cs);
                        w[0] = 0.25 * (1.0 - sn); w[1] = 0.25 * (1.0 + cs);
                        w[2] = 0.25 * (1.0 + sn); w[3] = 0.25 * (1.0 - cs);
                    } else {
                        const double q = sqrt(1.0 + 4.0 * r - 4.0 * r * r);
                        w[0] = 0.125 * (3.0 - 2.0 * r - q); w[1] = 0.125 * (3.0 - 2.0 * r + q);
                        w[2] = 0.125 * (1.0 + 2.0 * r + q); w[3] = 0.125 * (1.0 + 2.0 * r - q);
                    }
                }
                coef[pi * DIM + c] = F[(int64_t)k * DIM + c] * wgt[k] * invhd;
            }
            __syncthreads();
            // owner accumulation, no atomics: in 3D a thread owns a z-column (c, tx, ty) of the
            // tile, in 2D a node; it visits the chunk's points and adds those whose 4-point
            // support covers it
            constexpr int NOWN = DIM * T * T;
            for (int o = t; o < NOWN; o += NT) {
                const int c = o / (T * T), rem = o - c * T * T;
                const int ty = rem / T, tx = rem - ty * T;
                const int colo = c * TV + ty * T + tx;         // offset of the owned column in sm[]
                const int bofs = (int)(base - (int*)sm);        // int offset of base[] in sm (as ints)
                for (int pi = 0; pi < nc; ++pi) {
                    const int pc = pi * DIM + c;
                    const int* bsp = (const int*)sm + bofs + pc * DIM;
                    const int dx = tx - bsp[0], dy = ty - bsp[1];
                    if ((unsigned)dx < 4u && (unsigned)dy < 4u) {
                        const int wo = (int)(W - sm) + pc * DIM * 4;
                        const double v = sm[(int)(coef - sm) + pc] * sm[wo + dx] * sm[wo + 4 + dy];
                        if (DIM == 3) {
                            const int zo = colo + bsp[2] * T * T;
#pragma unroll
                            for (int dz = 0; dz < 4; ++dz) sm[zo + dz * T * T] += v * sm[wo + 8 + dz];
                        } else {
                            sm[colo] += v;
                        }
                    }
                }
            }
        }
        __syncthreads();
        // flush the tile into G (and f) with periodic wrap
        double* gc[3] = {g0, g1, g2};
        double* fc[3] = {f0, f1, f2};
        for (int e = t; e < DIM * TV; e += NT) {
            const double v = tile[e];
            if (v == 0.0) continue;
            const int c = e / TV;
            int r = e - c * TV;
            size_t q = 0, mul = 1;
#pragma unroll
            for (int a = 0; a < DIM; ++a) {
                int gi = bo[a] + (r % T);
                r /= T;
                gi = (gi < 0) ? gi + n : (gi >= n ? gi - n : gi);
                q += (size_t)gi * mul;
                mul *= (size_t)n;
            }
            atomicAdd(gc[c] + q, two_rho * v);
            if (KEEP) atomicAdd(fc[c] + q, v);
        }
        __syncthreads();
    }
}

// -------------------------------------------------------------------------------
// Box-staged interpolation and spreading (Steps 1a and 2b).  The points are stored in
// Morton order of their initial cells (ib_set_boundary), so the kBoxPts consecutive
// points of a CTA lie close together: the CTA takes the bounding box of their 4-point
// supports (all components), and
//   interpolation  loads the box of u once (coalesced along x) into shared memory and
//                  gathers each point's 4^d stencil from there;
//   spreading      accumulates every contribution into the box in shared memory, then
//                  adds the non-zero box entries into G (and f) with one global fp64
//                  reduction each -- instead of 4^d d scattered global atomics per point.
// Thread (p, c) owns point p of the chunk and velocity component c.  A chunk whose box
// exceeds the shared-memory budget (points far apart) falls back to direct global
// gathers / atomics for that chunk, so the result does not depend on the ordering.
// -------------------------------------------------------------------------------
constexpr int kBoxPts = 64;
template <int DIM> struct BoxCap;
template <> struct BoxCap<3> { static constexpr int EXT = 16, VOL = 2048; };
template <> struct BoxCap<2> { static constexpr int EXT = 40, VOL = 1024; };

// 1D weights with the UNWRAPPED base node index (base = floor(x) - 1)
template <int KER>
__device__ __forceinline__ void weights4u(double x, int& base, double w[4])
{
    const double fl = floor(x);
    const double r = x - fl;
    base = (int)fl - 1;
    if (KER == IB_DELTA_COS4) {
        double sn, cs;
        sincospi(0.5 * r, &sn, &cs);
        w[0] = 0.25 * (1.0 - sn);
        w[1] = 0.25 * (1.0 + cs);
        w[2] = 0.25 * (1.0 + sn);
        w[3] = 0.25 * (1.0 - cs);
    } else {
        const double q = sqrt(1.0 + 4.0 * r - 4.0 * r * r);
        w[0] = 0.125 * (3.0 - 2.0 * r - q);
        w[1] = 0.125 * (3.0 - 2.0 * r + q);
        w[2] = 0.125 * (1.0 + 2.0 * r + q);
        w[3] = 0.125 * (1.0 + 2.0 * r - q);
    }
}

__device__ __forceinline__ int wrapm(int i, int n)
{
    i %= n;
    return i < 0 ? i + n : i;
}

// chunk box: origin o (unwrapped node index) and extents e per axis; false if it does
// not fit.  Every thread of the CTA must call it (two barriers).
template <int DIM>
__device__ __forceinline__ bool chunk_box(const double* Xk, bool lead, double invh, int* sh, int o[3], int e[3], int& V)
{
    if (threadIdx.x < 3) { sh[threadIdx.x] = INT_MAX; sh[3 + threadIdx.x] = INT_MIN; }
    __syncthreads();
    if (lead)
#pragma unroll
        for (int a = 0; a < DIM; ++a) {
            const int ci = (int)floor(Xk[a] * invh);
            atomicMin(sh + a, ci);
            atomicMax(sh + 3 + a, ci);
        }
    __syncthreads();
    bool ok = true;
    V = 1;
#pragma unroll
    for (int a = 0; a < DIM; ++a) {
        o[a] = sh[a] - 2;
        e[a] = sh[3 + a] - sh[a] + 5;
        ok = ok && e[a] <= BoxCap<DIM>::EXT;
        V *= e[a];
    }
    return ok && V <= BoxCap<DIM>::VOL;
}

// Walk the box row by row: XL lanes along x (no per-element division), rows (c, y[, z])
// spread over the remaining lanes.  f(c, i, q): i the box index, q the global index.
template <int DIM, class Fn>
__device__ __forceinline__ void for_box(const int o[3], const int e[3], int V, int n, Fn&& f)
{
    constexpr int XL = (DIM == 3) ? 16 : 32;
    const int xl = threadIdx.x % XL, rstep = blockDim.x / XL;
    const int rows_c = (DIM == 3) ? e[1] * e[2] : e[1];
    const int ox = wrapm(o[0], n);
    const size_t nn = (size_t)n;
    for (int r = threadIdx.x / XL; r < DIM * rows_c; r += rstep) {
        const int c = r / rows_c;
        const int rr = r - c * rows_c;
        const int z = (DIM == 3) ? rr / e[1] : 0;
        const int y = rr - z * e[1];
        size_t rowg = nn * (size_t)wrapm(o[1] + y, n);
        if (DIM == 3) rowg += nn * nn * (size_t)wrapm(o[2] + z, n);
        const int rowb = c * V + (z * e[1] + y) * e[0];
        for (int x = xl; x < e[0]; x += XL) {
            int gx = ox + x;
            while (gx >= n) gx -= n;
            f(c, rowb + x, rowg + (size_t)gx);
        }
    }
}

template <int DIM, int KER>
__global__ void __launch_bounds__(kBoxPts * DIM) k_interp_box(const double* __restrict__ u0, const double* __restrict__ u1,
                                                            const double* __restrict__ u2, double* __restrict__ X,
                                                            double* __restrict__ Xh, double* __restrict__ Uprev,
                                                            double* __restrict__ Xold, double* __restrict__ Uold,
                                                            int64_t npts, int n, double invh, double dt, int first)
{
    extern __shared__ double box[];
    __shared__ int sh[6];
    const int t = threadIdx.x;
    const int p = t % kBoxPts, c = t / kBoxPts;
    const int64_t k = blockIdx.x * (int64_t)kBoxPts + p;
    const bool valid = k < npts;
    double Xk[3] = {0, 0, 0};
    if (valid)
#pragma unroll
        for (int a = 0; a < DIM; ++a) Xk[a] = X[k * DIM + a];
    int o[3] = {0, 0, 0}, e[3] = {1, 1, 1}, V;
    const bool fits = chunk_box<DIM>(Xk, valid && c == 0, invh, sh, o, e, V);
    if (fits) {
        for_box<DIM>(o, e, V, n, [&](int cc, int i, size_t q) {
            const double* ucc = (cc == 0) ? u0 : (cc == 1 ? u1 : u2);
            box[i] = __ldg(ucc + q);
        });
        __syncthreads();
    }
    if (!valid) return;
    int b[3] = {0, 0, 0};
    double w[3][4];
#pragma unroll
    for (int a = 0; a < DIM; ++a) weights4u<KER>(Xk[a] * invh - (a == c ? 0.0 : 0.5), b[a], w[a]);
    double acc = 0.0;
    if (fits) {
        const double* bc = box + c * V;
        if (DIM == 2) {
#pragma unroll
            for (int m1 = 0; m1 < 4; ++m1) {
                const double* row = bc + (b[1] - o[1] + m1) * e[0] + (b[0] - o[0]);
                double r = 0.0;
#pragma unroll
                for (int m0 = 0; m0 < 4; ++m0) r += w[0][m0] * row[m0];
                acc += w[1][m1] * r;
            }
        } else {
#pragma unroll
            for (int m2 = 0; m2 < 4; ++m2) {
                double pa = 0.0;
#pragma unroll
                for (int m1 = 0; m1 < 4; ++m1) {
                    const double* row = bc + ((b[2] - o[2] + m2) * e[1] + (b[1] - o[1] + m1)) * e[0] + (b[0] - o[0]);
                    double r = 0.0;
#pragma unroll
                    for (int m0 = 0; m0 < 4; ++m0) r += w[0][m0] * row[m0];
                    pa += w[1][m1] * r;
                }
                acc += w[2][m2] * pa;
            }
        }
    } else {
        const double* u = (c == 0) ? u0 : (c == 1 ? u1 : u2);
        const size_t nn = (size_t)n;
        if (DIM == 2) {
#pragma unroll
            for (int m1 = 0; m1 < 4; ++m1) {
                const size_t row = nn * (size_t)wrapm(b[1] + m1, n);
                double r = 0.0;
#pragma unroll
                for (int m0 = 0; m0 < 4; ++m0) r += w[0][m0] * u[row + wrapm(b[0] + m0, n)];
                acc += w[1][m1] * r;
            }
        } else {
#pragma unroll
            for (int m2 = 0; m2 < 4; ++m2) {
                const size_t pl = nn * nn * (size_t)wrapm(b[2] + m2, n);
                double pa = 0.0;
#pragma unroll
                for (int m1 = 0; m1 < 4; ++m1) {
                    const size_t row = pl + nn * (size_t)wrapm(b[1] + m1, n);
                    double r = 0.0;
#pragma unroll
                    for (int m0 = 0; m0 < 4; ++m0) r += w[0][m0] * u[row + wrapm(b[0] + m0, n)];
                    pa += w[1][m1] * r;
                }
                acc += w[2][m2] * pa;
            }
        }
    }
    // Steps 1b-1c for component c of this point
    const double xc = (c == 0) ? Xk[0] : (c == 1 ? Xk[1] : Xk[2]);
    const double up = Uprev[k * DIM + c];
    const double xn = first ? xc + dt * acc : xc + dt * (1.5 * acc - 0.5 * up);
    Xh[k * DIM + c] = 0.5 * (xn + xc);
    X[k * DIM + c] = xn;
    Uprev[k * DIM + c] = acc;
    Xold[k * DIM + c] = xc;
    Uold[k * DIM + c] = up;
}

// shared layout of the spread: box [DIM][VOL], then per (component, point) the weights
// [DIM axes][4] and the scaled force; the box-relative base nodes are static shared
template <int DIM>
__host__ __device__ constexpr size_t spread_box_doubles()
{
    return (size_t)DIM * (DIM == 3 ? BoxCap<3>::VOL : BoxCap<2>::VOL) + (size_t)DIM * kBoxPts * (DIM * 4 + 1);
}

template <int DIM, int KER, bool KEEP>
__global__ void __launch_bounds__(kBoxPts * DIM) k_spread_box(const double* __restrict__ Xh, const double* __restrict__ F,
                                                            const double* __restrict__ wgt, double* __restrict__ g0,
                                                            double* __restrict__ g1, double* __restrict__ g2,
                                                            double* __restrict__ f0, double* __restrict__ f1,
                                                            double* __restrict__ f2, int64_t npts, int n, double invh,
                                                            double invhd, double two_rho)
{
    constexpr int VOL = (DIM == 3) ? BoxCap<3>::VOL : BoxCap<2>::VOL;
    extern __shared__ double box[];
    double* W = box + DIM * VOL;                      // [c][p][a][4]
    double* coef = W + DIM * kBoxPts * DIM * 4;       // [c][p]
    __shared__ int sh[6];
    __shared__ int bs[DIM * kBoxPts * 4];             // [c][p][a] (padded to 4)
    const int t = threadIdx.x;
    const int p = t % kBoxPts, c = t / kBoxPts;
    const int64_t k = blockIdx.x * (int64_t)kBoxPts + p;
    const bool valid = k < npts;
    double Xk[3] = {0, 0, 0};
    if (valid)
#pragma unroll
        for (int a = 0; a < DIM; ++a) Xk[a] = Xh[k * DIM + a];
    int o[3] = {0, 0, 0}, e[3] = {1, 1, 1}, V;
    const bool fits = chunk_box<DIM>(Xk, valid && c == 0, invh, sh, o, e, V);
    double* gcc = (c == 0) ? g0 : (c == 1 ? g1 : g2);
    double* fcc = (c == 0) ? f0 : (c == 1 ? f1 : f2);
    int b[3] = {0, 0, 0};
    double w[3][4];
    double Fc = 0.0;
    if (valid) {
#pragma unroll
        for (int a = 0; a < DIM; ++a) weights4u<KER>(Xk[a] * invh - (a == c ? 0.0 : 0.5), b[a], w[a]);
        Fc = F[k * DIM + c] * wgt[k] * invhd;
    }
    if (!fits) {
        // direct fallback: 4^d global reductions for this (point, component)
        if (!valid) return;
        const size_t nn = (size_t)n;
        if (DIM == 2) {
#pragma unroll
            for (int m1 = 0; m1 < 4; ++m1) {
                const size_t row = nn * (size_t)wrapm(b[1] + m1, n);
                const double a1 = Fc * w[1][m1];
#pragma unroll
                for (int m0 = 0; m0 < 4; ++m0) {
                    const size_t q = row + wrapm(b[0] + m0, n);
                    const double v = a1 * w[0][m0];
                    atomicAdd(gcc + q, two_rho * v);
                    if (KEEP) atomicAdd(fcc + q, v);
                }
            }
        } else {
#pragma unroll
            for (int m2 = 0; m2 < 4; ++m2) {
                const size_t pl = nn * nn * (size_t)wrapm(b[2] + m2, n);
                const double a2 = Fc * w[2][m2];
#pragma unroll
                for (int m1 = 0; m1 < 4; ++m1) {
                    const size_t row = pl + nn * (size_t)wrapm(b[1] + m1, n);
                    const double a1 = a2 * w[1][m1];
#pragma unroll
                    for (int m0 = 0; m0 < 4; ++m0) {
                        const size_t q = row + wrapm(b[0] + m0, n);
                        const double v = a1 * w[0][m0];
                        atomicAdd(gcc + q, two_rho * v);
                        if (KEEP) atomicAdd(fcc + q, v);
                    }
                }
            }
        }
        return;
    }
    // per (component, point): box-relative base nodes, weights, scaled force
    {
        const int cp = c * kBoxPts + p;
#pragma unroll
        for (int a = 0; a < DIM; ++a) {
            bs[cp * 4 + a] = valid ? b[a] - o[a] : -1000;
#pragma unroll
            for (int m = 0; m < 4; ++m) W[(cp * DIM + a) * 4 + m] = w[a][m];
        }
        coef[cp] = Fc;
    }
    for (int i = t; i < DIM * V; i += blockDim.x) box[i] = 0.0;
    __syncthreads();
    // owner accumulation (no atomics): a thread owns a z-column (c, x, y) of the box in
    // 3D (a node (c, x, y) in 2D) and adds every point of the chunk whose support covers it
    const int plane = e[0] * e[1];
    for (int col = t; col < DIM * plane; col += blockDim.x) {
        const int cc = col / plane;
        const int rem = col - cc * plane;
        const int y = rem / e[0];
        const int x = rem - y * e[0];
        double* colp = box + cc * V + rem;
        const int* bsc = bs + cc * kBoxPts * 4;
        const double* Wc = W + cc * kBoxPts * DIM * 4;
        const double* cfc = coef + cc * kBoxPts;
        double acc2 = 0.0;
        for (int q = 0; q < kBoxPts; ++q) {
            const int dx = x - bsc[q * 4], dy = y - bsc[q * 4 + 1];
            if ((unsigned)dx < 4u && (unsigned)dy < 4u) {
                const double* wq = Wc + q * DIM * 4;
                const double v = cfc[q] * wq[dx] * wq[4 + dy];
                if (DIM == 3) {
                    double* zp = colp + bsc[q * 4 + 2] * plane;
#pragma unroll
                    for (int dz = 0; dz < 4; ++dz) zp[dz * plane] += v * wq[8 + dz];
                } else {
                    acc2 += v;
                }
            }
        }
        if (DIM == 2) *colp = acc2;
    }
    __syncthreads();
    for_box<DIM>(o, e, V, n, [&](int cc, int i, size_t q) {
        const double v = box[i];
        if (v == 0.0) return;
        atomicAdd(((cc == 0) ? g0 : (cc == 1 ? g1 : g2)) + q, two_rho * v);
        if (KEEP) atomicAdd(((cc == 0) ? f0 : (cc == 1 ? f1 : f2)) + q, v);
    });
}

// -------------------------------------------------------------------------------
// Quad-lane interpolation and spreading (Steps 1a, 2b): 4 lanes per (point,
// component), lane m0 owns the stencil nodes i0+m0 along x, so one warp instruction
// touches 8 rows of 4 consecutive nodes (coalesced sectors) instead of 32 scattered
// nodes.  Groups of a warp are 8 consecutive points (Morton order) of one component.
// -------------------------------------------------------------------------------
template <int DIM, int KER>
__device__ __forceinline__ void quad_weights(const double* Xk, int c, double invh, int n, int b[3], double w[3][4])
{
#pragma unroll
    for (int a = 0; a < DIM; ++a) {
        weights4u<KER>(Xk[a] * invh - (a == c ? 0.0 : 0.5), b[a], w[a]);
        b[a] = wrapm(b[a], n);
    }
}

template <int DIM, int KER>
__global__ void __launch_bounds__(256) k_interp_quad(const double* __restrict__ u0, const double* __restrict__ u1,
                                                     const double* __restrict__ u2, double* __restrict__ X,
                                                     double* __restrict__ Xh, double* __restrict__ Uprev,
                                                     double* __restrict__ Xold, double* __restrict__ Uold,
                                                     int64_t npts, int n, double invh, double dt, int first)
{
    const int64_t g = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 2;   // (component, point) group
    const int m0 = threadIdx.x & 3;
    // groups ordered (point block of 8, component, point): a warp = 8 points x 1 component
    const int64_t blk = g / (8 * DIM);
    const int rem = (int)(g - blk * 8 * DIM);
    const int c = rem >> 3;
    const int64_t k = blk * 8 + (rem & 7);
    const bool valid = k < npts;
    double Xk[3] = {0, 0, 0};
    const int64_t kk = valid ? k : 0;
#pragma unroll
    for (int a = 0; a < DIM; ++a) Xk[a] = X[kk * DIM + a];
    // the DIM component groups of a point live in this block (blockDim is a multiple of
    // 32 DIM), and each writes its component of X^{n+1} below: every read of X^n first
    __syncthreads();
    int b[3];
    double w[3][4];
    quad_weights<DIM, KER>(Xk, c, invh, n, b, w);
    const double* u = (c == 0) ? u0 : (c == 1 ? u1 : u2);
    int ix = b[0] + m0;
    if (ix >= n) ix -= n;
    const double wx = (m0 == 0) ? w[0][0] : (m0 == 1 ? w[0][1] : (m0 == 2 ? w[0][2] : w[0][3]));
    const size_t nn = (size_t)n;
    double acc = 0.0;
    if (DIM == 2) {
#pragma unroll
        for (int m1 = 0; m1 < 4; ++m1) {
            int iy = b[1] + m1;
            if (iy >= n) iy -= n;
            acc += w[1][m1] * __ldg(u + nn * iy + ix);
        }
    } else {
#pragma unroll
        for (int m2 = 0; m2 < 4; ++m2) {
            int iz = b[2] + m2;
            if (iz >= n) iz -= n;
            double pa = 0.0;
#pragma unroll
            for (int m1 = 0; m1 < 4; ++m1) {
                int iy = b[1] + m1;
                if (iy >= n) iy -= n;
                pa += w[1][m1] * __ldg(u + nn * (nn * iz + iy) + ix);
            }
            acc += w[2][m2] * pa;
        }
    }
    acc *= wx;
    acc += __shfl_xor_sync(0xffffffffu, acc, 1);
    acc += __shfl_xor_sync(0xffffffffu, acc, 2);
    if (!valid || m0 != 0) return;
    const double xc = (c == 0) ? Xk[0] : (c == 1 ? Xk[1] : Xk[2]);
    const double up = Uprev[k * DIM + c];
    const double xn = first ? xc + dt * acc : xc + dt * (1.5 * acc - 0.5 * up);
    Xh[k * DIM + c] = 0.5 * (xn + xc);
    X[k * DIM + c] = xn;
    Uprev[k * DIM + c] = acc;
    Xold[k * DIM + c] = xc;
    Uold[k * DIM + c] = up;
}

// PART (z-slab, slab.cu): the items are the `*count` points of `list` whose support meets
// this slab's planes z0 .. z0+nzl-1 of the last axis, and only rows inside the slab are
// accumulated (into the slab's fields, addressed by local plane).
template <int DIM, int KER, bool KEEP, bool PART>
__global__ void __launch_bounds__(256) k_spread_quad(const double* __restrict__ Xh, const double* __restrict__ F,
                                                     const double* __restrict__ wgt, double* __restrict__ g0,
                                                     double* __restrict__ g1, double* __restrict__ g2,
                                                     double* __restrict__ f0, double* __restrict__ f1,
                                                     double* __restrict__ f2, int64_t npts, int n, double invh,
                                                     double invhd, double two_rho, int red,
                                                     const int* __restrict__ list, const int* __restrict__ count,
                                                     int z0, int nzl)
{
    pdl_wait();
    pdl_trigger();
    const int64_t g = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 2;
    const int m0 = threadIdx.x & 3;
    const int64_t blk = g / (8 * DIM);
    const int rem = (int)(g - blk * 8 * DIM);
    const int c = rem >> 3;
    const int64_t item = blk * 8 + (rem & 7);
    const int64_t nitem = PART ? (int64_t)*count : npts;
    bool valid = item < nitem;
    if (PART && blk * 8 >= nitem) return;  // the whole warp is past the list
    if (!red && !valid) return;
    int64_t k = valid ? item : nitem - 1;  // red: every lane takes part in the shuffles
    if (PART) {
        k = list[k];
        if (k < 0) {                        // padding of a warp-aligned chunk (k_slab_select)
            if (!red) return;
            k = 0;
            valid = false;
        }
    }
    double Xk[3] = {0, 0, 0};
#pragma unroll
    for (int a = 0; a < DIM; ++a) Xk[a] = Xh[k * DIM + a];
    int b[3];
    double w[3][4];
    quad_weights<DIM, KER>(Xk, c, invh, n, b, w);
    double* gc = (c == 0) ? g0 : (c == 1 ? g1 : g2);
    double* fc = (c == 0) ? f0 : (c == 1 ? f1 : f2);
    int ix = b[0] + m0;
    if (ix >= n) ix -= n;
    const double wx = (m0 == 0) ? w[0][0] : (m0 == 1 ? w[0][1] : (m0 == 2 ? w[0][2] : w[0][3]));
    const double Fx = valid ? F[k * DIM + c] * wgt[k] * invhd * wx : 0.0;
    const size_t nn = (size_t)n;
    // warp-level pre-reduction (red): a warp's 8 lane groups hold 8 consecutive points
    // (Morton order) of one component; groups with the same base node touch the same
    // 4^d nodes in the same iteration, so a run of them sums its contributions by a
    // segmented suffix scan over the groups and only the run's first group issues the
    // atomics.  Skipped when the warp has no such run.
    const int grp = (threadIdx.x & 31) >> 2;
    bool head = valid;
    int last = grp;          // last group of this group's run
    bool dup = false;
    if (red) {
        const unsigned FULL = 0xffffffffu;
        const long long key = valid ? ((DIM == 3 ? (long long)b[2] * n : 0LL) + b[1]) * n + b[0] : -1LL - grp;
        const long long kprev = __shfl_up_sync(FULL, key, 4);
        const bool h = (grp == 0) || (kprev != key);
        const unsigned hb = __ballot_sync(FULL, h && m0 == 0);     // bit 4g: group g starts a run
        dup = (hb != 0x11111111u);
        const unsigned above = hb & ~((2u << (4 * grp)) - 1u);
        last = above ? ((__ffs(above) - 1) >> 2) - 1 : 7;
        head = valid && h;
    }
    auto reduce = [&](double v) -> double {
        if (dup) {
#pragma unroll
            for (int d = 1; d < 8; d <<= 1) {
                const double o = __shfl_down_sync(0xffffffffu, v, 4 * d);
                if (grp + d <= last) v += o;
            }
        }
        return v;
    };
    if (DIM == 2) {
#pragma unroll
        for (int m1 = 0; m1 < 4; ++m1) {
            int iy = b[1] + m1;
            if (iy >= n) iy -= n;
            const double v = reduce(Fx * w[1][m1]);
            const int ly = PART ? iy - z0 : iy;
            if (head && (!PART || (unsigned)ly < (unsigned)nzl)) {
                atomicAdd(gc + nn * ly + ix, two_rho * v);
                if (KEEP) atomicAdd(fc + nn * ly + ix, v);
            }
        }
    } else {
#pragma unroll
        for (int m2 = 0; m2 < 4; ++m2) {
            int iz = b[2] + m2;
            if (iz >= n) iz -= n;
            const int lz = PART ? iz - z0 : iz;
            const bool in = !PART || (unsigned)lz < (unsigned)nzl;
            const double a2 = Fx * w[2][m2];
#pragma unroll
            for (int m1 = 0; m1 < 4; ++m1) {
                int iy = b[1] + m1;
                if (iy >= n) iy -= n;
                const double v = reduce(a2 * w[1][m1]);
                const size_t q = nn * (nn * (size_t)(in ? lz : 0) + iy) + ix;
                if (head && in) {
                    atomicAdd(gc + q, two_rho * v);
                    if (KEEP) atomicAdd(fc + q, v);
                }
            }
        }
    }
}

// -------------------------------------------------------------------------------
// Window-staged spreading and interpolation (Steps 2b and 1a).  A warp takes a window
// of 32 consecutive points (Morton order, R30) and one velocity component in 3D (both
// components, one per half-warp, in 2D).  The 4^d supports of a window's points overlap
// heavily (dense membranes: at config 4 a window of 32 points touches ~170 distinct
// nodes, against 32 x 64 contributions), so the warp works in a box of shared memory
// covering the window's supports (origin = the smallest base node, extents = spread of
// the base nodes + 4):
//   spreading      iterates over the window's points; for each point the lanes own the
//                  distinct nodes of its support (2 per lane in 3D, 1 per half-warp lane
//                  in 2D) and add their contributions to the box -- no two lanes touch
//                  the same entry in one iteration, so no atomics -- then every non-zero
//                  box entry goes to G (and f) with ONE global fp64 reduction;
//   interpolation  loads the box of u_c once (rows contiguous along x) and every lane
//                  gathers its point's 4^d stencil from shared memory.
// Only warp barriers: warps never wait for each other.  A window whose box exceeds the
// budget (points far apart, or a window across the periodic seam) falls back to direct
// global reductions / gathers, so results never depend on the ordering.
// -------------------------------------------------------------------------------
template <int DIM>
struct WinCfg {
    static constexpr int CPW = (DIM == 3) ? 1 : 2;             // components per warp
    static constexpr int WPW = DIM / CPW;                      // warps per window
    static constexpr int CAP = (DIM == 3) ? 640 : 320;         // box doubles per component
    static constexpr int REC = 4 * DIM;                        // per point: w_x F, w_y[, w_z]
    static constexpr int WARP_DOUBLES = CPW * (CAP + 32 * REC);
    static constexpr int WARP_INTS = CPW * 32;
};

template <int DIM>
__host__ __device__ constexpr size_t win_smem(int warps)
{
    return (size_t)warps * (WinCfg<DIM>::WARP_DOUBLES * sizeof(double) + WinCfg<DIM>::WARP_INTS * sizeof(int));
}

// box entry i -> unwrapped offsets (x, y, z) inside a box of extents e (exact for the
// box sizes used: i < 2^20)
template <int DIM>
__device__ __forceinline__ void win_unflat(int i, const int e[3], float r0, float r01, int& x, int& y, int& z)
{
    if (DIM == 3) {
        z = (int)((float)i * r01 + 0.5f * r01);
        const int rem = i - z * e[0] * e[1];
        y = (int)((float)rem * r0 + 0.5f * r0);
        x = rem - y * e[0];
    } else {
        z = 0;
        y = (int)((float)i * r0 + 0.5f * r0);
        x = i - y * e[0];
    }
}

// window bounding box of the lanes' base nodes (unwrapped); false if it does not fit
template <int DIM, int CAP>
__device__ __forceinline__ bool win_box(const int bl[3], bool valid, int n, int o[3], int e[3], int& V)
{
    const unsigned FULL = 0xffffffffu;
    bool ok = true;
    V = 1;
#pragma unroll
    for (int a = 0; a < DIM; ++a) {
        const int lo = __reduce_min_sync(FULL, valid ? bl[a] : INT_MAX);
        const int hi = __reduce_max_sync(FULL, valid ? bl[a] : INT_MIN);
        o[a] = lo;
        e[a] = (hi >= lo) ? hi - lo + 4 : 1;
        ok = ok && e[a] <= CAP && e[a] <= n;
    }
    if (!ok) return false;
#pragma unroll
    for (int a = 0; a < DIM; ++a) V *= e[a];
    return V <= CAP;
}

template <int DIM, int KER, bool KEEP, bool PART>
__global__ void __launch_bounds__(256) k_spread_win(const double* __restrict__ Xh, const double* __restrict__ F,
                                                    const double* __restrict__ wgt, double* __restrict__ g0,
                                                    double* __restrict__ g1, double* __restrict__ g2,
                                                    double* __restrict__ f0, double* __restrict__ f1,
                                                    double* __restrict__ f2, int64_t npts, int n, double invh,
                                                    double invhd, double two_rho, const int* __restrict__ list,
                                                    const int* __restrict__ count, int z0, int nzl)
{
    using W = WinCfg<DIM>;
    constexpr int CPW = W::CPW, CAP = W::CAP, REC = W::REC;
    extern __shared__ double wsm[];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    double* box = wsm + (size_t)wib * W::WARP_DOUBLES;          // [CPW][CAP]
    double* rec = box + CPW * CAP;                              // [CPW][32][REC]
    int* rel = (int*)(wsm + (size_t)(blockDim.x >> 5) * W::WARP_DOUBLES) + wib * W::WARP_INTS;   // [CPW][32]
    const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t win = gw / W::WPW;
    const int cw = (int)(gw - win * W::WPW);
    const int64_t nitem = PART ? (int64_t)*count : npts;
    if (win * 32 >= nitem) return;                              // warp-uniform
    const int64_t item = win * 32 + lane;
    bool valid = item < nitem;
    int64_t k = valid ? item : 0;
    if (PART && valid) {
        k = list[item];
        if (k < 0) { valid = false; k = 0; }     // padding of a warp-aligned chunk (k_slab_select)
    }
    double Xk[3] = {0, 0, 0};
    double ws = 0.0;
    if (valid) {
#pragma unroll
        for (int a = 0; a < DIM; ++a) Xk[a] = Xh[k * DIM + a];
        ws = wgt[k] * invhd;
    }
    const size_t nn = (size_t)n;
    int bl[CPW][3], o[CPW][3], e[CPW][3], V[CPW], myrel[CPW];
    double w[CPW][3][4];
    bool fits[CPW];
#pragma unroll
    for (int q = 0; q < CPW; ++q) {
        const int c = (DIM == 3) ? cw : q;
        bl[q][2] = 0;
#pragma unroll
        for (int a = 0; a < DIM; ++a) weights4u<KER>(Xk[a] * invh - (a == c ? 0.0 : 0.5), bl[q][a], w[q][a]);
        const double Fs = valid ? F[k * DIM + c] * ws : 0.0;
#pragma unroll
        for (int m = 0; m < 4; ++m) w[q][0][m] *= Fs;
        fits[q] = win_box<DIM, CAP>(bl[q], valid, n, o[q], e[q], V[q]);
        myrel[q] = -1;
        if (fits[q]) {
            double* R = rec + (q * 32 + lane) * REC;
#pragma unroll
            for (int a = 0; a < DIM; ++a)
#pragma unroll
                for (int m = 0; m < 4; ++m) R[4 * a + ((a == 2) ? ((m & 1) * 2 + (m >> 1)) : m)] = w[q][a][m];
            myrel[q] = valid ? (bl[q][0] - o[q][0]) + e[q][0] * ((bl[q][1] - o[q][1]) +
                                                               (DIM == 3 ? e[q][1] * (bl[q][2] - o[q][2]) : 0)) : -1;
            rel[q * 32 + lane] = myrel[q];
            for (int i = lane; i < V[q]; i += 32) box[q * CAP + i] = 0.0;
        }
    }
    __syncwarp();
    // accumulate: the lanes own distinct nodes of a support.  3D: the window's points are
    // taken in groups with the same base node (ballot), whose contributions to the lane's
    // two nodes sum in registers; one read-modify-write of the box per group (a window of
    // 32 points has ~9 distinct base nodes at config 4).  The record holds w_z as
    // (w0, w2, w1, w3): lane dz reads its pair (w_dz, w_dz+2) with one 16-byte load.
    if (DIM == 3) {
        if (fits[0]) {
            const int dx = lane & 3, dy = (lane >> 2) & 3, dz = lane >> 4;
            const int e01 = e[0][0] * e[0][1];
            const int loff = dx + e[0][0] * dy + e01 * dz;
            const int st2 = 2 * e01;
            unsigned pend = __ballot_sync(0xffffffffu, valid);
            while (pend) {
                const int p0 = __ffs(pend) - 1;
                const int r0 = __shfl_sync(0xffffffffu, myrel[0], p0);
                const unsigned grp = __ballot_sync(0xffffffffu, myrel[0] == r0) & pend;
                pend &= ~grp;
                double a0 = 0.0, a1 = 0.0;
                for (unsigned g = grp; g; g &= g - 1) {
                    const double* R = rec + (__ffs(g) - 1) * REC;
                    const double2 wz = *reinterpret_cast<const double2*>(R + 8 + 2 * dz);
                    const double a = R[dx] * R[4 + dy];
                    a0 = fma(a, wz.x, a0);
                    a1 = fma(a, wz.y, a1);
                }
                box[r0 + loff] += a0;
                box[r0 + loff + st2] += a1;
                __syncwarp();
            }
        }
    } else {
        const int h = lane >> 4, j = lane & 15;
        const int dx = j & 3, dy = j >> 2;
        const bool fh = h ? fits[CPW - 1] : fits[0];
        const int eh = h ? e[CPW - 1][0] : e[0][0];
        const int loff = dx + eh * dy;
        double* bh = box + h * CAP;
        const double* rh = rec + h * 32 * REC;
        const int* relh = rel + h * 32;
        for (int p = 0; p < 32; ++p) {
            const int r = relh[p];                      // -1: no point in this lane
            if (fh && r >= 0) {
                const double* R = rh + p * REC;
                bh[r + loff] += R[dx] * R[4 + dy];
            }
            __syncwarp();
        }
    }
    // flush: one reduction per non-zero box entry; fall back to direct reductions
#pragma unroll
    for (int q = 0; q < CPW; ++q) {
        const int c = (DIM == 3) ? cw : q;
        double* gc = (c == 0) ? g0 : (c == 1 ? g1 : g2);
        double* fc = (c == 0) ? f0 : (c == 1 ? f1 : f2);
        if (fits[q]) {
            int wo[3] = {0, 0, 0};
#pragma unroll
            for (int a = 0; a < DIM; ++a) wo[a] = wrapm(o[q][a], n);
            const float r0 = 1.0f / (float)e[q][0];
            const float r01 = 1.0f / (float)(e[q][0] * e[q][1]);
            for (int i = lane; i < V[q]; i += 32) {
                const double v = box[q * CAP + i];
                if (v == 0.0) continue;
                int x, y, z;
                win_unflat<DIM>(i, e[q], r0, r01, x, y, z);
                int gx = wo[0] + x, gy = wo[1] + y, gz = wo[2] + z;
                if (gx >= n) gx -= n;
                if (gy >= n) gy -= n;
                if (gz >= n) gz -= n;
                int ll = (DIM == 3) ? gz : gy;                  // the last axis
                if (PART) {
                    ll -= z0;
                    if ((unsigned)ll >= (unsigned)nzl) continue;
                }
                const size_t qa = (DIM == 3) ? nn * (nn * (size_t)ll + gy) + gx : nn * (size_t)ll + gx;
                atomicAdd(gc + qa, two_rho * v);
                if (KEEP) atomicAdd(fc + qa, v);
            }
        } else if (valid) {
            int wb[3] = {0, 0, 0};
#pragma unroll
            for (int a = 0; a < DIM; ++a) wb[a] = wrapm(bl[q][a], n);
            const int m2n = (DIM == 3) ? 4 : 1;
            for (int m2 = 0; m2 < m2n; ++m2) {
                const int gz = (DIM == 3) ? wrap1(wb[2] + m2, n) : 0;
#pragma unroll
                for (int m1 = 0; m1 < 4; ++m1) {
                    const int gy = wrap1(wb[1] + m1, n);
                    int ll = (DIM == 3) ? gz : gy;
                    if (PART) {
                        ll -= z0;
                        if ((unsigned)ll >= (unsigned)nzl) continue;
                    }
                    const double a1 = w[q][1][m1] * ((DIM == 3) ? w[q][2][m2] : 1.0);
#pragma unroll
                    for (int m0 = 0; m0 < 4; ++m0) {
                        const int gx = wrap1(wb[0] + m0, n);
                        const size_t qa = (DIM == 3) ? nn * (nn * (size_t)ll + gy) + gx : nn * (size_t)ll + gx;
                        const double v = a1 * w[q][0][m0];
                        atomicAdd(gc + qa, two_rho * v);
                        if (KEEP) atomicAdd(fc + qa, v);
                    }
                }
            }
        }
    }
}

// Window-staged interpolation + Steps 1b-1c.  3D: a 192-thread block = 2 windows x 3
// components (warp = window x component); the block barrier orders every read of X^n
// before the writes of X^{n+1} (all components of a point are in the block).  2D: a warp
// = one window, both components (boxes [2][CAP]), each lane owns one point.
// PART (z-slab, slab.cu): the items are the listed points (warp-aligned chunks, -1 =
// none), the box holds only the nodes of this slab's planes z0 .. z0+nzl-1 (0 elsewhere),
// and the partial sums go to Upart (U^n = their sum over the slabs; no Steps 1b-1c).
template <int DIM, int KER, bool PART>
__global__ void __launch_bounds__(256) k_interp_win(const double* __restrict__ u0, const double* __restrict__ u1,
                                                    const double* __restrict__ u2, double* __restrict__ X,
                                                    double* __restrict__ Xh, double* __restrict__ Uprev,
                                                    double* __restrict__ Xold, double* __restrict__ Uold,
                                                    int64_t npts, int n, double invh, double dt, int first,
                                                    double* __restrict__ Upart, const int* __restrict__ list,
                                                    const int* __restrict__ count, int z0, int nzl)
{
    using W = WinCfg<DIM>;
    constexpr int CPW = W::CPW, CAP = W::CAP;
    extern __shared__ double wsm[];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    double* box = wsm + (size_t)wib * CPW * CAP;
    const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t win = gw / W::WPW;
    const int cw = (int)(gw - win * W::WPW);
    const int64_t nitem = PART ? (int64_t)*count : npts;
    const int64_t item = win * 32 + lane;
    bool valid = item < nitem;
    int64_t k = item;
    if (PART && valid) {
        k = list[item];
        valid = k >= 0;
    }
    double Xk[3] = {0, 0, 0};
    if (valid)
#pragma unroll
        for (int a = 0; a < DIM; ++a) Xk[a] = X[k * DIM + a];
    if (DIM == 3 && !PART) __syncthreads();   // every X^n read of the block precedes any X^{n+1} write
    if (win * 32 >= nitem) return;            // warp-uniform
    const size_t nn = (size_t)n;
#pragma unroll
    for (int q = 0; q < CPW; ++q) {
        const int c = (DIM == 3) ? cw : q;
        const double* uc = (c == 0) ? u0 : (c == 1 ? u1 : u2);
        int bl[3] = {0, 0, 0}, o[3], e[3], V;
        double w[3][4];
#pragma unroll
        for (int a = 0; a < DIM; ++a) weights4u<KER>(Xk[a] * invh - (a == c ? 0.0 : 0.5), bl[a], w[a]);
        const bool fits = win_box<DIM, CAP>(bl, valid, n, o, e, V);
        double acc = 0.0;
        if (fits) {
            double* bq = box + q * CAP;
            int wo[3] = {0, 0, 0};
#pragma unroll
            for (int a = 0; a < DIM; ++a) wo[a] = wrapm(o[a], n);
            const float r0 = 1.0f / (float)e[0];
            const float r01 = 1.0f / (float)(e[0] * e[1]);
            for (int i = lane; i < V; i += 32) {
                int x, y, z;
                win_unflat<DIM>(i, e, r0, r01, x, y, z);
                int gx = wo[0] + x, gy = wo[1] + y, gz = wo[2] + z;
                if (gx >= n) gx -= n;
                if (gy >= n) gy -= n;
                if (gz >= n) gz -= n;
                if (PART) {
                    const int l = ((DIM == 3) ? gz : gy) - z0;      // local plane of the last axis
                    bq[i] = ((unsigned)l < (unsigned)nzl)
                                ? __ldg(uc + ((DIM == 3) ? nn * (nn * (size_t)l + gy) + gx : nn * (size_t)l + gx))
                                : 0.0;
                } else {
                    bq[i] = __ldg(uc + ((DIM == 3) ? nn * (nn * (size_t)gz + gy) + gx : nn * (size_t)gy + gx));
                }
            }
            __syncwarp();
            if (valid) {
                const int rx = bl[0] - o[0], ry = bl[1] - o[1], rz = (DIM == 3) ? bl[2] - o[2] : 0;
                const double* b0 = bq + rx + e[0] * (ry + e[1] * rz);
                const int m2n = (DIM == 3) ? 4 : 1;
#pragma unroll
                for (int m2 = 0; m2 < m2n; ++m2) {
                    double pa = 0.0;
#pragma unroll
                    for (int m1 = 0; m1 < 4; ++m1) {
                        const double* row = b0 + e[0] * (m1 + e[1] * m2);
                        double r = 0.0;
#pragma unroll
                        for (int m0 = 0; m0 < 4; ++m0) r += w[0][m0] * row[m0];
                        pa += w[1][m1] * r;
                    }
                    acc += (DIM == 3) ? w[2][m2] * pa : pa;
                }
            }
            __syncwarp();
        } else if (valid) {
            int wb[3] = {0, 0, 0};
#pragma unroll
            for (int a = 0; a < DIM; ++a) wb[a] = wrapm(bl[a], n);
            const int m2n = (DIM == 3) ? 4 : 1;
#pragma unroll
            for (int m2 = 0; m2 < m2n; ++m2) {
                int lz = (DIM == 3) ? wrap1(wb[2] + m2, n) : 0;
                if (PART && DIM == 3) {
                    lz -= z0;
                    if ((unsigned)lz >= (unsigned)nzl) continue;
                }
                const size_t pl = (DIM == 3) ? nn * nn * (size_t)lz : 0;
                double pa = 0.0;
#pragma unroll
                for (int m1 = 0; m1 < 4; ++m1) {
                    int ly = wrap1(wb[1] + m1, n);
                    if (PART && DIM == 2) {
                        ly -= z0;
                        if ((unsigned)ly >= (unsigned)nzl) continue;
                    }
                    const size_t row = pl + nn * (size_t)ly;
                    double r = 0.0;
#pragma unroll
                    for (int m0 = 0; m0 < 4; ++m0) r += w[0][m0] * __ldg(uc + row + wrap1(wb[0] + m0, n));
                    pa += w[1][m1] * r;
                }
                acc += (DIM == 3) ? w[2][m2] * pa : pa;
            }
        }
        if (PART) {
            if (valid) Upart[k * DIM + c] = acc;
        } else if (valid) {
            // Steps 1b-1c for component c of this point
            const double xc = (c == 0) ? Xk[0] : (c == 1 ? Xk[1] : Xk[2]);
            const double up = Uprev[k * DIM + c];
            const double xn = first ? xc + dt * acc : xc + dt * (1.5 * acc - 0.5 * up);
            Xh[k * DIM + c] = 0.5 * (xn + xc);
            X[k * DIM + c] = xn;
            Uprev[k * DIM + c] = acc;
            Xold[k * DIM + c] = xc;
            Uold[k * DIM + c] = up;
        }
    }
}

// Step 1a restricted to the nodes of one z-slab (slab.cu): one thread per (listed point,
// component), 64 points per 64*DIM block; the partial sums over ranks form U^n.
template <int DIM, int KER>
__global__ void __launch_bounds__(64 * DIM) k_interp_comp_part(const double* __restrict__ u0,
                                                             const double* __restrict__ u1,
                                                             const double* __restrict__ u2,
                                                             const double* __restrict__ X, double* __restrict__ Upart,
                                                             const int* __restrict__ list,
                                                             const int* __restrict__ count, int n, int z0, int nzl,
                                                             double invh)
{
    const int c = threadIdx.x >> 6;
    const int64_t i = blockIdx.x * 64LL + (threadIdx.x & 63);
    if (i >= *count) return;
    const int64_t k = list[i];
    if (k < 0) return;                  // padding of a warp-aligned chunk (k_slab_select)
    const double* uc = (c == 0) ? u0 : (c == 1 ? u1 : u2);
    const size_t nn = (size_t)n;
    int b[3] = {0, 0, 0};
    double w[3][4];
#pragma unroll
    for (int a = 0; a < DIM; ++a) {
        weights4u<KER>(X[k * DIM + a] * invh - (a == c ? 0.0 : 0.5), b[a], w[a]);
        b[a] = wrapm(b[a], n);
    }
    double acc = 0.0;
#pragma unroll
    for (int mL = 0; mL < 4; ++mL) {
        int iL = b[DIM - 1] + mL;
        if (iL >= n) iL -= n;
        const int l = iL - z0;
        if ((unsigned)l >= (unsigned)nzl) continue;
        double pa = 0.0;
        if (DIM == 2) {
#pragma unroll
            for (int m0 = 0; m0 < 4; ++m0) pa += w[0][m0] * __ldg(uc + nn * l + wrap1(b[0] + m0, n));
        } else {
#pragma unroll
            for (int m1 = 0; m1 < 4; ++m1) {
                const size_t row = nn * (nn * (size_t)l + (size_t)wrap1(b[1] + m1, n));
                double r = 0.0;
#pragma unroll
                for (int m0 = 0; m0 < 4; ++m0) r += w[0][m0] * __ldg(uc + row + wrap1(b[0] + m0, n));
                pa += w[1][m1] * r;
            }
        }
        acc += w[DIM - 1][mL] * pa;
    }
    Upart[k * DIM + c] = acc;
}

// list capacity of a slab selection: npts rounded up to k_slab_select's 128-thread blocks
static int64_t sel_cap(int64_t npts) { return (npts + 127) / 128 * 128; }

template <int ID, class K>
static cudaError_t box_attr(K kern, size_t sm);

cudaError_t launch_interp_part(Ctx* top, Ctx* s, double* Upart, const int* list, const int* count)
{
    if (s->dim == 3) {
        // window-staged (as on one GPU): 6 warps = 2 windows x 3 components per block
        const int64_t warps = ((sel_cap(top->npts) + 31) / 32) * 3;
        const unsigned nbk = (unsigned)((warps + 5) / 6);
        const size_t sm = (size_t)6 * WinCfg<3>::CAP * sizeof(double);
        const double invh = 1.0 / s->h;
#define IBGM_IWP(K)                                                                                          \
    do {                                                                                                     \
        const cudaError_t ae_ = box_attr<330 + K>(k_interp_win<3, K, true>, sm);                             \
        if (ae_ != cudaSuccess) return ae_;                                                                  \
        k_interp_win<3, K, true><<<nbk, 192, sm, s->stream>>>(s->u[0], s->u[1], s->u[2], top->X, nullptr,   \
                nullptr, nullptr, nullptr, top->npts, (int)s->n, invh, 0.0, 0, Upart, list, count, (int)s->z0, (int)s->nl); \
    } while (0)
        if (top->kernel == IB_DELTA_COS4) IBGM_IWP(0); else IBGM_IWP(1);
#undef IBGM_IWP
        s->launches++;
        return cudaGetLastError();
    }
    const unsigned nb = (unsigned)((sel_cap(top->npts) + 63) / 64);
    const double invh = 1.0 / s->h;
#define IBGM_ICP(D, K) k_interp_comp_part<D, K><<<nb, 64 * D, 0, s->stream>>>(s->u[0], s->u[1], s->u[2], top->X, Upart, \
        list, count, (int)s->n, (int)s->z0, (int)s->nl, invh)
    if (s->dim == 2) { if (top->kernel == IB_DELTA_COS4) IBGM_ICP(2, 0); else IBGM_ICP(2, 1); }
    else { if (top->kernel == IB_DELTA_COS4) IBGM_ICP(3, 0); else IBGM_ICP(3, 1); }
#undef IBGM_ICP
    s->launches++;
    return cudaGetLastError();
}

template <bool PART>
static cudaError_t launch_spread_win(Ctx* top, Ctx* s, const int* list, const int* count);

cudaError_t launch_spread_part(Ctx* top, Ctx* s, const int* list, const int* count)
{
    if (s->dim == 3) return launch_spread_win<true>(top, s, list, count);
    const int64_t thr = ((sel_cap(top->npts) + 7) / 8) * 8 * s->dim * 4;
    const unsigned nbk = (unsigned)((thr + 255) / 256);
    const double invh = 1.0 / s->h;
    const double invhd = (s->dim == 3) ? invh * invh * invh : invh * invh;
    const double two_rho = 2.0 / s->rho;
    const int red = (s->dim == 3) ? 1 : 0;
#define IBGM_SQP(D, K, KP) k_spread_quad<D, K, KP, true><<<nbk, 256, 0, s->stream>>>(top->Xh, top->F, top->wgt, \
        s->nprev[0], s->nprev[1], s->nprev[2], s->f[0], s->f[1], s->f[2], top->npts, (int)s->n, invh, invhd, two_rho, \
        red, list, count, (int)s->z0, (int)s->nl)
    const bool kp = top->debug_keep_f != 0;
    if (s->dim == 2) {
        if (top->kernel == IB_DELTA_COS4) { if (kp) IBGM_SQP(2, 0, true); else IBGM_SQP(2, 0, false); }
        else { if (kp) IBGM_SQP(2, 1, true); else IBGM_SQP(2, 1, false); }
    } else {
        if (top->kernel == IB_DELTA_COS4) { if (kp) IBGM_SQP(3, 0, true); else IBGM_SQP(3, 0, false); }
        else { if (kp) IBGM_SQP(3, 1, true); else IBGM_SQP(3, 1, false); }
    }
#undef IBGM_SQP
    s->launches++;
    return cudaGetLastError();
}

// dst[idx[i]] = src[i] per point (internal -> caller order)
__global__ void k_scatter_pts(const double* __restrict__ src, const int32_t* __restrict__ idx, double* __restrict__ dst,
                              int64_t npts, int dim)
{
    const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e >= npts * dim) return;
    const int64_t k = e / dim;
    dst[(int64_t)idx[k] * dim + (e - k * dim)] = src[e];
}

__global__ void k_check_finite(const double* __restrict__ a, size_t cnt, int* __restrict__ flag)
{
    for (size_t q = blockIdx.x * (size_t)blockDim.x + threadIdx.x; q < cnt; q += (size_t)gridDim.x * blockDim.x)
        if (!isfinite(a[q])) { *(volatile int*)flag = 1; return; }
}

// X^{n+1} - X^{n+1/2} = (X^{n+1} - X^n)/2: a point that moved more than one cell h in a
// step (or a non-finite position) sets *flag (IB_EDOMAIN; "support stencil
// exceeds resident+halo region")
__global__ void k_check_domain(const double* __restrict__ X, const double* __restrict__ Xh, size_t cnt,
                               double half_h, int* __restrict__ flag)
{
    for (size_t q = blockIdx.x * (size_t)blockDim.x + threadIdx.x; q < cnt; q += (size_t)gridDim.x * blockDim.x)
        if (!(fabs(X[q] - Xh[q]) <= half_h)) { *(volatile int*)flag = 1; return; }
}

static unsigned nblk(int64_t cnt, int thr) { return (unsigned)((cnt + thr - 1) / thr); }

static size_t box_smem(int dim) { return (size_t)dim * (dim == 3 ? BoxCap<3>::VOL : BoxCap<2>::VOL) * sizeof(double); }
static size_t spread_smem(int dim)
{
    return (dim == 3 ? spread_box_doubles<3>() : spread_box_doubles<2>()) * sizeof(double);
}

// opt in to the box's dynamic shared memory once per kernel instantiation (ID tells the
// instantiations apart: they share one function type)
template <int ID, class K>
static cudaError_t box_attr(K kern, size_t sm)
{
    static unsigned long long mask = 0;   // per instantiation (ID), per device
    return smem_attr_once(mask, kern, (int)sm);
}

cudaError_t launch_interp_evolve(Ctx* s, int first)
{
    if (s->npts == 0) return cudaSuccess;
    // auto: quad-lane in 2D (config 2 0.0762 -> 0.0748 ms/step; window-staged 0.0700),
    // window-staged in 3D (config 4 interp 169 -> 140 us, 4.730 -> 4.710 ms/step; config 3
    // 19.5 -> 17.7 us, 0.1695 -> 0.1680 ms/step, against one thread per (point, component))
    const int im = s->interp_mode ? s->interp_mode : (s->dim == 2 ? 3 : 5);
    if (im == 5) {
        // window-staged: 3D 6 warps (2 windows x 3 components), 2D 8 warps (8 windows)
        const int D = s->dim;
        const int wpb = (D == 3) ? 6 : 8;
        const int64_t warps = ((s->npts + 31) / 32) * (D == 3 ? 3 : 1);
        const unsigned nbk = (unsigned)((warps + wpb - 1) / wpb);
        const size_t sm = (size_t)wpb * (D == 3 ? WinCfg<3>::CPW * WinCfg<3>::CAP : WinCfg<2>::CPW * WinCfg<2>::CAP) *
                          sizeof(double);
        const double invh = 1.0 / s->h;
#define IBGM_IW(Dd, K)                                                                                           \
    do {                                                                                                         \
        const cudaError_t ae_ = box_attr<300 + 10 * Dd + K>(k_interp_win<Dd, K, false>, sm);                    \
        if (ae_ != cudaSuccess) return ae_;                                                                      \
        k_interp_win<Dd, K, false><<<nbk, 32 * wpb, sm, s->stream>>>(s->u[0], s->u[1], s->u[2], s->X, s->Xh,     \
                s->Uprev, s->Xold, s->Uold, s->npts, (int)s->n, invh, s->dt, first, nullptr, nullptr, nullptr, 0, 0); \
    } while (0)
        if (D == 2) { if (s->kernel == IB_DELTA_COS4) IBGM_IW(2, 0); else IBGM_IW(2, 1); }
        else { if (s->kernel == IB_DELTA_COS4) IBGM_IW(3, 0); else IBGM_IW(3, 1); }
#undef IBGM_IW
        s->launches++;
        return cudaGetLastError();
    }
    if (im == 3) {
        // a block holds whole 8-point groups of every component (32 DIM threads each):
        // 256 threads in 2D, 192 in 3D, so the X^n reads of all components of a point
        // precede its X^{n+1} writes (barrier in the kernel)
        const int bs = s->dim == 3 ? 192 : 256;
        const int64_t thr = ((s->npts + 7) / 8) * 8 * s->dim * 4;
        const unsigned nbk = (unsigned)((thr + bs - 1) / bs);
        const double invh = 1.0 / s->h;
#define IBGM_IQ(D, K) k_interp_quad<D, K><<<nbk, bs, 0, s->stream>>>(s->u[0], s->u[1], s->u[2], s->X, s->Xh, \
                                                                      s->Uprev, s->Xold, s->Uold, s->npts, (int)s->n, invh, \
                                                                      s->dt, first)
        if (s->dim == 2) { if (s->kernel == IB_DELTA_COS4) IBGM_IQ(2, 0); else IBGM_IQ(2, 1); }
        else { if (s->kernel == IB_DELTA_COS4) IBGM_IQ(3, 0); else IBGM_IQ(3, 1); }
#undef IBGM_IQ
        s->launches++;
        return cudaGetLastError();
    }
    if (im == 2) {
        const unsigned nbk = (unsigned)((s->npts + kBoxPts - 1) / kBoxPts);
        const size_t sm = box_smem(s->dim);
        const double invh = 1.0 / s->h;
#define IBGM_IB(D, K)                                                                                   \
    do {                                                                                                \
        const cudaError_t ae_ = box_attr<10 * D + K>(k_interp_box<D, K>, sm);                                         \
        if (ae_ != cudaSuccess) return ae_;                                                             \
        k_interp_box<D, K><<<nbk, kBoxPts * D, sm, s->stream>>>(s->u[0], s->u[1], s->u[2], s->X, s->Xh, \
                                                                    s->Uprev, s->Xold, s->Uold, s->npts, (int)s->n, invh, s->dt, first); \
    } while (0)
        if (s->dim == 2) { if (s->kernel == IB_DELTA_COS4) IBGM_IB(2, 0); else IBGM_IB(2, 1); }
        else { if (s->kernel == IB_DELTA_COS4) IBGM_IB(3, 0); else IBGM_IB(3, 1); }
#undef IBGM_IB
        s->launches++;
        return cudaGetLastError();
    }
    const double invh = 1.0 / s->h;
    if (im == 4) {
        const unsigned nb = (unsigned)((s->npts + 63) / 64);
#define IBGM_IC(D, K) k_interp_comp<D, K><<<nb, 64 * D, 0, s->stream>>>(s->u[0], s->u[1], s->u[2], s->X, s->Xh, \
        s->Uprev, s->Xold, s->Uold, s->npts, (int)s->n, invh, s->dt, first)
        if (s->dim == 2) { if (s->kernel == IB_DELTA_COS4) IBGM_IC(2, 0); else IBGM_IC(2, 1); }
        else { if (s->kernel == IB_DELTA_COS4) IBGM_IC(3, 0); else IBGM_IC(3, 1); }
#undef IBGM_IC
        s->launches++;
        return cudaGetLastError();
    }
    const int thr = 128;
#define IBGM_IE(D, K) launch_pdl_if(D == 2, k_interp_evolve<D, K>, dim3(nblk(s->npts, thr)), dim3(thr), 0, s->stream, \
        s->u[0], s->u[1], s->u[2], s->X, s->Xh, s->Uprev, s->Xold, s->Uold, s->npts, (int)s->n, invh, s->dt, first)
    if (s->dim == 2) { if (s->kernel == IB_DELTA_COS4) IBGM_IE(2, 0); else IBGM_IE(2, 1); }
    else { if (s->kernel == IB_DELTA_COS4) IBGM_IE(3, 0); else IBGM_IE(3, 1); }
#undef IBGM_IE
    s->launches++;
    return cudaGetLastError();
}

cudaError_t launch_force(Ctx* s)
{
    if (s->npts == 0) return cudaSuccess;
    const int thr = 128;
    if (s->dim == 2)
        launch_pdl_if(true, k_force<2>, dim3(nblk(s->npts, thr)), dim3(thr), 0, s->stream, s->Xh, s->csr_ptr, s->csr_nbr,
                   s->csr_kappa, s->csr_rest, s->has_rest, s->F, s->npts, s->H, 1.0 / s->H, s->err_d);
    else
        launch_pdl_if(false, k_force<3>, dim3(nblk(s->npts, thr)), dim3(thr), 0, s->stream, s->Xh, s->csr_ptr, s->csr_nbr,
                   s->csr_kappa, s->csr_rest, s->has_rest, s->F, s->npts, s->H, 1.0 / s->H, s->err_d);
    s->launches++;
    return cudaGetLastError();
}

static size_t brick_smem(int dim, int B)
{
    const int T = B + 4;
    const int TV = (dim == 3) ? T * T * T : T * T;
    const int CH = 128;
    return (size_t)(dim * TV + CH * dim * dim * 4 + CH * dim) * sizeof(double) + (size_t)CH * dim * dim * sizeof(int);
}

constexpr int kBrick3 = 4, kBrick2 = 8;

template <int DIM, int KER, int B, bool KEEP>
static cudaError_t go_brick_spread(Ctx* s)
{
    auto kern = k_brick_spread<DIM, KER, B, KEEP>;
    const size_t sm = brick_smem(DIM, B);
    static unsigned long long attr = 0;
    {
        const cudaError_t e = smem_attr_once(attr, kern, (int)sm);
        if (e != cudaSuccess) return e;
    }
    const double invh = 1.0 / s->h;
    const double invhd = (DIM == 3) ? invh * invh * invh : invh * invh;
    const int64_t cap = 148 * 16;
    int grid = (int)(s->nbricks < cap ? s->nbricks : cap);
    if (grid < 1) grid = 1;
    kern<<<grid, 256, sm, s->stream>>>(s->Xh, s->F, s->wgt, s->bin_sorted, s->bin_start, s->bin_count, s->bin_list,
                                       s->bin_nlist, s->nprev[0], s->nprev[1], s->nprev[2], s->f[0], s->f[1], s->f[2],
                                       (int)s->n, s->nb, invh, invhd, 2.0 / s->rho);
    s->launches++;
    return cudaGetLastError();
}

static cudaError_t launch_spread_direct(Ctx* s)
{
    const int thr = 128;
    const double invh = 1.0 / s->h;
    const double invhd = (s->dim == 3) ? invh * invh * invh : invh * invh;
    const double two_rho = 2.0 / s->rho;
#define IBGM_SP(D, K, KP) k_spread<D, K, KP><<<nblk(s->npts, thr), thr, 0, s->stream>>>( \
        s->Xh, s->F, s->wgt, s->nprev[0], s->nprev[1], s->nprev[2], s->f[0], s->f[1], s->f[2], s->npts, \
        (int)s->n, invh, invhd, two_rho)
    const bool kp = s->debug_keep_f != 0;
    if (s->dim == 2) {
        if (s->kernel == IB_DELTA_COS4) { if (kp) IBGM_SP(2, 0, true); else IBGM_SP(2, 0, false); }
        else { if (kp) IBGM_SP(2, 1, true); else IBGM_SP(2, 1, false); }
    } else {
        if (s->kernel == IB_DELTA_COS4) { if (kp) IBGM_SP(3, 0, true); else IBGM_SP(3, 0, false); }
        else { if (kp) IBGM_SP(3, 1, true); else IBGM_SP(3, 1, false); }
    }
#undef IBGM_SP
    s->launches++;
    return cudaGetLastError();
}

static cudaError_t launch_spread_box(Ctx* s)
{
    const unsigned nbk = (unsigned)((s->npts + kBoxPts - 1) / kBoxPts);
    const size_t sm = spread_smem(s->dim);
    const double invh = 1.0 / s->h;
    const double invhd = (s->dim == 3) ? invh * invh * invh : invh * invh;
    const double two_rho = 2.0 / s->rho;
#define IBGM_SB(D, K, KP)                                                                                  \
    do {                                                                                                   \
        const cudaError_t ae_ = box_attr<100 + 10 * D + 2 * K + KP>(k_spread_box<D, K, KP>, sm);                                      \
        if (ae_ != cudaSuccess) return ae_;                                                                \
        k_spread_box<D, K, KP><<<nbk, kBoxPts * D, sm, s->stream>>>(s->Xh, s->F, s->wgt, s->nprev[0],   \
                s->nprev[1], s->nprev[2], s->f[0], s->f[1], s->f[2], s->npts, (int)s->n, invh, invhd, two_rho); \
    } while (0)
    const bool kp = s->debug_keep_f != 0;
    if (s->dim == 2) {
        if (s->kernel == IB_DELTA_COS4) { if (kp) IBGM_SB(2, 0, true); else IBGM_SB(2, 0, false); }
        else { if (kp) IBGM_SB(2, 1, true); else IBGM_SB(2, 1, false); }
    } else {
        if (s->kernel == IB_DELTA_COS4) { if (kp) IBGM_SB(3, 0, true); else IBGM_SB(3, 0, false); }
        else { if (kp) IBGM_SB(3, 1, true); else IBGM_SB(3, 1, false); }
    }
#undef IBGM_SB
    s->launches++;
    return cudaGetLastError();
}

cudaError_t launch_scatter_pts(Ctx* s, const double* src, double* dst)
{
    const int64_t cnt = s->npts * s->dim;
    if (cnt == 0) return cudaSuccess;
    k_scatter_pts<<<nblk(cnt, 256), 256, 0, s->stream>>>(src, s->pt_user, dst, s->npts, s->dim);
    s->launches++;
    return cudaGetLastError();
}

static cudaError_t launch_spread_quad(Ctx* s)
{
    const int64_t thr = ((s->npts + 7) / 8) * 8 * s->dim * 4;
    const unsigned nbk = (unsigned)((thr + 255) / 256);
    const double invh = 1.0 / s->h;
    const double invhd = (s->dim == 3) ? invh * invh * invh : invh * invh;
    const double two_rho = 2.0 / s->rho;
    // mode 5: with the warp pre-reduction (config 4 spread 460 -> 348 us, config 3
    // 30.3 -> 24.9 us); 2D auto: without (no runs of equal base nodes on a curve)
    const int red = (s->spread_mode == 5) ? 1 : 0;
#define IBGM_SQ(D, K, KP) launch_pdl_if(D == 2, k_spread_quad<D, K, KP, false>, dim3(nbk), dim3(256), 0, s->stream, s->Xh, \
        s->F, s->wgt, s->nprev[0], s->nprev[1], s->nprev[2], s->f[0], s->f[1], s->f[2], s->npts, (int)s->n, invh, invhd, \
        two_rho, red, (const int*)nullptr, (const int*)nullptr, 0, 0)
    const bool kp = s->debug_keep_f != 0;
    if (s->dim == 2) {
        if (s->kernel == IB_DELTA_COS4) { if (kp) IBGM_SQ(2, 0, true); else IBGM_SQ(2, 0, false); }
        else { if (kp) IBGM_SQ(2, 1, true); else IBGM_SQ(2, 1, false); }
    } else {
        if (s->kernel == IB_DELTA_COS4) { if (kp) IBGM_SQ(3, 0, true); else IBGM_SQ(3, 0, false); }
        else { if (kp) IBGM_SQ(3, 1, true); else IBGM_SQ(3, 1, false); }
    }
#undef IBGM_SQ
    s->launches++;
    return cudaGetLastError();
}

// window-staged spreading (k_spread_win): 8 warps per block; PART: the listed points of
// a z-slab (top: the replicated Lagrangian data, s: the slab)
template <bool PART>
static cudaError_t launch_spread_win(Ctx* top, Ctx* s, const int* list, const int* count)
{
    const int D = s->dim;
    static int wpb = -1;             // warps per block (IBGM_WIN_WPB, A/B)
    if (wpb < 0) {
        const char* ev = getenv("IBGM_WIN_WPB");
        wpb = ev ? atoi(ev) : 8;
        if (wpb < 1 || wpb > 8) wpb = 8;
    }
    const int64_t items = PART ? sel_cap(top->npts) : top->npts;
    const int64_t warps = ((items + 31) / 32) * (D == 3 ? 3 : 1);
    const unsigned nbk = (unsigned)((warps + wpb - 1) / wpb);
    const size_t sm = (D == 3) ? win_smem<3>(wpb) : win_smem<2>(wpb);
    const double invh = 1.0 / s->h;
    const double invhd = (D == 3) ? invh * invh * invh : invh * invh;
    const double two_rho = 2.0 / s->rho;
    const bool kp = top->debug_keep_f != 0;
    const int z0 = PART ? (int)s->z0 : 0, nzl = PART ? (int)s->nl : 0;
#define IBGM_SW(Dd, K, KP)                                                                                  \
    do {                                                                                                    \
        const cudaError_t ae_ = box_attr<200 + 10 * Dd + 4 * K + 2 * KP + PART>(k_spread_win<Dd, K, KP, PART>, sm); \
        if (ae_ != cudaSuccess) return ae_;                                                                 \
        k_spread_win<Dd, K, KP, PART><<<nbk, 32 * wpb, sm, s->stream>>>(top->Xh, top->F, top->wgt, s->nprev[0],  \
                s->nprev[1], s->nprev[2], s->f[0], s->f[1], s->f[2], top->npts, (int)s->n, invh, invhd, two_rho, \
                list, count, z0, nzl);                                                                      \
    } while (0)
    if (D == 2) {
        if (top->kernel == IB_DELTA_COS4) { if (kp) IBGM_SW(2, 0, true); else IBGM_SW(2, 0, false); }
        else { if (kp) IBGM_SW(2, 1, true); else IBGM_SW(2, 1, false); }
    } else {
        if (top->kernel == IB_DELTA_COS4) { if (kp) IBGM_SW(3, 0, true); else IBGM_SW(3, 0, false); }
        else { if (kp) IBGM_SW(3, 1, true); else IBGM_SW(3, 1, false); }
    }
#undef IBGM_SW
    s->launches++;
    return cudaGetLastError();
}

cudaError_t launch_spread(Ctx* s)
{
    if (s->npts == 0) return cudaSuccess;
    // auto in 3D: window-staged (config 4 spread 354 -> 264 us, 4.854 -> 4.759 ms/step;
    // config 3 0.1727 -> 0.1709 ms/step); 2D keeps the quad-lane kernel (config 2:
    // 8.1 us vs 12.8 window-staged -- a curve gives short windows little overlap)
    if (s->spread_mode == 6 || (s->spread_mode == 0 && s->dim == 3)) return launch_spread_win<false>(s, s, nullptr, nullptr);
    // 0 (auto) and 4: quad-lane atomics; 1: per-point atomics; 2: brick-binned; 3: box-staged
    if (s->spread_mode == 0 || s->spread_mode == 4 || s->spread_mode == 5) return launch_spread_quad(s);   // 0: 2D
    if (s->spread_mode == 3) return launch_spread_box(s);
    if (s->spread_mode == 1) return launch_spread_direct(s);
    const int thr = 256;
    const double invh = 1.0 / s->h;
    cudaError_t e = cudaMemsetAsync(s->bin_count, 0, sizeof(int) * s->nbricks, s->stream);
    if (e != cudaSuccess) return e;
    if (s->dim == 3)
        k_bin_count<3, kBrick3><<<nblk(s->npts, thr), thr, 0, s->stream>>>(s->Xh, s->npts, (int)s->n, s->nb, invh,
                                                                          s->bin_bid, s->bin_count);
    else
        k_bin_count<2, kBrick2><<<nblk(s->npts, thr), thr, 0, s->stream>>>(s->Xh, s->npts, (int)s->n, s->nb, invh,
                                                                          s->bin_bid, s->bin_count);
    const int nparts = (int)((s->nbricks + kScanB - 1) / kScanB);
    k_scan_partial<<<nparts, kScanB, 0, s->stream>>>(s->bin_count, (int)s->nbricks, s->bin_partial);
    k_scan_top<<<1, kScanB, 0, s->stream>>>(s->bin_partial, nparts, s->bin_nlist);
    k_scan_final<<<nparts, kScanB, 0, s->stream>>>(s->bin_count, (int)s->nbricks, s->bin_partial, s->bin_start,
                                                   s->bin_cursor, s->bin_list, s->bin_nlist);
    k_bin_fill<<<nblk(s->npts, thr), thr, 0, s->stream>>>(s->bin_bid, s->npts, s->bin_start, s->bin_cursor,
                                                          s->bin_sorted);
    s->launches += 5;
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    const bool kp = s->debug_keep_f != 0;
    if (s->dim == 3) {
        if (s->kernel == IB_DELTA_COS4)
            return kp ? go_brick_spread<3, 0, kBrick3, true>(s) : go_brick_spread<3, 0, kBrick3, false>(s);
        return kp ? go_brick_spread<3, 1, kBrick3, true>(s) : go_brick_spread<3, 1, kBrick3, false>(s);
    }
    if (s->kernel == IB_DELTA_COS4)
        return kp ? go_brick_spread<2, 0, kBrick2, true>(s) : go_brick_spread<2, 0, kBrick2, false>(s);
    return kp ? go_brick_spread<2, 1, kBrick2, true>(s) : go_brick_spread<2, 1, kBrick2, false>(s);
}

cudaError_t launch_check_finite(Ctx* s, int* flag)
{
    const int thr = 256;
    if (s->nlocal > 0) {
        for (int c = 0; c < s->dim; ++c) {
            k_check_finite<<<592, thr, 0, s->stream>>>(s->u[c], (size_t)s->nlocal, flag);
            s->launches++;
        }
        k_check_finite<<<592, thr, 0, s->stream>>>(s->p, (size_t)s->nlocal, flag);
        s->launches++;
    }
    if (s->npts) {
        k_check_finite<<<592, thr, 0, s->stream>>>(s->X, (size_t)s->npts * s->dim, flag);
        s->launches++;
    }
    return cudaGetLastError();
}

cudaError_t launch_check_domain(Ctx* s, int* flag)
{
    if (s->npts == 0) return cudaSuccess;
    k_check_domain<<<nblk(s->npts * s->dim, 256), 256, 0, s->stream>>>(s->X, s->Xh, (size_t)s->npts * s->dim,
                                                                       0.5 * s->h, flag);
    s->launches++;
    return cudaGetLastError();
}

}  // namespace ibgm
