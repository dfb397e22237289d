// Immersed-boundary kernels of the IB-GM step (sm_100a, fp64): Steps 1a-1c and 2a-2b
// of PAPER.md:577-621.  Lagrangian arrays are point-major [npts][dim].
#include <cuda_runtime.h>

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
                                double* __restrict__ Uprev, int64_t npts, int n,
                                double invh, double dt, int first)
{
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
    }
}

// Step 2a: F_k = sum_{e=(k,m)} kappa_e (X_m - X_k)(1 - L_e/|X_m - X_k|) at X^{n+1/2}
// (PAPER.md:607-614 in the force-connection form of PAPER.md:856-861), gathered per
// point from a CSR adjacency (no atomics).
template <int DIM>
__global__ void k_force(const double* __restrict__ Xh, const int32_t* __restrict__ ptr,
                        const int32_t* __restrict__ nbr, const double* __restrict__ kap,
                        const double* __restrict__ rest, int has_rest, double* __restrict__ F, int64_t npts)
{
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
            l2 += d[a] * d[a];
        }
        double t = kap[e];
        if (has_rest) {
            const double L = rest[e];
            if (L != 0.0) t *= 1.0 - L / sqrt(l2);
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
__global__ void k_spread(const double* __restrict__ Xh, const double* __restrict__ F,
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

__global__ void k_check_finite(const double* __restrict__ a, size_t cnt, int* __restrict__ flag)
{
    for (size_t q = blockIdx.x * (size_t)blockDim.x + threadIdx.x; q < cnt; q += (size_t)gridDim.x * blockDim.x)
        if (!isfinite(a[q])) { atomicOr(flag, 1); return; }
}

static unsigned nblk(int64_t cnt, int thr) { return (unsigned)((cnt + thr - 1) / thr); }

cudaError_t launch_interp_evolve(Ctx* s, int first)
{
    if (s->npts == 0) return cudaSuccess;
    const int thr = 128;
    const double invh = 1.0 / s->h;
#define IBGM_IE(D, K) k_interp_evolve<D, K><<<nblk(s->npts, thr), thr, 0, s->stream>>>( \
        s->u[0], s->u[1], s->u[2], s->X, s->Xh, s->Uprev, s->npts, (int)s->n, invh, s->dt, first)
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
        k_force<2><<<nblk(s->npts, thr), thr, 0, s->stream>>>(s->Xh, s->csr_ptr, s->csr_nbr, s->csr_kappa,
                                                              s->csr_rest, s->has_rest, s->F, s->npts);
    else
        k_force<3><<<nblk(s->npts, thr), thr, 0, s->stream>>>(s->Xh, s->csr_ptr, s->csr_nbr, s->csr_kappa,
                                                              s->csr_rest, s->has_rest, s->F, s->npts);
    s->launches++;
    return cudaGetLastError();
}

cudaError_t launch_spread(Ctx* s)
{
    if (s->npts == 0) return cudaSuccess;
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

cudaError_t launch_check_finite(Ctx* s)
{
    const int thr = 256;
    cudaError_t e = cudaMemsetAsync(s->d_flag, 0, sizeof(int), s->stream);
    if (e != cudaSuccess) return e;
    for (int c = 0; c < s->dim; ++c) {
        k_check_finite<<<592, thr, 0, s->stream>>>(s->u[c], (size_t)s->ncell, s->d_flag);
        s->launches++;
    }
    k_check_finite<<<592, thr, 0, s->stream>>>(s->p, (size_t)s->ncell, s->d_flag);
    s->launches++;
    if (s->npts) {
        k_check_finite<<<592, thr, 0, s->stream>>>(s->X, (size_t)s->npts * s->dim, s->d_flag);
        s->launches++;
    }
    return cudaGetLastError();
}

}  // namespace ibgm
