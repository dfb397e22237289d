// Z-slab decomposition of the IB-GM step, sm_100a, fp64.
//
// The grid is cut along its last axis (z in 3D, y in 2D) into P slabs of nz = N/P
// planes; slab s owns global planes [s nz, (s+1) nz).  Every field keeps one halo plane
// on each side (planes -1 and nz), which is all the stencils of Steps 3b/3e need
// (PAPER.md:807-833).  The Lagrangian data is replicated on every rank:
//   - interpolation (Step 1a): each rank sums the delta-weighted velocities of the grid
//     nodes it owns; one all-reduce over ranks forms U^n, then every rank evolves all
//     points identically (Steps 1b-1c);
//   - spreading (Step 2b): each rank spreads every point into the nodes it owns only,
//     so no reverse halo sum is needed.
// Lines along x and y lie inside a slab and use the single-GPU line kernels.  Lines
// along the cut axis are solved with the paper's Schur-complement splitting across
// ranks: slab s is part s of every line -- its first plane is the
// interface unknown y_s and planes 1..nz-1 are the interior block B_s.  Each rank
// solves B_s f*_s = d_s (Thomas, one thread per line, coalesced across x), publishes
// per line the scalars the reduced system needs to that line's master rank (line index
// mod P, as in the paper's PAPER.md:1270-1276), the master applies the precomputed
// S^{-1} and sends each rank back only its y_s, y_{s+1} and the line-mean correction,
// and each rank corrects x_s = f*_s - B_s^{-1} E_s y.
//
// Two transports move the halo planes, the reduced system and the partial U:
//   EMULATE  P virtual slabs in one context on one GPU (device-to-device copies and
//            shared exchange buffers) -- the same kernels in the same order, used to
//            test the decomposition at the parity bar with a single GPU;
//   NCCL     one slab per process (one process per GPU), grouped ncclSend/ncclRecv for
//            halos and for the two all-to-alls of the reduced system (scalars to the
//            masters, y values back), ncclAllReduce for U.  NCCL is
//            loaded at run time (the copy torch already loaded if present).
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>

#include <algorithm>

#include "ibgm_internal.cuh"

namespace ibgm {

// ------------------------------------------------------------------------------------
// NCCL, loaded at run time (minimal ABI: ncclUniqueId is 128 bytes, enums are int)
// ------------------------------------------------------------------------------------
struct NcclApi {
    bool ok = false;
    int (*GetUniqueId)(NcclUid*) = nullptr;
    int (*CommInitRank)(void**, int, NcclUid, int) = nullptr;
    int (*CommDestroy)(void*) = nullptr;
    int (*AllReduce)(const void*, void*, size_t, int, int, void*, cudaStream_t) = nullptr;
    int (*AllGather)(const void*, void*, size_t, int, void*, cudaStream_t) = nullptr;
    int (*Send)(const void*, size_t, int, int, void*, cudaStream_t) = nullptr;
    int (*Recv)(void*, size_t, int, int, void*, cudaStream_t) = nullptr;
    int (*CommSplit)(void*, int, int, void**, void*) = nullptr;   // optional (NCCL >= 2.18)
    int (*GroupStart)() = nullptr;
    int (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(int) = nullptr;
};
constexpr int kNcclDouble = 8, kNcclSum = 0;

static NcclApi g_nccl;

const char* nccl_load(void)
{
    static char err[256] = "";
    if (g_nccl.ok) return nullptr;
    void* h = nullptr;
    const char* env = getenv("IBGM_NCCL_LIB");
    if (env && *env) h = dlopen(env, RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);   // the copy torch loaded
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
        snprintf(err, sizeof(err), "cannot load libnccl.so.2: %s", dlerror());
        return err;
    }
#define IBGM_SYM(field, name)                                             \
    g_nccl.field = reinterpret_cast<decltype(g_nccl.field)>(dlsym(h, name)); \
    if (!g_nccl.field) {                                                  \
        snprintf(err, sizeof(err), "libnccl.so.2 lacks %s", name);        \
        return err;                                                       \
    }
    IBGM_SYM(GetUniqueId, "ncclGetUniqueId");
    IBGM_SYM(CommInitRank, "ncclCommInitRank");
    IBGM_SYM(CommDestroy, "ncclCommDestroy");
    IBGM_SYM(AllReduce, "ncclAllReduce");
    IBGM_SYM(AllGather, "ncclAllGather");
    IBGM_SYM(Send, "ncclSend");
    IBGM_SYM(Recv, "ncclRecv");
    IBGM_SYM(GroupStart, "ncclGroupStart");
    IBGM_SYM(GroupEnd, "ncclGroupEnd");
    IBGM_SYM(GetErrorString, "ncclGetErrorString");
#undef IBGM_SYM
    g_nccl.CommSplit = reinterpret_cast<decltype(g_nccl.CommSplit)>(dlsym(h, "ncclCommSplit"));
    g_nccl.ok = true;
    return nullptr;
}

int nccl_unique_id(NcclUid* id) { return g_nccl.GetUniqueId(id); }
int nccl_comm_init(void** comm, int nranks, const NcclUid* id, int rank) { return g_nccl.CommInitRank(comm, nranks, *id, rank); }
void nccl_comm_destroy(void* comm) { if (comm && g_nccl.ok) g_nccl.CommDestroy(comm); }
int nccl_comm_split(void* comm, int rank, void** out)
{
    if (!g_nccl.ok || !g_nccl.CommSplit) return -1;
    return g_nccl.CommSplit(comm, 0, rank, out, nullptr);
}
const char* nccl_error_string(int rc) { return g_nccl.ok ? g_nccl.GetErrorString(rc) : "nccl not loaded"; }

// ------------------------------------------------------------------------------------
// Slab line solve: device coefficient block (built on the host in long double by
// make_slab_coef): header, then inv[m], cp[m], g[m], h[m] of the interior block
// B = tridiag(c, a, b) of m = nz-1 unknowns, then S^{-1} (P x P) and its column sums.
// ------------------------------------------------------------------------------------
struct SlabCf {
    const double* p;
    int m, P;
    __device__ __forceinline__ double c() const { return p[SC_C]; }
    __device__ __forceinline__ double b() const { return p[SC_B]; }
    __device__ __forceinline__ const double* inv() const { return p + SC_HDR; }
    __device__ __forceinline__ const double* cp() const { return p + SC_HDR + m; }
    __device__ __forceinline__ const double* g() const { return p + SC_HDR + 2 * m; }
    __device__ __forceinline__ const double* h() const { return p + SC_HDR + 3 * m; }
    __device__ __forceinline__ const double* sinv() const { return p + SC_HDR + 4 * m; }
    __device__ __forceinline__ const double* colsum() const { return p + SC_HDR + 4 * m + P * P; }
};

enum SlabSrc { SRC_FIELD = 0, SRC_DIV = 1 };
enum SlabEpi { EPI_STORE = 0, EPI_ADD_UN = 1 };

struct SlabArgs {
    double* io[3];            // per component: the slab field (plane-0 pointer)
    const double* un[3];      // u^n (EPI_ADD_UN; SRC_DIV)
    const double* unew[3];    // u^{n+1} (SRC_DIV)
    double* p;                // SRC_DIV: p -> q = p - chi mu D.(u^{n+1}+u^n)/2
    const double* divn;       // SRC_DIV: D.u^n written by S1 (else gathered from u^n)
    // reduced-system exchange with a master rank per line (m = line mod P)
    double* up_w;             // writer: this rank's block for master 0; + m * up_mstride for master m
    long long up_mstride;
    const double* up_r;       // master: [rank][Q][ns][nidx] it received (+ z * up_rmstride)
    long long up_rmstride;
    double* dn_w;             // master: block for rank 0; + r * dn_rstride for rank r (+ z * dn_wmstride)
    long long dn_rstride, dn_wmstride;
    const double* dn_r;       // rank: [master][comp][nb][nidx] it received
    int nidx;                 // lines per master = plane / P
    int nb;                   // values per rank, line and component returned: y_{rQ..rQ+Q}, corr
    double neg_rho_dt, chimu_half, invh;
    int n, nz, rank;
    int Q, Lseg;              // Schur parts per slab and their length (nz = Q Lseg)
    int ns;                   // gather slots per part of this solve (6 viscous: 2 per component; 4 psi)
    long long plane;          // N^{d-1}
    // visc_local (S^{-1} diagonal): this slab's scalars A_t, fm_t in edge_w [comp][Q][2][plane],
    // the neighbours' in edge_r [2][comp][plane] (fm of the part below, A of the part above)
    int local;
    double w0;
    double* edge_w;
    const double* edge_r;
};

// forward phase: interior Thomas solve of every line of this slab, in place (plane 0
// keeps d_0), and the per-line scalars of the reduced system:
//   A_s = d_{s,0} - b f*_{s,1},  fm_s = f*_{s,m},  (mean fix) D_s = sum d,  F_s = sum f*.
template <int DIM, int SRC, int MF>
__global__ void __launch_bounds__(128) k_slab_fwd(SlabCf C, SlabArgs A, int slot0)
{
    const long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (q >= A.plane) return;
    const int comp = blockIdx.y;
    const int k0 = blockIdx.z * A.Lseg;                  // first plane of this Schur part
    const int part = A.rank * A.Q + blockIdx.z;          // its index along the whole line
    double* io = ((comp == 0) ? A.io[0] : (comp == 1 ? A.io[1] : A.io[2])) + (long long)k0 * A.plane;
    const long long PL = A.plane;
    const int n = A.n;
    long long off[3] = {1, n, PL};      // +e_x, +e_y, +e_last (periodic in x, y within the slab)
    if (SRC == SRC_DIV) {
        const int i = (int)(q % n);
        if (i == n - 1) off[0] = -(long long)(n - 1);
        if (DIM == 3) {
            const int j = (int)(q / n);
            if (j == n - 1) off[1] = -(long long)(n - 1) * n;
        } else {
            off[1] = PL;                 // 2D: the cut axis is y
        }
    }
    auto src = [&](int kl) -> double {
        const long long f = kl * PL + q;
        if (SRC == SRC_FIELD) return io[f];
        // Step 3e RHS r = -(rho/dt) D.u^{n+1} and the explicit part of Step 3f
        // (PAPER.md:484-491, 668-683); the +e_last neighbour of plane nz-1 is the halo
        double dn = 0.0, dol = 0.0;
        const long long fg = f + (long long)k0 * PL;   // offset in the slab fields
#pragma unroll
        for (int c = 0; c < DIM; ++c) {
            const long long o = (c == DIM - 1) ? PL : off[c];
            dn += A.unew[c][fg + o] - A.unew[c][fg];
            if (!A.divn) dol += A.un[c][fg + o] - A.un[c][fg];
        }
        dn *= A.invh;
        dol = A.divn ? A.divn[fg] : dol * A.invh;
        A.p[fg] = A.p[fg] - A.chimu_half * (dn + dol);
        const double r = A.neg_rho_dt * dn;
        io[f] = r;
        return r;
    };
    const double c = C.c(), b = C.b();
    const double* inv = C.inv();
    const double* cpv = C.cp();
    const int m = C.m;
    const double d0 = src(0);
    double dsum = d0, prev = 0.0;
    for (int i = 1; i <= m; ++i) {
        const double d = src(i);
        dsum += d;
        prev = (d - c * prev) * inv[i - 1];
        io[i * PL + q] = prev;
    }
    double x = prev, fsum = prev;
    const double fm = prev;
    for (int i = m - 1; i >= 1; --i) {
        x = io[i * PL + q] - cpv[i - 1] * x;
        io[i * PL + q] = x;
        fsum += x;
    }
    if (A.local) {                      // A_t and fm_t of this part (visc_local)
        double* e = A.edge_w + ((long long)(comp * A.Q + blockIdx.z) * 2) * PL + q;
        e[0] = d0 - b * x;
        e[PL] = fm;
        return;
    }
    // to the line's master: [sub][slot][idx] in the block for master m
    {
        const int P = C.P / A.Q, mst = (int)(q % P);
        const long long idx = q / P;
        double* g = A.up_w + mst * A.up_mstride + ((long long)(part - A.rank * A.Q) * A.ns + slot0 + 2 * comp) * A.nidx + idx;
        g[0] = d0 - b * x;              // x = f*_1 here
        g[A.nidx] = fm;
        if (MF) {
            g[2 * (long long)A.nidx] = dsum;
            g[3 * (long long)A.nidx] = fsum;
        }
    }
}

// The forward phase with the part's column held in registers (parts of at most MAXM+1
// planes; fully unrolled, predicated on the runtime length): one read of d and one write
// of f* per cell instead of the two-pass recurrence through global memory above.
template <int DIM, int SRC, int MF, int MAXM>
__global__ void __launch_bounds__(128) k_slab_fwd_reg(SlabCf C, SlabArgs A, int slot0)
{
    const long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (q >= A.plane) return;
    const int comp = blockIdx.y;
    const int k0 = blockIdx.z * A.Lseg;
    const int part = A.rank * A.Q + blockIdx.z;
    double* io = ((comp == 0) ? A.io[0] : (comp == 1 ? A.io[1] : A.io[2])) + (long long)k0 * A.plane;
    const long long PL = A.plane;
    const int n = A.n;
    long long off[3] = {1, n, PL};
    if (SRC == SRC_DIV) {
        const int i = (int)(q % n);
        if (i == n - 1) off[0] = -(long long)(n - 1);
        if (DIM == 3) {
            const int j = (int)(q / n);
            if (j == n - 1) off[1] = -(long long)(n - 1) * n;
        } else {
            off[1] = PL;
        }
    }
    // (the updated p of each plane is kept and stored after the loads of the whole column:
    //  a store between them would keep the next plane's loads from being issued early)
    double pq[(SRC == SRC_DIV) ? MAXM + 1 : 1];
    auto src = [&](int kl) -> double {
        const long long f = kl * PL + q;
        if (SRC == SRC_FIELD) return io[f];
        double dn = 0.0, dol = 0.0;
        const long long fg = f + (long long)k0 * PL;
#pragma unroll
        for (int c = 0; c < DIM; ++c) {
            const long long o = (c == DIM - 1) ? PL : off[c];
            dn += __ldg(A.unew[c] + fg + o) - __ldg(A.unew[c] + fg);
            if (!A.divn) dol += __ldg(A.un[c] + fg + o) - __ldg(A.un[c] + fg);
        }
        dn *= A.invh;
        dol = A.divn ? __ldg(A.divn + fg) : dol * A.invh;
        pq[(SRC == SRC_DIV) ? kl : 0] = A.p[fg] - A.chimu_half * (dn + dol);
        return A.neg_rho_dt * dn;
    };
    const double c = C.c(), b = C.b();
    const double* inv = C.inv();
    const double* cpv = C.cp();
    const int m = C.m;
    double d[MAXM + 1];
#pragma unroll
    for (int i = 0; i <= MAXM; ++i) d[i] = (i <= m) ? src(i) : 0.0;
    if (SRC == SRC_DIV) {
#pragma unroll
        for (int i = 0; i <= MAXM; ++i)
            if (i <= m) A.p[(long long)(k0 + i) * PL + q] = pq[i];
    }
    double dsum = 0.0;
#pragma unroll
    for (int i = 0; i <= MAXM; ++i) dsum += d[i];
    double prev = 0.0;
#pragma unroll
    for (int i = 1; i <= MAXM; ++i)
        if (i <= m) {
            prev = (d[i] - c * prev) * __ldg(inv + i - 1);
            d[i] = prev;
        }
    const double fm = prev;
    double x = prev;
#pragma unroll
    for (int i = MAXM - 1; i >= 1; --i)
        if (i < m) {
            x = d[i] - __ldg(cpv + i - 1) * x;
            d[i] = x;
        }
    double fsum = 0.0;
#pragma unroll
    for (int i = 1; i <= MAXM; ++i)
        if (i <= m) {
            io[i * PL + q] = d[i];
            fsum += d[i];
        }
    if (A.local) {                      // A_t and fm_t of this part (visc_local)
        double* e = A.edge_w + ((long long)(comp * A.Q + blockIdx.z) * 2) * PL + q;
        e[0] = d[0] - b * d[1];
        e[PL] = fm;
        return;
    }
    {
        const int P = C.P / A.Q, mst = (int)(q % P);
        const long long idx = q / P;
        double* g = A.up_w + mst * A.up_mstride + ((long long)(part - A.rank * A.Q) * A.ns + slot0 + 2 * comp) * A.nidx + idx;
        g[0] = d[0] - b * d[1];
        g[A.nidx] = fm;
        if (MF) {
            g[2 * (long long)A.nidx] = dsum;
            g[3 * (long long)A.nidx] = fsum;
        }
    }
}

// correction phase: with y_s, y_{s+1} and the line-mean correction returned by the line's
// master (k_slab_master), x = f* - c y_s g - b y_{s+1} h (+ correction) on this part's
// planes.
template <int EPI, int MF>
__global__ void __launch_bounds__(128) k_slab_corr(SlabCf C, SlabArgs A, int slot0)
{
    const long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (q >= A.plane) return;
    const int comp = blockIdx.y;
    const long long k0 = (long long)blockIdx.z * A.Lseg;
    const int part = A.rank * A.Q + blockIdx.z;
    double* io = ((comp == 0) ? A.io[0] : (comp == 1 ? A.io[1] : A.io[2])) + k0 * A.plane;
    const double* un = ((comp == 0) ? A.un[0] : (comp == 1 ? A.un[1] : A.un[2])) + k0 * A.plane;
    const long long PL = A.plane;
    const int P = C.P / A.Q;
    const double c = C.c(), b = C.b();
    const int sub = part - A.rank * A.Q;
    double ys, ys1, corr = 0.0;
    if (A.local) {
        // visc_local: y_t = w0 (A_t - c fm_{t-1}), y_{t+1} = w0 (A_{t+1} - c fm_t), the
        // neighbour parts of the slab's first / last part from the exchanged planes
        const double* e = A.edge_w + (long long)comp * A.Q * 2 * PL + q;
        const double At = e[(long long)(2 * sub) * PL], fmt = e[(long long)(2 * sub + 1) * PL];
        const double fmp = (sub > 0) ? e[(long long)(2 * sub - 1) * PL] : A.edge_r[(long long)comp * PL + q];
        const double An = (sub < A.Q - 1) ? e[(long long)(2 * sub + 2) * PL]
                                          : A.edge_r[(long long)(3 + comp) * PL + q];
        ys = A.w0 * (At - c * fmp);
        ys1 = A.w0 * (An - c * fmt);
    } else {
        // y_s, y_{s+1} and the line-mean correction from the line's master
        const int mst = (int)(q % P);
        const long long idx = q / P;
        const double* y = A.dn_r + ((long long)mst * 3 + comp) * A.nb * A.nidx + idx;
        ys = y[(long long)sub * A.nidx];
        ys1 = y[(long long)(sub + 1) * A.nidx];
        corr = MF ? y[(long long)(A.Q + 1) * A.nidx] : 0.0;
    }
    (void)slot0;
    const double* g = C.g();
    const double* h = C.h();
    const double cy = c * ys, by = b * ys1;
    for (int kl = 0; kl <= C.m; ++kl) {
        const long long f = kl * PL + q;
        double x = (kl == 0) ? ys : io[f] - (cy * g[kl - 1] + by * h[kl - 1]);
        x += corr;
        if (EPI == EPI_ADD_UN) io[f] = un[f] + x;     // u^{n+1} = u^n + delta (R23)
        else io[f] = x;
    }
}

// The reduced system of the lines a rank is master of (q = m + P idx): r_t = A_t -
// c fm_{t-1} over the P Q parts t (every rank sent its scalars here), y_t = (S^{-1} r)_t,
// the exact line-mean correction (R16: sum(y) = colsum(S^{-1}) . r and sum(x)
// = (1 - c gsum - b hsum) sum(y) + sum_t F_t), and back to every rank r its
// y_{rQ} .. y_{rQ+Q} and the correction.  A block takes 32 lines: r is staged in shared
// memory once, the 8 warps split the rows t of S^{-1} (a row read is a warp broadcast).
// blockIdx.z is the master among those this launch handles (all P with EMULATE, this
// rank with NCCL).
constexpr int kMasterWarps = 8;
template <int MF>
__global__ void __launch_bounds__(32 * kMasterWarps) k_slab_master(SlabCf C, SlabArgs A, int slot0)
{
    __shared__ double rs[kSlabMaxParts * 32];   // [t][lane]
    const int lane = threadIdx.x & 31, tg = threadIdx.x >> 5;
    const long long idx = blockIdx.x * 32LL + lane;
    const bool ok = idx < A.nidx;
    const int comp = blockIdx.y;
    const int PQ = C.P, Q = A.Q, P = PQ / Q;
    const double c = C.c(), b = C.b();
    const double* SI = C.sinv();
    const long long NI = A.nidx;
    const double* in = A.up_r + (long long)blockIdx.z * A.up_rmstride;     // [rank][Q][ns][nidx]
    auto slot = [&](int t, int k) -> double { return in[((long long)t * A.ns + slot0 + 2 * comp + k) * NI + idx]; };
    for (int t = tg; t < PQ; t += kMasterWarps)
        rs[t * 32 + lane] = ok ? slot(t, 0) - c * slot(t == 0 ? PQ - 1 : t - 1, 1) : 0.0;
    __syncthreads();
    if (!ok) return;
    double* out = A.dn_w + (long long)blockIdx.z * A.dn_wmstride + (long long)comp * A.nb * NI + idx;
    for (int t = tg; t < PQ; t += kMasterWarps) {
        const double* row = SI + (long long)t * PQ;
        double y = 0.0;
        for (int u = 0; u < PQ; ++u) y = fma(row[u], rs[u * 32 + lane], y);
        const int r = t / Q, j = t - r * Q;
        out[(long long)r * A.dn_rstride + (long long)j * NI] = y;                 // y_{rQ+j} of rank r
        if (j == 0)                                                               // y_{(r'+1)Q} of rank r' = r-1
            out[(long long)((r + P - 1) % P) * A.dn_rstride + (long long)Q * NI] = y;
    }
    if (MF && tg == kMasterWarps - 1) {
        const double* CS = C.colsum();
        double ysum = 0.0, D = 0.0, F = 0.0;
        for (int t = 0; t < PQ; ++t) {
            ysum = fma(CS[t], rs[t * 32 + lane], ysum);
            D += slot(t, 2);
            F += slot(t, 3);
        }
        const double X = (1.0 - c * C.p[SC_GSUM] - b * C.p[SC_HSUM]) * ysum + F;
        const double corr = (D * C.p[SC_INVROW] - X) / C.p[SC_N];
        for (int r = 0; r < P; ++r) out[(long long)r * A.dn_rstride + (long long)(Q + 1) * NI] = corr;
    }
}

static unsigned nb128(long long cnt) { return (unsigned)((cnt + 127) / 128); }

template <int DIM, int SRC, int MF>
static cudaError_t launch_fwd(Ctx* s, const SlabCf& C, const SlabArgs& a, int ncomp)
{
    const dim3 grid(nb128(s->plane), (unsigned)ncomp, (unsigned)a.Q);
    // parts of <= 17 planes: column in registers (config 3 on 2 slabs 0.427 -> 0.388 ms)
    static int reg = -1;   // IBGM_SLAB_REG=0: the two-pass kernel (A/B)
    if (reg < 0) {
        const char* e = getenv("IBGM_SLAB_REG");
        reg = (e && atoi(e) == 0) ? 0 : 1;
    }
    if (reg && C.m <= 16) {
        k_slab_fwd_reg<DIM, SRC, MF, 16><<<grid, 128, 0, s->stream>>>(C, a, 0);
        s->launches++;
        return cudaGetLastError();
    }
    // (a 32-plane register variant measured slower than the two-pass kernel at config 4:
    //  8 slabs of 2 x 24 planes, 8.61 vs 8.15 ms; register pressure halves occupancy)
    k_slab_fwd<DIM, SRC, MF><<<grid, 128, 0, s->stream>>>(C, a, 0);
    s->launches++;
    return cudaGetLastError();
}

// exchange layouts (ns slots per part, nb = Q + 2 values back per line and component),
// one set per rank -- with EMULATE, slab r's set sits at r * (per-rank size) in the
// same buffers, so both transports run the same layouts and only the copy primitive
// differs (ncclSend/ncclRecv pairs, or one device copy per (sender, receiver) block):
//   up_s  [master][Q][ns][nidx]  -> up_rv [rank][Q][ns][nidx]   (scalars to the masters)
//   dn_s  [rank][3][nb][nidx]    -> dn_rv [master][3][nb][nidx] (y values back)
static size_t up_rank_size(const Group* G, long long plane)
{
    return (size_t)G->P * G->Q * kSlabSlots * (size_t)(plane / G->P);
}
static size_t dn_rank_size(const Group* G, long long plane)
{
    return (size_t)G->P * 3 * (size_t)(G->Q + 2) * (size_t)(plane / G->P);
}

static SlabArgs slab_args(Ctx* s, Group* G, int ns)
{
    SlabArgs a{};
    const int P = G->P, Q = G->Q;
    a.n = (int)s->n;
    a.nz = (int)s->nl;
    a.rank = s->rank;
    a.Q = Q;
    a.Lseg = (int)(s->nl / Q);
    a.plane = s->plane;
    a.invh = 1.0 / s->h;
    a.neg_rho_dt = -s->rho / s->dt;
    a.chimu_half = 0.5 * s->chi * s->mu;
    a.ns = ns;
    a.nidx = (int)(s->plane / P);
    a.nb = Q + 2;
    const long long NI = a.nidx, blk = (long long)Q * ns * NI, blk2 = 3LL * a.nb * NI;
    const bool emu = G->transport == IB_TRANSPORT_EMULATE;
    const long long us = (long long)up_rank_size(G, s->plane), ds = (long long)dn_rank_size(G, s->plane);
    const long long me = emu ? s->rank : 0;               // this slab's buffer set
    a.up_w = G->up_s + me * us;
    a.up_mstride = blk;
    a.up_r = G->up_rv;                                    // the master kernel's z-th master
    a.up_rmstride = emu ? us : 0;
    a.dn_w = G->dn_s;
    a.dn_wmstride = emu ? ds : 0;
    a.dn_rstride = blk2;
    a.dn_r = G->dn_rv + me * ds;
    a.edge_w = a.up_w;                                    // visc_local layouts (set by the sweeps)
    a.edge_r = G->up_rv + me * us;
    return a;
}

// the masters' reduced systems of one solve (EMULATE: every master in one launch)
cudaError_t slab_master(Ctx* s, Group* G, int sys, int ncomp, int ns, int mf)
{
    SlabArgs a = slab_args(s, G, ns);
    SlabCf C{G->coef[sys], (int)(s->nl / G->Q) - 1, G->P * G->Q};
    const unsigned nz = (G->transport == IB_TRANSPORT_EMULATE) ? (unsigned)G->P : 1u;
    const dim3 grid((unsigned)((a.nidx + 31) / 32), (unsigned)ncomp, nz);
    if (mf) k_slab_master<1><<<grid, 32 * kMasterWarps, 0, s->stream>>>(C, a, 0);
    else k_slab_master<0><<<grid, 32 * kMasterWarps, 0, s->stream>>>(C, a, 0);
    s->launches++;
    return cudaGetLastError();
}

// viscous sweep along the cut axis, all components: st = u^n + (1 - A_last)^{-1} st
cudaError_t slab_sweep_last_fwd(Ctx* s, Group* G)
{
    SlabArgs a = slab_args(s, G, 2 * s->dim);
    a.local = G->visc_local;
    a.w0 = G->visc_w0;
    for (int c = 0; c < s->dim; ++c) { a.io[c] = s->st[c]; a.un[c] = s->u[c]; }
    SlabCf C{G->coef[SYS_VISC], (int)(s->nl / G->Q) - 1, G->P * G->Q};
    if (s->dim == 3) return launch_fwd<3, SRC_FIELD, 0>(s, C, a, 3);
    return launch_fwd<2, SRC_FIELD, 0>(s, C, a, 2);
}

cudaError_t slab_sweep_last_corr(Ctx* s, Group* G)
{
    SlabArgs a = slab_args(s, G, 2 * s->dim);
    a.local = G->visc_local;
    a.w0 = G->visc_w0;
    for (int c = 0; c < s->dim; ++c) { a.io[c] = s->st[c]; a.un[c] = s->u[c]; }
    SlabCf C{G->coef[SYS_VISC], (int)(s->nl / G->Q) - 1, G->P * G->Q};
    k_slab_corr<EPI_ADD_UN, 0><<<dim3(nb128(s->plane), (unsigned)s->dim, (unsigned)a.Q), 128, 0, s->stream>>>(C, a, 0);
    s->launches++;
    return cudaGetLastError();
}

// Step 3e RHS, explicit part of 3f and the psi factor along the cut axis (into p*)
cudaError_t slab_divpsi_fwd(Ctx* s, Group* G)
{
    SlabArgs a = slab_args(s, G, 4);
    a.io[0] = a.io[1] = a.io[2] = s->pstar;
    for (int c = 0; c < s->dim; ++c) { a.un[c] = s->u[c]; a.unew[c] = s->st[c]; }
    a.p = s->p;
    a.divn = divn_fused(s) ? s->tmp : nullptr;
    SlabCf C{G->coef[SYS_PSI], (int)(s->nl / G->Q) - 1, G->P * G->Q};
    if (s->dim == 3) return launch_fwd<3, SRC_DIV, 1>(s, C, a, 1);
    return launch_fwd<2, SRC_DIV, 1>(s, C, a, 1);
}

cudaError_t slab_divpsi_corr(Ctx* s, Group* G)
{
    SlabArgs a = slab_args(s, G, 4);
    a.io[0] = a.io[1] = a.io[2] = s->pstar;
    SlabCf C{G->coef[SYS_PSI], (int)(s->nl / G->Q) - 1, G->P * G->Q};
    k_slab_corr<EPI_STORE, 1><<<dim3(nb128(s->plane), 1, (unsigned)a.Q), 128, 0, s->stream>>>(C, a, 0);
    s->launches++;
    return cudaGetLastError();
}

// stand-alone solve along the cut axis of data (in place) with coefficient block sys
cudaError_t slab_user_fwd(Ctx* s, Group* G, double* data, int mf)
{
    SlabArgs a = slab_args(s, G, mf ? 4 : 2);
    a.io[0] = a.io[1] = a.io[2] = data;
    SlabCf C{G->coef[SYS_USER], (int)(s->nl / G->Q) - 1, G->P * G->Q};
    if (mf) {
        if (s->dim == 3) return launch_fwd<3, SRC_FIELD, 1>(s, C, a, 1);
        return launch_fwd<2, SRC_FIELD, 1>(s, C, a, 1);
    }
    if (s->dim == 3) return launch_fwd<3, SRC_FIELD, 0>(s, C, a, 1);
    return launch_fwd<2, SRC_FIELD, 0>(s, C, a, 1);
}

cudaError_t slab_user_corr(Ctx* s, Group* G, double* data, int mf)
{
    SlabArgs a = slab_args(s, G, mf ? 4 : 2);
    a.io[0] = a.io[1] = a.io[2] = data;
    SlabCf C{G->coef[SYS_USER], (int)(s->nl / G->Q) - 1, G->P * G->Q};
    const dim3 grid(nb128(s->plane), 1, (unsigned)a.Q);
    if (mf) k_slab_corr<EPI_STORE, 1><<<grid, 128, 0, s->stream>>>(C, a, 0);
    else k_slab_corr<EPI_STORE, 0><<<grid, 128, 0, s->stream>>>(C, a, 0);
    s->launches++;
    return cudaGetLastError();
}

// ------------------------------------------------------------------------------------
// IB on a slab
// ------------------------------------------------------------------------------------
template <int KER>
__device__ __forceinline__ void w4(double x, int n, int& i0, double w[4])
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
        const double qq = sqrt(1.0 + 4.0 * r - 4.0 * r * r);
        w[0] = 0.125 * (3.0 - 2.0 * r - qq);
        w[1] = 0.125 * (3.0 - 2.0 * r + qq);
        w[2] = 0.125 * (1.0 + 2.0 * r + qq);
        w[3] = 0.125 * (1.0 + 2.0 * r - qq);
    }
}

__device__ __forceinline__ int wrapp(int i, int n) { return i >= n ? i - n : i; }

// Step 1a restricted to the nodes this slab owns (global planes z0 .. z0+nz-1 of the
// last axis): Upart_k = sum over owned stencil nodes of u phi phi (phi).  The sum over
// ranks (all-reduce) is U^n of PAPER.md:581-586.
// The points whose 4-point support (any staggering: cells cz-2 .. cz+2 of the last axis)
// meets this slab's planes, appended to list (warp-aggregated; order irrelevant).
template <int DIM>
__global__ void k_slab_select(const double* __restrict__ X, long long npts, int n, int z0, int nz, double invh,
                              int* __restrict__ list, int* __restrict__ count)
{
    const long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    bool hit = false;
    if (k < npts) {
        const int cz = (int)floor(X[k * DIM + DIM - 1] * invh);
#pragma unroll
        for (int d = -2; d <= 2; ++d) {
            int g = (cz + d) % n;
            if (g < 0) g += n;
            hit = hit || (unsigned)(g - z0) < (unsigned)nz;
        }
    }
    // a warp with any hit appends one 32-slot chunk in its own (Morton) order, -1 where
    // a lane has no hit: a window of 32 list entries is then one source warp's points
    // (spatially compact for the window-staged IB kernels), wherever the chunk lands
    const unsigned m = __ballot_sync(0xffffffffu, hit);
    if (m == 0) return;
    const int lane = threadIdx.x & 31;
    int base = 0;
    if (lane == 0) base = atomicAdd(count, 32);
    base = __shfl_sync(0xffffffffu, base, 0);
    list[base + lane] = hit ? (int)k : -1;
}

template <int DIM, int KER>
__global__ void k_interp_part(const double* __restrict__ u0, const double* __restrict__ u1,
                              const double* __restrict__ u2, const double* __restrict__ X,
                              double* __restrict__ Upart, const int* __restrict__ list, const int* __restrict__ count,
                              int n, int z0, int nz, double invh)
{
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i >= *count) return;
    const long long k = list[i];
    if (k < 0) return;                  // padding of a warp-aligned chunk (k_slab_select)
    double Xk[3];
#pragma unroll
    for (int a = 0; a < DIM; ++a) Xk[a] = X[k * DIM + a];
    const long long nn = n;
#pragma unroll
    for (int c = 0; c < DIM; ++c) {
        const double* uc = (c == 0) ? u0 : (c == 1 ? u1 : u2);
        int i0[3] = {0, 0, 0};
        double w[3][4];
#pragma unroll
        for (int a = 0; a < DIM; ++a) w4<KER>(Xk[a] * invh - (a == c ? 0.0 : 0.5), n, i0[a], w[a]);
        double acc = 0.0;
#pragma unroll
        for (int mL = 0; mL < 4; ++mL) {
            const int kl = wrapp(i0[DIM - 1] + mL, n) - z0;
            if (kl < 0 || kl >= nz) continue;
            double pa = 0.0;
            if (DIM == 2) {
                const long long row = nn * kl;
#pragma unroll
                for (int m0 = 0; m0 < 4; ++m0) pa += w[0][m0] * uc[row + wrapp(i0[0] + m0, n)];
            } else {
                const long long pl = nn * nn * kl;
#pragma unroll
                for (int m1 = 0; m1 < 4; ++m1) {
                    const long long row = pl + nn * wrapp(i0[1] + m1, n);
                    double r = 0.0;
#pragma unroll
                    for (int m0 = 0; m0 < 4; ++m0) r += w[0][m0] * uc[row + wrapp(i0[0] + m0, n)];
                    pa += w[1][m1] * r;
                }
            }
            acc += w[DIM - 1][mL] * pa;
        }
        Upart[k * DIM + c] = acc;
    }
}

// sum of the P partial interpolations (EMULATE transport; NCCL all-reduces instead)
__global__ void k_sum_slots(const double* __restrict__ part, int P, long long cnt, double* __restrict__ out)
{
    for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < cnt; q += (long long)gridDim.x * blockDim.x) {
        double a = 0.0;
        for (int r = 0; r < P; ++r) a += part[r * cnt + q];
        out[q] = a;
    }
}

// Steps 1b-1c on every point from the reduced U^n (identical on every rank)
__global__ void k_evolve(const double* __restrict__ U, double* __restrict__ X, double* __restrict__ Xh,
                         double* __restrict__ Uprev, double* __restrict__ Xold, double* __restrict__ Uold,
                         long long cnt, double dt, int first)
{
    const long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (e >= cnt) return;
    const double x = X[e], u = U[e], up = Uprev[e];
    const double xn = first ? x + dt * u : x + dt * (1.5 * u - 0.5 * up);
    Xh[e] = 0.5 * (xn + x);
    X[e] = xn;
    Uprev[e] = u;
    Xold[e] = x;        // X^n, U^{n-1}: the state before this IB phase (read while ahead)
    Uold[e] = up;
}

// Step 2b restricted to the nodes this slab owns (into G = N^{n-1} + (2/rho) f, R24)
template <int DIM, int KER, bool KEEP>
__global__ void __launch_bounds__(128) k_spread_part(const double* __restrict__ Xh, const double* __restrict__ F,
                                                     const double* __restrict__ wgt, double* g0, double* g1, double* g2,
                                                     double* f0, double* f1, double* f2, const int* __restrict__ list,
                                                     const int* __restrict__ count, int n, int z0,
                                                     int nz, double invh, double invhd, double two_rho)
{
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i >= *count) return;
    const long long k = list[i];
    if (k < 0) return;                  // padding of a warp-aligned chunk (k_slab_select)
    double Xk[3];
#pragma unroll
    for (int a = 0; a < DIM; ++a) Xk[a] = Xh[k * DIM + a];
    const double wk = wgt[k] * invhd;
    const long long nn = n;
#pragma unroll
    for (int c = 0; c < DIM; ++c) {
        double* gc = (c == 0) ? g0 : (c == 1 ? g1 : g2);
        double* fc = (c == 0) ? f0 : (c == 1 ? f1 : f2);
        int i0[3] = {0, 0, 0};
        double w[3][4];
#pragma unroll
        for (int a = 0; a < DIM; ++a) w4<KER>(Xk[a] * invh - (a == c ? 0.0 : 0.5), n, i0[a], w[a]);
        const double Fc = F[k * DIM + c] * wk;
#pragma unroll
        for (int mL = 0; mL < 4; ++mL) {
            const int kl = wrapp(i0[DIM - 1] + mL, n) - z0;
            if (kl < 0 || kl >= nz) continue;
            const double aL = Fc * w[DIM - 1][mL];
            if (DIM == 2) {
                const long long row = nn * kl;
#pragma unroll
                for (int m0 = 0; m0 < 4; ++m0) {
                    const long long q = row + wrapp(i0[0] + m0, n);
                    const double v = aL * w[0][m0];
                    atomicAdd(gc + q, two_rho * v);
                    if (KEEP) atomicAdd(fc + q, v);
                }
            } else {
                const long long pl = nn * nn * kl;
#pragma unroll
                for (int m1 = 0; m1 < 4; ++m1) {
                    const long long row = pl + nn * wrapp(i0[1] + m1, n);
                    const double a1 = aL * w[1][m1];
#pragma unroll
                    for (int m0 = 0; m0 < 4; ++m0) {
                        const long long q = row + wrapp(i0[0] + m0, n);
                        const double v = a1 * w[0][m0];
                        atomicAdd(gc + q, two_rho * v);
                        if (KEEP) atomicAdd(fc + q, v);
                    }
                }
            }
        }
    }
}

// select the points of slab s (list r of the group) from positions Xsrc
static cudaError_t slab_select(Ctx* top, Ctx* s, const double* Xsrc, int* list, int* count)
{
    cudaError_t e = cudaMemsetAsync(count, 0, sizeof(int), s->stream);
    if (e != cudaSuccess) return e;
    const double invh = 1.0 / s->h;
    if (s->dim == 3)
        k_slab_select<3><<<nb128(top->npts), 128, 0, s->stream>>>(Xsrc, top->npts, (int)s->n, (int)s->z0, (int)s->nl,
                                                                  invh, list, count);
    else
        k_slab_select<2><<<nb128(top->npts), 128, 0, s->stream>>>(Xsrc, top->npts, (int)s->n, (int)s->z0, (int)s->nl,
                                                                  invh, list, count);
    s->launches++;
    return cudaGetLastError();
}

// the slab IB kernels: one thread per (point, component) for the interpolation and the
// quad-lane spread with warp pre-reduction (ib.cu) on the selected points; IBGM_SLAB_IB=0
// keeps the per-point kernels below (A/B)
static bool slab_ib_fast()
{
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("IBGM_SLAB_IB");
        v = (e && atoi(e) == 0) ? 0 : 1;
    }
    return v == 1;
}

cudaError_t slab_interp_part(Ctx* top, Ctx* s, double* Upart, int* list, int* count)
{
    const double invh = 1.0 / s->h;
    cudaError_t e = cudaMemsetAsync(Upart, 0, sizeof(double) * top->npts * top->dim, s->stream);
    if (e != cudaSuccess) return e;
    if ((e = slab_select(top, s, top->X, list, count)) != cudaSuccess) return e;
    if (slab_ib_fast()) return launch_interp_part(top, s, Upart, list, count);
#define IBGM_IP(D, K) k_interp_part<D, K><<<nb128(nb128(top->npts) * 128LL), 128, 0, s->stream>>>( \
        s->u[0], s->u[1], s->u[2], top->X, Upart, list, count, (int)s->n, (int)s->z0, (int)s->nl, invh)
    if (s->dim == 2) { if (top->kernel == IB_DELTA_COS4) IBGM_IP(2, 0); else IBGM_IP(2, 1); }
    else { if (top->kernel == IB_DELTA_COS4) IBGM_IP(3, 0); else IBGM_IP(3, 1); }
#undef IBGM_IP
    s->launches++;
    return cudaGetLastError();
}

cudaError_t slab_sum_slots(Ctx* top, const double* part, int P, double* out)
{
    const long long cnt = top->npts * top->dim;
    k_sum_slots<<<(unsigned)((cnt + 255) / 256 < 592 ? (cnt + 255) / 256 : 592), 256, 0, top->stream>>>(part, P, cnt, out);
    top->launches++;
    return cudaGetLastError();
}

cudaError_t slab_evolve(Ctx* top, const double* U, int first)
{
    const long long cnt = top->npts * top->dim;
    k_evolve<<<nb128(cnt), 128, 0, top->stream>>>(U, top->X, top->Xh, top->Uprev, top->Xold, top->Uold, cnt, top->dt,
                                                  first);
    top->launches++;
    return cudaGetLastError();
}

cudaError_t slab_spread_part(Ctx* top, Ctx* s, int* list, int* count)
{
    const double invh = 1.0 / s->h;
    const double invhd = (s->dim == 3) ? invh * invh * invh : invh * invh;
    const bool kp = top->debug_keep_f != 0;
    cudaError_t e = slab_select(top, s, top->Xh, list, count);
    if (e != cudaSuccess) return e;
    if (slab_ib_fast()) return launch_spread_part(top, s, list, count);
#define IBGM_SPP(D, K, KP) k_spread_part<D, K, KP><<<nb128(nb128(top->npts) * 128LL), 128, 0, s->stream>>>(                  \
        top->Xh, top->F, top->wgt, s->nprev[0], s->nprev[1], s->nprev[2], s->f[0], s->f[1], s->f[2], list, count, \
        (int)s->n, (int)s->z0, (int)s->nl, invh, invhd, 2.0 / s->rho)
    if (s->dim == 2) {
        if (top->kernel == IB_DELTA_COS4) { if (kp) IBGM_SPP(2, 0, true); else IBGM_SPP(2, 0, false); }
        else { if (kp) IBGM_SPP(2, 1, true); else IBGM_SPP(2, 1, false); }
    } else {
        if (top->kernel == IB_DELTA_COS4) { if (kp) IBGM_SPP(3, 0, true); else IBGM_SPP(3, 0, false); }
        else { if (kp) IBGM_SPP(3, 1, true); else IBGM_SPP(3, 1, false); }
    }
#undef IBGM_SPP
    s->launches++;
    return cudaGetLastError();
}

// ------------------------------------------------------------------------------------
// transports
// ------------------------------------------------------------------------------------
#define NCK(call)                                   \
    do {                                            \
        const int r_ = (call);                      \
        if (r_ != 0) return r_;                     \
    } while (0)

// EMULATE transport: the P x P (sender, receiver) block copies of one all-to-all in a
// single launch -- block (r, m) of `cnt` doubles goes from src + r sr + m sm to
// dst + m dr + r dm (blockIdx.y = r P + m), exactly the ncclSend/ncclRecv pairs of the
// NCCL transport.
__global__ void k_alltoall_copy(const double* __restrict__ src, double* __restrict__ dst, int P, long long cnt,
                                long long sr, long long sm, long long dr, long long dm)
{
    const int r = blockIdx.y / P, m = blockIdx.y - r * P;
    const double* a = src + r * sr + m * sm;
    double* b = dst + m * dr + r * dm;
    for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < cnt; q += (long long)gridDim.x * blockDim.x)
        b[q] = a[q];
}

static cudaError_t alltoall_copy(const double* src, double* dst, int P, long long cnt, long long sr, long long sm,
                                 long long dr, long long dm, cudaStream_t st)
{
    const long long bx = std::min((cnt + 255) / 256, 64LL);
    k_alltoall_copy<<<dim3((unsigned)std::max(bx, 1LL), (unsigned)(P * P)), 256, 0, st>>>(src, dst, P, cnt, sr, sm, dr,
                                                                                        dm);
    return cudaGetLastError();
}

// Halo exchange (EMULATE): every slab's boundary planes of up to kHaloMax fields into the
// neighbours' halo planes in one launch (blockIdx.y = field, slab, direction)
constexpr int kHaloMax = 4;
struct HaloPtrs {
    const double* src[kHaloMax * kMaxRanks * 2];
    double* dst[kHaloMax * kMaxRanks * 2];
};
__global__ void k_halo_copy(const HaloPtrs H, long long PL)
{
    const double* a = H.src[blockIdx.y];
    double* b = H.dst[blockIdx.y];
    if (!a) return;
    for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < PL; q += (long long)gridDim.x * blockDim.x)
        b[q] = a[q];
}

// Halo exchange of the listed fields.  dir_up: plane nz-1 of slab s
// -> plane -1 of slab s+1; dir_down: plane 0 of slab s -> plane nz of slab s-1 (periodic).
// Returns 0, a cudaError_t (as int, transport EMULATE) or an ncclResult_t (NCCL).
int group_halo(Group* G, int nf, const HaloSpec* spec, cudaStream_t st, void* comm)
{
    if (!comm) comm = G->comm;
    const int P = G->P;
    if (G->transport == IB_TRANSPORT_EMULATE) {
        // the same sends and receives as the NCCL branch below, one launch for all of them
        HaloPtrs H{};
        int np = 0;
        const long long nz = G->slab[0]->nl, PL = G->slab[0]->plane;
        if (nf > kHaloMax) return (int)cudaErrorInvalidValue;
        for (int f = 0; f < nf; ++f)
            for (int r = 0; r < P; ++r) {
                Ctx* a = G->slab[r];
                if (spec[f].up) {
                    Ctx* b = G->slab[(r + 1) % P];
                    H.src[np] = spec[f].field(a) + (nz - 1) * PL;
                    H.dst[np++] = spec[f].field(b) - PL;
                }
                if (spec[f].down) {
                    Ctx* b = G->slab[(r + P - 1) % P];
                    H.src[np] = spec[f].field(a);
                    H.dst[np++] = spec[f].field(b) + nz * PL;
                }
            }
        if (np == 0) return 0;
        const long long bx = std::min((PL + 255) / 256, 32LL);
        k_halo_copy<<<dim3((unsigned)bx, (unsigned)np), 256, 0, st>>>(H, PL);
        return (int)cudaGetLastError();
    }
    Ctx* a = G->slab[0];
    const long long nz = a->nl, PL = a->plane;
    const int up = (G->rank + 1) % P, dn = (G->rank + P - 1) % P;
    NCK(g_nccl.GroupStart());
    for (int f = 0; f < nf; ++f) {
        double* fld = spec[f].field(a);
        if (spec[f].up) {
            NCK(g_nccl.Send(fld + (nz - 1) * PL, (size_t)PL, kNcclDouble, up, comm, st));
            NCK(g_nccl.Recv(fld - PL, (size_t)PL, kNcclDouble, dn, comm, st));
        }
        if (spec[f].down) {
            NCK(g_nccl.Send(fld, (size_t)PL, kNcclDouble, dn, comm, st));
            NCK(g_nccl.Recv(fld + nz * PL, (size_t)PL, kNcclDouble, up, comm, st));
        }
    }
    NCK(g_nccl.GroupEnd());
    return 0;
}

// each line's scalars to its master (all-to-all): rank r's block for master m
// (up_s[r] + m blk) lands in master m's receive buffer at r blk
int group_up(Group* G, int ns, cudaStream_t st)
{
    const long long plane = G->slab[0]->plane;
    const size_t blk = (size_t)G->Q * ns * (plane / G->P);
    if (G->transport == IB_TRANSPORT_EMULATE) {
        const long long us = (long long)up_rank_size(G, plane);
        return (int)alltoall_copy(G->up_s, G->up_rv, G->P, (long long)blk, us, (long long)blk, us, (long long)blk, st);
    }
    NCK(g_nccl.GroupStart());
    for (int m = 0; m < G->P; ++m) {
        NCK(g_nccl.Send(G->up_s + m * blk, blk, kNcclDouble, m, G->comm, st));
        NCK(g_nccl.Recv(G->up_rv + m * blk, blk, kNcclDouble, m, G->comm, st));
    }
    NCK(g_nccl.GroupEnd());
    return 0;
}

// the masters' y values and corrections back to the ranks (all-to-all): master m's
// block for rank r (dn_s[m] + r stride) lands in rank r's receive buffer at m stride
int group_dn(Group* G, int ncomp, cudaStream_t st)
{
    const long long plane = G->slab[0]->plane;
    const size_t NI = plane / G->P, nb = (size_t)G->Q + 2;
    const size_t stride = 3 * nb * NI, cnt = (size_t)ncomp * nb * NI;
    if (G->transport == IB_TRANSPORT_EMULATE) {
        // sender = master m (block for rank r at r stride) -> receiver r (at m stride)
        const long long ds = (long long)dn_rank_size(G, plane);
        return (int)alltoall_copy(G->dn_s, G->dn_rv, G->P, (long long)cnt, ds, (long long)stride, ds,
                                  (long long)stride, st);
    }
    NCK(g_nccl.GroupStart());
    for (int r = 0; r < G->P; ++r) {
        NCK(g_nccl.Send(G->dn_s + r * stride, cnt, kNcclDouble, r, G->comm, st));
        NCK(g_nccl.Recv(G->dn_rv + r * stride, cnt, kNcclDouble, r, G->comm, st));
    }
    NCK(g_nccl.GroupEnd());
    return 0;
}

// visc_local: the scalars of each slab's boundary parts to its neighbours (the
// nearest-neighbour exchange of PAPER.md:807-833 applied to the reduced system): fm of
// the last part -> the slab above (receive slot 0), A of the first part -> the slab
// below (receive slot 1); one plane per component each way
int group_edge(Group* G, int ncomp, cudaStream_t st)
{
    const int P = G->P, Q = G->Q;
    const long long PL = G->slab[0]->plane;
    const long long us = (long long)up_rank_size(G, PL);
    if (G->transport == IB_TRANSPORT_EMULATE) {
        HaloPtrs H{};
        int np = 0;
        for (int c = 0; c < ncomp; ++c)
            for (int r = 0; r < P; ++r) {
                const double* e = G->up_s + r * us + (long long)c * Q * 2 * PL;
                H.src[np] = e + (long long)(2 * (Q - 1) + 1) * PL;                     // fm of the last part
                H.dst[np++] = G->up_rv + ((r + 1) % P) * us + (long long)c * PL;      // -> above, slot 0
                H.src[np] = e;                                                        // A of the first part
                H.dst[np++] = G->up_rv + ((r + P - 1) % P) * us + (long long)(3 + c) * PL;   // -> below, slot 1
            }
        const long long bx = std::min((PL + 255) / 256, 32LL);
        k_halo_copy<<<dim3((unsigned)bx, (unsigned)np), 256, 0, st>>>(H, PL);
        return (int)cudaGetLastError();
    }
    const int up = (G->rank + 1) % P, dn = (G->rank + P - 1) % P;
    NCK(g_nccl.GroupStart());
    for (int c = 0; c < ncomp; ++c) {
        const double* e = G->up_s + (long long)c * Q * 2 * PL;
        NCK(g_nccl.Send(e + (long long)(2 * (Q - 1) + 1) * PL, (size_t)PL, kNcclDouble, up, G->comm, st));
        NCK(g_nccl.Recv(G->up_rv + (long long)c * PL, (size_t)PL, kNcclDouble, dn, G->comm, st));
        NCK(g_nccl.Send(e, (size_t)PL, kNcclDouble, dn, G->comm, st));
        NCK(g_nccl.Recv(G->up_rv + (long long)(3 + c) * PL, (size_t)PL, kNcclDouble, up, G->comm, st));
    }
    NCK(g_nccl.GroupEnd());
    return 0;
}

// U^n = sum over ranks of the partial interpolations
int group_allreduce_U(Group* G, Ctx* top, cudaStream_t st, bool side)
{
    const long long cnt = top->npts * top->dim;
    if (G->transport == IB_TRANSPORT_EMULATE) return (int)slab_sum_slots(top, G->Upart, G->P, G->Ured);
    return g_nccl.AllReduce(G->Upart, G->Ured, (size_t)cnt, kNcclDouble, kNcclSum, side ? G->comm_side : G->comm, st);
}

}  // namespace ibgm
