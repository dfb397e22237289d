// Internal declarations shared by the CUDA translation units of libibgm.so.
// Product code; shares nothing with oracle/.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <utility>

#include "../../include/ibgm.h"

namespace ibgm {

constexpr int kMaxSeg = 32;   // max segments P per line (reduced Schur system size)
constexpr int kMaxL = 32;     // max segment length L
constexpr int kMaxBand = 4;   // max half-width of a banded S^{-1} (LineCoef::w)

// Constant-coefficient cyclic tridiagonal system  c x_{i-1} + a x_i + b x_{i+1} = d_i
// solved by the paper's Schur-complement splitting applied
// inside a thread block: each line of N = P*L unknowns is cut into P parts; part p
// is one interface unknown y_p = x_{pL} followed by an interior block of m = L-1
// unknowns (the B_p of eq. BlockSchurSystem).  Everything here is line-independent
// and precomputed once on the host in long double (PAPER.md:1260-1262:
// "S and B^{-1}E can be precomputed").  Passed to kernels BY VALUE (constant bank).
struct LineCoef {
    double c, a, b;
    double inv_rowsum;        // 1/(a+b+c): mean(x) = mean(d)/(a+b+c) for circulant A
    double gsum, hsum;        // sum_i g_i, sum_i h_i
    double inv_n;             // 1/N
    int L, P, N, mean_fix;
    const double* ext;        // L > kMaxL (2D N > 1024): device inv, cp, g, h [m each]
    double inv[kMaxL];        // Thomas: 1/den_i of B (i = 0..m-1)
    double cp[kMaxL];         // Thomas: b/den_i
    double g[kMaxL];          // B^{-1} e_1   (first column of B^{-1})
    double h[kMaxL];          // B^{-1} e_m   (last column of B^{-1})
    // S is circulant (P equal parts, constant coefficients), so S^{-1} is too.  When every
    // entry of S^{-1} farther than `band` parts from the diagonal is below 1e-18 of the
    // diagonal (well-conditioned viscous systems: the coupling between parts decays like
    // lambda^L, lambda ~ kappa), y_s = sum_{|d| <= band} w[kMaxBand + d] r_{s+d} replaces the
    // dense product; band = -1: dense S^{-1} (SchurInv).
    int band;
    double w[2 * kMaxBand + 1];
    // circ = 1: S^{-1} is circulant, row 0 in wf (y_s = sum_d wf[d] r_{(s+d) mod P}, the
    // coefficients uniform across lanes: constant-bank operands instead of a staged
    // P x P matrix); 0: dense S^{-1} (SchurInv)
    int circ;
    double wf[kMaxSeg];
};

// dense inverse of the P x P periodic Schur matrix S and its column sums (device)
struct SchurInv {
    double sinv[kMaxSeg * kMaxSeg];
    double sinvT[kMaxSeg * kMaxSeg];  // transposed: sinvT[q P + p] = sinv[p P + q]
    double colsum[kMaxSeg];
};

enum SysId { SYS_VISC = 0, SYS_PSI = 1, SYS_USER = 2, SYS_COUNT = 3 };

// indices of the sticky error words (Ctx::err_h / err_d)
enum ErrWord { ERR_NONFINITE = 0, ERR_DOMAIN = 1, ERR_DEGENERATE = 2, ERR_WORDS = 4 };

struct Group;

struct Ctx {
    int dim;
    int64_t n, ncell;
    // local extent: the last axis (z in 3D, y in 2D) has nl planes starting at global
    // plane z0; nl = n, z0 = 0, wrap = 1 on a single GPU; on a z-slab wrap = 0 and the
    // fields carry one halo plane on each side (pointers address plane 0, hoff doubles
    // in from the allocation)
    int64_t nl, z0, plane, nlocal, hoff;
    int wrap, rank;
    Group* grp;                       // z-slab decomposition (nullptr on a single GPU)
    double h, H, mu, rho, dt, chi;   // h = H/N, H the box side
    int kernel, advection, device;
    cudaStream_t stream;
    bool own_stream;
    int L, P;                         // line segmentation: N = P*L
    // Eulerian state (device), each ncell doubles
    double* u[3];                     // u^n
    double* st[3];                    // Douglas increments delta1, delta2, then u^{n+1}
    double* nadv[3];                  // N(u^n), written this step
    double* nprev[3];                 // G = N(u^{n-1}) + (2/rho) f^{n+1/2} (spread adds f here)
    double* f[3];                     // debug only: f^{n+1/2} kept for ib_get_aux
    double* p;                        // p^{n-1/2}  (holds q = p - chi mu D.u_bar mid-step)
    double* pstar;                    // p* = p^{n-1/2} + psi^{n-1/2}; psi factors mid-step
    double* tmp;                      // scratch field (ib_get_fields psi, ib_line_solve)
    SchurInv* sinv;                   // device, SYS_COUNT entries
    double* lcext[SYS_COUNT];         // device long-segment factors (LineCoef::ext)
    LineCoef hcoef[SYS_COUNT];        // host copies (passed by value)
    // Lagrangian state (device)
    int64_t npts, nedges;
    double *X, *Xh, *Uprev, *F, *wgt;   // Uprev: U interpolated in the last step
    double *Xold, *Uold;              // X and Uprev before the last IB phase (see ib_ahead)
    int32_t* csr_ptr;                 // [npts+1]
    int32_t* csr_nbr;                 // [2*nedges]
    double* csr_kappa;                // [2*nedges]
    double* csr_rest;                 // [2*nedges]
    int has_rest;
    // brick binning of the points for the spread (Step 2b)
    int nb;                           // bricks per axis
    int64_t nbricks;
    int *bin_bid, *bin_count, *bin_start, *bin_cursor, *bin_list, *bin_nlist, *bin_sorted, *bin_partial;
    int debug_keep_f;                 // ib_set_debug: also accumulate f for ib_get_aux
    int spread_mode;                  // ib_set_debug bits 1-3: 0 auto (quad), 1 per-point, 2 brick, 3 box, 4 quad
    int interp_mode;                  // ib_set_debug bits 4-5: 0 auto (per-point), 1 per-point, 2 box, 3 quad
    // internal point order (Morton order of the initial cells): pt_user[i] = caller index
    int32_t* pt_user;
    double* lag_tmp;                  // [npts][dim] scratch for returning points in caller order
    int64_t step;                     // steps completed since set_fields/set_boundary
    bool fields_set;
    int64_t launches;
    int* d_flag;                      // device flag for finiteness checks
    // sticky device-raised errors (mapped pinned host words, written by kernels with plain
    // stores, read by the host without a synchronisation): ERR_* below.  Slabs share the
    // top context's words.
    int* err_h;
    int* err_d;
    int64_t check_every;              // in-step state check every K steps (0: off)
    // IB look-ahead: the IB phase of step n+1 (Steps 1-2, which need only u^{n+1} and X)
    // runs on a side stream concurrently with the psi passes of step n; ib_ahead says
    // it has been done, so X, Uprev, Xh, F and G already belong to the next step
    cudaStream_t side;
    cudaEvent_t ev_fork, ev_join;
    // z-slabs: the u^{n+1} halos the next step's S1 needs are exchanged on `comm` as soon as
    // the last Douglas sweep has formed u^{n+1}, concurrently with the psi passes
    // (ev_h0 fork, ev_h1 join); u_halo_ready: the current u's halo planes are valid
    cudaStream_t comm;
    cudaEvent_t ev_h0, ev_h1;
    bool u_halo_ready;
    bool ib_ahead;
    int lookahead;                    // 1 (default) enables the overlap
    // CUDA graphs of one regular step, per pointer parity (u <-> st, N <-> G swaps) and
    // per look-ahead state at entry
    int parity;
    bool use_graphs;
    cudaGraphExec_t gexec[4];
    bool gvalid[4];
    int64_t glaunches[4];             // kernels per captured step
    // per-phase profiling (ib_set_profiling)
    int profiling;
    cudaEvent_t ev[IB_NPHASES][2];
    bool ev_made;
    double ph_ms[IB_NPHASES];
    int64_t ph_cnt[IB_NPHASES];
    bool ph_pending[IB_NPHASES];
};

// ---------------------------------------------------------------------------------
// z-slab decomposition (slab.cu)
// ---------------------------------------------------------------------------------
struct NcclUid { char internal[128]; };

// slab coefficient block header (doubles), followed by inv, cp, g, h [m], S^{-1} [P*P],
// colsum(S^{-1}) [P]
enum { SC_C = 0, SC_A, SC_B, SC_INVROW, SC_GSUM, SC_HSUM, SC_N, SC_MF, SC_HDR = 8 };
constexpr int kSlabMaxParts = 128;  // parts of the cut-axis reduced system (P Q), k_slab_master
constexpr int kSlabSlots = 6;         // max gather slots per part: 2 per velocity component / 4 for psi
constexpr int kMaxRanks = 64;

struct Group {
    int P;                            // ranks (slabs)
    int transport;                    // IB_TRANSPORT_EMULATE | IB_TRANSPORT_NCCL
    int rank;                         // NCCL: this process's rank
    int nloc;                         // slabs held by this context (P emulated, 1 with NCCL)
    int Q;                            // Schur parts per slab along the cut axis (nz = Q Lseg)
    Ctx* slab[kMaxRanks];
    double *up_s, *up_rv;             // reduced-system scalars to the line masters (slab.cu layouts)
    double *dn_s, *dn_rv;             // y values and corrections back from the masters
    double* Upart;                    // partial interpolation ([P][npts*d] emulated, [npts*d] NCCL)
    double* Ured;                     // U^n after the sum over ranks
    int64_t ucap;                     // capacity (points*d) of Upart/Ured
    int* sel[kMaxRanks];              // per local slab: the points whose support meets it
    int* sel_cnt;                     // [nloc] counters
    double* coef[SYS_COUNT];          // device slab coefficient blocks
    void* comm;                       // ncclComm_t
    void* comm_side;                  // a second communicator (ncclCommSplit) for the IB
                                      // look-ahead's all-reduce on the side stream
    void* comm_halo;                  // a third one for the early u halos on the comm stream
    // the viscous cut-axis system's S^{-1} is diagonal to rounding (every off-diagonal
    // entry below 1e-18 of the diagonal): y_t = w0 r_t, so each part needs only its
    // neighbour parts' scalars -- a nearest-neighbour exchange instead of the line masters
    int visc_local;
    double visc_w0;
};

struct HaloSpec {
    double* (*field)(Ctx*);
    bool up, down;
};

const char* nccl_load(void);
int nccl_unique_id(NcclUid* id);
int nccl_comm_init(void** comm, int nranks, const NcclUid* id, int rank);
void nccl_comm_destroy(void* comm);
const char* nccl_error_string(int rc);

cudaError_t slab_sweep_last_fwd(Ctx* s, Group* G);
cudaError_t slab_sweep_last_corr(Ctx* s, Group* G);
cudaError_t slab_divpsi_fwd(Ctx* s, Group* G);
cudaError_t slab_divpsi_corr(Ctx* s, Group* G);
cudaError_t slab_user_fwd(Ctx* s, Group* G, double* data, int mf);
cudaError_t slab_user_corr(Ctx* s, Group* G, double* data, int mf);
cudaError_t slab_interp_part(Ctx* top, Ctx* s, double* Upart, int* list, int* count);
cudaError_t slab_sum_slots(Ctx* top, const double* part, int P, double* out);
cudaError_t slab_evolve(Ctx* top, const double* U, int first);   // also keeps X^n, U^{n-1} in Xold, Uold
cudaError_t slab_spread_part(Ctx* top, Ctx* s, int* list, int* count);
int group_halo(Group* G, int nf, const HaloSpec* spec, cudaStream_t st, void* comm = nullptr);
int group_up(Group* G, int ns, cudaStream_t st);          // scalars to the line masters
int group_dn(Group* G, int ncomp, cudaStream_t st);       // y and corrections back
int group_edge(Group* G, int ncomp, cudaStream_t st);     // neighbour parts' scalars (visc_local)
cudaError_t slab_master(Ctx* s, Group* G, int sys, int ncomp, int ns, int mf);
int group_allreduce_U(Group* G, Ctx* top, cudaStream_t st, bool side = false);
int nccl_comm_split(void* comm, int rank, void** out);      // ncclCommSplit (0 ok; -1 unavailable)

// ---------------------------------------------------------------------------------
// Programmatic dependent launch: a kernel launched with launch_pdl may become resident
// while its predecessor in the stream drains; pdl_wait() (griddepcontrol.wait) blocks
// until the predecessor has completed and its writes are visible, so it must precede
// every read of data the predecessor produced.  pdl_trigger() lets the successor launch.
// Without the launch attribute both are no-ops.
// ---------------------------------------------------------------------------------
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

bool pdl_enabled();

// Set a kernel's dynamic shared-memory limit once per device (function attributes are
// per device): `mask` is the caller's static bitmask of devices already done.
template <class K>
inline cudaError_t smem_attr_once(unsigned long long& mask, K kern, int bytes)
{
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    const unsigned long long bit = 1ull << (dev & 63);
    if (mask & bit) return cudaSuccess;
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e == cudaSuccess) mask |= bit;
    return e;
}

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl_if(bool on, void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                                 Args&&... args)
{
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = (on && pdl_enabled()) ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args&&... args)
{
    return launch_pdl_if(true, kern, grid, block, smem, st, std::forward<Args>(args)...);
}

// host-side precompute (api.cu)
void make_line_coef(LineCoef* C, SchurInv* S, int64_t N, int L, double c, double a, double b, int mean_fix,
                    double* ext_host = nullptr);   // ext_host: 4 (L-1) doubles when L > kMaxL

// launchers (fluid.cu)
cudaError_t launch_s1_x(Ctx* s, int first_step);             // Steps 3a-3c: p*, momentum, x sweep
bool divn_fused(const Ctx* s);                               // S1 stores D.u^n for the first psi pass
cudaError_t launch_sweep_mid(Ctx* s, int axis);              // Step 3d: a middle Douglas sweep
cudaError_t launch_sweep_last(Ctx* s, int axis);             // last Douglas sweep, u^{n+1} = u^n + delta
cudaError_t launch_div_psi_first(Ctx* s, int axis);          // Step 3e RHS + first psi factor + q (3f)
cudaError_t launch_psi_mid(Ctx* s, int axis);                // middle psi factor (3D)
cudaError_t launch_psi_last_x(Ctx* s);                       // last psi factor, p = q + psi, p* = p + psi
cudaError_t launch_line_solve(Ctx* s, int axis, int sys, double* data);  // stand-alone solve
cudaError_t launch_sub(Ctx* s, const double* a, const double* b, double* out);  // out = a - b
// IB (ib.cu)
cudaError_t launch_interp_evolve(Ctx* s, int first_step);    // Steps 1a-1c
cudaError_t launch_force(Ctx* s);                            // Step 2a
cudaError_t launch_spread(Ctx* s);                           // Step 2b (into G, and f in debug mode)
cudaError_t launch_check_finite(Ctx* s, int* flag);          // u, p (if held) and X non-finite -> *flag = 1
cudaError_t launch_check_domain(Ctx* s, int* flag);          // a point moved > h in one step -> *flag = 1
cudaError_t launch_scatter_pts(Ctx* s, const double* src, double* dst);   // internal -> caller order
// z-slab IB (slab.cu calls): the listed points, restricted to slab s's planes
cudaError_t launch_interp_part(Ctx* top, Ctx* s, double* Upart, const int* list, const int* count);
cudaError_t launch_spread_part(Ctx* top, Ctx* s, const int* list, const int* count);

}  // namespace ibgm
