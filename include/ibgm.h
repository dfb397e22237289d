/*
 * ibgm.h -- C-ABI of the B200-native IB-GM hot path.
 *
 * The method: the immersed-boundary / Guermond-Minev (IB-GM) time step of
 * Wiens & Stockie, "An Efficient Parallel Immersed Boundary Algorithm using a
 * Pseudo-Compressible Fluid Solver", arXiv:1305.3976, Section 3.4, Steps 1a-3f
 * (PAPER.md:574-697), on a periodic MAC grid in 2D or 3D,
 * coupled to an elastic force-connection network through a
 * 4-point delta kernel.
 *
 * Conventions common to every entry point
 *   - Return value: IB_OK (0) or a negative IB_E* code; ib_last_error() returns a
 *     thread-local message for the last failure.  No exception crosses the ABI.
 *   - Host pointers: every pointer argument is a caller-owned HOST buffer.  Inputs
 *     are copied during the call; outputs are written into caller-allocated
 *     buffers of the documented size before the call returns.
 *   - Field layout: a field of the N^d grid is N^d doubles, x fastest:
 *     flat index i + N*(j + N*k).  u (x-velocity) lives at (i h, (j+1/2) h, (k+1/2) h),
 *     v at ((i+1/2) h, j h, (k+1/2) h), w at ((i+1/2) h, (j+1/2) h, k h), p and psi at
 *     cell centres ((i+1/2) h, ...) with h = H/N.
 *   - Lagrangian arrays: X, U are [npts][dim] doubles (point-major), unwrapped
 *     positions (only grid indices wrap periodically).
 *   - Device memory and the CUDA stream are owned by the context (unless a stream
 *     is passed in ib_options.stream); all device work of a call is ordered on that
 *     stream.  Calls on one context are not thread-safe.
 *   - Z-slab decomposition (nranks > 1): the grid is cut along its
 *     last axis (z in 3D, y in 2D) into nranks slabs of nz = N/nranks planes; rank r
 *     owns global planes [r nz, (r+1) nz) (ib_slab_range).  Lines along the cut axis
 *     are solved by the paper's Schur-complement splitting across ranks
 *     (PAPER.md:1025-1276); halos move by NCCL.  Lagrangian arrays
 *     are replicated and always global.  Field arrays are:
 *       transport IB_TRANSPORT_NCCL    the rank's LOCAL slab, N^{d-1} * nz doubles
 *                                      (same x-fastest layout, planes z0 .. z0+nz-1);
 *       transport IB_TRANSPORT_EMULATE the GLOBAL N^d field: the context holds all
 *                                      nranks slabs on one GPU and runs the same
 *                                      per-slab kernels and exchanges (copies) in the
 *                                      same order -- the single-GPU test vehicle of
 *                                      the decomposition.
 */
#ifndef IBGM_H
#define IBGM_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define IB_OK 0
#define IB_EINVAL (-1)      /* invalid argument (dim, N, dt, rho, nu, chi, edge index ...) */
#define IB_ESTATE (-2)      /* call out of order (ib_step before ib_set_fields, ...)           */
#define IB_ECUDA (-3)       /* a CUDA runtime call failed (message names it)                  */
#define IB_ENCCL (-4)       /* NCCL could not be loaded or an NCCL call failed                */
#define IB_ENONFINITE (-5)  /* NaN/Inf in u, p or X (ib_check_finite, or the in-step check)    */
#define IB_EDOMAIN (-6)     /* an IB point moved more than one cell h in one step, so its
                               4-point support left the halo a step assumes (
                               an explicit-coupling stability failure: reduce dt)            */
#define IB_ENOMEM (-7)      /* device allocation failed                                       */
#define IB_EDEGENERATE (-8) /* a force connection with rest length L != 0 has zero length
                               |X_m - X_k| = 0: singular strain                 */

#define IB_TRANSPORT_NCCL 0     /* one slab per process, one process per GPU (nranks > 1) */
#define IB_TRANSPORT_EMULATE 1  /* all nranks slabs in this context, one GPU               */

#define IB_DELTA_COS4 0     /* phi(r) = (1 + cos(pi r/2))/4, |r| < 2: BASELINE.json configs */
#define IB_DELTA_PESKIN4 1  /* the paper's kernel, eq. (discretedelta)    */

typedef struct ib_ctx ib_ctx; /* opaque; owned by the library until ib_destroy */

typedef struct {
    int32_t dim; /* 2 or 3 */
    int64_t n;   /* cells per side N; must have a divisor L in {2,3,4,6,8,12,16,24,32}
                    (or 64, 128 in 2D) with N/L <= 32 (line-solve segmentation);
                    8 <= N <= 1024 in 3D, <= 4096 in 2D                                */
    double H;    /* box side H > 0 (1 in every BASELINE config); h = H/N in every
                    operator, including the literal psi operator (1 - D_aa),
                    D_aa = delta_aa/h^2 (R2); positions live in [0, H)^d */
} ib_grid;

typedef struct {
    int32_t kernel;    /* IB_DELTA_COS4 (default) | IB_DELTA_PESKIN4                  */
    double chi;        /* rotational correction weight chi in (0,1], default 0.6
                                                                      */
    int32_t advection; /* 1 (default): skew-symmetric advection;
                          0: Stokes mode (closed-form tests)                            */
    int32_t device;    /* CUDA ordinal, default 0                                       */
    void* stream;      /* cudaStream_t to order all work on, or NULL (own stream)       */
    int32_t rank;      /* z-slab rank in [0, nranks) (NCCL transport; 0 otherwise)     */
    int32_t nranks;    /* number of z-slabs, default 1 (no decomposition); N % nranks
                          == 0 and N/nranks >= 2.  nranks = 1 with transport EMULATE or
                          with an nccl_id runs the slab code path on one slab (a 1-rank
                          communicator for NCCL: tests the transport on one GPU)        */
    int32_t transport; /* IB_TRANSPORT_NCCL (default) | IB_TRANSPORT_EMULATE            */
    const void* nccl_id; /* NCCL transport, nranks > 1: the 128-byte unique id that rank 0
                          obtained from ib_nccl_unique_id and shared with every rank
                          (e.g. a torch.distributed broadcast); read during ib_create */
} ib_options;

/* Fill *opt with the defaults listed above. */
void ib_default_options(ib_options* opt);

/* Create a context for the grid with kinematic viscosity nu = mu/rho, density rho
 * and time step dt (epsilon = dt).  Allocates every device
 * buffer and precomputes the line-solver factors.  *out receives the context.
 * With nranks > 1 and the NCCL transport every rank calls ib_create collectively
 * (ncclCommInitRank on device `device`).
 * Errors: IB_EINVAL (dim not 2/3, N unsupported, H <= 0, dt <= 0, rho <= 0, nu < 0,
 * chi not in (0,1], N % nranks != 0, N/nranks < 2, rank out of range, NCCL transport
 * without nccl_id), IB_ENCCL, IB_ECUDA, IB_ENOMEM. */
int ib_create(const ib_grid* grid, double nu, double rho, double dt, const ib_options* opt,
              ib_ctx** out);

/* Set the initial state: velocity u^0, v^0, (w^0: NULL in 2D) on the MAC faces and
 * pressure p^{-1/2} (NULL -> 0); psi^{-1/2} = 0 and the step counter is reset to 0,
 * which arms the start-up rules of PAPER.md:686-697.  Each array is N^d doubles.
 * The immersed boundary keeps its current position X^n (the one ib_get_fields
 * returns); a look-ahead IB phase already run for the next step is undone.  Clears
 * raised faults. */
int ib_set_fields(ib_ctx* ctx, const double* u, const double* v, const double* w,
                  const double* p);

/* Set the immersed boundary as a force-connection network:
 * X[npts][dim] positions; edges[nedges][2] point indices; kappa[nedges] stiffness;
 * rest[nedges] rest lengths (NULL -> 0); weight[npts] quadrature weights w_k used
 * by spreading (NULL -> 1).  Edge e=(a,b) exerts F_a += kappa_e (X_b - X_a)
 * (1 - rest_e/|X_b - X_a|) and the opposite on b (Step 2a).  A closed 2D fibre of
 * PAPER.md:607-614 is kappa = sigma/h_s^2, rest = L h_s, weight = h_s.  Resets the
 * step counter to 0.  Errors: IB_EINVAL (edge index out of range, npts < 0). */
int ib_set_boundary(ib_ctx* ctx, int64_t npts, const double* X, int64_t nedges,
                    const int64_t* edges, const double* kappa, const double* rest,
                    const double* weight);

/* BASELINE.json's ib_set_boundary(X, stiffness) for closed 2D fibres: n_fibers
 * closed fibres, fibre f has pts_per_fiber[f] consecutive points in X, stiffness
 * sigma, rest length 0; builds kappa = sigma/h_s^2, weight = h_s, h_s = 1/pts. */
int ib_set_fibers(ib_ctx* ctx, int32_t n_fibers, const int64_t* pts_per_fiber,
                  const double* X, double sigma);

/* Advance nsteps time steps (Steps 1a-3f each).  All work is enqueued on the
 * context's stream; the call returns after enqueueing (use ib_sync to wait).
 * Device-detected faults are sticky: the force kernel raises IB_EDEGENERATE (a
 * connection with L != 0 and zero length; its force is dropped instead of spreading
 * NaN), and every K-th step (ib_set_check_interval, default K = 100) a state check
 * raises IB_ENONFINITE (NaN/Inf in u, p or X) or IB_EDOMAIN (a point moved more than
 * h).  A raised fault is returned by the first ib_step / ib_sync / ib_get_state after
 * the kernel that raised it has run (ib_step checks on entry and after enqueueing,
 * without waiting), and by every later ib_step until ib_set_fields, ib_set_state or
 * ib_set_boundary clears it.  With the NCCL transport each rank detects its own
 * faults; a rank that reports one must abort the job (the others would wait in the
 * next collective).  Errors: IB_ESTATE (no ib_set_fields yet), IB_ECUDA, IB_ENCCL,
 * IB_EDEGENERATE, IB_ENONFINITE, IB_EDOMAIN. */
int ib_step(ib_ctx* ctx, int64_t nsteps);

/* Run the in-step state check (see ib_step) every `every` steps; 0 turns it off.
 * Default 100.  The check reads u, p and X once (~4 fields of traffic).
 * Errors: IB_EINVAL (every < 0). */
int ib_set_check_interval(ib_ctx* ctx, int64_t every);

/* Block until all work enqueued on the context's stream has completed; then return
 * any device-raised fault (see ib_step). */
int ib_sync(ib_ctx* ctx);

/* Checkpoint / resume: the complete state the next step reads (u^n, the momentum
 * history G = N(u^{n-1}) [+ (2/rho) f^{n+3/2} once the look-ahead ran], p^{n-1/2},
 * p* = p^{n-1/2} + psi^{n-1/2}, X^n, U^{n-1}, the look-ahead's X^{n+1}/U^n, the step
 * counter) as an opaque host blob of ib_state_size bytes, valid for a context with the
 * same grid, parameters, decomposition and rank and the same immersed boundary
 * (ib_set_boundary with the same points).  ib_set_state followed by ib_step(k) gives
 * bit for bit the steps the saving context would have taken (same kernels, same
 * order; spreading atomics aside, R18).  Both synchronise the stream
 * before returning (the buffer may be reused at once).  ib_set_state clears any
 * raised fault.  Errors: IB_EINVAL (null, buffer too small, blob of another
 * grid/parameters/decomposition/boundary), IB_ESTATE (ib_get_state before
 * ib_set_fields), IB_ECUDA. */
int ib_state_size(ib_ctx* ctx, int64_t* bytes);
int ib_get_state(ib_ctx* ctx, void* buf, int64_t bytes);
int ib_set_state(ib_ctx* ctx, const void* buf, int64_t bytes);

/* Copy the state to host buffers (any pointer may be NULL): u^n, v^n, w^n,
 * p^{n-1/2}, psi^{n-1/2} (N^d each), X^n and U^{n-1} (the velocity interpolated in
 * the last step) ([npts][dim]).  Synchronises the stream. */
int ib_get_fields(ib_ctx* ctx, double* u, double* v, double* w, double* p, double* psi,
                  double* X, double* U);

/* Intermediates of the last step (any pointer may be NULL): the spread force
 * f^{n+1/2} per component (N^d each; requires ib_set_debug bit 0 before the step,
 * else IB_ESTATE), the stored advection N(u^n) per component,
 * the Lagrangian force F^{n+1/2} and X^{n+1/2} ([npts][dim]).  F is the force of
 * Step 2a BEFORE the quadrature weight is applied.  Without ib_set_debug bit 0 the
 * single-GPU path runs the IB phase (Steps 1-2) of step n+1 concurrently with the psi
 * passes of step n, so F, X^{n+1/2} and the history then already belong to the next
 * step; set bit 0 (before stepping) to inspect the intermediates of each step. */
int ib_get_aux(ib_ctx* ctx, double* fu, double* fv, double* fw, double* nu, double* nv,
               double* nw, double* F, double* Xh);

/* Stand-alone batched cyclic tridiagonal solve on the GPU (the line solver of
 * PAPER.md:946-1276 used by every step): for every grid line of the N^d array `d`
 * along `axis` (0 = x, 1 = y, 2 = z) solve  c x_{i-1} + a x_i + c x_{i+1} = d_i
 * (indices mod N) with a = 1 + 2 kappa, c = -kappa, and write x (N^d, may alias d).
 * Uses the same kernels, segmentation and mean correction as ib_step.  Host buffers.
 * On a z-slab context, d and x follow the field convention above and `axis` must be
 * the cut axis (dim-1): the lines are solved with the cross-rank Schur splitting
 * (collective across ranks with the NCCL transport).
 * Errors: IB_EINVAL (kappa < 0, axis >= dim, slab context and axis != dim-1). */
int ib_line_solve(ib_ctx* ctx, int32_t axis, double kappa, const double* d, double* x);

/* Stand-alone directional-split solve (eq. PoissonGMProblem with
 * A = (1 - D_xx)(1 - D_yy)[(1 - D_zz)], D_aa = delta_aa / h^2, H = 1): copies the
 * cell-centred right-hand side f (N^d doubles, host) to the device, applies A^{-1}
 * `repeats` times in place (each application = one batched cyclic line pass per axis,
 * the same kernels and mean correction as the psi factors of ib_step), and copies
 * A^{-repeats} f to psi (host; may alias f).  *device_ms (may be NULL) receives the
 * average device time of one application, measured with CUDA events on the context's
 * stream around the line passes only.  Single-GPU contexts only.
 * Errors: IB_EINVAL (repeats < 1, null f/psi, slab context). */
int ib_psi_solve(ib_ctx* ctx, const double* f, double* psi, int32_t repeats, double* device_ms);

/* Synchronous device-side finiteness check of u, p and X now; IB_ENONFINITE if any
 * NaN/Inf (independent of the sticky in-step faults). */
int ib_check_finite(ib_ctx* ctx);

/* Statistics (any pointer may be NULL): ms_per_phase[IB_NPHASES] the average device
 * milliseconds per step of each phase over the steps timed since ib_set_profiling(1)
 * (0 for phases never timed; see the IB_PH_* list), the number of completed steps, and
 * the number of kernels this library launched since the context was created. */
int ib_get_stats(ib_ctx* ctx, double* ms_per_phase, int64_t* steps_done, int64_t* kernel_launches);

/* Phases of one step, for ib_get_phase_times (one kernel launch each). */
#define IB_PH_INTERP 0   /* Steps 1a-1c: interpolate U^n, evolve X                         */
#define IB_PH_FORCE 1    /* Step 2a: force-connection forces                              */
#define IB_PH_SPREAD 2   /* Step 2b: spread F into the momentum history                    */
#define IB_PH_S1 3       /* Steps 3a-3c: p*, explicit momentum, x sweep                    */
#define IB_PH_SWEEP_Y 4  /* Step 3d: y sweep (2D: the last sweep, u^{n+1} = u^n + d)       */
#define IB_PH_SWEEP_Z 5  /* z sweep, u^{n+1} = u^n + d (3D)                                */
#define IB_PH_DIVPSI 6   /* Step 3e RHS D.u^{n+1} + first psi factor + explicit part of 3f */
#define IB_PH_PSI_Y 7    /* psi factor (1 - D_yy) (3D)                                      */
#define IB_PH_PSI_X 8    /* psi factor (1 - D_xx) + Step 3f p = q + psi, p* = p + psi      */
#define IB_PH_CLEAR 9    /* history clear at n = 0 and debug clears                        */
#define IB_NPHASES 10

/* Debug flags: bit 0 keeps the spread force f^{n+1/2} as a separate field so that
 * ib_get_aux can return it (costs one extra atomic per spread contribution and a
 * clear per step).  Bits 1-3 select the spreading method: 0 automatic (6 in 3D,
 * 4 in 2D),
 * 1 one thread per point (4^d global fp64 reductions per component), 2 brick-binned
 * (points counting-sorted into 4^3-cell bricks every step, shared-memory tiles),
 * 3 box-staged (chunks of 64 consecutive points accumulate in a shared-memory box,
 * one global reduction per box node), 4 quad-lane (4 lanes per point and component,
 * one per x-node of a stencil row, so each warp reduction is coalesced), 5 quad-lane
 * with a warp pre-reduction (consecutive points of a warp with the same base node sum
 * their contributions by shuffles and one lane group issues the reductions), 6 window-
 * staged (a warp accumulates the contributions of 32 consecutive points into a
 * shared-memory box of their supports without atomics, then one global reduction per
 * non-zero box node).  Bits 4-6
 * select the interpolation: 0 automatic (3 in 2D, 5 in 3D), 1 one thread per point, 2 box-staged,
 * 3 quad-lane, 4 one thread per (point, component), 5 window-staged (a warp loads the
 * box of u covering the supports of 32 consecutive points into shared memory once).  The points are kept internally in Morton order of their initial
 * cells (outputs are returned in the caller's order).  Automatic by default.  Only
 * the single-GPU path honours bits 1-6.  Set bit 0 before the first ib_step (or right
 * after ib_set_fields): once the look-ahead has run the next step's IB phase, turning
 * it on returns IB_ESTATE.  Errors: IB_EINVAL (spreading method > 6, interpolation
 * method > 5, or a bit above 6 set). */
int ib_set_debug(ib_ctx* ctx, int32_t flags);

/* Turn per-phase CUDA-event timing on (1) or off (0).  While on, ib_step records an
 * event pair around every phase on the context's stream and synchronises at the end
 * of each ib_step call to accumulate the elapsed times; turning it on resets them. */
int ib_set_profiling(ib_ctx* ctx, int32_t on);

/* Accumulated milliseconds and launch counts per phase (arrays of IB_NPHASES). */
int ib_get_phase_times(ib_ctx* ctx, double* ms, int64_t* count);

/* Write a fresh 128-byte NCCL unique id into out[128] (call on rank 0 only, then
 * share it).  Loads NCCL at run time (the copy already in the process if any).
 * Needs no GPU.  Errors: IB_EINVAL (null), IB_ENCCL (NCCL missing or failed). */
int ib_nccl_unique_id(void* out);

/* Global first plane z0 and depth nz of rank `rank`'s slab of an N-cell axis cut into
 * nranks slabs (z0 = rank N/nranks, nz = N/nranks).  Host-only arithmetic.
 * Errors: IB_EINVAL (N % nranks != 0, N/nranks < 2, rank out of range). */
int ib_slab_range(int64_t n, int32_t nranks, int32_t rank, int64_t* z0, int64_t* nz);

/* Release every device buffer, the stream (if owned) and the context. */
int ib_destroy(ib_ctx* ctx);

/* Thread-local message describing the last non-zero return of this thread. */
const char* ib_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* IBGM_H */
