/*
 * stencil_b200.h — C-ABI of the B200-native folded stencil sweep
 * (arXiv 2103.09235, "Reducing Redundancy in Data Organization and Arithmetic
 * Calculation for Stencil Computations").
 *
 * Citations: P:<line> = /reference PAPER.md line; S:<line> = SPEC.md line.
 *
 * The operation (§1): a d-dimensional grid updated iteratively in time;
 * "the value of one point at time t is a weighted sum of itself and its
 * neighboring points at the previous time":
 *
 *     u^{t+1}[p] = sum_j w_j * u^t[p + o_j]            (correlation form, the
 *                                                       v_{i+t} index of Eq.4,
 *                                                       P:385; R3)
 *
 * Temporal computation folding (§3.2-3.3, Eq.2, Eq.4-6):
 * m time steps are applied as ONE sweep with the reassigned weights
 * lambda^(m) = w * w * ... * w (the m-fold self-convolution of the tap map;
 * P:335 "weights are all reassigned based on the m-step expansion").
 *
 * Boundary (the paper is silent — DESIGN.md reading R1): FIXED = an r-wide
 * ring around the interior that holds u0 and is never updated.  The folded
 * weights are not valid within (m-1)*r of a FIXED face (R2); the
 * library evaluates that band step by step, exactly.
 *
 * Conventions for every entry point:
 *  - Return value: STENCIL_OK (0) or a negative stencil_status.  Nothing
 *    aborts or throws across this boundary.  On error, stencil_last_error()
 *    returns a thread-local message.
 *  - Device pointers are CUDA device pointers on the current device; they are
 *    OWNED BY THE CALLER (PyTorch is the only allocator).  Host pointers are
 *    plain host memory, owned by the caller.
 *  - `stream` is a cudaStream_t (NULL = legacy default stream).  Runs are
 *    asynchronous on it; kernel faults surface at the caller's next
 *    synchronisation, as with any CUDA library.  A plan owns device scratch
 *    for its sweep schedule, so the runs of ONE plan must be ordered (one
 *    stream, or streams synchronised by the caller); different plans run
 *    concurrently.  A plan is not thread-safe for concurrent calls.
 *  - CUDA graphs: runs may be captured (cudaStreamBeginCapture) and replayed.
 *    A captured 2D/3D sweep zeroes the plan's schedule scratch before and
 *    after its kernel (memset nodes), so replays do not depend on the launch
 *    order.  Run the same call once eagerly before capturing it (the scratch
 *    may have to grow, which is not allowed while capturing: EUNSUPPORTED).
 *    A graph is valid while its plan lives and the scratch does not grow
 *    (a later eager call on a larger domain reallocates it).
 *  - Axes are listed slowest first (z, y, x); x has unit stride.
 */
#ifndef STENCIL_B200_H
#define STENCIL_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define STENCIL_MAX_DIMS 3
#define STENCIL_MAX_FOLD 8
/* Largest counterpart count (rank) the 2D counterpart evaluation is compiled for. */
#define STENCIL_MAX_COUNTERPARTS 2

typedef enum {
    STENCIL_OK = 0,
    STENCIL_EINVAL = -1,        /* bad argument (dims, radius, ncoeffs, fold_m<1, T<0, null, aliasing, misalignment) */
    STENCIL_EUNSUPPORTED = -2,  /* valid request this build does not compile (e.g. PERIODIC dist runs, fold_m*r too large) */
    STENCIL_ECUDA = -3,         /* CUDA runtime/driver error (message in stencil_last_error) */
    STENCIL_ENCCL = -4,         /* NCCL error or NCCL library not loadable */
    STENCIL_ENOMEM = -5,        /* host allocation failed */
    STENCIL_ETIMEOUT = -6       /* stencil_comm_wait: the stream did not drain in time (comm aborted) */
} stencil_status;

typedef enum { STENCIL_STAR = 0, STENCIL_BOX = 1 } stencil_shape;
typedef enum { STENCIL_F32 = 0, STENCIL_F64 = 1 } stencil_dtype;
typedef enum { STENCIL_BC_FIXED = 0, STENCIL_BC_PERIODIC = 1 } stencil_boundary;

typedef struct stencil_plan_s *stencil_plan;
typedef struct stencil_comm_s *stencil_comm;

/*
 * Buffer layout the library requires.  The caller allocates
 * `bytes` bytes (device, >= 256-byte aligned as cudaMalloc/PyTorch give) and
 * addresses interior point (i_0, .., i_{d-1}) at element index
 *     sum_a (origin[a] + i_a) * stride[a].
 * The physical ring occupies interior coordinates [-r, 0) and [N_a, N_a + r)
 * on every axis.  The unit-stride axis has a left pad so interior x = 0 is
 * 128-byte aligned, and its row pitch (stride of the next axis) is a multiple
 * of 128 bytes (TMA needs 16-byte multiples).  Pad cells outside the ring are
 * never used for any result.  For dist layouts (stencil_plan_layout_dist)
 * axis 0 carries `halo` ghost planes on each side instead of the ring; at the
 * global ends the r planes next to the interior are the physical ring.
 */
typedef struct {
    int ndim;
    int radius;               /* r */
    int64_t interior[STENCIL_MAX_DIMS]; /* N_a (local N for dist layouts) */
    int64_t extent[STENCIL_MAX_DIMS];   /* allocated extent per axis (elements) */
    int64_t stride[STENCIL_MAX_DIMS];   /* element stride per axis */
    int64_t origin[STENCIL_MAX_DIMS];   /* index of interior coordinate 0 per axis */
    int64_t elem_bytes;       /* 4 (F32) or 8 (F64) */
    int64_t bytes;            /* allocation size */
    int64_t global_offset0;   /* dist: global interior index of local plane 0 on axis 0 (else 0) */
} stencil_layout;

/*
 * Create a plan (host only; no CUDA call).
 *   ndim     1..3; dims[ndim] interior extents, slowest first, each >= 1.
 *   radius   r >= 1.
 *   shape    STAR: taps = offsets in [-r,r]^d with at most one nonzero
 *            coordinate (k = 2dr+1); BOX: all of [-r,r]^d (k = (2r+1)^d)
 *            (SPEC.md:31-32).
 *   coeffs   ncoeffs == k fp64 weights in CANONICAL tap order: offsets in
 *            lexicographic order, slowest axis outermost, each axis -r..r
 *            (R4).  Copied.
 *   dtype    storage + arithmetic type on the GPU.  Folded weights are computed
 *            in fp64 and rounded once to dtype.
 *   boundary FIXED: an r-wide frozen ring holding u0 (R1); PERIODIC
 *            (SURVEY §8(f) NEXT-4): the layout carries a ghost ring of
 *            STENCIL_MAX_FOLD * r cells per side on every axis, refilled from
 *            the wrapped interior after every sweep (single-GPU runs only;
 *            dist layouts/runs return EUNSUPPORTED).
 * Errors: EINVAL on any bad argument.
 */
int stencil_plan_create(stencil_plan *plan, int ndim, const int64_t *dims, int radius,
                        stencil_shape shape, const double *coeffs, int ncoeffs,
                        stencil_dtype dtype, stencil_boundary boundary);
int stencil_plan_destroy(stencil_plan plan);

/* Single-GPU buffer layout (for `in`, `out` and the workspace). */
int stencil_plan_layout(stencil_plan plan, stencil_layout *out);

/* Number of taps k, and the canonical offsets (k * ndim ints, slowest first). */
int stencil_plan_ntaps(stencil_plan plan, int *ntaps);
int stencil_plan_taps(stencil_plan plan, int *offsets, int cap);

/*
 * The library's folding matrix lambda^(m) (Eq.2; the counterpart rows
 * of Eq.4-6) as a dense (2mr+1)^ndim fp64 array, index [o + m r],
 * slowest axis first.  Host only.  cap = capacity in doubles.
 * Errors: EINVAL if m < 1 or cap too small; EUNSUPPORTED if m > STENCIL_MAX_FOLD.
 */
int stencil_plan_fold_coeffs(stencil_plan plan, int m, double *dense, int64_t cap);

/*
 * Counterpart decomposition of the 2D folded weights (
 * vertical/horizontal folding Eq.4-6, counterpart reuse Eq.7
 * P:443-466).  Lambda = lambda^(m) viewed as a W x W matrix (W = 2 m r + 1,
 * rows = offset along axis 0, columns = offset along x) is written as
 *   Lambda[i][j] = sum_{k < rank} a[k W + i] * b[k W + j]
 * by LU with complete pivoting, stopped when the largest residual entry is
 * <= 1e-13 max|Lambda|.  The paper's uniform 2D9P, m = 2 example has rank 1
 * (P:387).  When 2 W rank < |supp Lambda| and rank <=
 * STENCIL_MAX_COUNTERPARTS, stencil_run evaluates the folded pass through the
 * counterparts: each loaded row is folded horizontally with every b_k, and the
 * counterparts are folded vertically with the a_k into the sliding window.
 * rank: out; a, b: caller arrays of `cap` >= rank * W doubles (either may be
 * NULL).  Errors: EINVAL (m < 1, NULL rank, cap too small), EUNSUPPORTED
 * (ndim != 2, m > STENCIL_MAX_FOLD).
 */
int stencil_plan_fold_rank(stencil_plan plan, int m, int *rank, double *a, double *b, int64_t cap);

/*
 * Enable (default) or disable the counterpart evaluation for this plan
 * (disabling forces the dense folded pass; used to compare the two).
 */
int stencil_plan_set_counterparts(stencil_plan plan, int enable);

/*
 * fold_m = 0 in stencil_run / stencil_run_ex / stencil_run_host /
 * stencil_run_dist means "auto": this fold, chosen per family from the B200
 * measurements: 1D 2; 2D FIXED radius 1: 6 for fp64 stars
 * and 8 otherwise (the on-chip temporal block: that many single steps per HBM
 * round trip), or 4 when lambda^(4) has a counterpart decomposition of rank
 * <= 2; 2D PERIODIC: star 3, box 2; 3D FIXED radius-1: star 4, fp64 box 2 (the
 * 3D temporal block); other 3D stars 2, other 3D boxes 1; radius > 1: 1.
 * Errors: EINVAL (NULL).
 */
int stencil_plan_auto_fold(stencil_plan plan, int *fold_m);

/*
 * Fault injection for tests (the mutation idea of S:464): add
 * `delta` to entry `index` of the plan's cached lambda^(m) (dense layout of
 * stencil_plan_fold_coeffs).  Every later run with fold_m = m uses the
 * perturbed weights, so a parity check against the oracle must fail.
 * Errors: EINVAL (NULL, m out of 1..STENCIL_MAX_FOLD, index out of range).
 */
int stencil_plan_perturb_fold(stencil_plan plan, int m, int64_t index, double delta);

/*
 * The evaluation stencil_run(..., fold_m = m, stages = 0) chooses for the
 * main region (the GPU form of the profitability index Eq.3):
 * `stages` passes of lambda^(q) (m = q * stages); rank > 0 = one pass through
 * `rank` counterparts.  Errors: EINVAL (NULL, m < 1), EUNSUPPORTED (m too large).
 */
int stencil_plan_variant(stencil_plan plan, int m, int *q, int *stages, int *rank);

/* Workspace bytes stencil_run needs (one more buffer of the plan's layout). */
int stencil_workspace_size(stencil_plan plan, int64_t *bytes);

/*
 * K-G0: fill a device buffer (plan layout) with the seeded input field
 * u0 = U(seed, i), i = row-major index of the point in the UNALIGNED padded
 * frame prod(N_a + 2r) (R6), over the interior and the ring.  Pads
 * are set to 0.  Async on stream.
 */
int stencil_fill_random(stencil_plan plan, void *buf, uint64_t seed, void *stream);

/*
 * Run T time steps: out = S^T(in), with fold_m steps per sweep (Eq.2; 0 = auto,
 * stencil_plan_auto_fold):
 *   floor(T / fold_m) folded sweeps, then one sweep of fold T mod fold_m
 *   (R10).  Jacobi ping-pong between `out` and `workspace`
 *    arranged so the last sweep writes `out`; `in` is never written.
 *   T = 0 copies in -> out.  Every sweep = the folded interior sweep plus the
 *   stepwise band within (fold_m-1)*r of each face.
 * in, out, workspace: device buffers of the plan layout (workspace may be NULL
 *   when at most one sweep runs).  `out` is fully written, ring included.
 * Errors: EINVAL (T < 0, fold_m < 1, null/aliased/misaligned pointers),
 *   EUNSUPPORTED (fold_m > STENCIL_MAX_FOLD), ECUDA.  PERIODIC plans need a
 *   workspace for every T > 0 (`in` is copied into the ping-pong first).
 */
int stencil_run(stencil_plan plan, const void *in, void *out, int64_t T, int fold_m,
                void *workspace, void *stream);

/*
 * As stencil_run, selecting the on-chip evaluation of each m-step sweep:
 *   stages = 1 : the folded sweep (one pass of lambda^(m), §3.3);
 *   stages = m : the on-chip m-step temporal block (m single steps per tile,
 *                "time loop fusion");
 *   1 < stages < m, stages | m : stages on-chip passes of lambda^(m/stages);
 *   stages = 0 : the plan's choice (FMA-vs-byte budget).
 * Results are identical up to fp rounding for every choice.
 */
int stencil_run_ex(stencil_plan plan, const void *in, void *out, int64_t T, int fold_m,
                   int stages, void *workspace, void *stream);

/*
 * End-to-end call with HOST buffers (for the e2e measurement): copies
 * in_host (plan layout, pinned recommended) -> dev_in, runs stencil_run_ex,
 * copies dev_out -> out_host, all enqueued on `stream`.  Does not synchronise.
 */
int stencil_run_host(stencil_plan plan, const void *in_host, void *out_host, int64_t T,
                     int fold_m, int stages, void *dev_in, void *dev_out, void *workspace,
                     void *stream);

/*
 * A batch of `nbatch` independent problems from HOST memory (the e2e path of
 * the measurement): problem k copies in_hosts[k] -> device, runs
 * stencil_run_ex(T, fold_m, stages) and copies the result -> out_hosts[k].
 * Pipelined: the library's two internal copy streams overlap problem k's
 * H2D and problem k-2's D2H with problem k-1's run on `stream`, using two
 * device buffer sets alternately.  dev = 6 device pointers {in0, out0, ws0,
 * in1, out1, ws1} of the plan layout (set 1 unused when nbatch == 1; ws may
 * be NULL when a run needs no workspace).  Host buffers: plan layout, pinned
 * (page-locked) for the copies to be asynchronous.  Ordered after prior work
 * on `stream`; `stream` waits for every copy of the batch, so synchronising
 * it makes all out_hosts valid.  Errors: EINVAL (NULL), as stencil_run_ex, ECUDA.
 */
int stencil_run_host_batch(stencil_plan plan, int nbatch, const void *const *in_hosts,
                           void *const *out_hosts, int64_t T, int fold_m, int stages,
                           void *const *dev, void *stream);

/*
 * Dynamic-schedule controls and counters of the 2D/3D sweep (tests and
 * tuning).  The persistent CTAs claim `chunk`-plane pieces of their own column
 * segment, then grab never-started segments, then steal the upper half of the
 * largest remaining segment if it has at least `min_steal` planes
 * (DESIGN.md §5.1); max_ctas > 0 caps the persistent grid (so CTAs must
 * grab).  stencil_plan_set_schedule(plan, 0, 0, 0) restores the defaults.
 * stencil_plan_sched_stats returns the successful grabs and steals
 * counted by the kernels since the plan's scratch was allocated or last reset
 * (synchronous device read; reset != 0 zeroes them).
 * Errors: EINVAL (NULL, negative values), ECUDA.
 */
int stencil_plan_set_schedule(stencil_plan plan, int chunk, int min_steal, int max_ctas);
int stencil_plan_sched_stats(stencil_plan plan, int64_t *grabs, int64_t *steals, int reset);

/* Number of kernel launches the last run on this plan enqueued (host count). */
int stencil_plan_last_launches(stencil_plan plan, int64_t *launches);

/*
 * Measurement support.  While timing is enabled, every kernel launch of the
 * main-region sweep (kind 0; the 1D on-chip kernel for ndim = 1) and of the
 * boundary band (kind 1) is bracketed by CUDA events recorded on the launch
 * stream.  stencil_plan_timing waits for those events and returns, for one
 * kind, the summed kernel time (ms), the number of launches, the algorithmic
 * bytes (2 * elem_bytes per output point: one read + one write per sweep) and
 * the algorithmic FMAs (per output point: stages * |supp lambda^(q)|) of the
 * launches recorded since the last reset.  Host only bookkeeping + event sync.
 */
int stencil_plan_set_timing(stencil_plan plan, int enable);
int stencil_plan_timing(stencil_plan plan, int kind, double *ms, int64_t *launches, int64_t *bytes,
                        int64_t *fmas);
int stencil_plan_timing_reset(stencil_plan plan);

/* ---------------------------------------------------------------- multi-GPU
 * Slab decomposition along axis 0 (the slowest axis), one process per GPU
 * (SURVEY §8(e)).  Rank g owns interior planes [g*N0/G, (g+1)*N0/G) plus
 * `halo` ghost planes per side (halo >= fold_m * r for every run).  Per sweep
 * the first/last fold_m*r local planes are computed first and exchanged with
 * rank g-1 / g+1 (grouped ncclSend/ncclRecv on a comm stream) while the rest
 * of the slab is computed.  Slab seams are not physical faces: no band there.
 */

/* 128-byte NCCL unique id (rank 0 creates, caller broadcasts). */
int stencil_comm_unique_id(unsigned char id[128]);
/* Create a communicator on the current CUDA device. */
int stencil_comm_create(stencil_comm *comm, const unsigned char id[128], int rank, int nranks);
int stencil_comm_destroy(stencil_comm comm);

/* Local layout of rank `rank` of `nranks` with `halo` ghost planes.
 * EINVAL if N0 is not divisible by nranks or a slab is thinner than halo. */
int stencil_plan_layout_dist(stencil_plan plan, int rank, int nranks, int halo,
                             stencil_layout *out);

/* K-G0 for a local slab: the same global field, ghost planes included. */
int stencil_fill_random_dist(stencil_plan plan, int rank, int nranks, int halo, void *buf,
                             uint64_t seed, void *stream);

/*
 * Distributed run.  in_local / out_local / workspace: local slab buffers
 * (stencil_plan_layout_dist with the same halo).  in_local's ghost planes must
 * hold the neighbours' planes (stencil_fill_random_dist provides that, or call
 * stencil_halo_exchange first).  All ranks call collectively.
 */
int stencil_run_dist(stencil_plan plan, stencil_comm comm, const void *in_local,
                     void *out_local, int64_t T, int fold_m, int stages, int halo,
                     void *workspace, void *stream);

/* Exchange the ghost planes of a local slab buffer (collective).  NCCL comms
 * only (a peer comm returns EINVAL: its ghosts are written by the sweep). */
int stencil_halo_exchange(stencil_plan plan, stencil_comm comm, void *buf, int halo,
                          void *stream);

/*
 * Diagnostic: the per-sweep NCCL exchange of stencil_run_dist (the same
 * grouped ncclSend/ncclRecv calls, counts, datatype and plane addresses) with
 * THIS rank as both neighbours, so the transport can be exercised on a box
 * with one GPU (a 1-rank communicator has no neighbours otherwise).  Within
 * the group, sends and receives to one peer match in issue order: afterwards
 * buf's lower ghost planes [-halo, 0) hold its planes [0, halo) and its upper
 * ghost planes [n0, n0 + halo) hold its planes [n0 - halo, n0).  NCCL comms
 * only (EINVAL for a peer comm, a slab thinner than halo, or a halo beyond the
 * planes the rank's layout holds outside its slab: ghost planes, or the
 * r-ring at a physical face, which this call overwrites); every rank that
 * calls it exchanges with itself only (not collective).
 */
int stencil_halo_exchange_loopback(stencil_plan plan, stencil_comm comm, void *buf, int halo,
                                   void *stream);

/*
 * Failure detection.  Wait until `stream` has drained, polling
 * the NCCL communicator's asynchronous error (ncclCommGetAsyncError) every
 * 0.2 ms.  On an asynchronous NCCL error the communicator is aborted
 * (ncclCommAbort) and ENCCL is returned; if the stream has not drained after
 * timeout_ms (< 0: no limit) the communicator is aborted and ETIMEOUT is
 * returned.  An aborted comm makes every later run/exchange on it return
 * ENCCL.  Every NCCL call inside run_dist/halo_exchange is checked and the
 * async error is also polled before each exchange.  Host-blocking.
 */
int stencil_comm_wait(stencil_comm comm, void *stream, int64_t timeout_ms);

/*
 * Fused halo exchange over peer memory (one process per
 * GPU, NVLink/NVSwitch peers).  Instead of an NCCL kernel per sweep, the sweep
 * kernel stores the outputs of its first/last fold_m*r planes a second time,
 * straight into the neighbours' ghost planes (CUDA IPC peer pointers), so the
 * transfer overlaps the math tile by tile; GPUs order their sweeps with
 * stream memory operations on small flag words (cuStreamWriteValue32 after
 * each sweep, cuStreamWaitValue32 before the next: no spinning kernel).
 *   1. stencil_comm_create_peer(&c, rank, nranks, buf0, buf1): buf0/buf1 =
 *      this rank's ping-pong buffers; every run on every rank must pass
 *      buf0 as `out` and buf1 as `workspace` (a rank stores into the
 *      neighbour's buffer of the same registered index; EINVAL otherwise);
 *   2. stencil_comm_peer_handles(c, rec): writes 3 * STENCIL_PEER_HANDLE_BYTES;
 *   3. all-gather the records (rank order) and stencil_comm_peer_attach(c, all);
 *   4. stencil_run_dist(plan, c, ...) as with an NCCL comm.  Every sweep,
 *      the last one included, stores into the neighbours' ghost planes, so
 *      after the run out_local's ghosts hold the neighbours' final planes and
 *      a copy of out_local (ghosts included) is a complete in_local for a
 *      chained run.  Between runs all ranks must synchronise (stream sync +
 *      process barrier) before touching their buffers.
 * Errors: EINVAL (NULL, bad rank, buffers not the registered pair), ECUDA
 * (IPC / stream memory operations unavailable or failing).
 */
#define STENCIL_PEER_HANDLE_BYTES 72
int stencil_comm_create_peer(stencil_comm *comm, int rank, int nranks, void *buf0, void *buf1);
int stencil_comm_peer_handles(stencil_comm comm, unsigned char *out);
int stencil_comm_peer_attach(stencil_comm comm, const unsigned char *all);

/*
 * The same distributed algorithm with all `nranks` ranks in THIS process on
 * the current device (identical kernels, boxes and ordering; used by tests on
 * one GPU).  exchange = 0: the NCCL path's schedule, its transport done with
 * device-to-device copies; exchange = 1: the fused peer-store path (the
 * neighbours' buffers are plain device pointers here).  Arrays of nranks
 * pointers.
 */
int stencil_run_dist_emulated(stencil_plan plan, int nranks, const void *const *in_locals,
                              void *const *out_locals, int64_t T, int fold_m, int stages,
                              int halo, void *const *workspaces, int exchange, void *stream);

/* Thread-local message for the last error on this thread ("" if none). */
const char *stencil_last_error(void);

/* Library version string. */
const char *stencil_version(void);

#ifdef __cplusplus
}
#endif
#endif /* STENCIL_B200_H */
