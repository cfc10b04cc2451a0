/*
 * pft.h — C ABI of the B200-native PROFusion tracking-and-fusion hot path
 * (arXiv 2509.24236).  "pft" = particle fitness tracker.
 *
 * The calls follow the paper's statement of the problem (BASELINE.json north_star):
 *   volume_create / reset            the TSDF scene representation   (§III "Method overview")
 *   integrate(depth, K, T)           KinectFusion fusion of a frame
 *   track(depth, K, T_init, pst, iters) -> T and per-particle fitness
 *                                    randomized optimization          (§III-B)
 *   eval_poses(depth, K, poses)      the fitness E of eq. (§III-B) of arbitrary poses
 *
 * Every call returns a pft_status; nothing throws or aborts.  All device work is enqueued on
 * the caller's CUDA stream (`stream` = cudaStream_t, NULL = legacy default stream) and is
 * asynchronous unless the call says "syncs".  The library never allocates device memory (NCCL
 * internals excepted): the caller owns every buffer and sizes it with the *_bytes queries.
 *
 * Conventions (DESIGN.md §3 lists every reading of the paper):
 *   - pose = double[12], row-major 3x4 [R|t], camera -> world: p_w = R p_c + t.
 *   - camera frame x right, y down, z forward; depth is z-depth, uint16 raw * depth_unit_m.
 *   - voxel (i,j,k) samples the world point origin + voxel*(i+1/2, j+1/2, k+1/2).
 *   - stored TSDF values V are normalised by tau (metric / tau, in [-1,1]); unobserved voxels
 *     hold V = 1, W = 0 (reading L2/L3).
 *   - canonical volume arrays (upload / download) are nx*ny*nz elements, x fastest, then y,
 *     then z, in the storage precision (fp32, or fp16 as raw 16-bit patterns).
 */
#ifndef PFT_H
#define PFT_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PFT_ABI_VERSION 4

typedef enum {
  PFT_OK = 0,
  PFT_ERR_INVALID_ARG = -1,     /* null required pointer or out-of-range parameter            */
  PFT_ERR_BUFFER_TOO_SMALL = -2,/* caller buffer smaller than the matching *_bytes query         */
  PFT_ERR_EMPTY_CLOUD = -3,     /* reserved: an empty strided cloud is reported asynchronously,
                                   see pft_track (trace flag bit 2 and pft_track_info)            */
  PFT_ERR_CUDA = -4,            /* a CUDA launch/runtime error (sticky per volume handle)          */
  PFT_ERR_NCCL = -5,            /* NCCL missing or an NCCL call failed                             */
  PFT_ERR_UNSUPPORTED = -6,     /* valid but unsupported (e.g. > 2^31 voxels)                      */
  PFT_ERR_STATE = -7            /* call out of order (e.g. comm not initialised)                   */
} pft_status;

typedef enum { PFT_STORE_F32 = 0, PFT_STORE_F16 = 1 } pft_storage; /* value AND weight precision */

/* Reading L10: how the delta pose dP = (dR, u) multiplies the current pose P = (R, t)
 * (PAPER.md:196 "dP_k P", :207).  CAMERA_CENTRED (default): (dR R, t + u).
 * WORLD_LITERAL: (dR R, dR t + u), the literal left product of [dR|u] and [R|t]. */
typedef enum { PFT_DELTA_CAMERA_CENTRED = 0, PFT_DELTA_WORLD_LITERAL = 1 } pft_delta_conv;

/* Reading L14: the advantage-set average.  MEAN is the paper's plain mean;
 * WEIGHTED (NEXT F3) weights member k by E_base - E_k > 0; TOPK (NEXT F3, north_star "top-k")
 * averages the `topk` (1..32) best members by (E_k, k), plain mean in ascending k; K <= 65536.
 * With TOPK, trace[1] reports the number of members averaged. */
typedef enum { PFT_UPDATE_MEAN = 0, PFT_UPDATE_WEIGHTED = 1, PFT_UPDATE_TOPK = 2 } pft_update_rule;

#define PFT_MAX_SCHED 4

typedef struct {
  int32_t nx, ny, nz;   /* voxels per axis, each in [2, 4096]                                */
  double voxel_m;       /* voxel edge (m), > 0                                               */
  double origin_m[3];   /* min corner of the grid (m)                                        */
  double trunc_m;       /* tau (m), >= 2 * voxel_m                              */
  double max_weight;    /* W cap (SPEC.md:218 default 128), >= 1                              */
  double max_depth_m;   /* depths >= this are invalid (default 8 m)                          */
  pft_storage storage;
} pft_volume_desc;

typedef struct {
  double fx, fy, cx, cy;  /* pinhole intrinsics (pixels), fx, fy > 0                          */
  int32_t width, height;  /* depth image size, 1..16384 each                                 */
  double depth_unit_m;    /* metres per raw unit: 0.001 for uint16 millimetres                */
} pft_intrinsics;

typedef struct {
  double omega0_deg;      /* s^(1) rotation range, degrees, in [0,100]  (10)    */
  double v0_cm;           /* s^(1) translation range, cm, >= 0          (10)    */
  double beta;            /* search-size momentum in [0,1)              (0.1)   */
  int32_t iters;          /* iterations, >= 1 (fixed count, no early stop)      */
  int32_t stride;         /* point down-sampling stride sigma >= 1: pixels (sigma*c, sigma*r)  */
  double min_inband_frac; /* rho in [0,1]: E = 1 unless n >= rho * N (reading L6; default 0)  */
  pft_delta_conv delta_conv;
  pft_update_rule update_rule;
  int32_t topk;           /* PFT_UPDATE_TOPK: members averaged, 1..32                         */
  /* NEXT F1, the paper's schedule: nsched in [1, PFT_MAX_SCHED] cycles
   * (sched_K, sched_sx, sched_sy): iteration i uses the first min(sched_K, K) template rows and the
   * points of column/row strides (sched_sx, sched_sy); its baseline E(P^(i-1)) is recomputed when
   * the point set changes (reading L11).  nsched = 0: every iteration uses all rows and `stride`. */
  int32_t nsched;
  int32_t sched_K[PFT_MAX_SCHED], sched_sx[PFT_MAX_SCHED], sched_sy[PFT_MAX_SCHED];
  /* F1 convergence stop: stop after an iteration whose new s has omega < min_search_deg
   * AND v < min_search_cm (both 0: off).  Later trace rows are flagged "not run" (bit 5). */
  double min_search_deg, min_search_cm;
  /* NEXT F3: guard != 0 keeps P^(i-1) when E(P^(i)) > E_base (a stall,
   * trace bit 3); stall_limit > 0 stops after that many consecutive iterations without a pose change. */
  int32_t guard, stall_limit;
} pft_track_params;

/* Per-iteration trace record, PFT_TRACE_DOUBLES doubles:
 *  [0] E_base = E(P^(i-1))  [1] |A|  [2] omega_i (deg)  [3] v_i (cm)  [4..15] P^(i) (12)
 *  [16] E(P^(i))  [17] omega_{i+1}  [18] v_{i+1}
 *  [19] flags: bit0 advantage set empty, bit1 lost (E_base == 1), bit2 empty cloud (N == 0),
 *       bit3 guard rejected the update, bit4 stopped after this iteration, bit5 not run
 *  [20] n_c = in-band count of P^(i)  [21] N = valid points of the iteration's set
 *  [22] K_i particles evaluated  [23] stride code sx + 1000 sy.
 * Rows of iterations that did not run (after a stop) are zero except flags = 32. */
#define PFT_TRACE_DOUBLES 24

typedef struct pft_volume pft_volume; /* opaque handle */

/* ---------------------------------------------------------------- volume */

/* Bytes of device storage a volume of this description needs (values, weights and the
 * scratch the library uses for checksums and integration culling).  INVALID_ARG on a bad
 * desc; UNSUPPORTED if the padded grid exceeds 2^31 voxels. */
pft_status pft_volume_bytes(const pft_volume_desc* desc, size_t* bytes_out);

/* Creates a handle that BORROWS dev_storage (device pointer, 256-byte aligned, >= the
 * pft_volume_bytes size) for its lifetime; contents are undefined until reset/upload.
 * *out is a host object freed by pft_volume_destroy (which does not free dev_storage). */
pft_status pft_volume_create(const pft_volume_desc* desc, void* dev_storage, size_t bytes,
                             pft_volume** out);

/* V = 1, W = 0 everywhere ("unobserved", reading L3). */
pft_status pft_volume_reset(pft_volume* vol, void* stream);

/* Canonical (x-fastest) device arrays -> the library's internal brick order.  Each array is
 * nx*ny*nz elements of the storage precision.  Neither pointer may be NULL. */
pft_status pft_volume_upload(pft_volume* vol, const void* dev_values, const void* dev_weights,
                             void* stream);

/* Internal brick order -> canonical device arrays (either pointer may be NULL to skip). */
pft_status pft_volume_download(const pft_volume* vol, void* dev_values, void* dev_weights,
                               void* stream);

/* Order-independent 64-bit hash of every voxel's (index, V bits, W bits); layout-independent,
 * so two replicas with identical contents hash identically.  Syncs `stream`. */
pft_status pft_volume_checksum(const pft_volume* vol, uint64_t* host_out, void* stream);

/* Frees the handle (and its NCCL communicator, if any).  Does not free dev_storage. */
pft_status pft_volume_destroy(pft_volume* vol);

/* ---------------------------------------------------------------- fusion */

/* KinectFusion TSDF integration of one depth frame (dev_depth: height x width uint16,
 * row-major) at camera->world pose dev_T (device, 12 doubles).  Per voxel (reading L22):
 *   p_c = R^T (g_w - t); skip unless z_c > 0; (u,v) = (fx x/z + cx, fy y/z + cy);
 *   pixel (floor(u+1/2), floor(v+1/2)) must be inside and valid; sdf = d - z_c;
 *   if sdf > -tau: V' = (V W + min(1, sdf/tau)) / (W + 1), W' = min(W + 1, W_max),
 *   each rounded once (RNE) to the storage precision.
 * Decisions and the update are evaluated in fp64 in the stated operation order, so stored
 * bits equal those of a plain fp64 evaluation of the same formulas.  Must not overlap a
 * track / eval_poses on the same volume (one writer). */
pft_status pft_integrate(pft_volume* vol, const uint16_t* dev_depth, const pft_intrinsics* K,
                         const double* dev_T, void* stream);

/* pft_integrate with flags: bit0 = full sweep over every voxel (no brick culling; the
 * verification path — results are identical by construction). */
#define PFT_INTEGRATE_FULL_SWEEP 1
pft_status pft_integrate_ex(pft_volume* vol, const uint16_t* dev_depth, const pft_intrinsics* K,
                            const double* dev_T, int32_t flags, void* stream);

/* Work counters of the last culled pft_integrate call on this volume (measurement):
 * out[0] bricks kept by the cull (4^3 voxels each), out[1] of those classified free space (every
 * voxel provably updated with v_new = 1, no projection), out[2] voxels updated (W or V written),
 * out[3] cell-bricks whose tracker records were rebuilt.  Syncs `stream`.  After a full-sweep
 * call the counters are not maintained (out[] = -1). */
pft_status pft_integrate_stats(const pft_volume* vol, int64_t out[4], void* stream);

/* NEXT F4: zero-crossing surface points, input of the completeness / accuracy
 * metrics of PAPER.md:562-563.  For every voxel and axis whose +1 neighbour is in the grid, both
 * observed (W > 0), values of different sign (not both 0): t = V0/(V0 - V1), point = voxel centre
 * + t * voxel along the axis (fp64, bit-identical to a plain evaluation).  dev_points: max_points x 3
 * doubles (world, metres), unordered; *dev_count (device int64) = total crossings (may exceed
 * max_points: only the first max_points are written; call with max_points = 0 to size). */
pft_status pft_extract_surface(const pft_volume* vol, double* dev_points, int64_t max_points,
                               int64_t* dev_count, void* stream);

/* ---------------------------------------------------------------- tracking */

/* Workspace bytes pft_track / pft_eval_poses need for this frame geometry and K particles
 * (K = number of poses for pft_eval_poses). */
pft_status pft_track_workspace_bytes(const pft_volume* vol, const pft_intrinsics* K, int32_t nparticles,
                                     const pft_track_params* prm, size_t* bytes_out);
/* (E_k / n_k outputs are those of the last iteration that ran; rows k >= that iteration's K_i
 *  report E = 1, n = 0.) */

/* Randomized optimisation of PAPER.md:192-208:
 *   points: strided back-projection of the depth (stride prm->stride);
 *   P = T_init, s = (omega0, v0), E_c = E(P);
 *   for i = 1..iters:
 *     dP_k = (Rodrigues(r_k), u_k), r_k = pst[k][0:3] * omega*pi/180, u_k = pst[k][3:6] * v/100;
 *     E_k = E(dP_k P) for every k;  A = {k : E_k < E_c};
 *     if A nonempty: q = normalised sum of the unit quaternions of A, u = mean of u_k over A,
 *                    P = (R(q), u) P (delta_conv), E_c = E(P);
 *     s = (beta + (1 - beta) E_c) s.
 * E(T) = mean over in-band points of |V(T p)| (trilinear, all 8 corners |V| < 1), or 1 when
 * no point is in band (or fewer than rho * N).
 * Arguments (device pointers): dev_depth (height x width uint16), dev_T_init (12 doubles),
 * dev_pst (nparticles x 6 fp32 in [-1,1]: rotation vector then translation, reused every
 * iteration), dev_ws (>= pft_track_workspace_bytes), outputs dev_T_out (12 doubles),
 * dev_E (nparticles doubles) and dev_inband (nparticles int32) of the LAST iteration, and
 * dev_trace (NULL, or iters x PFT_TRACE_DOUBLES).
 * Prefix-stable: the first i iterations of an iters = n run equal an iters = i run bit for bit.
 * An empty cloud (no valid strided pixel) is not an error: T_out = T_init, every E = 1,
 * every count 0, trace flag bit 2 set.
 * After pft_comm_init this is a collective: every rank passes identical arguments; rank r
 * evaluates particles [r*ceil(K/G), ...) and per-particle results are all-gathered. */
pft_status pft_track(pft_volume* vol, const uint16_t* dev_depth, const pft_intrinsics* K,
                     const double* dev_T_init, const float* dev_pst, int32_t nparticles,
                     const pft_track_params* prm, void* dev_ws, size_t ws_bytes,
                     double* dev_T_out, double* dev_E, int32_t* dev_inband, double* dev_trace,
                     void* stream);

/* Fitness E (and in-band count n) of M arbitrary poses (dev_poses: M x 12 doubles) on the
 * frame's strided points (uses prm->stride and prm->min_inband_frac only).  Local to this
 * rank (never a collective). */
pft_status pft_eval_poses(const pft_volume* vol, const uint16_t* dev_depth, const pft_intrinsics* K,
                          const pft_track_params* prm, const double* dev_poses, int32_t M,
                          void* dev_ws, size_t ws_bytes, double* dev_E, int32_t* dev_inband,
                          void* stream);

/* Number of valid strided points N of the last pft_track / pft_eval_poses that used dev_ws.
 * Syncs `stream`. */
pft_status pft_track_info(const void* dev_ws, int32_t* npoints_out, void* stream);

/* Device-side pose chaining (the sequence driver O11 / reading L25: T_init = P_{t-1} * rel_t):
 * dev_out = dev_A * dev_B for rigid 3x4 row-major [R|t] poses, i.e. (R_A R_B, R_A t_B + t_A), in
 * fp64 (dev_out may alias an input).  Enqueued on `stream`. */
pft_status pft_pose_compose(const double* dev_A, const double* dev_B, double* dev_out, void* stream);

/* ---------------------------------------------------------------- multi-GPU (north_star) */

/* NCCL unique id for pft_comm_init (call on one rank, broadcast the 128 bytes). */
pft_status pft_comm_get_unique_id(uint8_t id_out[128]);

/* Attaches an NCCL communicator (one rank per GPU) to the volume handle; afterwards
 * pft_track shards particles across the nranks GPUs.  The volume is replicated: every rank
 * calls pft_integrate with the same inputs.  The current CUDA device must be this rank's.
 * nranks = 1 attaches a real single-rank communicator, and pft_track then runs the collective
 * (multi-launch) path -- the NCCL plumbing exercised on one GPU, results unchanged.
 * PFT_ERR_STATE if virtual ranks or peer exchange buffers are set on the handle.  Collective
 * failures, including asynchronous ones (ncclCommGetAsyncError, polled after each collective),
 * return PFT_ERR_NCCL. */
pft_status pft_comm_init(pft_volume* vol, const uint8_t id[128], int32_t nranks, int32_t rank);

/* F2 fused exchange (Sec. III-C "Randomized optimization": every
 * particle's E_k is needed by every rank for the advantage-set update).  With peer buffers
 * attached, pft_track runs the whole RO loop as one persistent launch per GPU: each rank
 * evaluates its shard (rows [r*ceil(K/G), ...)), then its CTAs store their finished per-particle
 * records (16 B each) straight into every rank's exchange buffer over NVLink (P2P stores), the
 * rank signals each peer with one system-scope atomic, and waits for all G shards before the
 * update -- no NCCL launch and no host round trip per iteration.  Counters are monotone across
 * calls (each rank stores the number of completed rounds in its own buffer), so calls need no
 * reset handshake; all ranks must call pft_track with the same arguments the same number of
 * times.  A rank that waits longer than the watchdog for a peer traps (a launch error instead of
 * a hang; environment PFT_WATCHDOG_MS, default 5000, read once per process).
 *
 * pft_comm_p2p_init: allocates (cudaMalloc, zero-filled) this rank's exchange buffer sized for
 *   up to max_particles particles and nranks <= PFT_MAX_FUSED_RANKS ranks, and writes its
 *   CUDA IPC handle (PFT_IPC_HANDLE_BYTES) to handle_out.  The library owns the buffer (freed
 *   by pft_volume_destroy).  Call on the rank's own device.
 * pft_comm_p2p_attach: `handles` = the nranks handles in rank order (gathered by the caller,
 *   e.g. torch.distributed.all_gather); opens the peers' buffers with peer access enabled.  The
 *   caller must barrier all ranks after attach and before the first pft_track.
 * Errors: PFT_ERR_STATE if another communicator is attached; PFT_ERR_CUDA if IPC fails (the
 * GPUs must be peers on one node). */
#define PFT_MAX_FUSED_RANKS 8
#define PFT_IPC_HANDLE_BYTES 64
pft_status pft_comm_p2p_init(pft_volume* vol, int32_t nranks, int32_t rank, int32_t max_particles,
                             uint8_t handle_out[PFT_IPC_HANDLE_BYTES]);
pft_status pft_comm_p2p_attach(pft_volume* vol, const uint8_t* handles);
/* Undoes pft_comm_p2p_init/attach on this rank (closes the peers' mappings, frees the buffer);
 * the volume is then single-rank again (or keeps an attached NCCL communicator).  For a job
 * whose ranks could not all attach: every rank detaches and falls back to pft_comm_init. */
pft_status pft_comm_p2p_detach(pft_volume* vol);
/* Pre-flight of the attached peer exchange, before the first pft_track: one small kernel writes a
 * token into every rank's buffer over NVLink (system-scope release stores) and waits, at most
 * timeout_ms, for every peer's token in its own buffer (acquire loads).  *ok_out = 1 when all G
 * arrived intact, 0 otherwise (no trap: the caller agrees with the other ranks and falls back to
 * pft_comm_init).  All ranks must call it; syncs `stream`.  PFT_ERR_STATE if not attached. */
pft_status pft_comm_p2p_preflight(pft_volume* vol, int32_t timeout_ms, int32_t* ok_out, void* stream);

/* F2b (SURVEY.md §8(e) "alternative partition"): how pft_track splits the work across the ranks
 * of an NCCL communicator (or virtual shards).  PARTICLES (default): rank r evaluates template rows
 * [r*ceil(K/G), ...) on all points; the per-particle records are all-gathered.  POINTS: every rank
 * evaluates all K_i particles on its contiguous slice of the strided point slots (whole 8x4 tiles),
 * and the per-particle fixed-point sums -- and the centre's -- are summed by an integer all-reduce
 * (exact, so results equal the 1-rank run bit for bit).  PFT_ERR_UNSUPPORTED with the peer exchange. */
#define PFT_PARTITION_PARTICLES 0
#define PFT_PARTITION_POINTS 1
pft_status pft_comm_set_partition(pft_volume* vol, int32_t partition);

/* ---------------------------------------------------------------- instrumentation */

/* Kernel classes of the per-launch profile. */
#define PFT_PROF_EVAL 0        /* k_particle_eval: the particle x point hot loop (a3/a4)      */
#define PFT_PROF_CENTRE 1      /* k_centre: E(P) + s-law (a5/a8)                              */
#define PFT_PROF_UPDATE 2      /* k_update: advantage set + pose update (a7)                  */
#define PFT_PROF_PREP 3        /* k_track_init + k_backproject (a1/a2)                        */
#define PFT_PROF_INTEGRATE 4   /* fusion sweep (a10)                                          */
#define PFT_PROF_CULL 5        /* depth tiles + brick cull (a10)                              */
#define PFT_PROF_COMM 6        /* ncclAllGather (a6)                                          */
#define PFT_PROF_OTHER 7       /* volume reset / upload / download / checksum                 */
#define PFT_PROF_RECORDS 8     /* tracker cell-record / in-band-mask maintenance (a10)        */
#define PFT_PROF_TRACK 9       /* k_track_persistent: the whole RO loop in one launch         */
#define PFT_PROF_CLASSES 10

/* Cumulative number of CUDA kernels (and NCCL collectives) this library has launched. */
uint64_t pft_launch_count(void);

/* While profiling is on, every launch is bracketed by CUDA events recorded on its own stream.
 * pft_profile_stop syncs those events, returns per-class total milliseconds and launch counts
 * (arrays of PFT_PROF_CLASSES; either may be NULL) and turns profiling off.  Process-global;
 * at most 65536 launches are recorded per start/stop. */
pft_status pft_profile_start(void);
pft_status pft_profile_stop(double* ms_out, int64_t* launches_out);

/* Test/debug: emulate nranks particle shards on this one GPU (SURVEY.md §4 "virtual shards"):
 * pft_track then runs the multi-GPU code path with rank r's evaluation launched in turn and the
 * all-gather replaced by device copies; results must equal the 1-rank run bit for bit.  Not for
 * production (the shards run sequentially). */
pft_status pft_comm_init_virtual(pft_volume* vol, int32_t nranks);

/* Test/debug: emulate the F2 fused exchange on this one GPU: pft_track runs ONE persistent
 * launch holding nranks (<= PFT_MAX_FUSED_RANKS) groups of CTAs, each group a rank with its own
 * workspace region (pft_track_workspace_bytes grows nranks-fold) and exchange buffer, pushing
 * its shard into every group's buffer and waiting on the same counters the multi-GPU path uses.
 * Results (T, E, n, trace) must equal the 1-rank run bit for bit; group 0 writes the outputs. */
pft_status pft_comm_init_virtual_fused(pft_volume* vol, int32_t nranks);

/* Thread-local message describing the last non-OK status of this thread. */
const char* pft_last_error(void);

/* Library ABI version (PFT_ABI_VERSION). */
int32_t pft_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* PFT_H */
