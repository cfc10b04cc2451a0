// pft_internal.cuh — internal declarations shared by the libpft translation units.
// Nothing here is part of the ABI (include/pft.h is).
#pragma once
#include <cuda_runtime.h>
#include <cuda_fp16.h>
#include <stdint.h>
#include <stddef.h>

#include "../../include/pft.h"

namespace pft {

// ------------------------------------------------------------------ volume layout
// TSDF storage is SoA (values, weights) in 4x4x4-voxel bricks: a brick is 64
// consecutive elements, z-major inside (z*16 + y*4 + x), bricks x-fastest.  The element
// offset of voxel (x,y,z) is separable: offx(x) + offy(y) + offz(z), so the 8 trilinear
// corners cost 6 offset terms and 8 adds.
constexpr int kBrick = 4;
constexpr int kBrickVox = 64;

struct Geom {
  int nx, ny, nz;          // voxels
  int nbx, nby, nbz;       // bricks
  uint32_t sy, sz;         // brick-row / brick-slab strides in elements (64*nbx, 64*nbx*nby)
  double voxel, ox, oy, oz;
  double trunc, max_weight, max_depth;
};

__host__ __device__ __forceinline__ uint32_t offx(int x) { return ((uint32_t)(x >> 2) << 6) | (uint32_t)(x & 3); }
__host__ __device__ __forceinline__ uint32_t offy(int y, uint32_t sy) { return (uint32_t)(y >> 2) * sy + ((uint32_t)(y & 3) << 2); }
__host__ __device__ __forceinline__ uint32_t offz(int z, uint32_t sz) { return (uint32_t)(z >> 2) * sz + ((uint32_t)(z & 3) << 4); }

// Cell records: the tracker reads, for trilinear cell (cx,cy,cz), ONE 32-byte
// (fp32) / 16-byte (fp16) record at record index offx(cx)+offy(cy)+offz(cz) (same brick order as
// the voxels), rebuilt by the fusion step for every touched brick.  fp32 volumes store the
// trilinear polynomial coefficients [a b c d e f g h] of the cell (fp64-computed, rounded once);
// fp16 volumes store the 8 corner values [v000 v100 v010 v110 v001 v101 v011 v111].
// Beside them, a 1-bit-per-cell in-band mask (bit w of the brick's uint64, w = cell index inside
// the brick) says whether all 8 corners have |V| < 1 (reading L3); the tracker loads a record
// only for in-band cells, so its working set is the band, not the search volume.
// Byte layout of the caller-owned volume storage.
struct VolLayout {
  size_t scratch_off, scratch_bytes;  // checksum / counters
  size_t v_off, w_off, elems;         // elems = nbx*nby*nbz*64 per array
  size_t r_off;                       // cell records: elems x 8 values
  size_t m_off;                       // in-band mask: one uint64 per brick, bit w = cell w
  size_t list_off, list_bytes;        // integration: active brick list (uint32 per brick)
  size_t dirty_off, dlist_off;        // records: dirty flag per cell-brick + dirty list (uint32 each)
  size_t slist_off;                   // integration: surviving super-bricks (8^3 bricks) list
  size_t tiles_off, tiles_bytes;      // integration: per-tile depth max (float)
  size_t axis_off;                    // integration: per-frame axis tables, 4*(nbx+nby+nbz) double4
  size_t total;
};

}  // namespace pft

namespace pft {
constexpr int kMaxFusedRanks = PFT_MAX_FUSED_RANKS;  // F2 fused exchange: ranks per job

// ------------------------------------------------------------------ programmatic dependent launch
// The integration chain (frame prep -> culls -> fusion -> record refresh) launches each kernel with
// programmatic stream serialization: its CTAs are scheduled while the previous kernel drains and
// wait in pdl_wait() (griddepcontrol.wait: the previous grid has completed and its memory is
// visible) before touching anything it wrote; pdl_trigger() lets the next kernel be launched
// early.  Without the launch attribute both are no-ops.  Every grid of the chain fits in one wave,
// so early-launched CTAs never hold SM slots a predecessor still needs.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
bool pdl_enabled();  // PFT_PDL=0 disables (abi.cu)
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, args...);
  if (e != cudaSuccess && cfg.numAttrs) {  // (not expected on sm_100a) the plain stream-ordered launch
    cudaGetLastError();
    cfg.numAttrs = 0;
    e = cudaLaunchKernelEx(&cfg, kern, args...);
  }
  return e;
}
}

struct pft_volume {
  pft_volume_desc desc;
  pft::Geom g;
  pft::VolLayout L;
  size_t esize;     // 4 (fp32) or 2 (fp16)
  char* base;
  int device;
  // multi-GPU
  void* nccl_comm;
  int nranks, rank;
  int virtual_ranks;  // > 1: pft_comm_init_virtual (sequential shards, no NCCL)
  int virtual_fused;  // pft_comm_init_virtual_fused: G rank groups in one persistent launch
  // F2 peer exchange (pft_comm_p2p_init / _attach): xbuf[q] = rank q's exchange buffer mapped
  // into this process (xbuf[rank] = xown); records at 0, counters at xcnt_off
  int p2p;
  char* xbuf[PFT_MAX_FUSED_RANKS];
  char* xown;
  size_t xbytes, xcnt_off;
  int32_t xmax_particles;
  int partition;      // PFT_PARTITION_PARTICLES (default) | PFT_PARTITION_POINTS (F2b)
  unsigned long long preflight_round;  // pft_comm_p2p_preflight calls so far
  // one-GPU emulation: the exchange counters are zeroed when the workspace changes
  const char* xws_last;
  size_t xws_total, xws_region, xws_xcnt;  // workspace + layout the counters were zeroed for
};

namespace pft {

// ------------------------------------------------------------------ tracking state / records
// Per-particle accumulator, exchanged as-is by the all-gather (16 B).
// S = sum over in-band points of |v| in fixed point (units of 2^-kFixBits), n = in-band count.
struct PartRec {
  unsigned long long S;
  unsigned int n;
  unsigned int pad;
};
constexpr int kFixBits = 29;  // per-thread partial sums of <= 7 terms in [0,1) fit in uint32

// Device-resident state of one pft_track call (lives at the start of the workspace).
struct TrackState {
  double P[12];        // current pose P^(i)
  double Pprev[12];    // P^(i-1) (F3 guard, multi-launch path)
  double omega, v;     // current search size s^(i) (deg, cm)
  double Ec;           // E(P) of the current pose on the current point set
  double Ebase;        // E of the pose the current iteration started from
  double Wsum;         // sum of member weights of the last update
  unsigned long long Sc_acc;  // centre accumulators (zeroed after use)
  unsigned int nc_acc;
  unsigned int nc;     // in-band count of the current pose
  unsigned int nc_base;  // in-band count of the iteration's starting pose
  int nA;              // |A| of the last update
  int iter;            // iterations completed
  int Nvalid[4];       // valid points per point set (Nvalid[0]: the first iteration's set)
  int cur_set;         // point set E_c refers to (-1: none yet)
  int stalls;          // consecutive iterations without a pose change
  int stopped;         // a stop rule fired: later iterations are no-ops
  int K_last;          // K_i of the last iteration that ran
  unsigned int ticket_upd, ticket_ctr;
  unsigned long long pmax_bits;  // max |point coordinate| over all sets (persistent path)
  unsigned long long bar_mono;      // persistent path: grid-barrier arrivals (monotone within a launch)
  unsigned int sm_cnt[256];   // persistent path, SM pairing: CTAs arrived per SM id
  unsigned int sm_pair[256];  //   pair index + 1 of the SM (published by its first CTA)
  unsigned int npairs, pad2;
  double pad[4];
};

// One strided point set (2-D strides sx on columns, sy on rows; reading L20), 8x4-pixel tiles.
struct PointSetL { int sx, sy, nr, nc, ntx, nty, npad; size_t off; };

struct TrackLayout {
  size_t state_off;
  int nsets;
  PointSetL sets[4];   // distinct (sx, sy) of the schedule; set of schedule entry j: sched_set[j]
  int nsched;          // >= 1 (0 in the params maps to one entry (K, stride, stride))
  int sched_K[4], sched_set[4];
  int npad_max;
  size_t acc_local_off, acc_full_off;
  size_t part_off;     // update partials: nblk_upd * kUpdW doubles
  size_t ptab_off;     // persistent path: K x 12 folded candidate poses + K flags
  size_t mtab_off;     // persistent path: K x 8 member deltas (q, u, pad) for the update
  size_t cpart_off;    // persistent path: per-CTA centre partials (S, n)
  size_t work_off;     // persistent path: per-iteration work counters
  size_t topk_off;     // F3 top-k: per-block candidate lists and the merged result
  size_t cacc_off;     // F2b point shards: the centre's partial (S, n) as 2 uint64 (all-reduced)
  int points_part;     // F2b: particles unsharded (kloc = K), points sharded across the ranks
  size_t total;         // bytes of the whole workspace (G regions in the fused emulation)
  size_t region;        // bytes of one rank's region
  size_t xch_off;       // fused emulation: the rank's exchange buffer inside its region
  size_t xcnt_rel;      //   its counters: kMaxFusedRanks words + the completed-round word
  int kloc, kfull, nblk_upd;
};

constexpr int kUpdW = 10;  // update partial width: q(4), u(3), |A|, sum of weights, pad

}  // namespace pft

namespace pft {
// Error reporting (abi.cu): records a thread-local message and returns s.
pft_status fail(pft_status s, const char* fmt, ...);
// cudaGetLastError() after a launch sequence -> PFT_OK or PFT_ERR_CUDA with the message.
pft_status cuda_check(const char* what);
// F2 peer exchange pre-flight (track.cu): one exchange of tokens with every attached peer.
pft_status p2p_preflight(pft_volume* vol, int timeout_ms, int32_t* ok_out, cudaStream_t st);
// Launch instrumentation (abi.cu): call prof_begin before and prof_end after each launch.
void prof_begin(int cls, cudaStream_t st);
void prof_end(int cls, cudaStream_t st, const char* what);
// Cell-record maintenance (volume.cu): rebuild every record, or those of the listed bricks
// (cells [4b-1, 4b+3] per axis, i.e. every cell with a corner in the brick).
void records_rebuild_all(pft_volume* vol, cudaStream_t st);
void records_rebuild_dirty(pft_volume* vol, cudaStream_t st);
// Marks (dedup'ed) the cell-bricks whose records depend on a changed voxel of brick (bx,by,bz):
// nbmask bit (dz*4 + dy*2 + dx) = cell-brick (bx-dx, by-dy, bz-dz) is affected.  Called by a whole
// warp (nbmask warp-uniform): lane q < 8 claims neighbour q (atomicExch on its dirty flag), then the
// newly claimed ones are appended with one warp-aggregated atomicAdd -- two atomic round trips in
// total instead of up to 8 serial pairs.
__device__ __forceinline__ void mark_dirty_cells_warp(const Geom& g, int bx, int by, int bz, unsigned nbmask,
                                                      uint32_t* dirty, uint32_t* dlist, uint32_t* dcount) {
  const int q = threadIdx.x & 31;
  bool mine = false;
  uint32_t cb = 0;
  if (q < 8 && ((nbmask >> q) & 1u)) {
    const int cx = bx - (q & 1), cy = by - ((q >> 1) & 1), cz = bz - (q >> 2);
    if (cx >= 0 && cy >= 0 && cz >= 0) {
      cb = ((uint32_t)cz * g.nby + (uint32_t)cy) * g.nbx + (uint32_t)cx;
      mine = atomicExch(dirty + cb, 1u) == 0u;
    }
  }
  const unsigned ball = __ballot_sync(0xffffffffu, mine);
  if (ball) {
    uint32_t base = 0;
    if (q == 0) base = atomicAdd(dcount, (uint32_t)__popc(ball));
    base = __shfl_sync(0xffffffffu, base, 0);
    if (mine) dlist[base + __popc(ball & ((1u << q) - 1u))] = cb;
  }
}
#define PFT_LAUNCH(cls, st, ...)        \
  do {                                  \
    ::pft::prof_begin((cls), (st));     \
    __VA_ARGS__;                        \
    ::pft::prof_end((cls), (st), #__VA_ARGS__); \
  } while (0)
// Validation helpers shared by the entry points.
pft_status check_intrinsics(const pft_intrinsics* K);
pft_status track_layout(const pft_volume* vol, const pft_intrinsics* K, int32_t nparticles,
                        const pft_track_params* prm, int nranks, TrackLayout* L);
}  // namespace pft
