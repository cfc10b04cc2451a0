// integrate.cu — KinectFusion TSDF fusion of one depth frame ("The fusion process
// remains the same as KinectFusion"; reading L22/L23 in DESIGN.md §3).
//
// Per voxel, in this exact fp64 operation order (no FMA contraction, IEEE division), so the
// stored bits equal a plain fp64 evaluation of the same formulas:
//   g_w = o + s*(i + 1/2);  p_c = R^T (g_w - t);  skip unless z_c > 0;
//   u = fx*x/z + cx, v = fy*y/z + cy;  pixel = (floor(u + 1/2), floor(v + 1/2)) inside and valid;
//   sdf = d - z_c;  skip unless sdf > -tau;  v_new = min(1, sdf/tau);
//   V' = (V W + v_new)/(W + 1), W' = min(W + 1, W_max), each rounded once (RNE) to storage.
//
// B200 design: the update set of a frame is the camera frustum up to the
// surface + tau, a few % of a room-scale grid.  A per-brick cull (conservative, fp32 with
// margins) compacts the 4^3 bricks that can contain an updated voxel; the fusion kernel then
// sweeps only those bricks, 64 consecutive elements (one brick = 2 x 128 B lines per array
// at fp32) per pair of warps, fully coalesced.  The full sweep is kept for verification.
#include "pft_internal.cuh"

namespace pft {

struct Intr {
  double fx, fy, cx, cy, unit;
  int W, H;
};

template <typename T> __device__ __forceinline__ double to_double(T x);
template <> __device__ __forceinline__ double to_double<float>(float x) { return (double)x; }
template <> __device__ __forceinline__ double to_double<__half>(__half x) { return (double)__half2float(x); }
template <typename T> __device__ __forceinline__ T store_rn(double x);
template <> __device__ __forceinline__ float store_rn<float>(double x) { return __double2float_rn(x); }
template <> __device__ __forceinline__ __half store_rn<__half>(double x) { return __double2half(x); }

template <typename T> __device__ __forceinline__ bool same_bits(T a, T b);
template <> __device__ __forceinline__ bool same_bits<float>(float a, float b) { return __float_as_uint(a) == __float_as_uint(b); }
template <> __device__ __forceinline__ bool same_bits<__half>(__half a, __half b) { return __half_as_ushort(a) == __half_as_ushort(b); }

// Exact int -> double without the conversion pipe (XU): 2^52 + i has i in its low mantissa bits.
__device__ __forceinline__ double i2d(int i) {  // 0 <= i < 2^31
  return __dsub_rn(__hiloint2double(0x43300000, i), 4503599627370496.0);
}
// floor(x) as an int for |x| < 2^30 (exact; no FRND): x + 1.5*2^52 rounded toward -inf holds
// floor(x) in its low word.
__device__ __forceinline__ int floor_lo(double x) { return __double2loint(__dadd_rd(x, 6755399441055744.0)); }

// Returns true iff the stored value V changed (its cell records must then be refreshed).
template <typename T>
__device__ __forceinline__ bool fuse_voxel(const Geom& g, const Intr& K, const uint16_t* __restrict__ depth,
                                           const double* T_, int i, int j, int k, T* __restrict__ V,
                                           T* __restrict__ W, uint32_t o) {
  const double gw0 = __dadd_rn(g.ox, __dmul_rn(g.voxel, __dadd_rn(i2d(i), 0.5)));
  const double gw1 = __dadd_rn(g.oy, __dmul_rn(g.voxel, __dadd_rn(i2d(j), 0.5)));
  const double gw2 = __dadd_rn(g.oz, __dmul_rn(g.voxel, __dadd_rn(i2d(k), 0.5)));
  const double d0 = __dsub_rn(gw0, T_[3]), d1 = __dsub_rn(gw1, T_[7]), d2 = __dsub_rn(gw2, T_[11]);
  const double z = __dadd_rn(__dadd_rn(__dmul_rn(T_[2], d0), __dmul_rn(T_[6], d1)), __dmul_rn(T_[10], d2));
  if (!(z > 0.0)) return false;
  const double x = __dadd_rn(__dadd_rn(__dmul_rn(T_[0], d0), __dmul_rn(T_[4], d1)), __dmul_rn(T_[8], d2));
  const double y = __dadd_rn(__dadd_rn(__dmul_rn(T_[1], d0), __dmul_rn(T_[5], d1)), __dmul_rn(T_[9], d2));
  // pixel = floor(u + 1/2): out of [0, W) also for |u + 1/2| >= 2^30 and NaN
  const double u2 = __dadd_rn(__dadd_rn(__ddiv_rn(__dmul_rn(K.fx, x), z), K.cx), 0.5);
  if (!(fabs(u2) < 1073741824.0)) return false;
  const int ui = floor_lo(u2);
  if ((unsigned)ui >= (unsigned)K.W) return false;
  const double v2 = __dadd_rn(__dadd_rn(__ddiv_rn(__dmul_rn(K.fy, y), z), K.cy), 0.5);
  if (!(fabs(v2) < 1073741824.0)) return false;
  const int vi = floor_lo(v2);
  if ((unsigned)vi >= (unsigned)K.H) return false;
  const uint16_t raw = __ldg(depth + (size_t)vi * K.W + (size_t)ui);
  const double d = __dmul_rn(i2d((int)raw), K.unit);
  if (raw == 0 || !(d < g.max_depth)) return false;
  const double sdf = __dsub_rn(d, z);
  if (!(sdf > -g.trunc)) return false;
  double vnew = __ddiv_rn(sdf, g.trunc);
  if (vnew > 1.0) vnew = 1.0;
  const T Vs = V[o];
  const double Vo = to_double<T>(Vs), Wo = to_double<T>(W[o]);
  const double Wp = __dadd_rn(Wo, 1.0);
  const double Vn = __ddiv_rn(__dadd_rn(__dmul_rn(Vo, Wo), vnew), Wp);
  const double Wn = Wp > g.max_weight ? g.max_weight : Wp;
  const T Vnew = store_rn<T>(Vn);
  V[o] = Vnew;
  W[o] = store_rn<T>(Wn);
  return !same_bits<T>(Vs, Vnew);
}

// Full sweep: one thread per brick element (the verification path).
template <typename T>
__global__ __launch_bounds__(256) void k_integrate_sweep(Geom g, Intr K, const uint16_t* __restrict__ depth,
                                                         const double* __restrict__ Tdev, T* __restrict__ V,
                                                         T* __restrict__ W, size_t nelem) {
  __shared__ double sT[12];
  if (threadIdx.x < 12) sT[threadIdx.x] = Tdev[threadIdx.x];
  __syncthreads();
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < nelem; e += (size_t)gridDim.x * blockDim.x) {
    const uint32_t b = (uint32_t)(e >> 6), w = (uint32_t)(e & 63);
    const int bx = (int)(b % (uint32_t)g.nbx);
    const uint32_t r = b / (uint32_t)g.nbx;
    const int by = (int)(r % (uint32_t)g.nby), bz = (int)(r / (uint32_t)g.nby);
    const int i = bx * 4 + (int)(w & 3), j = by * 4 + (int)((w >> 2) & 3), k = bz * 4 + (int)(w >> 4);
    if (i >= g.nx || j >= g.ny || k >= g.nz) continue;
    fuse_voxel<T>(g, K, depth, sT, i, j, k, V, W, (uint32_t)e);
  }
}

// ---- culling ---------------------------------------------------------------------------------
constexpr int kTile = 8;  // depth tiles of 8x8 pixels

// Per tile: the maximum valid raw depth (0 if the tile has no valid pixel).  Validity is the
// exact fp64 test of O1 (raw > 0 and raw*unit < max_depth).
__global__ void k_depth_tiles(Intr K, double max_depth, const uint16_t* __restrict__ depth, uint32_t* __restrict__ tiles,
                              int ntx, int nty) {
  const int t = blockIdx.x * blockDim.y + threadIdx.y;  // one warp per tile
  if (t >= ntx * nty) return;
  const int tx = t % ntx, ty = t / ntx;
  uint32_t m = 0;
  for (int p = threadIdx.x; p < kTile * kTile; p += 32) {
    const int u = tx * kTile + (p & 7), v = ty * kTile + (p >> 3);
    if (u < K.W && v < K.H) {
      const uint16_t raw = depth[(size_t)v * K.W + u];
      if (raw != 0 && __dmul_rn((double)raw, K.unit) < max_depth) m = max(m, (uint32_t)raw);
    }
  }
  for (int s = 16; s > 0; s >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, s));
  if (threadIdx.x == 0) {
    tiles[t] = m;
    if (m) atomicMax(tiles + ntx * nty + (ty >> 3) * ((ntx + 7) >> 3) + (tx >> 3), m);  // coarse 64x64-px level
  }
}

// Conservative visibility test of a box of voxel centres given by its centre (world, fp64) and
// bounding-sphere radius: false only when no voxel centre inside can pass the voxel-level tests
// (all z_c <= 0, projection misses the image, or every pixel it can project to is invalid or has
// d + tau <= z_c).  fp32 with margins (1 mm, 2 px) far above fp32 rounding at room scale.  Boxes
// straddling the camera plane, or covering more than max_tiles depth tiles, are kept.
struct Footprint {
  int verdict;  // 0 reject, 1 keep, 2 decided by the max depth over tiles [t0x,t1x] x [t0y,t1y] of lvl
  const uint32_t* lvl;
  int stride, t0x, t1x, t0y, t1y;
  float zn;
};

__device__ __forceinline__ Footprint box_footprint(const Intr& K, const double* __restrict__ Tdev,
                                                   const uint32_t* __restrict__ tiles, int ntx, double cxw, double cyw,
                                                   double czw, float rad, int max_tiles) {
  Footprint f;
  f.verdict = 0;
  const float cwx = (float)(cxw - Tdev[3]), cwy = (float)(cyw - Tdev[7]), cwz = (float)(czw - Tdev[11]);
  const float x = (float)Tdev[0] * cwx + (float)Tdev[4] * cwy + (float)Tdev[8] * cwz;
  const float y = (float)Tdev[1] * cwx + (float)Tdev[5] * cwy + (float)Tdev[9] * cwz;
  const float z = (float)Tdev[2] * cwx + (float)Tdev[6] * cwy + (float)Tdev[10] * cwz;
  if (!(z + rad > 0.f)) return f;
  f.verdict = 1;
  if (z - rad <= 1e-3f) return f;  // straddles the camera plane: no projection bound
  const float zn = z - rad, zf = z + rad;
  const float fx = (float)K.fx, fy = (float)K.fy, cx = (float)K.cx, cy = (float)K.cy;
  const float u0 = fx * fminf((x - rad) / zn, (x - rad) / zf) + cx - 2.f;
  const float u1 = fx * fmaxf((x + rad) / zn, (x + rad) / zf) + cx + 2.f;
  const float v0 = fy * fminf((y - rad) / zn, (y - rad) / zf) + cy - 2.f;
  const float v1 = fy * fmaxf((y + rad) / zn, (y + rad) / zf) + cy + 2.f;
  f.verdict = 0;
  if (!(u1 >= -0.5f && v1 >= -0.5f && u0 < (float)K.W && v0 < (float)K.H)) return f;
  const int pu0 = max(0, (int)floorf(u0 + 0.5f)), pu1 = min(K.W - 1, (int)floorf(u1 + 0.5f));
  const int pv0 = max(0, (int)floorf(v0 + 0.5f)), pv1 = min(K.H - 1, (int)floorf(v1 + 0.5f));
  f.t0x = pu0 / kTile; f.t1x = pu1 / kTile; f.t0y = pv0 / kTile; f.t1y = pv1 / kTile;
  f.lvl = tiles;
  f.stride = ntx;
  f.zn = zn;
  f.verdict = 2;
  if ((f.t1x - f.t0x + 1) * (f.t1y - f.t0y + 1) > 64) {  // large footprint: the coarse (8x8-tile) level
    const int nty_f = (K.H + kTile - 1) / kTile;
    f.lvl = tiles + ntx * nty_f;
    f.stride = (ntx + 7) >> 3;
    f.t0x >>= 3; f.t1x >>= 3; f.t0y >>= 3; f.t1y >>= 3;
    if ((f.t1x - f.t0x + 1) * (f.t1y - f.t0y + 1) > max_tiles) f.verdict = 1;
  }
  return f;
}

__device__ __forceinline__ bool footprint_keep(const Geom& g, const Intr& K, const Footprint& f, uint32_t m) {
  if (m == 0) return false;
  const float dmax = (float)((double)m * K.unit);
  return f.zn - 1e-3f < dmax + (float)g.trunc;
}

__device__ __forceinline__ bool box_visible(const Geom& g, const Intr& K, const double* __restrict__ Tdev,
                                            const uint32_t* __restrict__ tiles, int ntx, double cxw, double cyw,
                                            double czw, float rad, int max_tiles) {
  const Footprint f = box_footprint(K, Tdev, tiles, ntx, cxw, cyw, czw, rad, max_tiles);
  if (f.verdict != 2) return f.verdict == 1;
  uint32_t m = 0;
  for (int ty = f.t0y; ty <= f.t1y; ++ty)
    for (int tx = f.t0x; tx <= f.t1x; ++tx) m = max(m, __ldg(f.lvl + ty * f.stride + tx));
  return footprint_keep(g, K, f, m);
}

// Kept-brick list entries carry the brick coordinates packed 10:10:10 bits (grids up to 4096
// voxels per axis, checked at volume creation), so the sweep decodes them with shifts instead of
// two runtime integer divisions per thread.
__device__ __forceinline__ uint32_t pack_brick(int bx, int by, int bz) {
  return ((uint32_t)bz << 20) | ((uint32_t)by << 10) | (uint32_t)bx;
}

__device__ __forceinline__ void append_warp(bool keep, uint32_t v, uint32_t* __restrict__ list,
                                            uint32_t* __restrict__ count) {
  const unsigned ball = __ballot_sync(0xffffffffu, keep);
  if (ball) {
    const int lane = threadIdx.x & 31;
    uint32_t base = 0;
    if (lane == 0) base = atomicAdd(count, (uint32_t)__popc(ball));
    base = __shfl_sync(0xffffffffu, base, 0);
    if (keep) list[base + __popc(ball & ((1u << lane) - 1))] = v;
  }
}

constexpr int kSuper = 8;  // super-brick = 8^3 bricks = 32^3 voxels

// Level 1: one warp per super-brick; the lanes share the footprint's tile loads.
__global__ void k_cull_super(Geom g, Intr K, const double* __restrict__ Tdev, const uint32_t* __restrict__ tiles,
                             int ntx, int nsx, int nsy, int nsz, uint32_t* __restrict__ slist,
                             uint32_t* __restrict__ scount) {
  const uint32_t ns = (uint32_t)nsx * nsy * nsz;
  const uint32_t sb = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;  // warp-uniform
  const int lane = threadIdx.x & 31;
  if (sb >= ns) return;
  const int sx = (int)(sb % (uint32_t)nsx);
  const uint32_t r = sb / (uint32_t)nsx;
  const int sy = (int)(r % (uint32_t)nsy), sz = (int)(r / (uint32_t)nsy);
  // voxel-centre box of the super-brick: voxels [32 s, 32 s + 31] per axis
  const double h = 16.0;
  const Footprint f = box_footprint(K, Tdev, tiles, ntx, g.ox + g.voxel * (32.0 * sx + h), g.oy + g.voxel * (32.0 * sy + h),
                                    g.oz + g.voxel * (32.0 * sz + h), (float)(15.5 * 1.7320508 * g.voxel) + 1e-3f, 64);
  bool keep = f.verdict == 1;
  if (f.verdict == 2) {
    const int nx = f.t1x - f.t0x + 1, nt = nx * (f.t1y - f.t0y + 1);
    uint32_t m = 0;
    for (int t = lane; t < nt; t += 32) m = max(m, __ldg(f.lvl + (f.t0y + t / nx) * f.stride + f.t0x + t % nx));
    for (int s = 16; s > 0; s >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, s));
    keep = footprint_keep(g, K, f, m);
  }
  if (lane == 0 && keep) slist[atomicAdd(scount, 1u)] = sb;
}

// Level 2: the 512 bricks of every surviving super-brick (one CTA of 512 threads per super-brick).
__global__ __launch_bounds__(512) void k_cull_bricks(Geom g, Intr K, const double* __restrict__ Tdev,
                                                     const uint32_t* __restrict__ tiles, int ntx, int nsx, int nsy,
                                                     const uint32_t* __restrict__ slist,
                                                     const uint32_t* __restrict__ scount, uint32_t* __restrict__ list,
                                                     uint32_t* __restrict__ count) {
  const uint32_t n = *scount;
  const int t = threadIdx.x;
  for (uint32_t li = blockIdx.x; li < n; li += gridDim.x) {
    const uint32_t sb = slist[li];
    const int sx = (int)(sb % (uint32_t)nsx);
    const uint32_t r = sb / (uint32_t)nsx;
    const int sy = (int)(r % (uint32_t)nsy), sz = (int)(r / (uint32_t)nsy);
    const int bx = sx * kSuper + (t & 7), by = sy * kSuper + ((t >> 3) & 7), bz = sz * kSuper + (t >> 6);
    bool keep = false;
    if (bx < g.nbx && by < g.nby && bz < g.nbz)
      keep = box_visible(g, K, Tdev, tiles, ntx, g.ox + g.voxel * (4.0 * bx + 2.0), g.oy + g.voxel * (4.0 * by + 2.0),
                         g.oz + g.voxel * (4.0 * bz + 2.0), (float)(1.5 * 1.7320508 * g.voxel) + 1e-3f, 64);
    append_warp(keep, pack_brick(bx, by, bz), list, count);
  }
}

// Sweep of the compacted bricks: 4 bricks per 256-thread CTA, grid-stride over the list.
template <typename T>
__global__ __launch_bounds__(256) void k_integrate_list(Geom g, Intr K, const uint16_t* __restrict__ depth,
                                                        const double* __restrict__ Tdev, const uint32_t* __restrict__ list,
                                                        const uint32_t* __restrict__ count, T* __restrict__ V,
                                                        T* __restrict__ W, uint32_t* __restrict__ dirty,
                                                        uint32_t* __restrict__ dlist, uint32_t* __restrict__ dcount) {
  __shared__ double sT[12];
  if (threadIdx.x < 12) sT[threadIdx.x] = Tdev[threadIdx.x];
  __syncthreads();
  const uint32_t n = *count;
  const uint32_t w = threadIdx.x & 63;
  for (uint32_t li = blockIdx.x * 4 + (threadIdx.x >> 6); li < n; li += gridDim.x * 4) {
    const uint32_t e = list[li];
    const int bx = (int)(e & 1023u), by = (int)((e >> 10) & 1023u), bz = (int)(e >> 20);
    const uint32_t b = ((uint32_t)bz * g.nby + (uint32_t)by) * g.nbx + (uint32_t)bx;
    const int i = bx * 4 + (int)(w & 3), j = by * 4 + (int)((w >> 2) & 3), k = bz * 4 + (int)(w >> 4);
    bool changed = false;
    if (i < g.nx && j < g.ny && k < g.nz) changed = fuse_voxel<T>(g, K, depth, sT, i, j, k, V, W, b * 64u + w);
    // cell-bricks whose records read this voxel: (b - d) for d in {0,1}^3, the -1 neighbours
    // only from the brick's low faces
    unsigned nbm = 0u;
    if (changed) {
      const unsigned ex = (w & 3) == 0, ey = ((w >> 2) & 3) == 0, ez = (w >> 4) == 0;
#pragma unroll
      for (int q = 0; q < 8; ++q)
        if ((!(q & 1) || ex) && (!(q & 2) || ey) && (!(q & 4) || ez)) nbm |= 1u << q;
    }
    nbm = __reduce_or_sync(0xffffffffu, nbm);
    if ((threadIdx.x & 31) == 0 && nbm) mark_dirty_cells(g, bx, by, bz, nbm, dirty, dlist, dcount);
  }
}

pft_status integrate_impl(pft_volume* vol, const uint16_t* depth, const pft_intrinsics* Kp, const double* T,
                          int full_sweep, cudaStream_t st) {
  Intr K{Kp->fx, Kp->fy, Kp->cx, Kp->cy, Kp->depth_unit_m, Kp->width, Kp->height};
  const Geom& g = vol->g;
  const int ntx = (K.W + kTile - 1) / kTile, nty = (K.H + kTile - 1) / kTile;
  const size_t ntiles_all = (size_t)ntx * nty + (size_t)((ntx + 7) >> 3) * ((nty + 7) >> 3);
  if (ntiles_all * 4 > vol->L.tiles_bytes) full_sweep = 1;
  if (full_sweep) {
    size_t n = vol->L.elems;
    size_t blocks = (n + 255) / 256;
    int grid = (int)(blocks < 148 * 64 ? blocks : 148 * 64);
    if (vol->esize == 4)
      PFT_LAUNCH(PFT_PROF_INTEGRATE, st, k_integrate_sweep<float><<<grid, 256, 0, st>>>(g, K, depth, T, (float*)(vol->base + vol->L.v_off),
                                                     (float*)(vol->base + vol->L.w_off), n));
    else
      PFT_LAUNCH(PFT_PROF_INTEGRATE, st, k_integrate_sweep<__half><<<grid, 256, 0, st>>>(g, K, depth, T, (__half*)(vol->base + vol->L.v_off),
                                                      (__half*)(vol->base + vol->L.w_off), n));
    records_rebuild_all(vol, st);
    return cuda_check("integrate (full sweep)");
  }
  uint32_t* tiles = (uint32_t*)(vol->base + vol->L.tiles_off);
  uint32_t* list = (uint32_t*)(vol->base + vol->L.list_off);
  uint32_t* count = (uint32_t*)(vol->base + vol->L.scratch_off + 64);
  uint32_t* dcount = (uint32_t*)(vol->base + vol->L.scratch_off + 128);
  uint32_t* dirty = (uint32_t*)(vol->base + vol->L.dirty_off);
  uint32_t* dlist = (uint32_t*)(vol->base + vol->L.dlist_off);
  cudaMemsetAsync(count, 0, 192, st);  // active, dirty and super-brick counts (scratch +64..+255)
  cudaMemsetAsync(tiles + (size_t)ntx * nty, 0, 4 * (size_t)((ntx + 7) >> 3) * ((nty + 7) >> 3), st);  // coarse level
  {
    dim3 blk(32, 8);
    int nt = ntx * nty;
    PFT_LAUNCH(PFT_PROF_CULL, st, k_depth_tiles<<<(nt + 7) / 8, blk, 0, st>>>(K, g.max_depth, depth, tiles, ntx, nty));
  }
  const int nsx = (g.nbx + kSuper - 1) / kSuper, nsy = (g.nby + kSuper - 1) / kSuper, nsz = (g.nbz + kSuper - 1) / kSuper;
  const uint32_t ns = (uint32_t)nsx * nsy * nsz;
  uint32_t* slist = (uint32_t*)(vol->base + vol->L.slist_off);
  uint32_t* scount = (uint32_t*)(vol->base + vol->L.scratch_off + 192);
  PFT_LAUNCH(PFT_PROF_CULL, st, k_cull_super<<<(ns * 32 + 255) / 256, 256, 0, st>>>(g, K, T, tiles, ntx, nsx, nsy, nsz, slist, scount));
  PFT_LAUNCH(PFT_PROF_CULL, st, k_cull_bricks<<<148 * 4, 512, 0, st>>>(g, K, T, tiles, ntx, nsx, nsy, slist, scount, list, count));
  const int grid = 148 * 8;
  if (vol->esize == 4)
    PFT_LAUNCH(PFT_PROF_INTEGRATE, st, k_integrate_list<float><<<grid, 256, 0, st>>>(g, K, depth, T, list, count, (float*)(vol->base + vol->L.v_off),
                                                  (float*)(vol->base + vol->L.w_off), dirty, dlist, dcount));
  else
    PFT_LAUNCH(PFT_PROF_INTEGRATE, st, k_integrate_list<__half><<<grid, 256, 0, st>>>(g, K, depth, T, list, count, (__half*)(vol->base + vol->L.v_off),
                                                   (__half*)(vol->base + vol->L.w_off), dirty, dlist, dcount));
  records_rebuild_dirty(vol, st);
  return cuda_check("integrate");
}

}  // namespace pft

using namespace pft;

extern "C" {

pft_status pft_integrate_ex(pft_volume* vol, const uint16_t* dev_depth, const pft_intrinsics* K, const double* dev_T,
                            int32_t flags, void* stream) {
  if (!vol || !dev_depth || !dev_T) return fail(PFT_ERR_INVALID_ARG, "NULL argument");
  pft_status s = check_intrinsics(K);
  if (s != PFT_OK) return s;
  return integrate_impl(vol, dev_depth, K, dev_T, flags & 1, (cudaStream_t)stream);
}

pft_status pft_integrate(pft_volume* vol, const uint16_t* dev_depth, const pft_intrinsics* K, const double* dev_T,
                         void* stream) {
  return pft_integrate_ex(vol, dev_depth, K, dev_T, 0, stream);
}

}  // extern "C"
