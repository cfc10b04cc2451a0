// volume.cu — TSDF volume storage: layout, reset, canonical<->brick conversion, checksum.
// The TSDF is "a tensor that records the distance value in each 3D grid";
// unobserved voxels hold V = 1, W = 0 (reading L3).
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <new>

#include "pft_internal.cuh"
#include "records.cuh"

namespace pft {

static size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

static pft_status check_desc(const pft_volume_desc* d) {
  if (!d) return fail(PFT_ERR_INVALID_ARG, "desc is NULL");
  if (d->nx < 2 || d->ny < 2 || d->nz < 2) return fail(PFT_ERR_INVALID_ARG, "dims must be >= 2 (got %d %d %d)", d->nx, d->ny, d->nz);
  if (d->nx > 4096 || d->ny > 4096 || d->nz > 4096)
    return fail(PFT_ERR_INVALID_ARG, "dims must be <= 4096 (got %d %d %d)", d->nx, d->ny, d->nz);
  if (!(d->voxel_m > 0.0)) return fail(PFT_ERR_INVALID_ARG, "voxel_m must be > 0");
  if (!(d->trunc_m >= 2.0 * d->voxel_m)) return fail(PFT_ERR_INVALID_ARG, "trunc_m must be >= 2*voxel_m (SPEC.md:219)");
  if (!(d->max_weight >= 1.0)) return fail(PFT_ERR_INVALID_ARG, "max_weight must be >= 1");
  if (!(d->max_depth_m > 0.0)) return fail(PFT_ERR_INVALID_ARG, "max_depth_m must be > 0");
  for (int a = 0; a < 3; ++a)
    if (!(d->origin_m[a] == d->origin_m[a]) || d->origin_m[a] > 1e30 || d->origin_m[a] < -1e30)
      return fail(PFT_ERR_INVALID_ARG, "origin_m must be finite");
  if (d->storage != PFT_STORE_F32 && d->storage != PFT_STORE_F16) return fail(PFT_ERR_INVALID_ARG, "bad storage");
  return PFT_OK;
}

static pft_status make_layout(const pft_volume_desc* d, Geom* g, VolLayout* L, size_t* esize) {
  pft_status s = check_desc(d);
  if (s != PFT_OK) return s;
  g->nx = d->nx; g->ny = d->ny; g->nz = d->nz;
  g->nbx = (d->nx + kBrick - 1) / kBrick;
  g->nby = (d->ny + kBrick - 1) / kBrick;
  g->nbz = (d->nz + kBrick - 1) / kBrick;
  size_t nb = (size_t)g->nbx * g->nby * g->nbz;
  size_t elems = nb * kBrickVox;
  if (elems > ((size_t)1 << 31)) return fail(PFT_ERR_UNSUPPORTED, "padded grid has %zu voxels (> 2^31)", elems);
  g->sy = (uint32_t)(kBrickVox * g->nbx);
  g->sz = (uint32_t)((size_t)kBrickVox * g->nbx * g->nby);
  g->voxel = d->voxel_m;
  g->ox = d->origin_m[0]; g->oy = d->origin_m[1]; g->oz = d->origin_m[2];
  g->trunc = d->trunc_m; g->max_weight = d->max_weight; g->max_depth = d->max_depth_m;
  *esize = d->storage == PFT_STORE_F32 ? 4 : 2;
  size_t off = 0;
  L->scratch_off = off; L->scratch_bytes = 4096; off += 4096;
  L->v_off = off; L->elems = elems; off = align_up(off + elems * *esize, 256);
  L->w_off = off; off = align_up(off + elems * *esize, 256);
  L->r_off = off; off = align_up(off + elems * 8 * *esize, 256);
  L->m_off = off; off = align_up(off + nb * 8, 256);
  L->list_off = off; L->list_bytes = nb * 4; off = align_up(off + L->list_bytes, 256);
  L->dirty_off = off; off = align_up(off + nb * 4, 256);
  {
    const size_t nsup = (size_t)((g->nbx + 3) / 4) * ((g->nby + 3) / 4) * ((g->nbz + 3) / 4);  // 4^3-brick super-bricks
    L->slist_off = off; off = align_up(off + (nsup + 64) * 4, 256);  // super-brick list
  }
  L->dlist_off = off; off = align_up(off + nb * 4, 256);
  L->tiles_off = off; L->tiles_bytes = 64 * 1024 * 4; off = align_up(off + L->tiles_bytes, 256);
  L->axis_off = off; off = align_up(off + 4 * (size_t)(g->nbx + g->nby + g->nbz) * 4 * sizeof(double), 256);
  L->total = off;
  return PFT_OK;
}

// ------------------------------------------------------------------ kernels
template <typename T> __device__ __forceinline__ T from_double(double x);
template <> __device__ __forceinline__ float from_double<float>(double x) { return __double2float_rn(x); }
template <> __device__ __forceinline__ __half from_double<__half>(double x) { return __double2half(x); }

template <typename T>
__global__ void k_reset(T* __restrict__ V, T* __restrict__ W, size_t n) {
  const T one = from_double<T>(1.0), zero = from_double<T>(0.0);
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    V[i] = one;
    W[i] = zero;
  }
}

template <typename T>
__global__ void k_fill(T* __restrict__ R, size_t n, float val) {
  const T v = from_double<T>((double)val);
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) R[i] = v;
}

// (build_record, records_dirty_pass: records.cuh)

// Every cell: one thread per brick element (cells beyond n-2 are never read and are skipped).
// Every cell: one thread per brick element; a warp covers half a brick, so the two 32-bit
// halves of each brick's mask word are written by ballots without atomics.
template <typename T>
__global__ void k_records_all(Geom g, const T* __restrict__ V, T* __restrict__ R, uint32_t* __restrict__ mask,
                              size_t nelem) {
  for (size_t e0 = blockIdx.x * (size_t)blockDim.x; e0 < nelem; e0 += (size_t)gridDim.x * blockDim.x) {
    const size_t e = e0 + threadIdx.x;
    bool in = false;
    if (e < nelem) {
      const uint32_t b = (uint32_t)(e >> 6), w = (uint32_t)(e & 63);
      const int bx = (int)(b % (uint32_t)g.nbx);
      const uint32_t r = b / (uint32_t)g.nbx;
      const int by = (int)(r % (uint32_t)g.nby), bz = (int)(r / (uint32_t)g.nby);
      const int cx = bx * 4 + (int)(w & 3), cy = by * 4 + (int)((w >> 2) & 3), cz = bz * 4 + (int)(w >> 4);
      if (cx <= g.nx - 2 && cy <= g.ny - 2 && cz <= g.nz - 2) in = build_record<T>(g, V, R, cx, cy, cz);
    }
    const unsigned bal = __ballot_sync(0xffffffffu, in);
    if ((threadIdx.x & 31) == 0 && e < nelem) mask[e >> 5] = bal;
  }
}

// Dirty cell-bricks (records.cuh records_dirty_pass), one launch.
template <typename T>
__global__ __launch_bounds__(256) void k_records_dirty(Geom g, const T* __restrict__ V, T* __restrict__ R,
                                                       uint32_t* __restrict__ mask, uint32_t* __restrict__ dirty,
                                                       const uint32_t* __restrict__ dlist,
                                                       const uint32_t* __restrict__ dcount) {
  pdl_wait();  // the fusion kernel's dirty list
  pdl_trigger();
  records_dirty_pass<T>(g, V, R, mask, dirty, dlist, *dcount, blockIdx.x, gridDim.x);
}

// canonical index -> brick element offset
__device__ __forceinline__ uint32_t brick_of(const Geom& g, size_t idx) {
  int x = (int)(idx % (size_t)g.nx);
  size_t r = idx / (size_t)g.nx;
  int y = (int)(r % (size_t)g.ny);
  int z = (int)(r / (size_t)g.ny);
  return offx(x) + offy(y, g.sy) + offz(z, g.sz);
}

template <typename T>
__global__ void k_upload(Geom g, const T* __restrict__ sv, const T* __restrict__ sw, T* __restrict__ V,
                         T* __restrict__ W, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint32_t o = brick_of(g, i);
    V[o] = sv[i];
    W[o] = sw[i];
  }
}

template <typename T>
__global__ void k_download(Geom g, const T* __restrict__ V, const T* __restrict__ W, T* __restrict__ dv,
                           T* __restrict__ dw, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint32_t o = brick_of(g, i);
    if (dv) dv[i] = V[o];
    if (dw) dw[i] = W[o];
  }
}

__device__ __forceinline__ unsigned long long mix64(unsigned long long z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// h = sum over canonical voxels of mix64(idx * GOLDEN + (Vbits | Wbits << 32)) mod 2^64.
template <typename T>
__global__ void k_checksum(Geom g, const T* __restrict__ V, const T* __restrict__ W, size_t n,
                           unsigned long long* out) {
  unsigned long long h = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint32_t o = brick_of(g, i);
    unsigned long long vb, wb;
    if (sizeof(T) == 4) {
      vb = __float_as_uint(*(const float*)&V[o]);
      wb = __float_as_uint(*(const float*)&W[o]);
    } else {
      vb = *(const unsigned short*)&V[o];
      wb = *(const unsigned short*)&W[o];
    }
    h += mix64((unsigned long long)i * 0x9E3779B97F4A7C15ull + (vb | (wb << 32)));
  }
  for (int s = 16; s > 0; s >>= 1) h += __shfl_xor_sync(0xffffffffu, h, s);
  if ((threadIdx.x & 31) == 0) atomicAdd(out, h);
}

static int grid_for(size_t n, int threads) {
  size_t b = (n + threads - 1) / threads;
  size_t cap = 148 * 32;
  return (int)(b < cap ? (b ? b : 1) : cap);
}

pft_status volume_reset_impl(pft_volume* vol, cudaStream_t st) {
  size_t n = vol->L.elems;
  if (vol->esize == 4) {
    PFT_LAUNCH(PFT_PROF_OTHER, st, k_reset<float><<<grid_for(n, 256), 256, 0, st>>>((float*)(vol->base + vol->L.v_off), (float*)(vol->base + vol->L.w_off), n));
    PFT_LAUNCH(PFT_PROF_OTHER, st, k_fill<float><<<grid_for(8 * n, 256), 256, 0, st>>>((float*)(vol->base + vol->L.r_off), 8 * n, 1.0f));
  } else {
    PFT_LAUNCH(PFT_PROF_OTHER, st, k_reset<__half><<<grid_for(n, 256), 256, 0, st>>>((__half*)(vol->base + vol->L.v_off), (__half*)(vol->base + vol->L.w_off), n));
    PFT_LAUNCH(PFT_PROF_OTHER, st, k_fill<__half><<<grid_for(8 * n, 256), 256, 0, st>>>((__half*)(vol->base + vol->L.r_off), 8 * n, 1.0f));
  }
  cudaMemsetAsync(vol->base + vol->L.m_off, 0, (n / 64) * 8, st);  // nothing is in band
  cudaMemsetAsync(vol->base + vol->L.dirty_off, 0, (n / 64) * 4, st);
  return cuda_check("volume_reset");
}

void records_rebuild_all(pft_volume* vol, cudaStream_t st) {
  size_t n = vol->L.elems;
  if (vol->esize == 4)
    PFT_LAUNCH(PFT_PROF_RECORDS, st, k_records_all<float><<<grid_for(n, 256), 256, 0, st>>>(vol->g, (const float*)(vol->base + vol->L.v_off), (float*)(vol->base + vol->L.r_off), (uint32_t*)(vol->base + vol->L.m_off), n));
  else
    PFT_LAUNCH(PFT_PROF_RECORDS, st, k_records_all<__half><<<grid_for(n, 256), 256, 0, st>>>(vol->g, (const __half*)(vol->base + vol->L.v_off), (__half*)(vol->base + vol->L.r_off), (uint32_t*)(vol->base + vol->L.m_off), n));
}

void records_rebuild_dirty(pft_volume* vol, cudaStream_t st) {
  const int grid = 148 * 8;
  uint32_t* dirty = (uint32_t*)(vol->base + vol->L.dirty_off);
  const uint32_t* dlist = (const uint32_t*)(vol->base + vol->L.dlist_off);
  const uint32_t* dcount = (const uint32_t*)(vol->base + vol->L.scratch_off + 128);
  if (vol->esize == 4)
    PFT_LAUNCH(PFT_PROF_RECORDS, st, launch_pdl(k_records_dirty<float>, dim3(grid), dim3(256), 0, st, vol->g, (const float*)(vol->base + vol->L.v_off), (float*)(vol->base + vol->L.r_off), (uint32_t*)(vol->base + vol->L.m_off), dirty, dlist, dcount));
  else
    PFT_LAUNCH(PFT_PROF_RECORDS, st, launch_pdl(k_records_dirty<__half>, dim3(grid), dim3(256), 0, st, vol->g, (const __half*)(vol->base + vol->L.v_off), (__half*)(vol->base + vol->L.r_off), (uint32_t*)(vol->base + vol->L.m_off), dirty, dlist, dcount));
}

}  // namespace pft

using namespace pft;

extern "C" {

pft_status pft_volume_bytes(const pft_volume_desc* desc, size_t* bytes_out) {
  if (!bytes_out) return fail(PFT_ERR_INVALID_ARG, "bytes_out is NULL");
  Geom g; VolLayout L; size_t es;
  pft_status s = make_layout(desc, &g, &L, &es);
  if (s != PFT_OK) return s;
  *bytes_out = L.total;
  return PFT_OK;
}

pft_status pft_volume_create(const pft_volume_desc* desc, void* dev_storage, size_t bytes, pft_volume** out) {
  if (!out) return fail(PFT_ERR_INVALID_ARG, "out is NULL");
  *out = nullptr;
  if (!dev_storage) return fail(PFT_ERR_INVALID_ARG, "dev_storage is NULL");
  if (((uintptr_t)dev_storage) % 256) return fail(PFT_ERR_INVALID_ARG, "dev_storage must be 256-byte aligned");
  Geom g; VolLayout L; size_t es;
  pft_status s = make_layout(desc, &g, &L, &es);
  if (s != PFT_OK) return s;
  if (bytes < L.total) return fail(PFT_ERR_BUFFER_TOO_SMALL, "storage %zu B < required %zu B", bytes, L.total);
  pft_volume* v = new (std::nothrow) pft_volume;
  if (!v) return fail(PFT_ERR_INVALID_ARG, "host allocation failed");
  v->desc = *desc; v->g = g; v->L = L; v->esize = es; v->base = (char*)dev_storage;
  cudaGetDevice(&v->device);
  v->nccl_comm = nullptr; v->nranks = 1; v->rank = 0; v->virtual_ranks = 0; v->virtual_fused = 0;
  v->p2p = 0; v->xown = nullptr; v->xbytes = 0; v->xcnt_off = 0; v->xmax_particles = 0;
  v->partition = PFT_PARTITION_PARTICLES; v->preflight_round = 0;
  for (int q = 0; q < PFT_MAX_FUSED_RANKS; ++q) v->xbuf[q] = nullptr;
  v->xws_last = nullptr; v->xws_total = v->xws_region = v->xws_xcnt = 0;
  *out = v;
  return PFT_OK;
}

pft_status pft_volume_reset(pft_volume* vol, void* stream) {
  if (!vol) return fail(PFT_ERR_INVALID_ARG, "vol is NULL");
  return volume_reset_impl(vol, (cudaStream_t)stream);
}

pft_status pft_volume_upload(pft_volume* vol, const void* dv, const void* dw, void* stream) {
  if (!vol || !dv || !dw) return fail(PFT_ERR_INVALID_ARG, "NULL argument");
  cudaStream_t st = (cudaStream_t)stream;
  pft_status s = volume_reset_impl(vol, st);  // padding voxels of partial bricks: V=1, W=0
  if (s != PFT_OK) return s;
  size_t n = (size_t)vol->g.nx * vol->g.ny * vol->g.nz;
  if (vol->esize == 4)
    PFT_LAUNCH(PFT_PROF_OTHER, st, k_upload<float><<<grid_for(n, 256), 256, 0, st>>>(vol->g, (const float*)dv, (const float*)dw,
        (float*)(vol->base + vol->L.v_off), (float*)(vol->base + vol->L.w_off), n));
  else
    PFT_LAUNCH(PFT_PROF_OTHER, st, k_upload<__half><<<grid_for(n, 256), 256, 0, st>>>(vol->g, (const __half*)dv, (const __half*)dw,
        (__half*)(vol->base + vol->L.v_off), (__half*)(vol->base + vol->L.w_off), n));
  records_rebuild_all(vol, st);
  return cuda_check("volume_upload");
}

pft_status pft_volume_download(const pft_volume* vol, void* dv, void* dw, void* stream) {
  if (!vol) return fail(PFT_ERR_INVALID_ARG, "vol is NULL");
  if (!dv && !dw) return PFT_OK;
  cudaStream_t st = (cudaStream_t)stream;
  size_t n = (size_t)vol->g.nx * vol->g.ny * vol->g.nz;
  if (vol->esize == 4)
    PFT_LAUNCH(PFT_PROF_OTHER, st, k_download<float><<<grid_for(n, 256), 256, 0, st>>>(vol->g, (const float*)(vol->base + vol->L.v_off),
        (const float*)(vol->base + vol->L.w_off), (float*)dv, (float*)dw, n));
  else
    PFT_LAUNCH(PFT_PROF_OTHER, st, k_download<__half><<<grid_for(n, 256), 256, 0, st>>>(vol->g, (const __half*)(vol->base + vol->L.v_off),
        (const __half*)(vol->base + vol->L.w_off), (__half*)dv, (__half*)dw, n));
  return cuda_check("volume_download");
}

pft_status pft_volume_checksum(const pft_volume* vol, uint64_t* host_out, void* stream) {
  if (!vol || !host_out) return fail(PFT_ERR_INVALID_ARG, "NULL argument");
  cudaStream_t st = (cudaStream_t)stream;
  unsigned long long* acc = (unsigned long long*)(vol->base + vol->L.scratch_off);
  cudaMemsetAsync(acc, 0, 8, st);
  size_t n = (size_t)vol->g.nx * vol->g.ny * vol->g.nz;
  if (vol->esize == 4)
    PFT_LAUNCH(PFT_PROF_OTHER, st, k_checksum<float><<<grid_for(n, 256), 256, 0, st>>>(vol->g, (const float*)(vol->base + vol->L.v_off),
        (const float*)(vol->base + vol->L.w_off), n, acc));
  else
    PFT_LAUNCH(PFT_PROF_OTHER, st, k_checksum<__half><<<grid_for(n, 256), 256, 0, st>>>(vol->g, (const __half*)(vol->base + vol->L.v_off),
        (const __half*)(vol->base + vol->L.w_off), n, acc));
  pft_status s = cuda_check("volume_checksum");
  if (s != PFT_OK) return s;
  unsigned long long h = 0;
  if (cudaMemcpyAsync(&h, acc, 8, cudaMemcpyDeviceToHost, st) != cudaSuccess || cudaStreamSynchronize(st) != cudaSuccess)
    return cuda_check("volume_checksum copy");
  *host_out = h;
  return PFT_OK;
}

}  // extern "C"
