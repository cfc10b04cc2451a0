// abi.cu — error reporting, shared validation, volume destruction and the NCCL plumbing of
// the multi-GPU path (north_star: particles sharded across the GPUs of one box, volume
// replicated, per-particle fitness all-gathered over NVLink).
//
// NCCL is loaded with dlopen at pft_comm_init time ("libnccl.so.2", normally already mapped
// by torch), so the library loads and runs single-GPU without NCCL on the link line.
#include <dlfcn.h>

#include <cstdarg>
#include <cstdio>
#include <atomic>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>

#include <nccl.h>

#include "pft_internal.cuh"

namespace pft {

static thread_local char g_err[512] = "";

pft_status fail(pft_status s, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof g_err, fmt, ap);
  va_end(ap);
  return s;
}

pft_status cuda_check(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) return PFT_OK;
  return fail(PFT_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

pft_status check_intrinsics(const pft_intrinsics* K) {
  if (!K) return fail(PFT_ERR_INVALID_ARG, "intrinsics is NULL");
  if (!(K->fx > 0.0) || !(K->fy > 0.0)) return fail(PFT_ERR_INVALID_ARG, "fx, fy must be > 0 (SPEC.md:149)");
  if (K->width < 1 || K->height < 1 || K->width > 16384 || K->height > 16384)
    return fail(PFT_ERR_INVALID_ARG, "bad image size %dx%d", K->width, K->height);
  if (!(K->depth_unit_m > 0.0)) return fail(PFT_ERR_INVALID_ARG, "depth_unit_m must be > 0");
  if (!(K->cx == K->cx) || !(K->cy == K->cy)) return fail(PFT_ERR_INVALID_ARG, "cx, cy must be finite");
  return PFT_OK;
}

// ------------------------------------------------------------------ instrumentation

static std::atomic<unsigned long long> g_launches{0};
static std::atomic<bool> g_prof_on{false};
struct ProfRec { int cls; cudaEvent_t a, b; };
static std::mutex g_prof_mu;
static std::vector<ProfRec> g_prof;       // recorded this session
static std::vector<cudaEvent_t> g_pool;   // reusable events
static thread_local cudaEvent_t t_open = nullptr;
constexpr size_t kProfMax = 65536;

static cudaEvent_t ev_get() {
  if (!g_pool.empty()) { cudaEvent_t e = g_pool.back(); g_pool.pop_back(); return e; }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}

bool pdl_enabled() {
  static const bool on = [] {
    const char* e = getenv("PFT_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}

void prof_begin(int cls, cudaStream_t st) {
  (void)cls;
  g_launches.fetch_add(1, std::memory_order_relaxed);
  if (!g_prof_on.load(std::memory_order_relaxed)) return;
  std::lock_guard<std::mutex> lk(g_prof_mu);
  if (g_prof.size() >= kProfMax) return;
  t_open = ev_get();
  cudaEventRecord(t_open, st);
}

// PFT_SYNC_DEBUG=1: synchronise after every launch and name the kernel that failed (stderr).
static const bool g_sync_debug = [] {
  const char* e = getenv("PFT_SYNC_DEBUG");
  return e && e[0] == '1';
}();

void prof_end(int cls, cudaStream_t st, const char* what) {
  if (g_sync_debug) {
    cudaError_t e = cudaStreamSynchronize(st);
    if (e == cudaSuccess) e = cudaGetLastError();
    if (e != cudaSuccess) fprintf(stderr, "pft: launch failed (%s): %.160s\n", cudaGetErrorString(e), what);
  }
  if (!g_prof_on.load(std::memory_order_relaxed) || !t_open) return;
  std::lock_guard<std::mutex> lk(g_prof_mu);
  cudaEvent_t b = ev_get();
  cudaEventRecord(b, st);
  g_prof.push_back(ProfRec{cls, t_open, b});
  t_open = nullptr;
}

// ------------------------------------------------------------------ NCCL via dlopen
struct Nccl {
  void* h = nullptr;
  decltype(&ncclGetUniqueId) getUniqueId = nullptr;
  decltype(&ncclCommInitRank) commInitRank = nullptr;
  decltype(&ncclCommDestroy) commDestroy = nullptr;
  decltype(&ncclAllGather) allGather = nullptr;
  decltype(&ncclAllReduce) allReduce = nullptr;
  decltype(&ncclGetErrorString) errStr = nullptr;
  decltype(&ncclCommGetAsyncError) asyncErr = nullptr;
};

static Nccl* nccl() {
  static Nccl n;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (h) {
      n.getUniqueId = (decltype(n.getUniqueId))dlsym(h, "ncclGetUniqueId");
      n.commInitRank = (decltype(n.commInitRank))dlsym(h, "ncclCommInitRank");
      n.commDestroy = (decltype(n.commDestroy))dlsym(h, "ncclCommDestroy");
      n.allGather = (decltype(n.allGather))dlsym(h, "ncclAllGather");
      n.allReduce = (decltype(n.allReduce))dlsym(h, "ncclAllReduce");
      n.errStr = (decltype(n.errStr))dlsym(h, "ncclGetErrorString");
      n.asyncErr = (decltype(n.asyncErr))dlsym(h, "ncclCommGetAsyncError");
      if (n.getUniqueId && n.commInitRank && n.commDestroy && n.allGather && n.allReduce && n.errStr) n.h = h;
    }
  }
  return n.h ? &n : nullptr;
}

// Asynchronous NCCL failures (a peer died, a network error) surface through the communicator's
// async error state, not through the enqueue call: polled after every collective, mapped to
// PFT_ERR_NCCL (include/pft.h).
static pft_status nccl_async_check(Nccl* n, pft_volume* vol, const char* what) {
  if (!n->asyncErr) return PFT_OK;
  ncclResult_t a = ncclSuccess;
  if (n->asyncErr((ncclComm_t)vol->nccl_comm, &a) != ncclSuccess) return PFT_OK;
  if (a != ncclSuccess && a != ncclInProgress) return fail(PFT_ERR_NCCL, "%s: asynchronous error %s", what, n->errStr(a));
  return PFT_OK;
}

pft_status comm_allgather(pft_volume* vol, const void* send, void* recv, size_t bytes_per_rank, cudaStream_t st) {
  Nccl* n = nccl();
  if (!n || !vol->nccl_comm) return fail(PFT_ERR_STATE, "communicator not initialised");
  prof_begin(PFT_PROF_COMM, st);
  ncclResult_t r = n->allGather(send, recv, bytes_per_rank, ncclUint8, (ncclComm_t)vol->nccl_comm, st);
  prof_end(PFT_PROF_COMM, st, "ncclAllGather");
  if (r != ncclSuccess) return fail(PFT_ERR_NCCL, "ncclAllGather: %s", n->errStr(r));
  return nccl_async_check(n, vol, "ncclAllGather");
}

// In-place sum of `count` uint64 words over the ranks (point-sharded partition, F2b).
pft_status comm_allreduce_u64(pft_volume* vol, void* buf, size_t count, cudaStream_t st) {
  Nccl* n = nccl();
  if (!n || !vol->nccl_comm) return fail(PFT_ERR_STATE, "communicator not initialised");
  prof_begin(PFT_PROF_COMM, st);
  ncclResult_t r = n->allReduce(buf, buf, count, ncclUint64, ncclSum, (ncclComm_t)vol->nccl_comm, st);
  prof_end(PFT_PROF_COMM, st, "ncclAllReduce");
  if (r != ncclSuccess) return fail(PFT_ERR_NCCL, "ncclAllReduce: %s", n->errStr(r));
  return nccl_async_check(n, vol, "ncclAllReduce");
}

}  // namespace pft

using namespace pft;

extern "C" {

const char* pft_last_error(void) { return g_err; }

int32_t pft_abi_version(void) { return PFT_ABI_VERSION; }

uint64_t pft_launch_count(void) { return g_launches.load(); }

pft_status pft_profile_start(void) {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  for (auto& r : g_prof) { g_pool.push_back(r.a); g_pool.push_back(r.b); }
  g_prof.clear();
  g_prof_on.store(true);
  return PFT_OK;
}

pft_status pft_profile_stop(double* ms_out, int64_t* launches_out) {
  g_prof_on.store(false);
  std::lock_guard<std::mutex> lk(g_prof_mu);
  double ms[PFT_PROF_CLASSES] = {0};
  int64_t cnt[PFT_PROF_CLASSES] = {0};
  pft_status s = PFT_OK;
  for (auto& r : g_prof) {
    if (cudaEventSynchronize(r.b) != cudaSuccess) { s = cuda_check("profile_stop"); break; }
    float t = 0.f;
    cudaEventElapsedTime(&t, r.a, r.b);
    if (r.cls >= 0 && r.cls < PFT_PROF_CLASSES) { ms[r.cls] += t; cnt[r.cls] += 1; }
  }
  for (auto& r : g_prof) { g_pool.push_back(r.a); g_pool.push_back(r.b); }
  g_prof.clear();
  for (int i = 0; i < PFT_PROF_CLASSES; ++i) {
    if (ms_out) ms_out[i] = ms[i];
    if (launches_out) launches_out[i] = cnt[i];
  }
  return s;
}

pft_status pft_volume_destroy(pft_volume* vol) {
  if (!vol) return PFT_OK;
  if (vol->nccl_comm) {
    Nccl* n = nccl();
    if (n) n->commDestroy((ncclComm_t)vol->nccl_comm);
  }
  if (vol->p2p)
    for (int q = 0; q < vol->nranks; ++q)
      if (q != vol->rank && vol->xbuf[q]) cudaIpcCloseMemHandle(vol->xbuf[q]);
  if (vol->xown) cudaFree(vol->xown);
  delete vol;
  return PFT_OK;
}

pft_status pft_comm_get_unique_id(uint8_t id_out[128]) {
  if (!id_out) return fail(PFT_ERR_INVALID_ARG, "id_out is NULL");
  Nccl* n = nccl();
  if (!n) return fail(PFT_ERR_NCCL, "libnccl.so.2 not loadable: %s", dlerror());
  ncclUniqueId id;
  ncclResult_t r = n->getUniqueId(&id);
  if (r != ncclSuccess) return fail(PFT_ERR_NCCL, "ncclGetUniqueId: %s", n->errStr(r));
  memcpy(id_out, id.internal, 128);
  return PFT_OK;
}

pft_status pft_comm_init_virtual(pft_volume* vol, int32_t nranks) {
  if (!vol) return fail(PFT_ERR_INVALID_ARG, "vol is NULL");
  if (nranks < 1) return fail(PFT_ERR_INVALID_ARG, "nranks must be >= 1");
  if (vol->nccl_comm) return fail(PFT_ERR_STATE, "a real communicator is attached");
  if (vol->p2p) return fail(PFT_ERR_STATE, "peer exchange buffers are attached");
  vol->nranks = nranks;
  vol->rank = 0;
  vol->virtual_ranks = nranks > 1 ? nranks : 0;
  vol->virtual_fused = 0;
  return PFT_OK;
}

pft_status pft_comm_init_virtual_fused(pft_volume* vol, int32_t nranks) {
  if (!vol) return fail(PFT_ERR_INVALID_ARG, "vol is NULL");
  if (nranks < 1 || nranks > PFT_MAX_FUSED_RANKS)
    return fail(PFT_ERR_INVALID_ARG, "nranks must be in [1,%d]", PFT_MAX_FUSED_RANKS);
  if (vol->nccl_comm) return fail(PFT_ERR_STATE, "a real communicator is attached");
  if (vol->p2p) return fail(PFT_ERR_STATE, "peer exchange buffers are attached");
  vol->nranks = nranks;
  vol->rank = 0;
  vol->virtual_ranks = nranks > 1 ? nranks : 0;
  vol->virtual_fused = nranks > 1 ? 1 : 0;
  vol->xws_last = nullptr;
  vol->xws_total = vol->xws_region = vol->xws_xcnt = 0;
  return PFT_OK;
}

pft_status pft_comm_p2p_init(pft_volume* vol, int32_t nranks, int32_t rank, int32_t max_particles,
                             uint8_t handle_out[PFT_IPC_HANDLE_BYTES]) {
  if (!vol || !handle_out) return fail(PFT_ERR_INVALID_ARG, "NULL argument");
  if (nranks < 2 || nranks > PFT_MAX_FUSED_RANKS)
    return fail(PFT_ERR_INVALID_ARG, "nranks must be in [2,%d]", PFT_MAX_FUSED_RANKS);
  if (rank < 0 || rank >= nranks) return fail(PFT_ERR_INVALID_ARG, "bad rank %d of %d", rank, nranks);
  if (max_particles < 1) return fail(PFT_ERR_INVALID_ARG, "max_particles must be >= 1");
  if (vol->p2p || vol->xown) return fail(PFT_ERR_STATE, "peer exchange already initialised");
  if (vol->nccl_comm || vol->virtual_ranks) return fail(PFT_ERR_STATE, "another communicator is attached");
  const size_t kloc = ((size_t)max_particles + nranks - 1) / nranks;
  const size_t rec = (2 * sizeof(pft::PartRec) * kloc * (size_t)nranks + 255) / 256 * 256;
  // records (2 halves), then kMaxFusedRanks round counters + the completed-round word, then
  // kMaxFusedRanks preflight tokens and the preflight result word (pft_comm_p2p_preflight)
  const size_t bytes = rec + (2 * pft::kMaxFusedRanks + 2) * sizeof(unsigned long long);
  char* p = nullptr;
  cudaError_t e = cudaMalloc(&p, bytes);
  if (e != cudaSuccess) return fail(PFT_ERR_CUDA, "exchange buffer (%zu B): %s", bytes, cudaGetErrorString(e));
  e = cudaMemset(p, 0, bytes);
  cudaIpcMemHandle_t h;
  if (e == cudaSuccess) e = cudaIpcGetMemHandle(&h, p);
  if (e != cudaSuccess) {
    cudaFree(p);
    return fail(PFT_ERR_CUDA, "exchange buffer IPC handle: %s", cudaGetErrorString(e));
  }
  static_assert(sizeof(h) == PFT_IPC_HANDLE_BYTES, "IPC handle size");
  memcpy(handle_out, &h, sizeof(h));
  vol->xown = p;
  vol->xbytes = bytes;
  vol->xcnt_off = rec;
  vol->xmax_particles = max_particles;
  vol->nranks = nranks;
  vol->rank = rank;
  return PFT_OK;
}

pft_status pft_comm_p2p_detach(pft_volume* vol) {
  if (!vol) return fail(PFT_ERR_INVALID_ARG, "vol is NULL");
  if (vol->p2p)
    for (int q = 0; q < vol->nranks; ++q)
      if (q != vol->rank && vol->xbuf[q]) cudaIpcCloseMemHandle(vol->xbuf[q]);
  for (int q = 0; q < PFT_MAX_FUSED_RANKS; ++q) vol->xbuf[q] = nullptr;
  vol->p2p = 0;
  if (vol->xown) cudaFree(vol->xown);
  vol->xown = nullptr;
  vol->xbytes = vol->xcnt_off = 0;
  vol->xmax_particles = 0;
  if (!vol->nccl_comm) { vol->nranks = 1; vol->rank = 0; }
  return PFT_OK;
}

pft_status pft_comm_p2p_attach(pft_volume* vol, const uint8_t* handles) {
  if (!vol || !handles) return fail(PFT_ERR_INVALID_ARG, "NULL argument");
  if (!vol->xown) return fail(PFT_ERR_STATE, "pft_comm_p2p_init was not called");
  if (vol->p2p) return fail(PFT_ERR_STATE, "peers already attached");
  for (int q = 0; q < vol->nranks; ++q) {
    if (q == vol->rank) { vol->xbuf[q] = vol->xown; continue; }
    cudaIpcMemHandle_t h;
    memcpy(&h, handles + (size_t)q * PFT_IPC_HANDLE_BYTES, sizeof(h));
    void* p = nullptr;
    cudaError_t e = cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) {
      for (int r = 0; r < q; ++r)
        if (r != vol->rank && vol->xbuf[r]) { cudaIpcCloseMemHandle(vol->xbuf[r]); vol->xbuf[r] = nullptr; }
      return fail(PFT_ERR_CUDA, "opening rank %d's exchange buffer: %s", q, cudaGetErrorString(e));
    }
    vol->xbuf[q] = (char*)p;
  }
  vol->p2p = 1;
  return PFT_OK;
}

pft_status pft_comm_p2p_preflight(pft_volume* vol, int32_t timeout_ms, int32_t* ok_out, void* stream) {
  if (!vol || !ok_out) return fail(PFT_ERR_INVALID_ARG, "NULL argument");
  if (!vol->p2p) return fail(PFT_ERR_STATE, "peers are not attached (pft_comm_p2p_attach)");
  if (timeout_ms < 1) return fail(PFT_ERR_INVALID_ARG, "timeout_ms must be >= 1");
  return pft::p2p_preflight(vol, timeout_ms, ok_out, (cudaStream_t)stream);
}

pft_status pft_comm_set_partition(pft_volume* vol, int32_t partition) {
  if (!vol) return fail(PFT_ERR_INVALID_ARG, "vol is NULL");
  if (partition != PFT_PARTITION_PARTICLES && partition != PFT_PARTITION_POINTS)
    return fail(PFT_ERR_INVALID_ARG, "bad partition %d", partition);
  if (partition == PFT_PARTITION_POINTS && (vol->p2p || vol->virtual_fused))
    return fail(PFT_ERR_UNSUPPORTED, "the point-sharded partition runs on the NCCL / virtual-shard path only");
  vol->partition = partition;
  return PFT_OK;
}

pft_status pft_comm_init(pft_volume* vol, const uint8_t id[128], int32_t nranks, int32_t rank) {
  if (!vol || !id) return fail(PFT_ERR_INVALID_ARG, "NULL argument");
  if (nranks < 1 || rank < 0 || rank >= nranks) return fail(PFT_ERR_INVALID_ARG, "bad rank %d of %d", rank, nranks);
  if (vol->nccl_comm) return fail(PFT_ERR_STATE, "communicator already initialised");
  if (vol->virtual_ranks || vol->virtual_fused) return fail(PFT_ERR_STATE, "virtual ranks are set (pft_comm_init_virtual*)");
  if (vol->p2p || vol->xown) return fail(PFT_ERR_STATE, "peer exchange buffers are attached (pft_comm_p2p_detach first)");
  // (nranks = 1 attaches a real single-rank communicator: pft_track then runs its collective path)
  Nccl* n = nccl();
  if (!n) return fail(PFT_ERR_NCCL, "libnccl.so.2 not loadable");
  ncclUniqueId uid;
  memcpy(uid.internal, id, 128);
  ncclComm_t comm;
  ncclResult_t r = n->commInitRank(&comm, nranks, uid, rank);
  if (r != ncclSuccess) return fail(PFT_ERR_NCCL, "ncclCommInitRank: %s", n->errStr(r));
  vol->nccl_comm = comm;
  vol->nranks = nranks;
  vol->rank = rank;
  return PFT_OK;
}

}  // extern "C"
