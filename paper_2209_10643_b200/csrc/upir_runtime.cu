// upir_runtime.cu -- host runtime behind include/upir.h.
//
// Context (streams, workspace, NCCL communicator), the upir.data present
// table (Figs. 5-6; reading c18), descriptor validation and
// normalisation of upir.spmd / upir.loop / loop_parallel (Figs. 1, 3), launch
// dispatch to the sm_100a kernels, upir.sync (Fig. 7) and CUDA-graph capture.
// No C++ exception crosses the ABI; every entry point returns upir_status.
#include <cuda.h>
#include <cuda_runtime.h>
#include <nccl.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "dev_tma.cuh"
#include "upir_internal.h"

using namespace upir;

// ------------------------------------------------------------------ errors
static thread_local std::string g_err;

static upir_status fail(upir_status s, const char *fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return s;
}

#define CUDA_TRY(expr)                                                                      \
  do {                                                                                      \
    cudaError_t _e = (expr);                                                                \
    if (_e != cudaSuccess)                                                                  \
      return fail(UPIR_E_CUDA, "%s failed: %s (%s:%d)", #expr, cudaGetErrorString(_e), __FILE__, __LINE__); \
  } while (0)

#define NCCL_TRY(expr)                                                                      \
  do {                                                                                      \
    ncclResult_t _r = (expr);                                                               \
    if (_r != ncclSuccess)                                                                  \
      return fail(UPIR_E_NCCL, "%s failed: %s", #expr, ncclGetErrorString(_r));             \
  } while (0)

extern "C" const char *upir_last_error(void) { return g_err.c_str(); }
extern "C" const char *upir_version(void) { return "upir-b200 0.1 (sm_100a)"; }

// ------------------------------------------------------------------ objects
struct upir_map_s {
  upir_ctx ctx;
  void *host;
  size_t bytes;          // global bytes of the host array (or adopted bytes)
  int kind;
  void *dev;             // local device buffer
  size_t dev_bytes;      // local bytes
  bool owned;            // dev allocated by us
  int refcount;
  // distribution
  upir_dist dist;
  int64_t row_lo, row_hi;        // owned rows
  int64_t loc_row_lo, loc_row_hi;  // rows held locally (halo included)
  int64_t elems_local;           // local elements (rows*row_elems)
  int64_t elem_offset;           // global element index of local element 0
  int64_t elem_bytes;
  void *pin_reg = nullptr; // registration this map took a user count on (or null)
  // peer mode (fused halo): exported from a cudaMalloc block; neighbours'
  // buffers mapped by CUDA IPC ([0] = rank - 1, [1] = rank + 1)
  bool ipc_alloc = false;
  void *peer_base[2] = {nullptr, nullptr};
  float *peer_dev[2] = {nullptr, nullptr};
  int64_t peer_row0[2] = {0, 0};
  bool halo_fused = false;  // last written by a peer-mode sweep: halos already exchanged
};

struct upir_event_s {
  cudaEvent_t ev;
};

struct upir_graph_s {
  cudaGraph_t graph;
  cudaGraphExec_t exec;
  int64_t kernels = 0;   // library kernels captured (counted per graph launch)
};

struct upir_spmd_s {
  upir_ctx ctx;
  upir_spmd_desc d;
};

struct upir_ctx_s {
  int device = 0;
  int rank = 0, nranks = 1;
  int num_sms = 148;
  cudaStream_t compute = nullptr, copy = nullptr;
  bool own_compute = false, own_copy = false;
  ncclComm_t comm = nullptr;
  // workspace
  unsigned long long *slots = nullptr;
  size_t slots_teams = 0;
  unsigned int *done = nullptr;
  unsigned long long *dyn = nullptr;
  void *scratch = nullptr;      // world-reduce gather buffer
  size_t scratch_bytes = 0;
  void *one = nullptr;          // 1-element buffer for the world barrier
  // guided-schedule boundary tables, one device table per (T, p, c, simd),
  // never overwritten: a captured graph keeps the pointer it was built with
  struct GTab { int64_t T, p, c, s, n; int64_t *dev; };
  std::vector<GTab> gtabs;
  // workspace a captured graph may still reference after it was outgrown:
  // released at upir_finalize, never while the context lives
  std::vector<void *> retired;
  // present table: host pointer -> map
  std::map<void *, upir_map> present;
  std::vector<upir_map> adopted;
  // host ranges this context pinned with cudaHostRegister: {ptr, bytes, live maps}
  struct Reg { void *ptr; size_t bytes; int users; };
  std::vector<Reg> registered;
  std::vector<upir_spmd> regions;
  cudaError_t sticky = cudaSuccess;
  bool capturing = false;
  // peer window (WinWord layout) and the other ranks' windows mapped by IPC
  unsigned long long *win = nullptr;
  unsigned long long *peer_win[WIN_MAX_RANKS] = {};
  void *peer_win_base[WIN_MAX_RANKS] = {};
  // statistics
  int64_t h2d_bytes = 0, d2h_bytes = 0, launches = 0;
  int64_t launches_at_capture = 0;
};

static upir_status sticky_check(upir_ctx c) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess && c->sticky == cudaSuccess) c->sticky = e;
  if (c->sticky != cudaSuccess)
    return fail(UPIR_E_CUDA, "asynchronous CUDA error: %s", cudaGetErrorString(c->sticky));
  return UPIR_OK;
}

static upir_status ensure_slots(upir_ctx c, size_t teams) {
  if (teams <= c->slots_teams) return UPIR_OK;
  if (c->capturing) return fail(UPIR_E_INVALID, "workspace must grow (teams=%zu) but a graph is being captured", teams);
  if (c->slots) c->retired.push_back(c->slots);   // graphs may hold it
  size_t n = std::max(teams, (size_t)1 << 16);
  CUDA_TRY(cudaMalloc(&c->slots, n * 2 * sizeof(unsigned long long)));
  c->slots_teams = n;
  return UPIR_OK;
}

// ------------------------------------------------------------------ lifecycle
extern "C" upir_status upir_init(int cuda_device, const upir_world *world, upir_ctx *out) {
  if (!out) return fail(UPIR_E_INVALID, "out is NULL");
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess || ndev == 0)
    return fail(UPIR_E_CUDA, "no CUDA device available (%s); this runtime has no CPU fallback",
                cudaGetErrorString(e));
  if (cuda_device < 0 || cuda_device >= ndev) return fail(UPIR_E_INVALID, "device %d out of range", cuda_device);
  cudaDeviceProp prop;
  CUDA_TRY(cudaGetDeviceProperties(&prop, cuda_device));
  if (prop.major != 10)
    return fail(UPIR_E_UNSUPPORTED, "device %d is sm_%d%d; this build targets sm_100a only", cuda_device,
                prop.major, prop.minor);
  if (world && (world->nranks < 1 || world->rank < 0 || world->rank >= world->nranks))
    return fail(UPIR_E_INVALID, "bad world rank %d / nranks %d", world->rank, world->nranks);
  CUDA_TRY(cudaSetDevice(cuda_device));
  upir_ctx c = new upir_ctx_s();
  c->device = cuda_device;
  c->num_sms = prop.multiProcessorCount;
  if (world) {
    c->rank = world->rank;
    c->nranks = world->nranks;
    c->compute = (cudaStream_t)world->compute_stream;
    c->copy = (cudaStream_t)world->copy_stream;
  }
  auto cleanup = [&](upir_status s) {   // release whatever was created before the failure
    if (c->slots) cudaFree(c->slots);
    if (c->done) cudaFree(c->done);
    if (c->one) cudaFree(c->one);
    if (c->win) cudaFree(c->win);
    if (c->own_compute && c->compute) cudaStreamDestroy(c->compute);
    if (c->own_copy && c->copy) cudaStreamDestroy(c->copy);
    delete c;
    return s;
  };
  if (!c->compute) {
    if (cudaStreamCreateWithFlags(&c->compute, cudaStreamNonBlocking) != cudaSuccess)
      return cleanup(fail(UPIR_E_CUDA, "stream create failed"));
    c->own_compute = true;
  }
  if (!c->copy) {
    if (cudaStreamCreateWithFlags(&c->copy, cudaStreamNonBlocking) != cudaSuccess)
      return cleanup(fail(UPIR_E_CUDA, "stream create failed"));
    c->own_copy = true;
  }
  // stream-ordered allocations of map(to/from/alloc) stay cached in the
  // device's default pool across map exit / enter (no re-mapping per map)
  {
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, cuda_device) == cudaSuccess) {
      uint64_t thr = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    cudaGetLastError();
  }
  if (cudaMalloc(&c->done, 256) != cudaSuccess || cudaMemset(c->done, 0, 256) != cudaSuccess)
    return cleanup(fail(UPIR_E_OOM, "workspace allocation failed"));
  c->dyn = reinterpret_cast<unsigned long long *>(reinterpret_cast<char *>(c->done) + 64);
  if (cudaMalloc(&c->one, 64) != cudaSuccess) return cleanup(fail(UPIR_E_OOM, "workspace allocation failed"));
  if (ensure_slots(c, (size_t)1 << 16) != UPIR_OK) return cleanup(UPIR_E_OOM);
  // peer window: plain cudaMalloc block (CUDA-IPC exportable), zeroed; its own
  // entry of the peer table points at itself
  if (cudaMalloc(&c->win, WIN_BYTES) != cudaSuccess || cudaMemset(c->win, 0, WIN_BYTES) != cudaSuccess)
    return cleanup(fail(UPIR_E_OOM, "peer window allocation failed"));
  if (c->rank < WIN_MAX_RANKS) {
    c->peer_win[c->rank] = c->win;
    unsigned long long self = (unsigned long long)(uintptr_t)c->win;
    if (cudaMemcpy(c->win + WIN_PEERS + c->rank, &self, 8, cudaMemcpyHostToDevice) != cudaSuccess)
      return cleanup(fail(UPIR_E_CUDA, "peer window init failed"));
  }
  // nccl_id NULL with nranks > 1: a communicator-less world -- only the peer
  // window paths (fused world reduction / halo, peer barrier) exchange data
  if (c->nranks > 1 && world->nccl_id) {
    ncclUniqueId id;
    memcpy(&id, world->nccl_id, sizeof id);
    ncclResult_t r = ncclCommInitRank(&c->comm, c->nranks, id, c->rank);
    if (r != ncclSuccess) return cleanup(fail(UPIR_E_NCCL, "ncclCommInitRank: %s", ncclGetErrorString(r)));
  }
  *out = c;
  return UPIR_OK;
}

extern "C" upir_status upir_comm_unique_id(void *out128) {
  if (!out128) return fail(UPIR_E_INVALID, "out is NULL");
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
  ncclUniqueId id;
  NCCL_TRY(ncclGetUniqueId(&id));
  memcpy(out128, &id, sizeof id);
  return UPIR_OK;
}

extern "C" upir_status upir_ctx_stream(upir_ctx c, int which, uintptr_t *out) {
  if (!c || !out || (which != 0 && which != 1)) return fail(UPIR_E_INVALID, "bad argument");
  *out = (uintptr_t)(which == 0 ? c->compute : c->copy);
  return UPIR_OK;
}

extern "C" upir_status upir_ctx_stats(upir_ctx c, int64_t out[4]) {
  if (!c || !out) return fail(UPIR_E_INVALID, "bad argument");
  out[0] = c->h2d_bytes;
  out[1] = c->d2h_bytes;
  out[2] = (int64_t)(c->present.size() + c->adopted.size());
  out[3] = c->launches;
  return UPIR_OK;
}

extern "C" upir_status upir_finalize(upir_ctx c) {
  if (!c) return fail(UPIR_E_INVALID, "ctx is NULL");
  cudaSetDevice(c->device);
  cudaStreamSynchronize(c->compute);
  cudaStreamSynchronize(c->copy);
  if (!c->present.empty() || !c->adopted.empty())
    return fail(UPIR_E_LEAK, "finalize with %zu live maps", c->present.size() + c->adopted.size());
  upir_status st = sticky_check(c);
  for (auto &r : c->registered) cudaHostUnregister(r.ptr);
  for (auto s : c->regions) delete s;
  for (int q = 0; q < WIN_MAX_RANKS; ++q)
    if (c->peer_win_base[q]) cudaIpcCloseMemHandle(c->peer_win_base[q]);
  cudaFree(c->win);
  if (c->comm) ncclCommDestroy(c->comm);
  cudaFree(c->slots);
  cudaFree(c->done);
  cudaFree(c->one);
  if (c->scratch) cudaFree(c->scratch);
  for (auto &g : c->gtabs) cudaFree(g.dev);
  for (void *p : c->retired) cudaFree(p);
  if (c->own_compute) cudaStreamDestroy(c->compute);
  if (c->own_copy) cudaStreamDestroy(c->copy);
  delete c;
  return st;
}

// ------------------------------------------------------------------ distribution
extern "C" upir_status upir_dist_owned_rows(int64_t n_rows, int32_t rank, int32_t nranks, int64_t *lo,
                                            int64_t *hi) {
  if (!lo || !hi || nranks < 1 || rank < 0 || rank >= nranks || n_rows < 0)
    return fail(UPIR_E_INVALID, "bad distribution arguments");
  // reading c20: the static block rule over ranks
  const int64_t q = n_rows / nranks, r = n_rows % nranks;
  *lo = rank * q + std::min<int64_t>(rank, r);
  *hi = *lo + q + (rank < r ? 1 : 0);
  return UPIR_OK;
}

extern "C" upir_status upir_halo_plan(int64_t n_rows, int32_t halo, int32_t rank, int32_t nranks, int64_t out[8]) {
  if (!out || halo < 0) return fail(UPIR_E_INVALID, "bad halo plan arguments");
  int64_t lo, hi;
  upir_status st = upir_dist_owned_rows(n_rows, rank, nranks, &lo, &hi);
  if (st != UPIR_OK) return st;
  for (int i = 0; i < 8; ++i) out[i] = 0;
  if (rank > 0) {
    int64_t ulo, uhi;
    upir_dist_owned_rows(n_rows, rank - 1, nranks, &ulo, &uhi);
    const int64_t s = std::min<int64_t>(halo, std::min(hi - lo, uhi - ulo));
    if (s > 0) {
      out[0] = lo; out[1] = lo + s;        // my first owned rows -> up's bottom halo
      out[2] = lo - s; out[3] = lo;        // up's last owned rows -> my top halo
    }
  }
  if (rank < nranks - 1) {
    int64_t dlo, dhi;
    upir_dist_owned_rows(n_rows, rank + 1, nranks, &dlo, &dhi);
    const int64_t s = std::min<int64_t>(halo, std::min(hi - lo, dhi - dlo));
    if (s > 0) {
      out[4] = hi - s; out[5] = hi;        // my last owned rows -> down's top halo
      out[6] = hi; out[7] = hi + s;        // down's first owned rows -> my bottom halo
    }
  }
  return UPIR_OK;
}

static upir_status layout_map(upir_ctx c, upir_map m, size_t bytes, const upir_dist *dist) {
  if (dist && dist->pattern == UPIR_PATTERN_BLOCK) {
    if (dist->n_rows < 1 || dist->row_elems < 1 || dist->elem_bytes < 1 || dist->halo_rows < 0)
      return fail(UPIR_E_INVALID, "bad upir_dist");
    if ((size_t)(dist->n_rows * dist->row_elems * dist->elem_bytes) != bytes)
      return fail(UPIR_E_INVALID, "upir_dist extent (%lld rows x %lld x %lld B) != bytes %zu",
                  (long long)dist->n_rows, (long long)dist->row_elems, (long long)dist->elem_bytes, bytes);
    m->dist = *dist;
    upir_dist_owned_rows(dist->n_rows, c->rank, c->nranks, &m->row_lo, &m->row_hi);
    m->loc_row_lo = std::max<int64_t>(0, m->row_lo - dist->halo_rows);
    m->loc_row_hi = std::min<int64_t>(dist->n_rows, m->row_hi + dist->halo_rows);
    m->elem_bytes = dist->elem_bytes;
    m->elems_local = (m->loc_row_hi - m->loc_row_lo) * dist->row_elems;
    m->elem_offset = m->loc_row_lo * dist->row_elems;
    m->dev_bytes = (size_t)(m->elems_local * dist->elem_bytes);
  } else {
    if (dist && dist->pattern != UPIR_PATTERN_NONE) return fail(UPIR_E_INVALID, "unknown pattern");
    memset(&m->dist, 0, sizeof m->dist);
    m->elem_bytes = 1;
    m->row_lo = m->loc_row_lo = 0;
    m->row_hi = m->loc_row_hi = (int64_t)bytes;
    m->elems_local = (int64_t)bytes;
    m->elem_offset = 0;
    m->dev_bytes = bytes;
  }
  return UPIR_OK;
}

// bytes of host / device ranges moved by a map: local rows (halo included) on
// enter; owned rows on exit.
static void map_range(upir_map m, bool owned_only, size_t &host_off, size_t &dev_off, size_t &len) {
  if (m->dist.pattern == UPIR_PATTERN_BLOCK) {
    const int64_t rb = m->dist.row_elems * m->dist.elem_bytes;
    const int64_t r0 = owned_only ? m->row_lo : m->loc_row_lo;
    const int64_t r1 = owned_only ? m->row_hi : m->loc_row_hi;
    host_off = (size_t)(r0 * rb);
    dev_off = (size_t)((r0 - m->loc_row_lo) * rb);
    len = (size_t)((r1 - r0) * rb);
  } else {
    host_off = dev_off = 0;
    len = m->bytes;
  }
}

// Pin a caller host range for async DMA.  Memory the caller already pinned
// (cudaHostAlloc / torch pin_memory) is used as is.  Ranges we register are
// released at the first upir_sync (or finalize) after their last map is gone
// -- the contract keeps host buffers valid until that sync.
// Returns the registration it took a user count on, or null when it took none
// (small buffer, memory pinned by someone else, failed registration).
static void *pin_host(upir_ctx c, void *host, size_t bytes) {
  // small buffers are copied from pageable memory (the driver stages them);
  // registering / unregistering a page per map costs more than the copy
  if (bytes < ((size_t)1 << 20)) return nullptr;
  for (auto &r : c->registered)
    if ((char *)host >= (char *)r.ptr && (char *)host + bytes <= (char *)r.ptr + r.bytes) {
      r.users++;
      return r.ptr;
    }
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, host) == cudaSuccess &&
      (at.type == cudaMemoryTypeHost || at.type == cudaMemoryTypeManaged))
    return nullptr;
  cudaGetLastError();
  cudaError_t e = cudaHostRegister(host, bytes, cudaHostRegisterDefault);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return nullptr;   // pageable copies still work (staged by the driver)
  }
  c->registered.push_back({host, bytes, 1});
  return host;
}

// drop the user count a map took on registration `reg`
static void unpin_host(upir_ctx c, void *reg) {
  for (auto &r : c->registered)
    if (r.ptr == reg) {
      r.users--;
      return;
    }
}

// after all copies completed: drop registrations without live maps
static void release_pins(upir_ctx c) {
  for (size_t i = 0; i < c->registered.size();) {
    if (c->registered[i].users <= 0) {
      cudaHostUnregister(c->registered[i].ptr);
      cudaGetLastError();
      c->registered.erase(c->registered.begin() + i);
    } else {
      ++i;
    }
  }
}

// compute stream waits for everything enqueued on the copy stream so far
static upir_status copy_to_compute(upir_ctx c) {
  cudaEvent_t ev;
  CUDA_TRY(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  CUDA_TRY(cudaEventRecord(ev, c->copy));
  CUDA_TRY(cudaStreamWaitEvent(c->compute, ev, 0));
  CUDA_TRY(cudaEventDestroy(ev));
  return UPIR_OK;
}
static upir_status peer_release(upir_ctx c, upir_map m);

static upir_status compute_to_copy(upir_ctx c) {
  cudaEvent_t ev;
  CUDA_TRY(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  CUDA_TRY(cudaEventRecord(ev, c->compute));
  CUDA_TRY(cudaStreamWaitEvent(c->copy, ev, 0));
  CUDA_TRY(cudaEventDestroy(ev));
  return UPIR_OK;
}

extern "C" upir_status upir_data_map(upir_ctx c, void *host, size_t bytes, upir_map_kind kind,
                                     const upir_dist *dist, upir_map *out) {
  if (!c || !host || !out) return fail(UPIR_E_INVALID, "NULL argument");
  if (kind < UPIR_MAP_TO || kind > UPIR_MAP_ALLOC) return fail(UPIR_E_INVALID, "bad map kind %d", (int)kind);
  if (bytes == 0) return fail(UPIR_E_INVALID, "zero-byte map");
  auto it = c->present.find(host);
  if (it != c->present.end()) {   // present: refcount only (reading c18)
    if (it->second->bytes != bytes) return fail(UPIR_E_INVALID, "host pointer already mapped with %zu bytes", it->second->bytes);
    it->second->refcount++;
    *out = it->second;
    return UPIR_OK;
  }
  upir_map m = new upir_map_s();
  m->ctx = c;
  m->host = host;
  m->bytes = bytes;
  m->kind = kind;
  m->owned = true;
  m->refcount = 1;
  upir_status st = layout_map(c, m, bytes, dist);
  if (st != UPIR_OK) { delete m; return st; }
  cudaSetDevice(c->device);
  // mm_allocator (Fig. 6): stream-ordered allocation, rounded to 256 B so
  // vector paths may read the last partial vector's bytes safely.
  size_t alloc = (m->dev_bytes + 255) & ~(size_t)255;
  cudaError_t e = cudaMallocAsync(&m->dev, alloc, c->copy);
  if (e != cudaSuccess) {
    cudaGetLastError();
    delete m;
    return fail(UPIR_E_OOM, "device allocation of %zu bytes failed: %s", alloc, cudaGetErrorString(e));
  }
  if (kind != UPIR_MAP_ALLOC) m->pin_reg = pin_host(c, host, bytes);
  if (kind == UPIR_MAP_TO || kind == UPIR_MAP_TOFROM) {   // data_movement forward
    size_t ho, dof, len;
    map_range(m, false, ho, dof, len);
    e = cudaMemcpyAsync((char *)m->dev + dof, (char *)host + ho, len, cudaMemcpyHostToDevice, c->copy);
    if (e != cudaSuccess) {
      if (m->pin_reg) unpin_host(c, m->pin_reg);
      cudaFreeAsync(m->dev, c->copy);
      delete m;
      return fail(UPIR_E_CUDA, "H2D copy failed: %s", cudaGetErrorString(e));
    }
    c->h2d_bytes += (int64_t)len;
  }
  st = copy_to_compute(c);
  if (st != UPIR_OK) {
    if (m->pin_reg) unpin_host(c, m->pin_reg);
    cudaFreeAsync(m->dev, c->copy);
    delete m;
    return st;
  }
  c->present[host] = m;
  *out = m;
  return UPIR_OK;
}

extern "C" upir_status upir_data_adopt(upir_ctx c, void *dev_ptr, size_t bytes, const upir_dist *dist,
                                       upir_map *out) {
  if (!c || !dev_ptr || !out || bytes == 0) return fail(UPIR_E_INVALID, "bad argument");
  upir_map m = new upir_map_s();
  m->ctx = c;
  m->host = nullptr;
  m->bytes = bytes;
  m->kind = 0;
  m->owned = false;
  m->refcount = 1;
  m->dev = dev_ptr;
  // an adopted buffer holds this rank's local rows of a distributed array
  upir_status st = layout_map(c, m, dist ? (size_t)(dist->n_rows * dist->row_elems * dist->elem_bytes) : bytes, dist);
  if (st != UPIR_OK) { delete m; return st; }
  if (dist && dist->pattern == UPIR_PATTERN_BLOCK && (size_t)m->dev_bytes > bytes) {
    delete m;
    return fail(UPIR_E_INVALID, "adopted buffer (%zu B) smaller than the local block (%zu B)", bytes, m->dev_bytes);
  }
  if (!dist || dist->pattern != UPIR_PATTERN_BLOCK) m->dev_bytes = bytes;
  c->adopted.push_back(m);
  *out = m;
  return UPIR_OK;
}

extern "C" upir_status upir_data_unmap(upir_ctx c, upir_map m) {
  if (!c || !m || m->ctx != c) return fail(UPIR_E_INVALID, "bad map");
  if (!m->owned) {
    auto it = std::find(c->adopted.begin(), c->adopted.end(), m);
    if (it == c->adopted.end()) return fail(UPIR_E_INVALID, "map not live");
    upir_status pst = peer_release(c, m);
    if (pst != UPIR_OK) return pst;
    c->adopted.erase(it);
    delete m;
    return sticky_check(c);
  }
  auto it = c->present.find(m->host);
  if (it == c->present.end() || it->second != m) return fail(UPIR_E_INVALID, "map not live");
  if (--m->refcount > 0) return UPIR_OK;
  upir_status st = peer_release(c, m);
  if (st != UPIR_OK) return st;
  st = compute_to_copy(c);
  if (st != UPIR_OK) return st;
  if (m->kind == UPIR_MAP_FROM || m->kind == UPIR_MAP_TOFROM) {   // data_movement backward
    size_t ho, dof, len;
    map_range(m, true, ho, dof, len);
    CUDA_TRY(cudaMemcpyAsync((char *)m->host + ho, (char *)m->dev + dof, len, cudaMemcpyDeviceToHost, c->copy));
    c->d2h_bytes += (int64_t)len;
  }
  if (m->ipc_alloc) {   // exported block: plain free once the copy is done
    CUDA_TRY(cudaStreamSynchronize(c->copy));
    CUDA_TRY(cudaFree(m->dev));
  } else {
    CUDA_TRY(cudaFreeAsync(m->dev, c->copy));   // mm_deallocator
  }
  if (m->pin_reg) unpin_host(c, m->pin_reg);
  c->present.erase(it);
  delete m;
  return sticky_check(c);
}

extern "C" upir_status upir_data_update(upir_ctx c, upir_map m, int direction) {
  if (!c || !m || m->ctx != c || !m->owned || !m->host) return fail(UPIR_E_INVALID, "bad map");
  if (direction < 0 || direction > UPIR_UPDATE_FORWARD_ASYNC)
    return fail(UPIR_E_INVALID, "direction must be 0 (forward), 1 (backward) or 2 (forward async)");
  upir_status st = compute_to_copy(c);
  if (st != UPIR_OK) return st;
  size_t ho, dof, len;
  if (direction == 0) {
    map_range(m, false, ho, dof, len);
    CUDA_TRY(cudaMemcpyAsync((char *)m->dev + dof, (char *)m->host + ho, len, cudaMemcpyHostToDevice, c->copy));
    c->h2d_bytes += (int64_t)len;
  } else {
    map_range(m, true, ho, dof, len);
    CUDA_TRY(cudaMemcpyAsync((char *)m->host + ho, (char *)m->dev + dof, len, cudaMemcpyDeviceToHost, c->copy));
    c->d2h_bytes += (int64_t)len;
  }
  return copy_to_compute(c);
}

extern "C" upir_status upir_data_update_section(upir_ctx c, upir_map m, int64_t off, int64_t bytes, int direction) {
  if (!c || !m || m->ctx != c || !m->owned || !m->host) return fail(UPIR_E_INVALID, "bad map");
  if (direction < 0 || direction > UPIR_UPDATE_FORWARD_ASYNC)
    return fail(UPIR_E_INVALID, "direction must be 0 (forward), 1 (backward) or 2 (forward async)");
  if (off < 0 || bytes < 0 || off + bytes > (int64_t)m->dev_bytes)
    return fail(UPIR_E_INVALID, "section [%lld, +%lld) outside the local buffer (%zu B)", (long long)off,
                (long long)bytes, m->dev_bytes);
  if (bytes == 0) return UPIR_OK;
  // host offset of local byte 0: the first local row of a BLOCK map
  size_t ho, dof, len;
  map_range(m, false, ho, dof, len);
  char *h = (char *)m->host + ho - dof + off;
  if (direction != UPIR_UPDATE_FORWARD_ASYNC) {   // ordered after the compute work so far
    upir_status st = compute_to_copy(c);
    if (st != UPIR_OK) return st;
  }
  if (direction != 1) {
    CUDA_TRY(cudaMemcpyAsync((char *)m->dev + off, h, (size_t)bytes, cudaMemcpyHostToDevice, c->copy));
    c->h2d_bytes += bytes;
  } else {
    CUDA_TRY(cudaMemcpyAsync(h, (char *)m->dev + off, (size_t)bytes, cudaMemcpyDeviceToHost, c->copy));
    c->d2h_bytes += bytes;
  }
  return copy_to_compute(c);
}

extern "C" upir_status upir_data_device_ptr(upir_map m, void **dptr, int64_t *local_elems, int64_t *global_offset) {
  if (!m) return fail(UPIR_E_INVALID, "map is NULL");
  if (dptr) *dptr = m->dev;
  if (local_elems) *local_elems = m->elems_local;
  if (global_offset) *global_offset = m->elem_offset;
  return UPIR_OK;
}

// ------------------------------------------------------------------ peer windows (CUDA IPC)
static upir_status check_map(upir_ctx c, upir_map m, const char *what);
// A record carries one CUDA-IPC handle plus the layout facts the importer
// checks; the caller moves records between ranks (e.g. torch.distributed).
namespace {
struct PeerRec {
  uint32_t magic;            // PEER_MAGIC
  uint32_t kind;             // 0 = context window, 1 = map buffer
  int32_t rank, nranks;
  cudaIpcMemHandle_t handle;
  int64_t offset;            // byte offset of the buffer inside the exported allocation
  int64_t loc_row_lo, row_elems, elem_bytes, n_rows;
  int32_t halo_rows, pad;
};
static_assert(sizeof(PeerRec) <= UPIR_PEER_REC_BYTES, "peer record size");
constexpr uint32_t PEER_MAGIC = 0x52495055u;   // "UPIR"
}  // namespace

// Allocation base of a device pointer (driver cuMemGetAddressRange).
static bool alloc_base(void *p, void **base) {
  typedef CUresult (*Fn)(CUdeviceptr *, size_t *, CUdeviceptr);
  static Fn fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void *f = nullptr;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !f)
      return false;
    fn = reinterpret_cast<Fn>(f);
  }
  CUdeviceptr b = 0;
  size_t sz = 0;
  if (fn(&b, &sz, (CUdeviceptr)(uintptr_t)p) != CUDA_SUCCESS) return false;
  *base = (void *)(uintptr_t)b;
  return true;
}

static bool world_ready(upir_ctx c) {
  if (c->nranks > WIN_MAX_RANKS) return false;
  for (int q = 0; q < c->nranks; ++q)
    if (!c->peer_win[q]) return false;
  return true;
}

extern "C" upir_status upir_peer_export(upir_ctx c, upir_map m, void *rec) {
  if (!c || !rec) return fail(UPIR_E_INVALID, "NULL argument");
  cudaSetDevice(c->device);
  PeerRec r;
  memset(&r, 0, sizeof r);
  r.magic = PEER_MAGIC;
  r.rank = c->rank;
  r.nranks = c->nranks;
  if (!m) {
    r.kind = 0;
    CUDA_TRY(cudaIpcGetMemHandle(&r.handle, c->win));
  } else {
    upir_status st = check_map(c, m, "map");
    if (st != UPIR_OK) return st;
    if (m->dist.pattern != UPIR_PATTERN_BLOCK)
      return fail(UPIR_E_INVALID, "peer export needs a BLOCK-distributed map (its halo rows are the peers' targets)");
    if (c->capturing) return fail(UPIR_E_INVALID, "peer export during graph capture");
    if (m->owned && !m->ipc_alloc) {
      // stream-ordered pool blocks are not IPC-exportable: move the buffer to
      // a plain cudaMalloc block (device pointers taken earlier go stale)
      CUDA_TRY(cudaStreamSynchronize(c->compute));
      CUDA_TRY(cudaStreamSynchronize(c->copy));
      void *nb = nullptr;
      const size_t alloc = std::max<size_t>(256, (m->dev_bytes + 255) / 256 * 256);
      if (cudaMalloc(&nb, alloc) != cudaSuccess) {
        cudaGetLastError();
        return fail(UPIR_E_OOM, "peer buffer of %zu bytes", alloc);
      }
      CUDA_TRY(cudaMemcpy(nb, m->dev, m->dev_bytes, cudaMemcpyDeviceToDevice));
      CUDA_TRY(cudaFreeAsync(m->dev, c->copy));
      CUDA_TRY(cudaStreamSynchronize(c->copy));
      m->dev = nb;
      m->ipc_alloc = true;
    }
    void *base = m->dev;
    if (!m->owned && !alloc_base(m->dev, &base)) return fail(UPIR_E_CUDA, "cannot resolve the allocation of an adopted buffer");
    CUDA_TRY(cudaIpcGetMemHandle(&r.handle, base));
    r.kind = 1;
    r.offset = (int64_t)((char *)m->dev - (char *)base);
    r.loc_row_lo = m->loc_row_lo;
    r.row_elems = m->dist.row_elems;
    r.elem_bytes = m->dist.elem_bytes;
    r.n_rows = m->dist.n_rows;
    r.halo_rows = m->dist.halo_rows;
  }
  memset(rec, 0, UPIR_PEER_REC_BYTES);
  memcpy(rec, &r, sizeof r);
  return UPIR_OK;
}

extern "C" upir_status upir_peer_import(upir_ctx c, upir_map m, int32_t peer, const void *rec) {
  if (!c || !rec) return fail(UPIR_E_INVALID, "NULL argument");
  PeerRec r;
  memcpy(&r, rec, sizeof r);
  if (r.magic != PEER_MAGIC) return fail(UPIR_E_INVALID, "not a peer record");
  if (peer < 0 || peer >= c->nranks || r.rank != peer || r.nranks != c->nranks)
    return fail(UPIR_E_INVALID, "peer record of rank %d/%d imported as rank %d/%d", r.rank, r.nranks, peer, c->nranks);
  cudaSetDevice(c->device);
  if (!m) {
    if (r.kind != 0) return fail(UPIR_E_INVALID, "record is not a context window");
    if (peer >= WIN_MAX_RANKS) return fail(UPIR_E_UNSUPPORTED, "peer windows support at most %d ranks", WIN_MAX_RANKS);
    if (peer == c->rank || c->peer_win[peer]) return UPIR_OK;
    void *p = nullptr;
    CUDA_TRY(cudaIpcOpenMemHandle(&p, r.handle, cudaIpcMemLazyEnablePeerAccess));
    c->peer_win_base[peer] = p;
    c->peer_win[peer] = reinterpret_cast<unsigned long long *>((char *)p + r.offset);
    const unsigned long long v = (unsigned long long)(uintptr_t)c->peer_win[peer];
    CUDA_TRY(cudaMemcpy(c->win + WIN_PEERS + peer, &v, 8, cudaMemcpyHostToDevice));
    return UPIR_OK;
  }
  upir_status st = check_map(c, m, "map");
  if (st != UPIR_OK) return st;
  if (r.kind != 1) return fail(UPIR_E_INVALID, "record is not a map buffer");
  if (m->dist.pattern != UPIR_PATTERN_BLOCK || r.n_rows != m->dist.n_rows || r.row_elems != m->dist.row_elems ||
      r.elem_bytes != m->dist.elem_bytes)
    return fail(UPIR_E_INVALID, "peer map layout differs from this map's");
  const int side = peer == c->rank - 1 ? 0 : (peer == c->rank + 1 ? 1 : -1);
  if (side < 0) return fail(UPIR_E_INVALID, "map buffers are imported from the halo neighbours (rank +- 1) only");
  if (m->peer_base[side]) {
    CUDA_TRY(cudaStreamSynchronize(c->compute));
    cudaIpcCloseMemHandle(m->peer_base[side]);
    m->peer_base[side] = nullptr;
    m->peer_dev[side] = nullptr;
  }
  void *p = nullptr;
  CUDA_TRY(cudaIpcOpenMemHandle(&p, r.handle, cudaIpcMemLazyEnablePeerAccess));
  m->peer_base[side] = p;
  m->peer_dev[side] = reinterpret_cast<float *>((char *)p + r.offset);
  m->peer_row0[side] = r.loc_row_lo;
  return UPIR_OK;
}

// Before a peer-attached buffer is read back or released: the neighbours'
// last sweeps (which store into its halo rows) must have been delivered, and
// this rank's kernels must be done with the neighbours' buffers.
static upir_status peer_release(upir_ctx c, upir_map m) {
  if (!m->peer_base[0] && !m->peer_base[1] && !m->ipc_alloc) return UPIR_OK;
  const bool up = c->rank > 0 && c->peer_win[c->rank - 1];
  const bool dn = c->rank + 1 < c->nranks && c->rank + 1 < WIN_MAX_RANKS && c->peer_win[c->rank + 1];
  if (up || dn) {
    cudaError_t e = launch_peer_drain(c->win, up, dn, c->compute);
    if (e != cudaSuccess) return fail(UPIR_E_CUDA, "peer drain launch failed: %s", cudaGetErrorString(e));
  }
  CUDA_TRY(cudaStreamSynchronize(c->compute));
  for (int side = 0; side < 2; ++side)
    if (m->peer_base[side]) {
      cudaIpcCloseMemHandle(m->peer_base[side]);
      m->peer_base[side] = nullptr;
      m->peer_dev[side] = nullptr;
    }
  return UPIR_OK;
}

// ------------------------------------------------------------------ spmd
static upir_status validate_spmd(const upir_spmd_desc *d) {
  if (!d) return fail(UPIR_E_INVALID, "spmd descriptor is NULL");
  // lesson of PAPER.md:1578-1587: honour the requested geometry or reject it
  if (d->num_units < 1 || d->num_units > 1024)
    return fail(UPIR_E_INVALID, "num_units=%d outside [1,1024] (geometry is never clamped)", d->num_units);
  if (d->num_teams < 1) return fail(UPIR_E_INVALID, "num_teams=%d < 1", d->num_teams);
  if (d->target != UPIR_TARGET_GPU && d->target != UPIR_TARGET_CLUSTER)
    return fail(UPIR_E_INVALID, "target must be GPU or CLUSTER");
  return UPIR_OK;
}

extern "C" upir_status upir_spmd_launch(upir_ctx c, const upir_spmd_desc *d, upir_spmd *out) {
  if (!c || !out) return fail(UPIR_E_INVALID, "NULL argument");
  upir_status st = validate_spmd(d);
  if (st != UPIR_OK) return st;
  upir_spmd s = new upir_spmd_s();
  s->ctx = c;
  s->d = *d;
  c->regions.push_back(s);
  *out = s;
  return UPIR_OK;
}

extern "C" upir_status upir_spmd_end(upir_spmd s) {
  if (!s) return fail(UPIR_E_INVALID, "NULL region");
  upir_ctx c = s->ctx;
  auto it = std::find(c->regions.begin(), c->regions.end(), s);
  if (it == c->regions.end()) return fail(UPIR_E_INVALID, "region not open");
  c->regions.erase(it);
  delete s;
  return UPIR_OK;
}

// ------------------------------------------------------------------ loop normalisation
static int64_t trip(int64_t lb, int64_t ub, int64_t step) {
  if (step > 0) return ub <= lb ? 0 : (ub - lb + step - 1) / step;
  return lb <= ub ? 0 : (lb - ub + (-step) - 1) / (-step);
}

extern "C" upir_status upir_loop_normalize(const upir_loop_desc *l, int64_t *T_total, int64_t T_d[3]) {
  if (!l || !T_total) return fail(UPIR_E_INVALID, "NULL argument");
  if (l->collapse < 1 || l->collapse > 2) return fail(UPIR_E_INVALID, "collapse=%d outside [1,2]", l->collapse);
  int64_t T = 1, Td[3] = {1, 1, 1};
  for (int d = 0; d < l->collapse; ++d) {
    if (l->step[d] == 0) return fail(UPIR_E_INVALID, "step[%d] == 0", d);
    Td[d] = trip(l->lb[d], l->ub[d], l->step[d]);
    if (Td[d] > 0 && T > INT64_MAX / Td[d]) return fail(UPIR_E_INVALID, "iteration space overflows int64");
    T *= Td[d];
  }
  *T_total = T;
  if (T_d) for (int d = 0; d < 3; ++d) T_d[d] = Td[d];
  return UPIR_OK;
}

// Resolve (policy, chunk) -> (SchedKind, chunk) (readings c3, c8).
static upir_status resolve_sched(int policy, int64_t chunk, int &sk, int64_t &c) {
  if (chunk < 0) return fail(UPIR_E_INVALID, "chunk < 0");
  switch (policy) {
    case UPIR_SCHED_RUNTIME:
    case UPIR_SCHED_AUTO:
      sk = SK_STATIC_BLOCK;
      c = 0;
      return UPIR_OK;
    case UPIR_SCHED_STATIC:
      sk = chunk > 0 ? SK_STATIC_CHUNK : SK_STATIC_BLOCK;
      c = chunk;
      return UPIR_OK;
    case UPIR_SCHED_DYNAMIC:
      sk = SK_DYNAMIC;
      c = chunk > 0 ? chunk : 1;
      return UPIR_OK;
    case UPIR_SCHED_GUIDED:
      sk = SK_GUIDED;
      c = chunk > 0 ? chunk : 1;
      return UPIR_OK;
  }
  return fail(UPIR_E_INVALID, "unknown schedule policy %d", policy);
}

extern "C" upir_status upir_schedule_chunks(int32_t policy, int64_t chunk, int64_t T, int64_t p, int64_t u,
                                            int64_t *lo, int64_t *hi, int64_t cap, int64_t *count) {
  if (!count || p < 1 || u < 0 || u >= p || T < 0 || cap < 0 || (cap > 0 && (!lo || !hi)))
    return fail(UPIR_E_INVALID, "bad argument");
  int sk;
  int64_t c;
  upir_status st = resolve_sched(policy, chunk, sk, c);
  if (st != UPIR_OK) return st;
  if (sk == SK_DYNAMIC || sk == SK_GUIDED)
    return fail(UPIR_E_INVALID, "dynamic / guided assignment is decided at run time");
  int64_t n = 0;
  if (sk == SK_STATIC_BLOCK) {
    const int64_t q = T / p, r = T % p;
    const int64_t len = q + (u < r ? 1 : 0);
    if (len > 0) {
      if (cap > 0) { lo[0] = u * q + std::min(u, r); hi[0] = lo[0] + len; }
      n = 1;
    }
  } else {
    const int64_t nc = (T + c - 1) / c;
    for (int64_t k = u; k < nc; k += p, ++n)
      if (n < cap) { lo[n] = k * c; hi[n] = std::min((k + 1) * c, T); }
  }
  *count = n;
  return UPIR_OK;
}

static int body_dtype_ok(int kind, int dtype) {
  switch (kind) {
    case UPIR_BODY_AXPY: return dtype == UPIR_F32;
    case UPIR_BODY_REDUCE: return dtype == UPIR_I64 || dtype == UPIR_F32;
    case UPIR_BODY_JACOBI5: return dtype == UPIR_F32;
    case UPIR_BODY_MATMUL: return dtype == UPIR_BF16 || dtype == UPIR_F32;
    case UPIR_BODY_MATVEC: return dtype == UPIR_F32;
    case UPIR_BODY_STENCIL2D: return dtype == UPIR_F32;
  }
  return 0;
}

// simd(simdlen) (reading c33): SIMD group size, and a chunk rounded up to
// whole groups (OpenMP's simd schedule modifier).
static int64_t simd_of(const upir_loop_desc *l) { return l->simdlen > 1 ? (int64_t)l->simdlen : 1; }
static int64_t simd_chunk(int64_t c, int64_t s) { return s > 1 && c > 0 ? (c + s - 1) / s * s : c; }

static upir_status validate_loop(const upir_spmd_desc *sd, const upir_loop_desc *l, int kind, int dtype,
                                 const upir_reduction *reds, int n_reds) {
  upir_status st = validate_spmd(sd);
  if (st != UPIR_OK) return st;
  if (!l) return fail(UPIR_E_INVALID, "loop descriptor is NULL");
  if (l->simdlen > 4096) return fail(UPIR_E_INVALID, "simdlen %u outside [0, 4096]", l->simdlen);
  if ((l->flags & (UPIR_TILE_COLMAJOR | UPIR_TILE_REVERSE)) && kind != UPIR_BODY_JACOBI5)
    return fail(UPIR_E_UNSUPPORTED, "UPIR_TILE_COLMAJOR / UPIR_TILE_REVERSE are implemented for JACOBI5 tiled nests only");
  int64_t T;
  st = upir_loop_normalize(l, &T, nullptr);
  if (st != UPIR_OK) return st;
  int sk;
  int64_t c;
  st = resolve_sched(l->policy, l->chunk, sk, c);
  if (st != UPIR_OK) return st;
  if (l->distribute != UPIR_DIST_TEAMS && l->distribute != UPIR_DIST_UNITS && l->distribute != UPIR_DIST_TEAMS_UNITS)
    return fail(UPIR_E_INVALID, "distribute must be TEAMS, UNITS or TEAMS_UNITS");
  const bool tiled = l->collapse == 2 && (l->tile[0] > 0 || l->tile[1] > 0);
  if (l->distribute == UPIR_DIST_UNITS && sd->num_teams > 1 && !tiled)
    return fail(UPIR_E_INVALID, "distribute(units) with num_teams > 1 would replicate the loop per team (reading c7)");
  if (kind < UPIR_BODY_AXPY || kind > UPIR_BODY_STENCIL2D) return fail(UPIR_E_INVALID, "unknown body kind %d", kind);
  if (dtype >= 0 && !body_dtype_ok(kind, dtype)) return fail(UPIR_E_INVALID, "dtype %d not valid for body %d", dtype, kind);
  if (n_reds < 0 || n_reds > 2) return fail(UPIR_E_INVALID, "n_reds=%d outside [0,2]", n_reds);
  if (n_reds > 0 && !reds) return fail(UPIR_E_INVALID, "reds is NULL");
  if (kind == UPIR_BODY_REDUCE && n_reds == 0) return fail(UPIR_E_INVALID, "REDUCE body needs a reduction");
  if ((kind == UPIR_BODY_JACOBI5 || kind == UPIR_BODY_MATMUL || kind == UPIR_BODY_MATVEC ||
       kind == UPIR_BODY_STENCIL2D) && n_reds > 0)
    return fail(UPIR_E_INVALID, "reductions are not defined for this body");
  if (kind == UPIR_BODY_MATVEC) {
    if (l->collapse != 1 || l->step[0] != 1) return fail(UPIR_E_INVALID, "MATVEC is a collapse(1) row loop with step 1");
    if (l->distribute == UPIR_DIST_UNITS && sd->num_teams > 1)
      return fail(UPIR_E_INVALID, "distribute(units) with num_teams > 1 would replicate rows (reading c7)");
    if (l->distribute == UPIR_DIST_TEAMS && l->inner_policy != UPIR_SCHED_STATIC)
      return fail(UPIR_E_UNSUPPORTED, "the k-loop inside a team is schedule(static, c) over units");
    return UPIR_OK;
  }
  for (int r = 0; r < n_reds; ++r) {
    if (reds[r].op < UPIR_OP_SUM || reds[r].op > UPIR_OP_MIN) return fail(UPIR_E_INVALID, "bad reduction op");
    if (reds[r].dtype != UPIR_I64 && reds[r].dtype != UPIR_F32) return fail(UPIR_E_INVALID, "reduction dtype must be I64 or F32");
    if (dtype >= 0 && reds[r].dtype != (kind == UPIR_BODY_AXPY ? UPIR_F32 : dtype))
      return fail(UPIR_E_INVALID, "reduction dtype does not match the body's element type");
  }
  if (kind == UPIR_BODY_AXPY || kind == UPIR_BODY_REDUCE) {
    if (l->collapse != 1) return fail(UPIR_E_INVALID, "AXPY/REDUCE loops have collapse 1");
  } else {
    if (l->collapse != 2) return fail(UPIR_E_INVALID, "JACOBI5/MATMUL loops are collapse(2) nests");
    for (int d = 0; d < 2; ++d)
      if (l->step[d] != 1) return fail(UPIR_E_INVALID, "JACOBI5/MATMUL levels need step 1");
  }
  if (kind == UPIR_BODY_JACOBI5 || kind == UPIR_BODY_STENCIL2D) {
    if (l->tile[0] <= 0 || l->tile[1] <= 0) return fail(UPIR_E_INVALID, "tiled stencils need tile[0], tile[1] > 0");
    if (l->distribute != UPIR_DIST_TEAMS) return fail(UPIR_E_INVALID, "the tile loop of a tiled nest is distributed over teams");
    if (l->inner_policy != UPIR_SCHED_STATIC || l->inner_chunk < 1)
      return fail(UPIR_E_UNSUPPORTED, "intra-tile loop supports schedule(static, c>=1) over units");
  }
  return UPIR_OK;
}

extern "C" upir_status upir_loop_validate(const upir_spmd_desc *sd, const upir_loop_desc *l, int32_t body_kind,
                                         const upir_reduction *reds, int32_t n_reds) {
  return validate_loop(sd, l, body_kind, -1, reds, n_reds);
}

// ------------------------------------------------------------------ stream loops
static upir_status check_map(upir_ctx c, upir_map m, const char *what) {
  if (!m) return fail(UPIR_E_NOT_MAPPED, "%s is not mapped (NULL)", what);
  if (m->ctx != c) return fail(UPIR_E_NOT_MAPPED, "%s belongs to another context", what);
  if (m->owned) {
    auto it = c->present.find(m->host);
    if (it == c->present.end() || it->second != m) return fail(UPIR_E_NOT_MAPPED, "%s is not in the present table", what);
  } else if (std::find(c->adopted.begin(), c->adopted.end(), m) == c->adopted.end()) {
    return fail(UPIR_E_NOT_MAPPED, "%s is not live", what);
  }
  return UPIR_OK;
}

// element view of a map for a body with element size esz
struct ElemView {
  char *base_shifted;   // element i at base_shifted + i*esz
  int64_t lo, hi;       // valid global element indices
  bool aligned16;
  int32_t esh;          // base_shifted = 128-B aligned address + esh * esz
};

static upir_status elem_view(upir_map m, int64_t esz, ElemView &v) {
  int64_t off, n;
  if (m->dist.pattern == UPIR_PATTERN_BLOCK) {
    if (m->elem_bytes != esz) return fail(UPIR_E_INVALID, "map element size %lld != body element size %lld",
                                          (long long)m->elem_bytes, (long long)esz);
    off = m->elem_offset;
    n = m->elems_local;
  } else {
    off = 0;
    n = (int64_t)(m->dev_bytes / esz);
  }
  v.base_shifted = (char *)m->dev - off * esz;
  v.lo = off;
  v.hi = off + n;
  v.aligned16 = ((uintptr_t)v.base_shifted % 16) == 0;
  if ((uintptr_t)v.base_shifted % esz != 0)
    return fail(UPIR_E_INVALID, "buffer is not aligned to its %lld-byte elements", (long long)esz);
  v.esh = (int32_t)(((uintptr_t)v.base_shifted % 128) / esz);
  return UPIR_OK;
}

// L2 promotion of the 4-column halo boxes of the Jacobi window (16 B per
// row).  64 B measured best (ncu, C5b 32768^2 sweep: DRAM reads 4.95 GB with
// 256 B promotion -> 4.70 GB, +2.5 % GLUP/s; each missed 16-B halo segment
// otherwise pulls 256 B).  Experiment hook UPIR_JACOBI_HALO_PROMO = 0 none,
// 1 64 B, 2 128 B, 3 256 B.
static CUtensorMapL2promotion jacobi_halo_promotion() {
  const char *v = getenv("UPIR_JACOBI_HALO_PROMO");
  const int k = v ? atoi(v) : 1;
  return k == 0 ? CU_TENSOR_MAP_L2_PROMOTION_NONE
         : k == 1 ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
         : k == 2 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B
                  : CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
}

static const char *env_path() {
  const char *p = getenv("UPIR_PATH");
  return p ? p : "";
}

// Guided chunk boundaries b_0 = 0, b_{g+1} = b_g + max(ceil((T - b_g)/p), c)
// (PAPER.md:644 'guided'), cached on the device per (T, p, c).
static upir_status guided_table(upir_ctx c, int64_t T, int64_t p, int64_t ch, int64_t simd, const int64_t **tab,
                                int64_t *nc) {
  for (auto &g : c->gtabs)
    if (g.T == T && g.p == p && g.c == ch && g.s == simd) {
      *tab = g.dev;
      *nc = g.n;
      return UPIR_OK;
    }
  if (c->capturing) return fail(UPIR_E_INVALID, "guided table must be built before graph capture");
  // chunk sequence over the G = ceil(T/s) SIMD groups (s = 1: iterations),
  // boundaries scaled back to iterations (reading c33)
  std::vector<int64_t> b;
  b.push_back(0);
  const int64_t G = (T + simd - 1) / simd, chg = (ch + simd - 1) / simd;
  int64_t start = 0;
  while (start < G) {
    const int64_t rem = G - start;
    int64_t len = (rem + p - 1) / p;
    if (len < chg) len = chg;
    if (len > rem) len = rem;
    start += len;
    b.push_back(std::min(start * simd, T));
  }
  const size_t bytes = b.size() * sizeof(int64_t);
  int64_t *dev = nullptr;
  CUDA_TRY(cudaMalloc(&dev, bytes));
  CUDA_TRY(cudaMemcpy(dev, b.data(), bytes, cudaMemcpyHostToDevice));
  c->gtabs.push_back({T, p, ch, simd, (int64_t)b.size() - 1, dev});
  *tab = dev;
  *nc = (int64_t)b.size() - 1;
  return UPIR_OK;
}

static upir_status exec_stream(upir_spmd s, const upir_loop_desc *l, const upir_body *b, const upir_reduction *reds,
                               int n_reds, upir_map trace) {
  upir_ctx c = s->ctx;
  const upir_spmd_desc &sd = s->d;
  int64_t T;
  upir_loop_normalize(l, &T, nullptr);
  int sk;
  int64_t chunk;
  resolve_sched(l->policy, l->chunk, sk, chunk);
  const int64_t simd = simd_of(l);
  if (sk != SK_GUIDED) chunk = simd_chunk(chunk, simd);   // guided: rounded in its table
  int64_t lb = l->lb[0], step = l->step[0];
  // cluster target: block-distribute the normalised space over ranks (c20),
  // whole SIMD groups per rank (c33)
  if (sd.target == UPIR_TARGET_CLUSTER && c->nranks > 1) {
    int64_t klo, khi;
    upir_dist_owned_rows((T + simd - 1) / simd, c->rank, c->nranks, &klo, &khi);
    klo = std::min(klo * simd, T);
    khi = std::min(khi * simd, T);
    lb = lb + klo * step;
    T = khi - klo;
  }
  const int body = b->kind == UPIR_BODY_AXPY ? SB_AXPY : (b->dtype == UPIR_I64 ? SB_RED_I64 : SB_RED_F32);
  const int64_t esz = b->dtype == UPIR_I64 ? 8 : 4;
  const int VEC = (int)(16 / esz);
  upir_status st = check_map(c, b->in0, "in0");
  if (st != UPIR_OK) return st;
  ElemView vx, vy{};
  if ((st = elem_view(b->in0, esz, vx)) != UPIR_OK) return st;
  if (body == SB_AXPY) {
    if ((st = check_map(c, b->out, "out")) != UPIR_OK) return st;
    if ((st = elem_view(b->out, esz, vy)) != UPIR_OK) return st;
  }
  // every touched element must lie inside the mapped (local) buffers
  if (T > 0) {
    const int64_t i0 = lb, i1 = lb + (T - 1) * step;
    const int64_t imin = std::min(i0, i1), imax = std::max(i0, i1);
    if (imin < vx.lo || imax >= vx.hi) return fail(UPIR_E_INVALID, "iterations [%lld,%lld] outside in0's elements [%lld,%lld)",
                                                  (long long)imin, (long long)imax, (long long)vx.lo, (long long)vx.hi);
    if (body == SB_AXPY && (imin < vy.lo || imax >= vy.hi))
      return fail(UPIR_E_INVALID, "iterations outside out's elements");
  }
  if (trace) {
    if ((st = check_map(c, trace, "trace")) != UPIR_OK) return st;
    if ((int64_t)trace->dev_bytes < 3 * T * 4) return fail(UPIR_E_INVALID, "trace map needs 3*T int32");
  }
  StreamArgs a;
  memset(&a, 0, sizeof a);
  a.T = T;
  a.lb = lb;
  a.step = step;
  a.sched = sk;
  a.distribute = l->distribute;
  a.chunk = sk == SK_STATIC_BLOCK ? 1 : chunk;
  a.simd = simd;
  a.in0 = vx.base_shifted;
  a.out = body == SB_AXPY ? vy.base_shifted : nullptr;
  // vector accesses are aligned by address (an adopted view with a storage
  // offset, or a BLOCK slice starting mid-line, is not 32-B aligned by index);
  // x and y at different offsets within a line: scalar accesses only
  a.esh = vx.esh;
  a.vecok = body != SB_AXPY || vy.esh == vx.esh;
  a.alpha = (float)b->alpha;
  a.safe_hi = body == SB_AXPY ? std::min(vx.hi, vy.hi) : vx.hi;
  a.safe_lo = body == SB_AXPY ? std::max(vx.lo, vy.lo) : vx.lo;
  a.nred = n_reds;
  for (int r = 0; r < n_reds; ++r) {
    a.red[r].op = reds[r].op;
    a.red[r].dtype = reds[r].dtype;
    a.red[r].result = reds[r].dev_result;
    if (!reds[r].dev_result) return fail(UPIR_E_INVALID, "reduction %d has no dev_result", r);
    if (reds[r].dtype == UPIR_I64) {
      int64_t v = reds[r].op == UPIR_OP_SUM ? 0 : (reds[r].op == UPIR_OP_MAX ? INT64_MIN : INT64_MAX);
      if (reds[r].init) memcpy(&v, reds[r].init, 8);
      a.red[r].init_bits = (uint64_t)v;
    } else {
      double v = reds[r].op == UPIR_OP_SUM ? 0.0 : (reds[r].op == UPIR_OP_MAX ? -HUGE_VAL : HUGE_VAL);
      if (reds[r].init) { float f; memcpy(&f, reds[r].init, 4); v = f; }
      memcpy(&a.red[r].init_bits, &v, 8);
    }
  }
  // UPIR_WORLD_REDUCE: upir.sync allreduce fused into the loop (peer windows),
  // or through the communicator: the last team writes the rank's partials,
  // NCCL all-gathers them and one kernel combines init (+) P_0 (+) ... -- the
  // same arithmetic as the fused path
  bool world_after = false;
  // (nranks == 1 with UPIR_WORLD_VIA_COMM: the same partial / combine path
  // with a device copy for the gather -- its arithmetic is testable on one GPU)
  const bool via_comm = (l->flags & UPIR_WORLD_VIA_COMM) != 0;
  if ((l->flags & UPIR_WORLD_REDUCE) && n_reds > 0 && (c->nranks > 1 || via_comm)) {
    if (c->nranks > 1 && world_ready(c) && !(via_comm && c->comm)) {
      a.wwin = c->win;
      a.wrank = c->rank;
      a.wranks = c->nranks;
    } else if (c->comm || c->nranks == 1) {
      // each rank's int64 / fp64 partials are all-gathered and combined with
      // init in ascending rank order, rounded once -- the same arithmetic as
      // the fused peer path
      world_after = true;
      a.wpart = reinterpret_cast<unsigned long long *>(reinterpret_cast<char *>(c->done) + 128);
      const size_t need = (size_t)c->nranks * 16;
      if (need > c->scratch_bytes) {
        if (c->capturing) return fail(UPIR_E_INVALID, "scratch must grow during capture");
        if (c->scratch) c->retired.push_back(c->scratch);   // graphs may hold it
        CUDA_TRY(cudaMalloc(&c->scratch, need));
        c->scratch_bytes = need;
      }
    } else {
      return fail(UPIR_E_INVALID, "UPIR_WORLD_REDUCE needs every rank's peer window (upir_peer_import) or a communicator");
    }
  }
  a.trace = trace ? (int32_t *)trace->dev : nullptr;
  // long per-unit chunks: 256-bit loads, 4 in flight (dvar 1); for AXPY teams
  // of > 256 units the main loop is aligned to whole 128-B lines (dvar 8) --
  // teams of <= 256 units take the axpy_long setting below (round-1 / round-2
  // sweeps, tools/sweep_r2.py)
  a.dvar = body == SB_AXPY ? 8 : 1;
  if (const char *dv = getenv("UPIR_DVAR")) a.dvar = atoi(dv);
  // dynamic tickets: m chunks per unit so a ticket covers >= ~256 KiB
  const int p_team = l->distribute == UPIR_DIST_TEAMS ? 1 : sd.num_units;
  const int64_t p_sched = l->distribute == UPIR_DIST_TEAMS ? sd.num_teams
                         : l->distribute == UPIR_DIST_UNITS ? sd.num_units
                         : (int64_t)sd.num_teams * sd.num_units;
  if (sk == SK_GUIDED) {
    st = guided_table(c, T, p_sched, chunk, simd, &a.gtab, &a.gchunks);
    if (st != UPIR_OK) return st;
    a.dyn_counter = c->dyn;
  }
  if (sk == SK_DYNAMIC) {
    const int64_t want = (256 * 1024) / esz;
    a.ticket_m = std::max<int64_t>(1, (want + (int64_t)p_team * chunk - 1) / ((int64_t)p_team * chunk));
    a.dyn_counter = c->dyn;
  }
  a.slots = c->slots;
  a.done = c->done;
  st = ensure_slots(c, (size_t)sd.num_teams);
  if (st != UPIR_OK) return st;
  a.slots = c->slots;
  // memory path: per-unit chunk longer than one vector -> staged
  const int64_t p = l->distribute == UPIR_DIST_TEAMS ? sd.num_teams
                   : l->distribute == UPIR_DIST_UNITS ? sd.num_units
                   : (int64_t)sd.num_teams * sd.num_units;
  int64_t unit_chunk = sk == SK_STATIC_BLOCK ? ((T + simd - 1) / simd + p - 1) / p * simd : chunk;
  // the staged path is warp-cooperative: it needs whole warps
  const bool can_stage = (step == 1 || step == -1) && vx.aligned16 && (body != SB_AXPY || vy.aligned16) &&
                         sd.num_units % 32 == 0;
  // Default: DIRECT (long per-unit chunks use 256-bit loads with a 256-B L2
  // prefetch, measured at ~1.0x the copy bandwidth on B200, above the staged
  // variant); UPIR_PATH=staged selects the TMA-bulk staged path.
  bool staged = false;
  const char *ep = env_path();
  if (!strcmp(ep, "direct")) staged = false;
  if (!strcmp(ep, "staged") && can_stage) staged = true;
  int segv = 0, nst = 0;
  size_t smem = 0;
  if (staged) {
    // pick (SEGV, NST) maximising bytes in flight per SM under the smem budget
    const int cfg[5][2] = {{16, 3}, {16, 2}, {8, 3}, {8, 2}, {4, 2}};
    double best = -1;
    const int warps = (sd.num_units + 31) / 32;
    for (auto &cf : cfg) {
      size_t sm = staged_smem_bytes(body, sd.num_units, cf[0], cf[1]);
      if (sm > 227 * 1024) continue;
      int ctas = std::min<int>(std::min<int>((int)((227 * 1024) / std::max<size_t>(sm, 1)), 2048 / (warps * 32)), 32);
      ctas = std::min<int64_t>(ctas, (sd.num_teams + c->num_sms - 1) / c->num_sms);
      if (ctas < 1) ctas = 1;
      double inflight = std::min(128.0 * 1024, (double)ctas * warps * (cf[1] - 1) * cf[0] * 16 * 32);
      if (inflight > best + 1e-9) { best = inflight; segv = cf[0]; nst = cf[1]; smem = sm; }
    }
    if (best < 0) staged = false;
    // experiment hook: UPIR_STAGE=segv,nst forces a configuration
    const char *fc = getenv("UPIR_STAGE");
    int fs = 0, fn = 0;
    if (fc && sscanf(fc, "%d,%d", &fs, &fn) == 2) {
      size_t sm = staged_smem_bytes(body, sd.num_units, fs, fn);
      if (sm > 0 && sm <= 227 * 1024) { segv = fs; nst = fn; smem = sm; staged = true; }
    }
  }
  if (!staged) { segv = 0; nst = 0; smem = 0; }
  // AXPY with long per-unit chunks (static block): every unit streams its own
  // x, y and y' ranges -- 3 DRAM streams per unit.  Measured best with 2 x
  // 32-B loads per array in flight per unit (dvar 1, no line alignment) and
  // ONE resident team per SM (fewer concurrent streams, better DRAM row
  // locality): 0.69 -> 0.82 of the copy bandwidth at 592 x 256 over 2^28
  // (tools/sweep_r2.py); reserved dynamic shared memory enforces the
  // residency (the direct path uses none).
  const bool axpy_long = body == SB_AXPY && !staged && unit_chunk >= 256 && sd.num_units <= 256;
  if (axpy_long && !getenv("UPIR_DVAR")) a.dvar = 1;
  if (axpy_long && !getenv("UPIR_DIRECT_OCC")) smem = (size_t)(228 * 1024) / 2 + 1024;
  // experiment hook UPIR_DIRECT_OCC = k: reserve dynamic shared memory so
  // that at most k teams are resident per SM (fewer concurrent per-unit
  // streams; the direct path itself uses no dynamic shared memory)
  if (!staged)
    if (const char *v = getenv("UPIR_DIRECT_OCC")) {
      const int k = atoi(v);
      if (k > 0) smem = (size_t)(228 * 1024) / (size_t)(k + 1) + 1024;
    }
  cudaError_t e = launch_stream_loop(body, staged ? PATH_STAGED : PATH_DIRECT, segv, nst, trace != nullptr,
                                     sd.num_teams, sd.num_units, smem, a, c->compute);
  if (e != cudaSuccess) return fail(UPIR_E_CUDA, "loop kernel launch failed: %s", cudaGetErrorString(e));
  c->launches++;
  if (world_after) {
    if (c->nranks > 1) NCCL_TRY(ncclAllGather(a.wpart, c->scratch, 2, ncclUint64, c->comm, c->compute));
    else CUDA_TRY(cudaMemcpyAsync(c->scratch, a.wpart, 16, cudaMemcpyDeviceToDevice, c->compute));
    e = launch_world_combine(reinterpret_cast<const unsigned long long *>(c->scratch), c->nranks, n_reds, a.red,
                             c->compute);
    if (e != cudaSuccess) return fail(UPIR_E_CUDA, "world combine launch failed: %s", cudaGetErrorString(e));
    c->launches++;
  }
  return UPIR_OK;
}

static upir_status exec_jacobi(upir_spmd s, const upir_loop_desc *l, const upir_body *b, upir_map trace);
static upir_status exec_matvec(upir_spmd s, const upir_loop_desc *l, const upir_body *b, upir_map trace);
static upir_status exec_stencil(upir_spmd s, const upir_loop_desc *l, const upir_body *b, upir_map trace);
static upir_status exec_matmul(upir_spmd s, const upir_loop_desc *l, const upir_body *b, upir_map trace);

extern "C" upir_status upir_loop_exec(upir_spmd s, const upir_loop_desc *l, const upir_body *b,
                                      const upir_reduction *reds, int32_t n_reds, upir_map trace) {
  if (!s || !b) return fail(UPIR_E_INVALID, "NULL argument");
  upir_ctx c = s->ctx;
  if (std::find(c->regions.begin(), c->regions.end(), s) == c->regions.end())
    return fail(UPIR_E_INVALID, "region is not open");
  upir_status st = validate_loop(&s->d, l, b->kind, b->dtype, reds, n_reds);
  if (st != UPIR_OK) return st;
  if (c->sticky != cudaSuccess) return sticky_check(c);
  cudaSetDevice(c->device);
  switch (b->kind) {
    case UPIR_BODY_AXPY:
    case UPIR_BODY_REDUCE: st = exec_stream(s, l, b, reds, n_reds, trace); break;
    case UPIR_BODY_JACOBI5: st = exec_jacobi(s, l, b, trace); break;
    case UPIR_BODY_MATMUL: st = exec_matmul(s, l, b, trace); break;
    case UPIR_BODY_MATVEC: st = exec_matvec(s, l, b, trace); break;
    case UPIR_BODY_STENCIL2D: st = exec_stencil(s, l, b, trace); break;
  }
  if (st != UPIR_OK) return st;
  // out was validated by the body (REDUCE ignores it): a write by anything but
  // a peer-mode sweep leaves the halos un-exchanged
  if (b->kind != UPIR_BODY_REDUCE && b->kind != UPIR_BODY_JACOBI5) b->out->halo_fused = false;
  // implicit barrier at the end of a worksharing loop: stream
  // order makes every later operation wait; the host waits only at upir_sync.
  return UPIR_OK;
}

// ------------------------------------------------------------------ jacobi / matmul
// Tile-loop schedule over teams (readings c3, c8, c24).
static upir_status tile_sched(const upir_loop_desc *l, int &sk, int64_t &chunk) {
  upir_status st = resolve_sched(l->policy, l->chunk, sk, chunk);
  if (st != UPIR_OK) return st;
  if (sk == SK_GUIDED) return fail(UPIR_E_UNSUPPORTED, "guided tile loops are not built (static / dynamic)");
  if (sk == SK_STATIC_BLOCK) chunk = 1;
  return UPIR_OK;
}

static upir_status exec_jacobi(upir_spmd s, const upir_loop_desc *l, const upir_body *b, upir_map trace) {
  upir_ctx c = s->ctx;
  const upir_spmd_desc &sd = s->d;
  upir_status st;
  if ((st = check_map(c, b->in0, "in0")) != UPIR_OK) return st;
  if ((st = check_map(c, b->out, "out")) != UPIR_OK) return st;
  const int64_t ny = b->dims[0], ld = b->ld[0];
  const int bm = (int)l->tile[0], bn = (int)l->tile[1];
  if (!jacobi_supported_tile(bm, bn))
    return fail(UPIR_E_UNSUPPORTED, "JACOBI5 tile %dx%d not built (32x256, 32x128, 16x256, 64x128, 8x64)", bm, bn);
  if (ny < 3 || ld < 3) return fail(UPIR_E_INVALID, "JACOBI5 needs dims[0] (rows) >= 3 and ld[0] (row pitch) >= 3");
  if (ld % 4 != 0) return fail(UPIR_E_UNSUPPORTED, "JACOBI5 row pitch must be a multiple of 4 elements (TMA stride)");
  ElemView vi, vo;
  if ((st = elem_view(b->in0, 4, vi)) != UPIR_OK) return st;
  if ((st = elem_view(b->out, 4, vo)) != UPIR_OK) return st;
  if (vi.lo != vo.lo || vi.hi != vo.hi) return fail(UPIR_E_INVALID, "in0 and out must have the same layout");
  if (vi.lo % ld != 0 || vi.hi % ld != 0) return fail(UPIR_E_INVALID, "maps must hold whole rows of ld elements");
  const int64_t row0 = vi.lo / ld, rows_local = (vi.hi - vi.lo) / ld;
  // the 5-point stencil reads i +- 1 and j +- 1
  int64_t lb0 = l->lb[0], ub0 = l->ub[0], lb1 = l->lb[1], ub1 = l->ub[1];
  if (lb0 < 1 || ub0 > ny - 1 || lb1 < 1 || ub1 > ld - 1)
    return fail(UPIR_E_INVALID, "JACOBI5 iteration space must lie in the grid interior [1,ny-1) x [1,ld-1)");
  // peer mode: the out map has imported neighbour buffers (fused halo)
  const upir_map mo = b->out;
  const bool peer = sd.target == UPIR_TARGET_CLUSTER && c->nranks > 1 && (mo->peer_dev[0] || mo->peer_dev[1]) &&
                    !(l->flags & UPIR_HALO_EXPLICIT);
  if (sd.target == UPIR_TARGET_CLUSTER && c->nranks > 1) {
    upir_map m = b->in0;
    if (m->dist.pattern != UPIR_PATTERN_BLOCK) return fail(UPIR_E_INVALID, "cluster JACOBI5 needs BLOCK-distributed maps");
    lb0 = std::max(lb0, m->row_lo);
    ub0 = std::min(ub0, m->row_hi);
  }
  if (ub0 > lb0 && (lb0 - 1 < row0 || ub0 + 1 > row0 + rows_local))
    return fail(UPIR_E_INVALID, "rows [%lld,%lld) need halo rows outside the local buffer [%lld,%lld)", (long long)lb0,
                (long long)ub0, (long long)row0, (long long)(row0 + rows_local));
  JacobiArgs a;
  memset(&a, 0, sizeof a);
  a.colmajor = (l->flags & UPIR_TILE_COLMAJOR) ? 1 : 0;
  a.reverse = (l->flags & UPIR_TILE_REVERSE) ? 1 : 0;
  if (peer) {
    int64_t plan[8];
    if ((st = upir_halo_plan(mo->dist.n_rows, mo->dist.halo_rows, c->rank, c->nranks, plan)) != UPIR_OK) return st;
    a.send_up_row = a.send_dn_row = a.halo_up_row = a.halo_dn_row = -1;
    if (plan[1] > plan[0]) {   // exchange with rank - 1: send row lo, read halo row lo - 1
      if (!mo->peer_dev[0] || !c->peer_win[c->rank - 1])
        return fail(UPIR_E_INVALID, "peer-mode JACOBI5: rank %d's buffer / window not imported", c->rank - 1);
      a.win_up = c->peer_win[c->rank - 1];
      a.peer_up = mo->peer_dev[0];
      a.peer_up_row0 = mo->peer_row0[0];
      a.send_up_row = plan[0];
      a.halo_up_row = plan[0] - 1;
    }
    if (plan[5] > plan[4]) {   // exchange with rank + 1: send row hi - 1, read halo row hi
      if (!mo->peer_dev[1] || c->rank + 1 >= WIN_MAX_RANKS || !c->peer_win[c->rank + 1])
        return fail(UPIR_E_INVALID, "peer-mode JACOBI5: rank %d's buffer / window not imported", c->rank + 1);
      a.win_dn = c->peer_win[c->rank + 1];
      a.peer_dn = mo->peer_dev[1];
      a.peer_dn_row0 = mo->peer_row0[1];
      a.send_dn_row = plan[5] - 1;
      a.halo_dn_row = plan[5];
    }
    a.win = c->win;
  }
  a.out = reinterpret_cast<float *>(b->out->dev);
  a.ld = ld;
  a.row0 = row0;
  a.lb0 = lb0;
  a.ub0 = ub0;
  a.lb1 = lb1;
  a.ub1 = ub1;
  const bool empty = ub0 <= lb0 || ub1 <= lb1;
  if (empty && !peer) {   // empty iteration space
    mo->halo_fused = false;
    return UPIR_OK;
  }
  if (!empty) {
    a.ti0 = lb0 / bm;
    a.tj0 = lb1 / bn;
    a.ntr = (ub0 + bm - 1) / bm - a.ti0;
    a.ntc = (ub1 + bn - 1) / bn - a.tj0;
  } else {
    a.ntc = 1;   // no tiles; the sweep still delivers to the neighbours
  }
  int sk;
  int64_t chunk;
  if ((st = tile_sched(l, sk, chunk)) != UPIR_OK) return st;
  a.sched = sk;
  a.chunk = chunk;
  a.inner_chunk = (int)simd_chunk(l->inner_chunk, simd_of(l));   // intra-tile SIMD groups (c33)
  a.dyn_counter = c->dyn;
  a.done = c->done;
  if (trace) {
    if ((st = check_map(c, trace, "trace")) != UPIR_OK) return st;
    const int64_t need = 3 * a.ntr * a.ntc * bm * bn * 4;
    if ((int64_t)trace->dev_bytes < need) return fail(UPIR_E_INVALID, "trace map needs %lld bytes", (long long)need);
    a.trace = (int32_t *)trace->dev;
  }
  CUtensorMap tmc, tmh;
  const void *base = b->in0->dev;
  if (!encode_tmap_2d(&tmc, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, base, (uint64_t)ld, (uint64_t)rows_local, (uint64_t)ld * 4,
                      (uint32_t)bn, (uint32_t)(bm + 2), CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B) ||
      !encode_tmap_2d(&tmh, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, base, (uint64_t)ld, (uint64_t)rows_local, (uint64_t)ld * 4, 4,
                      (uint32_t)(bm + 2), CU_TENSOR_MAP_SWIZZLE_NONE, jacobi_halo_promotion()))
    return fail(UPIR_E_CUDA, "cuTensorMapEncodeTiled failed for the JACOBI5 input");
  cudaError_t e = launch_jacobi_tma(a, &tmc, &tmh, sd.num_teams, sd.num_units, bm, bn, trace != nullptr, c->compute);
  if (e != cudaSuccess) return fail(UPIR_E_CUDA, "JACOBI5 launch failed: %s", cudaGetErrorString(e));
  c->launches++;
  mo->halo_fused = peer;
  return UPIR_OK;
}
static upir_status exec_stencil(upir_spmd s, const upir_loop_desc *l, const upir_body *b, upir_map trace) {
  upir_ctx c = s->ctx;
  const upir_spmd_desc &sd = s->d;
  upir_status st;
  if ((st = check_map(c, b->in0, "in0")) != UPIR_OK) return st;
  if ((st = check_map(c, b->in1, "in1 (weights)")) != UPIR_OK) return st;
  if ((st = check_map(c, b->out, "out")) != UPIR_OK) return st;
  const int64_t ny = b->dims[0], F = b->dims[1], ld = b->ld[0];
  const int R = (int)(F - 1) / 2;
  const int bm = (int)l->tile[0], bn = (int)l->tile[1];
  if (!stencil_supported((int)F, bm, bn))
    return fail(UPIR_E_UNSUPPORTED, "STENCIL2D: filter size %lld / tile %dx%d not built (F 3/5/7, tiles 16x128, 8x64, 16x512, 16x1024, 8x512, 8x1024)",
                (long long)F, bm, bn);
  if ((int64_t)b->in1->dev_bytes < F * F * 4) return fail(UPIR_E_INVALID, "weights map needs F*F fp32");
  if (ld % 4 != 0) return fail(UPIR_E_UNSUPPORTED, "STENCIL2D row pitch must be a multiple of 4 elements (TMA stride)");
  ElemView vi, vo;
  if ((st = elem_view(b->in0, 4, vi)) != UPIR_OK) return st;
  if ((st = elem_view(b->out, 4, vo)) != UPIR_OK) return st;
  if (vi.lo != vo.lo || vi.hi != vo.hi) return fail(UPIR_E_INVALID, "in0 and out must have the same layout");
  if (ld < 1 || vi.lo % ld != 0 || vi.hi % ld != 0) return fail(UPIR_E_INVALID, "maps must hold whole rows");
  const int64_t row0 = vi.lo / ld, rows_local = (vi.hi - vi.lo) / ld;
  int64_t lb0 = l->lb[0], ub0 = l->ub[0], lb1 = l->lb[1], ub1 = l->ub[1];
  if (lb0 < R || ub0 > ny - R || lb1 < R || ub1 > ld - R)
    return fail(UPIR_E_INVALID, "STENCIL2D iteration space must lie in [R, ny-R) x [R, ld-R)");
  if (sd.target == UPIR_TARGET_CLUSTER && c->nranks > 1) {
    upir_map m = b->in0;
    if (m->dist.pattern != UPIR_PATTERN_BLOCK || m->dist.halo_rows < R)
      return fail(UPIR_E_INVALID, "cluster STENCIL2D needs BLOCK maps with halo_rows >= R");
    lb0 = std::max(lb0, m->row_lo);
    ub0 = std::min(ub0, m->row_hi);
  }
  if (ub0 > lb0 && (lb0 - R < row0 || ub0 + R > row0 + rows_local))
    return fail(UPIR_E_INVALID, "rows need halo rows outside the local buffer");
  StencilArgs a;
  memset(&a, 0, sizeof a);
  a.in = (const float *)b->in0->dev;
  a.out = (float *)b->out->dev;
  a.w = (const float *)b->in1->dev;
  a.ld = ld;
  a.row0 = row0;
  a.ny = std::min(ny, row0 + rows_local);
  a.nx = ld;
  a.lb0 = lb0; a.ub0 = ub0; a.lb1 = lb1; a.ub1 = ub1;
  if (ub0 <= lb0 || ub1 <= lb1) return UPIR_OK;
  a.ti0 = lb0 / bm;
  a.tj0 = lb1 / bn;
  a.ntr = (ub0 + bm - 1) / bm - a.ti0;
  a.ntc = (ub1 + bn - 1) / bn - a.tj0;
  int sk;
  int64_t chunk;
  if ((st = tile_sched(l, sk, chunk)) != UPIR_OK) return st;
  a.sched = sk;
  a.chunk = chunk;
  a.inner_chunk = (int)simd_chunk(l->inner_chunk, simd_of(l));   // intra-tile SIMD groups (c33)
  a.dyn_counter = c->dyn;
  a.done = c->done;
  if (trace) {
    if ((st = check_map(c, trace, "trace")) != UPIR_OK) return st;
    const int64_t need = 3 * a.ntr * a.ntc * bm * bn * 4;
    if ((int64_t)trace->dev_bytes < need) return fail(UPIR_E_INVALID, "trace map needs %lld bytes", (long long)need);
    a.trace = (int32_t *)trace->dev;
  }
  cudaError_t e = launch_stencil(a, (int)F, bm, bn, sd.num_teams, sd.num_units, c->compute);
  if (e != cudaSuccess) return fail(UPIR_E_CUDA, "STENCIL2D launch failed: %s", cudaGetErrorString(e));
  c->launches++;
  return UPIR_OK;
}

static upir_status exec_matvec(upir_spmd s, const upir_loop_desc *l, const upir_body *b, upir_map trace) {
  upir_ctx c = s->ctx;
  const upir_spmd_desc &sd = s->d;
  upir_status st;
  if ((st = check_map(c, b->in0, "in0 (A)")) != UPIR_OK) return st;
  if ((st = check_map(c, b->in1, "in1 (x)")) != UPIR_OK) return st;
  if ((st = check_map(c, b->out, "out (y)")) != UPIR_OK) return st;
  const int64_t K = b->dims[0], M = b->dims[1], lda = b->ld[0];
  if (K < 1 || M < 1 || lda < K) return fail(UPIR_E_INVALID, "MATVEC needs dims = (K, M) >= 1 and ld[0] >= K");
  if ((int64_t)b->in0->dev_bytes < ((M - 1) * lda + K) * 4 || (int64_t)b->in1->dev_bytes < K * 4 ||
      (int64_t)b->out->dev_bytes < M * 4)
    return fail(UPIR_E_INVALID, "MATVEC maps smaller than A (M x K), x (K) and y (M)");
  int64_t T;
  upir_loop_normalize(l, &T, nullptr);
  const int64_t lb = l->lb[0];
  if (lb < 0 || lb + T > M) return fail(UPIR_E_INVALID, "MATVEC rows must lie in [0, M)");
  int sk;
  int64_t chunk;
  if ((st = resolve_sched(l->policy, l->chunk, sk, chunk)) != UPIR_OK) return st;
  if (sk == SK_GUIDED) return fail(UPIR_E_UNSUPPORTED, "guided MATVEC row loops are not built");
  if (sk == SK_DYNAMIC && l->distribute != UPIR_DIST_TEAMS)
    return fail(UPIR_E_UNSUPPORTED, "dynamic MATVEC rows are scheduled over teams only");
  if (sk == SK_STATIC_BLOCK) chunk = 1;
  // simd (c33): the loop the units execute -- the k-loop under
  // distribute(teams), else the row loop
  const int64_t simd = simd_of(l);
  const bool simd_rows = l->distribute != UPIR_DIST_TEAMS;
  if (simd_rows && sk != SK_STATIC_BLOCK) chunk = simd_chunk(chunk, simd);
  MatvecArgs a;
  memset(&a, 0, sizeof a);
  a.simd = simd_rows ? simd : 1;
  a.A = (const float *)b->in0->dev;
  a.x = (const float *)b->in1->dev;
  a.y = (float *)b->out->dev;
  a.K = K;
  a.lda = lda;
  a.lb = lb;
  a.T = T;
  a.sched = sk;
  a.chunk = chunk;
  a.distribute = l->distribute;
  a.inner_chunk = (int)simd_chunk(l->inner_chunk > 0 ? l->inner_chunk : 4, simd_rows ? 1 : simd);
  a.dyn_counter = c->dyn;
  a.done = c->done;
  if (trace) {
    if ((st = check_map(c, trace, "trace")) != UPIR_OK) return st;
    if ((int64_t)trace->dev_bytes < 3 * T * 4) return fail(UPIR_E_INVALID, "trace map needs 3*T int32");
    a.trace = (int32_t *)trace->dev;
  }
  if (T == 0) return UPIR_OK;
  cudaError_t e = launch_matvec(a, sd.num_teams, sd.num_units, c->compute);
  if (e != cudaSuccess) return fail(UPIR_E_CUDA, "MATVEC launch failed: %s", cudaGetErrorString(e));
  c->launches++;
  return UPIR_OK;
}

static upir_status exec_matmul(upir_spmd s, const upir_loop_desc *l, const upir_body *b, upir_map trace) {
  upir_ctx c = s->ctx;
  const upir_spmd_desc &sd = s->d;
  upir_status st;
  if ((st = check_map(c, b->in0, "in0 (A)")) != UPIR_OK) return st;
  if ((st = check_map(c, b->in1, "in1 (B)")) != UPIR_OK) return st;
  if ((st = check_map(c, b->out, "out (C)")) != UPIR_OK) return st;
  const int64_t K = b->dims[0], M = b->dims[1], N = b->dims[2];
  const int64_t lda = b->ld[0], ldb = b->ld[1], ldc = b->ld[2];
  if (M < 1 || N < 1 || K < 1) return fail(UPIR_E_INVALID, "MATMUL needs dims = (K, M, N) >= 1");
  if (lda < K || ldb < N || ldc < N) return fail(UPIR_E_INVALID, "MATMUL leading dimensions too small");
  if (lda % 8 || ldb % 8 || ldc % 8)
    return fail(UPIR_E_UNSUPPORTED, "MATMUL needs lda, ldb, ldc multiples of 8 elements (TMA / 32-B stores)");
  const int64_t es = b->dtype == UPIR_F32 ? 4 : 2;
  if (es == 4 && (lda % 4 || ldb % 4)) return fail(UPIR_E_UNSUPPORTED, "fp32 MATMUL needs lda, ldb multiples of 4");
  const int64_t MA = b->in0->dist.pattern == UPIR_PATTERN_BLOCK ? b->in0->loc_row_hi - b->in0->loc_row_lo : M;
  if (MA > 0 && ((int64_t)b->in0->dev_bytes < ((MA - 1) * lda + K) * es ||
                 (int64_t)b->in1->dev_bytes < ((K - 1) * ldb + N) * es ||
                 (int64_t)b->out->dev_bytes < ((MA - 1) * ldc + N) * 4))
    return fail(UPIR_E_INVALID, "MATMUL maps smaller than the matrices they hold");
  if (l->lb[0] < 0 || l->ub[0] > M || l->lb[1] < 0 || l->ub[1] > N)
    return fail(UPIR_E_INVALID, "MATMUL iteration space must lie in [0,M) x [0,N)");
  // rows of A and C may be BLOCK-distributed over ranks (B replicated): the
  // local buffers hold global rows [row0, row0 + local rows)
  int64_t row0 = 0, rows_here = M;
  const upir_map mA = b->in0, mC = b->out;
  if (mA->dist.pattern == UPIR_PATTERN_BLOCK || mC->dist.pattern == UPIR_PATTERN_BLOCK) {
    if (mA->dist.pattern != UPIR_PATTERN_BLOCK || mC->dist.pattern != UPIR_PATTERN_BLOCK ||
        mA->loc_row_lo != mC->loc_row_lo || mA->loc_row_hi != mC->loc_row_hi || mA->dist.n_rows != M ||
        mC->dist.n_rows != M)
      return fail(UPIR_E_INVALID, "distributed MATMUL needs A and C BLOCK-distributed over the same M rows");
    row0 = mA->loc_row_lo;
    rows_here = mA->loc_row_hi - mA->loc_row_lo;
  }
  if (!matmul_units_ok(b->dtype, sd.num_units))
    return fail(UPIR_E_INVALID,
                "the tcgen05 MATMUL body runs %d units per team for this dtype (bf16 also 512 = a CTA pair; got %d): "
                "geometry is not clamped", matmul_required_units(b->dtype), sd.num_units);
  int sk;
  int64_t chunk;
  if ((st = tile_sched(l, sk, chunk)) != UPIR_OK) return st;
  if (sk == SK_DYNAMIC) return fail(UPIR_E_UNSUPPORTED, "MATMUL tile loop supports static schedules");
  MatmulArgs a;
  memset(&a, 0, sizeof a);
  a.A = b->in0->dev;
  a.B = b->in1->dev;
  a.C = (float *)b->out->dev;
  a.M = M; a.N = N; a.K = K;
  a.lda = lda; a.ldb = ldb; a.ldc = ldc;
  a.lb0 = l->lb[0]; a.ub0 = l->ub[0]; a.lb1 = l->lb[1]; a.ub1 = l->ub[1];
  a.row0 = row0;
  if (sd.target == UPIR_TARGET_CLUSTER && c->nranks > 1) {
    // cluster SPMD: the (i) level is block-distributed over the ranks (c20)
    int64_t lo, hi;
    upir_dist_owned_rows(M, c->rank, c->nranks, &lo, &hi);
    a.lb0 = std::max(a.lb0, lo);
    a.ub0 = std::min(a.ub0, hi);
  }
  if (a.ub0 > a.lb0 && (a.lb0 < row0 || a.ub0 > row0 + rows_here))
    return fail(UPIR_E_INVALID, "MATMUL rows [%lld,%lld) are not held locally", (long long)a.lb0, (long long)a.ub0);
  if (a.ub0 <= a.lb0 || a.ub1 <= a.lb1) return UPIR_OK;
  a.sched = sk;
  a.chunk = chunk;
  const int64_t bm = matmul_tile_m_for(b->dtype, sd.num_units), bn = matmul_tile_n();
  const int64_t nt = ((a.ub0 + bm - 1) / bm - a.lb0 / bm) * ((a.ub1 + bn - 1) / bn - a.lb1 / bn);
  if (trace) {
    if ((st = check_map(c, trace, "trace")) != UPIR_OK) return st;
    if ((int64_t)trace->dev_bytes < 3 * nt * 4) return fail(UPIR_E_INVALID, "trace map needs 3*ntiles int32");
    a.trace = (int32_t *)trace->dev;
  }
  alignas(64) CUtensorMap ta, tb, ta2, tb2;
  // 3xTF32 on CTA pairs: split A and B into tf32 hi / lo copies first (one
  // elementwise pass each, stream-ordered scratch), the loop kernel streams
  // both copies with TMA
  const bool presplit = b->dtype == UPIR_F32 && matmul_f32_presplit(sd.num_units);
  float *scratch = nullptr;
  const int64_t nA = (rows_here - 1) * lda + K, nB = (K - 1) * ldb + N;
  if (presplit) {
    const size_t bytes = (size_t)(2 * (nA + nB) + 64) * 4;
    CUDA_TRY(cudaMallocAsync((void **)&scratch, bytes, c->compute));
    float *ahi = scratch, *alo = ahi + ((nA + 31) / 32) * 32, *bhi = alo + ((nA + 31) / 32) * 32,
          *blo = bhi + ((nB + 31) / 32) * 32;
    cudaError_t e1 = launch_tf32_split((const float *)a.A, ahi, alo, nA, c->num_sms, c->compute);
    cudaError_t e2 = launch_tf32_split((const float *)a.B, bhi, blo, nB, c->num_sms, c->compute);
    if (e1 != cudaSuccess || e2 != cudaSuccess) {
      cudaFreeAsync(scratch, c->compute);
      return fail(UPIR_E_CUDA, "3xTF32 split launch failed: %s", cudaGetErrorString(e1 != cudaSuccess ? e1 : e2));
    }
    c->launches += 2;
    if (!matmul_encode_tmaps(&ta, &tb, ahi, bhi, b->dtype, rows_here, N, K, lda, ldb) ||
        !matmul_encode_tmaps(&ta2, &tb2, alo, blo, b->dtype, rows_here, N, K, lda, ldb)) {
      cudaFreeAsync(scratch, c->compute);
      return fail(UPIR_E_CUDA, "cuTensorMapEncodeTiled failed for MATMUL operands");
    }
    a.tmap_a2 = &ta2;
    a.tmap_b2 = &tb2;
  } else if (!matmul_encode_tmaps(&ta, &tb, a.A, a.B, b->dtype, rows_here, N, K, lda, ldb)) {
    return fail(UPIR_E_CUDA, "cuTensorMapEncodeTiled failed for MATMUL operands");
  }
  a.tmap_a = &ta;
  a.tmap_b = &tb;
  cudaError_t e = launch_matmul(a, b->dtype, sd.num_teams, sd.num_units, c->compute);
  if (scratch) cudaFreeAsync(scratch, c->compute);   // stream-ordered: after the loop kernel
  if (e != cudaSuccess) return fail(UPIR_E_CUDA, "MATMUL launch failed: %s", cudaGetErrorString(e));
  c->launches++;
  return UPIR_OK;
}

// ------------------------------------------------------------------ upir.sync
extern "C" upir_status upir_reduce(upir_ctx c, int32_t op, int32_t dtype, const void *dev_in, int64_t count,
                                   void *dev_out, int32_t scope) {
  if (!c || !dev_in || !dev_out || count < 1) return fail(UPIR_E_INVALID, "bad argument");
  if (op < UPIR_OP_SUM || op > UPIR_OP_MIN) return fail(UPIR_E_INVALID, "bad op");
  if (dtype != UPIR_I64 && dtype != UPIR_F32) return fail(UPIR_E_INVALID, "dtype must be I64 or F32");
  cudaSetDevice(c->device);
  const size_t esz = dtype == UPIR_I64 ? 8 : 4;
  if (scope == UPIR_SCOPE_DEVICE) {
    StreamArgs a;
    memset(&a, 0, sizeof a);
    const int VEC = (int)(16 / esz);
    a.T = count;
    a.lb = 0;
    a.step = 1;
    a.sched = SK_STATIC_CHUNK;
    a.chunk = ((uintptr_t)dev_in % 16 == 0) ? VEC : 1;
    a.distribute = UPIR_DIST_TEAMS_UNITS;
    a.in0 = dev_in;
    a.safe_lo = 0;
    a.safe_hi = count;
    a.nred = 1;
    a.red[0].op = op;
    a.red[0].dtype = dtype;
    a.red[0].result = dev_out;
    if (dtype == UPIR_I64) {
      int64_t v = op == UPIR_OP_SUM ? 0 : (op == UPIR_OP_MAX ? INT64_MIN : INT64_MAX);
      a.red[0].init_bits = (uint64_t)v;
    } else {
      double v = op == UPIR_OP_SUM ? 0.0 : (op == UPIR_OP_MAX ? -HUGE_VAL : HUGE_VAL);
      memcpy(&a.red[0].init_bits, &v, 8);
    }
    int teams = (int)std::min<int64_t>((int64_t)c->num_sms * 4, std::max<int64_t>(1, (count + 1023) / 1024));
    upir_status st = ensure_slots(c, (size_t)teams);
    if (st != UPIR_OK) return st;
    a.slots = c->slots;
    a.done = c->done;
    cudaError_t e = launch_stream_loop(dtype == UPIR_I64 ? SB_RED_I64 : SB_RED_F32, PATH_DIRECT, 0, 0, false, teams,
                                       256, 0, a, c->compute);
    if (e != cudaSuccess) return fail(UPIR_E_CUDA, "reduce launch failed: %s", cudaGetErrorString(e));
    c->launches++;
    return UPIR_OK;
  }
  if (scope != UPIR_SCOPE_WORLD) return fail(UPIR_E_INVALID, "bad scope");
  // measurement hook: UPIR_REDUCE_VIA_COMM=1 keeps the communicator path
  const bool via_comm = c->comm && getenv("UPIR_REDUCE_VIA_COMM");
  if (c->nranks > 1 && world_ready(c) && count <= WIN_AR_ELEMS && !via_comm) {
    // every rank's window imported: stage, publish and combine over NVLink
    cudaError_t e = launch_peer_allreduce(c->win, c->nranks, op, dtype, dev_in, count, dev_out, c->compute);
    if (e != cudaSuccess) return fail(UPIR_E_CUDA, "peer allreduce launch failed: %s", cudaGetErrorString(e));
    c->launches++;
    return UPIR_OK;
  }
  // allreduce over ranks (Fig. 7): all-gather of the partials, then the
  // combine in ascending rank order on every rank (deterministic, c10).
  const size_t need = esz * (size_t)count * (size_t)c->nranks;
  if (need > c->scratch_bytes) {
    if (c->capturing) return fail(UPIR_E_INVALID, "scratch must grow during capture");
    if (c->scratch) c->retired.push_back(c->scratch);   // graphs may hold it
    CUDA_TRY(cudaMalloc(&c->scratch, need));
    c->scratch_bytes = need;
  }
  if (c->nranks > 1) {
    if (!c->comm) return fail(UPIR_E_UNSUPPORTED, "upir_reduce(WORLD) needs a communicator (or UPIR_WORLD_REDUCE on a loop)");
    NCCL_TRY(ncclAllGather(dev_in, c->scratch, (size_t)count, dtype == UPIR_I64 ? ncclInt64 : ncclFloat32, c->comm,
                           c->compute));
  } else {
    CUDA_TRY(cudaMemcpyAsync(c->scratch, dev_in, esz * count, cudaMemcpyDeviceToDevice, c->compute));
  }
  cudaError_t e = launch_rank_combine(op, dtype, c->scratch, count, c->nranks, dev_out, c->compute);
  if (e != cudaSuccess) return fail(UPIR_E_CUDA, "combine launch failed: %s", cudaGetErrorString(e));
  c->launches++;
  return UPIR_OK;
}

extern "C" upir_status upir_reduce_async(upir_ctx c, int32_t op, int32_t dtype, const void *dev_in, int64_t count,
                                         void *dev_out, upir_event *token) {
  if (!c || !dev_in || !dev_out || count < 1 || !token) return fail(UPIR_E_INVALID, "bad argument");
  if (*token) return fail(UPIR_E_INVALID, "token out-param must be NULL on entry");
  if (op < UPIR_OP_SUM || op > UPIR_OP_MIN) return fail(UPIR_E_INVALID, "bad op");
  if (dtype != UPIR_I64 && dtype != UPIR_F32) return fail(UPIR_E_INVALID, "dtype must be I64 or F32");
  const bool via_peer = c->nranks > 1 && world_ready(c) && count <= WIN_AR_ELEMS &&
                        !(c->comm && getenv("UPIR_REDUCE_VIA_COMM"));
  if (c->nranks > 1 && !c->comm && !via_peer)
    return fail(UPIR_E_UNSUPPORTED, "upir_reduce_async needs a communicator or every rank's peer window "
                                    "(count <= %lld)", (long long)WIN_AR_ELEMS);
  if (c->sticky != cudaSuccess) return sticky_check(c);
  cudaSetDevice(c->device);
  const size_t esz = dtype == UPIR_I64 ? 8 : 4;
  const size_t need = esz * (size_t)count * (size_t)c->nranks;
  upir_event ev = new upir_event_s();
  if (cudaEventCreateWithFlags(&ev->ev, cudaEventDisableTiming) != cudaSuccess) {
    delete ev;
    return fail(UPIR_E_CUDA, "event create failed");
  }
  auto undo = [&](upir_status st) {
    cudaEventDestroy(ev->ev);
    delete ev;
    return st;
  };
  // arrive-compute: ordered after the compute work so far, on the copy stream
  upir_status st = compute_to_copy(c);
  if (st != UPIR_OK) return undo(st);
  if (via_peer) {
    cudaError_t e = launch_peer_allreduce(c->win, c->nranks, op, dtype, dev_in, count, dev_out, c->copy);
    if (e != cudaSuccess) return undo(fail(UPIR_E_CUDA, "peer allreduce launch failed: %s", cudaGetErrorString(e)));
    c->launches++;
    e = cudaEventRecord(ev->ev, c->copy);
    if (e != cudaSuccess) return undo(fail(UPIR_E_CUDA, "event record: %s", cudaGetErrorString(e)));
    *token = ev;
    return UPIR_OK;
  }
  void *scr = nullptr;
  cudaError_t e = cudaMallocAsync(&scr, need, c->copy);
  if (e != cudaSuccess) return undo(fail(UPIR_E_OOM, "async allreduce scratch: %s", cudaGetErrorString(e)));
  if (c->nranks > 1) {
    ncclResult_t r = ncclAllGather(dev_in, scr, (size_t)count, dtype == UPIR_I64 ? ncclInt64 : ncclFloat32, c->comm,
                                   c->copy);
    if (r != ncclSuccess) {
      cudaFreeAsync(scr, c->copy);
      return undo(fail(UPIR_E_NCCL, "ncclAllGather: %s", ncclGetErrorString(r)));
    }
  } else {
    e = cudaMemcpyAsync(scr, dev_in, esz * count, cudaMemcpyDeviceToDevice, c->copy);
    if (e != cudaSuccess) {
      cudaFreeAsync(scr, c->copy);
      return undo(fail(UPIR_E_CUDA, "gather copy: %s", cudaGetErrorString(e)));
    }
  }
  e = launch_rank_combine(op, dtype, scr, count, c->nranks, dev_out, c->copy);
  cudaFreeAsync(scr, c->copy);
  if (e != cudaSuccess) return undo(fail(UPIR_E_CUDA, "combine launch failed: %s", cudaGetErrorString(e)));
  c->launches++;
  e = cudaEventRecord(ev->ev, c->copy);
  if (e != cudaSuccess) return undo(fail(UPIR_E_CUDA, "event record: %s", cudaGetErrorString(e)));
  *token = ev;
  return UPIR_OK;
}

static upir_status halo_exchange(upir_ctx c, upir_map m, cudaStream_t strm) {
  if (m->dist.pattern != UPIR_PATTERN_BLOCK || m->dist.halo_rows < 1)
    return fail(UPIR_E_INVALID, "HALO needs a BLOCK-distributed map with halo_rows >= 1");
  if (c->nranks == 1) return UPIR_OK;
  if (m->halo_fused) {
    // exchanged inside the peer-mode sweep that wrote it: a later peer-mode
    // sweep waits for the neighbours' deliveries in-kernel, anything else
    // (an explicit sweep, a read-back) needs them here -- drain them in
    // stream order
    const bool up = c->rank > 0 && c->peer_win[c->rank - 1];
    const bool dn = c->rank + 1 < c->nranks && c->rank + 1 < WIN_MAX_RANKS && c->peer_win[c->rank + 1];
    if (up || dn) {
      cudaError_t e = launch_peer_drain(c->win, up, dn, strm);
      if (e != cudaSuccess) return fail(UPIR_E_CUDA, "peer drain launch failed: %s", cudaGetErrorString(e));
      c->launches++;
    }
    return UPIR_OK;
  }
  int64_t plan[8];
  upir_status st = upir_halo_plan(m->dist.n_rows, m->dist.halo_rows, c->rank, c->nranks, plan);
  if (st != UPIR_OK) return st;
  const int64_t rb = m->dist.row_elems * m->dist.elem_bytes;
  char *base = (char *)m->dev;
  auto at = [&](int64_t row) { return base + (row - m->loc_row_lo) * rb; };
  const bool need_up = plan[1] > plan[0], need_dn = plan[5] > plan[4];
  const bool peer_ok = world_ready(c) && (!need_up || m->peer_dev[0]) && (!need_dn || m->peer_dev[1]) &&
                       (m->peer_dev[0] || m->peer_dev[1]);
  if (peer_ok) {
    // peer mappings: my send rows land at the same global rows of the neighbour's buffer
    PeerHaloArgs a;
    memset(&a, 0, sizeof a);
    a.win = c->win;
    if (need_up) {
      a.win_up = c->peer_win[c->rank - 1];
      a.src_up = at(plan[0]);
      a.dst_up = (char *)m->peer_dev[0] + (plan[0] - m->peer_row0[0]) * rb;
      a.bytes_up = (plan[1] - plan[0]) * rb;
    }
    if (need_dn) {
      a.win_dn = c->peer_win[c->rank + 1];
      a.src_dn = at(plan[4]);
      a.dst_dn = (char *)m->peer_dev[1] + (plan[4] - m->peer_row0[1]) * rb;
      a.bytes_dn = (plan[5] - plan[4]) * rb;
    }
    cudaError_t e = launch_peer_halo(a, strm);
    if (e != cudaSuccess) return fail(UPIR_E_CUDA, "peer halo launch failed: %s", cudaGetErrorString(e));
    c->launches++;
    return UPIR_OK;
  }
  if (!c->comm)
    return fail(UPIR_E_UNSUPPORTED,
                "communicator-less world: halos move through imported peer buffers (upir_peer_import) only");
  // Fig. 7 send/recv with rank units, in stream order before the next sweep
  NCCL_TRY(ncclGroupStart());
  if (plan[1] > plan[0]) {
    NCCL_TRY(ncclSend(at(plan[0]), (size_t)((plan[1] - plan[0]) * rb), ncclChar, c->rank - 1, c->comm, strm));
    NCCL_TRY(ncclRecv(at(plan[2]), (size_t)((plan[3] - plan[2]) * rb), ncclChar, c->rank - 1, c->comm, strm));
  }
  if (plan[5] > plan[4]) {
    NCCL_TRY(ncclSend(at(plan[4]), (size_t)((plan[5] - plan[4]) * rb), ncclChar, c->rank + 1, c->comm, strm));
    NCCL_TRY(ncclRecv(at(plan[6]), (size_t)((plan[7] - plan[6]) * rb), ncclChar, c->rank + 1, c->comm, strm));
  }
  NCCL_TRY(ncclGroupEnd());
  return UPIR_OK;
}

extern "C" upir_status upir_sync(upir_ctx c, int32_t kind, upir_map halo_map, upir_event *token) {
  if (!c) return fail(UPIR_E_INVALID, "ctx is NULL");
  cudaSetDevice(c->device);
  switch (kind) {
    case UPIR_SYNC_BARRIER: {
      cudaError_t e1 = cudaStreamSynchronize(c->compute);
      cudaError_t e2 = cudaStreamSynchronize(c->copy);
      if (e1 != cudaSuccess && c->sticky == cudaSuccess) c->sticky = e1;
      if (e2 != cudaSuccess && c->sticky == cudaSuccess) c->sticky = e2;
      if (e1 == cudaSuccess && e2 == cudaSuccess) release_pins(c);
      if (c->comm) {
        ncclResult_t ar;
        if (ncclCommGetAsyncError(c->comm, &ar) == ncclSuccess && ar != ncclSuccess)
          return fail(UPIR_E_NCCL, "NCCL asynchronous error: %s", ncclGetErrorString(ar));
      }
      return sticky_check(c);
    }
    case UPIR_SYNC_WORLD_BARRIER: {
      upir_status st = upir_sync(c, UPIR_SYNC_BARRIER, nullptr, nullptr);
      if (st != UPIR_OK) return st;
      if (c->nranks > 1) {
        if (c->comm) {
          NCCL_TRY(ncclAllReduce(c->one, c->one, 1, ncclInt32, ncclSum, c->comm, c->compute));
        } else if (world_ready(c)) {
          cudaError_t e = launch_peer_barrier(c->win, c->nranks, c->compute);
          if (e != cudaSuccess) return fail(UPIR_E_CUDA, "peer barrier launch failed: %s", cudaGetErrorString(e));
        } else {
          return fail(UPIR_E_UNSUPPORTED, "WORLD_BARRIER needs a communicator or every rank's peer window");
        }
        CUDA_TRY(cudaStreamSynchronize(c->compute));
      }
      return UPIR_OK;
    }
    case UPIR_SYNC_ARRIVE: {
      if (!token) return fail(UPIR_E_INVALID, "ARRIVE needs a token out-param");
      upir_event ev = new upir_event_s();
      if (cudaEventCreateWithFlags(&ev->ev, cudaEventDisableTiming) != cudaSuccess) {
        delete ev;
        return fail(UPIR_E_CUDA, "event create failed");
      }
      upir_status st = copy_to_compute(c);
      if (st != UPIR_OK) { cudaEventDestroy(ev->ev); delete ev; return st; }
      CUDA_TRY(cudaEventRecord(ev->ev, c->compute));
      *token = ev;
      return UPIR_OK;
    }
    case UPIR_SYNC_WAIT: {
      if (!token || !*token) return fail(UPIR_E_SYNC, "WAIT without a matching ARRIVE token");
      upir_event ev = *token;
      cudaError_t e = cudaEventSynchronize(ev->ev);
      cudaEventDestroy(ev->ev);
      delete ev;
      *token = nullptr;
      if (e != cudaSuccess) return fail(UPIR_E_CUDA, "wait failed: %s", cudaGetErrorString(e));
      return sticky_check(c);
    }
    case UPIR_SYNC_HALO: {
      if (!halo_map) return fail(UPIR_E_INVALID, "HALO needs a map");
      upir_status st = check_map(c, halo_map, "halo map");
      if (st != UPIR_OK) return st;
      if (!token) return halo_exchange(c, halo_map, c->compute);
      // async arrive-compute: exchange on the copy stream
      upir_event ev = new upir_event_s();
      if (cudaEventCreateWithFlags(&ev->ev, cudaEventDisableTiming) != cudaSuccess) {
        delete ev;
        return fail(UPIR_E_CUDA, "event create failed");
      }
      st = compute_to_copy(c);
      if (st == UPIR_OK) st = halo_exchange(c, halo_map, c->copy);
      if (st != UPIR_OK) {
        cudaEventDestroy(ev->ev);
        delete ev;
        return st;
      }
      CUDA_TRY(cudaEventRecord(ev->ev, c->copy));
      *token = ev;
      return UPIR_OK;
    }
    case UPIR_SYNC_JOIN: {
      if (!token || !*token) return fail(UPIR_E_SYNC, "JOIN without a matching async token");
      upir_event ev = *token;
      cudaError_t e = cudaStreamWaitEvent(c->compute, ev->ev, 0);
      cudaEventDestroy(ev->ev);   // destruction is deferred until the event completes
      delete ev;
      *token = nullptr;
      if (e != cudaSuccess) return fail(UPIR_E_CUDA, "join failed: %s", cudaGetErrorString(e));
      return UPIR_OK;
    }
  }
  return fail(UPIR_E_INVALID, "unknown sync kind %d", kind);
}

// ------------------------------------------------------------------ graphs
extern "C" upir_status upir_graph_begin(upir_ctx c) {
  if (!c) return fail(UPIR_E_INVALID, "ctx is NULL");
  if (c->capturing) return fail(UPIR_E_INVALID, "already capturing");
  cudaSetDevice(c->device);
  CUDA_TRY(cudaStreamBeginCapture(c->compute, cudaStreamCaptureModeRelaxed));
  c->capturing = true;
  c->launches_at_capture = c->launches;
  return UPIR_OK;
}

extern "C" upir_status upir_graph_end(upir_ctx c, upir_graph *out) {
  if (!c || !out) return fail(UPIR_E_INVALID, "bad argument");
  if (!c->capturing) return fail(UPIR_E_INVALID, "not capturing");
  c->capturing = false;
  upir_graph g = new upir_graph_s();
  // captured kernels did not run: they count when the graph is launched
  g->kernels = c->launches - c->launches_at_capture;
  c->launches = c->launches_at_capture;
  cudaError_t e = cudaStreamEndCapture(c->compute, &g->graph);
  if (e != cudaSuccess) { delete g; return fail(UPIR_E_CUDA, "end capture: %s", cudaGetErrorString(e)); }
  e = cudaGraphInstantiate(&g->exec, g->graph, 0);
  if (e != cudaSuccess) {
    cudaGraphDestroy(g->graph);
    delete g;
    return fail(UPIR_E_CUDA, "instantiate: %s", cudaGetErrorString(e));
  }
  *out = g;
  return UPIR_OK;
}

extern "C" upir_status upir_graph_launch(upir_ctx c, upir_graph g) {
  if (!c || !g) return fail(UPIR_E_INVALID, "bad argument");
  cudaSetDevice(c->device);
  CUDA_TRY(cudaGraphLaunch(g->exec, c->compute));
  c->launches += g->kernels;
  return UPIR_OK;
}

extern "C" upir_status upir_graph_destroy(upir_graph g) {
  if (!g) return fail(UPIR_E_INVALID, "graph is NULL");
  cudaGraphExecDestroy(g->exec);
  cudaGraphDestroy(g->graph);
  delete g;
  return UPIR_OK;
}

// ------------------------------------------------------------------ synthetic inputs
extern "C" upir_status upir_synth_fill(upir_ctx c, upir_map m, int32_t dist, uint64_t stream, int64_t index_base,
                                       int64_t n_rows, int64_t n_cols) {
  if (!c || !m) return fail(UPIR_E_INVALID, "bad argument");
  upir_status st = check_map(c, m, "map");
  if (st != UPIR_OK) return st;
  if (dist < 0 || dist > 4) return fail(UPIR_E_INVALID, "bad dist");
  const int64_t esz = dist == 2 ? 8 : (dist == 3 ? 2 : 4);
  if (dist == 4 && (n_rows < 1 || n_cols < 1)) return fail(UPIR_E_INVALID, "Jacobi fill needs n_rows, n_cols");
  int64_t n, off;
  if (m->dist.pattern == UPIR_PATTERN_BLOCK) {
    if (m->elem_bytes != esz) return fail(UPIR_E_INVALID, "element size mismatch");
    n = m->elems_local;
    off = m->elem_offset;
  } else {
    n = (int64_t)(m->dev_bytes / esz);
    off = 0;
  }
  cudaSetDevice(c->device);
  cudaError_t e = launch_synth_fill(dist, stream, m->dev, n, off + index_base, n_rows, n_cols, c->compute);
  if (e != cudaSuccess) return fail(UPIR_E_CUDA, "fill launch failed: %s", cudaGetErrorString(e));
  c->launches++;
  return UPIR_OK;
}
