// C ABI entry points (include/freqcache_b200.h). Each call validates on the host
// what the reference validates before mutation, launches the device sequence on
// the caller's stream and, where the reference returns scalars, synchronises.
#include <pthread.h>
#include <sched.h>

#include <cctype>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <unordered_map>
#include <vector>

#include <cuda.h>

#include "fc_internal.cuh"

namespace fc {

static thread_local char g_err[512] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int cuda_fail(cudaError_t e, const char* what) {
  set_error("CUDA error %s (%s) in %s", cudaGetErrorName(e), cudaGetErrorString(e), what);
  return FC_ERR_CUDA;
}

struct TraceEv {
  int tag;
  cudaEvent_t ev;
};

void trace_mark(fc_cache* h, int tag, cudaStream_t st) {
  if (!h->trace) return;
  auto* v = static_cast<std::vector<TraceEv>*>(h->trace);
  cudaEvent_t e;
  if (cudaEventCreate(&e) != cudaSuccess) return;
  cudaEventRecord(e, st);
  v->push_back(TraceEv{tag, e});
}

static void trace_clear(fc_cache* h) {
  if (!h->trace) return;
  auto* v = static_cast<std::vector<TraceEv>*>(h->trace);
  for (auto& t : *v) cudaEventDestroy(t.ev);
  delete v;
  h->trace = nullptr;
}

// CPUs attached to the GPU's PCIe root (its NUMA node's cores), from sysfs; empty if unknown.
std::vector<int> device_local_cpus(int device) {
  std::vector<int> cpus;
  char bus[64] = {0};
  if (cudaDeviceGetPCIBusId(bus, sizeof(bus), device) != cudaSuccess) {
    cudaGetLastError();
    return cpus;
  }
  for (char* c = bus; *c; ++c) *c = (char)std::tolower(*c);
  char path[256];
  std::snprintf(path, sizeof(path), "/sys/bus/pci/devices/%s/local_cpulist", bus);
  FILE* f = std::fopen(path, "r");
  if (!f) return cpus;
  char line[4096] = {0};
  if (std::fgets(line, sizeof(line), f)) {
    for (char* tok = std::strtok(line, ",\n"); tok; tok = std::strtok(nullptr, ",\n")) {
      int a = -1, b = -1;
      if (std::sscanf(tok, "%d-%d", &a, &b) == 2) {
        for (int x = a; x <= b; ++x) cpus.push_back(x);
      } else if (std::sscanf(tok, "%d", &a) == 1) {
        cpus.push_back(a);
      }
    }
  }
  std::fclose(f);
  cpu_set_t allowed;  // keep only CPUs this process may run on (containers, taskset)
  if (sched_getaffinity(0, sizeof(allowed), &allowed) == 0) {
    std::vector<int> ok;
    for (int c : cpus)
      if (c >= 0 && c < CPU_SETSIZE && CPU_ISSET(c, &allowed)) ok.push_back(c);
    cpus.swap(ok);
  }
  return cpus;
}

// Bind a thread (0 = the calling thread) to `cpus`; no-op when the list is empty.
void bind_thread(pthread_t t, const std::vector<int>& cpus) {
  if (cpus.empty()) return;
  cpu_set_t set;
  CPU_ZERO(&set);
  for (int c : cpus) CPU_SET(c, &set);
  pthread_setaffinity_np(t, sizeof(set), &set);
}

int ensure_scratch_buf(void** p, size_t* have, size_t bytes) {
  if (bytes <= *have) return FC_OK;
  size_t nb = std::max(bytes, *have + *have / 2);
  if (*p) FC_CUDA(cudaFree(*p));  // synchronising: no kernel still uses the old buffer
  *p = nullptr;
  *have = 0;
  FC_CUDA(cudaMalloc(p, nb));
  *have = nb;
  return FC_OK;
}

int ensure_scratch(fc_cache* h, size_t bytes) { return ensure_scratch_buf(&h->scratch, &h->scratch_bytes, bytes); }

// sync the stream through the handle's event and pull the counters
static int sync_counters(fc_cache* h, cudaStream_t st) {
  FC_CUDA(cudaMemcpyAsync(h->ctr_host, h->ctr, sizeof(Counters), cudaMemcpyDeviceToHost, st));
  FC_CUDA(cudaEventRecord(h->done, st));
  FC_CUDA(cudaEventSynchronize(h->done));
  h->host_free = h->ctr_host->free_count;
  return FC_OK;
}

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

static void release(fc_cache* h) {
  trace_clear(h);
  pipe_release(h);
  engine_release(h);
  void* dev[] = {h->arena, h->wb_stage, h->wb_stage_state, h->scratch};
  for (void* p : dev)
    if (p) cudaFree(p);
  if (h->ctr_host) cudaFreeHost(h->ctr_host);
  if (h->done) cudaEventDestroy(h->done);
  if (h->profile)
    for (int i = 0; i < 4; ++i) cudaEventDestroy(h->pev[i]);
  delete h;
}

}  // namespace fc

using namespace fc;

// Synchronous verbs see the state only after a prefetched prepare is committed.
#define FC_NO_OUTSTANDING(h)                                                          \
  do {                                                                                \
    if (pipe_outstanding(h)) {                                                        \
      set_error("a prefetched prepare is outstanding: call fc_prepare_commit first"); \
      return FC_ERR_BAD_ARG;                                                          \
    }                                                                                 \
  } while (0)

#define FC_TRY(expr)          \
  do {                        \
    int rc__ = (expr);        \
    if (rc__) return rc__;    \
  } while (0)

extern "C" {

const char* fc_last_error(void) { return g_err; }

int fc_host_alloc(int64_t bytes, void** out) {
  if (!out || bytes < 0) return FC_ERR_BAD_ARG;
  *out = nullptr;
  // The pages are faulted in (pinned) by the calling thread, and land on its NUMA node: run
  // the allocation on the current GPU's local CPUs so the slow tier sits next to its GPU
  // (on multi-socket boxes the host scatter and the DMA then stay on one socket).
  int dev = 0;
  cudaGetDevice(&dev);
  const std::vector<int> cpus = device_local_cpus(dev);
  cpu_set_t old;
  const bool have_old = !cpus.empty() && sched_getaffinity(0, sizeof(old), &old) == 0;
  if (have_old) bind_thread(pthread_self(), cpus);
  const cudaError_t e = cudaHostAlloc(out, std::max<int64_t>(bytes, 16), cudaHostAllocMapped | cudaHostAllocPortable);
  if (have_old) sched_setaffinity(0, sizeof(old), &old);
  FC_CUDA(e);
  return FC_OK;
}

int fc_host_free(void* p) {
  if (p) FC_CUDA(cudaFreeHost(p));
  return FC_OK;
}

int fc_create(int64_t num_ids, int64_t capacity, int32_t dim, int32_t state_width, int32_t write_back,
              int32_t evict_mode, int64_t buffer_bytes, int32_t device, fc_cache** out) {
  if (!out) return FC_ERR_BAD_ARG;
  *out = nullptr;
  if (capacity < 1) {
    set_error("capacity must be >= 1");
    return FC_ERR_BAD_ARG;
  }
  if (capacity > num_ids) {
    set_error("capacity %lld exceeds num_ids %lld", (long long)capacity, (long long)num_ids);
    return FC_ERR_BAD_ARG;
  }
  if (num_ids > INT32_MAX - 64 || dim < 1 || state_width < 0 || buffer_bytes < 1 ||
      (write_back != FC_WB_DIRTY_ONLY && write_back != FC_WB_ALWAYS) ||
      (evict_mode != FC_EVICT_OCCUPANCY_AWARE && evict_mode != FC_EVICT_PAPER_LITERAL)) {
    set_error("bad geometry or mode");
    return FC_ERR_BAD_ARG;
  }
  DeviceGuard dg(device);
  fc_cache* h = new fc_cache();
  std::memset(h, 0, sizeof(*h));
  h->num_ids = num_ids;
  h->capacity = (int32_t)capacity;
  h->dim = dim;
  h->sw = state_width;
  h->write_back = write_back;
  h->evict_mode = evict_mode;
  h->buffer_bytes = buffer_bytes;
  h->device = device;
  h->nw_ids = ((num_ids + 31) / 32 + 3) / 4 * 4;
  h->nw_slots = ((capacity + 31) / 32 + 3) / 4 * 4;
  const size_t C = (size_t)capacity;
  int rc = FC_OK;
  Arena ar;
  ar.add(&h->rank_of, num_ids);
  ar.add(&h->rank_to_slot, num_ids);
  ar.add(&h->aux, num_ids);
  ar.add(&h->slot_to_rank, C);
  ar.add(&h->dirty, C);
  ar.add(&h->fast, C * dim);
  if (state_width) ar.add(&h->fast_state, C * state_width);
  ar.add(&h->res_bits, h->nw_ids);
  ar.add(&h->id_bits, h->nw_ids);
  ar.add(&h->miss_bits, h->nw_ids);
  ar.add(&h->prot_bits, h->nw_ids);
  ar.add(&h->free_bits, h->nw_slots);
  ar.add(&h->evicted_ranks, C);
  ar.add(&h->victim_slots, C);
  ar.add(&h->wb_ranks, C);
  ar.add(&h->admitted_ranks, C);
  ar.add(&h->target_slots, C);
  ar.add(&h->block_cnt, kMaxScanBlocks + 1);
  ar.add(&h->block_cnt2, kMaxScanBlocks + 1);
  ar.add(&h->ctr, 1);
  {
    const cudaError_t ea = ar.alloc(&h->arena);
    if (ea != cudaSuccess) {
      rc = cuda_fail(ea, "fc_create: device arrays");
      release(h);
      return rc;
    }
    h->arena_bytes = (int64_t)ar.bytes;
  }
  cudaError_t e = cudaHostAlloc(reinterpret_cast<void**>(&h->ctr_host), sizeof(Counters), cudaHostAllocDefault);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&h->done, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaMemset(h->rank_to_slot, 0xff, num_ids * 4);
  if (e == cudaSuccess) e = cudaMemset(h->slot_to_rank, 0xff, C * 4);
  if (e == cudaSuccess) e = cudaMemset(h->aux, 0, num_ids * 4);
  if (e == cudaSuccess) e = cudaMemset(h->dirty, 0, C);
  if (e == cudaSuccess) e = cudaMemset(h->fast, 0, C * dim * 4);
  if (e == cudaSuccess && state_width) e = cudaMemset(h->fast_state, 0, C * state_width * 4);
  for (uint32_t* b : {h->res_bits, h->id_bits, h->miss_bits, h->prot_bits})
    if (e == cudaSuccess) e = cudaMemset(b, 0, h->nw_ids * 4);
  if (e == cudaSuccess) {  // every slot starts free
    std::vector<uint32_t> fb(h->nw_slots, 0u);
    for (int64_t s = 0; s < capacity; ++s) fb[s >> 5] |= 1u << (s & 31);
    e = cudaMemcpy(h->free_bits, fb.data(), fb.size() * 4, cudaMemcpyHostToDevice);
  }
  if (e == cudaSuccess) {
    Counters c0;
    std::memset(&c0, 0, sizeof(c0));
    c0.free_count = (int32_t)capacity;
    e = cudaMemcpy(h->ctr, &c0, sizeof(c0), cudaMemcpyHostToDevice);
  }
  if (e != cudaSuccess) {
    rc = cuda_fail(e, "fc_create");
    release(h);
    return rc;
  }
  h->host_free = (int32_t)capacity;
  h->live = h->ctr;
  h->ev_src = h->evicted_ranks;
  h->ad_src = h->admitted_ranks;
  *out = h;
  return FC_OK;
}

int fc_destroy(fc_cache* h) {
  if (!h) return FC_OK;
  DeviceGuard dg(h->device);
  cudaDeviceSynchronize();
  release(h);
  return FC_OK;
}

int fc_get_views(fc_cache* h, fc_views* v) {
  if (!h || !v) return FC_ERR_BAD_ARG;
  v->fast_rows = h->fast;
  v->slot_to_rank = h->slot_to_rank;
  v->rank_to_slot = h->rank_to_slot;
  v->dirty = h->dirty;
  v->rank_of = h->rank_of;
  v->fast_state = h->fast_state;
  v->capacity = h->capacity;
  v->num_ids = h->num_ids;
  v->dim = h->dim;
  v->state_width = h->sw;
  return FC_OK;
}

int fc_set_modes(fc_cache* h, int32_t write_back, int32_t evict_mode) {
  if (!h || (write_back != FC_WB_DIRTY_ONLY && write_back != FC_WB_ALWAYS) ||
      (evict_mode != FC_EVICT_OCCUPANCY_AWARE && evict_mode != FC_EVICT_PAPER_LITERAL))
    return FC_ERR_BAD_ARG;
  if (write_back == h->write_back && evict_mode == h->evict_mode) return FC_OK;  // no change: allowed any time
  FC_NO_OUTSTANDING(h);
  h->write_back = write_back;
  h->evict_mode = evict_mode;
  return FC_OK;
}

int64_t fc_free_count(fc_cache* h) { return h ? h->host_free : -1; }

int fc_set_buffer_bytes(fc_cache* h, int64_t buffer_bytes) {
  if (!h || buffer_bytes < 1) return FC_ERR_BAD_ARG;
  if (buffer_bytes == h->buffer_bytes) return FC_OK;
  FC_NO_OUTSTANDING(h);
  h->buffer_bytes = buffer_bytes;
  return FC_OK;
}

int fc_set_engine(fc_cache* h, int32_t engine) {
  if (!h) return FC_ERR_BAD_ARG;
  FC_NO_OUTSTANDING(h);
  DeviceGuard dg(h->device);
  return engine_set(h, engine);
}

int fc_drain(fc_cache* h) {
  if (!h) return FC_ERR_BAD_ARG;
  DeviceGuard dg(h->device);
  return engine_drain(h);
}

int fc_drain_stream(fc_cache* h, void* stream) {
  if (!h) return FC_ERR_BAD_ARG;
  DeviceGuard dg(h->device);
  return engine_drain_stream(h, as_stream(stream));
}

int fc_set_idx_map(fc_cache* h, const int64_t* rank_of_host, void* stream) {
  if (!h || !rank_of_host) return FC_ERR_BAD_ARG;
  DeviceGuard dg(h->device);
  std::vector<int32_t> r((size_t)h->num_ids);
  for (int64_t i = 0; i < h->num_ids; ++i) {
    const int64_t v = rank_of_host[i];
    if (v < 0 || v >= h->num_ids) {
      set_error("rank_of[%lld]=%lld outside [0, %lld)", (long long)i, (long long)v, (long long)h->num_ids);
      return FC_ERR_BAD_ARG;
    }
    r[(size_t)i] = (int32_t)v;
  }
  cudaStream_t st = as_stream(stream);
  FC_CUDA(cudaMemcpyAsync(h->rank_of, r.data(), r.size() * 4, cudaMemcpyHostToDevice, st));
  FC_CUDA(cudaStreamSynchronize(st));
  return FC_OK;
}

int fc_attach_slow_tier(fc_cache* h, float* rows_host, int64_t row_stride, float* state_host, int64_t state_stride) {
  if (!h || !rows_host || row_stride < h->dim) return FC_ERR_BAD_ARG;
  DeviceGuard dg(h->device);
  void* dptr = nullptr;
  cudaError_t e = cudaHostGetDevicePointer(&dptr, rows_host, 0);
  if (e != cudaSuccess) {
    cudaGetLastError();
    set_error("slow tier must live in pinned mapped host memory (fc_host_alloc): %s", cudaGetErrorString(e));
    return FC_ERR_BAD_ARG;
  }
  h->slow = static_cast<float*>(dptr);
  h->slow_host = rows_host;
  h->slow_ld = row_stride;
  if (h->sw) {
    if (!state_host || state_stride < h->sw) {
      set_error("optimizer-state rows required (state_width=%d)", h->sw);
      return FC_ERR_BAD_ARG;
    }
    e = cudaHostGetDevicePointer(&dptr, state_host, 0);
    if (e != cudaSuccess) {
      cudaGetLastError();
      set_error("slow state must be pinned mapped host memory");
      return FC_ERR_BAD_ARG;
    }
    h->slow_state = static_cast<float*>(dptr);
    h->slow_state_host = state_host;
    h->state_ld = state_stride;
  }
  return FC_OK;
}

int fc_warmup(fc_cache* h, int64_t k, void* stream) {
  if (!h) return FC_ERR_BAD_ARG;
  FC_NO_OUTSTANDING(h);
  if (k < 0 || k > h->capacity) {
    set_error("warmup k must be in [0, capacity=%d], got %lld", h->capacity, (long long)k);
    return FC_ERR_BAD_ARG;
  }
  if (h->host_free != h->capacity) {
    set_error("warmup requires an empty cache");
    return FC_ERR_NOT_EMPTY;
  }
  if (k == 0) return FC_OK;
  if (!h->slow) return FC_ERR_NO_SLOW_TIER;
  if ((int64_t)h->dim * 4 > h->buffer_bytes) {
    set_error("row of %d B cannot fit in a %lld B buffer", h->dim * 4, (long long)h->buffer_bytes);
    return FC_ERR_BUFFER_TOO_SMALL;
  }
  DeviceGuard dg(h->device);
  cudaStream_t st = as_stream(stream);
  FC_TRY(pipe_order(h, st));
  // ranks 0..k-1 are contiguous in the slow tier: one DMA copy, no gather
  FC_CUDA(cudaMemcpy2DAsync(h->fast, (size_t)h->dim * 4, h->slow, (size_t)h->slow_ld * 4, (size_t)h->dim * 4, (size_t)k,
                            cudaMemcpyDefault, st));
  if (h->sw)
    FC_CUDA(cudaMemcpy2DAsync(h->fast_state, (size_t)h->sw * 4, h->slow_state, (size_t)h->state_ld * 4,
                              (size_t)h->sw * 4, (size_t)k, cudaMemcpyDefault, st));
  FC_TRY(launch_warmup_state(h, k, st));
  return sync_counters(h, st);
}

int fc_prepare(fc_cache* h, const void* ids, int32_t ids_bytes, int64_t n, int64_t batch_seq, int32_t* uids,
               int32_t* ucnt, int32_t* uranks, int32_t* uslots, int32_t* inverse, void* stream, fc_prepare_info* info) {
  (void)batch_seq;
  if (!h || !info || (ids_bytes != 4 && ids_bytes != 8) || n < 0 || n > INT32_MAX) return FC_ERR_BAD_ARG;
  FC_NO_OUTSTANDING(h);
  std::memset(info, 0, sizeof(*info));
  info->free_count = h->host_free;
  if (n == 0) return FC_OK;
  if (!h->slow) return FC_ERR_NO_SLOW_TIER;
  DeviceGuard dg(h->device);
  cudaStream_t st = as_stream(stream);
  FC_TRY(pipe_order(h, st));
  FC_TRY(engine_begin(h, st));
  pipe_forget_sort_hist(h, inverse);  // this inverse buffer gets new contents, without histograms
  FC_TRY(launch_prepare(h, ids, ids_bytes, n, uids, ucnt, uranks, uslots, inverse, st));
  h->ev_src = h->evicted_ranks;
  h->ad_src = h->admitted_ranks;
  h->last_wb_dev = nullptr;
  FC_TRY(sync_counters(h, st));
  FC_TRY(engine_after_prepare(h, st));
  const Counters& c = *h->ctr_host;
  info->unique = c.unique;
  info->free_count = c.free_count;
  info->candidates = c.candidates;
  h->last_needed = 0;
  h->last_misses = 0;
  switch (c.err) {
    case FC_OK:
      break;
    case FC_ERR_ID_OUT_OF_RANGE:
      info->bad_id = (c.lo != LLONG_MAX) ? c.lo : c.hi;
      set_error("id out of range: %lld not in [0, %lld)", (long long)info->bad_id, (long long)h->num_ids);
      return c.err;
    case FC_ERR_BATCH_EXCEEDS_CAPACITY:
      set_error("batch has %d unique ids but the fast tier holds %d; the cache ratio is too small for this batch",
                c.unique, h->capacity);
      return c.err;
    case FC_ERR_INSUFFICIENT_FREE_SLOTS:
      set_error("%d rows to admit but only %d free slots (evict_mode='paper_literal' left the tier over-full)",
                c.misses, c.free_count + c.needed);
      return c.err;
    case FC_ERR_INSUFFICIENT_EVICTABLE:
      set_error("need %d victims but only %d evictable rows", c.needed, c.candidates);
      return c.err;
    case FC_ERR_BUFFER_TOO_SMALL:
      set_error("row of %d B cannot fit in a %lld B buffer", h->dim * 4, (long long)h->buffer_bytes);
      return c.err;
    default:
      set_error("internal error %d in prepare", c.err);
      return c.err;
  }
  info->misses = c.misses;
  info->hits = c.unique - c.misses;
  info->evictions = c.needed;
  info->rows_to_slow = c.wb_rows;
  h->last_needed = c.needed;
  h->last_misses = c.misses;
  if (h->profile) {
    float a = 0.f, b = 0.f;
    cudaEventElapsedTime(&a, h->pev[0], h->pev[3]);
    cudaEventElapsedTime(&b, h->pev[1], h->pev[2]);
    h->prof[0] += a;
    h->prof[1] += b;
    h->prof[2] += 1;
    // bytes the bracketed kernel moves over the host link: both directions for the
    // paired engine 0; admissions only for engine 1 (its write-back rides the copy engine)
    h->prof[3] += 4.0 * (h->dim + h->sw) * ((double)c.misses + (h->engine == 1 ? 0 : c.wb_rows));
    h->prof[4] += 4.0 * (h->dim + h->sw) * (double)c.wb_rows;
  }
  return FC_OK;
}

int fc_prepare_begin(fc_cache* h, const void* ids, int32_t ids_bytes, int64_t n, int64_t batch_seq, int32_t* uids,
                     int32_t* ucnt, int32_t* uranks, int32_t* uslots, int32_t* inverse, void* stream) {
  (void)batch_seq;
  if (!h || (ids_bytes != 4 && ids_bytes != 8) || n < 1 || n > INT32_MAX) return FC_ERR_BAD_ARG;
  if (!h->slow) return FC_ERR_NO_SLOW_TIER;
  DeviceGuard dg(h->device);
  return pipe_begin(h, ids, ids_bytes, n, uids, ucnt, uranks, uslots, inverse, as_stream(stream));
}

int fc_prepare_commit(fc_cache* h, void* stream, fc_prepare_info* info) {
  if (!h || !info) return FC_ERR_BAD_ARG;
  DeviceGuard dg(h->device);
  const int rc = pipe_commit(h, as_stream(stream), info);
  switch (rc) {
    case FC_OK:
      break;
    case FC_ERR_ID_OUT_OF_RANGE:
      set_error("id out of range: %lld not in [0, %lld)", (long long)info->bad_id, (long long)h->num_ids);
      break;
    case FC_ERR_BATCH_EXCEEDS_CAPACITY:
      set_error("batch has %lld unique ids but the fast tier holds %d; the cache ratio is too small for this batch",
                (long long)info->unique, h->capacity);
      break;
    case FC_ERR_BUFFER_TOO_SMALL:
      set_error("row of %d B cannot fit in a %lld B buffer", h->dim * 4, (long long)h->buffer_bytes);
      break;
    case FC_ERR_INSUFFICIENT_FREE_SLOTS:
    case FC_ERR_INSUFFICIENT_EVICTABLE:
      set_error("not enough free or evictable slots for this batch");
      break;
    default:
      break;
  }
  return rc;
}

int fc_memory_bytes(fc_cache* h, int64_t* out, int32_t n_out) {
  if (!h || !out || n_out < FC_MEM_FIELDS) return FC_ERR_BAD_ARG;
  int64_t e[7];
  engine_memory(h, e);
  const int64_t C = h->capacity, N = h->num_ids;
  const int64_t wb0 = h->wb_stage ? 4 * C * (int64_t)(h->dim + (h->wb_stage_state ? h->sw : 0)) : 0;
  int64_t v[FC_MEM_FIELDS] = {};
  v[FC_MEM_FAST_ROWS] = 4 * C * (int64_t)(h->dim + (h->fast_state ? h->sw : 0));
  v[FC_MEM_ID_SPACE] = 3 * 4 * N + e[1];  // rank_of, rank_to_slot, aux (+ pending marks)
  v[FC_MEM_BITMAPS] = 4 * 4 * h->nw_ids + 4 * h->nw_slots;
  v[FC_MEM_STAGING] = e[0] + wb0;
  v[FC_MEM_SCRATCH] = (int64_t)h->scratch_bytes;
  // what the allocations reserve: the arenas and the separately grown buffers in 2 MiB pages
  int64_t reserved = reserved_bytes(h->arena_bytes) + e[6] + reserved_bytes(v[FC_MEM_SCRATCH]);
  if (h->wb_stage) reserved += reserved_bytes(4 * C * (int64_t)h->dim);
  if (h->wb_stage_state) reserved += reserved_bytes(4 * C * (int64_t)h->sw);
  // slot tables, per-slot lists, counters and the 256-byte padding of the arenas' parts
  v[FC_MEM_SLOT_SPACE] = h->arena_bytes - v[FC_MEM_FAST_ROWS] - 3 * 4 * N - v[FC_MEM_BITMAPS] + e[2];
  int64_t sum = 0;
  for (int i = 0; i < FC_MEM_ALLOC_SLACK; ++i) sum += v[i];
  v[FC_MEM_ALLOC_SLACK] = reserved - sum;
  v[FC_MEM_TOTAL_DEVICE] = reserved;
  v[FC_MEM_PINNED_STAGING] = e[3];
  v[FC_MEM_WB_STAGE_ROWS] = e[4];
  v[FC_MEM_ADMIT_STAGE_ROWS] = e[5];
  for (int i = 0; i < FC_MEM_FIELDS; ++i) out[i] = v[i];
  return FC_OK;
}

int fc_last_writebacks(fc_cache* h, int64_t* rows) {
  if (!h || !rows) return FC_ERR_BAD_ARG;
  DeviceGuard dg(h->device);
  *rows = 0;
  if (!h->last_wb_dev) return FC_OK;
  int32_t v = 0;
  FC_TRY(pipe_sync_commits(h));  // the commit's kernels have run
  FC_CUDA(cudaMemcpy(&v, h->last_wb_dev, sizeof(v), cudaMemcpyDeviceToHost));
  *rows = v;
  return FC_OK;
}

int fc_trace(fc_cache* h, int32_t enable) {
  if (!h) return FC_ERR_BAD_ARG;
  DeviceGuard dg(h->device);
  trace_clear(h);
  if (enable) h->trace = new std::vector<TraceEv>();
  return FC_OK;
}

int fc_trace_mark(fc_cache* h, int32_t tag, void* stream) {
  if (!h) return FC_ERR_BAD_ARG;
  DeviceGuard dg(h->device);
  trace_mark(h, tag, as_stream(stream));
  return FC_OK;
}

int64_t fc_trace_read(fc_cache* h, int32_t* tags, double* ms, int64_t max) {
  if (!h || !h->trace) return 0;
  DeviceGuard dg(h->device);
  auto* v = static_cast<std::vector<TraceEv>*>(h->trace);
  const int64_t n = std::min<int64_t>(max, (int64_t)v->size());
  for (int64_t i = 0; i < n; ++i) {
    cudaEventSynchronize((*v)[i].ev);
    float t = 0.f;
    cudaEventElapsedTime(&t, (*v)[0].ev, (*v)[i].ev);
    tags[i] = (*v)[i].tag;
    ms[i] = t;
  }
  return n;
}

int fc_profile(fc_cache* h, int32_t enable, double* out) {
  if (!h) return FC_ERR_BAD_ARG;
  DeviceGuard dg(h->device);
  if (out) {
    for (int i = 0; i < 6; ++i) out[i] = h->prof[i];
    double es[4];
    engine_stats(h, es);
    out[6] = es[0];
    out[7] = es[1];
    out[8] = h->prof[6];
    out[9] = es[2];
    out[10] = es[3];
    out[11] = (double)engine_threads(h);
  }
  if (enable && !h->profile) {
    for (int i = 0; i < 4; ++i) FC_CUDA(cudaEventCreate(&h->pev[i]));
  }
  if (!enable && h->profile) {
    for (int i = 0; i < 4; ++i) cudaEventDestroy(h->pev[i]);
  }
  h->profile = enable ? 1 : 0;
  for (int i = 0; i < 8; ++i) h->prof[i] = 0;
  return FC_OK;
}

int fc_last_events(fc_cache* h, int64_t* evicted_host, int64_t* admitted_host, void* stream) {
  if (!h) return FC_ERR_BAD_ARG;
  DeviceGuard dg(h->device);
  cudaStream_t st = as_stream(stream);
  std::vector<int32_t> a((size_t)h->last_needed), b((size_t)h->last_misses);
  if (!a.empty()) FC_CUDA(cudaMemcpyAsync(a.data(), h->ev_src, a.size() * 4, cudaMemcpyDeviceToHost, st));
  if (!b.empty()) FC_CUDA(cudaMemcpyAsync(b.data(), h->ad_src, b.size() * 4, cudaMemcpyDeviceToHost, st));
  FC_CUDA(cudaStreamSynchronize(st));
  for (size_t i = 0; i < a.size(); ++i) evicted_host[i] = a[i];
  for (size_t i = 0; i < b.size(); ++i) admitted_host[i] = b[i];
  return FC_OK;
}

int fc_flush(fc_cache* h, void* stream, int64_t* rows_written) {
  if (!h) return FC_ERR_BAD_ARG;
  FC_NO_OUTSTANDING(h);
  if (!h->slow) return FC_ERR_NO_SLOW_TIER;
  DeviceGuard dg(h->device);
  cudaStream_t st = as_stream(stream);
  FC_TRY(pipe_order(h, st));
  FC_TRY(engine_drain(h));  // queued write-backs land before flush's own
  FC_TRY(launch_reset_counters(h, st));
  FC_TRY(launch_flush(h, st));
  FC_TRY(sync_counters(h, st));
  if (rows_written) *rows_written = h->ctr_host->flush_rows;
  return FC_OK;
}

int fc_mark_dirty(fc_cache* h, const int64_t* slots, int64_t n, void* stream) {
  if (!h || n < 0) return FC_ERR_BAD_ARG;
  FC_NO_OUTSTANDING(h);
  if (n == 0) return FC_OK;
  DeviceGuard dg(h->device);
  cudaStream_t st = as_stream(stream);
  FC_TRY(pipe_order(h, st));
  FC_TRY(launch_mark_dirty(h, slots, n, st));
  FC_TRY(sync_counters(h, st));
  if (h->ctr_host->err) {
    set_error("slot out of range [0, %d)", h->capacity);
    return FC_ERR_SLOT_OUT_OF_RANGE;
  }
  return FC_OK;
}

int fc_select_evictions(fc_cache* h, int64_t needed, const int64_t* prot, int64_t nprot, int64_t* slots_host,
                        void* stream) {
  if (!h || needed < 0 || nprot < 0) return FC_ERR_BAD_ARG;
  FC_NO_OUTSTANDING(h);
  if (needed == 0) return FC_OK;
  DeviceGuard dg(h->device);
  cudaStream_t st = as_stream(stream);
  FC_TRY(pipe_order(h, st));
  FC_TRY(launch_select_evictions(h, needed, prot, nprot, st));
  FC_TRY(sync_counters(h, st));
  if (h->ctr_host->err) {
    set_error("need %lld victims but only %d evictable rows", (long long)needed, h->ctr_host->candidates);
    return h->ctr_host->err;
  }
  std::vector<int32_t> v((size_t)needed);
  FC_CUDA(cudaMemcpy(v.data(), h->victim_slots, v.size() * 4, cudaMemcpyDeviceToHost));
  for (size_t i = 0; i < v.size(); ++i) slots_host[i] = v[i];
  return FC_OK;
}

int fc_pooled_forward(fc_cache* h, const int32_t* uslots, const int32_t* inv, int64_t n, const void* offsets,
                      int32_t off_bytes, int64_t nbags, int32_t include_last, const float* psw, int32_t mode,
                      float* out, void* stream) {
  if (!h || (mode != FC_POOL_SUM && mode != FC_POOL_MEAN) || (offsets && off_bytes != 4 && off_bytes != 8))
    return FC_ERR_BAD_ARG;
  DeviceGuard dg(h->device);
  return launch_pool(h, uslots, inv, n, offsets, off_bytes, nbags, include_last, psw, mode, out, as_stream(stream));
}

int fc_gather_rows(fc_cache* h, const int32_t* slots, int64_t n, float* out, void* stream) {
  if (!h) return FC_ERR_BAD_ARG;
  DeviceGuard dg(h->device);
  return launch_gather_rows(h, slots, n, out, as_stream(stream));
}

int fc_pool_to_peers(fc_cache* h, const int32_t* uslots, const int32_t* inv, int64_t n, const int64_t* seg_dev,
                     int32_t world, float* const* dst_ptrs_dev, const int64_t* dst_off_dev, void* stream) {
  if (!h || world < 1 || world > 64 || n < 0) return FC_ERR_BAD_ARG;
  DeviceGuard dg(h->device);
  return launch_pool_to_peers(h, uslots, inv, n, seg_dev, world, dst_ptrs_dev, dst_off_dev, as_stream(stream));
}

int fc_gather_from_peers(const float* const* src_ptrs_dev, const int64_t* src_off_dev, const int64_t* seg_dev,
                         int32_t world, int64_t n, int32_t dim, float* out, void* stream) {
  if (world < 1 || world > 64 || n < 0 || dim < 1 || dim % 4) return FC_ERR_BAD_ARG;
  return launch_gather_from_peers(src_ptrs_dev, src_off_dev, seg_dev, world, n, dim, out, as_stream(stream));
}

int fc_pool_cols_to_peers(fc_cache* h, const int32_t* uslots, const int32_t* inv, int64_t n, const int64_t* seg_dev,
                          int32_t world, float* const* dst_ptrs_dev, const int64_t* dst_off_dev, int64_t ld,
                          int64_t col, const float* psw, void* stream) {
  if (!h || world < 1 || world > 64 || n < 0 || ld < 1 || col < 0) return FC_ERR_BAD_ARG;
  DeviceGuard dg(h->device);
  return launch_pool_cols_to_peers(h, uslots, inv, n, seg_dev, world, dst_ptrs_dev, dst_off_dev, ld, col, psw,
                                   as_stream(stream));
}

int fc_gather_cols_from_peers(const float* const* src_ptrs_dev, const int64_t* src_off_dev, const int64_t* seg_dev,
                              int32_t world, int64_t n, int32_t dim, int64_t ld, int64_t col, float* out,
                              void* stream) {
  if (world < 1 || world > 64 || n < 0 || dim < 1 || ld < 1 || col < 0) return FC_ERR_BAD_ARG;
  return launch_gather_cols_from_peers(src_ptrs_dev, src_off_dev, seg_dev, world, n, dim, ld, col, out,
                                       as_stream(stream));
}

// A CUDA IPC handle names a whole cudaMalloc allocation and cudaIpcOpenMemHandle maps its
// BASE; a pointer inside a caching allocator's segment (torch) sits at an offset from it.
// The exported handle therefore carries that offset, and the importer adds it back.
struct IpcHandle {
  cudaIpcMemHandle_t h;
  int64_t offset;
};
static_assert(sizeof(IpcHandle) <= FC_IPC_HANDLE_BYTES, "IPC handle size");

typedef CUresult (*AddrRangeFn)(CUdeviceptr*, size_t*, CUdeviceptr);
static AddrRangeFn addr_range_fn() {
  static AddrRangeFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return reinterpret_cast<AddrRangeFn>(p);
  }();
  return fn;
}

static std::mutex g_ipc_m;
static std::unordered_map<void*, void*> g_ipc_base;  // opened pointer -> mapped base (for close)

int fc_ipc_handle(void* dev_ptr, void* handle_out) {
  if (!dev_ptr || !handle_out) return FC_ERR_BAD_ARG;
  IpcHandle x;
  std::memset(&x, 0, sizeof(x));
  FC_CUDA(cudaIpcGetMemHandle(&x.h, dev_ptr));
  CUdeviceptr base = 0;
  size_t size = 0;
  AddrRangeFn fn = addr_range_fn();
  if (!fn || fn(&base, &size, reinterpret_cast<CUdeviceptr>(dev_ptr)) != CUDA_SUCCESS) {
    set_error("cuMemGetAddressRange failed for the IPC export");
    return FC_ERR_CUDA;
  }
  x.offset = (int64_t)(reinterpret_cast<CUdeviceptr>(dev_ptr) - base);
  std::memset(handle_out, 0, FC_IPC_HANDLE_BYTES);
  std::memcpy(handle_out, &x, sizeof(x));
  return FC_OK;
}

int fc_ipc_open(const void* handle, int32_t device, void** dev_ptr_out) {
  if (!handle || !dev_ptr_out) return FC_ERR_BAD_ARG;
  DeviceGuard dg(device);
  IpcHandle x;
  std::memcpy(&x, handle, sizeof(x));
  void* base = nullptr;
  FC_CUDA(cudaIpcOpenMemHandle(&base, x.h, cudaIpcMemLazyEnablePeerAccess));
  *dev_ptr_out = static_cast<char*>(base) + x.offset;
  std::lock_guard<std::mutex> lk(g_ipc_m);
  g_ipc_base[*dev_ptr_out] = base;
  return FC_OK;
}

int fc_ipc_close(void* dev_ptr) {
  if (!dev_ptr) return FC_OK;
  void* base = dev_ptr;
  {
    std::lock_guard<std::mutex> lk(g_ipc_m);
    auto it = g_ipc_base.find(dev_ptr);
    if (it != g_ipc_base.end()) {
      base = it->second;
      g_ipc_base.erase(it);
    }
  }
  FC_CUDA(cudaIpcCloseMemHandle(base));
  return FC_OK;
}

int fc_apply_unique_update(fc_cache* h, const int32_t* uslots, int64_t u, const float* add, void* stream) {
  if (!h) return FC_ERR_BAD_ARG;
  DeviceGuard dg(h->device);
  return launch_unique_add(h, uslots, u, add, as_stream(stream));
}

int fc_apply_synthetic_update(fc_cache* h, const int32_t* uids, const int32_t* ucnt, const int32_t* uslots, int64_t u,
                              uint64_t salt, const float* colw, void* stream) {
  if (!h) return FC_ERR_BAD_ARG;
  DeviceGuard dg(h->device);
  return launch_synthetic(h, uids, ucnt, uslots, u, salt, colw, as_stream(stream));
}

int fc_scatter_update(fc_cache* h, const int32_t* uslots, const int32_t* inv, const int32_t* ucnt, int64_t u, int64_t n,
                      const float* deltas, void* stream) {
  if (!h) return FC_ERR_BAD_ARG;
  DeviceGuard dg(h->device);
  return launch_scatter_update(h, uslots, inv, ucnt, u, n, deltas, as_stream(stream));
}

int fc_backward_update(fc_cache* h, const int32_t* uslots, const int32_t* inv, const int32_t* ucnt, int64_t u, int64_t n,
                       const void* offsets, int32_t off_bytes, int64_t nbags, int32_t include_last, const float* psw,
                       int32_t mode, const float* grad, int32_t optim, float lr, float eps, void* stream) {
  if (!h || (optim != FC_OPT_SGD && optim != FC_OPT_ADAGRAD) || (offsets && off_bytes != 4 && off_bytes != 8))
    return FC_ERR_BAD_ARG;
  DeviceGuard dg(h->device);
  cudaStream_t st = as_stream(stream);
  FC_TRY(launch_backward(h, uslots, inv, ucnt, u, n, offsets, off_bytes, nbags, include_last, psw, mode, grad, optim,
                         lr, eps, st));
  return pipe_launch_xfer(h, st, true);  // deferred miss staging of a prefetched batch runs after this update
}

}  // extern "C"
