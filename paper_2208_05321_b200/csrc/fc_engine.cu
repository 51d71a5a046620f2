// Async write-back engine (engine 1).
//
// The paired zero-copy kernel (engine 0, fc_rows.cu) moves victims and admissions
// with SM loads/stores over PCIe; concurrent SM-issued reads and writes top out near
// 75 GB/s on this box (tools/zerocopy_bench.cu) where the DMA engines reach ~100.
// Engine 1 takes the write-back direction off the SMs and off the critical path:
//
//   prepare t:  victims' dirty rows are compacted into HBM stage[b] (b rotates over
//               kWbBufs buffers, one per prepare that wrote rows back) and marked
//               pending[rank] = (b, k); admissions read their row from the newest
//               copy: the HBM stage when the rank is pending, else the pinned slow
//               tier (TMA bulk copies or SM loads over the host link);
//   after sync: stage[b] (+ ranks) goes D2H by cudaMemcpyAsync on a side stream
//               into pinned staging, and a host thread pool scatters the rows into
//               the slow tier at their ranks — overlapped with the pooled forward /
//               backward of step t and the index work of step t+1;
//   the next prepare that reuses stage[b] (kWbBufs write-backs later) waits for that
//               job, then clears the pending marks that still point into stage[b].
//
// Jobs run strictly FIFO so a rank written back twice lands its newest value last.
// `flush` drains every job before its own write-back, so after flush the slow tier
// is authoritative exactly as in the reference.
#include <emmintrin.h>

#include <algorithm>
#include <cmath>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <deque>
#include <mutex>
#include <thread>
#include <vector>

#include <climits>

#include <cuda.h>

#include "fc_rowutil.cuh"
#include "fc_tma.cuh"

namespace fc {

// FC_DEBUG_WAITS=1: report host waits longer than 5 ms on stderr (diagnostics)
static void slow_wait_note(const char* what, std::chrono::steady_clock::time_point t0) {
  static const bool on = std::getenv("FC_DEBUG_WAITS") != nullptr;
  if (!on) return;
  const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  if (ms > 5.0) fprintf(stderr, "[freqcache] slow host wait %.1f ms: %s\n", ms, what);
}

// Write-back stage buffers in rotation: a host scatter job may lag this many commits
// behind before a stage reuse has to wait for it (absorbs host-thread jitter).
constexpr int kWbBufs = 4;

struct Job {
  int buf;
  int64_t rows;      // -1: a pipeline commit's count is on device (d2h[buf] brings it back)
  uint64_t seq;
  int64_t victims = 0;  // pipeline commit: rows the stage may hold (every victim)
  bool shipped = false; // pipeline commit: all `victims` rows already queued D2H behind the commit
  bool copied = false;  // the copier issued the rows' D2H itself (cev[buf] marks its end)
};

struct AsyncWB {
  int32_t* pending = nullptr;   // device int32[num_ids], -1 or buf*rows + k
  int32_t rows = 0;             // rows per write-back stage buffer (grown on demand, engine_grow)
  void* fixed_arena = nullptr;  // pending marks + dev_rows
  int64_t fixed_bytes = 0;
  void* stage_arena = nullptr;  // every stage / sstage / sranks buffer
  int64_t stage_bytes = 0;
  int grows = 0;
  float* stage[kWbBufs] = {};
  float* sstage[kWbBufs] = {};
  int32_t* sranks[kWbBufs] = {};
  float* hstage[kWbBufs] = {};   // pinned
  float* hsstage[kWbBufs] = {};
  int32_t* hranks[kWbBufs] = {};
  volatile uint32_t* done_host = nullptr;  // pinned mapped: last finished job's sequence number
  CUdeviceptr done_dev = 0;                // its device address (stream wait-value target)
  int32_t* dev_rows = nullptr;             // device int32[kWbBufs]: rows staged by a pipeline commit
  int32_t* hrows = nullptr;                // pinned int32[kWbBufs]: their D2H copies
  int64_t rows_in[kWbBufs] = {};           // rows currently staged in each buffer (upper bound)
  bool rows_on_dev[kWbBufs] = {};          // the exact count is dev_rows[b]
  uint64_t seq_of[kWbBufs] = {};           // job sequence number using each buffer
  cudaStream_t side = nullptr;
  cudaStream_t dside = nullptr;            // the dispatcher's own D2H stream (exact-size write-back copies)
  cudaEvent_t d2h[kWbBufs] = {};
  cudaEvent_t cev[kWbBufs] = {};           // end of the copier's exact-size D2H of a buffer's job
  int cur = 0;
  int device = 0;
  bool vec = true;                         // rows move as 16-byte units (dim % 4 == 0, aligned)

  // FIFO scatter jobs, one dispatcher + helpers
  std::mutex m;
  std::condition_variable cv_q, cv_done, cv_help, cv_helped;
  std::deque<Job> q;       // jobs whose rows are (being) copied, in order: the dispatcher scatters them
  std::deque<Job> qc;      // jobs in commit order: the copier ships their rows D2H
  std::condition_variable cv_qc;
  uint64_t next_seq = 1, done_seq = 0, started_seq = 0;
  std::condition_variable cv_started;
  bool stop = false;
  bool copier_done = false;  // the copier has exited (everything it queued is in q)
  bool helpers_stop = false; // set after the dispatcher has exited
  std::thread dispatcher;
  std::thread copier;
  std::vector<std::thread> helpers;
  // parallel-for state
  uint64_t gen = 0;
  int helpers_left = 0;
  std::atomic<int64_t> next_row{0};
  const float* src = nullptr;
  const float* ssrc = nullptr;
  const int32_t* ranks = nullptr;
  int64_t nrows = 0;
  fc_cache* h = nullptr;
  double scatter_ms = 0;  // host scatter time (stats, under m)
  int64_t jobs_done = 0;
  double dirty_frac = 1.0;  // recent dirty share of the victims (pipeline commits; under m)
  int threads = 0;          // host scatter threads (dispatcher + helpers)
  int64_t rows_done = 0;  // rows written back to the slow tier (stats, under m)
  int64_t d2h_bytes = 0;  // bytes shipped device -> host for them (stats, under m)
};

void engine_stats(fc_cache* h, double* out) {
  AsyncWB* a = h->awb;
  if (!a) {
    out[0] = out[1] = out[2] = out[3] = 0;
    return;
  }
  std::lock_guard<std::mutex> lk(a->m);
  out[0] = a->scatter_ms;
  out[1] = (double)a->jobs_done;
  out[2] = (double)a->rows_done;
  out[3] = (double)a->d2h_bytes;
  a->scatter_ms = 0;
  a->jobs_done = 0;
  a->rows_done = 0;
  a->d2h_bytes = 0;
}


// ------------------------------------------------------------------ host scatter
// Rows land at scattered ranks of a table far larger than the caches: stream them
// with non-temporal 16-byte stores (no read-for-ownership of the destination lines).
static inline void copy_row_nt(float* dst, const float* src, int64_t n) {
  if (((reinterpret_cast<uintptr_t>(dst) | reinterpret_cast<uintptr_t>(src)) & 15) == 0 && n % 4 == 0) {
    __m128i* d = reinterpret_cast<__m128i*>(dst);
    const __m128i* s = reinterpret_cast<const __m128i*>(src);
    for (int64_t k = 0; k < n / 4; ++k) _mm_stream_si128(d + k, _mm_load_si128(s + k));
  } else {
    std::memcpy(dst, src, (size_t)n * 4);
  }
}

static void scatter_range(AsyncWB* a) {
  fc_cache* h = a->h;
  constexpr int64_t kGrain = 128;
  while (true) {
    const int64_t i0 = a->next_row.fetch_add(kGrain);
    if (i0 >= a->nrows) break;
    const int64_t i1 = std::min(a->nrows, i0 + kGrain);
    for (int64_t i = i0; i < i1; ++i) {
      const int64_t r = a->ranks[i];
      if (i + 4 < i1) __builtin_prefetch(h->slow_host + a->ranks[i + 4] * h->slow_ld, 1, 0);
      copy_row_nt(h->slow_host + r * h->slow_ld, a->src + i * h->dim, h->dim);
      if (h->sw) copy_row_nt(h->slow_state_host + r * h->state_ld, a->ssrc + i * h->sw, h->sw);
    }
  }
  _mm_sfence();  // make the streaming stores visible before the job is marked done
}

static void helper_main(AsyncWB* a) {
  uint64_t seen = 0;
  std::unique_lock<std::mutex> lk(a->m);
  while (true) {
    a->cv_help.wait(lk, [&] { return a->helpers_stop || a->gen != seen; });
    if (a->gen == seen) return;  // helpers_stop and no new work
    seen = a->gen;
    lk.unlock();
    scatter_range(a);
    lk.lock();
    if (--a->helpers_left == 0) a->cv_helped.notify_all();
  }
}

// Copier: jobs in commit order. A pipeline commit's dirty filter ran on device and only
// its row count came back (d2h[buf]); the copier then ships exactly those rows -- not
// every victim -- on its own stream, so job j+1's copy overlaps job j's host scatter.
static void copier_main(AsyncWB* a) {
  cudaSetDevice(a->device);
  fc_cache* h = a->h;
  std::unique_lock<std::mutex> lk(a->m);
  while (true) {
    a->cv_qc.wait(lk, [&] { return a->stop || !a->qc.empty(); });
    if (a->stop && a->qc.empty()) {
      a->copier_done = true;
      a->cv_q.notify_all();
      return;
    }
    Job j = a->qc.front();
    a->qc.pop_front();
    lk.unlock();
    const auto tw = std::chrono::steady_clock::now();
    cudaEventSynchronize(a->d2h[j.buf]);  // the staged rows (sync prepare) or their count (pipeline) are in pinned memory
    slow_wait_note("copier: write-back count / D2H event", tw);
    if (j.rows < 0) {
      const int b = j.buf;
      j.rows = a->hrows[b];
      if (j.rows > 0 && !j.shipped) {
        cudaMemcpyAsync(a->hranks[b], a->sranks[b], (size_t)j.rows * 4, cudaMemcpyDeviceToHost, a->dside);
        cudaMemcpyAsync(a->hstage[b], a->stage[b], (size_t)j.rows * h->dim * 4, cudaMemcpyDeviceToHost, a->dside);
        if (h->sw)
          cudaMemcpyAsync(a->hsstage[b], a->sstage[b], (size_t)j.rows * h->sw * 4, cudaMemcpyDeviceToHost, a->dside);
        cudaEventRecord(a->cev[b], a->dside);
        j.copied = true;
      }
    }
    lk.lock();
    if (j.victims > 0) a->dirty_frac = 0.75 * a->dirty_frac + 0.25 * (double)j.rows / (double)j.victims;
    a->started_seq = j.seq;  // d2h[j.buf] / hrows[j.buf] may be re-recorded from here on
    a->cv_started.notify_all();
    a->q.push_back(j);
    a->cv_q.notify_one();
  }
}

static void dispatcher_main(AsyncWB* a) {
  cudaSetDevice(a->device);
  std::unique_lock<std::mutex> lk(a->m);
  while (true) {
    a->cv_q.wait(lk, [&] { return a->copier_done || !a->q.empty(); });
    if (a->copier_done && a->q.empty()) return;
    Job j = a->q.front();
    a->q.pop_front();
    lk.unlock();
    if (j.copied) {
      const auto tw = std::chrono::steady_clock::now();
      cudaEventSynchronize(a->cev[j.buf]);
      slow_wait_note("dispatcher: write-back D2H", tw);
    }
    lk.lock();
    a->src = a->hstage[j.buf];
    a->ssrc = a->hsstage[j.buf];
    a->ranks = a->hranks[j.buf];
    a->nrows = j.rows;
    a->next_row.store(0);
    a->helpers_left = (int)a->helpers.size();
    ++a->gen;
    a->cv_help.notify_all();
    lk.unlock();
    const auto t0 = std::chrono::steady_clock::now();
    scatter_range(a);
    lk.lock();
    a->cv_helped.wait(lk, [&] { return a->helpers_left == 0; });
    a->scatter_ms += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    slow_wait_note("dispatcher: host scatter of one job", t0);
    a->jobs_done += 1;  // rows and bytes are counted with the job's completion, so the ratios hold mid-run
    a->rows_done += j.rows;
    if (!j.shipped) a->d2h_bytes += j.rows * (4 + 4 * (int64_t)(a->h->dim + a->h->sw));
    a->done_seq = j.seq;
    *a->done_host = (uint32_t)j.seq;  // releases streams waiting on this job (stream wait-value)
    a->cv_done.notify_all();
  }
}

// cuStreamWaitValue32 through the runtime's driver entry point (no -lcuda link)
typedef CUresult (*WaitValueFn)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
static WaitValueFn wait_value_fn() {
  static WaitValueFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return reinterpret_cast<WaitValueFn>(p);
  }();
  return fn;
}

static void wait_seq(AsyncWB* a, uint64_t seq) {
  std::unique_lock<std::mutex> lk(a->m);
  a->cv_done.wait(lk, [&] { return a->done_seq >= seq; });
}

// ------------------------------------------------------------------ kernels
__global__ void k_clear_pending(const int32_t* __restrict__ ranks, int64_t n, int32_t* pending, int32_t base,
                                int32_t cap, const int32_t* n_dev) {
  if (n_dev) n = *n_dev;
  for (int64_t k = (int64_t)blockIdx.x * kNT + threadIdx.x; k < n; k += (int64_t)gridDim.x * kNT) {
    const int r = ranks[k];
    if (pending[r] == base + (int32_t)k) pending[r] = -1;  // unless re-staged since
  }
  (void)cap;
}

// Copy 32 rows per warp: lane i owns row i (src/dst row pointers, active flag); the
// lanes then sweep the rows' units (16-byte when VEC, else single floats) with 4
// loads in flight per lane.
template <bool VEC>
__device__ __forceinline__ void warp_copy_rows(const float* sp, float* dp, bool act, Units un) {
  const int lane = threadIdx.x & 31;
  const int total = 32 * un.upr;
  constexpr int W = VEC ? 4 : 1;
  for (int u0 = 0; u0 < total; u0 += 32 * 4) {
    float4 v[4];
    float* d[4];
    bool a[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int u = u0 + q * 32 + lane;
      const int rr = min(un.row(u), 31);
      const int c = (u - rr * un.upr) * W;
      const float* s = reinterpret_cast<const float*>(__shfl_sync(FC_FULL, reinterpret_cast<long long>(sp), rr));
      d[q] = reinterpret_cast<float*>(__shfl_sync(FC_FULL, reinterpret_cast<long long>(dp), rr)) + c;
      a[q] = __shfl_sync(FC_FULL, (int)act, rr) && u < total;
      if (a[q]) {
        if (VEC) v[q] = ld4(s + c);
        else v[q].x = s[c];
      }
    }
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if (a[q]) {
        if (VEC) st4(d[q], v[q]);
        else *d[q] = v[q].x;
      }
  }
}

// 16-byte units per row when VEC, else one unit per float
inline Units row_units(int width, bool vec) {
  if (vec) return units_for(width);
  Units un;
  un.upr = width > 0 ? width : 1;
  un.lg = (un.upr & (un.upr - 1)) == 0 ? __builtin_ctz(un.upr) : -1;
  return un;
}

struct EngArgs {
  float* fast;
  float* fstate;
  const float* slow;
  const float* sstate;
  int64_t ld, sld;
  int D, S;
  int32_t* slot_to_rank;
  int32_t* rank_to_slot;
  uint8_t* dirty;
  uint32_t* res;
  uint32_t* freeb;
  const int32_t* evicted;
  const int32_t* admitted;
  const int32_t* target;
  int32_t* pending;
  float* stage[kWbBufs];
  float* sstage[kWbBufs];
  int32_t* sranks;
  int buf;
  int32_t cap;
  int always;
  Counters* c;
  Units ud, us;
};

// victims -> slot, dirty filter, compacted staging into stage[buf] + pending marks, state cleared
template <bool VEC>
__global__ void __launch_bounds__(kNT) k_evict_async(EngArgs x) {
  if (!gate_open(x.c, G_EVICT)) return;
  const int needed = x.c->needed;
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * kNT + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * kNT) >> 5;
  for (int64_t base = warp * 32; base < needed; base += nwarps * 32) {
    const int64_t v = base + lane;
    const bool act = v < needed;
    int r = 0, s = 0;
    bool wb = false;
    if (act) {
      r = x.evicted[v];
      s = x.rank_to_slot[r];
      wb = x.always || x.dirty[s];
    }
    const unsigned m = __ballot_sync(FC_FULL, wb);
    int k0 = 0;
    if (lane == 0 && m) k0 = atomicAdd(&x.c->wb_rows, __popc(m));
    k0 = __shfl_sync(FC_FULL, k0, 0);
    const int k = k0 + __popc(m & ((1u << lane) - 1u));
    warp_copy_rows<VEC>(x.fast + (int64_t)s * x.D, x.stage[x.buf] + (int64_t)k * x.D, wb, x.ud);
    if (x.S) warp_copy_rows<VEC>(x.fstate + (int64_t)s * x.S, x.sstage[x.buf] + (int64_t)k * x.S, wb, x.us);
    if (act) {
      if (wb) {
        x.sranks[k] = r;
        x.pending[r] = x.buf * x.cap + k;
      }
      x.slot_to_rank[s] = -1;
      x.rank_to_slot[r] = -1;
      x.dirty[s] = 0;
      atomicAnd(&x.res[r >> 5], ~(1u << (r & 31)));
      atomicOr(&x.freeb[s >> 5], 1u << (s & 31));
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) x.c->free_count += needed;
}

// admissions: newest copy of each admitted rank -> its target slot
template <bool VEC>
__global__ void __launch_bounds__(kNT) k_admit_async(EngArgs x) {
  if (!gate_open(x.c, G_OK)) return;
  const int m = x.c->misses;
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * kNT + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * kNT) >> 5;
  for (int64_t base = warp * 32; base < m; base += nwarps * 32) {
    const int64_t j = base + lane;
    const bool act = j < m;
    int r = 0, s = 0;
    const float* src = nullptr;
    const float* ssrc = nullptr;
    if (act) {
      r = x.admitted[j];
      s = x.target[j];
      const int pk = x.pending[r];
      src = pk >= 0 ? x.stage[pk / x.cap] + (int64_t)(pk % x.cap) * x.D : x.slow + (int64_t)r * x.ld;
      if (x.S) ssrc = pk >= 0 ? x.sstage[pk / x.cap] + (int64_t)(pk % x.cap) * x.S : x.sstate + (int64_t)r * x.sld;
    }
    warp_copy_rows<VEC>(src, x.fast + (int64_t)s * x.D, act, x.ud);
    if (x.S) warp_copy_rows<VEC>(ssrc, x.fstate + (int64_t)s * x.S, act, x.us);
    if (act) {
      x.slot_to_rank[s] = r;
      x.rank_to_slot[r] = s;
      x.dirty[s] = 0;
      atomicOr(&x.res[r >> 5], 1u << (r & 31));
      atomicAnd(&x.freeb[s >> 5], ~(1u << (s & 31)));
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) x.c->free_count -= m;
}

// ------------------------------------------------------------------ hooks
static bool vec_ok_engine(fc_cache* h) {
  auto al = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  bool v = (h->dim % 4 == 0) && (h->slow_ld % 4 == 0) && al(h->slow) && al(h->fast);
  if (h->sw) v = v && (h->sw % 4 == 0) && (h->state_ld % 4 == 0) && al(h->slow_state) && al(h->fast_state);
  return v;
}

#define FC_TRY_A(expr)     \
  do {                     \
    int rc__ = (expr);     \
    if (rc__) return rc__; \
  } while (0)

// Staging buffers are bounded like the reference's TransferBuffer (transmitter.py:19,75-94):
// they start at buffer_bytes worth of rows (64 MiB by default) and grow only when a batch
// needs more (engine_grow / pipe_grow_admission), instead of holding capacity-sized copies.
// FC_STAGE_ROWS forces the initial row count (tests exercise the overflow paths with it).
int32_t initial_stage_rows(const fc_cache* h) {
  int64_t r = h->buffer_bytes / std::max<int64_t>(1, 4 * (int64_t)(h->dim + h->sw));
  r = std::max<int64_t>(r, 1024);
  if (const char* env = std::getenv("FC_STAGE_ROWS")) r = std::max<int64_t>(1, std::atoll(env));
  return (int32_t)std::min<int64_t>(r, h->capacity);
}

static void free_wb_stages(AsyncWB* a) {
  if (a->stage_arena) cudaFree(a->stage_arena);
  a->stage_arena = nullptr;
  a->stage_bytes = 0;
  for (int b = 0; b < kWbBufs; ++b) {
    cudaFreeHost(a->hstage[b]);
    cudaFreeHost(a->hranks[b]);
    cudaFreeHost(a->hsstage[b]);
    a->stage[b] = a->sstage[b] = a->hstage[b] = a->hsstage[b] = nullptr;
    a->sranks[b] = a->hranks[b] = nullptr;
  }
  a->rows = 0;
}

static cudaError_t alloc_wb_stages(AsyncWB* a, const fc_cache* h, int32_t rows) {
  const size_t R = (size_t)rows;
  Arena ar;
  for (int b = 0; b < kWbBufs; ++b) {
    ar.add(&a->stage[b], R * h->dim);
    if (h->sw) ar.add(&a->sstage[b], R * h->sw);
    ar.add(&a->sranks[b], R);
  }
  cudaError_t e = ar.alloc(&a->stage_arena);
  if (e == cudaSuccess) a->stage_bytes = (int64_t)ar.bytes;
  for (int b = 0; b < kWbBufs && e == cudaSuccess; ++b) {
    e = cudaHostAlloc(&a->hstage[b], R * h->dim * 4, cudaHostAllocDefault);
    if (e == cudaSuccess) e = cudaHostAlloc(&a->hranks[b], R * 4, cudaHostAllocDefault);
    if (e == cudaSuccess && h->sw) e = cudaHostAlloc(&a->hsstage[b], R * h->sw * 4, cudaHostAllocDefault);
  }
  if (e == cudaSuccess) a->rows = rows;
  return e;
}

// Make every write-back stage hold `need` rows: wait for every queued job (the slow tier is
// then authoritative, so all pending marks are dropped), then reallocate the buffers.
// Rare: a batch evicting more rows than any before it.
int engine_grow(fc_cache* h, int64_t need) {
  AsyncWB* a = h->awb;
  if (!a || need <= a->rows) return FC_OK;
  FC_TRY_A(engine_drain(h));
  FC_CUDA(cudaDeviceSynchronize());  // no kernel reads a stage or a pending mark any more
  const int64_t grown = std::min<int64_t>(h->capacity, std::max<int64_t>(need + need / 4, 2 * (int64_t)a->rows));
  free_wb_stages(a);
  FC_CUDA(alloc_wb_stages(a, h, (int32_t)grown));
  FC_CUDA(cudaMemset(a->pending, 0xff, (size_t)h->num_ids * 4));
  for (int b = 0; b < kWbBufs; ++b) {
    a->rows_in[b] = 0;
    a->rows_on_dev[b] = false;
  }
  a->grows += 1;
  return FC_OK;
}

// Synchronous prepare: the eviction count is known on the device only. When the batch could
// evict more rows than a stage holds (min(n, C) > rows), read it back before the eviction
// kernel and grow first; otherwise no host round trip.
int engine_reserve(fc_cache* h, int64_t n, cudaStream_t st) {
  AsyncWB* a = h->awb;
  if (!a || std::min<int64_t>(n, h->capacity) <= a->rows) return FC_OK;
  FC_CUDA(cudaMemcpyAsync(h->ctr_host, h->ctr, sizeof(Counters), cudaMemcpyDeviceToHost, st));
  FC_CUDA(cudaStreamSynchronize(st));
  if (h->ctr_host->err == 0 && h->ctr_host->needed > a->rows) return engine_grow(h, h->ctr_host->needed);
  return FC_OK;
}

int engine_set(fc_cache* h, int engine) {
  if (engine == h->engine) return FC_OK;
  if (engine == 0) {
    int rc = engine_drain(h);
    if (rc) return rc;
    engine_release(h);
    h->engine = 0;
    return FC_OK;
  }
  if (engine != 1) return FC_ERR_BAD_ARG;
  if (!h->slow) {
    set_error("attach the slow tier before selecting the async engine");
    return FC_ERR_NO_SLOW_TIER;
  }
  if ((int64_t)h->capacity * kWbBufs > INT32_MAX) {  // stage rows <= capacity
    set_error("capacity too large for the async engine's pending-row encoding");
    return FC_ERR_BAD_ARG;
  }
  AsyncWB* a = new AsyncWB();
  a->h = h;
  a->vec = vec_ok_engine(h);
  a->device = h->device;
  Arena fx;
  fx.add(&a->pending, (size_t)h->num_ids);
  fx.add(&a->dev_rows, kWbBufs);
  cudaError_t e = fx.alloc(&a->fixed_arena);
  if (e == cudaSuccess) a->fixed_bytes = (int64_t)fx.bytes;
  if (e == cudaSuccess) e = cudaMemset(a->pending, 0xff, (size_t)h->num_ids * 4);
  if (e == cudaSuccess) e = alloc_wb_stages(a, h, initial_stage_rows(h));
  for (int b = 0; b < kWbBufs && e == cudaSuccess; ++b) {
    // the dispatcher sleeps on these (a spinning cudaEventSynchronize would contend for
    // the driver with the caller's launches)
    e = cudaEventCreateWithFlags(&a->d2h[b], cudaEventDisableTiming | cudaEventBlockingSync);
  }
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&a->side, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&a->dside, cudaStreamNonBlocking);
  for (int b = 0; b < kWbBufs && e == cudaSuccess; ++b)
    e = cudaEventCreateWithFlags(&a->cev[b], cudaEventDisableTiming | cudaEventBlockingSync);
  if (e == cudaSuccess) e = cudaHostAlloc((void**)&a->done_host, 64, cudaHostAllocMapped);
  if (e == cudaSuccess) {
    *a->done_host = 0;
    void* dp = nullptr;
    e = cudaHostGetDevicePointer(&dp, (void*)a->done_host, 0);
    a->done_dev = reinterpret_cast<CUdeviceptr>(dp);
  }
  if (e == cudaSuccess) e = cudaHostAlloc(&a->hrows, kWbBufs * sizeof(int32_t), cudaHostAllocDefault);
  h->awb = a;
  if (e != cudaSuccess) {
    engine_release(h);
    return cuda_fail(e, "engine_set");
  }
  // Host threads of this cache: on the GPU's own socket (its local CPUs, where the slow tier
  // was pinned by fc_host_alloc), and at most half of this rank's share of those cores --
  // one process per GPU shares the socket with its peers (LOCAL_WORLD_SIZE from torchrun)
  // and leaves the other half to the caller's threads.
  const std::vector<int> cpus = device_local_cpus(h->device);
  int cores = cpus.empty() ? (int)std::thread::hardware_concurrency() : (int)cpus.size();
  int local_ranks = 1;
  if (const char* env = std::getenv("LOCAL_WORLD_SIZE")) local_ranks = std::max(1, std::atoi(env));
  if (!cpus.empty() && local_ranks > 1) {  // ranks sharing this socket: the GPUs whose local CPUs match
    int same = 0, ndev = 0;
    cudaGetDeviceCount(&ndev);
    for (int d = 0; d < ndev; ++d) same += device_local_cpus(d) == cpus;
    local_ranks = std::max(1, std::min(local_ranks, same));
  }
  const int share = std::max(1, cores / local_ranks);
  int nh = std::max(1, std::min(7, share / 2 - 1));
  if (const char* env = std::getenv("FC_SCATTER_THREADS")) nh = std::max(0, std::atoi(env) - 1);
  for (int i = 0; i < nh; ++i) a->helpers.emplace_back(helper_main, a);
  a->dispatcher = std::thread(dispatcher_main, a);
  a->copier = std::thread(copier_main, a);
  for (auto& t : a->helpers) bind_thread(t.native_handle(), cpus);
  bind_thread(a->dispatcher.native_handle(), cpus);
  bind_thread(a->copier.native_handle(), cpus);
  a->threads = nh + 1;
  h->engine = 1;
  return FC_OK;
}

int engine_begin(fc_cache* h, cudaStream_t st) {
  if (h->engine != 1) return FC_OK;
  AsyncWB* a = h->awb;
  const int b = a->cur;
  if (a->rows_in[b] > 0) {  // stage[b] still holds rows from kWbBufs prepares ago
    const auto t0 = std::chrono::steady_clock::now();
    wait_seq(a, a->seq_of[b]);
    h->prof[5] += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    k_clear_pending<<<grid_for(a->rows_in[b], kNT, kSMs * 4), kNT, 0, st>>>(
        a->sranks[b], a->rows_in[b], a->pending, (int32_t)(b * a->rows), a->rows,
        a->rows_on_dev[b] ? a->dev_rows + b : nullptr);
    a->rows_in[b] = 0;
    a->rows_on_dev[b] = false;
    FC_CUDA(cudaGetLastError());
  }
  return FC_OK;
}

static EngArgs eng_args(fc_cache* h) {
  AsyncWB* a = h->awb;
  EngArgs x;
  x.fast = h->fast;
  x.fstate = h->fast_state;
  x.slow = h->slow;
  x.sstate = h->slow_state;
  x.ld = h->slow_ld;
  x.sld = h->state_ld;
  x.D = h->dim;
  x.S = h->sw;
  x.slot_to_rank = h->slot_to_rank;
  x.rank_to_slot = h->rank_to_slot;
  x.dirty = h->dirty;
  x.res = h->res_bits;
  x.freeb = h->free_bits;
  x.evicted = h->evicted_ranks;
  x.admitted = h->admitted_ranks;
  x.target = h->target_slots;
  x.pending = a->pending;
  for (int b = 0; b < kWbBufs; ++b) {
    x.stage[b] = a->stage[b];
    x.sstage[b] = a->sstage[b];
  }
  x.sranks = a->sranks[a->cur];
  x.buf = a->cur;
  x.cap = a->rows;
  x.always = h->write_back == FC_WB_ALWAYS;
  x.c = h->ctr;
  x.ud = row_units(h->dim, a->vec);
  x.us = row_units(h->sw ? h->sw : 4, a->vec);
  return x;
}

int engine_evict(fc_cache* h, cudaStream_t st) {
  EngArgs x = eng_args(h);
  if (h->awb->vec) k_evict_async<true><<<kSMs * 8, kNT, 0, st>>>(x);
  else k_evict_async<false><<<kSMs * 8, kNT, 0, st>>>(x);
  FC_CUDA(cudaGetLastError());
  return FC_OK;
}

static int launch_admit_async_tma(fc_cache* h, const EngArgs& x, cudaStream_t st);  // below, with the TMA helpers
static bool tma_fits(const fc_cache* h);

int engine_admit(fc_cache* h, cudaStream_t st) {
  EngArgs x = eng_args(h);
  if (h->awb->vec && tma_fits(h) && !std::getenv("FC_NO_TMA")) return launch_admit_async_tma(h, x, st);
  if (h->awb->vec) k_admit_async<true><<<kSMs * 4, kNT, 0, st>>>(x);
  else k_admit_async<false><<<kSMs * 4, kNT, 0, st>>>(x);
  FC_CUDA(cudaGetLastError());
  return FC_OK;
}

int engine_after_prepare(fc_cache* h, cudaStream_t st) {
  (void)st;
  if (h->engine != 1) return FC_OK;
  AsyncWB* a = h->awb;
  const int b = a->cur;
  const int64_t rows = h->ctr_host->err ? 0 : h->ctr_host->wb_rows;
  if (rows > 0) {
    // the prepare's stream is synchronised: stage[b] is complete; ship it on the side stream
    FC_CUDA(cudaMemcpyAsync(a->hranks[b], a->sranks[b], rows * 4, cudaMemcpyDeviceToHost, a->side));
    FC_CUDA(cudaMemcpyAsync(a->hstage[b], a->stage[b], rows * h->dim * 4, cudaMemcpyDeviceToHost, a->side));
    if (h->sw)
      FC_CUDA(cudaMemcpyAsync(a->hsstage[b], a->sstage[b], rows * h->sw * 4, cudaMemcpyDeviceToHost, a->side));
    FC_CUDA(cudaEventRecord(a->d2h[b], a->side));
    {
      std::lock_guard<std::mutex> lk(a->m);
      const uint64_t seq = a->next_seq++;
      a->qc.push_back(Job{b, rows, seq});
      a->seq_of[b] = seq;
    }
    a->cv_qc.notify_one();
    a->rows_in[b] = rows;
    a->cur = (a->cur + 1) % kWbBufs;
  }
  return FC_OK;
}

int engine_drain(fc_cache* h) {
  if (h->engine != 1 || !h->awb) return FC_OK;
  AsyncWB* a = h->awb;
  uint64_t last;
  {
    std::lock_guard<std::mutex> lk(a->m);
    last = a->next_seq - 1;
  }
  wait_seq(a, last);
  return FC_OK;
}

// The same drain as a stream-ordered wait: work queued on `st` after this call starts only
// once every write-back queued so far has landed in the slow tier (no host block).
int engine_drain_stream(fc_cache* h, cudaStream_t st) {
  if (h->engine != 1 || !h->awb) return FC_OK;
  AsyncWB* a = h->awb;
  uint64_t last;
  {
    std::lock_guard<std::mutex> lk(a->m);
    last = a->next_seq - 1;
    if (a->done_seq >= last) return FC_OK;
  }
  WaitValueFn wv = wait_value_fn();
  if (!wv || wv(reinterpret_cast<CUstream>(st), a->done_dev, (cuuint32_t)last, CU_STREAM_WAIT_VALUE_GEQ) !=
                 CUDA_SUCCESS)
    wait_seq(a, last);
  return FC_OK;
}

int engine_threads(const fc_cache* h) { return h->awb ? h->awb->threads : 0; }

void engine_release(fc_cache* h) {
  AsyncWB* a = h->awb;
  if (!a) return;
  {
    std::lock_guard<std::mutex> lk(a->m);
    a->stop = true;
  }
  a->cv_qc.notify_all();
  if (a->copier.joinable()) a->copier.join();  // drains its queue into the dispatcher's, then sets copier_done
  if (a->dispatcher.joinable()) a->dispatcher.join();  // scatters what is left
  {
    std::lock_guard<std::mutex> lk(a->m);
    a->helpers_stop = true;
  }
  a->cv_help.notify_all();
  for (auto& t : a->helpers)
    if (t.joinable()) t.join();
  if (a->fixed_arena) cudaFree(a->fixed_arena);
  cudaFreeHost(a->hrows);
  if (a->done_host) cudaFreeHost((void*)a->done_host);
  free_wb_stages(a);
  for (int b = 0; b < kWbBufs; ++b)
    if (a->d2h[b]) cudaEventDestroy(a->d2h[b]);
  if (a->side) cudaStreamDestroy(a->side);
  if (a->dside) cudaStreamDestroy(a->dside);
  for (int b = 0; b < kWbBufs; ++b)
    if (a->cev[b]) cudaEventDestroy(a->cev[b]);
  delete a;
  h->awb = nullptr;
}

// ------------------------------------------------------------------ prefetch pipeline
// fc_prepare_begin / fc_prepare_commit split one prepare (cache_manager.py:234-348)
// so that batch t+1's cache work overlaps batch t's forward/backward:
//
//   begin(t+1), caller's index stream:  launch_index_phase (every decision and every
//       slot-table change; no row, no dirty bit) -> counters D2H;
//   begin(t+1), transfer stream:        k_admit_stage — the admitted rows' newest
//       copies (HBM write-back stage if pending, else the pinned slow tier over the
//       host link) -> HBM admission stage[t+1 % 2];
//   commit(t+1), caller's main stream (after backward(t) in stream order):
//       k_evict_commit — dirty victims -> write-back stage, pending marks, dirty
//       cleared (the victim rows already carry backward(t)'s update);
//       k_admit_commit — admission stage -> target slots (HBM -> HBM), dirty cleared;
//       then the async engine ships the write-back stage D2H as usual.
//
// The outcome is bit-identical to sequential prepares: the index phase reads only
// slot tables, which forward/backward never touch; victims are staged after the
// previous batch's update; admitted rows are read after the previous commit's
// write-back marks exist. Ordering is enforced with events:
//   index(t+1)  after index(t), and after commit(t-1) (its parity's buffers);
//   stage(t+1)  after index(t+1) and commit(t) (pending marks, stage reuse);
//   commit(t+1) after stage(t+1) (and the caller's stream order).

constexpr int kTmaStages = 4;  // k_admit_stage_tma: row groups in flight per block
constexpr int kTmaBlocks = 64;
// rows per TMA group so that one stage holds <= 32 KB
static inline int tma_group_rows(int row_bytes) { return std::max(1, std::min(32, 32768 / row_bytes)); }
// Staging blocks of the prefetch pipeline: enough bulk copies in flight to keep the host
// link busy (~2.5 MB), and no more -- extra requests queued on the link raise the memory
// latency of every kernel running beside the staging. Measured optima on
// the B200/PCIe box: 40 blocks for 512 B rows (64 KB in flight per block), 64 for 256 B,
// 32 for 1 KB rows (profiles/r01_tma_blocks_sweep.txt).
static inline int tma_pipe_blocks(int row_bytes) {
  const double per_block = (double)kTmaStages * tma_group_rows(row_bytes) * row_bytes;
  return std::max(32, std::min(64, (int)std::lround(2.5 * 1024 * 1024 / per_block)));
}
// Paced miss-staging rate (GB/s), FC_XFER_GBPS; 0 = unpaced (default). Alone, pacing the
// staging below ~36 GB/s keeps every other kernel at its isolated speed
// (profiles/r02_launch_latency.txt, runs 3-4), but in the pipeline the write-back's D2H copy
// runs at the same time and its posted writes hold the staging's read requests in the same
// upstream queue: with that copy beside it, even a 20 GB/s staging leaves kernel boundaries
// at ~40 us (run 4). The in-pipeline sweep (profiles/r02_pace_sweep.txt) found no rate that
// beats the unpaced ring, so pacing stays off.
constexpr double kPacedGBps = 0.0;
// the TMA ring must fit in shared memory (rows wider than ~12K floats use the SM kernels)
static bool tma_fits(const fc_cache* h) {
  const size_t rb = (size_t)(h->dim + h->sw) * 4;
  return (size_t)kTmaStages * tma_group_rows((int)rb) * rb <= 200 * 1024;
}

struct Pipe {
  IndexBufs ib[2];
  Counters* hctr[2] = {nullptr, nullptr};  // pinned mapped copies of the index counters
  Counters* hctr_dev[2] = {nullptr, nullptr};
  float* astage[2] = {nullptr, nullptr};   // admission stage [arows, D]
  float* astage_s[2] = {nullptr, nullptr}; // [arows, S]
  int32_t arows = 0;                       // rows per admission stage (grown on demand)
  int32_t scap[2] = {0, 0};                // rows the last staging of each parity staged at most
  // digit histograms of each begun batch's inverse for its backward's radix sort, in a ring
  // deep enough that a batch's backward has run before its buffer is zeroed again (the index
  // phase of batch t+4 follows commit(t+2), which follows backward(t+1) on the compute stream)
  static constexpr int kHistRing = 4;
  int32_t* sort_hist[kHistRing] = {};
  const int32_t* hist_inv[kHistRing] = {};
  int64_t hist_n[kHistRing] = {};
  int hist_next = 0;
  void* fixed_arena = nullptr;             // counters + index lists of both parities
  int64_t fixed_bytes = 0;
  void* stage_arena = nullptr;             // both admission stages
  int64_t stage_bytes = 0;
  int grows = 0;
  cudaStream_t xfer = nullptr;             // transfer stream (k_admit_stage)
  cudaEvent_t ev_index[2] = {nullptr, nullptr};
  cudaEvent_t ev_xfer[2] = {nullptr, nullptr};
  cudaEvent_t ev_commit[2] = {nullptr, nullptr};
  cudaEvent_t px[2][2] = {{nullptr, nullptr}, {nullptr, nullptr}};  // profiling: around k_admit_stage
  bool has_index[2] = {false, false};
  bool has_commit[2] = {false, false};
  bool timed[2] = {false, false};
  int par = 0;   // parity of the next prepare_begin
  int nout = 0;  // begun and not yet committed (0..2); the oldest has parity par ^ (nout & 1)
  int xfer_blocks = kSMs;                  // k_admit_stage grid (one block per SM: enough loads in flight)
  bool defer_xfer = false;                 // launch the staging after the next row update (fc_backward_update)
  bool tma = false;                        // stage through the bulk-copy engine (k_admit_stage_tma)
  int tma_blocks = kTmaBlocks;
  double xfer_gbps = 0.0;                  // paced staging rate (GB/s = B/ns); 0: unpaced
  bool xfer_pending = false;
  bool xfer_behind = false;                // the pending staging was begun behind an uncommitted prepare:
                                           // only that prepare's commit may launch it
  int xfer_par = 0;
  cudaEvent_t ev_after = nullptr;
};

#define FC_TRY_E(expr)     \
  do {                     \
    int rc__ = (expr);     \
    if (rc__) return rc__; \
  } while (0)

// FC_DEBUG_NOOP_INDEX / FC_DEBUG_NOOP_XFER=k: measurement only -- k empty kernels at the end of
// every pipelined index phase / before every staging, to price a kernel boundary on that chain
__global__ void k_noop_e() {}
static int debug_noops(const char* name) {
  const char* e = std::getenv(name);
  return e ? std::max(0, std::atoi(e)) : 0;
}

bool pipe_outstanding(const fc_cache* h) { return h->pipe && h->pipe->nout > 0; }

// Host wait for every recorded pipeline commit (their kernels have finished).
int pipe_sync_commits(fc_cache* h) {
  Pipe* q = h->pipe;
  if (!q) return FC_OK;
  for (int p = 0; p < 2; ++p)
    if (q->has_commit[p]) FC_CUDA(cudaEventSynchronize(q->ev_commit[p]));
  return FC_OK;
}

// A synchronous verb on stream `st` runs after every committed pipeline step.
int pipe_order(fc_cache* h, cudaStream_t st) {
  Pipe* q = h->pipe;
  if (!q) return FC_OK;
  for (int p = 0; p < 2; ++p) {
    if (q->has_commit[p]) FC_CUDA(cudaStreamWaitEvent(st, q->ev_commit[p], 0));
  }
  return FC_OK;
}

void pipe_release(fc_cache* h) {
  Pipe* q = h->pipe;
  if (!q) return;
  if (q->fixed_arena) cudaFree(q->fixed_arena);
  if (q->stage_arena) cudaFree(q->stage_arena);
  for (int p = 0; p < 2; ++p) {
    cudaFreeHost(q->hctr[p]);
    for (cudaEvent_t ev : {q->ev_index[p], q->ev_xfer[p], q->ev_commit[p], q->px[p][0], q->px[p][1]})
      if (ev) cudaEventDestroy(ev);
  }
  if (q->xfer) cudaStreamDestroy(q->xfer);
  if (q->ev_after) cudaEventDestroy(q->ev_after);
  delete q;
  h->pipe = nullptr;
}

static int pipe_create(fc_cache* h) {
  Pipe* q = new Pipe();
  std::memset(q->ib, 0, sizeof(q->ib));
  h->pipe = q;
  const size_t C = (size_t)h->capacity;
  q->arows = initial_stage_rows(h);
  Arena fx, sa;
  for (int k = 0; k < Pipe::kHistRing; ++k) fx.add(&q->sort_hist[k], kSortHistInts);
  for (int p = 0; p < 2; ++p) {
    fx.add(&q->ib[p].ctr, 1);
    fx.add(&q->ib[p].evicted, C);
    fx.add(&q->ib[p].vslots, C);
    fx.add(&q->ib[p].admitted, C);
    fx.add(&q->ib[p].target, C);
    sa.add(&q->astage[p], (size_t)q->arows * h->dim);
    if (h->sw) sa.add(&q->astage_s[p], (size_t)q->arows * h->sw);
  }
  cudaError_t e = fx.alloc(&q->fixed_arena);
  if (e == cudaSuccess) e = sa.alloc(&q->stage_arena);
  if (e == cudaSuccess) {
    q->fixed_bytes = (int64_t)fx.bytes;
    q->stage_bytes = (int64_t)sa.bytes;
  }
  for (int p = 0; p < 2 && e == cudaSuccess; ++p) {
    e = cudaMemset(q->ib[p].ctr, 0, sizeof(Counters));
    // mapped: the index phase publishes its counters with a kernel store instead of a
    // cudaMemcpy that would queue behind the write-back D2H on the copy engine
    if (e == cudaSuccess) e = cudaHostAlloc(&q->hctr[p], sizeof(Counters), cudaHostAllocMapped);
    if (e == cudaSuccess) e = cudaHostGetDevicePointer(reinterpret_cast<void**>(&q->hctr_dev[p]), q->hctr[p], 0);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&q->ev_index[p], cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&q->ev_xfer[p], cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&q->ev_commit[p], cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreate(&q->px[p][0]);
    if (e == cudaSuccess) e = cudaEventCreate(&q->px[p][1]);
  }
  // the transfer kernel is latency-bound on the host link and needs few SM resources,
  // but it is on the critical path: give its stream the highest priority
  int lo = 0, hi = 0;
  if (e == cudaSuccess) e = cudaDeviceGetStreamPriorityRange(&lo, &hi);
  if (e == cudaSuccess) e = cudaStreamCreateWithPriority(&q->xfer, cudaStreamNonBlocking, hi);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&q->ev_after, cudaEventDisableTiming);
  if (const char* env = std::getenv("FC_XFER_AFTER_UPDATE")) q->defer_xfer = std::atoi(env) != 0;
  // TMA staging needs 16-byte rows at 16-byte aligned addresses (the async engine's vec
  // condition); FC_XFER_TMA=0 selects the SM-load kernel
  q->tma = h->awb && h->awb->vec && tma_fits(h);
  if (const char* env = std::getenv("FC_XFER_TMA")) q->tma = q->tma && std::atoi(env) != 0;
  q->tma_blocks = tma_pipe_blocks((h->dim + h->sw) * 4);
  if (const char* env = std::getenv("FC_TMA_BLOCKS")) q->tma_blocks = std::max(1, std::atoi(env));
  q->xfer_gbps = kPacedGBps;
  if (const char* env = std::getenv("FC_XFER_GBPS")) q->xfer_gbps = std::max(0.0, std::atof(env));

  q->xfer_blocks = kSMs;
  if (const char* env = std::getenv("FC_XFER_BLOCKS")) q->xfer_blocks = std::max(1, std::atoi(env));
  if (e != cudaSuccess) {
    pipe_release(h);
    return cuda_fail(e, "pipeline buffers");
  }
  return FC_OK;
}

struct PipeArgs {
  float* fast;
  float* fstate;
  const float* slow;
  const float* sstate;
  int64_t ld, sld;
  int D, S;
  uint8_t* dirty;
  const int32_t* evicted;
  const int32_t* vslots;
  const int32_t* admitted;
  const int32_t* target;
  int32_t* pending;
  float* wstage[kWbBufs];   // write-back stage (AsyncWB)
  float* wstage_s[kWbBufs];
  int32_t* sranks;
  int32_t* stage_rows;
  float* astage;
  float* astage_s;
  int buf;
  int32_t cap;   // rows per write-back stage (pending-mark encoding)
  int32_t acap;  // rows per admission stage: admitted rows past it are copied at commit
  int always;
  Counters* c;
  Units ud, us;
};


// transfer stream: newest copy of each admitted rank -> admission stage (host link)
template <bool VEC>
__global__ void __launch_bounds__(kNT) k_admit_stage(PipeArgs x) {
  if (!gate_open(x.c, G_ADMIT)) return;
  const int m = min(x.c->misses, x.acap);  // the rest is copied by k_admit_commit
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * kNT + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * kNT) >> 5;
  for (int64_t base = warp * 32; base < m; base += nwarps * 32) {
    const int64_t j = base + lane;
    const bool act = j < m;
    const float* src = nullptr;
    const float* ssrc = nullptr;
    if (act) {
      const int r = x.admitted[j];
      const int pk = x.pending[r];
      src = pk >= 0 ? x.wstage[pk / x.cap] + (int64_t)(pk % x.cap) * x.D : x.slow + (int64_t)r * x.ld;
      if (x.S) ssrc = pk >= 0 ? x.wstage_s[pk / x.cap] + (int64_t)(pk % x.cap) * x.S : x.sstate + (int64_t)r * x.sld;
    }
    warp_copy_rows<VEC>(src, x.astage + j * x.D, act, x.ud);
    if (x.S) warp_copy_rows<VEC>(ssrc, x.astage_s + j * x.S, act, x.us);
  }
}

// ---- TMA bulk-copy staging (sm_100a) -------------------------------------------
// The same job as k_admit_stage, issued through the bulk-copy (TMA) engine: one
// thread per block queues cp.async.bulk loads of whole rows (host-mapped slow tier
// or the HBM write-back stage) into a shared-memory ring tracked by mbarriers, and
// writes each group of G staged rows back with ONE bulk store (the admission stage is
// contiguous). Measured (tools/interference_bench.cu, profiles/r01_interference_bench_tma.txt):
// 50 GB/s alone vs 43 for SM loads, and a concurrent HBM-bound kernel slows by ~5%
// instead of ~4x — the miss staging can overlap the backward.
// Pacing (gap_ns > 0): this block queues its k-th group no earlier than t0 + k * gap_ns
// (%globaltimer), so the staging offers the host link a fixed request rate instead of as
// many bulk copies as the ring allows. Unpaced, the requests queue up in front of the
// link (it serves random 512 B reads at ~42 GB/s), and while that queue exists every
// kernel boundary and memory fence anywhere on the GPU waits behind it: 60-100 us per
// launch instead of ~4 (tools/launch_latency.cu, profiles/r02_launch_latency.txt). Paced
// just below the link's rate the queue never forms and the index phase, pooled gather
// and backward that run beside the staging keep their isolated speed.
__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__global__ void __launch_bounds__(32) k_admit_stage_tma(PipeArgs x, int G, unsigned gap_ns) {
  extern __shared__ __align__(128) unsigned char ring[];  // kTmaStages x G x (D + S) floats
  __shared__ uint64_t bar[kTmaStages];
  const int lane = threadIdx.x;
  if (!gate_open(x.c, G_ADMIT)) return;
  const int m = min(x.c->misses, x.acap);  // the rest is copied by k_admit_commit
  const unsigned rb = (unsigned)x.D * 4, sb = (unsigned)x.S * 4;
  const size_t stage_bytes = (size_t)G * (rb + sb);
  if (lane == 0) {
    for (int i = 0; i < kTmaStages; ++i) mbar_init(&bar[i]);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  const uint64_t pol = l2_evict_first();
  unsigned phase_bits = 0;
  const int ngroups = (m + G - 1) / G;
  // group k of this block = blockIdx.x + k * gridDim.x; up to kTmaStages groups in flight.
  // The warp resolves a group's sources in parallel (admitted rank, pending mark: one
  // row per lane), lane 0 arms the stage's mbarrier, every lane queues its own row.
  int issued = 0, retired = 0;
  const int mine = ngroups > (int)blockIdx.x ? (ngroups - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
  // blocks start staggered across one gap so the link sees an even request stream
  const unsigned long long t0 =
      gap_ns ? __shfl_sync(FC_FULL, global_ns(), 0) + (unsigned long long)blockIdx.x * gap_ns / gridDim.x : 0ull;
  while (retired < mine) {
    const bool slot_free = issued < mine && issued - retired < kTmaStages;
    bool due = true;
    if (gap_ns && slot_free) due = __shfl_sync(FC_FULL, global_ns(), 0) >= t0 + (unsigned long long)issued * gap_ns;
    if (slot_free && !due && issued == retired) continue;  // nothing in flight: wait for the clock
    if (slot_free && !due) {  // something in flight: retire it if it has landed, else keep polling
      unsigned done = 0;
      if (lane == 0) {
        const int st0 = retired % kTmaStages;
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(done)
            : "r"(smem_u32(&bar[st0])), "r"((phase_bits >> st0) & 1u)
            : "memory");
      }
      if (!__shfl_sync(FC_FULL, done, 0)) continue;
    }
    if (slot_free && due) {
      const int st = issued % kTmaStages;
      if (issued >= kTmaStages) {  // the stage's previous bulk store has finished reading it
        if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        __syncwarp();
      }
      const int g = blockIdx.x + issued * gridDim.x;
      const int j0 = g * G, cnt = min(G, m - j0);
      unsigned char* rows = ring + st * stage_bytes;
      unsigned char* srows = rows + (size_t)G * rb;
      if (lane == 0) mbar_expect_tx(&bar[st], cnt * (rb + sb));
      __syncwarp();
      for (int i = lane; i < cnt; i += 32) {
        const int r = x.admitted[j0 + i];
        const int pk = x.pending[r];
        const float* src = pk >= 0 ? x.wstage[pk / x.cap] + (int64_t)(pk % x.cap) * x.D : x.slow + (int64_t)r * x.ld;
        bulk_g2s_ef(rows + (size_t)i * rb, src, rb, &bar[st], pol);
        if (x.S) {
          const float* ss =
              pk >= 0 ? x.wstage_s[pk / x.cap] + (int64_t)(pk % x.cap) * x.S : x.sstate + (int64_t)r * x.sld;
          bulk_g2s_ef(srows + (size_t)i * sb, ss, sb, &bar[st], pol);
        }
      }
      ++issued;
      continue;
    }
    // retire the oldest group: wait for its rows, one bulk store per array
    const int st = retired % kTmaStages;
    mbar_wait(&bar[st], (phase_bits >> st) & 1u);
    phase_bits ^= 1u << st;
    if (lane == 0) {
      const int g = blockIdx.x + retired * gridDim.x;
      const int j0 = g * G, cnt = min(G, m - j0);
      unsigned char* rows = ring + st * stage_bytes;
      bulk_s2g_ef(x.astage + (int64_t)j0 * x.D, rows, cnt * rb, pol);
      if (x.S) bulk_s2g_ef(x.astage_s + (int64_t)j0 * x.S, rows + (size_t)G * rb, cnt * sb, pol);
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
    __syncwarp();
    ++retired;
  }
  if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// Synchronous-prepare admission through the bulk-copy engine: like k_admit_stage_tma,
// but each staged row is stored straight to its target slot (one 16-byte-multiple bulk
// store per row) and the lanes apply the admissions to the slot tables as they queue
// them (nothing reads the rows before the next kernel).
__global__ void __launch_bounds__(32) k_admit_async_tma(EngArgs x, int G) {
  extern __shared__ __align__(128) unsigned char ring[];
  __shared__ uint64_t bar[kTmaStages];
  const int lane = threadIdx.x;
  if (!gate_open(x.c, G_OK)) return;
  const int m = x.c->misses;
  const unsigned rb = (unsigned)x.D * 4, sb = (unsigned)x.S * 4;
  const size_t stage_bytes = (size_t)G * (rb + sb);
  if (lane == 0) {
    for (int i = 0; i < kTmaStages; ++i) mbar_init(&bar[i]);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if (blockIdx.x == 0) x.c->free_count -= m;
  }
  __syncwarp();
  unsigned phase_bits = 0;
  const int ngroups = (m + G - 1) / G;
  int issued = 0, retired = 0;
  const int mine = ngroups > (int)blockIdx.x ? (ngroups - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
  while (retired < mine) {
    if (issued < mine && issued - retired < kTmaStages) {
      const int st = issued % kTmaStages;
      if (issued >= kTmaStages) {
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // every lane stored rows of this stage
        __syncwarp();
      }
      const int g = blockIdx.x + issued * gridDim.x;
      const int j0 = g * G, cnt = min(G, m - j0);
      unsigned char* rows = ring + st * stage_bytes;
      unsigned char* srows = rows + (size_t)G * rb;
      if (lane == 0) mbar_expect_tx(&bar[st], cnt * (rb + sb));
      __syncwarp();
      for (int i = lane; i < cnt; i += 32) {
        const int r = x.admitted[j0 + i];
        const int s = x.target[j0 + i];
        const int pk = x.pending[r];
        const float* src = pk >= 0 ? x.stage[pk / x.cap] + (int64_t)(pk % x.cap) * x.D : x.slow + (int64_t)r * x.ld;
        bulk_g2s(rows + (size_t)i * rb, src, rb, &bar[st]);
        if (x.S) {
          const float* ss = pk >= 0 ? x.sstage[pk / x.cap] + (int64_t)(pk % x.cap) * x.S : x.sstate + (int64_t)r * x.sld;
          bulk_g2s(srows + (size_t)i * sb, ss, sb, &bar[st]);
        }
        x.slot_to_rank[s] = r;
        x.rank_to_slot[r] = s;
        x.dirty[s] = 0;
        atomicOr(&x.res[r >> 5], 1u << (r & 31));
        atomicAnd(&x.freeb[s >> 5], ~(1u << (s & 31)));
      }
      ++issued;
      continue;
    }
    const int st = retired % kTmaStages;
    mbar_wait(&bar[st], (phase_bits >> st) & 1u);
    phase_bits ^= 1u << st;
    const int g = blockIdx.x + retired * gridDim.x;
    const int j0 = g * G, cnt = min(G, m - j0);
    unsigned char* rows = ring + st * stage_bytes;
    for (int i = lane; i < cnt; i += 32) {  // rows go to scattered slots: one bulk store each
      const int s = x.target[j0 + i];
      bulk_s2g(x.fast + (int64_t)s * x.D, rows + (size_t)i * rb, rb);
      if (x.S) bulk_s2g(x.fstate + (int64_t)s * x.S, rows + (size_t)G * rb + (size_t)i * sb, sb);
    }
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    __syncwarp();
    ++retired;
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

static int launch_admit_async_tma(fc_cache* h, const EngArgs& x, cudaStream_t st) {
  const int G = tma_group_rows((h->dim + h->sw) * 4);
  const size_t smem = (size_t)kTmaStages * G * (h->dim + h->sw) * 4;
  if (smem > 48 * 1024)
    FC_CUDA(cudaFuncSetAttribute(k_admit_async_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  k_admit_async_tma<<<kTmaBlocks, 32, smem, st>>>(x, G);
  FC_CUDA(cudaGetLastError());
  return FC_OK;
}

// commit: dirty victims (rows already carry the previous batch's update) -> write-back stage
template <bool VEC>
__global__ void __launch_bounds__(kNT) k_evict_commit(PipeArgs x) {
  if (!gate_open(x.c, G_EVICT)) return;
  const int needed = x.c->needed;
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * kNT + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * kNT) >> 5;
  for (int64_t base = warp * 32; base < needed; base += nwarps * 32) {
    const int64_t v = base + lane;
    const bool act = v < needed;
    int r = 0, s = 0;
    bool wb = false;
    if (act) {
      r = x.evicted[v];
      s = x.vslots[v];
      wb = x.always || x.dirty[s];
    }
    const unsigned m = __ballot_sync(FC_FULL, wb);
    int k0 = 0;
    if (lane == 0 && m) {
      k0 = atomicAdd(x.stage_rows, __popc(m));
      atomicAdd(&x.c->wb_rows, __popc(m));
    }
    k0 = __shfl_sync(FC_FULL, k0, 0);
    const int k = k0 + __popc(m & ((1u << lane) - 1u));
    warp_copy_rows<VEC>(x.fast + (int64_t)s * x.D, x.wstage[x.buf] + (int64_t)k * x.D, wb, x.ud);
    if (x.S) warp_copy_rows<VEC>(x.fstate + (int64_t)s * x.S, x.wstage_s[x.buf] + (int64_t)k * x.S, wb, x.us);
    if (wb) {
      x.sranks[k] = r;
      x.pending[r] = x.buf * x.cap + k;
    }
    if (act) x.dirty[s] = 0;
  }
}

// commit: admission stage -> target slots
template <bool VEC>
__global__ void __launch_bounds__(kNT) k_admit_commit(PipeArgs x) {
  if (!gate_open(x.c, G_ADMIT)) return;
  const int m = x.c->misses;
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * kNT + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * kNT) >> 5;
  for (int64_t base = warp * 32; base < m; base += nwarps * 32) {
    const int64_t j = base + lane;
    const bool act = j < m;
    const int t = act ? x.target[j] : 0;
    // rows past the admission stage (a batch with more misses than it holds; the stage grows
    // after this commit) come straight from their newest copy, as the synchronous path does
    const float* src = x.astage + j * x.D;
    const float* ssrc = x.S ? x.astage_s + j * x.S : nullptr;
    if (act && j >= x.acap) {
      const int r = x.admitted[j];
      const int pk = x.pending[r];
      src = pk >= 0 ? x.wstage[pk / x.cap] + (int64_t)(pk % x.cap) * x.D : x.slow + (int64_t)r * x.ld;
      if (x.S) ssrc = pk >= 0 ? x.wstage_s[pk / x.cap] + (int64_t)(pk % x.cap) * x.S : x.sstate + (int64_t)r * x.sld;
    }
    warp_copy_rows<VEC>(src, x.fast + (int64_t)t * x.D, act, x.ud);
    if (x.S) warp_copy_rows<VEC>(ssrc, x.fstate + (int64_t)t * x.S, act, x.us);
    if (act) x.dirty[t] = 0;
  }
}

static PipeArgs pipe_args(fc_cache* h, int p) {
  AsyncWB* a = h->awb;
  Pipe* q = h->pipe;
  PipeArgs x;
  x.fast = h->fast;
  x.fstate = h->fast_state;
  x.slow = h->slow;
  x.sstate = h->slow_state;
  x.ld = h->slow_ld;
  x.sld = h->state_ld;
  x.D = h->dim;
  x.S = h->sw;
  x.dirty = h->dirty;
  x.evicted = q->ib[p].evicted;
  x.vslots = q->ib[p].vslots;
  x.admitted = q->ib[p].admitted;
  x.target = q->ib[p].target;
  x.pending = a->pending;
  for (int b = 0; b < kWbBufs; ++b) {
    x.wstage[b] = a->stage[b];
    x.wstage_s[b] = a->sstage[b];
  }
  x.sranks = a->sranks[a->cur];
  x.stage_rows = a->dev_rows + a->cur;
  x.astage = q->astage[p];
  x.astage_s = q->astage_s[p];
  x.buf = a->cur;
  x.cap = a->rows;
  x.acap = q->scap[p];  // what this parity's staging was launched with (the stage may have grown since)
  x.always = h->write_back == FC_WB_ALWAYS;
  x.c = q->ib[p].ctr;
  x.ud = row_units(h->dim, a->vec);
  x.us = row_units(h->sw ? h->sw : 4, a->vec);
  return x;
}

// Admission stages for `need` rows from now on: after a device sync (no staging in flight),
// new buffers take over the rows the old ones hold (a batch staged but not yet committed).
static int pipe_grow_admission(fc_cache* h, int64_t need) {
  Pipe* q = h->pipe;
  if (need <= q->arows) return FC_OK;
  FC_CUDA(cudaDeviceSynchronize());
  const int64_t grown = std::min<int64_t>(h->capacity, std::max<int64_t>(need + need / 4, 2 * (int64_t)q->arows));
  float* nd[2] = {nullptr, nullptr};
  float* ns[2] = {nullptr, nullptr};
  Arena sa;
  for (int p = 0; p < 2; ++p) {
    sa.add(&nd[p], (size_t)grown * h->dim);
    if (h->sw) sa.add(&ns[p], (size_t)grown * h->sw);
  }
  void* arena = nullptr;
  FC_CUDA(sa.alloc(&arena));
  for (int p = 0; p < 2; ++p) {
    FC_CUDA(cudaMemcpy(nd[p], q->astage[p], (size_t)q->arows * h->dim * 4, cudaMemcpyDeviceToDevice));
    if (h->sw) FC_CUDA(cudaMemcpy(ns[p], q->astage_s[p], (size_t)q->arows * h->sw * 4, cudaMemcpyDeviceToDevice));
    q->astage[p] = nd[p];
    q->astage_s[p] = ns[p];
  }
  cudaFree(q->stage_arena);
  q->stage_arena = arena;
  q->stage_bytes = (int64_t)sa.bytes;
  q->arows = (int32_t)grown;
  q->grows += 1;
  return FC_OK;
}

void pipe_forget_sort_hist(fc_cache* h, const int32_t* inverse) {
  Pipe* q = h->pipe;
  if (!q) return;
  for (int k = 0; k < Pipe::kHistRing; ++k)
    if (q->hist_inv[k] == inverse) q->hist_inv[k] = nullptr;
}

const int32_t* pipe_take_sort_hist(fc_cache* h, const int32_t* inverse, int64_t n) {
  Pipe* q = h->pipe;
  if (!q || !inverse) return nullptr;
  for (int k = 0; k < Pipe::kHistRing; ++k) {  // newest first
    const int i = (q->hist_next + Pipe::kHistRing - 1 - k) % Pipe::kHistRing;
    if (q->hist_inv[i] == inverse && q->hist_n[i] == n) {
      q->hist_inv[i] = nullptr;  // one backward per prepare
      return q->sort_hist[i];
    }
  }
  return nullptr;
}

int pipe_begin(fc_cache* h, const void* ids, int ids_bytes, int64_t n, int32_t* uids, int32_t* ucnt, int32_t* uranks,
               int32_t* uslots, int32_t* inverse, cudaStream_t st) {
  if (h->engine != 1) {
    set_error("the prefetch pipeline needs the async engine (fc_set_engine(h, 1))");
    return FC_ERR_BAD_ARG;
  }
  if (!h->pipe) {
    int rc = pipe_create(h);
    if (rc) return rc;
  }
  Pipe* q = h->pipe;
  if ((int64_t)h->dim * 4 > h->buffer_bytes) {
    // the reference's order for a row larger than the buffer (write-back raises before
    // mutation only when a victim is dirty) needs the dirty bits at decision time, which
    // the concurrent row update of the previous batch may still change
    set_error("the prefetch pipeline needs a staging buffer of at least one row (%d B > %lld B)", h->dim * 4,
              (long long)h->buffer_bytes);
    return FC_ERR_BUFFER_TOO_SMALL;
  }
  // Depth 2: batch t+1 may be begun while batch t is still uncommitted -- its index phase
  // only needs index(t) (state order) and commit(t-1) (this parity's buffers), so it can
  // start on the device the moment index(t) ends instead of after the host has committed
  // t. Its staging must still follow commit(t) (pending write-back marks) and is launched
  // by that commit.
  if (q->nout >= 2 || (q->nout == 1 && q->defer_xfer)) {
    set_error(q->nout >= 2 ? "two prefetched prepares are outstanding: commit one first"
                           : "a prefetched prepare is outstanding: commit it first");
    return FC_ERR_BAD_ARG;
  }
  const int p = q->par;
  const int o = p ^ 1;
  // index(t+1) after index(t) (state order) and after commit(t-1) (this parity's buffers)
  if (q->has_index[o]) FC_CUDA(cudaStreamWaitEvent(st, q->ev_index[o], 0));
  if (q->has_commit[p]) FC_CUDA(cudaStreamWaitEvent(st, q->ev_commit[p], 0));
  trace_mark(h, T_INDEX_BEGIN, st);
  pipe_forget_sort_hist(h, inverse);  // an older batch's histograms for this buffer are stale now
  const int hs = q->hist_next;
  q->hist_next = (hs + 1) % Pipe::kHistRing;
  q->hist_inv[hs] = inverse;
  q->hist_n[hs] = n;
  int rc = launch_index_phase(h, ids, ids_bytes, n, uids, ucnt, uranks, uslots, inverse, q->ib[p], q->hctr_dev[p],
                              q->sort_hist[hs], st);
  if (rc) return rc;
  for (int k = 0; k < debug_noops("FC_DEBUG_NOOP_INDEX"); ++k) k_noop_e<<<1, 32, 0, st>>>();
  trace_mark(h, T_INDEX_END, st);
  FC_CUDA(cudaEventRecord(q->ev_index[p], st));
  q->has_index[p] = true;
  const bool behind_commit = q->nout == 1;  // commit(t) not launched yet: it launches this staging
  q->nout += 1;
  q->par = o;
  q->xfer_pending = true;
  q->xfer_behind = behind_commit;
  q->xfer_par = p;
  if (!q->defer_xfer && !behind_commit) return pipe_launch_xfer(h, nullptr, false);
  return FC_OK;
}

// Launch the outstanding prefetch's miss staging on the transfer stream. With
// `after` set, the staging also waits for everything queued so far on that stream
// (deferred mode: launched at the end of the row update so that the host-link
// kernel does not run beside the HBM-bound backward).
// fc_profile: add a finished staging kernel's event time (block: wait for it; else only
// when its end event has already fired)
static void harvest_xfer_time(fc_cache* h, int par, bool block) {
  Pipe* q = h->pipe;
  if (!q->timed[par]) return;
  if (!block && cudaEventQuery(q->px[par][1]) != cudaSuccess) return;
  float ms = 0.f;
  if (cudaEventSynchronize(q->px[par][1]) == cudaSuccess &&
      cudaEventElapsedTime(&ms, q->px[par][0], q->px[par][1]) == cudaSuccess) {
    h->prof[1] += ms;
    h->prof[6] += 1;
  }
  q->timed[par] = false;
}

int pipe_launch_xfer(fc_cache* h, cudaStream_t after, bool from_update) {
  Pipe* q = h->pipe;
  if (!q || !q->xfer_pending) return FC_OK;
  // A row update may not launch a staging that waits for an uncommitted prepare: its wait
  // on that prepare's commit event would bind to a stale commit and the staging could
  // read pending marks before that commit writes them. pipe_commit launches it.
  if (from_update && q->xfer_behind) return FC_OK;
  q->xfer_pending = false;
  q->xfer_behind = false;
  const int p = q->xfer_par, o = p ^ 1;
  // stage(t+1) after index(t+1), after commit(t) (pending marks), and after commit(t-1),
  // the last reader of this parity's admission stage. (Waiting only for commit(t)'s
  // write-back marks lets the staging start ~20 us earlier, beside the admission copy and the
  // pooled gather, and measured ~3% slower: profiles/r02_index_fusion_ab.txt.)
  FC_CUDA(cudaStreamWaitEvent(q->xfer, q->ev_index[p], 0));
  if (q->has_commit[o]) FC_CUDA(cudaStreamWaitEvent(q->xfer, q->ev_commit[o], 0));
  if (q->has_commit[p]) FC_CUDA(cudaStreamWaitEvent(q->xfer, q->ev_commit[p], 0));
  if (from_update) {  // `after` may be the legacy default stream (NULL)
    FC_CUDA(cudaEventRecord(q->ev_after, after));
    FC_CUDA(cudaStreamWaitEvent(q->xfer, q->ev_after, 0));
  }
  q->scap[p] = q->arows;
  PipeArgs x = pipe_args(h, p);
  harvest_xfer_time(h, p, true);  // this parity's previous staging (long finished) before its events are reused
  q->timed[p] = h->profile != 0;
  if (q->timed[p]) FC_CUDA(cudaEventRecord(q->px[p][0], q->xfer));
  for (int k = 0; k < debug_noops("FC_DEBUG_NOOP_XFER"); ++k) k_noop_e<<<1, 32, 0, q->xfer>>>();
  trace_mark(h, T_XFER_BEGIN, q->xfer);
  // FC_DEBUG_SKIP_STAGING=1: measurement only (admitted rows are NOT staged, results are
  // wrong) -- how long the rest of the pipelined step takes without host-link traffic
  static const bool skip_staging = [] {
    const bool on = std::getenv("FC_DEBUG_SKIP_STAGING") != nullptr;
    if (on) std::fprintf(stderr, "[freqcache_b200] FC_DEBUG_SKIP_STAGING: admitted rows are NOT staged (timing only)\n");
    return on;
  }();
  if (skip_staging) {
  } else if (q->tma) {  // bulk-copy engine: rows are 16-byte multiples at 16-byte aligned addresses
    const int G = tma_group_rows((h->dim + h->sw) * 4);
    const size_t smem = (size_t)kTmaStages * G * (h->dim + h->sw) * 4;
    if (smem > 48 * 1024)
      FC_CUDA(cudaFuncSetAttribute(k_admit_stage_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    // gap between one block's groups for the paced rate: blocks x group bytes / rate
    const double group_bytes = (double)G * (h->dim + h->sw) * 4;
    const unsigned gap = q->xfer_gbps > 0 ? (unsigned)(q->tma_blocks * group_bytes / q->xfer_gbps) : 0u;
    k_admit_stage_tma<<<q->tma_blocks, 32, smem, q->xfer>>>(x, G, gap);
  } else if (h->awb->vec) {
    k_admit_stage<true><<<q->xfer_blocks, kNT, 0, q->xfer>>>(x);
  } else {
    k_admit_stage<false><<<q->xfer_blocks, kNT, 0, q->xfer>>>(x);
  }
  FC_CUDA(cudaGetLastError());
  trace_mark(h, T_XFER_END, q->xfer);
  if (q->timed[p]) FC_CUDA(cudaEventRecord(q->px[p][1], q->xfer));
  FC_CUDA(cudaEventRecord(q->ev_xfer[p], q->xfer));
  return FC_OK;
}



int pipe_commit(fc_cache* h, cudaStream_t st, fc_prepare_info* info) {
  Pipe* q = h->pipe;
  std::memset(info, 0, sizeof(*info));
  if (!q || q->nout == 0) {
    set_error("no prefetched prepare to commit");
    return FC_ERR_BAD_ARG;
  }
  const int p = q->par ^ (q->nout & 1);  // the oldest outstanding prepare
  // deferred staging of this batch not triggered by an update: launch it now
  if (q->xfer_pending && q->xfer_par == p) FC_TRY_E(pipe_launch_xfer(h, nullptr, false));
  q->nout -= 1;
  // a newer prepare begun behind this commit gets its staging once this commit is queued
  auto launch_next_xfer = [&]() -> int {
    if (q->xfer_pending && q->xfer_par == (p ^ 1)) return pipe_launch_xfer(h, nullptr, false);
    return FC_OK;
  };
  const auto tw0 = std::chrono::steady_clock::now();
  FC_CUDA(cudaEventSynchronize(q->ev_index[p]));
  slow_wait_note("commit: index phase event", tw0);
  const Counters c = *q->hctr[p];
  h->host_free = c.free_count;
  info->unique = c.unique;
  info->free_count = c.free_count;
  info->candidates = c.candidates;
  h->last_needed = 0;
  h->last_misses = 0;
  if (c.err) {
    // nothing was mutated; the transfer kernel was gated off as well
    FC_CUDA(cudaStreamWaitEvent(st, q->ev_xfer[p], 0));
    FC_CUDA(cudaEventRecord(q->ev_commit[p], st));
    q->has_commit[p] = true;
    FC_TRY_E(launch_next_xfer());
    if (c.err == FC_ERR_ID_OUT_OF_RANGE) info->bad_id = (c.lo != LLONG_MAX) ? c.lo : c.hi;
    return c.err;
  }
  AsyncWB* a = h->awb;
  if (c.needed > a->rows) FC_TRY_E(engine_grow(h, c.needed));  // more victims than a stage holds
  const int b = a->cur;
  if (a->rows_in[b] > 0) {  // stage b still holds a job (the previous commit could not free it: a synchronous
                            // prepare ran between them); this batch's staging may still read its marks
    FC_CUDA(cudaStreamWaitEvent(st, q->ev_xfer[p], 0));
    // the stream (not the host) waits until the host threads have scattered that job;
    // fall back to a host wait when stream memory operations are unavailable
    WaitValueFn wv = std::getenv("FC_HOST_WAIT") ? nullptr : wait_value_fn();
    if (!wv || wv(reinterpret_cast<CUstream>(st), a->done_dev, (cuuint32_t)a->seq_of[b], CU_STREAM_WAIT_VALUE_GEQ) !=
                   CUDA_SUCCESS) {
      const auto t0 = std::chrono::steady_clock::now();
      wait_seq(a, a->seq_of[b]);
      h->prof[5] += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    }
    k_clear_pending<<<grid_for(a->rows_in[b], kNT, kSMs * 4), kNT, 0, st>>>(
        a->sranks[b], a->rows_in[b], a->pending, (int32_t)(b * a->rows), a->rows,
        a->rows_on_dev[b] ? a->dev_rows + b : nullptr);
    a->rows_in[b] = 0;
    a->rows_on_dev[b] = false;
  }
  trace_mark(h, T_COMMIT_BEGIN, st);
  PipeArgs x = pipe_args(h, p);
  // Free the stage the next commit will use now, before the next staging is launched: wait
  // (on the stream) for its last host job -- kWbBufs - 1 commits old -- and drop the pending
  // marks that still point into it, so the next staging reads those rows from the slow tier.
  // Queued first, so that the wait (it polls host memory) overlaps the current staging's
  // tail. This batch's staging may read those marks meanwhile: the job is done, so the stage
  // rows and the slow-tier rows are equal, and stage nb is rewritten only by the next commit.
  const int nb = c.needed > 0 ? (b + 1) % kWbBufs : b;
  if (nb != b && a->rows_in[nb] > 0) {
    WaitValueFn wv = std::getenv("FC_HOST_WAIT") ? nullptr : wait_value_fn();
    if (!wv || wv(reinterpret_cast<CUstream>(st), a->done_dev, (cuuint32_t)a->seq_of[nb], CU_STREAM_WAIT_VALUE_GEQ) !=
                   CUDA_SUCCESS) {
      const auto t0 = std::chrono::steady_clock::now();
      wait_seq(a, a->seq_of[nb]);
      h->prof[5] += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    }
    k_clear_pending<<<grid_for(a->rows_in[nb], kNT, kSMs * 4), kNT, 0, st>>>(
        a->sranks[nb], a->rows_in[nb], a->pending, (int32_t)(nb * a->rows), a->rows,
        a->rows_on_dev[nb] ? a->dev_rows + nb : nullptr);
    a->rows_in[nb] = 0;
    a->rows_on_dev[nb] = false;
  }
  // The victims go to the write-back stage without waiting for this batch's staging: the
  // staging reads only ranks that are not resident, and never stage b, whose marks the
  // previous commit cleared before launching it (as above). Only the admission needs the
  // staged rows, so the critical path from the end of one staging to the start of the
  // next is the admission copy alone.
  if (c.needed > 0) {
    FC_CUDA(cudaMemsetAsync(a->dev_rows + b, 0, sizeof(int32_t), st));
    if (a->vec) k_evict_commit<true><<<kSMs * 8, kNT, 0, st>>>(x);
    else k_evict_commit<false><<<kSMs * 8, kNT, 0, st>>>(x);
  }
  FC_CUDA(cudaStreamWaitEvent(st, q->ev_xfer[p], 0));
  if (c.misses > 0) {
    if (a->vec) k_admit_commit<true><<<kSMs * 8, kNT, 0, st>>>(x);
    else k_admit_commit<false><<<kSMs * 8, kNT, 0, st>>>(x);
  }
  FC_CUDA(cudaGetLastError());
  trace_mark(h, T_COMMIT_END, st);
  FC_CUDA(cudaEventRecord(q->ev_commit[p], st));
  q->has_commit[p] = true;
  FC_TRY_E(launch_next_xfer());
  if (c.misses > q->arows) FC_TRY_E(pipe_grow_admission(h, c.misses));  // this commit copied the overflow itself
  h->last_wb_dev = c.needed > 0 ? a->dev_rows + b : nullptr;
  if (c.needed > 0) {  // ship the write-back stage (upper bound: every victim) D2H on the side stream
    {  // the dispatcher must have consumed d2h[b] of the previous job on stage b before it is re-recorded
      std::unique_lock<std::mutex> lk(a->m);
      const auto tw1 = std::chrono::steady_clock::now();
      a->cv_started.wait(lk, [&] { return a->started_seq >= a->seq_of[b]; });
      slow_wait_note("commit: previous write-back job on this stage to start", tw1);
    }
    // The dirty filter ran on device: the host learns the write-back count W only when the
    // commit has run. While most victims come back dirty (training: every victim was just
    // updated) the whole victim stage is queued D2H right behind the commit, with no host
    // round trip; once they are mostly clean (inference, read-mostly phases) only the count
    // comes back here and the copier thread ships exactly W rows. Either way the host
    // scatters exactly W rows. FC_WB_EXACT=1 always takes the exact path.
    static const int exact_env = std::getenv("FC_WB_EXACT") ? std::atoi(std::getenv("FC_WB_EXACT")) : -1;
    bool ship_all;
    {
      std::lock_guard<std::mutex> lk(a->m);
      ship_all = exact_env == -1 ? a->dirty_frac >= 0.5 : exact_env == 0;
    }
    FC_CUDA(cudaStreamWaitEvent(a->side, q->ev_commit[p], 0));
    FC_CUDA(cudaMemcpyAsync(a->hrows + b, a->dev_rows + b, sizeof(int32_t), cudaMemcpyDeviceToHost, a->side));
    if (ship_all) {
      FC_CUDA(cudaMemcpyAsync(a->hranks[b], a->sranks[b], (size_t)c.needed * 4, cudaMemcpyDeviceToHost, a->side));
      FC_CUDA(cudaMemcpyAsync(a->hstage[b], a->stage[b], (size_t)c.needed * h->dim * 4, cudaMemcpyDeviceToHost,
                              a->side));
      if (h->sw)
        FC_CUDA(cudaMemcpyAsync(a->hsstage[b], a->sstage[b], (size_t)c.needed * h->sw * 4, cudaMemcpyDeviceToHost,
                                a->side));
    }
    FC_CUDA(cudaEventRecord(a->d2h[b], a->side));
    {
      std::lock_guard<std::mutex> lk(a->m);
      const uint64_t seq = a->next_seq++;
      Job j{b, -1, seq};
      j.victims = c.needed;
      j.shipped = ship_all;
      a->qc.push_back(j);
      a->seq_of[b] = seq;
      a->d2h_bytes += ship_all ? c.needed * (4 + 4 * (int64_t)(h->dim + h->sw)) : 0;
    }
    a->cv_qc.notify_one();
    a->rows_in[b] = c.needed;
    a->rows_on_dev[b] = true;
    a->cur = (a->cur + 1) % kWbBufs;
  }
  info->misses = c.misses;
  info->hits = c.unique - c.misses;
  info->evictions = c.needed;
  info->rows_to_slow = -1;  // decided on device by the commit (dirty filter); see fc_profile
  h->last_needed = c.needed;
  h->last_misses = c.misses;
  h->ev_src = q->ib[p].evicted;
  h->ad_src = q->ib[p].admitted;
  if (h->profile) {
    for (int par = 0; par < 2; ++par) harvest_xfer_time(h, par, false);  // stagings that have finished
    h->prof[2] += 1;
    h->prof[3] += 4.0 * (h->dim + h->sw) * (double)c.misses;
    h->prof[4] += 4.0 * (h->dim + h->sw) * (double)c.needed;
  }
  return FC_OK;
}

// Device / pinned-host bytes the engine and the pipeline hold (fc_memory_bytes):
// out = {stage bytes (device), id-space bytes (pending marks), other device bytes,
//        pinned host staging bytes, write-back stage rows, admission stage rows,
//        device bytes reserved by these allocations (2 MiB pages)}
void engine_memory(const fc_cache* h, int64_t* out) {
  for (int i = 0; i < 7; ++i) out[i] = 0;
  if (const AsyncWB* a = h->awb) {
    out[0] += a->stage_bytes;
    out[1] += 4 * h->num_ids;
    out[2] += a->fixed_bytes - 4 * h->num_ids;
    out[3] += kWbBufs * (int64_t)a->rows * (4 * (int64_t)(h->dim + h->sw) + 4);
    out[4] = a->rows;
    out[6] += reserved_bytes(a->stage_bytes) + reserved_bytes(a->fixed_bytes);
  }
  if (const Pipe* q = h->pipe) {
    out[0] += q->stage_bytes;
    out[2] += q->fixed_bytes;
    out[5] = q->arows;
    out[6] += reserved_bytes(q->stage_bytes) + reserved_bytes(q->fixed_bytes);
  }
}

}  // namespace fc
