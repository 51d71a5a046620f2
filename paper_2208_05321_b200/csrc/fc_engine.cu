// Async write-back engine (engine 1).
//
// The paired zero-copy kernel (engine 0, fc_rows.cu) moves victims and admissions
// with SM loads/stores over PCIe; concurrent SM-issued reads and writes top out near
// 75 GB/s on this box (tools/zerocopy_bench.cu) where the DMA engines reach ~100.
// Engine 1 takes the write-back direction off the SMs and off the critical path:
//
//   prepare t:  victims' dirty rows are compacted into HBM stage[t%2] and marked
//               pending[rank] = (t%2, k); admissions read their row from the newest
//               copy: the HBM stage when the rank is pending, else the pinned slow
//               tier (zero-copy, the H2D direction alone);
//   after sync: stage[t%2] (+ ranks) goes D2H by cudaMemcpyAsync on a side stream
//               into pinned staging, and a host thread pool scatters the rows into
//               the slow tier at their ranks — overlapped with the pooled forward /
//               backward of step t and the index work of step t+1;
//   prepare t+2: waits for that job, then clears the pending marks that still point
//               into stage[t%2] before reusing it.
//
// Jobs run strictly FIFO so a rank written back twice lands its newest value last.
// `flush` drains every job before its own write-back, so after flush the slow tier
// is authoritative exactly as in the reference.
#include <emmintrin.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <mutex>
#include <thread>
#include <vector>

#include "fc_rowutil.cuh"

namespace fc {

struct Job {
  int buf;
  int64_t rows;
  uint64_t seq;
};

struct AsyncWB {
  int32_t* pending = nullptr;   // device int32[num_ids], -1 or buf*C + k
  float* stage[2] = {nullptr, nullptr};
  float* sstage[2] = {nullptr, nullptr};
  int32_t* sranks[2] = {nullptr, nullptr};
  float* hstage[2] = {nullptr, nullptr};   // pinned
  float* hsstage[2] = {nullptr, nullptr};
  int32_t* hranks[2] = {nullptr, nullptr};
  int64_t rows_in[2] = {0, 0};             // rows currently staged in each buffer
  uint64_t seq_of[2] = {0, 0};             // job sequence number using each buffer
  cudaStream_t side = nullptr;
  cudaEvent_t d2h[2] = {nullptr, nullptr};
  int cur = 0;
  int device = 0;

  // FIFO scatter jobs, one dispatcher + helpers
  std::mutex m;
  std::condition_variable cv_q, cv_done, cv_help, cv_helped;
  std::deque<Job> q;
  uint64_t next_seq = 1, done_seq = 0;
  bool stop = false;
  std::thread dispatcher;
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
};

void engine_stats(fc_cache* h, double* out) {
  AsyncWB* a = h->awb;
  if (!a) {
    out[0] = out[1] = 0;
    return;
  }
  std::lock_guard<std::mutex> lk(a->m);
  out[0] = a->scatter_ms;
  out[1] = (double)a->jobs_done;
  a->scatter_ms = 0;
  a->jobs_done = 0;
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
    a->cv_help.wait(lk, [&] { return a->stop || a->gen != seen; });
    if (a->stop) return;
    seen = a->gen;
    lk.unlock();
    scatter_range(a);
    lk.lock();
    if (--a->helpers_left == 0) a->cv_helped.notify_all();
  }
}

static void dispatcher_main(AsyncWB* a) {
  cudaSetDevice(a->device);
  std::unique_lock<std::mutex> lk(a->m);
  while (true) {
    a->cv_q.wait(lk, [&] { return a->stop || !a->q.empty(); });
    if (a->stop && a->q.empty()) return;
    Job j = a->q.front();
    a->q.pop_front();
    lk.unlock();
    cudaEventSynchronize(a->d2h[j.buf]);  // the staged rows are in pinned memory
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
    a->jobs_done += 1;
    a->done_seq = j.seq;
    a->cv_done.notify_all();
  }
}

static void wait_seq(AsyncWB* a, uint64_t seq) {
  std::unique_lock<std::mutex> lk(a->m);
  a->cv_done.wait(lk, [&] { return a->done_seq >= seq; });
}

// ------------------------------------------------------------------ kernels
__global__ void k_clear_pending(const int32_t* __restrict__ ranks, int64_t n, int32_t* pending, int32_t base,
                                int32_t cap) {
  for (int64_t k = (int64_t)blockIdx.x * kNT + threadIdx.x; k < n; k += (int64_t)gridDim.x * kNT) {
    const int r = ranks[k];
    if (pending[r] == base + (int32_t)k) pending[r] = -1;  // unless re-staged since
  }
  (void)cap;
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
  float* stage[2];
  float* sstage[2];
  int32_t* sranks;
  int buf;
  int32_t cap;
  int always;
  Counters* c;
  Units ud, us;
};

// victims -> slot, dirty filter, compacted staging into stage[buf] + pending marks, state cleared
__global__ void __launch_bounds__(kNT) k_evict_async(EngArgs x) {
  __shared__ int sm[kNT / 32 + 1];
  if (!gate_open(x.c, G_EVICT)) return;
  const int needed = x.c->needed;
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * kNT + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * kNT) >> 5;
  int wb_count = 0;
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
    // rows: lane i's victim row fast[s_i] -> stage[buf][k_i]
    const int total = 32 * x.ud.upr;
    for (int u0 = 0; u0 < total; u0 += 32 * 4) {
      float4 val[4];
      int dk[4], cc[4];
      bool aa[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int u = u0 + q * 32 + lane;
        const int rr = min(x.ud.row(u), 31);
        cc[q] = (u - rr * x.ud.upr) * 4;
        const int sr = __shfl_sync(FC_FULL, s, rr);
        dk[q] = __shfl_sync(FC_FULL, k, rr);
        aa[q] = __shfl_sync(FC_FULL, (int)wb, rr) && u < total;
        if (aa[q]) val[q] = ld4(x.fast + (int64_t)sr * x.D + cc[q]);
      }
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (aa[q]) st4(x.stage[x.buf] + (int64_t)dk[q] * x.D + cc[q], val[q]);
    }
    if (x.S) {
      const int totals = 32 * x.us.upr;
      for (int u = lane; u < totals; u += 32) {
        const int rr = min(x.us.row(u), 31);
        const int c = (u - rr * x.us.upr) * 4;
        const int sr = __shfl_sync(FC_FULL, s, rr);
        const int kr = __shfl_sync(FC_FULL, k, rr);
        if (__shfl_sync(FC_FULL, (int)wb, rr))
          st4(x.sstage[x.buf] + (int64_t)kr * x.S + c, ld4(x.fstate + (int64_t)sr * x.S + c));
      }
    }
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
    wb_count += wb;
  }
  (void)wb_count;
  (void)sm;
  if (blockIdx.x == 0 && threadIdx.x == 0) x.c->free_count += needed;
}

// admissions: newest copy of each admitted rank -> its target slot
__global__ void __launch_bounds__(kNT) k_admit_async(EngArgs x) {
  if (!gate_open(x.c, G_OK)) return;
  const int m = x.c->misses;
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * kNT + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * kNT) >> 5;
  for (int64_t base = warp * 32; base < m; base += nwarps * 32) {
    const int64_t j = base + lane;
    const bool act = j < m;
    int r = 0, s = 0, pk = -1;
    if (act) {
      r = x.admitted[j];
      s = x.target[j];
      pk = x.pending[r];
    }
    const int total = 32 * x.ud.upr;
    for (int u0 = 0; u0 < total; u0 += 32 * 4) {
      float4 val[4];
      int ds[4], cc[4];
      bool aa[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int u = u0 + q * 32 + lane;
        const int rr = min(x.ud.row(u), 31);
        cc[q] = (u - rr * x.ud.upr) * 4;
        const int rq = __shfl_sync(FC_FULL, r, rr);
        const int pq = __shfl_sync(FC_FULL, pk, rr);
        ds[q] = __shfl_sync(FC_FULL, s, rr);
        aa[q] = __shfl_sync(FC_FULL, (int)act, rr) && u < total;
        if (aa[q]) {
          const float* src = pq >= 0 ? x.stage[pq / x.cap] + (int64_t)(pq % x.cap) * x.D
                                     : x.slow + (int64_t)rq * x.ld;
          val[q] = ld4(src + cc[q]);
        }
      }
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (aa[q]) st4(x.fast + (int64_t)ds[q] * x.D + cc[q], val[q]);
    }
    if (x.S) {
      const int totals = 32 * x.us.upr;
      for (int u = lane; u < totals; u += 32) {
        const int rr = min(x.us.row(u), 31);
        const int c = (u - rr * x.us.upr) * 4;
        const int rq = __shfl_sync(FC_FULL, r, rr);
        const int pq = __shfl_sync(FC_FULL, pk, rr);
        const int sq = __shfl_sync(FC_FULL, s, rr);
        if (__shfl_sync(FC_FULL, (int)act, rr)) {
          const float* src = pq >= 0 ? x.sstage[pq / x.cap] + (int64_t)(pq % x.cap) * x.S
                                     : x.sstate + (int64_t)rq * x.sld;
          st4(x.fstate + (int64_t)sq * x.S + c, ld4(src + c));
        }
      }
    }
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
  if (!vec_ok_engine(h)) {
    set_error("async engine needs dim %% 4 == 0 and 16-byte aligned rows");
    return FC_ERR_BAD_ARG;
  }
  AsyncWB* a = new AsyncWB();
  a->h = h;
  a->device = h->device;
  const size_t C = (size_t)h->capacity;
  cudaError_t e = cudaMalloc(&a->pending, (size_t)h->num_ids * 4);
  if (e == cudaSuccess) e = cudaMemset(a->pending, 0xff, (size_t)h->num_ids * 4);
  for (int b = 0; b < 2 && e == cudaSuccess; ++b) {
    e = cudaMalloc(&a->stage[b], C * h->dim * 4);
    if (e == cudaSuccess) e = cudaMalloc(&a->sranks[b], C * 4);
    if (e == cudaSuccess) e = cudaHostAlloc(&a->hstage[b], C * h->dim * 4, cudaHostAllocDefault);
    if (e == cudaSuccess) e = cudaHostAlloc(&a->hranks[b], C * 4, cudaHostAllocDefault);
    if (e == cudaSuccess && h->sw) e = cudaMalloc(&a->sstage[b], C * h->sw * 4);
    if (e == cudaSuccess && h->sw) e = cudaHostAlloc(&a->hsstage[b], C * h->sw * 4, cudaHostAllocDefault);
    // the dispatcher sleeps on these (a spinning cudaEventSynchronize would contend for
    // the driver with the caller's launches)
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&a->d2h[b], cudaEventDisableTiming | cudaEventBlockingSync);
  }
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&a->side, cudaStreamNonBlocking);
  h->awb = a;
  if (e != cudaSuccess) {
    engine_release(h);
    return cuda_fail(e, "engine_set");
  }
  unsigned hw = std::thread::hardware_concurrency();
  int nh = (int)std::max(1u, std::min(7u, hw > 4 ? hw / 2 - 1 : 1u));  // half the cores: leave the rest to the caller
  if (const char* env = std::getenv("FC_SCATTER_THREADS")) nh = std::max(0, std::atoi(env) - 1);
  for (int i = 0; i < nh; ++i) a->helpers.emplace_back(helper_main, a);
  a->dispatcher = std::thread(dispatcher_main, a);
  h->engine = 1;
  return FC_OK;
}

int engine_begin(fc_cache* h, cudaStream_t st) {
  if (h->engine != 1) return FC_OK;
  AsyncWB* a = h->awb;
  const int b = a->cur;
  if (a->rows_in[b] > 0) {  // stage[b] still holds rows from two prepares ago
    const auto t0 = std::chrono::steady_clock::now();
    wait_seq(a, a->seq_of[b]);
    h->prof[5] += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    k_clear_pending<<<grid_for(a->rows_in[b], kNT, kSMs * 4), kNT, 0, st>>>(a->sranks[b], a->rows_in[b], a->pending,
                                                                            (int32_t)(b * h->capacity), h->capacity);
    a->rows_in[b] = 0;
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
  x.stage[0] = a->stage[0];
  x.stage[1] = a->stage[1];
  x.sstage[0] = a->sstage[0];
  x.sstage[1] = a->sstage[1];
  x.sranks = a->sranks[a->cur];
  x.buf = a->cur;
  x.cap = h->capacity;
  x.always = h->write_back == FC_WB_ALWAYS;
  x.c = h->ctr;
  x.ud = units_for(h->dim);
  x.us = units_for(h->sw ? h->sw : 4);
  return x;
}

int engine_evict(fc_cache* h, cudaStream_t st) {
  EngArgs x = eng_args(h);
  k_evict_async<<<kSMs * 8, kNT, 0, st>>>(x);
  FC_CUDA(cudaGetLastError());
  return FC_OK;
}

int engine_admit(fc_cache* h, cudaStream_t st) {
  EngArgs x = eng_args(h);
  k_admit_async<<<kSMs * 4, kNT, 0, st>>>(x);
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
      a->q.push_back(Job{b, rows, seq});
      a->seq_of[b] = seq;
    }
    a->cv_q.notify_one();
    a->rows_in[b] = rows;
    a->cur ^= 1;
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

void engine_release(fc_cache* h) {
  AsyncWB* a = h->awb;
  if (!a) return;
  {
    std::lock_guard<std::mutex> lk(a->m);
    a->stop = true;
  }
  a->cv_q.notify_all();
  a->cv_help.notify_all();
  if (a->dispatcher.joinable()) a->dispatcher.join();
  for (auto& t : a->helpers)
    if (t.joinable()) t.join();
  cudaFree(a->pending);
  for (int b = 0; b < 2; ++b) {
    cudaFree(a->stage[b]);
    cudaFree(a->sranks[b]);
    cudaFree(a->sstage[b]);
    cudaFreeHost(a->hstage[b]);
    cudaFreeHost(a->hranks[b]);
    cudaFreeHost(a->hsstage[b]);
    if (a->d2h[b]) cudaEventDestroy(a->d2h[b]);
  }
  if (a->side) cudaStreamDestroy(a->side);
  delete a;
  h->awb = nullptr;
}

}  // namespace fc
