// Internal declarations shared by the freqcache_b200 translation units.
//
// Device-resident layout of one cache (one reference CacheStack,
// /root/reference/pkg/src/freqcache/cache_manager.py:441-562):
//
//   rank_of       int32[num_ids]   IdxMap.rank_of (freq_stats.py:52-73)
//   rank_to_slot  int32[num_ids]   CacheState.rank_to_slot (-1 = ABSENT)
//   slot_to_rank  int32[C]         CacheState.slot_to_rank (-1 = EMPTY)
//   dirty         uint8[C]
//   fast          fp32[C, D]       FastTierStore.slots (row stride D)
//   fast_state    fp32[C, S]       optimizer state cached with the row (S may be 0)
//   res_bits      u32[ceil(num_ids/32)]  resident-rank bitmap (rank space)
//   free_bits     u32[ceil(C/32)]        empty-slot bitmap (slot space)
//   id_bits / miss_bits / prot_bits      per-batch bitmaps, all-zero between calls
//   aux           int32[num_ids]   per-batch id counts, then unique positions; zero between calls
//
// Ordered outputs (ascending unique ids, ascending admitted ranks, ascending free
// slots, descending victim ranks) all come from one primitive: an ordered
// compaction of set bits of a bitmap (count -> scan -> emit). Bitmaps over the id
// or rank space are a 1-pass radix (counting) sort: O(N + num_ids/32) with no
// key comparisons, instead of np.unique / np.sort / np.partition.
#pragma once

#include <cuda_runtime.h>
#include <pthread.h>
#include <stdint.h>

#include <algorithm>
#include <vector>

#include "../../include/freqcache_b200.h"

#define FC_FULL 0xffffffffu

namespace fc {

constexpr int kNT = 256;                 // threads per block for streaming kernels
constexpr int kSMs = 148;                // B200 SM count
constexpr int kMaxScanBlocks = kSMs * 8; // blocks of one bitmap pass (<= 1184)

enum Gate : int { G_ALWAYS = 0, G_OK = 1, G_EVICT = 2, G_ADMIT = 3, G_EMITTED = 4 };

// Per-call device counters. `free_count` is persistent across calls.
struct Counters {
  int32_t err;
  int32_t emitted;      // id compaction produced outputs (cleanup needed)
  long long lo;         // smallest negative id seen
  long long hi;         // largest id >= num_ids seen
  int32_t unique;
  int32_t misses;
  int32_t needed;
  int32_t free_count;
  int32_t wb_rows;
  int32_t candidates;
  int32_t win_evict[2]; // order-index window of the victim emission
  int32_t win_admit[2];
  int32_t flush_rows;
  int32_t bad_slot;
};

struct AsyncWB;  // async write-back engine state (fc_engine.cu)
struct Pipe;     // prefetch pipeline state (fc_engine.cu)

// Per-prepare index buffers of the prefetch pipeline (double-buffered by batch parity).
struct IndexBufs {
  Counters* ctr;
  int32_t* evicted;   // [C] victim ranks, descending
  int32_t* vslots;    // [C] their slots
  int32_t* admitted;  // [C] admitted ranks, ascending
  int32_t* target;    // [C] their slots, ascending
};

}  // namespace fc

struct fc_cache {
  int64_t num_ids;
  int32_t capacity;
  int32_t dim;
  int32_t sw;             // optimizer-state width
  int32_t write_back;
  int32_t evict_mode;
  int64_t buffer_bytes;
  int device;
  int64_t nw_ids;         // words of a rank/id bitmap (padded)
  int64_t nw_slots;       // words of the slot bitmap (padded)

  int32_t* rank_of;
  int32_t* rank_to_slot;
  int32_t* slot_to_rank;
  uint8_t* dirty;
  float* fast;
  float* fast_state;
  uint32_t* res_bits;
  uint32_t* free_bits;
  uint32_t* id_bits;
  uint32_t* miss_bits;
  uint32_t* prot_bits;
  int32_t* aux;

  int32_t* evicted_ranks;   // [C] descending
  int32_t* victim_slots;    // [C]
  int32_t* wb_ranks;        // [C] rank per staged write-back row or -1
  float* wb_stage;          // [C, D] engine 0 only, allocated on its first eviction
  float* wb_stage_state;    // [C, S]
  int32_t* admitted_ranks;  // [C] ascending
  int32_t* target_slots;    // [C] ascending
  int32_t* block_cnt;       // [kMaxScanBlocks + 1]
  int32_t* block_cnt2;      // second scan lane (concurrent compactions)
  fc::Counters* ctr;        // device (synchronous verbs)
  void* arena;              // the allocation every array above (but wb_stage) is carved from
  int64_t arena_bytes;
  fc::Counters* ctr_host;   // pinned mirror
  fc::Counters* live;       // counters of the last call: holds the current free_count
  cudaEvent_t done;

  // scratch for sort-based kernels (backward / scatter_update), grown on demand
  void* scratch;
  size_t scratch_bytes;
  // the fused backward's last kernel clears the sort state for the next sort: this many
  // bytes from sort_zero_for (inside `scratch`; the state's offset depends on the batch size)
  // are zero
  void* sort_zero_for;
  size_t sort_zero_bytes;

  float* slow;              // slow tier rows, device-mapped pointer
  int64_t slow_ld;
  float* slow_state;
  int64_t state_ld;
  float* slow_host;         // the same rows, host pointer (host-side scatter)
  float* slow_state_host;

  int32_t last_needed;
  int32_t last_misses;
  int32_t host_free;        // host mirror of free_count

  // optional per-kernel timing (fc_profile): events around the host-link transfer kernel
  int profile;
  cudaEvent_t pev[4];
  double prof[8];           // prepare_ms, xfer_ms, calls, host-link bytes, write-back bytes, host wait ms,
                            // timed transfer launches (pipeline)

  // async write-back engine (fc_engine.cu); engine 0 = paired zero-copy kernel
  int engine;
  fc::AsyncWB* awb;
  fc::Pipe* pipe;           // prefetch pipeline (fc_prepare_begin / fc_prepare_commit), lazily created
  void* trace;              // std::vector of tagged events (fc_trace), NULL when off
  const int32_t* last_wb_dev; // device count of the last pipeline commit's write-backs (or NULL)
  const int32_t* ev_src;    // device lists read by fc_last_events (last prepare's buffers)
  const int32_t* ad_src;
};

namespace fc {
// engine hooks (fc_engine.cu)
int engine_set(fc_cache* h, int engine);
int engine_begin(fc_cache* h, cudaStream_t st);              // before a prepare's kernels
int engine_evict(fc_cache* h, cudaStream_t st);              // replaces k_evict_rows
int engine_admit(fc_cache* h, cudaStream_t st);              // replaces k_transfer_rows
int engine_after_prepare(fc_cache* h, cudaStream_t st);      // after the prepare's sync
int engine_drain(fc_cache* h);                               // all write-backs landed in the slow tier
int engine_drain_stream(fc_cache* h, cudaStream_t st);       // the same, as a wait on `st`
int engine_threads(const fc_cache* h);                       // host scatter threads of the async engine
int engine_reserve(fc_cache* h, int64_t n, cudaStream_t st);  // sync prepare: stages hold this batch's victims
int engine_grow(fc_cache* h, int64_t need);                  // write-back stages of >= need rows
int32_t initial_stage_rows(const fc_cache* h);               // staging rows before any growth
void engine_memory(const fc_cache* h, int64_t* out);          // engine + pipeline allocations (fc_memory_bytes)
void engine_release(fc_cache* h);
void engine_stats(fc_cache* h, double* out);                 // host scatter ms, jobs, rows, D2H bytes (then reset)
// prefetch pipeline (fc_engine.cu)
int pipe_begin(fc_cache* h, const void* ids, int ids_bytes, int64_t n, int32_t* uids, int32_t* ucnt, int32_t* uranks,
               int32_t* uslots, int32_t* inverse, cudaStream_t st);
int pipe_commit(fc_cache* h, cudaStream_t st, fc_prepare_info* info);
bool pipe_outstanding(const fc_cache* h);
int pipe_order(fc_cache* h, cudaStream_t st);
int pipe_sync_commits(fc_cache* h);
int pipe_launch_xfer(fc_cache* h, cudaStream_t after, bool from_update);  // after: extra dependency
void pipe_release(fc_cache* h);
}  // namespace fc

namespace fc {

void set_error(const char* fmt, ...);
// host placement (fc_api.cu): the GPU's local CPUs (sysfs local_cpulist), thread binding
std::vector<int> device_local_cpus(int device);
void bind_thread(pthread_t t, const std::vector<int>& cpus);
// timeline tracing (fc_trace): record a tagged event on `st` when tracing is on
void trace_mark(fc_cache* h, int tag, cudaStream_t st);
enum TraceTag : int { T_INDEX_BEGIN = 1, T_INDEX_END = 2, T_XFER_BEGIN = 3, T_XFER_END = 4, T_COMMIT_BEGIN = 5,
                      T_COMMIT_END = 6, T_HOST_WAIT_END = 7 };
int cuda_fail(cudaError_t e, const char* what);

#define FC_CUDA(call)                                 \
  do {                                                \
    cudaError_t e__ = (call);                         \
    if (e__ != cudaSuccess) return fc::cuda_fail(e__, #call); \
  } while (0)

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// One cudaMalloc carved into many arrays (256-byte aligned): a cache's fixed arrays, the
// engine's stages and the pipeline's buffers each live in one such arena, so the device
// memory they take is the arena sizes rounded to the allocation granularity -- which is
// what fc_memory_bytes reports.
struct Arena {
  struct Part {
    void** p;
    size_t off;
  };
  std::vector<Part> parts;
  size_t bytes = 0;
  template <class T>
  void add(T** p, size_t count) {
    parts.push_back({reinterpret_cast<void**>(p), bytes});
    bytes += (std::max<size_t>(count, 1) * sizeof(T) + 255) & ~size_t(255);
  }
  // allocates and assigns every part; *base receives the allocation
  cudaError_t alloc(void** base) {
    cudaError_t e = cudaMalloc(base, std::max<size_t>(bytes, 256));
    if (e != cudaSuccess) return e;
    for (const Part& q : parts) *q.p = static_cast<char*>(*base) + q.off;
    return cudaSuccess;
  }
};
constexpr int64_t kAllocGranularity = 2 << 20;  // cudaMalloc reserves device memory in 2 MiB pages
inline int64_t reserved_bytes(int64_t b) { return b <= 0 ? 0 : (b + kAllocGranularity - 1) / kAllocGranularity * kAllocGranularity; }

inline int grid_for(int64_t items, int per_block, int max_blocks = kSMs * 8) {
  int64_t b = (items + per_block - 1) / per_block;
  if (b < 1) b = 1;
  if (b > max_blocks) b = max_blocks;
  return static_cast<int>(b);
}

// lanes per row group: enough lanes to cover a row with 16-byte (vec) or 4-byte accesses
inline int row_group(int width, bool vec) {
  int units = vec ? (width + 3) / 4 : width;
  int g = 1;
  while (g < units && g < 32) g <<= 1;
  return g;
}

// index-space kernels (fc_index.cu)
int launch_prepare(fc_cache* h, const void* ids, int ids_bytes, int64_t n, int32_t* uids, int32_t* ucnt,
                   int32_t* uranks, int32_t* uslots, int32_t* inverse, cudaStream_t st);
int launch_select_evictions(fc_cache* h, int64_t needed, const int64_t* prot, int64_t nprot, cudaStream_t st);
int launch_warmup_state(fc_cache* h, int64_t k, cudaStream_t st);
int launch_mark_dirty(fc_cache* h, const int64_t* slots, int64_t n, cudaStream_t st);
int launch_reset_counters(fc_cache* h, cudaStream_t st);
int launch_index_phase(fc_cache* h, const void* ids, int ids_bytes, int64_t n, int32_t* uids, int32_t* ucnt,
                       int32_t* uranks, int32_t* uslots, int32_t* inverse, const IndexBufs& b, Counters* publish,
                       int32_t* sort_hist, cudaStream_t st);
// the digit histograms a pipeline index phase made for this inverse (then forgotten), or NULL
const int32_t* pipe_take_sort_hist(fc_cache* h, const int32_t* inverse, int64_t n);
void pipe_forget_sort_hist(fc_cache* h, const int32_t* inverse);  // a synchronous prepare rewrites it

// row kernels (fc_rows.cu)
int launch_evict_rows(fc_cache* h, cudaStream_t st);
int launch_transfer_rows(fc_cache* h, cudaStream_t st);
int launch_flush(fc_cache* h, cudaStream_t st);
int launch_pool(fc_cache* h, const int32_t* uslots, const int32_t* inv, int64_t n, const void* offsets,
                int off_bytes, int64_t nbags, int include_last, const float* psw, int mode, float* out,
                cudaStream_t st);
int launch_gather_rows(fc_cache* h, const int32_t* slots, int64_t n, float* out, cudaStream_t st);
int launch_gather_from_peers(const float* const* src, const int64_t* src_off, const int64_t* seg, int W, int64_t n,
                             int D, float* out, cudaStream_t st);
int launch_pool_cols_to_peers(fc_cache* h, const int32_t* uslots, const int32_t* inv, int64_t n, const int64_t* seg,
                              int W, float* const* dst, const int64_t* dst_off, int64_t ld, int64_t col,
                              const float* psw, cudaStream_t st);
int launch_gather_cols_from_peers(const float* const* src, const int64_t* src_off, const int64_t* seg, int W,
                                  int64_t n, int D, int64_t ld, int64_t col, float* out, cudaStream_t st);
int launch_pool_to_peers(fc_cache* h, const int32_t* uslots, const int32_t* inv, int64_t n, const int64_t* seg, int W,
                         float* const* dst, const int64_t* dst_off, cudaStream_t st);
int launch_unique_add(fc_cache* h, const int32_t* uslots, int64_t u, const float* add, cudaStream_t st);
int launch_synthetic(fc_cache* h, const int32_t* uids, const int32_t* ucnt, const int32_t* uslots, int64_t u,
                     uint64_t salt, const float* colw, cudaStream_t st);
int launch_scatter_update(fc_cache* h, const int32_t* uslots, const int32_t* inv, const int32_t* ucnt,
                          int64_t u, int64_t n, const float* deltas, cudaStream_t st);
int launch_backward(fc_cache* h, const int32_t* uslots, const int32_t* inv, const int32_t* ucnt, int64_t u,
                    int64_t n, const void* offsets, int off_bytes, int64_t nbags, int include_last,
                    const float* psw, int mode, const float* grad, int optim, float lr, float eps,
                    cudaStream_t st);

// sort / scan helpers (fc_sort.cu)
size_t sort_scratch_bytes(int64_t n);
int radix_sort_pairs(const uint32_t* keys_in, const int32_t* vals_in, uint32_t* keys_out, int32_t* vals_out,
                     int64_t n, int key_bits, void* scratch, cudaStream_t st, bool state_zeroed = false,
                     const int32_t* ghist_pre = nullptr);
constexpr int kSortHistInts = 4 * 512;  // digit histograms of up to 4 passes of <= 9-bit digits
size_t sort_state_bytes(int64_t n, int key_bits);
int exclusive_scan_i32(const int32_t* in, int32_t* out, int64_t n, void* scratch, cudaStream_t st);
size_t scan_scratch_bytes(int64_t n);
int ensure_scratch(fc_cache* h, size_t bytes);
int ensure_scratch_buf(void** p, size_t* have, size_t bytes);
int launch_unique_grads(void** scratch, size_t* scratch_bytes, const int32_t* inv, int64_t u, int64_t n,
                        const void* offsets, int off_bytes, int64_t nbags, int include_last, const float* psw,
                        int mode, const float* grad, int D, float* gu, cudaStream_t st);
int launch_pool_rows(const float* rows, int D, const int32_t* uslots, const int32_t* inv, int64_t n,
                     const void* offsets, int off_bytes, int64_t nbags, int include_last, const float* psw, int mode,
                     float* out, cudaStream_t st);

// ---------------------------------------------------------------- device utils
__device__ __forceinline__ int warp_sum(int v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FC_FULL, v, o);
  return v;
}

// Block-wide exclusive scan of one int per thread. `sm` needs NT/32 + 1 ints.
template <int NT>
__device__ __forceinline__ int block_excl_scan(int v, int* sm, int& total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(FC_FULL, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) sm[wid] = x;
  __syncthreads();
  if (wid == 0) {
    int w = (lane < NT / 32) ? sm[lane] : 0;
    int s = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(FC_FULL, s, o);
      if (lane >= o) s += y;
    }
    if (lane < NT / 32) sm[lane] = s - w;
    if (lane == NT / 32 - 1) sm[NT / 32] = s;
  }
  __syncthreads();
  int r = x - v + sm[wid];
  total = sm[NT / 32];
  __syncthreads();
  return r;
}

template <int NT>
__device__ __forceinline__ int block_sum(int v, int* sm) {
  int t;
  block_excl_scan<NT>(v, sm, t);
  return t;
}

__device__ __forceinline__ bool gate_open(const Counters* c, int gate) {
  switch (gate) {
    case G_ALWAYS: return true;
    case G_OK: return c->err == 0;
    case G_EVICT: return c->err == 0 && c->needed > 0;
    case G_ADMIT: return c->err == 0 && c->misses > 0;
    case G_EMITTED: return c->emitted != 0;
  }
  return true;
}

}  // namespace fc
