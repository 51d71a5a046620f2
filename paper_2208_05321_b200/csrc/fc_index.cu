// Index-space kernels of prepare_cache (/root/reference/pkg/src/freqcache/cache_manager.py:234-348).
//
// Every ordered list the reference builds with a sort is produced here by an
// ordered compaction of a bitmap (count -> scan -> emit):
//
//   np.unique(ids, return_counts=True)      (:277)  -> id_bits   (id space, ascending)
//   np.sort(unique_ranks[miss_mask])        (:310)  -> miss_bits (rank space, ascending)
//   StaticFreqLfu.victim_ranks top-k        (:67-75,298-303) -> res_bits & ~prot_bits, last k set
//                                                    bits, emitted in descending order
//   state.free_slots()[:misses]             (:312-318) -> free_bits (slot space, first M)
//
// All kernels read their sizes from device counters, so one prepare is a fixed
// sequence of launches with a single host synchronisation at the end.
#include <algorithm>
#include <climits>
#include <cstddef>
#include <cstring>

#include "fc_internal.cuh"

namespace fc {

#define FC_TRY_I(expr)     \
  do {                     \
    int rc__ = (expr);     \
    if (rc__) return rc__; \
  } while (0)

// ------------------------------------------------------------------ word sources
struct ArrWords {
  uint32_t* w;
  __device__ __forceinline__ uint32_t operator()(int64_t i) const { return w[i]; }
  __device__ __forceinline__ void clear(int64_t i) const { w[i] = 0u; }
};

struct CandWords {  // resident and not protected by the current batch
  const uint32_t* res;
  const uint32_t* prot;
  __device__ __forceinline__ uint32_t operator()(int64_t i) const { return res[i] & ~prot[i]; }
  __device__ __forceinline__ void clear(int64_t) const {}
};

// ------------------------------------------------------------------ the primitive
// (the bodies take the block index so that two passes can share one launch, see
// launch_index_phase: every kernel boundary is expensive beside the miss staging)
template <class WF>
__device__ __forceinline__ void bits_count_body(WF wf, int64_t nwords, int64_t chunk, int32_t* cnt,
                                                const Counters* ctr, int gate, int blk) {
  __shared__ int sm[kNT / 32 + 1];
  if (!gate_open(ctr, gate)) return;
  const int64_t b0 = (int64_t)blk * chunk;
  const int64_t b1 = min(nwords, b0 + chunk);
  int c = 0;
  for (int64_t w = b0 + threadIdx.x; w < b1; w += kNT) c += __popc(wf(w));
  c = block_sum<kNT>(c, sm);
  if (threadIdx.x == 0) cnt[blk] = c;
}

template <class WF>
__global__ void __launch_bounds__(kNT) k_bits_count(WF wf, int64_t nwords, int64_t chunk, int32_t* cnt,
                                                    const Counters* ctr, int gate) {
  bits_count_body(wf, nwords, chunk, cnt, ctr, gate, blockIdx.x);
}

// Emit, with the block-offset scan folded in: every block sums the per-block counts
// before it (its base) and all of them (the total, <= kMaxScanBlocks loads per block),
// runs the finisher on the total itself (the finishers only set counters, so the
// blocks' identical writes are benign) and then emits its set bits in order.
template <class WF, class EM, class FIN>
__device__ __forceinline__ void bits_emit_body(WF wf, EM em, FIN fin, int64_t nwords, int64_t chunk,
                                               const int32_t* cnt, int nb, const int32_t* win, Counters* ctr,
                                               int gate, int blk) {
  __shared__ int sm[kNT / 32 + 1];
  __shared__ int s_base;
  __shared__ Counters lc;  // this block's view of the counters after the finisher
  if (!gate_open(ctr, gate)) return;
  int pre = 0, all = 0;
  for (int b = threadIdx.x; b < nb; b += kNT) {
    const int v = cnt[b];
    all += v;
    if (b < blk) pre += v;
  }
  pre = block_sum<kNT>(pre, sm);
  all = block_sum<kNT>(all, sm);
  if (threadIdx.x == 0) {
    s_base = pre;
    // every block applies the finisher to a private copy (it only derives fields from
    // the total and from fields earlier kernels set); block 0 alone publishes it, so
    // 1000+ blocks do not all write the same counters line
    lc = *ctr;
    fin(all, &lc);
    if (blk == 0) fin(all, ctr);
  }
  __syncthreads();
  if (!gate_open(&lc, gate)) return;  // the finisher may have raised an error
  int lo = 0, hi = INT_MAX;
  if (win != nullptr) {  // window fields read from the block's copy
    const int32_t* lw = reinterpret_cast<const int32_t*>(reinterpret_cast<const char*>(&lc) +
                                                         (reinterpret_cast<const char*>(win) -
                                                          reinterpret_cast<const char*>(ctr)));
    lo = lw[0];
    hi = lw[1];
  }
  const int base = s_base;
  const int bend = base + cnt[blk];
  if (!EM::kVisitAll && (bend <= lo || base >= hi)) return;
  EM e = em;
  e.init(&lc);
  const int64_t b0 = (int64_t)blk * chunk;
  const int64_t b1 = min(nwords, b0 + chunk);
  int run = base;
  int acc = 0;
  for (int64_t t0 = b0; t0 < b1; t0 += kNT) {
    const int64_t w = t0 + threadIdx.x;
    uint32_t x = (w < b1) ? wf(w) : 0u;
    int tot;
    int idx = run + block_excl_scan<kNT>(__popc(x), sm, tot);
    while (x) {
      const int bit = __ffs(x) - 1;
      x &= x - 1;
      if (idx >= lo && idx < hi) acc += e(w * 32 + bit, idx);
      ++idx;
    }
    if (EM::kClear && w < b1) wf.clear(w);
    run += tot;
  }
  if (EM::kCount) {
    acc = block_sum<kNT>(acc, sm);
    if (threadIdx.x == 0 && acc) atomicAdd(e.counter(ctr), acc);
  }
}

template <class WF, class EM, class FIN>
__global__ void __launch_bounds__(kNT) k_bits_emit(WF wf, EM em, FIN fin, int64_t nwords, int64_t chunk,
                                                   const int32_t* cnt, int nb, const int32_t* win, Counters* ctr,
                                                   int gate) {
  bits_emit_body(wf, em, fin, nwords, chunk, cnt, nb, win, ctr, gate, blockIdx.x);
}

// Two independent count passes in one launch (blocks [0, nb1) count the first bitmap).
template <class WF1, class WF2>
__global__ void __launch_bounds__(kNT) k_bits_count2(WF1 wf1, int64_t nw1, int64_t chunk1, int32_t* cnt1, int nb1,
                                                     int gate1, WF2 wf2, int64_t nw2, int64_t chunk2, int32_t* cnt2,
                                                     int gate2, const Counters* ctr) {
  if ((int)blockIdx.x < nb1) bits_count_body(wf1, nw1, chunk1, cnt1, ctr, gate1, blockIdx.x);
  else bits_count_body(wf2, nw2, chunk2, cnt2, ctr, gate2, blockIdx.x - nb1);
}

// An emit pass and an independent count pass in one launch (blocks [0, nb1) emit).
template <class WF1, class EM, class FIN, class WF2>
__global__ void __launch_bounds__(kNT) k_bits_emit_count(WF1 wf1, EM em, FIN fin, int64_t nw1, int64_t chunk1,
                                                         const int32_t* cnt1, int nb1, const int32_t* win, int gate1,
                                                         WF2 wf2, int64_t nw2, int64_t chunk2, int32_t* cnt2,
                                                         int gate2, Counters* ctr) {
  if ((int)blockIdx.x < nb1) bits_emit_body(wf1, em, fin, nw1, chunk1, cnt1, nb1, win, ctr, gate1, blockIdx.x);
  else bits_count_body(wf2, nw2, chunk2, cnt2, ctr, gate2, blockIdx.x - nb1);
}

template <class WF, class FIN, class EM>
static void compact(WF wf, FIN fin, EM em, int64_t nwords, int32_t* cnt, const int32_t* win, Counters* ctr,
                    int gate, cudaStream_t st) {
  // small bitmaps (the slot space) still get enough blocks to emit in parallel
  const int nb = grid_for(nwords, 128, kMaxScanBlocks);
  const int64_t chunk = (nwords + nb - 1) / nb;
  k_bits_count<WF><<<nb, kNT, 0, st>>>(wf, nwords, chunk, cnt, ctr, gate);
  k_bits_emit<WF, EM, FIN><<<nb, kNT, 0, st>>>(wf, em, fin, nwords, chunk, cnt, nb, win, ctr, gate);
}

// ------------------------------------------------------------------ unique ids (:268-289)
// Counts are aggregated per block in a shared-memory hash table before touching
// global memory: a Zipf head id occurs ~8% of a batch, and per-occurrence (or
// per-warp) global atomics on its counter serialise in one L2 slice.
constexpr int kMarkTile = 512;      // ids per block iteration (a batch spans ~800 blocks)
constexpr int kMarkHash = 4096;     // open-addressing slots (load <= 0.5)

template <typename IdT>
__global__ void __launch_bounds__(kNT) k_mark_ids(const IdT* __restrict__ ids, int64_t n, int64_t num_ids,
                                                  uint32_t* id_bits, int32_t* aux, Counters* c) {
  __shared__ int hk[kMarkHash];
  __shared__ int hc[kMarkHash];
  const int lane = threadIdx.x & 31;
  for (int e = threadIdx.x; e < kMarkHash; e += kNT) {
    hk[e] = -1;
    hc[e] = 0;
  }
  __syncthreads();
  for (int64_t tile = blockIdx.x; tile * kMarkTile < n; tile += gridDim.x) {
#pragma unroll
    for (int k = 0; k < kMarkTile / kNT; ++k) {
      const int64_t i = tile * kMarkTile + k * kNT + threadIdx.x;
      const bool valid = i < n;
      const long long id = valid ? (long long)ids[i] : 0;
      const bool inr = valid && id >= 0 && id < num_ids;
      if (valid && !inr) {
        if (id < 0) atomicMin(&c->lo, id);
        else atomicMax(&c->hi, id);
      }
      const int key = inr ? (int)id : -1;
      const unsigned peers = __match_any_sync(FC_FULL, key);
      if (inr && lane == __ffs(peers) - 1) {
        unsigned h = ((unsigned)key * 2654435761u) >> 20;  // 12-bit slot
        while (true) {
          const int prev = atomicCAS(&hk[h], -1, key);
          if (prev == -1 || prev == key) {
            atomicAdd(&hc[h], __popc(peers));
            break;
          }
          h = (h + 1) & (kMarkHash - 1);
        }
      }
    }
    __syncthreads();
    for (int e = threadIdx.x; e < kMarkHash; e += kNT) {
      const int key = hk[e];
      if (key >= 0) {
        atomicAdd(&aux[key], hc[e]);
        const uint32_t m = 1u << (key & 31);
        uint32_t* wp = &id_bits[key >> 5];
        if (!(*wp & m)) atomicOr(wp, m);
        hk[e] = -1;
        hc[e] = 0;
      }
    }
    __syncthreads();
  }
}

struct IdFin {
  int32_t cap;
  __device__ void operator()(int total, Counters* c) const {
    c->unique = total;
    if (c->lo != LLONG_MAX || c->hi != LLONG_MIN) c->err = FC_ERR_ID_OUT_OF_RANGE;        // :272-275
    else if (total > cap) c->err = FC_ERR_BATCH_EXCEEDS_CAPACITY;                          // :278-282
    c->emitted = (c->err == 0);
  }
};

// Ordered emission only places each id at its position; the gathers that depend
// on it run afterwards, one thread per unique id, with no barrier in between.
struct IdEmit {
  static constexpr bool kVisitAll = true, kClear = true, kCount = false;
  int32_t* aux;
  int32_t* uids;
  int ok;
  __device__ void init(const Counters* c) { ok = c->emitted; }
  __device__ int* counter(Counters*) const { return nullptr; }
  __device__ __forceinline__ int operator()(int64_t id, int p) const {
    if (!ok) aux[id] = 0;  // validation failed: undo the per-id counts, touch nothing else
    else uids[p] = (int32_t)id;
    return 0;
  }
};

// per unique id: count, rank (:283), slot or miss (:286-289), protection mark (:299).
// Three dependent random gathers per id (aux, rank_of, rank_to_slot): each thread
// works on kUiIlp ids at once so their loads overlap.
constexpr int kUiIlp = 4;

// sort_hist (pipeline only): also the digit histograms of the inverse this batch will have
// -- unique position p occurs cnt times -- in the layout the backward's radix sort reads
// ([passes][bins], digits of key_bits_for(u) bits), so the backward runs no histogram
// kernel of its own (a launch costs ~100 us on the compute stream beside the staging).
__global__ void __launch_bounds__(kNT) k_unique_info(const int32_t* __restrict__ uids, int32_t* aux,
                                                     const int32_t* __restrict__ rank_of,
                                                     const int32_t* __restrict__ rank_to_slot, uint32_t* prot,
                                                     uint32_t* miss, int32_t* __restrict__ ucnt,
                                                     int32_t* __restrict__ uranks, int32_t* __restrict__ uslots,
                                                     Counters* c, int32_t* sort_hist) {
  __shared__ int sh[kSortHistInts];
  if (!c->emitted) return;
  const int u = c->unique;
  const int lane = threadIdx.x & 31;
  const int stride = gridDim.x * kNT;
  int misses = 0;
  int passes = 0, dbits = 1, bins = 2;
  if (sort_hist) {  // key_bits_for(u) and radix_sort_pairs' digit split, on device
    int bits = 1;
    while ((1 << bits) < u) ++bits;
    passes = max(1, (bits + 8) / 9);
    dbits = max(1, (bits + passes - 1) / passes);
    bins = 1 << dbits;
    for (int i = threadIdx.x; i < passes * bins; i += kNT) sh[i] = 0;
    __syncthreads();
  }
  for (int base = (blockIdx.x * kNT + threadIdx.x) & ~31; base < u; base += stride * kUiIlp) {
    int id[kUiIlp], cnt[kUiIlp], r[kUiIlp], sl[kUiIlp];
    bool in[kUiIlp];
#pragma unroll
    for (int k = 0; k < kUiIlp; ++k) {
      const int p = base + k * stride + lane;
      in[k] = p < u;
      id[k] = in[k] ? uids[p] : 0;
    }
#pragma unroll
    for (int k = 0; k < kUiIlp; ++k) {
      cnt[k] = in[k] ? aux[id[k]] : 0;
      r[k] = in[k] ? rank_of[id[k]] : 0;
    }
#pragma unroll
    for (int k = 0; k < kUiIlp; ++k) sl[k] = in[k] ? rank_to_slot[r[k]] : 0;
#pragma unroll
    for (int k = 0; k < kUiIlp; ++k) {
      const int p = base + k * stride + lane;
      bool m = false;
      if (in[k]) {
        aux[id[k]] = p;  // position in the unique list, read by k_inverse
        ucnt[p] = cnt[k];
        uranks[p] = r[k];
        uslots[p] = sl[k];
        atomicOr(&prot[r[k] >> 5], 1u << (r[k] & 31));
        m = sl[k] < 0;
        if (m) atomicOr(&miss[r[k] >> 5], 1u << (r[k] & 31));
        for (int q = 0; q < passes; ++q) atomicAdd(&sh[q * bins + ((p >> (q * dbits)) & (bins - 1))], cnt[k]);
      }
      misses += __popc(__ballot_sync(FC_FULL, m));
    }
  }
  if (lane == 0 && misses) atomicAdd(&c->misses, misses);
  if (sort_hist) {
    __syncthreads();
    for (int i = threadIdx.x; i < passes * bins; i += kNT)
      if (sh[i]) atomicAdd(&sort_hist[i], sh[i]);
  }
}

template <typename IdT>
__global__ void __launch_bounds__(kNT) k_inverse(const IdT* __restrict__ ids, int64_t n, const int32_t* __restrict__ aux,
                                                 int32_t* __restrict__ inv, const Counters* c) {
  if (!c->emitted) return;
  for (int64_t i = (int64_t)blockIdx.x * kNT + threadIdx.x; i < n; i += (int64_t)gridDim.x * kNT)
    inv[i] = aux[(int64_t)ids[i]];
}

// ------------------------------------------------------------------ eviction count (:293-296)
__global__ void k_plan(Counters* c, int cap, int evict_mode) {
  if (c->err) return;
  const int m = c->misses, u = c->unique, fr = c->free_count;
  const int needed = evict_mode == FC_EVICT_OCCUPANCY_AWARE ? max(0, m - fr) : max(0, u - cap);
  c->needed = needed;
  if (fr + needed < m) c->err = FC_ERR_INSUFFICIENT_FREE_SLOTS;  // paper_literal (:313-317)
  c->win_admit[0] = 0;
  c->win_admit[1] = m;
}

// A row larger than the staging buffer (transmitter.py:85-88) -- launched only in that
// degenerate configuration, in the reference's order (cache_manager.py:298-323): the
// write-back of victims raises BEFORE any mutation when there is a row to write back
// (_write_back skips the move when every victim is clean); otherwise the evictions are
// applied and the admission raises (k_bts_after_evict). A batch of hits raises nothing.
__global__ void k_bts_before_evict(const int32_t* __restrict__ evicted, const int32_t* __restrict__ rank_to_slot,
                                   const uint8_t* __restrict__ dirty, int always, Counters* c) {
  if (c->err) return;
  const int needed = c->needed;
  if (needed == 0) {
    if (c->misses > 0 && blockIdx.x == 0 && threadIdx.x == 0) c->err = FC_ERR_BUFFER_TOO_SMALL;
    return;
  }
  for (int v = blockIdx.x * kNT + threadIdx.x; v < needed; v += gridDim.x * kNT)
    if (always || dirty[rank_to_slot[evicted[v]]]) c->err = FC_ERR_BUFFER_TOO_SMALL;
}

__global__ void k_bts_after_evict(Counters* c) {
  if (c->err == 0 && c->misses > 0) c->err = FC_ERR_BUFFER_TOO_SMALL;
}

// ------------------------------------------------------------------ victims (:298-303)
struct EvictFin {
  __device__ void operator()(int total, Counters* c) const {
    c->candidates = total;
    const int need = c->needed;
    if (need > total) {
      c->err = FC_ERR_INSUFFICIENT_EVICTABLE;
      return;
    }
    c->win_evict[0] = total - need;  // the `need` largest candidate ranks
    c->win_evict[1] = total;
  }
};

struct EvictEmit {
  static constexpr bool kVisitAll = false, kClear = false, kCount = false;
  int32_t* evicted;
  int total;
  __device__ void init(const Counters* c) { total = c->candidates; }
  __device__ int* counter(Counters*) const { return nullptr; }
  __device__ __forceinline__ int operator()(int64_t r, int a) const {
    evicted[total - 1 - a] = (int32_t)r;  // descending, like np.sort(top)[::-1] (:75)
    return 0;
  }
};

__global__ void k_victim_slots(const int32_t* __restrict__ evicted, const int32_t* __restrict__ rank_to_slot,
                               int32_t* vslots, const Counters* c) {
  if (c->err) return;
  for (int v = blockIdx.x * kNT + threadIdx.x; v < c->needed; v += gridDim.x * kNT) vslots[v] = rank_to_slot[evicted[v]];
}

// ------------------------------------------------------------------ admission (:310-323)
struct AdmitFin {
  __device__ void operator()(int total, Counters* c) const {
    if (total != c->misses) c->err = FC_ERR_CUDA;  // internal inconsistency guard
  }
};

struct RankEmit {
  static constexpr bool kVisitAll = false, kClear = false, kCount = false;
  int32_t* out;
  __device__ void init(const Counters*) {}
  __device__ int* counter(Counters*) const { return nullptr; }
  __device__ __forceinline__ int operator()(int64_t r, int a) const {
    out[a] = (int32_t)r;
    return 0;
  }
};

struct FreeFin {
  __device__ void operator()(int total, Counters* c) const {
    if (total < c->misses) c->err = FC_ERR_INSUFFICIENT_FREE_SLOTS;
  }
};

// Reset the per-call counters; the persistent free_count is carried over from the
// counters of the last call (`src`), which may be another counters block (the
// prefetch pipeline double-buffers its counters).
__global__ void k_begin(Counters* c, const Counters* src, int32_t* zero = nullptr, int nzero = 0) {
  for (int i = threadIdx.x; i < nzero; i += blockDim.x) zero[i] = 0;  // the sort histograms of this batch
  if (threadIdx.x) return;
  if (src != c) c->free_count = src->free_count;
  c->err = 0;
  c->emitted = 0;
  c->lo = LLONG_MAX;
  c->hi = LLONG_MIN;
  c->unique = 0;
  c->misses = 0;
  c->needed = 0;
  c->wb_rows = 0;
  c->candidates = 0;
  c->win_evict[0] = c->win_evict[1] = 0;
  c->win_admit[0] = c->win_admit[1] = 0;
  c->flush_rows = 0;
  c->bad_slot = -1;
}

// unique_slots after admission + clear every per-batch bitmap / aux entry
__global__ void __launch_bounds__(kNT) k_finish(const int32_t* __restrict__ uids, const int32_t* __restrict__ uranks,
                                                int32_t* __restrict__ uslots, int32_t* aux,
                                                const int32_t* __restrict__ rank_to_slot, uint32_t* prot,
                                                uint32_t* miss, const Counters* c) {
  if (!c->emitted) return;
  const int u = c->unique;
  const bool ok = c->err == 0;
  for (int p = blockIdx.x * kNT + threadIdx.x; p < u; p += gridDim.x * kNT) {
    aux[uids[p]] = 0;
    const int r = uranks[p];
    prot[r >> 5] = 0u;
    miss[r >> 5] = 0u;
    if (ok) uslots[p] = rank_to_slot[r];  // :325
  }
}

// device addresses of the order-index windows inside the (device) counters
static const int32_t* win_evict(Counters* c) {
  return reinterpret_cast<const int32_t*>(reinterpret_cast<char*>(c) + offsetof(Counters, win_evict));
}
static const int32_t* win_admit(Counters* c) {
  return reinterpret_cast<const int32_t*>(reinterpret_cast<char*>(c) + offsetof(Counters, win_admit));
}

int launch_reset_counters(fc_cache* h, cudaStream_t st) {
  k_begin<<<1, 1, 0, st>>>(h->ctr, h->live);
  h->live = h->ctr;
  return FC_OK;
}

int launch_prepare(fc_cache* h, const void* ids, int ids_bytes, int64_t n, int32_t* uids, int32_t* ucnt,
                   int32_t* uranks, int32_t* uslots, int32_t* inverse, cudaStream_t st) {
  Counters* c = h->ctr;
  if (h->profile) cudaEventRecord(h->pev[0], st);
  k_begin<<<1, 1, 0, st>>>(c, h->live);
  h->live = c;
  const int gn = grid_for(n, kNT, kSMs * 8);
  const int gm = grid_for(n, kMarkTile, kSMs * 6);
  if (ids_bytes == 8) k_mark_ids<long long><<<gm, kNT, 0, st>>>((const long long*)ids, n, h->num_ids, h->id_bits, h->aux, c);
  else k_mark_ids<int><<<gm, kNT, 0, st>>>((const int*)ids, n, h->num_ids, h->id_bits, h->aux, c);

  compact(ArrWords{h->id_bits}, IdFin{h->capacity}, IdEmit{h->aux, uids, 0}, h->nw_ids, h->block_cnt, nullptr, c,
          G_ALWAYS, st);
  const int gu = grid_for(std::min<int64_t>(n, h->capacity), kNT, kSMs * 8);
  k_unique_info<<<grid_for(std::min<int64_t>(n, h->capacity), kNT * kUiIlp, kSMs * 8), kNT, 0, st>>>(
      uids, h->aux, h->rank_of, h->rank_to_slot, h->prot_bits, h->miss_bits, ucnt,
                                    uranks, uslots, c, nullptr);

  if (ids_bytes == 8) k_inverse<long long><<<gn, kNT, 0, st>>>((const long long*)ids, n, h->aux, inverse, c);
  else k_inverse<int><<<gn, kNT, 0, st>>>((const int*)ids, n, h->aux, inverse, c);

  k_plan<<<1, 1, 0, st>>>(c, h->capacity, h->evict_mode);

  compact(CandWords{h->res_bits, h->prot_bits}, EvictFin{}, EvictEmit{h->evicted_ranks, 0}, h->nw_ids, h->block_cnt,
          win_evict(c), c, G_EVICT, st);
  const bool row_fits = (int64_t)h->dim * 4 <= h->buffer_bytes;
  if (!row_fits)
    k_bts_before_evict<<<grid_for(h->capacity, kNT, kSMs * 4), kNT, 0, st>>>(
        h->evicted_ranks, h->rank_to_slot, h->dirty, h->write_back == FC_WB_ALWAYS, c);
  if (h->engine == 1) FC_TRY_I(engine_reserve(h, n, st));  // grows the write-back stages if needed
  int rc = h->engine == 1 ? engine_evict(h, st) : launch_evict_rows(h, st);
  if (rc) return rc;
  if (!row_fits) k_bts_after_evict<<<1, 1, 0, st>>>(c);

  compact(ArrWords{h->miss_bits}, AdmitFin{}, RankEmit{h->admitted_ranks}, h->nw_ids, h->block_cnt,
          win_admit(c), c, G_ADMIT, st);
  compact(ArrWords{h->free_bits}, FreeFin{}, RankEmit{h->target_slots}, h->nw_slots, h->block_cnt2,
          win_admit(c), c, G_ADMIT, st);
  if (h->profile) cudaEventRecord(h->pev[1], st);
  rc = h->engine == 1 ? engine_admit(h, st) : launch_transfer_rows(h, st);
  if (rc) return rc;
  if (h->profile) cudaEventRecord(h->pev[2], st);

  k_finish<<<gu, kNT, 0, st>>>(uids, uranks, uslots, h->aux, h->rank_to_slot, h->prot_bits, h->miss_bits, c);
  if (h->profile) cudaEventRecord(h->pev[3], st);
  FC_CUDA(cudaGetLastError());
  return FC_OK;
}

// ------------------------------------------------------------------ select_evictions (:205-216)
__global__ void k_set_prot(const int64_t* __restrict__ ranks, int64_t n, int64_t num_ids, uint32_t* prot,
                           bool set) {
  for (int64_t i = (int64_t)blockIdx.x * kNT + threadIdx.x; i < n; i += (int64_t)gridDim.x * kNT) {
    const long long r = ranks[i];
    if (r < 0 || r >= num_ids) continue;  // a rank that is not resident cannot matter
    if (set) atomicOr(&prot[r >> 5], 1u << (r & 31));
    else prot[r >> 5] = 0u;
  }
}

__global__ void k_set_needed(Counters* c, int needed) { c->needed = needed; }

int launch_select_evictions(fc_cache* h, int64_t needed, const int64_t* prot, int64_t nprot, cudaStream_t st) {
  Counters* c = h->ctr;
  k_begin<<<1, 1, 0, st>>>(c, h->live);
  h->live = c;
  const int g = grid_for(nprot, kNT, kSMs * 4);
  if (nprot) k_set_prot<<<g, kNT, 0, st>>>(prot, nprot, h->num_ids, h->prot_bits, true);
  k_set_needed<<<1, 1, 0, st>>>(c, (int)needed);
  compact(CandWords{h->res_bits, h->prot_bits}, EvictFin{}, EvictEmit{h->evicted_ranks, 0}, h->nw_ids, h->block_cnt,
          win_evict(c), c, G_EVICT, st);
  k_victim_slots<<<grid_for(needed, kNT, kSMs * 4), kNT, 0, st>>>(h->evicted_ranks, h->rank_to_slot, h->victim_slots, c);
  if (nprot) k_set_prot<<<g, kNT, 0, st>>>(prot, nprot, h->num_ids, h->prot_bits, false);
  FC_CUDA(cudaGetLastError());
  return FC_OK;
}

// ------------------------------------------------------------------ warmup (:351-390)
__global__ void k_warm_state(int32_t k, int32_t* slot_to_rank, int32_t* rank_to_slot, uint8_t* dirty,
                             uint32_t* res, uint32_t* freeb, Counters* c) {
  for (int s = blockIdx.x * kNT + threadIdx.x; s < k; s += gridDim.x * kNT) {
    slot_to_rank[s] = s;
    rank_to_slot[s] = s;
    dirty[s] = 0;
    atomicOr(&res[s >> 5], 1u << (s & 31));
    atomicAnd(&freeb[s >> 5], ~(1u << (s & 31)));
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) c->free_count -= k;
}

int launch_warmup_state(fc_cache* h, int64_t k, cudaStream_t st) {
  FC_TRY_I(launch_reset_counters(h, st));
  k_warm_state<<<grid_for(k, kNT, kSMs * 4), kNT, 0, st>>>((int32_t)k, h->slot_to_rank, h->rank_to_slot, h->dirty,
                                                           h->res_bits, h->free_bits, h->ctr);
  FC_CUDA(cudaGetLastError());
  return FC_OK;
}

// ------------------------------------------------------------------ mark_dirty (:393-400)
__global__ void k_check_slots(const int64_t* __restrict__ s, int64_t n, int cap, Counters* c) {
  for (int64_t i = (int64_t)blockIdx.x * kNT + threadIdx.x; i < n; i += (int64_t)gridDim.x * kNT)
    if (s[i] < 0 || s[i] >= cap) c->err = FC_ERR_SLOT_OUT_OF_RANGE;
}
__global__ void k_set_dirty(const int64_t* __restrict__ s, int64_t n, uint8_t* dirty, const Counters* c) {
  if (c->err) return;
  for (int64_t i = (int64_t)blockIdx.x * kNT + threadIdx.x; i < n; i += (int64_t)gridDim.x * kNT) dirty[s[i]] = 1;
}

int launch_mark_dirty(fc_cache* h, const int64_t* slots, int64_t n, cudaStream_t st) {
  FC_TRY_I(launch_reset_counters(h, st));
  const int g = grid_for(n, kNT, kSMs * 4);
  k_check_slots<<<g, kNT, 0, st>>>(slots, n, h->capacity, h->ctr);
  k_set_dirty<<<g, kNT, 0, st>>>(slots, n, h->dirty, h->ctr);
  FC_CUDA(cudaGetLastError());
  return FC_OK;
}

// ------------------------------------------------------------------ prefetch pipeline: index phase
// Everything Alg. 1 decides and every state-table change it makes, without
// touching a row or a dirty bit: victims leave the slot tables, admitted ranks
// take their target slots, and unique_slots are final. The row side runs later:
// the admitted rows are staged host -> HBM on the transfer stream
// (k_admit_stage, fc_engine.cu) and the commit phase writes victims back and
// moves the staged rows into their slots (k_evict_commit / k_admit_commit). So
// this phase may run while the previous batch's forward/backward still reads
// and updates rows: those kernels address rows through their own unique_slots.

// The pipeline's index phase runs beside the previous batch's miss staging, where every
// kernel boundary costs 60-100 us and the phase is on the critical path
// (the next staging waits for it). So it fuses what round 1 ran as separate kernels:
// the eviction count into k_inverse, the victims' and the admissions' slot-table updates
// into their compactions' emit passes, two independent count passes into one launch each,
// and the counters' publication into k_finish -- 11 launches instead of 17, same results.

// victims -> slots as they are emitted (k_evict_state's work); free_count by the finisher
struct EvictFinState {
  __device__ void operator()(int total, Counters* c) const {
    c->candidates = total;
    const int need = c->needed;
    if (need > total) {
      c->err = FC_ERR_INSUFFICIENT_EVICTABLE;
      return;
    }
    c->win_evict[0] = total - need;
    c->win_evict[1] = total;
    c->free_count += need;  // applied once, by block 0 on the shared counters (:305-308)
  }
};

struct EvictEmitState {
  static constexpr bool kVisitAll = false, kClear = false, kCount = false;
  int32_t* evicted;
  int32_t* vslots;
  int32_t* slot_to_rank;
  int32_t* rank_to_slot;
  uint32_t* res;
  uint32_t* freeb;
  int total;
  __device__ void init(const Counters* c) { total = c->candidates; }
  __device__ int* counter(Counters*) const { return nullptr; }
  __device__ __forceinline__ int operator()(int64_t r, int a) const {
    const int v = total - 1 - a;  // descending, like np.sort(top)[::-1] (:75)
    const int s = rank_to_slot[r];
    evicted[v] = (int32_t)r;
    vslots[v] = s;
    slot_to_rank[s] = -1;
    rank_to_slot[r] = -1;
    // this thread read r's residency word already (each word is read by one thread)
    atomicAnd(&res[r >> 5], ~(1u << (r & 31)));
    atomicOr(&freeb[s >> 5], 1u << (s & 31));
    return 0;
  }
};

// admitted ranks take the first free slots as the slots are emitted (k_admit_state's work)
struct FreeFinState {
  __device__ void operator()(int total, Counters* c) const {
    if (total < c->misses) {
      c->err = FC_ERR_INSUFFICIENT_FREE_SLOTS;
      return;
    }
    c->free_count -= c->misses;  // applied once, by block 0 on the shared counters
  }
};

struct FreeEmitState {
  static constexpr bool kVisitAll = false, kClear = false, kCount = false;
  int32_t* target;
  const int32_t* admitted;
  int32_t* slot_to_rank;
  int32_t* rank_to_slot;
  uint32_t* res;
  uint32_t* freeb;
  __device__ void init(const Counters*) {}
  __device__ int* counter(Counters*) const { return nullptr; }
  __device__ __forceinline__ int operator()(int64_t s, int a) const {
    const int r = admitted[a];
    target[a] = (int32_t)s;
    slot_to_rank[s] = r;
    rank_to_slot[r] = (int32_t)s;
    atomicOr(&res[r >> 5], 1u << (r & 31));
    atomicAnd(&freeb[s >> 5], ~(1u << (s & 31)));  // this thread read s's word already
    return 0;
  }
};

// k_inverse + the eviction count (k_plan, :293-296) by one thread of block 0
template <typename IdT>
__global__ void __launch_bounds__(kNT) k_inverse_plan(const IdT* __restrict__ ids, int64_t n,
                                                      const int32_t* __restrict__ aux, int32_t* __restrict__ inv,
                                                      Counters* c, int cap, int evict_mode) {
  if (blockIdx.x == 0 && threadIdx.x == 0 && c->err == 0) {  // misses are final (k_unique_info)
    const int m = c->misses, u = c->unique, fr = c->free_count;
    const int needed = evict_mode == FC_EVICT_OCCUPANCY_AWARE ? max(0, m - fr) : max(0, u - cap);
    c->needed = needed;
    if (fr + needed < m) c->err = FC_ERR_INSUFFICIENT_FREE_SLOTS;  // paper_literal (:313-317)
    c->win_admit[0] = 0;
    c->win_admit[1] = m;
  }
  if (!c->emitted) return;
  for (int64_t i = (int64_t)blockIdx.x * kNT + threadIdx.x; i < n; i += (int64_t)gridDim.x * kNT)
    inv[i] = aux[(int64_t)ids[i]];
}

// k_finish + the counters' publication to the pinned mapped host copy (k_publish)
__global__ void __launch_bounds__(kNT) k_finish_publish(const int32_t* __restrict__ uids,
                                                        const int32_t* __restrict__ uranks,
                                                        int32_t* __restrict__ uslots, int32_t* aux,
                                                        const int32_t* __restrict__ rank_to_slot, uint32_t* prot,
                                                        uint32_t* miss, const Counters* c, Counters* host) {
  if (blockIdx.x == 0 && threadIdx.x < 32) {  // the counters do not change any more in this phase
    const int* src = reinterpret_cast<const int*>(c);
    int* dst = reinterpret_cast<int*>(host);
    constexpr int kWords = (int)(sizeof(Counters) / sizeof(int));
    for (int i = threadIdx.x; i < kWords; i += 32) dst[i] = src[i];
    __threadfence_system();
  }
  if (!c->emitted) return;
  const int u = c->unique;
  const bool ok = c->err == 0;
  for (int p = blockIdx.x * kNT + threadIdx.x; p < u; p += gridDim.x * kNT) {
    aux[uids[p]] = 0;
    const int r = uranks[p];
    prot[r >> 5] = 0u;
    miss[r >> 5] = 0u;
    if (ok) uslots[p] = rank_to_slot[r];  // :325
  }
}

static void compaction_shape(int64_t nwords, int& nb, int64_t& chunk) {
  nb = grid_for(nwords, 128, kMaxScanBlocks);
  chunk = (nwords + nb - 1) / nb;
}

int launch_index_phase(fc_cache* h, const void* ids, int ids_bytes, int64_t n, int32_t* uids, int32_t* ucnt,
                       int32_t* uranks, int32_t* uslots, int32_t* inverse, const IndexBufs& b, Counters* publish,
                       int32_t* sort_hist, cudaStream_t st) {
  Counters* c = b.ctr;
  k_begin<<<1, kNT, 0, st>>>(c, h->live, sort_hist, sort_hist ? kSortHistInts : 0);
  h->live = c;
  const int gn = grid_for(n, kNT, kSMs * 8);
  const int gm = grid_for(n, kMarkTile, kSMs * 6);
  if (ids_bytes == 8) k_mark_ids<long long><<<gm, kNT, 0, st>>>((const long long*)ids, n, h->num_ids, h->id_bits, h->aux, c);
  else k_mark_ids<int><<<gm, kNT, 0, st>>>((const int*)ids, n, h->num_ids, h->id_bits, h->aux, c);
  trace_mark(h, 20, st);
  compact(ArrWords{h->id_bits}, IdFin{h->capacity}, IdEmit{h->aux, uids, 0}, h->nw_ids, h->block_cnt, nullptr, c,
          G_ALWAYS, st);
  trace_mark(h, 21, st);
  const int gu = grid_for(std::min<int64_t>(n, h->capacity), kNT, kSMs * 8);
  k_unique_info<<<grid_for(std::min<int64_t>(n, h->capacity), kNT * kUiIlp, kSMs * 8), kNT, 0, st>>>(
      uids, h->aux, h->rank_of, h->rank_to_slot, h->prot_bits, h->miss_bits, ucnt, uranks, uslots, c, sort_hist);
  // (the pipeline requires a row to fit the buffer: no BufferTooSmall ordering here)
  if (ids_bytes == 8)
    k_inverse_plan<long long><<<gn, kNT, 0, st>>>((const long long*)ids, n, h->aux, inverse, c, h->capacity,
                                                 h->evict_mode);
  else
    k_inverse_plan<int><<<gn, kNT, 0, st>>>((const int*)ids, n, h->aux, inverse, c, h->capacity, h->evict_mode);
  trace_mark(h, 22, st);
  // victims' and misses' counts in one launch; the misses' emission shares a launch with the
  // free slots' count (which needs the freed victim slots)
  int nb_id, nb_sl;
  int64_t ch_id, ch_sl;
  compaction_shape(h->nw_ids, nb_id, ch_id);
  compaction_shape(h->nw_slots, nb_sl, ch_sl);
  const CandWords cand{h->res_bits, h->prot_bits};
  k_bits_count2<CandWords, ArrWords><<<2 * nb_id, kNT, 0, st>>>(cand, h->nw_ids, ch_id, h->block_cnt, nb_id, G_EVICT,
                                                              ArrWords{h->miss_bits}, h->nw_ids, ch_id, h->block_cnt2,
                                                              G_ADMIT, c);
  k_bits_emit<CandWords, EvictEmitState, EvictFinState><<<nb_id, kNT, 0, st>>>(
      cand, EvictEmitState{b.evicted, b.vslots, h->slot_to_rank, h->rank_to_slot, h->res_bits, h->free_bits, 0},
      EvictFinState{}, h->nw_ids, ch_id, h->block_cnt, nb_id, win_evict(c), c, G_EVICT);
  trace_mark(h, 23, st);
  k_bits_emit_count<ArrWords, RankEmit, AdmitFin, ArrWords><<<nb_id + nb_sl, kNT, 0, st>>>(
      ArrWords{h->miss_bits}, RankEmit{b.admitted}, AdmitFin{}, h->nw_ids, ch_id, h->block_cnt2, nb_id, win_admit(c),
      G_ADMIT, ArrWords{h->free_bits}, h->nw_slots, ch_sl, h->block_cnt, G_ADMIT, c);
  k_bits_emit<ArrWords, FreeEmitState, FreeFinState><<<nb_sl, kNT, 0, st>>>(
      ArrWords{h->free_bits}, FreeEmitState{b.target, b.admitted, h->slot_to_rank, h->rank_to_slot, h->res_bits,
                                            h->free_bits},
      FreeFinState{}, h->nw_slots, ch_sl, h->block_cnt, nb_sl, win_admit(c), c, G_ADMIT);
  trace_mark(h, 24, st);
  k_finish_publish<<<gu, kNT, 0, st>>>(uids, uranks, uslots, h->aux, h->rank_to_slot, h->prot_bits, h->miss_bits, c,
                                       publish);
  FC_CUDA(cudaGetLastError());
  return FC_OK;
}

// ------------------------------------------------------------------ row-sharded exchange planner
// A requester's batch, routed to row owners (owner = id % world, the owner's local
// row = id / world): unique ids grouped by owner and ascending within each owner —
// one ordered compaction of a bitmap over the key space key = owner * S + id / world —
// plus every occurrence's position in that list (its inverse) and per-owner counts
// for the all-to-all splits. Same machinery as prepare's dedup (k_mark_ids / IdEmit).
// Owner and owner-local row of a global id, as the routing key owner * S + local:
//   RowMap   — row-wise: owner = id % W, local = id / W;
//   TableMap — table-wise: whole tables (contiguous id ranges [starts[t], starts[t+1]))
//              belong to owner[t] and sit at lbase[t] in that owner's local id space.
struct RowMap {
  uint32_t w, s;
  __device__ __forceinline__ int key(long long id) const {
    const uint32_t u = (uint32_t)id;
    return (int)((u % w) * s + u / w);
  }
};

struct TableMap {
  const long long* starts;  // [T + 1]
  const int* owner;         // [T]
  const long long* lbase;   // [T]
  int T;
  long long S;
  __device__ __forceinline__ int key(long long id) const {
    int lo = 0, hi = T - 1;  // the last table whose start is <= id
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (starts[mid] <= id) lo = mid;
      else hi = mid - 1;
    }
    return (int)(owner[lo] * S + lbase[lo] + (id - starts[lo]));
  }
};

template <typename IdT, class Map>
__global__ void __launch_bounds__(kNT) k_route_mark(const IdT* __restrict__ ids, int64_t n, int64_t num_ids, Map map,
                                                    uint32_t* bits, Counters* c) {
  const int lane = threadIdx.x & 31;
  for (int64_t base = (int64_t)blockIdx.x * kNT; base < n; base += (int64_t)gridDim.x * kNT) {
    const int64_t i = base + threadIdx.x;
    const bool valid = i < n;
    const long long id = valid ? (long long)ids[i] : 0;
    const bool inr = valid && id >= 0 && id < num_ids;
    if (valid && !inr) {
      if (id < 0) atomicMin(&c->lo, id);
      else atomicMax(&c->hi, id);
    }
    const int key = inr ? map.key(id) : -1;  // key space < 2^31 (checked at create)
    // one leader per distinct key of the warp; a read before the atomic skips the
    // bits already set (Zipf batches repeat head ids a lot)
    const unsigned peers = __match_any_sync(FC_FULL, key);
    if (inr && lane == __ffs(peers) - 1) {
      const uint32_t m = 1u << (key & 31);
      uint32_t* wp = &bits[key >> 5];
      if (!(*wp & m)) atomicOr(wp, m);
    }
  }
}

struct RouteFin {
  __device__ void operator()(int total, Counters* c) const {
    c->unique = total;
    if (c->lo != LLONG_MAX || c->hi != LLONG_MIN) c->err = FC_ERR_ID_OUT_OF_RANGE;
    c->emitted = (c->err == 0);
  }
};

struct RouteEmit {
  static constexpr bool kVisitAll = true, kClear = true, kCount = false;
  int32_t* ukeys;
  int32_t* ulocal;
  int32_t* aux;
  int64_t S;
  int ok;
  __device__ void init(const Counters* c) { ok = c->emitted; }
  __device__ int* counter(Counters*) const { return nullptr; }
  __device__ __forceinline__ int operator()(int64_t key, int p) const {
    if (ok) {
      ukeys[p] = (int32_t)key;
      ulocal[p] = (int32_t)(key % S);
      aux[key] = p;
    }
    return 0;
  }
};

template <typename IdT, class Map>
__global__ void __launch_bounds__(kNT) k_route_inverse(const IdT* __restrict__ ids, int64_t n, Map map,
                                                       const int32_t* __restrict__ aux, int32_t* __restrict__ inv,
                                                       const Counters* c) {
  if (!c->emitted) return;
  for (int64_t i = (int64_t)blockIdx.x * kNT + threadIdx.x; i < n; i += (int64_t)gridDim.x * kNT)
    inv[i] = aux[map.key((long long)ids[i])];
}

// clears the key->position map for the next call; block 0 also writes the per-owner
// counts: owner o's ids are the keys in [o*S, (o+1)*S) of the sorted unique list
__global__ void __launch_bounds__(kNT) k_route_finish(const int32_t* __restrict__ ukeys, int32_t* aux, int64_t S, int W,
                                                      const Counters* c, long long* owner_cnt) {
  const int u = c->emitted ? c->unique : 0;
  if (blockIdx.x == 0) {
    __shared__ int start[65];
    const int o = threadIdx.x;
    if (o <= W) {
      const long long target = (long long)o * S;
      int lo = 0, hi = u;  // first position with key >= o*S
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if ((long long)ukeys[mid] < target) lo = mid + 1;
        else hi = mid;
      }
      start[o] = (o == W) ? u : lo;
    }
    __syncthreads();
    if (o < W) owner_cnt[o] = start[o + 1] - start[o];
  }
  for (int p = blockIdx.x * kNT + threadIdx.x; p < u; p += gridDim.x * kNT) aux[ukeys[p]] = 0;
}

}  // namespace fc

struct fc_router {
  int64_t num_ids;
  int32_t world;
  int64_t S;       // keys per owner (multiple of 32)
  int64_t nw;      // bitmap words
  int device;
  uint32_t* bits;
  int32_t* aux;
  int32_t* ukeys;
  int64_t ukeys_cap;
  int32_t* block_cnt;
  fc::Counters* ctr;
  fc::Counters* ctr_host;
  long long* owner_cnt;
  long long* owner_cnt_host;
  void* scratch;
  size_t scratch_bytes;
  int32_t ntables;          // > 0: table-wise placement (fc_router_create_tables)
  long long* t_starts;      // device [T + 1]
  int* t_owner;             // device [T]
  long long* t_lbase;       // device [T]
};

namespace fc {

static void router_release(fc_router* r) {
  void* dev[] = {r->bits, r->aux, r->ukeys, r->block_cnt, r->ctr, r->owner_cnt, r->scratch, r->t_starts, r->t_owner,
                 r->t_lbase};
  for (void* p : dev)
    if (p) cudaFree(p);
  if (r->ctr_host) cudaFreeHost(r->ctr_host);
  if (r->owner_cnt_host) cudaFreeHost(r->owner_cnt_host);
  delete r;
}

}  // namespace fc

using namespace fc;

// keys per owner S: row-wise ceil(num_ids / world); table-wise the largest owner's rows
static int router_create(int64_t num_ids, int32_t world, int64_t S_rows, int32_t device, fc_router** out) {
  *out = nullptr;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(device);
  fc_router* r = new fc_router();
  std::memset(r, 0, sizeof(*r));
  r->num_ids = num_ids;
  r->world = world;
  r->S = (S_rows + 31) / 32 * 32;
  if (r->S * world > INT32_MAX - 64) {
    delete r;
    cudaSetDevice(prev);
    set_error("routing key space exceeds int32");
    return FC_ERR_BAD_ARG;
  }
  r->nw = (r->S * world / 32 + 3) / 4 * 4;
  r->device = device;
  cudaError_t e = cudaMalloc(&r->bits, r->nw * 4);
  if (e == cudaSuccess) e = cudaMemset(r->bits, 0, r->nw * 4);
  if (e == cudaSuccess) e = cudaMalloc(&r->aux, (size_t)r->S * world * 4);
  if (e == cudaSuccess) e = cudaMemset(r->aux, 0, (size_t)r->S * world * 4);
  if (e == cudaSuccess) e = cudaMalloc(&r->block_cnt, (kMaxScanBlocks + 1) * 4);
  if (e == cudaSuccess) e = cudaMalloc(&r->ctr, sizeof(Counters));
  if (e == cudaSuccess) e = cudaHostAlloc(&r->ctr_host, sizeof(Counters), cudaHostAllocDefault);
  if (e == cudaSuccess) e = cudaMalloc(&r->owner_cnt, 64 * sizeof(long long));
  if (e == cudaSuccess) e = cudaHostAlloc(&r->owner_cnt_host, 64 * sizeof(long long), cudaHostAllocDefault);
  cudaSetDevice(prev);
  if (e != cudaSuccess) {
    router_release(r);
    return cuda_fail(e, "fc_router_create");
  }
  *out = r;
  return FC_OK;
}

extern "C" int fc_router_create(int64_t num_ids, int32_t world, int32_t device, fc_router** out) {
  if (!out || num_ids < 1 || world < 1 || world > 64) return FC_ERR_BAD_ARG;
  return router_create(num_ids, world, (num_ids + world - 1) / world, device, out);
}

extern "C" int fc_router_create_tables(int64_t num_ids, int32_t world, int32_t num_tables, const int64_t* table_starts,
                                       const int32_t* table_owner, int32_t device, fc_router** out) {
  if (!out || num_ids < 1 || world < 1 || world > 64 || num_tables < 1 || !table_starts || !table_owner)
    return FC_ERR_BAD_ARG;
  *out = nullptr;
  if (table_starts[0] != 0 || table_starts[num_tables] != num_ids) {
    set_error("table starts must run from 0 to num_ids");
    return FC_ERR_BAD_ARG;
  }
  std::vector<long long> lbase(num_tables), load(world, 0);
  for (int t = 0; t < num_tables; ++t) {
    if (table_starts[t + 1] <= table_starts[t] || table_owner[t] < 0 || table_owner[t] >= world) {
      set_error("table %d: empty, unordered or owned by a rank outside [0, %d)", t, world);
      return FC_ERR_BAD_ARG;
    }
    lbase[t] = load[table_owner[t]];  // an owner's tables in table order
    load[table_owner[t]] += table_starts[t + 1] - table_starts[t];
  }
  const long long S = *std::max_element(load.begin(), load.end());
  int rc = router_create(num_ids, world, S, device, out);
  if (rc) return rc;
  fc_router* r = *out;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(device);
  r->ntables = num_tables;
  cudaError_t e = cudaMalloc(&r->t_starts, (num_tables + 1) * sizeof(long long));
  if (e == cudaSuccess) e = cudaMalloc(&r->t_owner, num_tables * sizeof(int));
  if (e == cudaSuccess) e = cudaMalloc(&r->t_lbase, num_tables * sizeof(long long));
  if (e == cudaSuccess)
    e = cudaMemcpy(r->t_starts, table_starts, (num_tables + 1) * sizeof(long long), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(r->t_owner, table_owner, num_tables * sizeof(int), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(r->t_lbase, lbase.data(), num_tables * sizeof(long long), cudaMemcpyHostToDevice);
  cudaSetDevice(prev);
  if (e != cudaSuccess) {
    router_release(r);
    *out = nullptr;
    return cuda_fail(e, "fc_router_create_tables");
  }
  return FC_OK;
}

extern "C" int fc_router_destroy(fc_router* r) {
  if (!r) return FC_OK;
  cudaDeviceSynchronize();
  router_release(r);
  return FC_OK;
}

extern "C" int fc_route(fc_router* r, const void* ids, int32_t ids_bytes, int64_t n, int32_t* local_ids,
                        int32_t* inverse, int64_t* owner_counts, int64_t* unique, void* stream) {
  if (!r || !owner_counts || !unique || (ids_bytes != 4 && ids_bytes != 8) || n < 0 || n > INT32_MAX)
    return FC_ERR_BAD_ARG;
  *unique = 0;
  for (int o = 0; o < r->world; ++o) owner_counts[o] = 0;
  if (n == 0) return FC_OK;
  int prev = 0;
  cudaGetDevice(&prev);
  if (prev != r->device) cudaSetDevice(r->device);
  cudaStream_t st = as_stream(stream);
  int rc = FC_OK;
  if (r->ukeys_cap < n) {
    if (r->ukeys) cudaFree(r->ukeys);
    r->ukeys = nullptr;
    r->ukeys_cap = 0;
    if (cudaMalloc(&r->ukeys, (size_t)n * 4) != cudaSuccess) {
      if (prev != r->device) cudaSetDevice(prev);
      return cuda_fail(cudaGetLastError(), "fc_route");
    }
    r->ukeys_cap = n;
  }
  Counters* c = r->ctr;
  k_begin<<<1, 1, 0, st>>>(c, c);
  const int g = grid_for(n, kNT, kSMs * 8);
  auto run = [&](auto map) {
    if (ids_bytes == 8)
      k_route_mark<long long><<<g, kNT, 0, st>>>((const long long*)ids, n, r->num_ids, map, r->bits, c);
    else k_route_mark<int><<<g, kNT, 0, st>>>((const int*)ids, n, r->num_ids, map, r->bits, c);
    compact(ArrWords{r->bits}, RouteFin{}, RouteEmit{r->ukeys, local_ids, r->aux, r->S, 0}, r->nw, r->block_cnt,
            nullptr, c, G_ALWAYS, st);
    if (ids_bytes == 8)
      k_route_inverse<long long><<<g, kNT, 0, st>>>((const long long*)ids, n, map, r->aux, inverse, c);
    else k_route_inverse<int><<<g, kNT, 0, st>>>((const int*)ids, n, map, r->aux, inverse, c);
  };
  if (r->ntables > 0) run(TableMap{r->t_starts, r->t_owner, r->t_lbase, r->ntables, r->S});
  else run(RowMap{(uint32_t)r->world, (uint32_t)r->S});
  k_route_finish<<<grid_for(n, kNT, kSMs * 4), kNT, 0, st>>>(r->ukeys, r->aux, r->S, r->world, c, r->owner_cnt);
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaMemcpyAsync(r->ctr_host, c, sizeof(Counters), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(r->owner_cnt_host, r->owner_cnt, r->world * sizeof(long long), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) rc = cuda_fail(e, "fc_route");
  if (rc == FC_OK && r->ctr_host->err) {
    const long long b = r->ctr_host->lo != LLONG_MAX ? r->ctr_host->lo : r->ctr_host->hi;
    set_error("id out of range: %lld not in [0, %lld)", b, (long long)r->num_ids);
    rc = FC_ERR_ID_OUT_OF_RANGE;
  }
  if (rc == FC_OK) {
    *unique = r->ctr_host->unique;
    for (int o = 0; o < r->world; ++o) owner_counts[o] = r->owner_cnt_host[o];
  }
  if (prev != r->device) cudaSetDevice(prev);
  return rc;
}

extern "C" int fc_route_grads(fc_router* r, const int32_t* inverse, int64_t u, int64_t n, const void* offsets,
                              int32_t off_bytes, int64_t nbags, int32_t include_last, const float* psw, int32_t mode,
                              const float* grad, int32_t dim, float* grad_unique, void* stream) {
  if (!r || (mode != FC_POOL_SUM && mode != FC_POOL_MEAN) || (offsets && off_bytes != 4 && off_bytes != 8))
    return FC_ERR_BAD_ARG;
  cudaStream_t st = as_stream(stream);  // every unique id has an occurrence: all u rows are written
  return launch_unique_grads(&r->scratch, &r->scratch_bytes, inverse, u, n, offsets, off_bytes, nbags, include_last, psw,
                             mode, grad, dim, grad_unique, st);
}

extern "C" int fc_pool_rows(const float* rows, int32_t dim, const int32_t* inverse, int64_t n, const void* offsets,
                            int32_t off_bytes, int64_t nbags, int32_t include_last, const float* psw, int32_t mode,
                            float* out, void* stream) {
  if (!rows || dim < 1 || (mode != FC_POOL_SUM && mode != FC_POOL_MEAN) || (offsets && off_bytes != 4 && off_bytes != 8))
    return FC_ERR_BAD_ARG;
  return launch_pool_rows(rows, dim, nullptr, inverse, n, offsets, off_bytes, nbags, include_last, psw, mode, out,
                          as_stream(stream));
}

