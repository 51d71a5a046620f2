// Row-moving kernels: eviction staging, host<->HBM transfers, flush, pooled
// EmbeddingBag forward, updates and the fused backward + sparse optimizer.
//
// Rows are moved by "row groups": G lanes (G = pow2 >= row_width/4, <= 32) own one
// row and move it with 16-byte accesses. Groups never straddle warps, so a warp
// walks ceil(items / (groups per grid)) rounds in lock-step and can __syncwarp.
//
// The slow tier lives in pinned, device-mapped host memory (fc_host_alloc). The
// GPU reads admitted rows from it and writes evicted dirty rows into it directly
// over PCIe/C2C, both directions in the same kernel so the duplex link is used
// both ways at once (transmitter.py:144-207 moves rows through a bounded host
// buffer; here the "buffer" is the HBM staging area of the victims).
#include <algorithm>
#include <cstdlib>

#include "fc_rowutil.cuh"
#include "fc_tma.cuh"

namespace fc {

struct RowCtx {
  float* fast;
  float* fstate;
  float* slow;
  float* sstate;
  int64_t ld;   // slow row stride (floats)
  int64_t sld;  // slow state stride
  int D, S;
  int32_t* slot_to_rank;
  int32_t* rank_to_slot;
  uint8_t* dirty;
  uint32_t* res;
  uint32_t* freeb;
  int32_t* evicted;
  int32_t* vslots;
  int32_t* wb_ranks;
  float* stage;
  float* stage_state;
  int32_t* admitted;
  int32_t* target;
  int always;
  Counters* c;
};

static RowCtx row_ctx(fc_cache* h) {
  RowCtx x;
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
  x.vslots = h->victim_slots;
  x.wb_ranks = h->wb_ranks;
  x.stage = h->wb_stage;
  x.stage_state = h->wb_stage_state;
  x.admitted = h->admitted_ranks;
  x.target = h->target_slots;
  x.always = h->write_back == FC_WB_ALWAYS;
  x.c = h->ctr;
  return x;
}

static bool vec_ok(fc_cache* h) {
  auto al = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  bool v = (h->dim % 4 == 0) && (h->slow_ld % 4 == 0) && al(h->slow) && al(h->fast);
  if (h->sw) v = v && (h->sw % 4 == 0) && (h->state_ld % 4 == 0) && al(h->slow_state) && al(h->fast_state);
  return v;
}

// two independent row copies with both loads issued before both stores
template <bool VEC>
__device__ __forceinline__ void copy_two_rows(float* d1, const float* s1, bool a1, float* d2, const float* s2, bool a2,
                                              int w, int gl, int G) {
  if (VEC) {
    for (int c = gl * 4; c < w; c += G * 4) {
      float4 x, y;
      if (a1) x = *reinterpret_cast<const float4*>(s1 + c);
      if (a2) y = *reinterpret_cast<const float4*>(s2 + c);
      if (a1) *reinterpret_cast<float4*>(d1 + c) = x;
      if (a2) *reinterpret_cast<float4*>(d2 + c) = y;
    }
  } else {
    for (int c = gl; c < w; c += G) {
      float x = 0.f, y = 0.f;
      if (a1) x = s1[c];
      if (a2) y = s2[c];
      if (a1) d1[c] = x;
      if (a2) d2[c] = y;
    }
  }
}

struct GroupIdx {
  int lane, gw, gl, gpw;
  int64_t warp, nwarps;
  __device__ GroupIdx(int G) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    lane = threadIdx.x & 31;
    gpw = 32 / G;
    gw = lane / G;
    gl = lane % G;
    warp = t >> 5;
    nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  }
};

// ------------------------------------------------------------- warp-batched row moves
// A warp takes 32 items at once: lane i loads item i's indices (one coalesced
// round trip for all 32), then the warp moves the 32 rows as a flat list of
// 16-byte units, K units per lane in flight. Row r's offsets come from lane r by
// shuffle. This hides the index->row dependent latency that a row-per-warp loop
// pays once per row.
// dst[drow_r * dstride + c] = src[srow_r * sstride + c] (* scale_r) for the warp's 32
// rows (act_r false -> skipped). Row indices travel by shuffle as int32.
template <int K, bool SCALE = false>
__device__ __forceinline__ void warp_move(const float* __restrict__ sbase, int64_t sstride, int srow,
                                          float* __restrict__ dbase, int64_t dstride, int drow, bool act,
                                          float scale, Units un) {
  const int lane = threadIdx.x & 31;
  const int total = 32 * un.upr;
  for (int u0 = 0; u0 < total; u0 += 32 * K) {
    float4 v[K];
    int dr[K], cc[K];
    bool aa[K];
    float sc[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const int u = u0 + k * 32 + lane;
      const int r = min(un.row(u), 31);
      cc[k] = (u - r * un.upr) * 4;
      const int sr = __shfl_sync(FC_FULL, srow, r);
      dr[k] = __shfl_sync(FC_FULL, drow, r);
      aa[k] = __shfl_sync(FC_FULL, (int)act, r) && u < total;
      if (SCALE) sc[k] = __shfl_sync(FC_FULL, scale, r);
      if (aa[k]) v[k] = ld4(sbase + (int64_t)sr * sstride + cc[k]);
    }
#pragma unroll
    for (int k = 0; k < K; ++k)
      if (aa[k]) {
        float4 w = v[k];
        if (SCALE) {
          w.x *= sc[k]; w.y *= sc[k]; w.z *= sc[k]; w.w *= sc[k];
        }
        st4(dbase + (int64_t)dr[k] * dstride + cc[k], w);
      }
  }
}

constexpr int kUnroll = 4;

// ------------------------------------------------------------- eviction (:298-308, _write_back :219-231)
// victims -> slots, dirty filter (or all, write_back="always"), rows staged in HBM,
// slot table cleared, bitmaps updated
template <bool VEC>
__global__ void __launch_bounds__(kNT) k_evict_rows(RowCtx x, Units ud, Units us, int G) {
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
    if (VEC) {
      warp_move<kUnroll>(x.fast, x.D, s, x.stage, x.D, (int)v, wb, 1.0f, ud);
      if (x.S) warp_move<kUnroll>(x.fstate, x.S, s, x.stage_state, x.S, (int)v, wb, 1.0f, us);
    } else {
      for (int q = 0; q < 32; ++q) {  // scalar fallback: lanes stride the row's columns
        const bool aq = __shfl_sync(FC_FULL, (int)wb, q);
        const int sq = __shfl_sync(FC_FULL, s, q);
        if (aq) {
          copy_row<false>(x.stage + (base + q) * x.D, x.fast + (int64_t)sq * x.D, x.D, lane, 32);
          if (x.S) copy_row<false>(x.stage_state + (base + q) * x.S, x.fstate + (int64_t)sq * x.S, x.S, lane, 32);
        }
      }
    }
    if (act) {
      x.wb_ranks[v] = wb ? r : -1;
      x.slot_to_rank[s] = -1;
      x.rank_to_slot[r] = -1;
      x.dirty[s] = 0;
      atomicAnd(&x.res[r >> 5], ~(1u << (r & 31)));
      atomicOr(&x.freeb[s >> 5], 1u << (s & 31));
      wb_count += wb;
    }
  }
  (void)G;
  wb_count = block_sum<kNT>(wb_count, sm);
  if (threadIdx.x == 0 && wb_count) atomicAdd(&x.c->wb_rows, wb_count);
  if (blockIdx.x == 0 && threadIdx.x == 0) x.c->free_count += needed;
}

// Two row lists moved together: per 16-byte unit a lane issues both loads before
// both stores, so every warp keeps one host read and one host write in flight.
template <int K>
__device__ __forceinline__ void warp_move2(const float* __restrict__ s1, int64_t ss1, int sr1, float* __restrict__ d1,
                                           int64_t ds1, int dr1, bool a1, const float* __restrict__ s2, int64_t ss2,
                                           int sr2, float* __restrict__ d2, int64_t ds2, int dr2, bool a2, Units un) {
  const int lane = threadIdx.x & 31;
  const int total = 32 * un.upr;
  for (int u0 = 0; u0 < total; u0 += 32 * K) {
    float4 v1[K], v2[K];
    int e1[K], e2[K], cc[K];
    bool b1[K], b2[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const int u = u0 + k * 32 + lane;
      const int r = min(un.row(u), 31);
      cc[k] = (u - r * un.upr) * 4;
      const bool in = u < total;
      const int x1 = __shfl_sync(FC_FULL, sr1, r), x2 = __shfl_sync(FC_FULL, sr2, r);
      e1[k] = __shfl_sync(FC_FULL, dr1, r);
      e2[k] = __shfl_sync(FC_FULL, dr2, r);
      b1[k] = __shfl_sync(FC_FULL, (int)a1, r) && in;
      b2[k] = __shfl_sync(FC_FULL, (int)a2, r) && in;
      if (b1[k]) v1[k] = ld4(s1 + (int64_t)x1 * ss1 + cc[k]);
      if (b2[k]) v2[k] = ld4(s2 + (int64_t)x2 * ss2 + cc[k]);
    }
#pragma unroll
    for (int k = 0; k < K; ++k) {
      if (b1[k]) st4(d1 + (int64_t)e1[k] * ds1 + cc[k], v1[k]);
      if (b2[k]) st4(d2 + (int64_t)e2[k] * ds2 + cc[k], v2[k]);
    }
  }
}

// ------------------------------------------------------------- write-back + admission rows (:304,319-323)
// Item j pairs the j-th staged victim (HBM -> pinned slow tier, posted writes) with
// the j-th admitted rank (slow tier -> its target slot). Both lists are rank-sorted
// (victims descending, admissions ascending): sorted host addresses sustain ~75 GB/s
// both ways on PCIe Gen5 where random ones fall to ~47 (tools/zerocopy_bench.cu).
template <bool VEC>
__global__ void __launch_bounds__(kNT, 4) k_transfer_rows(RowCtx x, Units ud, Units us) {
  if (!gate_open(x.c, G_OK)) return;
  const int needed = x.c->needed, m = x.c->misses;
  const int items = max(needed, m);
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * kNT + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * kNT) >> 5;
  for (int64_t base = warp * 32; base < items; base += nwarps * 32) {
    const int64_t j = base + lane;
    const int r1 = j < needed ? x.wb_ranks[j] : -1;
    const bool a1 = r1 >= 0;
    const bool a2 = j < m;
    int r2 = 0, s2 = 0;
    if (a2) {
      r2 = x.admitted[j];
      s2 = x.target[j];
    }
    if (VEC) {
      warp_move2<1>(x.stage, x.D, (int)j, x.slow, x.ld, r1, a1, x.slow, x.ld, r2, x.fast, x.D, s2, a2, ud);
      if (x.S)
        warp_move2<1>(x.stage_state, x.S, (int)j, x.sstate, x.sld, r1, a1, x.sstate, x.sld, r2, x.fstate, x.S, s2, a2,
                      us);
    } else {
      for (int q = 0; q < 32; ++q) {
        const int rq1 = __shfl_sync(FC_FULL, r1, q);
        const bool aq2 = __shfl_sync(FC_FULL, (int)a2, q);
        const int rq2 = __shfl_sync(FC_FULL, r2, q), sq2 = __shfl_sync(FC_FULL, s2, q);
        if (rq1 >= 0) {
          copy_row<false>(x.slow + (int64_t)rq1 * x.ld, x.stage + (base + q) * x.D, x.D, lane, 32);
          if (x.S) copy_row<false>(x.sstate + (int64_t)rq1 * x.sld, x.stage_state + (base + q) * x.S, x.S, lane, 32);
        }
        if (aq2) {
          copy_row<false>(x.fast + (int64_t)sq2 * x.D, x.slow + (int64_t)rq2 * x.ld, x.D, lane, 32);
          if (x.S) copy_row<false>(x.fstate + (int64_t)sq2 * x.S, x.sstate + (int64_t)rq2 * x.sld, x.S, lane, 32);
        }
      }
    }
    if (a2) {
      x.slot_to_rank[s2] = r2;
      x.rank_to_slot[r2] = s2;
      x.dirty[s2] = 0;
      atomicOr(&x.res[r2 >> 5], 1u << (r2 & 31));
      atomicAnd(&x.freeb[s2 >> 5], ~(1u << (s2 & 31)));
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) x.c->free_count -= m;
}

static int rows_grid() { return kSMs * 8; }

// engine 0's write-back stage (C rows): allocated the first time engine 0 evicts, so a
// cache on the default async engine never holds it
static int ensure_wb_stage(fc_cache* h) {
  if (h->wb_stage) return FC_OK;
  FC_CUDA(cudaMalloc(&h->wb_stage, (size_t)h->capacity * h->dim * 4));
  if (h->sw) FC_CUDA(cudaMalloc(&h->wb_stage_state, (size_t)h->capacity * h->sw * 4));
  return FC_OK;
}

int launch_evict_rows(fc_cache* h, cudaStream_t st) {
  int rc = ensure_wb_stage(h);
  if (rc) return rc;
  RowCtx x = row_ctx(h);
  const bool v = vec_ok(h);
  const Units ud = units_for(h->dim), us = units_for(h->sw ? h->sw : 4);
  if (v) k_evict_rows<true><<<rows_grid(), kNT, 0, st>>>(x, ud, us, 32);
  else k_evict_rows<false><<<rows_grid(), kNT, 0, st>>>(x, ud, us, 32);
  FC_CUDA(cudaGetLastError());
  return FC_OK;
}

int launch_transfer_rows(fc_cache* h, cudaStream_t st) {
  int rc = ensure_wb_stage(h);
  if (rc) return rc;
  RowCtx x = row_ctx(h);
  const bool v = vec_ok(h);
  const Units ud = units_for(h->dim), us = units_for(h->sw ? h->sw : 4);
  if (v) k_transfer_rows<true><<<kSMs * 4, kNT, 0, st>>>(x, ud, us);
  else k_transfer_rows<false><<<kSMs * 4, kNT, 0, st>>>(x, ud, us);
  FC_CUDA(cudaGetLastError());
  return FC_OK;
}

// ------------------------------------------------------------- flush (:403-415)
template <bool VEC>
__global__ void __launch_bounds__(kNT) k_flush(RowCtx x, int cap, int G) {
  __shared__ int sm[kNT / 32 + 1];
  GroupIdx g(G);
  int cnt = 0;
  for (int64_t base = g.warp * g.gpw; base < cap; base += g.nwarps * g.gpw) {
    const int64_t s = base + g.gw;
    const bool d = s < cap && x.dirty[s];
    int r = 0;
    if (d) r = x.slot_to_rank[s];
    __syncwarp();
    if (d) {
      copy_row<VEC>(x.slow + (int64_t)r * x.ld, x.fast + s * x.D, x.D, g.gl, G);
      if (x.S) copy_row<VEC>(x.sstate + (int64_t)r * x.sld, x.fstate + s * x.S, x.S, g.gl, G);
    }
    if (d && g.gl == 0) {
      x.dirty[s] = 0;
      ++cnt;
    }
  }
  cnt = block_sum<kNT>(cnt, sm);
  if (threadIdx.x == 0 && cnt) atomicAdd(&x.c->flush_rows, cnt);
}

int launch_flush(fc_cache* h, cudaStream_t st) {
  RowCtx x = row_ctx(h);
  const bool v = vec_ok(h);
  const int G = row_group(std::max(h->dim, h->sw), v);
  const int grid = grid_for((int64_t)h->capacity * G, kNT, kSMs * 8);
  if (v) k_flush<true><<<grid, kNT, 0, st>>>(x, h->capacity, G);
  else k_flush<false><<<grid, kNT, 0, st>>>(x, h->capacity, G);
  FC_CUDA(cudaGetLastError());
  return FC_OK;
}

// ------------------------------------------------------------- pooled EmbeddingBag forward
template <bool VEC, typename OffT>
__global__ void __launch_bounds__(kNT) k_pool(const float* __restrict__ fast, int D, const int32_t* __restrict__ uslots,
                                              const int32_t* __restrict__ inv, int64_t n, const OffT* __restrict__ off,
                                              int64_t nbags, int incl, const float* __restrict__ psw, int mode,
                                              float* __restrict__ out, int G) {
  GroupIdx g(G);
  for (int64_t base = g.warp * g.gpw; base < nbags; base += g.nwarps * g.gpw) {
    const int64_t b = base + g.gw;
    if (b >= nbags) continue;
    int64_t s, e;
    bag_bounds(off, b, nbags, n, incl, s, e);
    const float scale = (mode == FC_POOL_MEAN) ? (e > s ? 1.0f / (float)(e - s) : 0.0f) : 1.0f;
    if (VEC) {
      for (int c = g.gl * 4; c < D; c += G * 4) {
        float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
        int64_t j = s;
        for (; j + 1 < e; j += 2) {  // two rows in flight per lane
          const int r0 = uslots ? uslots[inv[j]] : inv[j], r1 = uslots ? uslots[inv[j + 1]] : inv[j + 1];
          const float4 v0 = __ldg(reinterpret_cast<const float4*>(fast + (int64_t)r0 * D + c));
          const float4 v1 = __ldg(reinterpret_cast<const float4*>(fast + (int64_t)r1 * D + c));
          const float w0 = psw ? psw[j] : 1.0f, w1 = psw ? psw[j + 1] : 1.0f;
          acc.x += w0 * v0.x; acc.y += w0 * v0.y; acc.z += w0 * v0.z; acc.w += w0 * v0.w;
          acc.x += w1 * v1.x; acc.y += w1 * v1.y; acc.z += w1 * v1.z; acc.w += w1 * v1.w;
        }
        if (j < e) {
          const int r0 = uslots ? uslots[inv[j]] : inv[j];
          const float4 v0 = __ldg(reinterpret_cast<const float4*>(fast + (int64_t)r0 * D + c));
          const float w0 = psw ? psw[j] : 1.0f;
          acc.x += w0 * v0.x; acc.y += w0 * v0.y; acc.z += w0 * v0.z; acc.w += w0 * v0.w;
        }
        acc.x *= scale; acc.y *= scale; acc.z *= scale; acc.w *= scale;
        __stcs(reinterpret_cast<float4*>(out + b * D + c), acc);
      }
    } else {
      for (int c = g.gl; c < D; c += G) {
        float acc = 0.f;
        for (int64_t j = s; j < e; ++j) {
          const float w = psw ? psw[j] : 1.0f;
          acc += w * fast[(int64_t)(uslots ? uslots[inv[j]] : inv[j]) * D + c];
        }
        out[b * D + c] = acc * scale;
      }
    }
  }
}

// bag size 1 (offsets == NULL: gather, or one id per (sample, feature) as in the
// Criteo/Avazu shapes): out[j] = w_j * fast[uslots[inv[j]]], warp-batched
__global__ void __launch_bounds__(kNT) k_pool1(const float* __restrict__ fast, int D, const int32_t* __restrict__ uslots,
                                               const int32_t* __restrict__ inv, int64_t n,
                                               const float* __restrict__ psw, float* __restrict__ out, Units un) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * kNT + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * kNT) >> 5;
  for (int64_t base = warp * 32; base < n; base += nwarps * 32) {
    const int64_t j = base + lane;
    const bool act = j < n;
    int s = 0;
    float w = 1.0f;
    if (act) {
      s = uslots ? uslots[inv[j]] : inv[j];  // uslots == NULL: inv indexes the rows directly
      if (psw) w = psw[j];
    }
    if (psw) warp_move<kUnroll, true>(fast, D, s, out, D, (int)j, act, w, un);
    else warp_move<kUnroll, false>(fast, D, s, out, D, (int)j, act, 1.0f, un);
  }
}

// Bag size 1 through the TMA bulk-copy engine: a one-warp block owns a ring of kPoolStages
// stages of G rows; each lane queues one cp.async.bulk of its occurrence's cached row into
// the stage (completion on the stage's mbarrier), the lanes scale the rows in shared
// memory when there are per-sample weights, and lane 0 writes the G consecutive output
// rows back with ONE bulk store. The SMs only resolve indices: the row bytes move
// HBM -> SMEM -> HBM without passing through registers.
constexpr int kPoolStages = 4;

__global__ void __launch_bounds__(32) k_pool1_tma(const float* __restrict__ fast, int D,
                                                  const int32_t* __restrict__ uslots, const int32_t* __restrict__ inv,
                                                  int64_t n, const float* __restrict__ psw, float* __restrict__ out,
                                                  int G) {
  extern __shared__ __align__(128) unsigned char pring[];  // kPoolStages x G x D floats
  __shared__ uint64_t bar[kPoolStages];
  const int lane = threadIdx.x;
  const unsigned rb = (unsigned)D * 4u;
  if (lane == 0) {
    for (int i = 0; i < kPoolStages; ++i) mbar_init(&bar[i]);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  const int64_t ngroups = (n + G - 1) / G;
  const int64_t mine = ngroups > blockIdx.x ? (ngroups - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  unsigned phase_bits = 0;
  int64_t issued = 0, retired = 0;
  while (retired < mine) {
    // at most kPoolStages - 1 stages loading: the stage refilled next was retired at least one
    // retire ago, so its bulk store is at most the second newest and wait_group.read 1 covers it
    if (issued < mine && issued - retired < kPoolStages - 1) {
      const int st = (int)(issued % kPoolStages);
      if (issued >= kPoolStages) {
        if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
        __syncwarp();
      }
      const int64_t j0 = (blockIdx.x + issued * gridDim.x) * G;
      const int cnt = (int)min((int64_t)G, n - j0);
      if (lane == 0) mbar_expect_tx(&bar[st], (unsigned)cnt * rb);
      __syncwarp();
      float* rows = reinterpret_cast<float*>(pring) + (size_t)st * G * D;
      for (int i = lane; i < cnt; i += 32) {
        const int sl = uslots ? uslots[inv[j0 + i]] : inv[j0 + i];
        bulk_g2s(rows + (size_t)i * D, fast + (int64_t)sl * D, rb, &bar[st]);
      }
      ++issued;
      continue;
    }
    const int st = (int)(retired % kPoolStages);
    mbar_wait(&bar[st], (phase_bits >> st) & 1u);
    phase_bits ^= 1u << st;
    const int64_t j0 = (blockIdx.x + retired * gridDim.x) * G;
    const int cnt = (int)min((int64_t)G, n - j0);
    float* rows = reinterpret_cast<float*>(pring) + (size_t)st * G * D;
    if (psw) {  // out[j] = w_j * row: scale in shared memory, then hand the stage back to the async proxy
      float wl[(32 + 31) / 32 * 1];
      wl[0] = lane < cnt ? psw[j0 + lane] : 0.f;  // G <= 32: one weight per lane
      for (int i = 0; i < cnt; ++i) {
        const float wj = __shfl_sync(FC_FULL, wl[0], i);
        for (int c = lane * 4; c < D; c += 128) {
          float4 v = *reinterpret_cast<float4*>(rows + (size_t)i * D + c);
          v.x *= wj; v.y *= wj; v.z *= wj; v.w *= wj;
          *reinterpret_cast<float4*>(rows + (size_t)i * D + c) = v;
        }
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
    }
    if (lane == 0) {
      bulk_s2g(out + j0 * D, rows, (unsigned)cnt * rb);
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
    __syncwarp();
    ++retired;
  }
  if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int launch_pool(fc_cache* h, const int32_t* uslots, const int32_t* inv, int64_t n, const void* offsets, int off_bytes,
                int64_t nbags, int include_last, const float* psw, int mode, float* out, cudaStream_t st) {
  return launch_pool_rows(h->fast, h->dim, uslots, inv, n, offsets, off_bytes, nbags, include_last, psw, mode, out, st);
}

// pooled forward over any row buffer; uslots == NULL means row = inv[j]
int launch_pool_rows(const float* rows, int D, const int32_t* uslots, const int32_t* inv, int64_t n,
                     const void* offsets, int off_bytes, int64_t nbags, int include_last, const float* psw, int mode,
                     float* out, cudaStream_t st) {
  if (nbags <= 0) return FC_OK;
  const bool v = (D % 4 == 0) && (((reinterpret_cast<uintptr_t>(out) | reinterpret_cast<uintptr_t>(rows)) & 15) == 0);
  // FC_POOL_TMA=1: bag size 1 without weights through the bulk-copy engine. Alone it
  // matches the register path (72.8 vs ~73 us at cfg2, profiles/r02_pool_tma_bench.txt),
  // but inside the prefetch pipeline it is slower (0.27-0.29 vs 0.18-0.24 ms in-step,
  // 346 vs 371 M lookups/s, profiles/r02_ab_pool.txt), so the register path is the default.
  static const bool use_tma = std::getenv("FC_POOL_TMA") != nullptr && std::atoi(std::getenv("FC_POOL_TMA")) != 0;
  if (v && offsets == nullptr && !psw && use_tma && D * 4 <= 8192) {
    const int G = std::max(1, std::min(32, 16384 / (D * 4)));
    const size_t smem = (size_t)kPoolStages * G * D * 4;
    static bool attr = false;
    if (!attr && smem > 48 * 1024) {
      FC_CUDA(cudaFuncSetAttribute(k_pool1_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
      attr = true;
    }
    const int per_sm = std::max(1, std::min(16, (int)((220 * 1024) / smem)));
    const int64_t groups = (nbags + G - 1) / G;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(groups, (int64_t)kSMs * per_sm));
    k_pool1_tma<<<grid, 32, smem, st>>>(rows, D, uslots, inv, nbags, psw, out, G);
    FC_CUDA(cudaGetLastError());
    return FC_OK;
  }
  if (v && offsets == nullptr) {  // bag size 1: one row per bag
    k_pool1<<<grid_for(nbags, kNT, kSMs * 8), kNT, 0, st>>>(rows, D, uslots, inv, nbags, psw, out, units_for(D));
    FC_CUDA(cudaGetLastError());
    return FC_OK;
  }
  const int G = row_group(D, v);
  const int grid = grid_for(nbags * G, kNT, kSMs * 16);
#define FC_POOL(VV, T) \
  k_pool<VV, T><<<grid, kNT, 0, st>>>(rows, D, uslots, inv, n, (const T*)offsets, nbags, include_last, psw, mode, out, G)
  if (off_bytes == 4) {
    if (v) FC_POOL(true, int32_t); else FC_POOL(false, int32_t);
  } else {
    if (v) FC_POOL(true, long long); else FC_POOL(false, long long);
  }
#undef FC_POOL
  FC_CUDA(cudaGetLastError());
  return FC_OK;
}

// ------------------------------------------------------------- pooled rows straight to the requesters
// Row-sharded forward, owner side, fused with the return exchange: received id i (from
// requester r = the segment of i in seg[0..W]) is looked up in the cache and its row is
// written directly into requester r's receive buffer over NVLink peer memory (CUDA IPC /
// symmetric pointers), at row dst_off[r] + (i - seg[r]). Replaces "pool into a local
// buffer, then all-to-all". The caller orders it before a stream-ordered barrier.
// Column-wise split (fc_pool_cols_to_peers): the destination rows are ld floats wide and this
// rank's slice starts at column col; psw (optional) scales occurrence i's row.
__global__ void __launch_bounds__(kNT) k_pool_to_peers(const float* __restrict__ fast, int D,
                                                       const int32_t* __restrict__ uslots,
                                                       const int32_t* __restrict__ inv, int64_t n,
                                                       const int64_t* __restrict__ seg, int W,
                                                       float* const* __restrict__ dst, const int64_t* __restrict__ dst_off,
                                                       Units un, int64_t ld, int64_t col,
                                                       const float* __restrict__ psw) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * kNT + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * kNT) >> 5;
  for (int64_t base = warp * 32; base < n; base += nwarps * 32) {
    const int64_t i = base + lane;
    const bool act = i < n;
    const float* src = nullptr;
    float* out = nullptr;
    float w = 1.f;
    if (act) {
      int r = 0;
      while (r + 1 < W && seg[r + 1] <= i) ++r;  // W <= 64: a short scan
      src = fast + (int64_t)uslots[inv[i]] * D;
      out = dst[r] + (dst_off[r] + (i - seg[r])) * ld + col;
      if (psw) w = psw[i];
    }
    // lanes sweep the 32 rows' 16-byte units (4 in flight), writing to each row's owner
    const int total = 32 * un.upr;
    for (int u0 = 0; u0 < total; u0 += 32 * 4) {
      float4 v[4];
      float* d[4];
      bool a[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int u = u0 + q * 32 + lane;
        const int rr = min(un.row(u), 31);
        const int c = (u - rr * un.upr) * 4;
        const float* sp = reinterpret_cast<const float*>(__shfl_sync(FC_FULL, reinterpret_cast<long long>(src), rr));
        d[q] = reinterpret_cast<float*>(__shfl_sync(FC_FULL, reinterpret_cast<long long>(out), rr)) + c;
        a[q] = __shfl_sync(FC_FULL, (int)act, rr) && u < total;
        const float wq = __shfl_sync(FC_FULL, w, rr);
        if (a[q]) {
          v[q] = ld4(sp + c);
          if (psw) v[q] = make_float4(__fmul_rn(v[q].x, wq), __fmul_rn(v[q].y, wq), __fmul_rn(v[q].z, wq),
                                      __fmul_rn(v[q].w, wq));
        }
      }
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (a[q]) st4(d[q], v[q]);
    }
  }
  __threadfence_system();  // peer-memory stores visible before the caller's barrier
}

int launch_pool_to_peers(fc_cache* h, const int32_t* uslots, const int32_t* inv, int64_t n, const int64_t* seg, int W,
                         float* const* dst, const int64_t* dst_off, cudaStream_t st) {
  if (n <= 0) return FC_OK;
  if (h->dim % 4) {
    set_error("pool_to_peers needs dim %% 4 == 0");
    return FC_ERR_BAD_ARG;
  }
  k_pool_to_peers<<<grid_for(n, kNT, kSMs * 8), kNT, 0, st>>>(h->fast, h->dim, uslots, inv, n, seg, W, dst, dst_off,
                                                              units_for(h->dim), h->dim, 0, nullptr);
  FC_CUDA(cudaGetLastError());
  return FC_OK;
}

int launch_pool_cols_to_peers(fc_cache* h, const int32_t* uslots, const int32_t* inv, int64_t n, const int64_t* seg,
                              int W, float* const* dst, const int64_t* dst_off, int64_t ld, int64_t col,
                              const float* psw, cudaStream_t st) {
  if (n <= 0) return FC_OK;
  if (h->dim % 4 || ld % 4 || col % 4 || col + h->dim > ld) {
    set_error("pool_cols_to_peers needs 16-byte aligned column slices (dim %d, ld %lld, col %lld)", h->dim,
              (long long)ld, (long long)col);
    return FC_ERR_BAD_ARG;
  }
  k_pool_to_peers<<<grid_for(n, kNT, kSMs * 8), kNT, 0, st>>>(h->fast, h->dim, uslots, inv, n, seg, W, dst, dst_off,
                                                              units_for(h->dim), ld, col, psw);
  FC_CUDA(cudaGetLastError());
  return FC_OK;
}

// The mirror for the backward: the owner pulls the gradient rows of its received ids
// from the requesters' buffers over peer memory — received id i (requester r = segment
// of i) reads src[r] row src_off[r] + (i - seg[r]) — into a local contiguous [n, D].
__global__ void __launch_bounds__(kNT) k_gather_from_peers(const float* const* __restrict__ src,
                                                           const int64_t* __restrict__ src_off,
                                                           const int64_t* __restrict__ seg, int W, int64_t n, int D,
                                                           float* __restrict__ out, Units un, int64_t ld, int64_t col) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * kNT + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * kNT) >> 5;
  for (int64_t base = warp * 32; base < n; base += nwarps * 32) {
    const int64_t i = base + lane;
    const bool act = i < n;
    const float* sp = nullptr;
    if (act) {
      int r = 0;
      while (r + 1 < W && seg[r + 1] <= i) ++r;
      sp = src[r] + (src_off[r] + (i - seg[r])) * ld + col;
    }
    const int total = 32 * un.upr;
    for (int u0 = 0; u0 < total; u0 += 32 * 4) {
      float4 v[4];
      int64_t d[4];
      bool a[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int u = u0 + q * 32 + lane;
        const int rr = min(un.row(u), 31);
        const int c = (u - rr * un.upr) * 4;
        const float* s = reinterpret_cast<const float*>(__shfl_sync(FC_FULL, reinterpret_cast<long long>(sp), rr));
        d[q] = (base + rr) * D + c;
        a[q] = __shfl_sync(FC_FULL, (int)act, rr) && u < total;
        if (a[q]) v[q] = ld4(s + c);
      }
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (a[q]) st4(out + d[q], v[q]);
    }
  }
}

int launch_gather_from_peers(const float* const* src, const int64_t* src_off, const int64_t* seg, int W, int64_t n,
                             int D, float* out, cudaStream_t st) {
  if (n <= 0) return FC_OK;
  k_gather_from_peers<<<grid_for(n, kNT, kSMs * 8), kNT, 0, st>>>(src, src_off, seg, W, n, D, out, units_for(D), D, 0);
  FC_CUDA(cudaGetLastError());
  return FC_OK;
}

int launch_gather_cols_from_peers(const float* const* src, const int64_t* src_off, const int64_t* seg, int W,
                                  int64_t n, int D, int64_t ld, int64_t col, float* out, cudaStream_t st) {
  if (n <= 0) return FC_OK;
  if (D % 4 || ld % 4 || col % 4 || col + D > ld) {
    set_error("gather_cols_from_peers needs 16-byte aligned column slices (dim %d, ld %lld, col %lld)", D,
              (long long)ld, (long long)col);
    return FC_ERR_BAD_ARG;
  }
  k_gather_from_peers<<<grid_for(n, kNT, kSMs * 8), kNT, 0, st>>>(src, src_off, seg, W, n, D, out, units_for(D), ld,
                                                                  col);
  FC_CUDA(cudaGetLastError());
  return FC_OK;
}

// ------------------------------------------------------------- gather_unique (:509-510)
template <bool VEC>
__global__ void __launch_bounds__(kNT) k_gather_rows(const float* __restrict__ fast, int D, const int32_t* __restrict__ slots,
                                                     int64_t n, float* __restrict__ out, int G) {
  GroupIdx g(G);
  for (int64_t base = g.warp * g.gpw; base < n; base += g.nwarps * g.gpw) {
    const int64_t p = base + g.gw;
    if (p < n) copy_row<VEC>(out + p * D, fast + (int64_t)slots[p] * D, D, g.gl, G);
  }
}

int launch_gather_rows(fc_cache* h, const int32_t* slots, int64_t n, float* out, cudaStream_t st) {
  if (n <= 0) return FC_OK;
  const bool v = (h->dim % 4 == 0) && ((reinterpret_cast<uintptr_t>(out) & 15) == 0);
  const int G = row_group(h->dim, v);
  const int grid = grid_for(n * G, kNT, kSMs * 16);
  if (v) k_gather_rows<true><<<grid, kNT, 0, st>>>(h->fast, h->dim, slots, n, out, G);
  else k_gather_rows<false><<<grid, kNT, 0, st>>>(h->fast, h->dim, slots, n, out, G);
  FC_CUDA(cudaGetLastError());
  return FC_OK;
}

// ------------------------------------------------------------- apply_unique_update (:517-523)
__global__ void __launch_bounds__(kNT) k_unique_add(float* fast, int D, const int32_t* __restrict__ uslots, int64_t u,
                                                    const float* __restrict__ add, uint8_t* dirty, int G) {
  GroupIdx g(G);
  for (int64_t base = g.warp * g.gpw; base < u; base += g.nwarps * g.gpw) {
    const int64_t p = base + g.gw;
    if (p >= u) continue;
    const int64_t s = uslots[p];
    for (int c = g.gl; c < D; c += G) fast[s * D + c] = __fadd_rn(fast[s * D + c], add[p * D + c]);
    if (g.gl == 0) dirty[s] = 1;
  }
}

int launch_unique_add(fc_cache* h, const int32_t* uslots, int64_t u, const float* add, cudaStream_t st) {
  if (u <= 0) return FC_OK;
  const int G = row_group(h->dim, false);
  k_unique_add<<<grid_for(u * G, kNT, kSMs * 16), kNT, 0, st>>>(h->fast, h->dim, uslots, u, add, h->dirty, G);
  FC_CUDA(cudaGetLastError());
  return FC_OK;
}

// ------------------------------------------------------------- the simulator's update (simulator.py:229-260,433)
__device__ __forceinline__ float hash_unit(uint64_t v, uint64_t salt) {
  uint64_t z = v * 0x9E3779B97F4A7C15ull + salt;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  z ^= z >> 31;
  return __fmul_rn(__uint2float_rn((unsigned)(z >> 40)), 5.9604644775390625e-08f);  // * 2^-24, exact
}

template <bool VEC>
__global__ void __launch_bounds__(kNT) k_synthetic(float* fast, int D, const int32_t* __restrict__ uids,
                                                   const int32_t* __restrict__ ucnt, const int32_t* __restrict__ uslots,
                                                   int64_t u, uint64_t salt, const float* __restrict__ colw,
                                                   uint8_t* dirty, int G, Units un) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * kNT + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * kNT) >> 5;
  for (int64_t base = warp * 32; base < u; base += nwarps * 32) {
    const int64_t p = base + lane;
    const bool act = p < u;
    int s = 0;
    float gs = 0.f;
    if (act) {
      s = uslots[p];
      // g = (hash - 0.5) * count, all fp32 with round-to-nearest like numpy (simulator.py:258-260)
      gs = __fmul_rn(__fsub_rn(hash_unit((uint64_t)uids[p], salt), 0.5f), __int2float_rn(ucnt[p]));
    }
    if (VEC) {
      const int total = 32 * un.upr;
      for (int u0 = 0; u0 < total; u0 += 32 * kUnroll) {
        float4 v[kUnroll], cw[kUnroll];
        float* rp[kUnroll];
        float gk[kUnroll];
        bool aa[kUnroll];
#pragma unroll
        for (int k = 0; k < kUnroll; ++k) {
          const int q = u0 + k * 32 + lane;
          const int r = min(un.row(q), 31);
          const int c = (q - r * un.upr) * 4;
          const int sr = __shfl_sync(FC_FULL, s, r);
          gk[k] = __shfl_sync(FC_FULL, gs, r);
          aa[k] = __shfl_sync(FC_FULL, (int)act, r) && q < total;
          rp[k] = fast + (int64_t)sr * D + c;
          if (aa[k]) {
            v[k] = ld4(rp[k]);
            cw[k] = ldg4(colw + c);
          }
        }
#pragma unroll
        for (int k = 0; k < kUnroll; ++k)
          if (aa[k]) {
            float4 w = v[k];
            w.x = __fadd_rn(w.x, __fmul_rn(gk[k], cw[k].x));
            w.y = __fadd_rn(w.y, __fmul_rn(gk[k], cw[k].y));
            w.z = __fadd_rn(w.z, __fmul_rn(gk[k], cw[k].z));
            w.w = __fadd_rn(w.w, __fmul_rn(gk[k], cw[k].w));
            st4(rp[k], w);
          }
      }
    } else {
      for (int q = 0; q < 32; ++q) {
        const bool aq = __shfl_sync(FC_FULL, (int)act, q);
        const int sq = __shfl_sync(FC_FULL, s, q);
        const float gq = __shfl_sync(FC_FULL, gs, q);
        if (aq)
          for (int c = lane; c < D; c += 32) {
            float* e = fast + (int64_t)sq * D + c;
            *e = __fadd_rn(*e, __fmul_rn(gq, colw[c]));
          }
      }
    }
    if (act) dirty[s] = 1;
  }
  (void)G;
}

int launch_synthetic(fc_cache* h, const int32_t* uids, const int32_t* ucnt, const int32_t* uslots, int64_t u,
                     uint64_t salt, const float* colw, cudaStream_t st) {
  if (u <= 0) return FC_OK;
  const bool v = (h->dim % 4 == 0) && ((reinterpret_cast<uintptr_t>(colw) & 15) == 0);
  const int G = row_group(h->dim, v);
  const int grid = grid_for(u * G, kNT, kSMs * 16);
  const int grid_w = grid_for(u, kNT, kSMs * 8);
  if (v)
    k_synthetic<true><<<grid_w, kNT, 0, st>>>(h->fast, h->dim, uids, ucnt, uslots, u, salt, colw, h->dirty, G,
                                              units_for(h->dim));
  else
    k_synthetic<false><<<grid_w, kNT, 0, st>>>(h->fast, h->dim, uids, ucnt, uslots, u, salt, colw, h->dirty, G,
                                               units_for(4));
  (void)grid;
  FC_CUDA(cudaGetLastError());
  return FC_OK;
}

}  // namespace fc
