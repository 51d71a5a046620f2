// Occurrence grouping, scatter_update and the fused backward + sparse optimizer.
//
// Both paths first group a batch's occurrences by unique row with a stable radix
// sort of `inverse` (so batch order is kept inside a group):
//   * scatter_update (/root/reference/pkg/src/freqcache/cache_manager.py:423-438)
//     then adds each group's deltas in batch order — bit-exact with np.add.at;
//   * the backward of the pooled forward (north star item 6) streams the sorted
//     occurrences once: each warp owns a chunk of kChunk consecutive sorted
//     occurrences and accumulates coef_j * grad_out[bag(j)] per run of equal rows in
//     registers (one float4 column unit per lane, kBwdUnroll grad rows in flight).
//     The optimizer step is fused into that pass: a run that starts and ends inside
//     its chunk (almost every row) updates its cached row (SGD, or Adagrad with the
//     state row) the moment it closes, with the row fetched when the run opened;
//     runs cut by chunk edges leave carries that one fix-up pass sums (a block per
//     split row, its warps summing contiguous slices of the chain, combined in warp
//     order) and then updates. No per-row gradient buffer; fixed order ->
//     deterministic. (FC_BWD_UNFUSED=1 selects sums-then-apply, k_bwd_apply.)
#include <algorithm>
#include <cstdlib>

#include "fc_rowutil.cuh"

namespace fc {

// (overridable at build time for tuning sweeps: tools/build_bwd_variants.sh)
#ifndef FC_BWD_CHUNK
#define FC_BWD_CHUNK 64
#endif
#ifndef FC_BWD_UNROLL
#define FC_BWD_UNROLL 4
#endif
#ifndef FC_BWD_MINBLOCKS
#define FC_BWD_MINBLOCKS 4
#endif
constexpr int kChunk = FC_BWD_CHUNK;  // sorted occurrences per warp in the backward stream
constexpr int kBwdUnroll = FC_BWD_UNROLL;

struct Grouping {
  uint32_t* keys;   // [n] sorted unique positions
  int32_t* order;   // [n] occurrence index of each sorted position
  void* sort_scr;   // the radix sort's scratch (its zero-initialised state at the head)
  char* rest;
};

static size_t grouping_bytes(int64_t n) { return align16(n * 4) * 2 + align16(sort_scratch_bytes(n)); }

static int build_grouping(void** scratch, size_t* scratch_bytes, const int32_t* inv, int64_t u, int64_t n,
                          size_t extra, Grouping& g, cudaStream_t st, bool state_zeroed = false,
                          const int32_t* sort_hist = nullptr) {
  int rc = ensure_scratch_buf(scratch, scratch_bytes, grouping_bytes(n) + extra);
  if (rc) return rc;
  char* p = static_cast<char*>(*scratch);
  g.keys = reinterpret_cast<uint32_t*>(p);
  p += align16(n * 4);
  g.order = reinterpret_cast<int32_t*>(p);
  p += align16(n * 4);
  void* sort_scr = p;
  g.sort_scr = sort_scr;
  p += align16(sort_scratch_bytes(n));
  g.rest = p;
  return radix_sort_pairs(reinterpret_cast<const uint32_t*>(inv), nullptr, g.keys, g.order, n, key_bits_for(u),
                          sort_scr, st, state_zeroed, sort_hist);
}

// ------------------------------------------------------------- scatter_update, bit-exact with np.add.at
__global__ void __launch_bounds__(kNT) k_seg_add_seq(float* fast, int D, const int32_t* __restrict__ uslots, int64_t u,
                                                     const int32_t* __restrict__ seg, const int32_t* __restrict__ order,
                                                     const float* __restrict__ deltas, uint8_t* dirty) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * kNT + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * kNT) >> 5;
  for (int64_t p = warp; p < u; p += nwarps) {  // one warp per unique row, lanes over columns
    const int64_t s = uslots[p];
    float* row = fast + s * D;
    const int j0 = seg[p], j1 = seg[p + 1];
    for (int c = lane; c < D; c += 32) {
      float acc = row[c];
      for (int j = j0; j < j1; ++j) acc = __fadd_rn(acc, deltas[(int64_t)order[j] * D + c]);  // batch order
      row[c] = acc;
    }
    if (lane == 0) dirty[s] = 1;
  }
}

int launch_scatter_update(fc_cache* h, const int32_t* uslots, const int32_t* inv, const int32_t* ucnt, int64_t u,
                          int64_t n, const float* deltas, cudaStream_t st) {
  if (u <= 0 || n <= 0) return FC_OK;
  Grouping g;
  const size_t extra = align16((u + 1) * 4) + align16(scan_scratch_bytes(u));
  h->sort_zero_for = nullptr;  // this sort leaves its state behind
  int rc = build_grouping(&h->scratch, &h->scratch_bytes, inv, u, n, extra, g, st);
  if (rc) return rc;
  int32_t* seg = reinterpret_cast<int32_t*>(g.rest);
  void* scan_scr = g.rest + align16((u + 1) * 4);
  rc = exclusive_scan_i32(ucnt, seg, u, scan_scr, st);
  if (rc) return rc;
  k_seg_add_seq<<<grid_for(u * 32, kNT, kSMs * 16), kNT, 0, st>>>(h->fast, h->dim, uslots, u, seg, g.order, deltas,
                                                                 h->dirty);
  FC_CUDA(cudaGetLastError());
  return FC_OK;
}

// ------------------------------------------------------------- backward + sparse optimizer
struct OptArgs {
  int optim;
  float lr, eps;
};

__device__ __forceinline__ float opt1(float w, float* st, float g, const OptArgs& o) {
  if (o.optim == FC_OPT_ADAGRAD) {  // torch.optim.Adagrad: G += g^2; w -= lr * g / (sqrt(G) + eps)
    const float s = *st + g * g;
    *st = s;
    return w - o.lr * g / (sqrtf(s) + o.eps);
  }
  return w - o.lr * g;  // torch.optim.SGD
}

// optimizer step on one 16-byte unit already in registers (row v, state sv), stored back
__device__ __forceinline__ void apply_unit_regs(float* w, float* st, float4 v, float4 sv, float4 g, const OptArgs& o) {
  if (st) {
    v.x = opt1(v.x, &sv.x, g.x, o);
    v.y = opt1(v.y, &sv.y, g.y, o);
    v.z = opt1(v.z, &sv.z, g.z, o);
    v.w = opt1(v.w, &sv.w, g.w, o);
    st4(st, sv);
  } else {
    v.x -= o.lr * g.x;
    v.y -= o.lr * g.y;
    v.z -= o.lr * g.z;
    v.w -= o.lr * g.w;
  }
  st4(w, v);
}

__device__ __forceinline__ void apply_unit(float* w, float* st, float4 g, const OptArgs& o) {
  float4 v = ld4(w);
  if (st) {
    v.x = opt1(v.x, st + 0, g.x, o);
    v.y = opt1(v.y, st + 1, g.y, o);
    v.z = opt1(v.z, st + 2, g.z, o);
    v.w = opt1(v.w, st + 3, g.w, o);
  } else {
    v.x -= o.lr * g.x;
    v.y -= o.lr * g.y;
    v.z -= o.lr * g.z;
    v.w -= o.lr * g.w;
  }
  st4(w, v);
}

template <typename OffT>
__global__ void __launch_bounds__(kNT) k_bag_coef(const OffT* __restrict__ off, int64_t nbags, int64_t n, int incl,
                                                  const float* __restrict__ psw, int mode, int32_t* bag_of,
                                                  float* coef) {
  for (int64_t b = (int64_t)blockIdx.x * kNT + threadIdx.x; b < nbags; b += (int64_t)gridDim.x * kNT) {
    int64_t s, e;
    bag_bounds(off, b, nbags, n, incl, s, e);
    const float scale = (mode == FC_POOL_MEAN) ? (e > s ? 1.0f / (float)(e - s) : 0.0f) : 1.0f;
    for (int64_t j = s; j < e; ++j) {
      bag_of[j] = (int32_t)b;
      coef[j] = psw ? scale * psw[j] : scale;
    }
  }
}

struct BwdArgs {
  float* fast;
  float* fstate;
  int D;
  const int32_t* uslots;
  const uint32_t* keys;
  const int32_t* order;
  int64_t n;
  const int32_t* bag_of;  // NULL: bag = occurrence
  const float* coef;      // NULL: coef = 1 (or psw)
  const float* psw;
  const float* grad;
  float* gu;              // [u, D] summed gradient per unique row
  float* carry;           // [nchunks * 2, D]
  int32_t* carry_key;     // [nchunks * 2] (-1 none)
  int32_t* carry_flag;    // bit0: run open at chunk start, bit1: open at chunk end
  uint8_t* dirty;
  OptArgs o;
  Units un;
  uint32_t* zero;     // the fix-up clears these words (the next sort's state) when set
  int64_t zero_words;
};

// One finished run of key `key` over sorted positions [a, b) of chunk c. A run that
// lies inside the chunk is final: APPLY updates the cached row right here with the
// row (and optimizer state) prefetched when the run started; otherwise its sum goes to
// gu[key] (coalesced). A run cut by a chunk edge is parked as a carry for the fix-up.
template <bool APPLY>
__device__ __forceinline__ void bwd_flush(const BwdArgs& x, int64_t c, int64_t j0, int64_t j1, int key, int64_t a,
                                          int64_t b, int prev_key, int next_key, float4 acc, int unit, bool has,
                                          bool first_col, int slot, float4 wrow, float4 srow) {
  const bool open_s = (a == j0) && (prev_key == key);
  const bool open_e = (b == j1) && (next_key == key);
  if (!open_s && !open_e) {
    if (APPLY) {
      if (has) {
        float* w = x.fast + (int64_t)slot * x.D + unit * 4;
        apply_unit_regs(w, x.fstate ? x.fstate + (w - x.fast) : nullptr, wrow, srow, acc, x.o);
      }
      if (first_col && (threadIdx.x & 31) == 0) x.dirty[slot] = 1;
    } else if (has) {
      st4(x.gu + (int64_t)key * x.D + unit * 4, acc);
    }
  } else {
    const int64_t cs = c * 2 + (open_s ? 0 : 1);
    if (has) st4(x.carry + cs * x.D + unit * 4, acc);
    if (first_col && (threadIdx.x & 31) == 0) {
      x.carry_key[cs] = key;
      x.carry_flag[cs] = (open_s ? 1 : 0) | (open_e ? 2 : 0);
    }
  }
}

template <bool APPLY>
__global__ void __launch_bounds__(kNT, FC_BWD_MINBLOCKS) k_bwd_stream(BwdArgs x) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * kNT + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * kNT) >> 5;
  const int64_t nchunks = (x.n + kChunk - 1) / kChunk;
  for (int64_t c = warp; c < nchunks; c += nwarps) {
    const int64_t j0 = c * kChunk, j1 = min(x.n, j0 + kChunk);
    // this chunk's two carry slots start empty (lane 0 may fill them in bwd_flush, later)
    if (lane == 0) {
      x.carry_key[c * 2] = -1;
      x.carry_key[c * 2 + 1] = -1;
    }
    const int prev_key = j0 > 0 ? (int)x.keys[j0 - 1] : -1;
    const int next_key = j1 < x.n ? (int)x.keys[j1] : -1;
    for (int cu0 = 0; cu0 < x.un.upr; cu0 += 32) {
      const int unit = cu0 + lane;
      const bool has = unit < x.un.upr;
      float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
      float4 wrow = acc, srow = acc;
      int cur = -1, cur_slot = 0;
      int64_t run_a = j0;
      for (int64_t r0 = j0; r0 < j1; r0 += 32) {
        const int64_t jj = r0 + lane;
        int kl = -1, bag = 0, sl = 0;
        float cf = 0.f;
        if (jj < j1) {
          kl = (int)x.keys[jj];
          const int occ = x.order[jj];
          bag = x.bag_of ? x.bag_of[occ] : occ;
          cf = x.coef ? x.coef[occ] : (x.psw ? x.psw[occ] : 1.0f);
          if (APPLY) sl = x.uslots[kl];
        }
        const int cnt = (int)(j1 - r0 < 32 ? j1 - r0 : 32);
        for (int q = 0; q < cnt; q += kBwdUnroll) {
          float4 g[kBwdUnroll];
          int kq[kBwdUnroll], sq[kBwdUnroll];
          float cq[kBwdUnroll];
#pragma unroll
          for (int k = 0; k < kBwdUnroll; ++k) {
            const int src = min(q + k, 31);
            const int bq = __shfl_sync(FC_FULL, bag, src);
            kq[k] = __shfl_sync(FC_FULL, kl, src);
            cq[k] = __shfl_sync(FC_FULL, cf, src);
            sq[k] = APPLY ? __shfl_sync(FC_FULL, sl, src) : 0;
            g[k] = make_float4(0.f, 0.f, 0.f, 0.f);
            if (has && q + k < cnt) g[k] = ldg4(x.grad + (int64_t)bq * x.D + unit * 4);
          }
#pragma unroll
          for (int k = 0; k < kBwdUnroll; ++k) {
            if (q + k >= cnt) break;
            if (kq[k] != cur) {
              if (cur >= 0)
                bwd_flush<APPLY>(x, c, j0, j1, cur, run_a, r0 + q + k, prev_key, next_key, acc, unit, has, cu0 == 0,
                                 cur_slot, wrow, srow);
              cur = kq[k];
              cur_slot = sq[k];
              run_a = r0 + q + k;
              acc = make_float4(0.f, 0.f, 0.f, 0.f);
              if (APPLY && has) {  // the run's row, fetched while its gradients stream in
                const float* w = x.fast + (int64_t)cur_slot * x.D + unit * 4;
                wrow = ld4(w);
                if (x.fstate) srow = ld4(x.fstate + (w - x.fast));
              }
            }
            acc.x += cq[k] * g[k].x;
            acc.y += cq[k] * g[k].y;
            acc.z += cq[k] * g[k].z;
            acc.w += cq[k] * g[k].w;
          }
        }
      }
      if (cur >= 0)
        bwd_flush<APPLY>(x, c, j0, j1, cur, run_a, j1, prev_key, next_key, acc, unit, has, cu0 == 0, cur_slot, wrow,
                         srow);
    }
  }
}

// Runs cut by chunk boundaries: chunk c's end-open run (slot 1) starts a split
// row; the following chunks' start-open runs (slot 0) continue it until one is
// closed at its end. One block per chunk index; blocks whose chunk starts no
// chain exit at once. A chain's carries are split into kFixWarps contiguous
// slices, each summed by one warp (16 loads in flight), and the slices are added
// in warp order: a hot row spanning hundreds of chunks costs a few latencies,
// not hundreds. The row's sum lands in gu like every other row's.
constexpr int kFixWarps = kNT / 32;

template <bool APPLY>
__global__ void __launch_bounds__(kNT) k_bwd_fixup(BwdArgs x) {
  extern __shared__ float4 part[];  // [kFixWarps][units per row]
  __shared__ int64_t s_m;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int64_t nchunks = (x.n + kChunk - 1) / kChunk;
  for (int64_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
    const int key = x.carry_key[c * 2 + 1];
    if (key < 0) continue;  // uniform across the block
    if (wid == 0) {  // extent: chunks c+1 .. c+m whose slot 0 carries `key`; the last is closed at its end
      int64_t m = 0;
      for (int64_t base = c + 1; base < nchunks; base += 32) {
        const int64_t cc = base + lane;
        const bool cont = cc < nchunks && x.carry_key[cc * 2] == key;
        const bool last = cont && !(x.carry_flag[cc * 2] & 2);
        const unsigned lastm = __ballot_sync(FC_FULL, last);
        const unsigned contm = __ballot_sync(FC_FULL, cont);
        if (lastm) {
          m += __ffs(lastm);
          break;
        }
        m += __popc(contm);
        if (contm != FC_FULL) break;
      }
      if (lane == 0) s_m = m;
    }
    __syncthreads();
    const int64_t m = s_m;
    // carries in chain order: k = 0 is chunk c's slot 1, k = 1..m are chunks c+k's slot 0
    const int64_t per = (m + 1 + kFixWarps - 1) / kFixWarps;
    const int64_t k0 = wid * per, k1 = min(m + 1, k0 + per);
    for (int cu0 = 0; cu0 < x.un.upr; cu0 += 32) {
      const int unit = cu0 + lane;
      const bool has = unit < x.un.upr;
      float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
      if (has) {
        int64_t k = k0;
        constexpr int kF = 16;
        for (; k + kF <= k1; k += kF) {
          float4 v[kF];
#pragma unroll
          for (int q = 0; q < kF; ++q) {
            const int64_t slot = (k + q == 0) ? c * 2 + 1 : (c + k + q) * 2;
            v[q] = ld4(x.carry + slot * x.D + unit * 4);
          }
#pragma unroll
          for (int q = 0; q < kF; ++q) {
            acc.x += v[q].x; acc.y += v[q].y; acc.z += v[q].z; acc.w += v[q].w;
          }
        }
        for (; k < k1; ++k) {
          const int64_t slot = (k == 0) ? c * 2 + 1 : (c + k) * 2;
          const float4 v = ld4(x.carry + slot * x.D + unit * 4);
          acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
        }
        part[wid * x.un.upr + unit] = acc;
      }
    }
    __syncthreads();
    if (wid == 0) {
      const int64_t slot = APPLY ? x.uslots[key] : 0;
      for (int unit = lane; unit < x.un.upr; unit += 32) {
        float4 acc = part[unit];
        for (int w = 1; w < kFixWarps; ++w) {
          const float4 v = part[w * x.un.upr + unit];
          acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
        }
        if (APPLY) {
          float* wr = x.fast + slot * x.D + unit * 4;
          apply_unit(wr, x.fstate ? x.fstate + (wr - x.fast) : nullptr, acc, x.o);
        } else {
          st4(x.gu + (int64_t)key * x.D + unit * 4, acc);
        }
      }
      if (APPLY && lane == 0) x.dirty[slot] = 1;
    }
    __syncthreads();
  }
  // the sort that produced keys/order is complete: clear its state for the next backward,
  // which then queues no memset (a launch costs ~90 us beside the miss staging, DESIGN 4b)
  if (x.zero)
    for (int64_t i = (int64_t)blockIdx.x * kNT + threadIdx.x; i < x.zero_words; i += (int64_t)gridDim.x * kNT)
      x.zero[i] = 0u;
}

// optimizer step on every unique row, 32 rows per warp, kBwdUnroll units in flight
__global__ void __launch_bounds__(kNT) k_bwd_apply(BwdArgs x, int64_t u) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * kNT + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * kNT) >> 5;
  const int total = 32 * x.un.upr;
  for (int64_t base = warp * 32; base < u; base += nwarps * 32) {
    const int64_t p = base + lane;
    const bool act = p < u;
    const int s = act ? x.uslots[p] : 0;
    for (int u0 = 0; u0 < total; u0 += 32 * kBwdUnroll) {
      float4 g[kBwdUnroll];
      float* w[kBwdUnroll];
      bool aa[kBwdUnroll];
#pragma unroll
      for (int k = 0; k < kBwdUnroll; ++k) {
        const int q = u0 + k * 32 + lane;
        const int r = min(x.un.row(q), 31);
        const int c = (q - r * x.un.upr) * 4;
        const int sr = __shfl_sync(FC_FULL, s, r);
        aa[k] = __shfl_sync(FC_FULL, (int)act, r) && q < total;
        w[k] = x.fast + (int64_t)sr * x.D + c;
        if (aa[k]) g[k] = ld4(x.gu + (base + r) * x.D + c);
      }
#pragma unroll
      for (int k = 0; k < kBwdUnroll; ++k)
        if (aa[k]) {
          float* stp = x.fstate ? x.fstate + (w[k] - x.fast) : nullptr;
          apply_unit(w[k], stp, g[k], x.o);
        }
    }
    if (act) x.dirty[s] = 1;
  }
}

// Every unique row has exactly one gradient row (u == n, no bags, no weights: the
// row-sharded owner receiving one row per distinct id): `inverse` is a permutation,
// so no grouping is needed -- occurrence i updates slot uslots[inv[i]] directly with
// the same arithmetic as a one-element run of k_bwd_stream.
__global__ void __launch_bounds__(kNT) k_bwd_direct(BwdArgs x, const int32_t* __restrict__ inv) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * kNT + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * kNT) >> 5;
  const int total = 32 * x.un.upr;
  for (int64_t base = warp * 32; base < x.n; base += nwarps * 32) {
    const int64_t i = base + lane;
    const bool act = i < x.n;
    const int s = act ? x.uslots[inv[i]] : 0;
    for (int u0 = 0; u0 < total; u0 += 32 * kBwdUnroll) {
      float4 g[kBwdUnroll];
      float* w[kBwdUnroll];
      bool aa[kBwdUnroll];
#pragma unroll
      for (int k = 0; k < kBwdUnroll; ++k) {
        const int q = u0 + k * 32 + lane;
        const int r = min(x.un.row(q), 31);
        const int c = (q - r * x.un.upr) * 4;
        const int sr = __shfl_sync(FC_FULL, s, r);
        aa[k] = __shfl_sync(FC_FULL, (int)act, r) && q < total;
        w[k] = x.fast + (int64_t)sr * x.D + c;
        if (aa[k]) {
          const float4 v = ld4(x.grad + (base + r) * x.D + c);
          g[k] = make_float4(0.f + v.x, 0.f + v.y, 0.f + v.z, 0.f + v.w);  // a run's sum starts at 0
        }
      }
#pragma unroll
      for (int k = 0; k < kBwdUnroll; ++k)
        if (aa[k]) {
          float* stp = x.fstate ? x.fstate + (w[k] - x.fast) : nullptr;
          apply_unit(w[k], stp, g[k], x.o);
        }
    }
    if (act) x.dirty[s] = 1;
  }
}

// Per-unique gradient of the pooled forward: group the occurrences by unique row
// (stable radix sort of `inverse`), stream the sorted occurrences accumulating
// coef_j * grad_out[bag(j)], fix up the runs cut by chunk edges. Leaves x ready for
// k_bwd_apply (x.gu = per-unique sums, in `gu_out` when given, else in scratch).
static int segment_grads(void** scratch, size_t* scratch_bytes, const int32_t* inv, int64_t u, int64_t n,
                         const void* offsets, int off_bytes, int64_t nbags, int include_last, const float* psw,
                         int mode, const float* grad, int D, float* gu_out, BwdArgs& x, bool apply, cudaStream_t st,
                         void** zero_for = nullptr, size_t* zero_bytes = nullptr,
                         const int32_t* sort_hist = nullptr) {
  if (D % 4 || (reinterpret_cast<uintptr_t>(grad) & 15) || (reinterpret_cast<uintptr_t>(gu_out) & 15)) {
    set_error("backward needs dim %% 4 == 0 and 16-byte aligned gradient rows");
    return FC_ERR_BAD_ARG;
  }
  if ((size_t)kFixWarps * (D / 4) * sizeof(float4) > 220 * 1024) {
    set_error("backward supports rows up to %d floats (the carry fix-up's shared memory)",
              (int)(220 * 1024 / (kFixWarps * sizeof(float4)) * 4));
    return FC_ERR_BAD_ARG;
  }
  const int64_t nchunks = (n + kChunk - 1) / kChunk;
  const bool bags = offsets != nullptr;
  const size_t extra = (gu_out || apply ? 0 : align16((size_t)u * D * 4)) + align16(nchunks * 2 * (size_t)D * 4) +
                       2 * align16(nchunks * 2 * 4) + (bags ? 2 * align16(n * 4) : 0);
  // sort state left zero by the previous fused backward (no memset); this one's fix-up clears
  // it again. The state sits after the keys and order arrays, so its address moves with n:
  // it counts as zero only where the previous fix-up cleared it (same address, no regrowth)
  const size_t state = sort_state_bytes(n, key_bits_for(u));
  const bool fits = *scratch != nullptr && grouping_bytes(n) + extra <= *scratch_bytes;
  const void* sort_at = fits ? static_cast<const void*>(static_cast<char*>(*scratch) + 2 * align16(n * 4)) : nullptr;
  const bool zeroed = zero_for && *zero_for != nullptr && fits && *zero_for == sort_at && *zero_bytes >= state;
  Grouping g;
  int rc = build_grouping(scratch, scratch_bytes, inv, u, n, extra, g, st, zeroed, sort_hist);
  if (zero_for) {  // valid again only once the fix-up below is queued
    *zero_for = nullptr;
    *zero_bytes = 0;
  }
  if (rc) return rc;
  x.zero = nullptr;
  x.zero_words = 0;
  char* p = g.rest;
  x.gu = gu_out;
  if (!gu_out && !apply) {
    x.gu = reinterpret_cast<float*>(p);
    p += align16((size_t)u * D * 4);
  }
  x.carry = reinterpret_cast<float*>(p);
  p += align16(nchunks * 2 * (size_t)D * 4);
  x.carry_key = reinterpret_cast<int32_t*>(p);
  p += align16(nchunks * 2 * 4);
  x.carry_flag = reinterpret_cast<int32_t*>(p);
  p += align16(nchunks * 2 * 4);
  x.bag_of = nullptr;
  x.coef = nullptr;
  x.psw = bags ? nullptr : psw;
  if (bags) {
    int32_t* bag_of = reinterpret_cast<int32_t*>(p);
    p += align16(n * 4);
    float* coef = reinterpret_cast<float*>(p);
    // occurrences outside every bag (include_last_offset with a short last offset) contribute 0
    FC_CUDA(cudaMemsetAsync(bag_of, 0, n * 4, st));
    FC_CUDA(cudaMemsetAsync(coef, 0, n * 4, st));
    const int gb = grid_for(nbags, kNT, kSMs * 8);
    if (off_bytes == 4)
      k_bag_coef<int32_t><<<gb, kNT, 0, st>>>((const int32_t*)offsets, nbags, n, include_last, psw, mode, bag_of, coef);
    else
      k_bag_coef<long long><<<gb, kNT, 0, st>>>((const long long*)offsets, nbags, n, include_last, psw, mode, bag_of,
                                               coef);
    x.bag_of = bag_of;
    x.coef = coef;
  }
  x.D = D;
  x.keys = g.keys;
  x.order = g.order;
  x.n = n;
  x.grad = grad;
  x.un = units_for(D);
  const int grid = grid_for(nchunks * 32, kNT, kSMs * 16);
  const size_t fix_smem = (size_t)kFixWarps * x.un.upr * sizeof(float4);
  const int fgrid = (int)std::min<int64_t>(nchunks, kSMs * 16);
  if (apply) {  // the optimizer step happens inside the reduction (no per-row gradient buffer)
    k_bwd_stream<true><<<grid, kNT, 0, st>>>(x);
    if (fix_smem > 48 * 1024) FC_CUDA(cudaFuncSetAttribute(k_bwd_fixup<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                           (int)fix_smem));
    if (zero_for) {
      x.zero = static_cast<uint32_t*>(g.sort_scr);
      x.zero_words = (int64_t)(state / 4);
    }
    k_bwd_fixup<true><<<fgrid, kNT, fix_smem, st>>>(x);
    if (zero_for) {
      FC_CUDA(cudaGetLastError());
      *zero_for = g.sort_scr;  // the address the fix-up cleared
      *zero_bytes = state;
    }
  } else {
    k_bwd_stream<false><<<grid, kNT, 0, st>>>(x);
    if (fix_smem > 48 * 1024) FC_CUDA(cudaFuncSetAttribute(k_bwd_fixup<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                           (int)fix_smem));
    k_bwd_fixup<false><<<fgrid, kNT, fix_smem, st>>>(x);
  }
  FC_CUDA(cudaGetLastError());
  return FC_OK;
}

__global__ void k_noop() {}

int launch_backward(fc_cache* h, const int32_t* uslots, const int32_t* inv, const int32_t* ucnt, int64_t u, int64_t n,
                    const void* offsets, int off_bytes, int64_t nbags, int include_last, const float* psw, int mode,
                    const float* grad, int optim, float lr, float eps, cudaStream_t st) {
  (void)ucnt;
  if (u <= 0 || n <= 0) return FC_OK;
  const int D = h->dim;
  if (optim == FC_OPT_ADAGRAD && (h->fast_state == nullptr || h->sw != D)) {
    set_error("Adagrad needs a cache created with state_width == dim");
    return FC_ERR_BAD_ARG;
  }
  BwdArgs x;
  x.uslots = uslots;
  x.fast = h->fast;
  x.fstate = optim == FC_OPT_ADAGRAD ? h->fast_state : nullptr;
  x.dirty = h->dirty;
  x.o = OptArgs{optim, lr, eps};
  static const bool fused = !std::getenv("FC_BWD_UNFUSED");
  static const bool direct_ok = !std::getenv("FC_BWD_NO_DIRECT");
  if (direct_ok && u == n && !offsets && !psw) {  // one gradient row per unique row: no grouping
    if (D % 4 || (reinterpret_cast<uintptr_t>(grad) & 15)) {
      set_error("backward needs dim %% 4 == 0 and 16-byte aligned gradient rows");
      return FC_ERR_BAD_ARG;
    }
    x.D = D;
    x.n = n;
    x.grad = grad;
    x.un = units_for(D);
    k_bwd_direct<<<grid_for(n, kNT, kSMs * 8), kNT, 0, st>>>(x, inv);
    FC_CUDA(cudaGetLastError());
    return FC_OK;
  }
  // the digit histograms of `inv`, when a pipeline index phase produced it (no histogram kernel)
  const int32_t* sort_hist = pipe_take_sort_hist(h, inv, n);
  // FC_DEBUG_NOOP_LAUNCHES=k: measurement only -- k empty kernels on the compute stream before a
  // pipelined backward, to price a kernel boundary inside the step (results unchanged)
  static const int noop_launches = [] {
    const char* e = std::getenv("FC_DEBUG_NOOP_LAUNCHES");
    return e ? std::max(0, std::atoi(e)) : 0;
  }();
  if (sort_hist)
    for (int k = 0; k < noop_launches; ++k) k_noop<<<1, 32, 0, st>>>();
  int rc = segment_grads(&h->scratch, &h->scratch_bytes, inv, u, n, offsets, off_bytes, nbags, include_last, psw, mode,
                         grad, D, nullptr, x, fused, st, &h->sort_zero_for, &h->sort_zero_bytes, sort_hist);
  if (rc || fused) return rc;
  k_bwd_apply<<<grid_for(u, kNT, kSMs * 8), kNT, 0, st>>>(x, u);  // the unfused variant: per-row sums, then apply
  FC_CUDA(cudaGetLastError());
  return FC_OK;
}

// Per-unique gradient rows without an optimizer step (the row-sharded exchange: a
// requester reduces its occurrences' gradients before sending them to the owners).
int launch_unique_grads(void** scratch, size_t* scratch_bytes, const int32_t* inv, int64_t u, int64_t n,
                        const void* offsets, int off_bytes, int64_t nbags, int include_last, const float* psw,
                        int mode, const float* grad, int D, float* gu, cudaStream_t st) {
  if (u <= 0 || n <= 0) return FC_OK;
  BwdArgs x;
  x.uslots = nullptr;
  x.fast = nullptr;
  x.fstate = nullptr;
  x.dirty = nullptr;
  return segment_grads(scratch, scratch_bytes, inv, u, n, offsets, off_bytes, nbags, include_last, psw, mode, grad, D,
                       gu, x, false, st);
}

}  // namespace fc
