// Stable LSD radix sort (32-bit keys, 32-bit values) and an exclusive int32 scan.
//
// Used by the backward / scatter_update path to group a batch's occurrences by
// unique row in batch order (the order np.add.at applies them,
// /root/reference/pkg/src/freqcache/cache_manager.py:437). One pass = per-tile
// digit histogram -> device-wide scan -> stable scatter. The stable in-tile rank
// is computed warp by warp with __match_any_sync: each warp walks its contiguous
// sub-tile in rounds of 32 keys, so (warp, round, lane) order equals input order.
#include <algorithm>

#include "fc_internal.cuh"

namespace fc {

constexpr int kRsWarps = 16;
constexpr int kRsRounds = 8;
constexpr int kRsTile = kRsWarps * kRsRounds * 32;  // 4096 keys per tile

// ---------------------------------------------------------------- exclusive scan
constexpr int kScanTile = kNT * 8;

__global__ void __launch_bounds__(kNT) k_scan_reduce(const int32_t* __restrict__ in, int64_t n, int64_t chunk,
                                                     int32_t* bsum) {
  __shared__ int sm[kNT / 32 + 1];
  const int64_t b0 = (int64_t)blockIdx.x * chunk, b1 = min(n, b0 + chunk);
  int s = 0;
  for (int64_t i = b0 + threadIdx.x; i < b1; i += kNT) s += in[i];
  s = block_sum<kNT>(s, sm);
  if (threadIdx.x == 0) bsum[blockIdx.x] = s;
}

__global__ void __launch_bounds__(1024) k_scan_top(int32_t* bsum, int nb) {
  __shared__ int sm[1024 / 32 + 1];
  const int per = (nb + 1023) / 1024, beg = threadIdx.x * per;
  int s = 0;
  for (int k = 0; k < per; ++k)
    if (beg + k < nb) s += bsum[beg + k];
  int tot;
  int off = block_excl_scan<1024>(s, sm, tot);
  for (int k = 0; k < per; ++k)
    if (beg + k < nb) {
      const int v = bsum[beg + k];
      bsum[beg + k] = off;
      off += v;
    }
  if (threadIdx.x == 0) bsum[nb] = tot;
}

// out[i] = sum(in[0..i)), out[n] = total; in == out allowed
__global__ void __launch_bounds__(kNT) k_scan_apply(const int32_t* in, int32_t* out, int64_t n, int64_t chunk,
                                                    const int32_t* bsum, int nb) {
  __shared__ int sm[kNT / 32 + 1];
  const int64_t b0 = (int64_t)blockIdx.x * chunk, b1 = min(n, b0 + chunk);
  int run = bsum[blockIdx.x];
  for (int64_t t0 = b0; t0 < b1; t0 += kNT) {
    const int64_t i = t0 + threadIdx.x;
    const int v = i < b1 ? in[i] : 0;
    int tot;
    const int e = block_excl_scan<kNT>(v, sm, tot);
    if (i < b1) out[i] = run + e;
    run += tot;
  }
  if (blockIdx.x == nb - 1 && threadIdx.x == 0) out[n] = bsum[nb];
}

size_t scan_scratch_bytes(int64_t) { return sizeof(int32_t) * (kMaxScanBlocks + 1); }

int exclusive_scan_i32(const int32_t* in, int32_t* out, int64_t n, void* scratch, cudaStream_t st) {
  int32_t* bsum = static_cast<int32_t*>(scratch);
  const int nb = grid_for(n, kScanTile, kMaxScanBlocks);
  const int64_t chunk = std::max<int64_t>(1, (n + nb - 1) / nb);
  k_scan_reduce<<<nb, kNT, 0, st>>>(in, n, chunk, bsum);
  k_scan_top<<<1, 1024, 0, st>>>(bsum, nb);
  k_scan_apply<<<nb, kNT, 0, st>>>(in, out, n, chunk, bsum, nb);
  FC_CUDA(cudaGetLastError());
  return FC_OK;
}

// ---------------------------------------------------------------- radix sort (one sweep per pass)
// Digits of up to 9 bits (512 bins): keys below 2^18 (U <= 262,144 unique rows) sort
// in two passes. Launches: one global histogram for every pass, then one kernel per
// pass that ranks a tile of keys, finds the tile's per-digit offset by decoupled
// look-back over the preceding tiles (tiles are claimed in order from an atomic
// counter, so a predecessor always makes progress), and scatters. Stable: within a
// tile the rank follows (warp, round, lane) = input order, across tiles tile order.
constexpr int kRsMaxBins = 512;
constexpr uint32_t kOsAgg = 1u << 30;     // status: tile's own count published
constexpr uint32_t kOsPrefix = 2u << 30;  // status: inclusive prefix published
constexpr uint32_t kOsMask = (1u << 30) - 1u;
constexpr int kOsMaxPasses = 4;

__global__ void __launch_bounds__(kNT) k_os_hist(const uint32_t* __restrict__ keys, int64_t n, int passes, int dbits,
                                                 int32_t* ghist) {
  __shared__ int h[kOsMaxPasses * kRsMaxBins];
  const int bins = 1 << dbits;
  for (int d = threadIdx.x; d < passes * bins; d += kNT) h[d] = 0;
  __syncthreads();
  for (int64_t i = (int64_t)blockIdx.x * kNT + threadIdx.x; i < n; i += (int64_t)gridDim.x * kNT) {
    const uint32_t k = keys[i];
    for (int p = 0; p < passes; ++p) atomicAdd(&h[p * bins + ((k >> (p * dbits)) & (bins - 1))], 1);
  }
  __syncthreads();
  for (int d = threadIdx.x; d < passes * bins; d += kNT)
    if (h[d]) atomicAdd(&ghist[d], h[d]);
}

__device__ __forceinline__ uint32_t ld_status(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_status(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__global__ void __launch_bounds__(kRsWarps * 32) k_os_scatter(const uint32_t* __restrict__ kin,
                                                              const int32_t* __restrict__ vin,
                                                              uint32_t* __restrict__ kout, int32_t* __restrict__ vout,
                                                              int64_t n, int shift, int bins,
                                                              const int32_t* __restrict__ ghist_pass,
                                                              uint32_t* status, int32_t* tile_ctr) {
  __shared__ int wc[kRsWarps][kRsMaxBins];
  __shared__ int base[kRsMaxBins];  // global digit start + exclusive tile prefix
  __shared__ int s_tile;
  __shared__ int sm[kRsWarps + 1];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (threadIdx.x == 0) s_tile = atomicAdd(tile_ctr, 1);
  for (int d = lane; d < bins; d += 32) wc[w][d] = 0;
  __syncthreads();
  const int tile = s_tile;
  const int64_t t0 = (int64_t)tile * kRsTile + (int64_t)w * kRsRounds * 32;
  const unsigned lt = (1u << lane) - 1u;
  uint32_t kk[kRsRounds];
  int32_t vv[kRsRounds];
  int dd[kRsRounds], loc[kRsRounds];
#pragma unroll
  for (int r = 0; r < kRsRounds; ++r) {
    const int64_t i = t0 + r * 32 + lane;
    const bool valid = i < n;
    kk[r] = valid ? kin[i] : 0u;
    vv[r] = valid ? (vin ? vin[i] : (int32_t)i) : 0;  // vin == NULL: values are the input positions
    const int d = valid ? (int)((kk[r] >> shift) & (bins - 1)) : kRsMaxBins;
    dd[r] = d;
    const unsigned peers = __match_any_sync(FC_FULL, d);
    int before = 0;
    if (valid) before = wc[w][d];
    loc[r] = before + __popc(peers & lt);
    __syncwarp();
    if (valid && lane == __ffs(peers) - 1) wc[w][d] += __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  // global digit starts (exclusive scan of the pass histogram, bins <= 512 = 2 per thread)
  {
    const int d0 = 2 * threadIdx.x;
    const int a = d0 < bins ? ghist_pass[d0] : 0, b = d0 + 1 < bins ? ghist_pass[d0 + 1] : 0;
    int tot;
    const int e = block_excl_scan<kRsWarps * 32>(a + b, sm, tot);
    if (d0 < bins) base[d0] = e;
    if (d0 + 1 < bins) base[d0 + 1] = e + a;
  }
  __syncthreads();
  // publish every digit's tile count first, then look back: a successor never waits on
  // this tile's look-back of another digit
  constexpr int kPer = kRsMaxBins / (kRsWarps * 32);
  int cnts[kPer];
#pragma unroll
  for (int q = 0; q < kPer; ++q) {
    const int d = threadIdx.x + q * kRsWarps * 32;
    cnts[q] = 0;
    if (d >= bins) continue;
    int cnt = 0;  // tile count of digit d; warp order = input order
#pragma unroll
    for (int wq = 0; wq < kRsWarps; ++wq) {
      const int t = wc[wq][d];
      wc[wq][d] = cnt;
      cnt += t;
    }
    cnts[q] = cnt;
    st_status(status + (int64_t)tile * bins + d, (tile == 0 ? kOsPrefix : kOsAgg) | (uint32_t)cnt);
  }
#pragma unroll
  for (int q = 0; q < kPer; ++q) {
    const int d = threadIdx.x + q * kRsWarps * 32;
    if (d >= bins || tile == 0) continue;
    // decoupled look-back, kLb predecessors' statuses loaded at once (independent loads)
    constexpr int kLb = 8;
    int excl = 0;
    bool done = false;
    for (int t0 = tile - 1; t0 >= 0 && !done; t0 -= kLb) {
      uint32_t v[kLb];
#pragma unroll
      for (int j = 0; j < kLb; ++j) v[j] = t0 - j >= 0 ? ld_status(status + (int64_t)(t0 - j) * bins + d) : 0u;
#pragma unroll
      for (int j = 0; j < kLb; ++j) {
        if (done || t0 - j < 0) continue;
        uint32_t x = v[j];
        while ((x & ~kOsMask) == 0u) x = ld_status(status + (int64_t)(t0 - j) * bins + d);  // not yet published
        excl += (int)(x & kOsMask);
        if (x & kOsPrefix) done = true;
      }
    }
    st_status(status + (int64_t)tile * bins + d, kOsPrefix | (uint32_t)(excl + cnts[q]));
    base[d] += excl;
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < kRsRounds; ++r) {
    if (dd[r] < kRsMaxBins) {
      const int64_t pos = (int64_t)base[dd[r]] + wc[w][dd[r]] + loc[r];
      if (pos < n) {  // always, unless a precomputed histogram did not match the keys
        kout[pos] = kk[r];
        vout[pos] = vv[r];
      }
    }
  }
}

size_t sort_scratch_bytes(int64_t n) {
  const int64_t ntiles = (n + kRsTile - 1) / kRsTile;
  return sizeof(int32_t) * (kOsMaxPasses * kRsMaxBins + kOsMaxPasses + 4) +
         sizeof(uint32_t) * (size_t)kOsMaxPasses * kRsMaxBins * ntiles + 2 * n * sizeof(int32_t) + 64;
}

// Bytes at the head of the scratch (histograms, tile counters, look-back status words)
// that must be zero when a sort of n keys of key_bits bits starts.
size_t sort_state_bytes(int64_t n, int key_bits) {
  const int64_t ntiles = (n + kRsTile - 1) / kRsTile;
  const int passes = std::max(1, (key_bits + 8) / 9);
  const int bins = 1 << std::max(1, (key_bits + passes - 1) / passes);
  return sizeof(int32_t) * (kOsMaxPasses * kRsMaxBins + kOsMaxPasses + 4) +
         sizeof(uint32_t) * (size_t)passes * bins * ntiles;
}

// Stable sort of (key, value) pairs by the low `key_bits` bits of the key.
// vals_in == NULL sorts the positions 0..n-1 (an argsort). Inputs are untouched.
// state_zeroed: the caller guarantees the first sort_state_bytes(n, key_bits) of the
// scratch are already zero (a previous kernel cleared them), so no memset is queued.
// ghist_pre: the digit histograms of keys_in, already computed ([passes][bins], the layout
// k_os_hist writes; the prefetch pipeline's index phase makes them for the backward's sort)
int radix_sort_pairs(const uint32_t* keys_in, const int32_t* vals_in, uint32_t* keys_out, int32_t* vals_out,
                     int64_t n, int key_bits, void* scratch, cudaStream_t st, bool state_zeroed,
                     const int32_t* ghist_pre) {
  if (n <= 0) return FC_OK;
  if (n > (int64_t)kOsMask) {
    set_error("radix sort of %lld keys exceeds the 30-bit tile counters", (long long)n);
    return FC_ERR_BAD_ARG;
  }
  const int ntiles = (int)((n + kRsTile - 1) / kRsTile);
  const int passes = std::max(1, (key_bits + 8) / 9);
  if (passes > kOsMaxPasses) return FC_ERR_BAD_ARG;
  const int dbits = std::max(1, (key_bits + passes - 1) / passes);
  const int bins = 1 << dbits;
  // scratch: [ghist passes*bins][tile counters passes] | status passes*ntiles*bins | ktmp | vtmp
  char* p = static_cast<char*>(scratch);
  int32_t* ghist = reinterpret_cast<int32_t*>(p);
  int32_t* tctr = ghist + kOsMaxPasses * kRsMaxBins;
  const size_t head = sizeof(int32_t) * (kOsMaxPasses * kRsMaxBins + kOsMaxPasses + 4);
  uint32_t* status = reinterpret_cast<uint32_t*>(p + head);
  const size_t status_bytes = sizeof(uint32_t) * (size_t)passes * bins * ntiles;
  p += head + status_bytes;
  p = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(p) + 15) & ~uintptr_t(15));
  uint32_t* ktmp = reinterpret_cast<uint32_t*>(p);
  int32_t* vtmp = reinterpret_cast<int32_t*>(p + n * sizeof(int32_t));
  if (!state_zeroed) FC_CUDA(cudaMemsetAsync(scratch, 0, head + status_bytes, st));  // histograms, counters, status
  if (ghist_pre) ghist = const_cast<int32_t*>(ghist_pre);  // read only below
  else k_os_hist<<<grid_for(n, kNT * 8, kSMs * 4), kNT, 0, st>>>(keys_in, n, passes, dbits, ghist);
  const uint32_t* ks = keys_in;
  const int32_t* vs = vals_in;
  for (int pass = 0; pass < passes; ++pass) {
    const bool to_out = ((passes - 1 - pass) % 2) == 0;  // last pass lands in the outputs
    uint32_t* kd = to_out ? keys_out : ktmp;
    int32_t* vd = to_out ? vals_out : vtmp;
    k_os_scatter<<<ntiles, kRsWarps * 32, 0, st>>>(ks, vs, kd, vd, n, pass * dbits, bins, ghist + pass * bins,
                                                   status + (size_t)pass * bins * ntiles, tctr + pass);
    ks = kd;
    vs = vd;
  }
  FC_CUDA(cudaGetLastError());
  return FC_OK;
}

}  // namespace fc
