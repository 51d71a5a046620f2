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

constexpr int kRsWarps = 8;
constexpr int kRsRounds = 8;
constexpr int kRsTile = kRsWarps * kRsRounds * 32;  // 2048 keys per tile

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

// ---------------------------------------------------------------- radix sort
// Digits of up to 9 bits (512 bins): keys below 2^18 (U <= 262,144 unique rows)
// sort in two passes. Each pass = tile histogram -> device-wide scan -> stable scatter.
constexpr int kRsMaxBins = 512;

__global__ void __launch_bounds__(kRsWarps * 32) k_rs_hist(const uint32_t* __restrict__ keys, int64_t n, int shift,
                                                           int bins, int32_t* hist, int ntiles) {
  __shared__ int h[kRsMaxBins];
  for (int d = threadIdx.x; d < bins; d += blockDim.x) h[d] = 0;
  __syncthreads();
  const int64_t base = (int64_t)blockIdx.x * kRsTile;
  for (int k = threadIdx.x; k < kRsTile; k += blockDim.x) {
    const int64_t i = base + k;
    if (i < n) atomicAdd(&h[(keys[i] >> shift) & (bins - 1)], 1);
  }
  __syncthreads();
  for (int d = threadIdx.x; d < bins; d += blockDim.x) hist[(int64_t)d * ntiles + blockIdx.x] = h[d];
}

__global__ void __launch_bounds__(kRsWarps * 32) k_rs_scatter(const uint32_t* __restrict__ kin,
                                                              const int32_t* __restrict__ vin,
                                                              uint32_t* __restrict__ kout, int32_t* __restrict__ vout,
                                                              int64_t n, int shift, int bins,
                                                              const int32_t* __restrict__ hist, int ntiles) {
  __shared__ int wc[kRsWarps][kRsMaxBins];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int d = lane; d < bins; d += 32) wc[w][d] = 0;
  __syncwarp();
  const int64_t base = (int64_t)blockIdx.x * kRsTile + (int64_t)w * kRsRounds * 32;
  const unsigned lt = (1u << lane) - 1u;
  uint32_t kk[kRsRounds];
  int32_t vv[kRsRounds];
  int dd[kRsRounds], loc[kRsRounds];
#pragma unroll
  for (int r = 0; r < kRsRounds; ++r) {
    const int64_t i = base + r * 32 + lane;
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
  for (int d = threadIdx.x; d < bins; d += blockDim.x) {  // warp order = input order
    int run = 0;
#pragma unroll
    for (int q = 0; q < kRsWarps; ++q) {
      const int t = wc[q][d];
      wc[q][d] = run;
      run += t;
    }
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < kRsRounds; ++r) {
    if (dd[r] < kRsMaxBins) {
      const int64_t pos = (int64_t)hist[(int64_t)dd[r] * ntiles + blockIdx.x] + wc[w][dd[r]] + loc[r];
      kout[pos] = kk[r];
      vout[pos] = vv[r];
    }
  }
}

size_t sort_scratch_bytes(int64_t n) {
  const int64_t ntiles = (n + kRsTile - 1) / kRsTile;
  return sizeof(int32_t) * (kRsMaxBins * ntiles + 1) + scan_scratch_bytes(kRsMaxBins * ntiles) +
         2 * n * sizeof(int32_t) + 64;
}

// Stable sort of (key, value) pairs by the low `key_bits` bits of the key.
// vals_in == NULL sorts the positions 0..n-1 (an argsort). Inputs are untouched.
int radix_sort_pairs(const uint32_t* keys_in, const int32_t* vals_in, uint32_t* keys_out, int32_t* vals_out,
                     int64_t n, int key_bits, void* scratch, cudaStream_t st) {
  if (n <= 0) return FC_OK;
  const int ntiles = (int)((n + kRsTile - 1) / kRsTile);
  char* p = static_cast<char*>(scratch);
  int32_t* hist = reinterpret_cast<int32_t*>(p);
  p += sizeof(int32_t) * ((int64_t)kRsMaxBins * ntiles + 1);
  void* scan_scr = p;
  p += scan_scratch_bytes(kRsMaxBins * ntiles);
  p = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(p) + 15) & ~uintptr_t(15));
  uint32_t* ktmp = reinterpret_cast<uint32_t*>(p);
  int32_t* vtmp = reinterpret_cast<int32_t*>(p + n * sizeof(int32_t));
  const int passes = std::max(1, (key_bits + 8) / 9);
  const int dbits = std::max(1, (key_bits + passes - 1) / passes);
  const int bins = 1 << dbits;
  const uint32_t* ks = keys_in;
  const int32_t* vs = vals_in;
  for (int pass = 0; pass < passes; ++pass) {
    const bool to_out = ((passes - 1 - pass) % 2) == 0;  // last pass lands in the outputs
    uint32_t* kd = to_out ? keys_out : ktmp;
    int32_t* vd = to_out ? vals_out : vtmp;
    k_rs_hist<<<ntiles, kRsWarps * 32, 0, st>>>(ks, n, pass * dbits, bins, hist, ntiles);
    int rc = exclusive_scan_i32(hist, hist, (int64_t)bins * ntiles, scan_scr, st);
    if (rc) return rc;
    k_rs_scatter<<<ntiles, kRsWarps * 32, 0, st>>>(ks, vs, kd, vd, n, pass * dbits, bins, hist, ntiles);
    ks = kd;
    vs = vd;
  }
  FC_CUDA(cudaGetLastError());
  return FC_OK;
}

}  // namespace fc
