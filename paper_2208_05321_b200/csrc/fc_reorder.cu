// Frequency reorder on the GPU: scan_frequencies + build_reorder
// (/root/reference/pkg/src/freqcache/freq_stats.py:97-111, 136-148).
//
//   counts  = bincount(trace, minlength=num_ids)            k_count_ids (block hash aggregation)
//   id_of   = argsort(-counts, kind="stable")               stable LSD radix sort of
//             key = max_count - count over the ids 0..num_ids-1 (ties keep ascending id)
//   rank_of[id_of] = arange(num_ids)                        k_rank_of
//
// Offline, once per run (the reference scans the whole trace before training,
// simulator.py:363-364); on the host this takes seconds at the Criteo scale.
#include <algorithm>
#include <climits>

#include "fc_rowutil.cuh"

namespace fc {

constexpr int kCountTile = 4096;  // ids per block iteration
constexpr int kCountHash = 4096;  // shared-memory open-addressing slots

// Per-block aggregation in a shared hash table, then one global 64-bit add per
// distinct id of the tile: Zipf head ids would otherwise serialise in L2 atomics.
template <typename IdT>
__global__ void __launch_bounds__(kNT) k_count_ids(const IdT* __restrict__ ids, int64_t n, int64_t num_ids,
                                                   unsigned long long* counts, long long* lohi) {
  __shared__ int hk[kCountHash];
  __shared__ int hc[kCountHash];
  const int lane = threadIdx.x & 31;
  for (int e = threadIdx.x; e < kCountHash; e += kNT) {
    hk[e] = -1;
    hc[e] = 0;
  }
  __syncthreads();
  for (int64_t tile = blockIdx.x; tile * kCountTile < n; tile += gridDim.x) {
    for (int k = 0; k < kCountTile / kNT; ++k) {
      const int64_t i = tile * kCountTile + k * kNT + threadIdx.x;
      const bool valid = i < n;
      const long long id = valid ? (long long)ids[i] : 0;
      const bool inr = valid && id >= 0 && id < num_ids;
      if (valid && !inr) {  // the reference names the smallest negative id, else the largest (freq_stats.py:82-90)
        if (id < 0) atomicMin(&lohi[0], id);
        else atomicMax(&lohi[1], id);
      }
      const int key = inr ? (int)id : -1;
      const unsigned peers = __match_any_sync(FC_FULL, key);
      if (inr && lane == __ffs(peers) - 1) {
        unsigned h = ((unsigned)key * 2654435761u) >> 20;
        while (true) {
          const int prev = atomicCAS(&hk[h], -1, key);
          if (prev == -1 || prev == key) {
            atomicAdd(&hc[h], __popc(peers));
            break;
          }
          h = (h + 1) & (kCountHash - 1);
        }
      }
    }
    __syncthreads();
    for (int e = threadIdx.x; e < kCountHash; e += kNT) {
      const int key = hk[e];
      if (key >= 0) {
        atomicAdd(&counts[key], (unsigned long long)hc[e]);
        hk[e] = -1;
        hc[e] = 0;
      }
    }
    __syncthreads();
  }
}

__global__ void k_max_count(const unsigned long long* __restrict__ counts, int64_t num_ids, unsigned long long* mx) {
  unsigned long long m = 0;
  for (int64_t i = (int64_t)blockIdx.x * kNT + threadIdx.x; i < num_ids; i += (int64_t)gridDim.x * kNT)
    m = max(m, counts[i]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(FC_FULL, m, o));
  if ((threadIdx.x & 31) == 0 && m) atomicMax(mx, m);
}

// descending count == ascending (max - count)
__global__ void k_count_keys(const unsigned long long* __restrict__ counts, int64_t num_ids,
                             const unsigned long long* __restrict__ mx, uint32_t* keys) {
  const unsigned long long m = *mx;
  for (int64_t i = (int64_t)blockIdx.x * kNT + threadIdx.x; i < num_ids; i += (int64_t)gridDim.x * kNT)
    keys[i] = (uint32_t)(m - counts[i]);
}

__global__ void k_rank_of(const int32_t* __restrict__ id_of, int64_t num_ids, int32_t* rank_of) {
  for (int64_t r = (int64_t)blockIdx.x * kNT + threadIdx.x; r < num_ids; r += (int64_t)gridDim.x * kNT)
    rank_of[id_of[r]] = (int32_t)r;
}

}  // namespace fc

using namespace fc;

extern "C" int fc_build_reorder(const void* ids, int32_t ids_bytes, int64_t n, int64_t num_ids, int64_t* counts_dev,
                                int32_t* id_of_dev, int32_t* rank_of_dev, int64_t* bad_id, void* stream) {
  if ((ids_bytes != 4 && ids_bytes != 8) || n < 0 || num_ids < 1 || num_ids > INT32_MAX - 64 || !counts_dev ||
      !id_of_dev || !rank_of_dev)
    return FC_ERR_BAD_ARG;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  unsigned long long* counts = reinterpret_cast<unsigned long long*>(counts_dev);
  // small device scratch: [0] max count, [1] smallest negative id, [2] largest id >= num_ids
  unsigned long long* small = nullptr;
  FC_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&small), 32, st));
  const long long init[3] = {0, LLONG_MAX, LLONG_MIN};
  FC_CUDA(cudaMemcpyAsync(small, init, 24, cudaMemcpyHostToDevice, st));
  FC_CUDA(cudaMemsetAsync(counts, 0, (size_t)num_ids * 8, st));
  long long* bad = reinterpret_cast<long long*>(small + 1);
  if (n > 0) {
    const int g = grid_for(n, kCountTile, kSMs * 4);
    if (ids_bytes == 8) k_count_ids<long long><<<g, kNT, 0, st>>>((const long long*)ids, n, num_ids, counts, bad);
    else k_count_ids<int><<<g, kNT, 0, st>>>((const int*)ids, n, num_ids, counts, bad);
  }
  k_max_count<<<grid_for(num_ids, kNT, kSMs * 8), kNT, 0, st>>>(counts, num_ids, small);
  long long host[3];
  FC_CUDA(cudaMemcpyAsync(host, small, 24, cudaMemcpyDeviceToHost, st));
  FC_CUDA(cudaStreamSynchronize(st));
  if (host[1] != LLONG_MAX || host[2] != LLONG_MIN) {  // freq_stats._check_id_range
    const long long b = host[1] != LLONG_MAX ? host[1] : host[2];
    if (bad_id) *bad_id = b;
    if (b < 0) set_error("id out of range: %lld < 0", b);
    else set_error("id out of range: %lld >= num_ids=%lld", b, (long long)num_ids);
    cudaFreeAsync(small, st);
    return FC_ERR_ID_OUT_OF_RANGE;
  }
  const unsigned long long mx = (unsigned long long)host[0];
  if (mx > 0xffffffffull) {
    set_error("a count above 2^32 does not fit the 32-bit sort key");
    cudaFreeAsync(small, st);
    return FC_ERR_BAD_ARG;
  }
  const int key_bits = std::max(1, key_bits_for((int64_t)mx + 1));
  // keys + sorted keys + sort scratch
  const size_t kb = align16((size_t)num_ids * 4);
  const size_t scr = sort_scratch_bytes(num_ids);
  char* buf = nullptr;
  FC_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&buf), 2 * kb + scr, st));
  uint32_t* keys = reinterpret_cast<uint32_t*>(buf);
  uint32_t* skeys = reinterpret_cast<uint32_t*>(buf + kb);
  const int gk = grid_for(num_ids, kNT, kSMs * 8);
  k_count_keys<<<gk, kNT, 0, st>>>(counts, num_ids, small, keys);
  int rc = radix_sort_pairs(keys, nullptr, skeys, id_of_dev, num_ids, key_bits, buf + 2 * kb, st);
  if (rc == FC_OK) {
    k_rank_of<<<gk, kNT, 0, st>>>(id_of_dev, num_ids, rank_of_dev);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) rc = cuda_fail(e, "fc_build_reorder");
  }
  cudaFreeAsync(buf, st);
  cudaFreeAsync(small, st);
  if (rc == FC_OK) FC_CUDA(cudaStreamSynchronize(st));
  return rc;
}
