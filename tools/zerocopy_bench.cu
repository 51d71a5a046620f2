// Host-link microbenchmark: what a kernel can pull from / push to pinned mapped
// host memory over PCIe, for contiguous and random 512-byte rows, one direction
// and both at once, versus cudaMemcpyAsync. Sets the ceiling for k_transfer_rows.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o zc tools/zerocopy_bench.cu
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1);} } while (0)

template <int K>
__global__ void rows_read(const float4* __restrict__ host, float4* __restrict__ dev, const int* __restrict__ idx,
                          int nrows, int upr) {
  const int lane = threadIdx.x & 31;
  const long warp = (blockIdx.x * (long)blockDim.x + threadIdx.x) >> 5;
  const long nw = (gridDim.x * (long)blockDim.x) >> 5;
  for (long r0 = warp * K; r0 < nrows; r0 += nw * K) {
    float4 v[K];
#pragma unroll
    for (int k = 0; k < K; ++k)
      if (r0 + k < nrows) v[k] = host[(long)idx[r0 + k] * upr + lane];
#pragma unroll
    for (int k = 0; k < K; ++k)
      if (r0 + k < nrows) dev[(r0 + k) * upr + lane] = v[k];
  }
}

template <int K>
__global__ void rows_write(float4* __restrict__ host, const float4* __restrict__ dev, const int* __restrict__ idx,
                           int nrows, int upr) {
  const int lane = threadIdx.x & 31;
  const long warp = (blockIdx.x * (long)blockDim.x + threadIdx.x) >> 5;
  const long nw = (gridDim.x * (long)blockDim.x) >> 5;
  for (long r0 = warp * K; r0 < nrows; r0 += nw * K) {
    float4 v[K];
#pragma unroll
    for (int k = 0; k < K; ++k)
      if (r0 + k < nrows) v[k] = dev[(r0 + k) * upr + lane];
#pragma unroll
    for (int k = 0; k < K; ++k)
      if (r0 + k < nrows) host[(long)idx[r0 + k] * upr + lane] = v[k];
  }
}

// one kernel, roles interleaved at warp granularity: even warps read host rows,
// odd warps write host rows, so both link directions are busy at once
template <int K>
__global__ void rows_both(const float4* __restrict__ hsrc, float4* __restrict__ hdst, float4* __restrict__ d1,
                          const float4* __restrict__ d2, const int* __restrict__ ir, const int* __restrict__ iw,
                          int nrows, int upr, int mod) {
  const int lane = threadIdx.x & 31;
  const long warp = (blockIdx.x * (long)blockDim.x + threadIdx.x) >> 5;
  const long nw = (gridDim.x * (long)blockDim.x) >> 5;
  const bool rd = (warp % mod) == 0;
  const long my = warp / mod * (mod - 1) + (rd ? 0 : (warp % mod) - 1);
  const long nmy = rd ? nw / mod : nw - nw / mod;
  const long w0 = rd ? warp / mod : my;
  for (long r0 = w0 * K; r0 < nrows; r0 += nmy * K) {
    float4 v[K];
    if (rd) {
#pragma unroll
      for (int k = 0; k < K; ++k) if (r0 + k < nrows) v[k] = hsrc[(long)ir[r0 + k] * upr + lane];
#pragma unroll
      for (int k = 0; k < K; ++k) if (r0 + k < nrows) d1[(r0 + k) * upr + lane] = v[k];
    } else {
#pragma unroll
      for (int k = 0; k < K; ++k) if (r0 + k < nrows) v[k] = d2[(r0 + k) * upr + lane];
#pragma unroll
      for (int k = 0; k < K; ++k) if (r0 + k < nrows) hdst[(long)iw[r0 + k] * upr + lane] = v[k];
    }
  }
}

// each warp moves one host->HBM row and one HBM->host row per iteration (both
// directions issued back to back by the same warp)
template <int K>
__global__ void rows_pair(const float4* __restrict__ hsrc, float4* __restrict__ hdst, float4* __restrict__ d1,
                          const float4* __restrict__ d2, const int* __restrict__ ir, const int* __restrict__ iw,
                          int nrows, int upr) {
  const int lane = threadIdx.x & 31;
  const long warp = (blockIdx.x * (long)blockDim.x + threadIdx.x) >> 5;
  const long nw = (gridDim.x * (long)blockDim.x) >> 5;
  for (long r0 = warp * K; r0 < nrows; r0 += nw * K) {
    float4 a[K], b[K];
#pragma unroll
    for (int k = 0; k < K; ++k) if (r0 + k < nrows) {
      a[k] = hsrc[(long)ir[r0 + k] * upr + lane];
      b[k] = d2[(r0 + k) * upr + lane];
    }
#pragma unroll
    for (int k = 0; k < K; ++k) if (r0 + k < nrows) {
      d1[(r0 + k) * upr + lane] = a[k];
      hdst[(long)iw[r0 + k] * upr + lane] = b[k];
    }
  }
}

int main() {
  const long slow_rows = 8l << 20;  // 8M rows x 512 B = 4 GiB pinned
  const int upr = 32;               // 128 floats
  const int n = 65536;              // rows per transfer (~ a cfg2 batch)
  float4* host;
  CK(cudaHostAlloc(&host, slow_rows * upr * 16, cudaHostAllocMapped));
  float4 *dev, *dev2;
  CK(cudaMalloc(&dev, (long)n * upr * 16));
  CK(cudaMalloc(&dev2, (long)n * upr * 16));
  std::vector<int> hi(n), hs(n);
  srand(1);
  for (int i = 0; i < n; ++i) { hi[i] = (int)(((long)rand() * 7919 + i) % slow_rows); hs[i] = i; }
  std::vector<int> hr = hi;
  for (int i = 0; i < n; ++i) hr[i] = (int)(((long)rand() * 104729 + 3 * i) % slow_rows);
  std::vector<int> hsa = hi, hsb = hr;
  std::sort(hsa.begin(), hsa.end());
  std::sort(hsb.begin(), hsb.end());
  int *idx_rand, *idx_seq, *idx_rand2, *idx_sa, *idx_sb;
  CK(cudaMalloc(&idx_sa, n * 4)); CK(cudaMalloc(&idx_sb, n * 4));
  CK(cudaMemcpy(idx_sa, hsa.data(), n * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(idx_sb, hsb.data(), n * 4, cudaMemcpyHostToDevice));
  CK(cudaMalloc(&idx_rand, n * 4)); CK(cudaMalloc(&idx_seq, n * 4)); CK(cudaMalloc(&idx_rand2, n * 4));
  CK(cudaMemcpy(idx_rand, hi.data(), n * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(idx_rand2, hr.data(), n * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(idx_seq, hs.data(), n * 4, cudaMemcpyHostToDevice));
  cudaStream_t s1, s2;
  CK(cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
  const double bytes = (double)n * upr * 16;
  int sms = 148;
  auto time_it = [&](auto fn, const char* name, double mult) {
    for (int w = 0; w < 3; ++w) fn();
    CK(cudaDeviceSynchronize());
    float best = 1e9;
    for (int r = 0; r < 10; ++r) {
      CK(cudaEventRecord(a, 0));
      fn();
      CK(cudaEventRecord(b, 0));
      CK(cudaEventSynchronize(b));
      float ms; CK(cudaEventElapsedTime(&ms, a, b));
      if (ms < best) best = ms;
    }
    printf("%-48s %8.3f ms  %7.2f GB/s\n", name, best, mult * bytes / best / 1e6);
  };
  for (int bps : {2, 4, 8, 16}) {
    for (int K : {1, 4}) {
      char nm[128];
      int grid = sms * bps;
      snprintf(nm, sizeof nm, "read rand   grid=%d K=%d", grid, K);
      if (K == 1) time_it([&] { rows_read<1><<<grid, 256>>>(host, dev, idx_rand, n, upr); }, nm, 1);
      else time_it([&] { rows_read<4><<<grid, 256>>>(host, dev, idx_rand, n, upr); }, nm, 1);
      snprintf(nm, sizeof nm, "write rand  grid=%d K=%d", grid, K);
      if (K == 1) time_it([&] { rows_write<1><<<grid, 256>>>(host, dev, idx_rand2, n, upr); }, nm, 1);
      else time_it([&] { rows_write<4><<<grid, 256>>>(host, dev, idx_rand2, n, upr); }, nm, 1);
    }
  }
  cudaEvent_t j;
  CK(cudaEventCreate(&j));
  auto both = [&](int grid) {
    CK(cudaEventRecord(j, 0));
    CK(cudaStreamWaitEvent(s1, j)); CK(cudaStreamWaitEvent(s2, j));
    rows_read<4><<<grid, 256, 0, s1>>>(host, dev, idx_rand, n, upr);
    rows_write<4><<<grid, 256, 0, s2>>>(host, dev2, idx_rand2, n, upr);
    CK(cudaEventRecord(j, s1)); CK(cudaStreamWaitEvent(0, j));
    CK(cudaEventRecord(j, s2)); CK(cudaStreamWaitEvent(0, j));
  };
  time_it([&] { both(148 * 4); }, "read+write rand concurrent grid=592 each", 2);
  time_it([&] { both(148 * 8); }, "read+write rand concurrent grid=1184 each", 2);
  time_it([&] { rows_read<4><<<592, 256>>>(host, dev, idx_seq, n, upr); }, "read seq   grid=592 K=4", 1);
  time_it([&] { rows_write<4><<<592, 256>>>(host, dev, idx_seq, n, upr); }, "write seq  grid=592 K=4", 1);
  time_it([&] { CK(cudaMemcpyAsync(dev, host, (size_t)bytes, cudaMemcpyHostToDevice, 0)); }, "memcpy H2D contiguous", 1);
  time_it([&] { CK(cudaMemcpyAsync(host, dev, (size_t)bytes, cudaMemcpyDeviceToHost, 0)); }, "memcpy D2H contiguous", 1);
  time_it([&] { rows_both<4><<<592, 256>>>(host, host, dev, dev2, idx_rand, idx_rand2, n, upr, 2); }, "both interleaved warps grid=592 mod2", 2);
  time_it([&] { rows_both<4><<<1184, 256>>>(host, host, dev, dev2, idx_rand, idx_rand2, n, upr, 2); }, "both interleaved warps grid=1184 mod2", 2);
  time_it([&] { rows_both<1><<<1184, 256>>>(host, host, dev, dev2, idx_rand, idx_rand2, n, upr, 2); }, "both interleaved warps grid=1184 K=1", 2);
  time_it([&] { rows_both<8><<<296, 256>>>(host, host, dev, dev2, idx_rand, idx_rand2, n, upr, 2); }, "both interleaved warps grid=296 K=8", 2);
  time_it([&] { rows_read<4><<<1184, 256>>>(host, dev, idx_sa, n, upr); }, "read sorted-rand grid=1184 K=4", 1);
  time_it([&] { rows_write<4><<<1184, 256>>>(host, dev, idx_sb, n, upr); }, "write sorted-rand grid=1184 K=4", 1);
  time_it([&] { rows_both<4><<<1184, 256>>>(host, host, dev, dev2, idx_sa, idx_sb, n, upr, 2); }, "both interleaved sorted grid=1184", 2);
  for (int g : {296, 592, 1184, 2368}) {
    char nm[96];
    snprintf(nm, sizeof nm, "pair rand grid=%d K=1", g);
    time_it([&] { rows_pair<1><<<g, 256>>>(host, host, dev, dev2, idx_rand, idx_rand2, n, upr); }, nm, 2);
    snprintf(nm, sizeof nm, "pair sorted grid=%d K=1", g);
    time_it([&] { rows_pair<1><<<g, 256>>>(host, host, dev, dev2, idx_sa, idx_sb, n, upr); }, nm, 2);
    snprintf(nm, sizeof nm, "pair sorted grid=%d K=2", g);
    time_it([&] { rows_pair<2><<<g, 256>>>(host, host, dev, dev2, idx_sa, idx_sb, n, upr); }, nm, 2);
  }
  return 0;
}
