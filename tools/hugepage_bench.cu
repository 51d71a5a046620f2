// Slow-tier page size experiment: does backing the pinned slow tier with 2 MB
// transparent huge pages (posix_memalign + madvise(MADV_HUGEPAGE) + cudaHostRegister)
// speed up (a) the host-thread write-back scatter and (b) SM zero-copy row gathers,
// compared with cudaHostAlloc'd (4 KB pages) memory?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -Xcompiler -fopenmp -o hp tools/hugepage_bench.cu
#include <sys/mman.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <thread>
#include <vector>

#include <cuda_runtime.h>
#include <emmintrin.h>

#define CK(x)                                                             \
  do {                                                                    \
    cudaError_t e = (x);                                                  \
    if (e != cudaSuccess) {                                               \
      printf("%s: %s (line %d)\n", #x, cudaGetErrorString(e), __LINE__); \
      exit(1);                                                            \
    }                                                                     \
  } while (0)

__global__ void zc_gather(const float4* __restrict__ host, float4* __restrict__ dev, const int* __restrict__ idx,
                          int nrows, int upr) {
  const int lane = threadIdx.x & 31;
  const long warp = (blockIdx.x * (long)blockDim.x + threadIdx.x) >> 5;
  const long nw = (gridDim.x * (long)blockDim.x) >> 5;
  for (long base = warp * 32; base < nrows; base += nw * 32) {
    const long j = base + lane;
    const long src = j < nrows ? (long)idx[j] : 0;
    for (int u0 = 0; u0 < 32 * upr; u0 += 128) {
      float4 v[4];
      long d[4];
      bool a[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int u = u0 + q * 32 + lane;
        const int rr = u / upr;
        const int c = u - rr * upr;
        const long s = __shfl_sync(0xffffffffu, src, rr);
        a[q] = base + rr < nrows;
        d[q] = (base + rr) * upr + c;
        if (a[q]) v[q] = host[s * upr + c];
      }
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (a[q]) dev[d[q]] = v[q];
    }
  }
}

static double scatter(float* table, const float* stage, const std::vector<int>& idx, int threads, bool gather) {
  const int rows = (int)idx.size();
  auto t0 = std::chrono::steady_clock::now();
  std::vector<std::thread> th;
  for (int t = 0; t < threads; ++t)
    th.emplace_back([&, t] {
      for (int i = t; i < rows; i += threads) {
        float* tr = table + (long)idx[i] * 128;
        const float* sr = stage + (long)i * 128;
        if (gather) {
          std::memcpy(const_cast<float*>(sr), tr, 512);
        } else {
          __m128i* d = reinterpret_cast<__m128i*>(tr);
          const __m128i* s = reinterpret_cast<const __m128i*>(sr);
          for (int k = 0; k < 32; ++k) _mm_stream_si128(d + k, _mm_load_si128(s + k));
        }
      }
      _mm_sfence();
    });
  for (auto& x : th) x.join();
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
}

int main() {
  const long table_rows = 33762577, bytes = table_rows * 512;
  const int rows = 67438;
  std::vector<int> idx(rows);
  std::mt19937_64 g(7);
  for (int i = 0; i < rows; ++i) idx[i] = (int)(g() % table_rows);
  std::sort(idx.begin(), idx.end());
  int* didx;
  CK(cudaMalloc(&didx, rows * 4));
  CK(cudaMemcpy(didx, idx.data(), rows * 4, cudaMemcpyHostToDevice));
  float4* dst;
  CK(cudaMalloc(&dst, (long)rows * 512));
  float* stage;
  CK(cudaHostAlloc(&stage, (long)rows * 512, cudaHostAllocDefault));
  memset(stage, 1, (long)rows * 512);

  FILE* f = fopen("/sys/kernel/mm/transparent_hugepage/enabled", "r");
  char buf[256] = "?";
  if (f) {
    if (!fgets(buf, sizeof buf, f)) buf[0] = 0;
    fclose(f);
  }
  printf("THP: %s", buf);

  for (int variant = 0; variant < 2; ++variant) {
    float* table = nullptr;
    auto t0 = std::chrono::steady_clock::now();
    if (variant == 0) {
      CK(cudaHostAlloc((void**)&table, bytes, cudaHostAllocMapped | cudaHostAllocPortable));
    } else {
      if (posix_memalign((void**)&table, 1 << 21, bytes)) return 1;
      madvise(table, bytes, MADV_HUGEPAGE);
      memset(table, 0, bytes);
      CK(cudaHostRegister(table, bytes, cudaHostRegisterMapped | cudaHostRegisterPortable));
    }
    const double alloc_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    if (variant == 0) memset(table, 0, bytes);
    float4* tdev;
    CK(cudaHostGetDevicePointer((void**)&tdev, table, 0));
    printf("== %s (alloc %.0f ms)\n", variant ? "THP + cudaHostRegister" : "cudaHostAlloc", alloc_ms);
    for (int th : {4, 8, 14}) {
      double best_s = 1e9, best_g = 1e9;
      for (int r = 0; r < 4; ++r) {
        best_s = std::min(best_s, scatter(table, stage, idx, th, false));
        best_g = std::min(best_g, scatter(table, stage, idx, th, true));
      }
      printf("  host %2d threads: scatter %.3f ms (%.1f GB/s), gather %.3f ms (%.1f GB/s)\n", th, best_s,
             rows * 512.0 / best_s / 1e6, best_g, rows * 512.0 / best_g / 1e6);
    }
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float best = 1e9;
    for (int r = 0; r < 6; ++r) {
      cudaEventRecord(a);
      zc_gather<<<148, 256>>>(tdev, dst, didx, rows, 32);
      cudaEventRecord(b);
      CK(cudaEventSynchronize(b));
      float t;
      cudaEventElapsedTime(&t, a, b);
      best = std::min(best, t);
    }
    printf("  zero-copy gather (148x256): %.3f ms (%.1f GB/s)\n", best, rows * 512.0 / best / 1e6);
    if (variant == 0) cudaFreeHost(table);
    else {
      cudaHostUnregister(table);
      free(table);
    }
  }
  return 0;
}
