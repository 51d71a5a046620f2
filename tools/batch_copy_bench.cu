// Copy-engine row gather/scatter between the pinned slow tier and HBM with
// cudaMemcpyBatchAsync (one descriptor per 512 B row), against the TMA staging it
// would replace: time alone, host submit cost, and next to an HBM-bound (H) and a
// latency-bound (L) kernel -- the interference that limits the prefetch pipeline
// (DESIGN.md 4a).
// argv[2] = "thp": the slow tier is 2 MB-aligned, madvise(MADV_HUGEPAGE) and
// cudaHostRegister'ed instead of cudaHostAlloc'ed (does a coarser host mapping cut the
// interference?). argv[3] = "quick": skip the batched-copy rows.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bcb tools/batch_copy_bench.cu -lcuda
#include <sys/mman.h>

#include <algorithm>
#include <chrono>
#include <cstring>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#include <cuda_runtime.h>

#define CK(x)                                                             \
  do {                                                                    \
    cudaError_t e = (x);                                                  \
    if (e != cudaSuccess) {                                               \
      printf("%s: %s (line %d)\n", #x, cudaGetErrorString(e), __LINE__); \
      exit(1);                                                            \
    }                                                                     \
  } while (0)

__global__ void hbm_copy(const float4* __restrict__ a, float4* __restrict__ b, long n) {
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) b[i] = a[i];
}

__global__ void dep_gather(const int* __restrict__ a, const int* __restrict__ b, const float4* __restrict__ rows,
                           float4* __restrict__ out, long n, int nrows) {
  const int lane = threadIdx.x & 31;
  const long warp = (blockIdx.x * (long)blockDim.x + threadIdx.x) >> 5;
  const long nw = (gridDim.x * (long)blockDim.x) >> 5;
  for (long j = warp; j < n; j += nw) {
    const int r = b[a[j] % nrows] % nrows;
    out[j * 32 + lane] = rows[(long)r * 32 + lane];
  }
}

// the TMA-free SM gather for reference (zero-copy loads)
__global__ void zc_gather(const float4* __restrict__ host, float4* __restrict__ dev, const int* __restrict__ idx,
                          int nrows) {
  const int lane = threadIdx.x & 31;
  const long warp = (blockIdx.x * (long)blockDim.x + threadIdx.x) >> 5;
  const long nw = (gridDim.x * (long)blockDim.x) >> 5;
  for (long r = warp; r < nrows; r += nw) dev[r * 32 + lane] = host[(long)idx[r] * 32 + lane];
}

struct Timer {
  cudaEvent_t a, b;
  Timer() {
    cudaEventCreate(&a);
    cudaEventCreate(&b);
  }
  float ms() {
    float t;
    cudaEventElapsedTime(&t, a, b);
    return t;
  }
};

int main(int argc, char** argv) {
  const long table_rows = argc > 1 ? atol(argv[1]) : 33762577;
  const int rows = 67438;
  const long nH = (1L << 30) / 16;
  float4 *ha, *hb;
  CK(cudaMalloc(&ha, nH * 16));
  CK(cudaMalloc(&hb, nH * 16));
  const bool thp = argc > 2 && !strcmp(argv[2], "thp");
  const bool quick = argc > 3 && !strcmp(argv[3], "quick");
  float4* host;
  auto ta = std::chrono::steady_clock::now();
  if (thp) {
    if (posix_memalign((void**)&host, 1 << 21, table_rows * 512)) return 1;
    madvise(host, table_rows * 512, MADV_HUGEPAGE);
    memset(host, 0, table_rows * 512);
    CK(cudaHostRegister(host, table_rows * 512, cudaHostRegisterMapped | cudaHostRegisterPortable));
  } else {
    CK(cudaHostAlloc(&host, table_rows * 512, cudaHostAllocMapped));
  }
  printf("slow tier: %s, alloc %.0f ms\n", thp ? "THP + cudaHostRegister" : "cudaHostAlloc",
         std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - ta).count());
  for (long i = 0; i < table_rows * 32; i += 997) host[i] = make_float4((float)i, 1.f, 2.f, 3.f);
  float4* hostd;
  CK(cudaHostGetDevicePointer((void**)&hostd, host, 0));
  float4* dst;
  CK(cudaMalloc(&dst, (long)rows * 512));
  std::vector<int> idx(rows);
  std::mt19937_64 g(1);
  for (int i = 0; i < rows; ++i) idx[i] = (int)(g() % table_rows);
  std::sort(idx.begin(), idx.end());
  int* didx;
  CK(cudaMalloc(&didx, rows * 4));
  CK(cudaMemcpy(didx, idx.data(), rows * 4, cudaMemcpyHostToDevice));
  const int nL = 1 << 20, nrows = 1 << 21;
  int *la, *lb;
  CK(cudaMalloc(&la, nL * 4));
  CK(cudaMalloc(&lb, nrows * 4));
  {
    std::vector<int> h1(nL), h2(nrows);
    for (int i = 0; i < nL; ++i) h1[i] = (int)(g() % nrows);
    for (int i = 0; i < nrows; ++i) h2[i] = (int)(g() % nrows);
    CK(cudaMemcpy(la, h1.data(), nL * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(lb, h2.data(), nrows * 4, cudaMemcpyHostToDevice));
  }
  float4* lout;
  CK(cudaMalloc(&lout, (long)nL * 512));
  cudaStream_t s1, s2;
  CK(cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));

  std::vector<void*> hsrc(rows), ddst(rows), dsrc(rows), hdst(rows);
  std::vector<size_t> sz(rows, 512);
  for (int i = 0; i < rows; ++i) {
    hsrc[i] = (char*)host + (long)idx[i] * 512;
    ddst[i] = (char*)dst + (long)i * 512;
    dsrc[i] = ddst[i];
    hdst[i] = hsrc[i];
  }
  double submit_us = 0;
  int submits = 0;
  auto batch = [&](cudaStream_t s, bool h2d, unsigned flags, int chunk) {
    cudaMemcpyAttributes attr = {};
    attr.srcAccessOrder = cudaMemcpySrcAccessOrderStream;
    attr.flags = flags;
    size_t attr_idx = 0, fail = 0;
    auto t0 = std::chrono::steady_clock::now();
    for (int b = 0; b < rows; b += chunk) {
      const int c = std::min(chunk, rows - b);
      cudaError_t e = h2d ? cudaMemcpyBatchAsync(ddst.data() + b, hsrc.data() + b, sz.data() + b, c, &attr, &attr_idx,
                                                 1, &fail, s)
                          : cudaMemcpyBatchAsync(hdst.data() + b, dsrc.data() + b, sz.data() + b, c, &attr, &attr_idx,
                                                 1, &fail, s);
      if (e != cudaSuccess) {
        printf("batch: %s (fail idx %zu)\n", cudaGetErrorString(e), fail);
        exit(1);
      }
    }
    submit_us += std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count();
    ++submits;
  };
  auto H = [&](cudaStream_t s) { hbm_copy<<<148 * 8, 256, 0, s>>>(ha, hb, nH); };
  auto L = [&](cudaStream_t s) { dep_gather<<<148 * 8, 256, 0, s>>>(la, lb, ha, lout, nL, nrows); };
  auto Z = [&](cudaStream_t s) { zc_gather<<<148 * 4, 256, 0, s>>>(hostd, dst, didx, rows); };

  auto alone = [&](const char* name, auto fn) {
    Timer t;
    for (int w = 0; w < 2; ++w) fn(s1);
    CK(cudaDeviceSynchronize());
    float best = 1e9;
    submit_us = 0;
    submits = 0;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(t.a, s1);
      fn(s1);
      cudaEventRecord(t.b, s1);
      CK(cudaEventSynchronize(t.b));
      best = std::min(best, t.ms());
    }
    printf("%-36s alone %8.3f ms  %6.1f GB/s", name, best, rows * 512.0 / best / 1e6);
    if (submits) printf("  (host submit %.0f us)", submit_us / submits);
    printf("\n");
    return best;
  };
  auto both = [&](const char* name, auto f1, auto f2) {
    Timer t1, t2, t0;
    float b1 = 1e9, b2 = 1e9;
    for (int r = 0; r < 5; ++r) {
      CK(cudaDeviceSynchronize());
      cudaEventRecord(t0.a, s1);
      cudaStreamWaitEvent(s2, t0.a, 0);
      cudaEventRecord(t1.a, s1);
      cudaEventRecord(t2.a, s2);
      f1(s1);
      f2(s2);
      cudaEventRecord(t1.b, s1);
      cudaEventRecord(t2.b, s2);
      CK(cudaDeviceSynchronize());
      b1 = std::min(b1, t1.ms());
      b2 = std::min(b2, t2.ms());
    }
    printf("%-36s together %8.3f | %8.3f ms\n", name, b1, b2);
  };
  printf("table %ld rows (%.1f GB pinned), %d random 512 B rows per copy\n", table_rows, table_rows * 512 / 1e9, rows);
  alone("H hbm copy 2x1GiB", H);
  alone("L dependent gather 1M rows", L);
  alone("Z zero-copy SM gather", Z);
  if (quick) {
    both("H + Z", H, Z);
    both("L + Z", L, Z);
    return 0;
  }
  for (int chunk : {rows, 8192, 1024}) {
    char nm[80];
    snprintf(nm, sizeof nm, "BA h2d batch chunk %d", chunk);
    alone(nm, [&](cudaStream_t s) { batch(s, true, 0, chunk); });
  }
  alone("BA h2d batch PreferOverlapWithCompute",
        [&](cudaStream_t s) { batch(s, true, cudaMemcpyFlagPreferOverlapWithCompute, rows); });
  alone("BD d2h batch (scatter into table)", [&](cudaStream_t s) { batch(s, false, 0, rows); });
  both("H + BA", H, [&](cudaStream_t s) { batch(s, true, 0, rows); });
  both("L + BA", L, [&](cudaStream_t s) { batch(s, true, 0, rows); });
  both("H + BD", H, [&](cudaStream_t s) { batch(s, false, 0, rows); });
  both("L + BD", L, [&](cudaStream_t s) { batch(s, false, 0, rows); });
  both("BA + BD", [&](cudaStream_t s) { batch(s, true, 0, rows); }, [&](cudaStream_t s) { batch(s, false, 0, rows); });
  both("H + Z", H, Z);
  both("L + Z", L, Z);
  {  // correctness: batch gather == SM gather
    std::vector<float> a((long)rows * 128), b((long)rows * 128);
    Z(s1);
    CK(cudaStreamSynchronize(s1));
    CK(cudaMemcpy(a.data(), dst, (long)rows * 512, cudaMemcpyDeviceToHost));
    CK(cudaMemset(dst, 0, (long)rows * 512));
    batch(s1, true, 0, rows);
    CK(cudaStreamSynchronize(s1));
    CK(cudaMemcpy(b.data(), dst, (long)rows * 512, cudaMemcpyDeviceToHost));
    printf("batch gather == SM gather: %s\n", a == b ? "yes" : "NO");
  }
  return 0;
}
