// Could part of the miss staging go through host threads + copy-engine DMA beside the TMA
// gather? Stages R random 512 B rows of a 16 GiB pinned table into HBM:
//   tma     : all R rows by the TMA gather kernel (40 blocks, as k_admit_stage_tma)
//   hyb f,T : a fraction f of the rows gathered by T host threads into pinned memory and
//             copied H2D by the copy engine, the rest by the TMA kernel, concurrently
//   + d2h   : the same with a 34.5 MB D2H copy running beside it (the write-back)
// Reports the wall time until both parts have landed (CUDA events + host clock).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/hyb tools/hybrid_staging_bench.cu -lpthread
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <thread>
#include <vector>

#include <cuda_runtime.h>

#define CK(x)                                                            \
  do {                                                                   \
    cudaError_t e = (x);                                                 \
    if (e != cudaSuccess) {                                              \
      printf("%s: %s (line %d)\n", #x, cudaGetErrorString(e), __LINE__); \
      exit(1);                                                           \
    }                                                                    \
  } while (0)

__device__ __forceinline__ unsigned su32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__global__ void tma_gather(const char* __restrict__ host, char* __restrict__ dev, const long* __restrict__ idx,
                           int nrows) {
  constexpr int ST = 4;
  extern __shared__ __align__(128) char ring[];
  __shared__ uint64_t bar[ST];
  if (threadIdx.x != 0) return;
  for (int s = 0; s < ST; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[s])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  const int ngroups = (nrows + 31) / 32;
  const int mine = ngroups > (int)blockIdx.x ? (ngroups - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
  unsigned ph = 0;
  int issued = 0, retired = 0;
  while (retired < mine) {
    if (issued < mine && issued - retired < ST) {
      const int st = issued % ST;
      if (issued >= ST) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      const int g = blockIdx.x + issued * gridDim.x;
      const int r0 = g * 32, cnt = min(32, nrows - r0);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar[st])), "r"(cnt * 512)
                   : "memory");
      for (int r = 0; r < cnt; ++r)
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 512, [%2];" ::"r"(
                su32(ring + (st * 32 + r) * 512)),
            "l"(host + idx[r0 + r] * 512), "r"(su32(&bar[st]))
            : "memory");
      ++issued;
      continue;
    }
    const int st = retired % ST;
    asm volatile(
        "{\n .reg .pred p;\n W_%=: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W_%=;\n}\n" ::"r"(
            su32(&bar[st])),
        "r"((ph >> st) & 1u)
        : "memory");
    ph ^= 1u << st;
    const int g = blockIdx.x + retired * gridDim.x;
    const int r0 = g * 32, cnt = min(32, nrows - r0);
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dev + (long)r0 * 512),
                 "r"(su32(ring + st * 32 * 512)), "r"(cnt * 512)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    ++retired;
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main() {
  const long table_rows = 32L << 20;  // 16 GiB of 512 B rows
  const int R = 67440;                // rows per step (cfg2 misses)
  char* host;
  CK(cudaHostAlloc(&host, table_rows * 512, cudaHostAllocMapped));
  {  // touch in parallel
    std::vector<std::thread> th;
    for (int t = 0; t < 16; ++t)
      th.emplace_back([&, t] { std::memset(host + (table_rows * 512 / 16) * t, 1, table_rows * 512 / 16); });
    for (auto& x : th) x.join();
  }
  char* hdev;
  CK(cudaHostGetDevicePointer((void**)&hdev, host, 0));
  std::mt19937_64 rng(3);
  std::vector<long> idx(R);
  char *dstage, *d2h_src, *hpin, *hd2h;
  long* didx;
  CK(cudaMalloc(&dstage, (long)R * 512));
  CK(cudaMalloc(&d2h_src, (long)R * 512));
  CK(cudaMalloc(&didx, R * 8));
  CK(cudaHostAlloc(&hpin, (long)R * 512, cudaHostAllocDefault));
  CK(cudaHostAlloc(&hd2h, (long)R * 512, cudaHostAllocDefault));
  CK(cudaFuncSetAttribute(tma_gather, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 32 * 512));
  cudaStream_t sk, sc, sd;
  CK(cudaStreamCreateWithFlags(&sk, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&sc, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&sd, cudaStreamNonBlocking));
  auto run = [&](double frac, int threads, bool d2h) {
    for (auto& v : idx) v = (long)(rng() % table_rows);
    std::sort(idx.begin(), idx.end());  // admitted ranks ascend
    const int nh = (int)(R * frac), nd = R - nh;  // host part = the last nh rows
    CK(cudaMemcpy(didx, idx.data(), R * 8, cudaMemcpyHostToDevice));
    CK(cudaDeviceSynchronize());
    const auto t0 = std::chrono::steady_clock::now();
    if (d2h) CK(cudaMemcpyAsync(hd2h, d2h_src, (long)R * 512, cudaMemcpyDeviceToHost, sd));
    if (nd > 0) tma_gather<<<40, 32, 4 * 32 * 512, sk>>>(hdev, dstage, didx, nd);
    if (nh > 0) {
      // host threads gather in pieces; each piece goes H2D as soon as it is packed
      const int piece = 4096;
      std::atomic<int> next{0};
      std::vector<std::thread> th;
      std::vector<std::atomic<int>> done((nh + piece - 1) / piece);
      for (auto& d : done) d = 0;
      for (int t = 0; t < threads; ++t)
        th.emplace_back([&] {
          for (int p; (p = next.fetch_add(1)) < (int)done.size();) {
            const int a = p * piece, b = std::min(nh, a + piece);
            for (int r = a; r < b; ++r) std::memcpy(hpin + (long)r * 512, host + idx[nd + r] * 512, 512);
            done[p] = 1;
          }
        });
      for (int p = 0; p < (int)done.size(); ++p) {
        while (!done[p]) std::this_thread::yield();
        const int a = p * piece, b = std::min(nh, a + piece);
        CK(cudaMemcpyAsync(dstage + (long)(nd + a) * 512, hpin + (long)a * 512, (long)(b - a) * 512,
                           cudaMemcpyHostToDevice, sc));
      }
      for (auto& x : th) x.join();
    }
    CK(cudaStreamSynchronize(sk));
    CK(cudaStreamSynchronize(sc));
    const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    CK(cudaStreamSynchronize(sd));
    // check
    for (int r = 0; r < R; r += 997) {
      char v[512];
      CK(cudaMemcpy(v, dstage + (long)r * 512, 512, cudaMemcpyDeviceToHost));
      if (std::memcmp(v, host + idx[r] * 512, 512)) {
        printf("MISMATCH row %d\n", r);
        break;
      }
    }
    return ms;
  };
  // distinct row contents so the check means something
  for (long r = 0; r < table_rows; r += 1) *reinterpret_cast<long*>(host + r * 512) = r;
  for (int rep = 0; rep < 2; ++rep) {
    for (bool d2h : {false, true}) {
      printf("d2h=%d tma only: %.3f ms\n", d2h, std::min({run(0, 0, d2h), run(0, 0, d2h), run(0, 0, d2h)}));
      for (double f : {0.2, 0.3, 0.4, 0.5})
        for (int t : {4, 8, 12}) {
          double best = 1e9;
          for (int k = 0; k < 3; ++k) best = std::min(best, run(f, t, d2h));
          printf("d2h=%d hybrid f=%.1f threads=%2d: %.3f ms\n", d2h, f, t, best);
        }
    }
  }
  return 0;
}
