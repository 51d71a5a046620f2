// Why does every small kernel take ~90 us while the miss staging runs?
// (profiles/r02_timeline_*.txt: k_plan, a <<<1,1>>> kernel, 2.5 us alone, ~100 us beside
// k_admit_stage_tma; a 53 KB memset 90 us; big HBM kernels only ~20% slower.)
//
// Background (stream bg): host-link traffic for ~25 ms --
//   none | TMA gather of random 512 B rows from pinned host memory (B blocks, 4-stage ring of
//   32 rows) | SM zero-copy gather | copy-engine H2D memcpy (contiguous).
// Foreground (stream fg), timed with events on fg:
//   chain   30 dependent 1-thread kernels, each launched from the host while bg runs
//   gated   the same 30 kernels queued behind an event of a 3 ms sleep kernel on a third
//           stream, so their launch commands are submitted long before they may start
//   graph   the 30 kernels as one CUDA graph (uploaded before), launched while bg runs
//   memset  10 x cudaMemsetAsync of 53 KB
//   hbm     a 256 MB device copy
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ll tools/launch_latency.cu
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <string>
#include <thread>
#include <chrono>
#include <vector>

#include <cooperative_groups.h>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

#define CK(x)                                                                     \
  do {                                                                            \
    cudaError_t e = (x);                                                          \
    if (e != cudaSuccess) {                                                       \
      printf("%s: %s (line %d)\n", #x, cudaGetErrorString(e), __LINE__);          \
      exit(1);                                                                    \
    }                                                                             \
  } while (0)

__device__ __forceinline__ unsigned su32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__global__ void tma_gather(const char* __restrict__ host, char* __restrict__ dev, const int* __restrict__ idx,
                           int nrows) {
  constexpr int ST = 4;
  extern __shared__ __align__(128) char ring[];  // ST x 32 rows x 512 B
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
            "l"(host + (long)idx[r0 + r] * 512), "r"(su32(&bar[st]))
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

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
// the same gather issued at a fixed rate: group k of block b no earlier than t0 + k * gap_ns
__global__ void tma_paced(const char* __restrict__ host, char* __restrict__ dev, const int* __restrict__ idx,
                          int nrows, unsigned gap_ns) {
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
  const unsigned long long t0 = gtimer() + (unsigned long long)blockIdx.x * gap_ns / gridDim.x;
  while (retired < mine) {
    if (issued < mine && issued - retired < ST && gtimer() >= t0 + (unsigned long long)issued * gap_ns) {
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
            "l"(host + (long)idx[r0 + r] * 512), "r"(su32(&bar[st]))
            : "memory");
      ++issued;
      continue;
    }
    if (issued == retired) continue;  // waiting for the pacing clock
    const int st = retired % ST;
    unsigned done = 0;
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                 : "=r"(done) : "r"(su32(&bar[st])), "r"((ph >> st) & 1u) : "memory");
    if (!done) continue;
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

__global__ void zc_gather(const float4* __restrict__ host, float4* __restrict__ dev, const int* __restrict__ idx,
                          int nrows) {
  const int lane = threadIdx.x & 31;
  const long warp = (blockIdx.x * (long)blockDim.x + threadIdx.x) >> 5;
  const long nw = (gridDim.x * (long)blockDim.x) >> 5;
  for (long r = warp; r < nrows; r += nw) dev[r * 32 + lane] = host[(long)idx[r] * 32 + lane];
}

__global__ void tiny(int* c) { c[1] = c[0] + 1; }
// 30 grid-wide barriers inside one cooperative kernel (one block per SM)
__global__ void coop30(int* c) {
  cg::grid_group g = cg::this_grid();
  for (int i = 0; i < 30; ++i) {
    if (threadIdx.x == 0 && blockIdx.x == 0) c[1] = c[0] + i;
    g.sync();
  }
}
// 30 barriers of a hand-rolled flag barrier: one atomic + a spin on a generation word
// mode 0: relaxed; 1: __threadfence() before arriving; 2: red.release.gpu arrive + ld.acquire.gpu spin
__global__ void flagm(unsigned* bar, int mode) {
  for (int i = 0; i < 30; ++i) {
    __syncthreads();
    if (threadIdx.x == 0) {
      const unsigned target = (unsigned)(i + 1) * gridDim.x;
      if (mode == 1) __threadfence();
      if (mode == 2) {
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
        unsigned v;
        do {
          asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar) : "memory");
        } while (v < target);
      } else {
        atomicAdd(&bar[0], 1u);
        while (atomicAdd(&bar[0], 0u) < target) {
        }
      }
    }
    __syncthreads();
  }
}
__global__ void flag30(unsigned* bar) {
  for (int i = 0; i < 30; ++i) {
    __syncthreads();
    if (threadIdx.x == 0) {
      const unsigned target = (unsigned)(i + 1) * gridDim.x;
      atomicAdd(&bar[0], 1u);
      while (atomicAdd(&bar[0], 0u) < target) {
      }
    }
    __syncthreads();
  }
}
// one thread, 2000 dependent loads over an L2-resident ring: per-access latency
__global__ void chase(const int* __restrict__ nxt, int* out) {
  int p = 0;
  for (int i = 0; i < 2000; ++i) p = nxt[p];
  out[0] = p;
}
__global__ void sleep_k(long ns) {
  long t0 = clock64();
  while (clock64() - t0 < ns * 2) {
  }
}
__global__ void hbm_copy(const float4* __restrict__ a, float4* __restrict__ b, long n) {
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) b[i] = a[i];
}

int main(int argc, char** argv) {
  const long host_rows = 8L << 20;  // 4 GiB of 512 B rows
  const int nrows = 1 << 19;         // 256 MiB per background pass (~5 ms at 50 GB/s)
  char* host;
  CK(cudaHostAlloc(&host, host_rows * 512, cudaHostAllocMapped));
  std::memset(host, 1, host_rows * 512);
  char* hdev;
  CK(cudaHostGetDevicePointer((void**)&hdev, host, 0));
  std::vector<int> idx(nrows);
  std::mt19937_64 rng(1);
  for (auto& v : idx) v = (int)(rng() % host_rows);
  int* didx;
  char* dstage;
  CK(cudaMalloc(&didx, nrows * 4));
  CK(cudaMemcpy(didx, idx.data(), nrows * 4, cudaMemcpyHostToDevice));
  CK(cudaMalloc(&dstage, (long)nrows * 512));
  const long hb = 256L << 20;
  float4 *ha, *hbuf;
  CK(cudaMalloc(&ha, hb));
  CK(cudaMalloc(&hbuf, hb));
  unsigned* bar;
  CK(cudaMalloc(&bar, 64));
  char* dsrc;  // device-resident source for the control case (same random rows, 4 GiB)
  CK(cudaMalloc(&dsrc, host_rows * 512));
  int* ctr;
  CK(cudaMalloc(&ctr, 64));
  char* dmem;
  CK(cudaMalloc(&dmem, 53 * 1024));
  int* dnext;  // random cyclic permutation over 1M ints (4 MB, L2 resident), stride-scattered
  {
    const int n = 1 << 20;
    std::vector<int> perm(n), nx(n);
    for (int i = 0; i < n; ++i) perm[i] = i;
    std::shuffle(perm.begin(), perm.end(), rng);
    for (int i = 0; i < n; ++i) nx[perm[i]] = perm[(i + 1) % n];
    CK(cudaMalloc(&dnext, n * 4));
    CK(cudaMemcpy(dnext, nx.data(), n * 4, cudaMemcpyHostToDevice));
  }
  CK(cudaFuncSetAttribute(tma_gather, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 32 * 512));
  CK(cudaFuncSetAttribute(tma_paced, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 32 * 512));
  cudaStream_t bg, fg, gs, bg2;
  CK(cudaStreamCreateWithFlags(&bg2, cudaStreamNonBlocking));
  char* hdst;  // pinned destination of the D2H background copies
  CK(cudaHostAlloc(&hdst, (long)nrows * 512, cudaHostAllocDefault));
  CK(cudaStreamCreateWithFlags(&bg, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&fg, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&gs, cudaStreamNonBlocking));
  cudaEvent_t e0, e1, eg;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  CK(cudaEventCreateWithFlags(&eg, cudaEventDisableTiming));
  // the chain as a graph
  cudaGraph_t g;
  cudaGraphExec_t ge;
  CK(cudaStreamBeginCapture(fg, cudaStreamCaptureModeThreadLocal));
  for (int i = 0; i < 30; ++i) tiny<<<1, 1, 0, fg>>>(ctr);
  CK(cudaStreamEndCapture(fg, &g));
  CK(cudaGraphInstantiate(&ge, g, 0));
  CK(cudaGraphUpload(ge, fg));
  CK(cudaDeviceSynchronize());

  auto launch_bg = [&](const std::string& kind0, int blocks) {
    std::string kind = kind0;
    if (kind.rfind("d2h", 0) == 0) {  // "d2h" alone, or "d2h+paced" with the paced gather beside it
      for (int rep = 0; rep < 5; ++rep)
        CK(cudaMemcpyAsync(hdst, dstage, (long)nrows * 512, cudaMemcpyDeviceToHost, bg2));
      if (kind == "d2h") return;
      kind = kind.substr(4);
    }
    for (int rep = 0; rep < 5; ++rep) {
      if (kind == "paced") {  // 40 blocks, 16 KB groups: gap = 40 * 16 KB / rate
        const unsigned gap = (unsigned)(40.0 * 16384.0 / blocks);  // ns (GB/s = B/ns)
        tma_paced<<<40, 32, 4 * 32 * 512, bg>>>(hdev, dstage, didx, nrows, gap);
      } else if (kind == "tmadev") tma_gather<<<blocks, 32, 4 * 32 * 512, bg>>>(dsrc, dstage, didx, nrows);
      else if (kind == "tma") tma_gather<<<blocks, 32, 4 * 32 * 512, bg>>>(hdev, dstage, didx, nrows);
      else if (kind == "zc") zc_gather<<<blocks, 256, 0, bg>>>((const float4*)hdev, (float4*)dstage, didx, nrows);
      else if (kind == "dma") CK(cudaMemcpyAsync(dstage, host, (long)nrows * 512, cudaMemcpyHostToDevice, bg));
    }
  };
  auto fg_case = [&](const std::string& c) {
    if (c == "gated") {
      sleep_k<<<1, 1, 0, gs>>>(3000000);
      CK(cudaEventRecord(eg, gs));
      CK(cudaStreamWaitEvent(fg, eg, 0));
      CK(cudaEventRecord(e0, fg));
      for (int i = 0; i < 30; ++i) tiny<<<1, 1, 0, fg>>>(ctr);
      CK(cudaEventRecord(e1, fg));
      return;
    }
    CK(cudaEventRecord(e0, fg));
    if (c == "chain")
      for (int i = 0; i < 30; ++i) tiny<<<1, 1, 0, fg>>>(ctr);
    else if (c == "graph")
      CK(cudaGraphLaunch(ge, fg));
    else if (c == "memset")
      for (int i = 0; i < 10; ++i) CK(cudaMemsetAsync(dmem, 0xff, 53 * 1024, fg));
    else if (c == "coop30") {
      void* a[] = {&ctr};
      CK(cudaLaunchCooperativeKernel((const void*)coop30, 148, 256, a, 0, fg));
    } else if (c == "flag30") {
      CK(cudaMemsetAsync(bar, 0, 64, fg));
      CK(cudaEventRecord(e0, fg));
      flag30<<<148, 256, 0, fg>>>(bar);
    } else if (c == "flagfence" || c == "flagrel") {
      CK(cudaMemsetAsync(bar, 0, 64, fg));
      CK(cudaEventRecord(e0, fg));
      flagm<<<148, 256, 0, fg>>>(bar, c == "flagfence" ? 1 : 2);
    } else if (c == "chase")
      chase<<<1, 1, 0, fg>>>(dnext, ctr + 4);
    else if (c == "hbm")
      hbm_copy<<<148 * 8, 256, 0, fg>>>(ha, hbuf, hb / 16);
    CK(cudaEventRecord(e1, fg));
  };
  struct Bg {
    const char* kind;
    int blocks;
  };
  // paced: blocks = 40, the number is the target rate in GB/s
  const Bg bgs[] = {{"none", 0}, {"paced", 30}, {"paced", 36}, {"d2h", 0}, {"d2h+paced", 20}, {"d2h+paced", 25},
                    {"d2h+paced", 30}, {"d2h+paced", 36}, {"d2h+tma", 40}};
  const char* fgs[] = {"chain", "flag30", "chase", "hbm"};
  // background throughput alone
  for (const Bg& b : bgs) {
    if (std::string(b.kind) == "none" || std::string(b.kind).rfind("d2h+", 0) == 0) continue;
    cudaEvent_t a0, a1;
    CK(cudaEventCreate(&a0));
    CK(cudaEventCreate(&a1));
    CK(cudaEventRecord(a0, bg));
    launch_bg(b.kind, b.blocks);
    CK(cudaEventRecord(a1, bg));
    CK(cudaDeviceSynchronize());
    float ms;
    CK(cudaEventElapsedTime(&ms, a0, a1));
    printf("bg %-4s %3d alone: %.2f ms for 5 x %d MB -> %.1f GB/s\n", b.kind, b.blocks, ms, nrows / 2048,
           5.0 * nrows * 512 / ms / 1e6);
  }
  for (const char* f : fgs) {
    for (const Bg& b : bgs) {
      float best = 1e9, sum = 0;
      const int reps = 3;
      for (int r = 0; r < reps; ++r) {
        CK(cudaDeviceSynchronize());
        launch_bg(b.kind, b.blocks);
        std::this_thread::sleep_for(std::chrono::microseconds(2000));  // bg is running
        fg_case(f);
        CK(cudaEventSynchronize(e1));
        float ms;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        best = std::min(best, ms);
        sum += ms;
        CK(cudaDeviceSynchronize());
      }
      printf("fg %-6s | bg %-4s %3d : min %8.1f us  avg %8.1f us\n", f, b.kind, b.blocks, best * 1e3,
             sum / reps * 1e3);
    }
  }
  return 0;
}
