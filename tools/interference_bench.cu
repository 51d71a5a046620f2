// Interference microbenchmark: how much host-link traffic slows a concurrent
// HBM-bound kernel (and vice versa). Decides how the prefetch pipeline may overlap
// the miss staging with the forward/backward.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ib tools/interference_bench.cu
// Cases (each timed alone and concurrently on two streams, CUDA events):
//   H  HBM stream copy, 1 GiB, float4, grid = 148*8
//   Z  zero-copy gather of random 512 B rows from pinned host memory (like k_admit_stage), 67k rows
//   ZS Z with its blocks limited (grid 148 / 32)
//   DH cudaMemcpyAsync H2D contiguous 34.5 MB;  DD cudaMemcpyAsync D2H 34.5 MB
//   BA cudaMemcpyBatchAsync of 67k random 512 B host rows -> HBM (copy engine gather)
// `ib chain`: a dependent chain of 17 small kernels (the shape of the prepare's index
// phase) alone and beside the TMA staging T(40) / zero-copy Z / copy-engine DH -- is the
// cost per kernel or per byte?
#include <algorithm>
#include <string>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#include <cuda.h>
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

// lane i of a warp owns row i; 4 units in flight per lane (mirrors warp_copy_rows)
template <int U>
__global__ void zc_gather(const float4* __restrict__ host, float4* __restrict__ dev, const int* __restrict__ idx,
                          int nrows, int upr) {
  const int lane = threadIdx.x & 31;
  const long warp = (blockIdx.x * (long)blockDim.x + threadIdx.x) >> 5;
  const long nw = (gridDim.x * (long)blockDim.x) >> 5;
  for (long base = warp * 32; base < nrows; base += nw * 32) {
    const long j = base + lane;
    const long src = j < nrows ? (long)idx[j] : 0;
    const int total = 32 * upr;
    for (int u0 = 0; u0 < total; u0 += 32 * U) {
      float4 v[U];
      long d[U];
      bool a[U];
#pragma unroll
      for (int q = 0; q < U; ++q) {
        const int u = u0 + q * 32 + lane;
        const int rr = u / upr;
        const int c = u - rr * upr;
        const long s = __shfl_sync(0xffffffffu, src, rr);
        a[q] = base + rr < nrows;
        d[q] = (base + rr) * upr + c;
        if (a[q]) v[q] = host[s * upr + c];
      }
#pragma unroll
      for (int q = 0; q < U; ++q)
        if (a[q]) dev[d[q]] = v[q];
    }
  }
}


// TMA (bulk-copy engine) gather: one thread per block issues cp.async.bulk loads of
// whole 512 B rows from host memory into a shared-memory ring (mbarrier-tracked),
// then one bulk store of the 32 contiguous rows to HBM.
__device__ __forceinline__ void mbar_init(uint64_t* b, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(b)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(b)),
               "r"(bytes));
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned phase) {
  asm volatile(
      "{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}\n" ::"r"(
          (unsigned)__cvta_generic_to_shared(b)),
      "r"(phase));
}
__device__ __forceinline__ void bulk_g2s(void* smem, const void* gmem, unsigned bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   (unsigned)__cvta_generic_to_shared(smem)),
               "l"(gmem), "r"(bytes), "r"((unsigned)__cvta_generic_to_shared(bar))
               : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* gmem, const void* smem, unsigned bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gmem),
               "r"((unsigned)__cvta_generic_to_shared(smem)), "r"(bytes)
               : "memory");
  asm volatile("cp.async.bulk.commit_group;");
}

template <int STAGES>
__global__ void tma_gather(const char* __restrict__ host, char* __restrict__ dev, const int* __restrict__ idx,
                           int nrows) {
  extern __shared__ __align__(128) char ring[];  // STAGES x 32 rows x 512 B
  __shared__ uint64_t bar[STAGES];
  if (threadIdx.x != 0) return;
  for (int s = 0; s < STAGES; ++s) mbar_init(&bar[s], 1);
  asm volatile("fence.mbarrier_init.release.cluster;");
  const int ngroups = (nrows + 31) / 32;
  int k = 0;
  unsigned phase[STAGES] = {0};
  // prologue + steady state: issue group g into stage g % STAGES, retire group g - STAGES + 1
  int issued = 0;
  for (int g = blockIdx.x; g < ngroups || issued > 0; g += gridDim.x) {
    if (g < ngroups) {
      const int st = k % STAGES;
      if (k >= STAGES) {  // the stage's previous store must have read the smem
        asm volatile("cp.async.bulk.wait_group.read 0;");
      }
      const int r0 = g * 32, cnt = min(32, nrows - r0);
      mbar_expect_tx(&bar[st], cnt * 512);
      for (int r = 0; r < cnt; ++r) bulk_g2s(ring + (st * 32 + r) * 512, host + (long)idx[r0 + r] * 512, 512, &bar[st]);
      ++k;
      ++issued;
    }
    if (issued == STAGES || (g >= ngroups && issued > 0)) {  // retire the oldest group
      const int kk = k - issued;
      const int st = kk % STAGES;
      mbar_wait(&bar[st], phase[st]);
      phase[st] ^= 1;
      const int gg = blockIdx.x + kk * gridDim.x;
      const int r0 = gg * 32, cnt = min(32, nrows - r0);
      bulk_s2g(dev + (long)r0 * 512, ring + st * 32 * 512, cnt * 512);
      --issued;
    }
    if (g >= ngroups && issued == 0) break;
  }
  asm volatile("cp.async.bulk.wait_group 0;");
}

// one tiny step of a kernel chain: a few dependent loads + a store (like k_begin / k_plan)
__global__ void tiny_step(int* c, int k) {
  int v = c[k];
  v = c[(v & 7) + 8];
  c[k + 1] = v + 1;
}
// one wide step: every thread loads one id and sets a bit (like k_mark_ids / k_bits_count)
__global__ void wide_step(const int* __restrict__ ids, unsigned* bits, int n) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int v = ids[i];
    if (!(bits[v >> 5] & (1u << (v & 31)))) atomicOr(&bits[v >> 5], 1u << (v & 31));
  }
}

// latency-bound: two dependent random index loads, then a random 512 B row per warp
__global__ void dep_gather(const int* __restrict__ a, const int* __restrict__ b, const float4* __restrict__ rows,
                           float4* __restrict__ out, int n, int nrows) {
  const int lane = threadIdx.x & 31;
  const long warp = (blockIdx.x * (long)blockDim.x + threadIdx.x) >> 5;
  const long nw = (gridDim.x * (long)blockDim.x) >> 5;
  for (long j = warp; j < n; j += nw) {
    const int r = b[a[j] % nrows] % nrows;
    out[j * 32 + lane] = rows[(long)r * 32 + lane];
  }
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
  const bool chain = argc > 1 && std::string(argv[1]) == "chain";
  const long nH = (1L << 30) / 16;  // 1 GiB of float4
  const int rows = 67438, upr = 32;  // 512 B rows
  const long table_rows = 33762577;
  float4 *ha, *hb;
  CK(cudaMalloc(&ha, nH * 16));
  CK(cudaMalloc(&hb, nH * 16));
  float4* host;
  CK(cudaHostAlloc(&host, table_rows * 512, cudaHostAllocMapped));
  float4* hostd;
  CK(cudaHostGetDevicePointer((void**)&hostd, host, 0));
  for (long i = 0; i < table_rows * 32; i += 997) host[i] = make_float4((float)i, 1.f, 2.f, 3.f);
  float4* zdst;
  CK(cudaMalloc(&zdst, (long)rows * 512));
  float4* hstage;
  CK(cudaHostAlloc(&hstage, (long)rows * 512, cudaHostAllocDefault));
  std::vector<int> idx(rows);
  std::mt19937_64 g(1);
  for (int i = 0; i < rows; ++i) idx[i] = (int)(g() % table_rows);
  std::sort(idx.begin(), idx.end());
  int* didx;
  CK(cudaMalloc(&didx, rows * 4));
  CK(cudaMemcpy(didx, idx.data(), rows * 4, cudaMemcpyHostToDevice));
  cudaStream_t s1, s2;
  CK(cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
  // batch copy descriptors
  std::vector<void*> bsrc(rows), bdst(rows);
  std::vector<size_t> bsz(rows, 512);
  for (int i = 0; i < rows; ++i) {
    bsrc[i] = (char*)host + (long)idx[i] * 512;
    bdst[i] = (char*)zdst + (long)i * 512;
  }

  auto H = [&](cudaStream_t s) { hbm_copy<<<148 * 8, 256, 0, s>>>(ha, hb, nH); };
  auto Z = [&](cudaStream_t s, int grid) { zc_gather<4><<<grid, 256, 0, s>>>(hostd, zdst, didx, rows, upr); };
  auto ZC = [&](int grid, int threads, int unroll) {
    return [=](cudaStream_t s) {
      if (unroll == 8) zc_gather<8><<<grid, threads, 0, s>>>(hostd, zdst, didx, rows, upr);
      else if (unroll == 16) zc_gather<16><<<grid, threads, 0, s>>>(hostd, zdst, didx, rows, upr);
      else zc_gather<4><<<grid, threads, 0, s>>>(hostd, zdst, didx, rows, upr);
    };
  };
  auto DH = [&](cudaStream_t s) { cudaMemcpyAsync(zdst, hstage, (long)rows * 512, cudaMemcpyHostToDevice, s); };
  auto DD = [&](cudaStream_t s) { cudaMemcpyAsync(hstage, zdst, (long)rows * 512, cudaMemcpyDeviceToHost, s); };
  auto BA = [&](cudaStream_t s) {
    cudaMemcpyAttributes attr = {};
    attr.srcAccessOrder = cudaMemcpySrcAccessOrderStream;
    attr.flags = cudaMemcpyFlagPreferOverlapWithCompute;
    size_t attr_idx = 0, fail = 0;
    cudaError_t e = cudaMemcpyBatchAsync(bdst.data(), bsrc.data(), bsz.data(), rows, &attr, &attr_idx, 1, &fail, s);
    if (e != cudaSuccess) printf("batch: %s\n", cudaGetErrorString(e));
  };

  auto alone = [&](const char* name, auto fn) {
    Timer t;
    for (int w = 0; w < 2; ++w) fn(s1);
    CK(cudaDeviceSynchronize());
    float best = 1e9;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(t.a, s1);
      fn(s1);
      cudaEventRecord(t.b, s1);
      CK(cudaEventSynchronize(t.b));
      best = std::min(best, t.ms());
    }
    printf("%-28s alone %8.3f ms\n", name, best);
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
    printf("%-28s together %8.3f | %8.3f ms\n", name, b1, b2);
  };
  if (chain) {
    CK(cudaFuncSetAttribute(tma_gather<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 32 * 512));
    int* cc;
    CK(cudaMalloc(&cc, 4096));
    CK(cudaMemset(cc, 0, 4096));
    const int nid = 425984;
    int* ids;
    unsigned* bits;
    CK(cudaMalloc(&ids, nid * 4));
    CK(cudaMalloc(&bits, (33762577 / 32 + 1) * 4));
    {
      std::vector<int> h(nid);
      for (int i = 0; i < nid; ++i) h[i] = (int)(g() % 33762577);
      CK(cudaMemcpy(ids, h.data(), nid * 4, cudaMemcpyHostToDevice));
    }
    auto E = [=](cudaStream_t s) {
      for (int k = 0; k < 17; ++k) tiny_step<<<1, 32, 0, s>>>(cc, k);
    };
    auto W = [=](cudaStream_t s) {
      for (int k = 0; k < 17; ++k) wide_step<<<148 * 8, 256, 0, s>>>(ids, bits, nid);
    };
    auto T40 = [=](cudaStream_t s) {
      tma_gather<4><<<40, 32, 4 * 32 * 512, s>>>((const char*)hostd, (char*)zdst, didx, rows);
    };
    auto T148 = [=](cudaStream_t s) {
      tma_gather<4><<<148, 32, 4 * 32 * 512, s>>>((const char*)hostd, (char*)zdst, didx, rows);
    };
    alone("E 17 tiny kernels", E);
    alone("W 17 wide kernels", W);
    alone("T(40)", T40);
    both("E + T(40)", E, T40);
    both("W + T(40)", W, T40);
    both("E + T(148)", E, T148);
    both("E + Z(148)", E, [&](cudaStream_t s) { Z(s, 148); });
    both("E + DH", E, DH);
    both("E + DD", E, DD);
    both("W + DH", W, DH);
    return 0;
  }
  const float tH = alone("H  hbm copy 2x1GiB", H);
  printf("   -> %.0f GB/s\n", 2.0 * nH * 16 / tH / 1e6);
  const float tZ = alone("Z  zc gather grid 148", [&](cudaStream_t s) { Z(s, 148); });
  printf("   -> %.1f GB/s\n", rows * 512.0 / tZ / 1e6);
  alone("Z  zc gather grid 592", [&](cudaStream_t s) { Z(s, 592); });
  alone("ZS zc gather grid 32", [&](cudaStream_t s) { Z(s, 32); });
  alone("DH memcpy H2D 34.5MB", DH);
  alone("DD memcpy D2H 34.5MB", DD);

  const int cfgs[][3] = {{64, 512, 8}, {148, 256, 8}};
  for (auto& c : cfgs) {
    char nm[64];
    snprintf(nm, sizeof nm, "Z grid %d x %d unroll %d", c[0], c[1], c[2]);
    const float t = alone(nm, ZC(c[0], c[1], c[2]));
    printf("   -> %.1f GB/s\n", rows * 512.0 / t / 1e6);
    snprintf(nm, sizeof nm, "H + Z(%d x %d u%d)", c[0], c[1], c[2]);
    both(nm, H, ZC(c[0], c[1], c[2]));
  }
  CK(cudaFuncSetAttribute(tma_gather<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 32 * 512));
  {  // latency-bound gather (the cache's index/backward kernels) next to the host-link staging
    const int nL = 1 << 20, nrows = 1 << 21;  // 1M row gathers from a 1 GiB table
    int *la, *lb;
    CK(cudaMalloc(&la, nL * 4));
    CK(cudaMalloc(&lb, nrows * 4));
    std::vector<int> h1(nL), h2(nrows);
    for (int i = 0; i < nL; ++i) h1[i] = (int)(g() % nrows);
    for (int i = 0; i < nrows; ++i) h2[i] = (int)(g() % nrows);
    CK(cudaMemcpy(la, h1.data(), nL * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(lb, h2.data(), nrows * 4, cudaMemcpyHostToDevice));
    float4* lout;
    CK(cudaMalloc(&lout, (long)nL * 512));
    auto L = [=](cudaStream_t s) { dep_gather<<<148 * 8, 256, 0, s>>>(la, lb, ha, lout, nL, nrows); };
    const float tl = alone("L  dependent gather 1M rows", L);
    printf("   -> %.0f GB/s\n", nL * 512.0 * 2 / tl / 1e6);
    both("L + T(64)", L, [=](cudaStream_t s) {
      tma_gather<4><<<64, 32, 4 * 32 * 512, s>>>((const char*)hostd, (char*)zdst, didx, rows);
    });
    both("L + Z(148)", L, [&](cudaStream_t s) { Z(s, 148); });
    both("L + DH", L, DH);
    {  // green contexts: the staging on its own SMs, the compute on the rest
      CUdevice cdev;
      cuDeviceGet(&cdev, 0);
      CUdevResource all, part[1], rest;
      unsigned nb = 1;
      CUresult r = cuDeviceGetDevResource(cdev, &all, CU_DEV_RESOURCE_TYPE_SM);
      if (r == CUDA_SUCCESS) r = cuDevSmResourceSplitByCount(part, &nb, &all, &rest, 0, 16);
      CUdevResourceDesc d1, d2;
      CUgreenCtx g1, g2;
      CUstream gs1 = nullptr, gs2 = nullptr;
      if (r == CUDA_SUCCESS) r = cuDevResourceGenerateDesc(&d1, part, 1);
      if (r == CUDA_SUCCESS) r = cuDevResourceGenerateDesc(&d2, &rest, 1);
      if (r == CUDA_SUCCESS) r = cuGreenCtxCreate(&g1, d1, cdev, CU_GREEN_CTX_DEFAULT_STREAM);
      if (r == CUDA_SUCCESS) r = cuGreenCtxCreate(&g2, d2, cdev, CU_GREEN_CTX_DEFAULT_STREAM);
      if (r == CUDA_SUCCESS) r = cuGreenCtxStreamCreate(&gs1, g1, CU_STREAM_NON_BLOCKING, 0);
      if (r == CUDA_SUCCESS) r = cuGreenCtxStreamCreate(&gs2, g2, CU_STREAM_NON_BLOCKING, 0);
      printf("green ctx setup: %d (staging SMs %u, compute SMs %u)\n", (int)r, part[0].sm.smCount, rest.sm.smCount);
      if (r == CUDA_SUCCESS) {
        cudaStream_t ts = (cudaStream_t)gs1, cs = (cudaStream_t)gs2;
        auto run = [&](bool withT, bool withL) {
          cudaEvent_t a, b, c, d;
          cudaEventCreate(&a); cudaEventCreate(&b); cudaEventCreate(&c); cudaEventCreate(&d);
          float bl = 1e9, bt = 1e9;
          for (int rep = 0; rep < 5; ++rep) {
            cudaDeviceSynchronize();
            cudaEventRecord(a, cs);
            cudaEventRecord(c, ts);
            if (withL) dep_gather<<<148 * 8, 256, 0, cs>>>(la, lb, ha, lout, nL, nrows);
            if (withT) tma_gather<4><<<64, 32, 4 * 32 * 512, ts>>>((const char*)hostd, (char*)zdst, didx, rows);
            cudaEventRecord(b, cs);
            cudaEventRecord(d, ts);
            cudaDeviceSynchronize();
            float x, y;
            cudaEventElapsedTime(&x, a, b);
            cudaEventElapsedTime(&y, c, d);
            bl = std::min(bl, x);
            bt = std::min(bt, y);
          }
          printf("green: L %s T %s -> L %.3f ms | T %.3f ms (err %s)\n", withL ? "on" : "off", withT ? "on" : "off", bl, bt,
                 cudaGetErrorString(cudaGetLastError()));
        };
        run(false, true);
        run(true, false);
        run(true, true);
      }
    }
    both("L + DD", L, DD);
  }
  for (int grid : {16, 32, 64, 148}) {
    auto T = [=](cudaStream_t s) {
      tma_gather<4><<<grid, 32, 4 * 32 * 512, s>>>((const char*)hostd, (char*)zdst, didx, rows);
    };
    char nm[64];
    snprintf(nm, sizeof nm, "T tma gather grid %d", grid);
    const float t = alone(nm, T);
    CK(cudaGetLastError());
    printf("   -> %.1f GB/s\n", rows * 512.0 / t / 1e6);
    snprintf(nm, sizeof nm, "H + T(%d)", grid);
    both(nm, H, T);
  }
  {  // correctness of the TMA gather against the zero-copy one
    std::vector<float> a((long)rows * 128), b((long)rows * 128);
    Z(s1, 148);
    CK(cudaStreamSynchronize(s1));
    CK(cudaMemcpy(a.data(), zdst, (long)rows * 512, cudaMemcpyDeviceToHost));
    CK(cudaMemset(zdst, 0, (long)rows * 512));
    tma_gather<4><<<64, 32, 4 * 32 * 512, s1>>>((const char*)hostd, (char*)zdst, didx, rows);
    CK(cudaStreamSynchronize(s1));
    CK(cudaMemcpy(b.data(), zdst, (long)rows * 512, cudaMemcpyDeviceToHost));
    printf("TMA gather == zero-copy gather: %s\n", a == b ? "yes" : "NO");
  }
  both("H + Z(148)", H, [&](cudaStream_t s) { Z(s, 148); });
  both("H + Z(32)", H, [&](cudaStream_t s) { Z(s, 32); });
  both("H + DH", H, DH);
  both("H + DD", H, DD);

  both("Z(148) + DD", [&](cudaStream_t s) { Z(s, 148); }, DD);

  return 0;
}
