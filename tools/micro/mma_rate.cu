// Microbenchmark: tcgen05.mma kind::f16 issue throughput vs N (operands resident
// in smem, no TMA), one CTA per SM, cta_group::1 (M=128) or ::2 (M=256 pairs).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma_rate mma_rate.cu && ./mma_rate
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t a, uint32_t lbo, uint32_t sbo) {
  uint64_t d = (uint64_t)((a >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= 1ull << 46;
  d |= 2ull << 61;
  return d;
}
__device__ __forceinline__ void wait_bar(uint32_t bar, uint32_t ph) {
  uint32_t ok = 0;
  do {
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(ok) : "r"(bar), "r"(ph) : "memory");
  } while (!ok);
}

template <bool kPair>
__global__ void __launch_bounds__(128, 1) k(int n, int iters, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* s = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x / 32;
  uint32_t rank = 0;
  if (kPair) asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) ((uint32_t*)s)[i] = 0;
  if (warp == 0) {
    if (kPair) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 256;" :: "r"(su32(&tslot)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" :: "r"(su32(&tslot)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  if (kPair) asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  else __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = tslot;
  const uint32_t M = kPair ? 256 : 128;
  const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((M >> 4) << 24);
  if (threadIdx.x == 0 && rank == 0) {
    const uint32_t a = su32(s), b = su32(s + 16384);
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        uint64_t ad = sdesc(a + kk * 32, 16, 1024), bd = sdesc(b + kk * 32, 16, 1024);
        uint32_t acc = (it | kk) ? 1 : 0;
        if (kPair)
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" :: "r"(tm), "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
        else
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" :: "r"(tm), "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
      }
    }
    if (kPair)
      asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" :: "r"(su32(&bar)), "h"((uint16_t)3) : "memory");
    else
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(su32(&bar)) : "memory");
    wait_bar(su32(&bar), 0);
    long long t1 = clock64();
    out[blockIdx.x] = t1 - t0;
  }
  if (kPair && threadIdx.x == 0 && rank == 1) wait_bar(su32(&bar), 0);
  asm volatile("tcgen05.fence::before_thread_sync;");
  if (kPair) asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  else __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (kPair) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 256;" :: "r"(tm));
    else asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" :: "r"(tm));
  }
}

int main() {
  long long* d;
  cudaMalloc(&d, 148 * sizeof(long long));
  long long h[148];
  const int iters = 2000;
  const int smem = 65536 + 1024;
  cudaFuncSetAttribute(k<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  int ns[] = {32, 64, 96, 112, 128, 160, 192, 224, 256};
  for (int pair = 0; pair < 2; ++pair) {
    for (int n : ns) {
      cudaMemset(d, 0, sizeof(h));
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(148);
      cfg.blockDim = dim3(128);
      cfg.dynamicSmemBytes = smem;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = 2; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = pair ? 1 : 0;
      cudaError_t e = pair ? cudaLaunchKernelEx(&cfg, k<true>, n, iters, d) : cudaLaunchKernelEx(&cfg, k<false>, n, iters, d);
      if (e != cudaSuccess || cudaDeviceSynchronize() != cudaSuccess) { printf("error %s\n", cudaGetErrorString(cudaGetLastError())); return 1; }
      cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
      double mx = 0, sum = 0; int c = 0;
      for (int i = 0; i < 148; ++i) if (h[i]) { mx = h[i] > mx ? h[i] : mx; sum += h[i]; ++c; }
      const double per_mma = sum / c / (iters * 4.0);
      const double M = pair ? 256 : 128;
      const double flop_per_sm_clk = M * n * 16 * 2 / per_mma / (pair ? 2 : 1);
      printf("%s N=%3d  cycles/MMA %.1f  FLOP/clk/SM %.0f\n", pair ? "pair M=256" : "1sm  M=128", n, per_mma, flop_per_sm_clk);
    }
  }
  return 0;
}
