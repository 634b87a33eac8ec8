// Development aid: tcgen05.mma.cta_group::2 (M=256 across a CTA pair) tf32
// throughput with A from TMEM, vs cta_group::1 M=128, per N. One cluster of 2
// CTAs per SM pair, 148 CTAs.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "ptx.cuh"
using namespace tobf;

__device__ __forceinline__ uint32_t cta_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

template <int N>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) probe2(int reps, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  for (int i = threadIdx.x; i < (2 * N * 128) / 4; i += 128) reinterpret_cast<float*>(smem)[i] = 0.f;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tslot)),
                 "r"(512) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  const uint32_t tb = tslot;
  if (cta_rank() == 0 && threadIdx.x == 0) {
    const uint32_t b = smem_u32(smem);
    constexpr uint32_t idesc = idesc_make(2u, 256, N);
    const long long t0 = clock64();
    for (int r = 0; r < reps; ++r)
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 1, 0;\n\t"
            "tcgen05.mma.cta_group::2.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tb),
            "r"(tb + 256 + kk * 8), "l"(sdesc_k128(b + kk * 32)), "r"(idesc)
            : "memory");
      }
    asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                 ::"r"(smem_u32(&bar)), "h"((uint16_t)1) : "memory");
    mbar_wait(&bar, 0, 1);
    const long long t1 = clock64();
    if (blockIdx.x == 0) out[0] = (unsigned long long)(t1 - t0);
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  tc_fence_after();
  if (threadIdx.x < 32)
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tb), "r"(512) : "memory");
}

template <int N>
void run() {
  unsigned long long* d;
  cudaMalloc(&d, 8);
  const int smem = 2 * N * 128 + 2048;
  cudaFuncSetAttribute(probe2<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int reps = 2048;
  probe2<N><<<148, 128, smem>>>(64, d);
  cudaError_t e = cudaDeviceSynchronize();
  probe2<N><<<148, 128, smem>>>(reps, d);
  e = cudaDeviceSynchronize();
  unsigned long long c = 0;
  cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
  const double per = (double)c / (reps * 4);
  const double macs_per_sm = 128.0 * N * 8;  // each SM of the pair does 128 rows
  printf("cta_group::2 tf32 TS M=256 N=%3d: %7.1f cycles/MMA  %7.0f MAC/clk/SM  err=%s\n", N, per,
         macs_per_sm / per, cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  run<64>();
  run<128>();
  run<256>();
  return 0;
}
