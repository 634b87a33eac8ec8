// Development aid: effective SM clock inside a kernel = clock64 delta /
// globaltimer delta, for an FMA-bound spin and for a tcgen05-MMA-bound spin.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "ptx.cuh"
using namespace tobf;

__global__ void spin_fma(int iters, unsigned long long* out) {
  float a = threadIdx.x, b = 1.0001f;
  const long long c0 = clock64();
  const unsigned long long g0 = globaltimer_ns();
  for (int i = 0; i < iters; ++i) { a = fmaf(a, b, 0.5f); b = fmaf(b, a, -0.25f); }
  const long long c1 = clock64();
  const unsigned long long g1 = globaltimer_ns();
  if (threadIdx.x == 0) { out[2 * blockIdx.x] = c1 - c0; out[2 * blockIdx.x + 1] = g1 - g0; }
  if (a == 12345.f) out[0] = 0;
}

__global__ void __launch_bounds__(128, 1) spin_mma(int reps, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  for (int i = threadIdx.x; i < (16384 + 2 * 128 * 128) / 4; i += 128) reinterpret_cast<float*>(smem)[i] = 0.f;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  if (threadIdx.x < 32) tmem_alloc(&tslot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tb = tslot;
  if (threadIdx.x == 0) {
    const uint32_t b = smem_u32(smem) + 16384;
    constexpr uint32_t idesc = idesc_make(2u, 128, 128);
    const long long c0 = clock64();
    const unsigned long long g0 = globaltimer_ns();
    for (int r = 0; r < reps; ++r)
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) mma_tf32_ts(tb, tb + 256 + kk * 8, sdesc_k128(b + kk * 32), idesc, 1u);
    mma_commit(&bar);
    mbar_wait(&bar, 0, 1);
    const long long c1 = clock64();
    const unsigned long long g1 = globaltimer_ns();
    out[2 * blockIdx.x] = c1 - c0;
    out[2 * blockIdx.x + 1] = g1 - g0;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x < 32) tmem_dealloc(tb, 512);
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 148 * 16);
  unsigned long long h[296];
  for (int rep = 0; rep < 3; ++rep) {
    spin_fma<<<148 * 4, 256>>>(2000000, d);
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    printf("fma spin: clock64/globaltimer = %.0f MHz (%.2f ms)\n", 1e3 * (double)h[0] / h[1], h[1] / 1e6);
  }
  const int smem = 16384 + 2 * 128 * 128 + 2048;
  cudaFuncSetAttribute(spin_mma, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int rep = 0; rep < 4; ++rep) {
    spin_mma<<<148, 128, smem>>>(20000, d);
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    double cyc = h[0], ns = h[1];
    printf("tf32 MMA spin (148 SMs): clock64/globaltimer = %.0f MHz, %.1f cycles/MMA, %.2f ms\n", 1e3 * cyc / ns,
           cyc / (20000.0 * 4), ns / 1e6);
  }
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
