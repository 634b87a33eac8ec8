// Development aid: tcgen05.mma issue-to-retire throughput per shape/kind on
// one SM (148 CTAs run concurrently, one per SM), cycles per MMA instruction.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "ptx.cuh"

using namespace tobf;

template <int N, int MODE>  // MODE 0: tf32 SS, 1: tf32 TS (A in TMEM), 2: bf16 SS
__global__ void __launch_bounds__(128, 1) probe(int reps, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  for (int i = threadIdx.x; i < (16384 + 2 * N * 128) / 4; i += 128) reinterpret_cast<float*>(smem)[i] = 0.f;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  if (threadIdx.x < 32) tmem_alloc(&tslot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tb = tslot;
  if (threadIdx.x == 0) {
    const uint32_t a = smem_u32(smem), b = a + 16384;
    constexpr uint32_t idesc = idesc_make(MODE == 2 ? 1u : 2u, 128, N);
    const long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        const uint64_t db = sdesc_k128(b + kk * 32);
        if (MODE == 0) mma_tf32(tb, sdesc_k128(a + kk * 32), db, idesc, 1u);
        if (MODE == 1) mma_tf32_ts(tb, tb + 256 + kk * 8, db, idesc, 1u);
        if (MODE == 2) mma_bf16(tb, sdesc_k128(a + kk * 32), db, idesc, 1u);
        if (MODE == 3) {  // the conv kernel's 3xTF32 pattern: two accumulators, hi/lo A and B
          const uint64_t dbl = sdesc_k128(b + N * 128 / 2 + kk * 32);
          mma_tf32_ts(tb + N, tb + 256 + 32 + kk * 8, db, idesc, 1u);
          mma_tf32_ts(tb + N, tb + 256 + kk * 8, dbl, idesc, 1u);
          mma_tf32_ts(tb, tb + 256 + kk * 8, db, idesc, 1u);
        }
        if (MODE == 4) {  // same, smem A
          const uint64_t dbl = sdesc_k128(b + N * 128 / 2 + kk * 32);
          mma_tf32(tb + N, sdesc_k128(a + 8192 + kk * 32), db, idesc, 1u);
          mma_tf32(tb + N, sdesc_k128(a + kk * 32), dbl, idesc, 1u);
          mma_tf32(tb, sdesc_k128(a + kk * 32), db, idesc, 1u);
        }
      }
    }
    mma_commit(&bar);
    mbar_wait(&bar, 0, 1);
    const long long t1 = clock64();
    if (blockIdx.x == 0) out[0] = (unsigned long long)(t1 - t0);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x < 32) tmem_dealloc(tb, 512);
}

template <int N, int MODE>
void run(const char* name) {
  unsigned long long* d;
  cudaMalloc(&d, 8);
  const int smem = 16384 + 2 * N * 128 + 2048;
  cudaFuncSetAttribute(probe<N, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int reps = 2048;
  probe<N, MODE><<<148, 128, smem>>>(64, d);
  cudaDeviceSynchronize();
  probe<N, MODE><<<148, 128, smem>>>(reps, d);
  unsigned long long c = 0;
  cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
  const double per = (double)c / (reps * 4 * (MODE >= 3 ? 3 : 1));
  const double macs = 128.0 * N * (MODE == 2 ? 16 : 8);
  printf("%-10s M=128 N=%3d: %7.1f cycles/MMA  %7.0f MAC/clk/SM  err=%s\n", name, N, per, macs / per,
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

int main() {
  run<64, 0>("tf32 SS"); run<128, 0>("tf32 SS"); run<256, 0>("tf32 SS");
  run<64, 1>("tf32 TS"); run<128, 1>("tf32 TS"); run<256, 1>("tf32 TS");
  run<64, 2>("bf16 SS"); run<128, 2>("bf16 SS"); run<256, 2>("bf16 SS");
  run<64, 3>("3xTF32 TS"); run<128, 3>("3xTF32 TS");
  run<64, 4>("3xTF32 SS"); run<128, 4>("3xTF32 SS");
  return 0;
}
