// Development aid: per-SM cp.async.bulk streaming throughput (global -> smem)
// with S stages of `bytes` each, all 148 SMs streaming concurrently, source
// either L2-resident (small buffer re-read) or HBM (large buffer). Mirrors the
// conv kernel's B-operand stream (32 KB per K block at BN=128).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "ptx.cuh"

using namespace tobf;

__global__ void __launch_bounds__(32, 1) stream(const uint8_t* src, size_t src_bytes, int stages, int bytes,
                                               int iters, unsigned long long* cyc, int parts) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t full[8];
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) mbar_init(&full[s], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  const size_t nchunks = src_bytes / bytes;
  size_t chunk = (size_t)blockIdx.x * 7919 % nchunks;
  const long long t0 = clock64();
  const int pb = bytes / parts;
  for (int s = 0; s < stages && s < iters; ++s) {
    mbar_arrive_expect_tx(&full[s], bytes);
    for (int q = 0; q < parts; ++q) bulk_g2s(smem + s * bytes + q * pb, src + chunk * bytes + q * pb, pb, &full[s]);
    chunk = (chunk + 148) % nchunks;
  }
  for (int i = 0; i < iters; ++i) {
    const int s = i % stages;
    mbar_wait(&full[s], (i / stages) & 1, 1);
    const int nx = i + stages;
    if (nx < iters) {
      mbar_arrive_expect_tx(&full[s], bytes);
      for (int q = 0; q < parts; ++q) bulk_g2s(smem + s * bytes + q * pb, src + chunk * bytes + q * pb, pb, &full[s]);
      chunk = (chunk + 148) % nchunks;
    }
  }
  cyc[blockIdx.x] = clock64() - t0;
}

int main() {
  const size_t big = (size_t)4 << 30, small = (size_t)48 << 20;
  uint8_t* buf;
  cudaMalloc(&buf, big);
  cudaMemset(buf, 1, big);
  unsigned long long* cyc;
  cudaMalloc(&cyc, 148 * 8);
  cudaFuncSetAttribute(stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int src_big = 0; src_big < 2; ++src_big)
    for (int bytes : {16384, 32768, 65536})
      for (int parts : {1, 2, 4})
      for (int stages : {2, 3}) {
        if (stages * bytes > 196 * 1024) continue;
        const int iters = 2000;
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        stream<<<148, 32, 200 * 1024>>>(buf, src_big ? big : small, stages, bytes, 50, cyc, parts);
        cudaEventRecord(a);
        stream<<<148, 32, 200 * 1024>>>(buf, src_big ? big : small, stages, bytes, iters, cyc, parts);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        unsigned long long h[148];
        cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
        double avg = 0;
        for (int i = 0; i < 148; ++i) avg += h[i] / 148.0;
        const double tot = 148.0 * iters * bytes;
        printf("%s parts %d bytes %6d stages %d: %8.1f GB/s total, %6.1f B/clk/SM, %7.0f cycles/copy\n",
               src_big ? "HBM" : "L2 ", parts, bytes, stages, tot / (ms * 1e6), (double)iters * bytes / avg,
               avg / iters);
      }
  cudaError_t e = cudaDeviceSynchronize();
  printf("%s\n", cudaGetErrorString(e));
  return 0;
}
