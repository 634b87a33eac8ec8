// Development aid: how tcgen05.mma kind::tf32 reads fp32 operand bits.
// One 128x64x8 MMA, A from TMEM (the conv's TS form): A[m][0] = 1 + m*2^-17
// (fractions of a tf32 ulp), B[0][0] = 1, B[1][0] = 1 + 3*2^-12 (SMEM),
// everything else 0. D[m][0] shows what the tensor core made of A[m][0],
// D[0][1] what it made of B[1][0]: truncation (low 13 bits ignored),
// round-to-nearest, or the full fp32 value.
// nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -Ipaper_2107_09789_b200/csrc scripts/tf32_trunc_probe.cu
#include <cmath>
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <cuda_runtime.h>
#include "ptx.cuh"
using namespace tobf;

__global__ void __launch_bounds__(128, 1) probe(float* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int t = threadIdx.x, warp = t >> 5;
  for (int i = t; i < 64 * 32; i += 128) reinterpret_cast<float*>(smem)[i] = 0.f;
  __syncthreads();
  if (t == 0) {
    *reinterpret_cast<float*>(smem + sw128_off(0, 0)) = 1.0f;                    // B[k=0][n=0]
    *reinterpret_cast<float*>(smem + sw128_off(1, 0)) = 1.0f + 3.0f / 4096.0f;   // B[k=0][n=1]
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  fence_proxy_async_smem();
  if (warp == 0) tmem_alloc(&tslot, 128);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tb = tslot;
  float a[16];
  for (int i = 0; i < 16; ++i) a[i] = 0.f;
  a[0] = 1.0f + (float)t * ldexpf(1.0f, -17);
  tmem_st16(tb + (static_cast<uint32_t>(warp * 32) << 16) + 64, a);
  tmem_wait_st();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (t == 0) {
    mma_tf32_ts(tb, tb + 64, sdesc_k128(smem_u32(smem)), idesc_make(2u, 128, 64), 0u);
    mma_commit(&bar);
  }
  mbar_wait(&bar, 0, 0x7ff);
  tc_fence_after();
  float d[16];
  tmem_ld16(tb + (static_cast<uint32_t>(warp * 32) << 16), d);
  out[t] = d[0];
  out[128 + t] = d[1];
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tb, 128);
}

static float tf32_trunc(float x) { uint32_t u; memcpy(&u, &x, 4); u &= 0xFFFFE000u; memcpy(&x, &u, 4); return x; }
static float tf32_rna(float x) { uint32_t u; memcpy(&u, &x, 4); u = (u + 0x1000u) & 0xFFFFE000u; memcpy(&x, &u, 4); return x; }
static float tf32_rne(float x) {
  uint32_t u; memcpy(&u, &x, 4);
  u = (u + 0xFFFu + ((u >> 13) & 1u)) & 0xFFFFE000u; memcpy(&x, &u, 4); return x;
}

int main() {
  float* d_out;
  cudaMalloc(&d_out, 256 * sizeof(float));
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384);
  probe<<<1, 128, 16384>>>(d_out);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
  float h[256];
  cudaMemcpy(h, d_out, sizeof h, cudaMemcpyDeviceToHost);
  int n_trunc = 0, n_rna = 0, n_rne = 0, n_full = 0;
  for (int m = 0; m < 128; ++m) {
    const float a = 1.0f + (float)m * ldexpf(1.0f, -17);
    n_trunc += h[m] == tf32_trunc(a);
    n_rna += h[m] == tf32_rna(a);
    n_rne += h[m] == tf32_rne(a);
    n_full += h[m] == a;
    if (m % 16 == 0 || m == 63 || m == 64 || m == 65) printf("A m=%3d a=%.9f hw=%.9f trunc=%.9f rna=%.9f\n", m, a, h[m], tf32_trunc(a), tf32_rna(a));
  }
  printf("A (TMEM): matches trunc %d rna %d rne %d full %d of 128\n", n_trunc, n_rna, n_rne, n_full);
  const float b = 1.0f + 3.0f / 4096.0f;
  printf("B (SMEM): b=%.9f hw=%.9f trunc=%.9f rna=%.9f\n", b, h[128], tf32_trunc(b), tf32_rna(b));
  return 0;
}
