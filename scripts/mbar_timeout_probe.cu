// Development aid: wall time of N mbarrier.try_wait expiries (suspend-time hint
// 0x989680) on a barrier that never completes, to size the bounded wait.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void probe(int tries, unsigned hint, unsigned long long* out) {
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) {
    uint32_t a = (uint32_t)__cvta_generic_to_shared(&bar);
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(a));
    asm volatile("fence.mbarrier_init.release.cluster;");
    unsigned long long t0, t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    int ok = 0;
    for (int i = 0; i < tries; ++i) {
      uint32_t p;
      asm volatile("{\n\t.reg .pred q;\n\tmbarrier.try_wait.parity.shared::cta.b64 q, [%1], %2, %3;\n\tselp.u32 %0,1,0,q;\n\t}"
                   : "=r"(p) : "r"(a), "r"(0u), "r"(hint) : "memory");
      ok |= p;
    }
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    out[0] = t1 - t0;
    out[1] = ok;
  }
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 16);
  unsigned hints[] = {0u, 1000u, 100000u, 0x989680u};
  for (unsigned h : hints) {
    for (int tries : {1, 16, 512}) {
      probe<<<1, 32>>>(tries, h, d);
      unsigned long long r[2];
      cudaMemcpy(r, d, 16, cudaMemcpyDeviceToHost);
      printf("hint %8u ns  tries %4d  total %10.3f us  per-try %8.3f us  completed=%llu  err=%s\n", h, tries,
             r[0] / 1e3, r[0] / 1e3 / tries, r[1], cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
