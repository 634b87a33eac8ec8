// Trace-feature kernels: the analytical cost model restated in fp64, bit-exact
// against the reference's Python arithmetic (compiled with -fmad=false: every
// formula is the same sequence of correctly rounded + - * / as CPython).
//
//   schedule_search_kernel  fusion.py:159-180 default_schedule — one CTA per
//                           kernel, lexicographic argmin of (cycles, ty, tx)
//                           over candidate_triples(H) x candidate_triples(W)
//                           (fusion.py:141-156), only `cycles` evaluated
//                           (costmodel.py:192-215)
//   profile_kernel_kernel   costmodel.py:166-232 profile_kernel — all 9 features
//   trace_total_kernel      costmodel.py:96-98 Trace.total_latency = CPython 3.12
//                           builtin sum() over floats (Neumaier compensation)
#include <cmath>
#include "tobf_internal.h"

namespace tobf {

// All factor triples over {1,2,4,8,16,32}^3 in lexicographic order, with
// their products: the candidate list for cap c is the subsequence with
// product <= c, still lexicographic (fusion.py:141-156).
__constant__ int8_t c_triples[216][3];
__constant__ int32_t c_tprod[216];

struct TripleTable {
  int8_t t[216][3];
  int32_t p[216];
};

static TripleTable make_table() {
  TripleTable tb{};
  const int f[6] = {1, 2, 4, 8, 16, 32};
  int n = 0;
  for (int a = 0; a < 6; ++a)
    for (int b = 0; b < 6; ++b)
      for (int c = 0; c < 6; ++c) {
        tb.t[n][0] = (int8_t)f[a];
        tb.t[n][1] = (int8_t)f[b];
        tb.t[n][2] = (int8_t)f[c];
        tb.p[n] = f[a] * f[b] * f[c];
        ++n;
      }
  return tb;
}

__host__ __device__ inline int64_t pow2_ceil(int64_t n) {
  int64_t v = 1;
  while (v < n) v <<= 1;  // 1 << bit_length(n-1), and 1 for n <= 1
  return v;
}

__host__ __device__ inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

struct ProfC {
  int64_t P, L, l1, l2, sm;
};

__device__ inline int64_t tile_footprint(const tobf_kern_desc& k, int64_t ey, int64_t ex) {
  // costmodel.py:150-163 (k1==k2==window for MaxPool, w_tile 0)
  const int64_t s = k.s;
  const int64_t in_tile = (ey * s + k.k1 - s) * (ex * s + k.k2 - s) * (int64_t)k.c;
  const int64_t w_tile = k.is_conv ? (int64_t)k.k1 * k.k2 * k.c : 0;
  return 4 * (ey * ex + in_tile + w_tile);
}

struct TiledTerms {
  int64_t fp_inner, fp_full, reuse_w, reuse_x;
  double eff;
};

__device__ inline TiledTerms tiled_terms(const tobf_kern_desc& k, const int* ty, const int* tx, int unroll,
                                         const ProfC& pr) {
  TiledTerms r;
  const int64_t inner_y = (int64_t)ty[1] * ty[2], inner_x = (int64_t)tx[1] * tx[2];
  const int64_t full_y = (int64_t)ty[0] * inner_y, full_x = (int64_t)tx[0] * inner_x;
  r.fp_inner = tile_footprint(k, inner_y, inner_x);
  r.fp_full = tile_footprint(k, full_y, full_x);
  const int64_t blocks = ceil_div(k.H, full_y) * ceil_div(k.W, full_x);
  // occupancy = min(1.0, blocks / sm_count): int/int true division
  double occ = (double)blocks / (double)pr.sm;
  if (!(occ < 1.0)) occ = 1.0;
  const int64_t fl1 = r.fp_full < pr.l1 ? r.fp_full : pr.l1;
  double eff = ((double)fl1 / (double)pr.l1) * occ;
  const double boost = 0.92 + 0.02 * (double)unroll;
  eff = eff * boost;
  if (!(eff < 1.0)) eff = 1.0;                  // min(1.0, ...)
  const double floor_ = 1.0 / 256.0;
  if (eff < floor_) eff = floor_;               // max(eff, floor)
  r.eff = eff;
  r.reuse_w = ceil_div(k.H, inner_y) * ceil_div(k.W, inner_x);
  r.reuse_x = ceil_div(k.channel_like, inner_y);
  return r;
}

__device__ inline double cycles_of(const tobf_kern_desc& k, double eff, const ProfC& pr) {
  // work / (P * eff) + fused_work / P + launch_overhead, left to right
  const double a = (double)k.work / ((double)pr.P * eff);
  const double b = (double)k.fused_work / (double)pr.P;
  return (a + b) + (double)pr.L;
}

__device__ inline bool key_less(double c, int i, double bc, int bi) {
  return c < bc || (c == bc && i < bi);
}

__global__ void schedule_search_kernel(tobf_kern_desc* __restrict__ descs, ProfC pr) {
  tobf_kern_desc& k = descs[blockIdx.x];
  __shared__ double s_c[256];
  __shared__ int s_i[256];
  const int64_t capy = pow2_ceil(k.H), capx = pow2_ceil(k.W);
  // candidate index lists: positions in the 216 table with product <= cap
  __shared__ uint8_t ly[216], lx[216];
  __shared__ int s_ny, s_nx;
  if (threadIdx.x == 0) {
    int ny = 0, nx = 0;
    for (int t = 0; t < 216; ++t) {
      if (c_tprod[t] <= capy) ly[ny++] = (uint8_t)t;
      if (c_tprod[t] <= capx) lx[nx++] = (uint8_t)t;
    }
    s_ny = ny;
    s_nx = nx;
  }
  __syncthreads();
  const int ny = s_ny, nx = s_nx;
  double best_c = INFINITY;
  int best_i = 0x7fffffff;
  if (k.resolved) return;  // memo hit: schedule already in the table
  if (!k.has_shape || k.label < 0) {
    // non-complex anchor -> TRIVIAL_SCHEDULE (fusion.py:168-170)
    if (threadIdx.x == 0) {
      for (int q = 0; q < 3; ++q) k.ty[q] = k.tx[q] = 1;
      k.unroll = 4;
    }
    return;
  }
  for (int i = threadIdx.x; i < ny * nx; i += blockDim.x) {
    const int iy = i / nx, ix = i - iy * nx;
    int ty[3], tx[3];
    for (int q = 0; q < 3; ++q) {
      ty[q] = c_triples[ly[iy]][q];
      tx[q] = c_triples[lx[ix]][q];
    }
    double eff = 1.0;
    if (k.tiled) eff = tiled_terms(k, ty, tx, 4, pr).eff;
    const double c = cycles_of(k, eff, pr);
    if (key_less(c, i, best_c, best_i)) {
      best_c = c;
      best_i = i;
    }
  }
  s_c[threadIdx.x] = best_c;
  s_i[threadIdx.x] = best_i;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) {
      const double oc = s_c[threadIdx.x + w];
      const int oi = s_i[threadIdx.x + w];
      if (key_less(oc, oi, s_c[threadIdx.x], s_i[threadIdx.x])) {
        s_c[threadIdx.x] = oc;
        s_i[threadIdx.x] = oi;
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const int i = s_i[0];
    const int iy = i / nx, ix = i - iy * nx;
    for (int q = 0; q < 3; ++q) {
      k.ty[q] = c_triples[ly[iy]][q];
      k.tx[q] = c_triples[lx[ix]][q];
    }
    k.unroll = 4;
  }
}

// fusion.py:105-121: strategy k forces slot k of a triple to 1 and keeps the
// product as the most balanced factor pair, smaller factor first.
__device__ inline void apply_strategy(int* t, int k) {
  const int prod = t[0] * t[1] * t[2];
  int a = 1;
  for (int d = 1; d * d <= prod; ++d)
    if (prod % d == 0) a = d;
  const int b = prod / a;
  int r0 = -1, r1 = -1;
  for (int i = 0; i < 3; ++i) {
    if (i == k - 1) continue;
    if (r0 < 0) r0 = i; else r1 = i;
  }
  t[k - 1] = 1;
  t[r0] = a;
  t[r1] = b;
}

__global__ void resolve_kernel(tobf_kern_desc* __restrict__ kern, int n, const tobf_kern_desc* __restrict__ sigs) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  tobf_kern_desc& k = kern[i];
  if (k.sig_index < 0) return;
  const tobf_kern_desc& s = sigs[k.sig_index];
  int ty[3] = {s.ty[0], s.ty[1], s.ty[2]}, tx[3] = {s.tx[0], s.tx[1], s.tx[2]};
  if (k.strategy >= 1 && k.strategy <= 3) {
    apply_strategy(ty, k.strategy);
    apply_strategy(tx, k.strategy);
  }
  for (int q = 0; q < 3; ++q) {
    k.ty[q] = ty[q];
    k.tx[q] = tx[q];
  }
  k.unroll = s.unroll;
}

__device__ inline double pct_hit(int64_t fp, int64_t working_set) {
  // float(np.clip(100.0 * (1.0 - fp / working_set), 5.0, 99.0))
  const double r = (double)fp / (double)working_set;
  double v = 100.0 * (1.0 - r);
  if (v < 5.0) v = 5.0;
  if (v > 99.0) v = 99.0;
  return v;
}

__global__ void profile_kernel_kernel(const tobf_kern_desc* __restrict__ descs, int n, ProfC pr,
                                      double* __restrict__ feats) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const tobf_kern_desc k = descs[i];
  double* f = feats + (int64_t)i * 9;
  if (!k.has_shape) {
    for (int q = 0; q < 9; ++q) f[q] = 0.0;
    return;
  }
  const int64_t working_set = k.in_bytes + k.w_bytes + k.out_bytes + k.fused_bytes;
  int64_t fp_inner, fp_full, reuse_w, reuse_x;
  double eff;
  if (k.tiled) {
    const TiledTerms t = tiled_terms(k, k.ty, k.tx, k.unroll, pr);
    fp_inner = t.fp_inner;
    fp_full = t.fp_full;
    reuse_w = t.reuse_w;
    reuse_x = t.reuse_x;
    eff = t.eff;
  } else {
    fp_inner = fp_full = working_set < 8192 ? working_set : 8192;  // _STREAM_FP
    eff = 1.0;
    reuse_w = 1;
    reuse_x = k.reuse_x_stream;
  }
  const int64_t read = k.w_bytes * reuse_w + k.in_bytes * reuse_x + k.fused_bytes;
  const int64_t write = k.out_bytes;
  f[0] = cycles_of(k, eff, pr);
  f[1] = (double)read;
  f[2] = (double)write;
  f[3] = (double)read / 32.0;
  f[4] = 100.0 * eff;
  f[5] = pct_hit(fp_inner, working_set);
  f[6] = (double)(read + write) / 32.0;
  const int64_t fl2 = fp_full < pr.l2 ? fp_full : pr.l2;
  f[7] = (100.0 * (double)fl2) / (double)pr.l2;
  f[8] = pct_hit(fp_full, working_set);
}

// CPython 3.12 builtin sum() over a float sequence (Objects/bltinmodule.c
// builtin_sum_impl): Neumaier-compensated, compensation added at the end only
// when non-zero and finite. One thread per candidate (traces are short).
__global__ void trace_total_kernel(const double* __restrict__ feats, const int32_t* __restrict__ offsets,
                                   int ncand, double* __restrict__ totals) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= ncand) return;
  double s = 0.0, comp = 0.0;
  for (int i = offsets[c]; i < offsets[c + 1]; ++i) {
    const double x = feats[(int64_t)i * 9];
    const double t = s + x;
    if (fabs(s) >= fabs(x)) comp += (s - t) + x;
    else comp += (x - t) + s;
    s = t;
  }
  if (comp != 0.0 && isfinite(comp)) s += comp;
  totals[c] = s;
}

static int ensure_tables() {
  static bool done = false;
  if (done) return TOBF_OK;
  const TripleTable tb = make_table();
  cudaError_t e = cudaMemcpyToSymbol(c_triples, tb.t, sizeof(tb.t));
  if (e == cudaSuccess) e = cudaMemcpyToSymbol(c_tprod, tb.p, sizeof(tb.p));
  if (e != cudaSuccess) return tobf_fail(TOBF_E_CUDA, "trace tables: %s", cudaGetErrorString(e));
  done = true;
  return TOBF_OK;
}

static ProfC to_profc(const tobf_device_profile* p) {
  return ProfC{p->macs_per_cycle, p->launch_overhead, p->l1_bytes, p->l2_bytes, p->sm_count};
}

}  // namespace tobf

using namespace tobf;

extern "C" int tobf_schedule_search(tobf_kern_desc* d_descs, int n, const tobf_device_profile* prof,
                                    void* stream) {
  if (n <= 0) return TOBF_OK;
  if (!d_descs || !prof || prof->macs_per_cycle <= 0 || prof->l1_bytes <= 0 || prof->l2_bytes <= 0 ||
      prof->sm_count <= 0)
    return tobf_fail(TOBF_E_INVALID, "tobf_schedule_search: bad arguments");
  int rc = ensure_tables();
  if (rc) return rc;
  schedule_search_kernel<<<n, 256, 0, (cudaStream_t)stream>>>(d_descs, to_profc(prof));
  return tobf_cuda_check("tobf_schedule_search");
}

extern "C" int tobf_resolve_schedules(tobf_kern_desc* d_kern, int n, const tobf_kern_desc* d_sigs, void* stream) {
  if (n <= 0) return TOBF_OK;
  if (!d_kern || !d_sigs) return tobf_fail(TOBF_E_INVALID, "tobf_resolve_schedules: bad arguments");
  resolve_kernel<<<(n + 127) / 128, 128, 0, (cudaStream_t)stream>>>(d_kern, n, d_sigs);
  return tobf_cuda_check("tobf_resolve_schedules");
}

extern "C" int tobf_profile_kernels(const tobf_kern_desc* d_descs, int n, const tobf_device_profile* prof,
                                    double* feats, void* stream) {
  if (n <= 0) return TOBF_OK;
  if (!d_descs || !prof || !feats) return tobf_fail(TOBF_E_INVALID, "tobf_profile_kernels: bad arguments");
  profile_kernel_kernel<<<(n + 127) / 128, 128, 0, (cudaStream_t)stream>>>(d_descs, n, to_profc(prof), feats);
  return tobf_cuda_check("tobf_profile_kernels");
}

extern "C" int tobf_trace_totals(const double* feats, const int32_t* offsets, int ncand, double* totals,
                                 void* stream) {
  if (ncand <= 0) return TOBF_OK;
  if (!feats || !offsets || !totals) return tobf_fail(TOBF_E_INVALID, "tobf_trace_totals: bad arguments");
  trace_total_kernel<<<(ncand + 127) / 128, 128, 0, (cudaStream_t)stream>>>(feats, offsets, ncand, totals);
  return tobf_cuda_check("tobf_trace_totals");
}
