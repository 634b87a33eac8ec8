// Fitness stage (no reference code exists — restated from PAPER.md:425-433,
// 458, 487, 623 and SPEC.md:471-486, 547-571; the CPU restatement lives in
// oracle/fitness_ref.c):
//   lstm_ctc_kernel    single-layer LSTM sequence predictor over the trace
//                      rows (log1p-normalised fp64 features -> fp32), linear
//                      head, greedy CTC decode (argmax, collapse repeats,
//                      drop blank 0). Fixed-order fmaf accumulation and the
//                      IEEE-only transcendental routines of detmath.h make the
//                      decoded tokens bit-exact against the CPU restatement.
//   levenshtein_kernel one warp per (prediction, truth) pair, anti-diagonal
//                      wavefront over 32-column strips of the truth.
//   eq10_kernel        R = mean(LER) / (eps + ((T - (1+B)T*)/T*)^2).
// Compiled with -fmad=false: every a*b+c that must match the CPU is an
// explicit fmaf, every other product/sum is separately rounded.
#include <cmath>
#include "detmath.h"
#include "tobf_internal.h"

namespace tobf {

constexpr int kMaxNC = 8;

// One CTA = TPC traces, blockDim = H threads (one per hidden unit).
// Weights: w_ihT [F][4H], w_hhT [H][4H] (gate-major columns i,f,g,o),
// bias [4H], w_out [NC][H], b_out [NC].
template <int TPC>
__global__ void lstm_ctc_kernel(const double* __restrict__ feats, const int32_t* __restrict__ offsets, int B, int F,
                                int H, int NC, const float* __restrict__ w_ihT, const float* __restrict__ w_hhT,
                                const float* __restrict__ bias, const float* __restrict__ w_out,
                                const float* __restrict__ b_out, int8_t* __restrict__ tokens, int T_max,
                                int32_t* __restrict__ ntok) {
  extern __shared__ float sh[];
  float* hbuf = sh;                          // [2][TPC][H]
  float* xbuf = hbuf + 2 * TPC * H;          // [TPC][16]
  float* lbuf = xbuf + TPC * 16;             // [TPC][kMaxNC]
  __shared__ int s_len[TPC], s_row0[TPC], s_prev[TPC], s_cnt[TPC];
  const int j = threadIdx.x;
  const int lane = j & 31, warp = j >> 5, nwarps = H >> 5;
  const int b0 = blockIdx.x * TPC;
  if (j < TPC) {
    const int b = b0 + j;
    s_len[j] = b < B ? offsets[b + 1] - offsets[b] : 0;
    s_row0[j] = b < B ? offsets[b] : 0;
    s_prev[j] = 0;
    s_cnt[j] = 0;
  }
  for (int i = j; i < 2 * TPC * H; i += H) hbuf[i] = 0.0f;
  __syncthreads();
  int tmax = 0;
  for (int q = 0; q < TPC; ++q) tmax = max(tmax, s_len[q]);
  float c[TPC];
#pragma unroll
  for (int q = 0; q < TPC; ++q) c[q] = 0.0f;
  const int G = 4 * H;
  for (int t = 0; t < tmax; ++t) {
    const float* hp = hbuf + (t & 1) * TPC * H;
    float* hn = hbuf + ((t + 1) & 1) * TPC * H;
    for (int idx = j; idx < TPC * F; idx += H) {
      const int q = idx / F, k = idx - q * F;
      xbuf[q * 16 + k] = t < s_len[q] ? (float)tobf_log1p_d(feats[(int64_t)(s_row0[q] + t) * 9 + k]) : 0.0f;
    }
    __syncthreads();
    float acc[4][TPC];
#pragma unroll
    for (int g = 0; g < 4; ++g) {
      const float bv = bias[g * H + j];
#pragma unroll
      for (int q = 0; q < TPC; ++q) acc[g][q] = bv;
    }
    for (int k = 0; k < F; ++k) {
      const float* wr = w_ihT + (int64_t)k * G + j;
      const float w0 = wr[0], w1 = wr[H], w2 = wr[2 * H], w3 = wr[3 * H];
#pragma unroll
      for (int q = 0; q < TPC; ++q) {
        const float xv = xbuf[q * 16 + k];
        acc[0][q] = fmaf(w0, xv, acc[0][q]);
        acc[1][q] = fmaf(w1, xv, acc[1][q]);
        acc[2][q] = fmaf(w2, xv, acc[2][q]);
        acc[3][q] = fmaf(w3, xv, acc[3][q]);
      }
    }
    for (int k = 0; k < H; ++k) {
      const float* wr = w_hhT + (int64_t)k * G + j;
      const float w0 = __ldg(wr), w1 = __ldg(wr + H), w2 = __ldg(wr + 2 * H), w3 = __ldg(wr + 3 * H);
#pragma unroll
      for (int q = 0; q < TPC; ++q) {
        const float hv = hp[q * H + k];
        acc[0][q] = fmaf(w0, hv, acc[0][q]);
        acc[1][q] = fmaf(w1, hv, acc[1][q]);
        acc[2][q] = fmaf(w2, hv, acc[2][q]);
        acc[3][q] = fmaf(w3, hv, acc[3][q]);
      }
    }
#pragma unroll
    for (int q = 0; q < TPC; ++q) {
      float hv = hp[q * H + j];
      if (t < s_len[q]) {
        const float ig = tobf_sigmoid(acc[0][q]);
        const float fg = tobf_sigmoid(acc[1][q]);
        const float gg = tobf_tanh(acc[2][q]);
        const float og = tobf_sigmoid(acc[3][q]);
        c[q] = fmaf(fg, c[q], ig * gg);
        hv = og * tobf_tanh(c[q]);
      }
      hn[q * H + j] = hv;
    }
    __syncthreads();
    // logits: warp w handles (trace, class) pairs w, w+nwarps, ...; lane-strided
    // fmaf partials then a fixed xor-butterfly (the order oracle/ restates).
    for (int pq = warp; pq < TPC * NC; pq += nwarps) {
      const int q = pq / NC, cls = pq - q * NC;
      float p = 0.0f;
      for (int k = lane; k < H; k += 32) p = fmaf(w_out[cls * H + k], hn[q * H + k], p);
      for (int off = 16; off; off >>= 1) p = p + __shfl_xor_sync(0xffffffffu, p, off);
      if (lane == 0) lbuf[q * kMaxNC + cls] = b_out[cls] + p;
    }
    __syncthreads();
    if (j < TPC && t < s_len[j] && b0 + j < B) {
      const float* lg = lbuf + j * kMaxNC;
      int best = 0;
      for (int cls = 1; cls < NC; ++cls)
        if (lg[cls] > lg[best]) best = cls;
      if (best != 0 && best != s_prev[j]) {
        tokens[(int64_t)(b0 + j) * T_max + s_cnt[j]] = (int8_t)best;
        s_cnt[j] += 1;
      }
      s_prev[j] = best;
    }
    // next iteration's first __syncthreads orders these smem updates
  }
  __syncthreads();
  if (j < TPC && b0 + j < B) ntok[b0 + j] = s_cnt[j];
}

// One warp per prediction; strips of 32 truth columns, anti-diagonal sweep.
__global__ void levenshtein_kernel(const int8_t* __restrict__ pred, const int32_t* __restrict__ ntok, int B,
                                   int T_max, const int8_t* __restrict__ truth, int m, int32_t* __restrict__ ed,
                                   double* __restrict__ ler, int colb_cap) {
  extern __shared__ int colb_all[];
  const int warps = blockDim.x >> 5;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int b = blockIdx.x * warps + w;
  if (b >= B) return;
  int* cola = colb_all + (2 * w) * colb_cap;      // boundary column read by lane 0
  int* colz = colb_all + (2 * w + 1) * colb_cap;  // boundary column written by the last lane
  const int n = ntok[b];
  const int8_t* p = pred + (int64_t)b * T_max;
  int result;
  if (m == 0) {
    result = n;
  } else if (n == 0) {
    result = m;
  } else {
    for (int i = lane; i <= n; i += 32) cola[i] = i;  // D[i][0]
    __syncwarp();
    int last = 0;
    for (int s0 = 0; s0 < m; s0 += 32) {
      const int jcol = s0 + lane + 1;  // 1-based truth column of this lane
      const bool active = jcol <= m;
      const int8_t tj = active ? truth[jcol - 1] : (int8_t)-1;
      int cur = jcol, old = jcol - 1;  // D[0][j], D[0][j-1] before row 1
      const int lastlane = min(31, m - 1 - s0);
      for (int st = 0; st < n + 32; ++st) {
        const int i = st - lane + 1;
        const int up_cur = __shfl_up_sync(0xffffffffu, cur, 1);  // D[i][j-1]
        const int up_old = __shfl_up_sync(0xffffffffu, old, 1);  // D[i-1][j-1]
        if (i >= 1 && i <= n && active) {
          const int left = lane == 0 ? cola[i] : up_cur;
          const int diag = lane == 0 ? cola[i - 1] : up_old;
          int v = cur + 1;
          v = min(v, left + 1);
          v = min(v, diag + (p[i - 1] != tj ? 1 : 0));
          old = cur;
          cur = v;
          if (lane == lastlane) colz[i] = v;
        } else if (i < 1) {
          old = cur;
        }
        __syncwarp();
      }
      if (lane == lastlane) {
        colz[0] = s0 + lastlane + 1;
        last = cur;
      }
      __syncwarp();
      int* tmp = cola;
      cola = colz;
      colz = tmp;
    }
    result = __shfl_sync(0xffffffffu, last, (m - 1) & 31);
  }
  if (lane == 0) {
    ed[b] = result;
    ler[b] = (double)result / (double)m;
  }
}

// CPython-3.12 float sum (Neumaier) of a short vector.
__device__ inline double py_sum(const double* v, int n, int stride) {
  double s = 0.0, comp = 0.0;
  for (int i = 0; i < n; ++i) {
    const double x = v[i * stride];
    const double t = s + x;
    if (fabs(s) >= fabs(x)) comp += (s - t) + x;
    else comp += (x - t) + s;
    s = t;
  }
  if (comp != 0.0 && isfinite(comp)) s += comp;
  return s;
}

__global__ void eq10_kernel(const double* __restrict__ ler, int npred, int ncand, const double* __restrict__ T,
                            const int32_t* __restrict__ feasible, double Tstar, double budget, double eps,
                            double* __restrict__ R, double* __restrict__ mean_ler) {
  const int cand = blockIdx.x * blockDim.x + threadIdx.x;
  if (cand >= ncand) return;
  const double mean = py_sum(ler + cand, npred, ncand) / (double)npred;
  mean_ler[cand] = mean;
  if (!feasible[cand]) {
    R[cand] = 0.0;
    return;
  }
  const double dev = (T[cand] - (1.0 + budget) * Tstar) / Tstar;
  R[cand] = mean / (eps + dev * dev);
}

}  // namespace tobf

using namespace tobf;

template <int TPC>
static int launch_lstm(const double* feats, const int32_t* offsets, int32_t B, int32_t F, int32_t H, int32_t NC,
                       const float* w_ihT, const float* w_hhT, const float* b, const float* w_out,
                       const float* b_out, int8_t* tokens, int32_t T_max, int32_t* ntok, cudaStream_t st) {
  const size_t smem = sizeof(float) * (2 * TPC * H + TPC * 16 + TPC * kMaxNC);
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(lstm_ctc_kernel<TPC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return tobf_fail(TOBF_E_CUDA, "lstm smem: %s", cudaGetErrorString(e));
  }
  lstm_ctc_kernel<TPC><<<(B + TPC - 1) / TPC, H, smem, st>>>(feats, offsets, B, F, H, NC, w_ihT, w_hhT, b, w_out,
                                                             b_out, tokens, T_max, ntok);
  return tobf_cuda_check("tobf_lstm_ctc");
}

extern "C" int tobf_lstm_ctc(const double* feats, const int32_t* offsets, int32_t B, int32_t F, int32_t H,
                             int32_t NC, const float* w_ihT, const float* w_hhT, const float* b, const float* w_out,
                             const float* b_out, int8_t* tokens, int32_t T_max, int32_t* ntok, void* stream) {
  if (B <= 0) return TOBF_OK;
  if (!feats || !offsets || !w_ihT || !w_hhT || !b || !w_out || !b_out || !tokens || !ntok || F < 1 || F > 9 ||
      NC < 2 || NC > kMaxNC || H < 32 || H > 1024 || H % 32 || T_max < 1)
    return tobf_fail(TOBF_E_INVALID, "tobf_lstm_ctc: bad arguments");
  cudaStream_t st = (cudaStream_t)stream;
  if (B >= 148 * 8) return launch_lstm<8>(feats, offsets, B, F, H, NC, w_ihT, w_hhT, b, w_out, b_out, tokens, T_max, ntok, st);
  return launch_lstm<2>(feats, offsets, B, F, H, NC, w_ihT, w_hhT, b, w_out, b_out, tokens, T_max, ntok, st);
}

extern "C" int tobf_levenshtein(const int8_t* pred, const int32_t* ntok, int32_t B, int32_t T_max,
                                const int8_t* truth, int32_t tlen, int32_t* ed, double* ler, void* stream) {
  if (B <= 0) return TOBF_OK;
  if (!pred || !ntok || (!truth && tlen > 0) || !ed || !ler || tlen < 0 || T_max < 1)
    return tobf_fail(TOBF_E_INVALID, "tobf_levenshtein: bad arguments");
  const int warps = 4;
  const int cap = T_max + 1;
  const size_t smem = sizeof(int) * 2 * warps * cap;
  if (smem > 200 * 1024) return tobf_fail(TOBF_E_INVALID, "tobf_levenshtein: T_max too large");
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(levenshtein_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  levenshtein_kernel<<<(B + warps - 1) / warps, 32 * warps, smem, (cudaStream_t)stream>>>(pred, ntok, B, T_max, truth,
                                                                                          tlen, ed, ler, cap);
  return tobf_cuda_check("tobf_levenshtein");
}

extern "C" int tobf_fitness_eq10(const double* ler, int32_t npred, int32_t ncand, const double* T,
                                 const int32_t* feasible, double Tstar, double budget, double eps, double* R,
                                 double* mean_ler, void* stream) {
  if (ncand <= 0) return TOBF_OK;
  if (!ler || !T || !feasible || !R || !mean_ler || npred < 1)
    return tobf_fail(TOBF_E_INVALID, "tobf_fitness_eq10: bad arguments");
  eq10_kernel<<<(ncand + 127) / 128, 128, 0, (cudaStream_t)stream>>>(ler, npred, ncand, T, feasible, Tstar, budget,
                                                                     eps, R, mean_ler);
  return tobf_cuda_check("tobf_fitness_eq10");
}
