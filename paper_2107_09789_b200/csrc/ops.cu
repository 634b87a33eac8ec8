// Memory-bound executor ops, grouped: one launch runs any mix of MaxPool,
// standalone injective chains, channel copies and SoftMax over many
// candidates. Work items are float4 channel groups (coalesced, vectorised)
// except for unaligned channel copies; descriptors are located by binary
// search over their work-item prefix.
//
// Replaces interpreter.py:33-35 (maxpool), :38-41 (softmax), :52-69
// (ReLU / BatchNorm / Add / Concat / Slice of _eval_node), :114-117 (the
// equivalence compare + max-reduce), and the NCHW<->NHWC staging of
// execute()'s input/output (interpreter.py:75-90).
#include <cmath>
#include "tobf_internal.h"

namespace tobf {

__device__ __forceinline__ float ew_epi(float v, const tobf_ew_desc& d, int64_t pix, int c, int64_t cbase) {
  for (int s = 0; s < d.nepi; ++s) {
    const tobf_epi_step st = d.epi[s];
    switch (st.op) {
      case TOBF_EPI_AFFINE:
        v = v * __ldg(st.ptr + c) + __ldg(st.ptr + st.aux + c);
        break;
      case TOBF_EPI_RELU:
        v = fmaxf(v, 0.0f);
        break;
      case TOBF_EPI_ADD_TENSOR:
        v = v + __ldg(st.ptr + pix * st.aux + c);
        break;
      case TOBF_EPI_ADD_CONST:
        v = v + __ldg(st.ptr + cbase + c);
        break;
      default:
        break;
    }
  }
  return v;
}

__device__ __forceinline__ int find_desc(const tobf_ew_desc* __restrict__ descs, int n, int64_t w) {
  int lo = 0, hi = n - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (descs[mid].work_start <= w) lo = mid; else hi = mid - 1;
  }
  return lo;
}

// Work items of one descriptor (tobf_ew_prepare's count, before its padding
// to a multiple of 32 so that no warp straddles two descriptors: SOFTMAX
// reduces with full-warp shuffles).
__host__ __device__ __forceinline__ int64_t ew_work(const tobf_ew_desc& d) {
  const int64_t pix_in = (int64_t)d.batch * d.H * d.W;
  switch (d.op) {
    case TOBF_OP_MAXPOOL: return (int64_t)d.batch * d.Ho * d.Wo * (d.Cpo / 4);
    case TOBF_OP_EPI: return pix_in * (d.Cpo / 4);
    case TOBF_OP_COPYCH: return pix_in * (d.Cpo - d.a0);
    case TOBF_OP_SOFTMAX: return pix_in * 32;
    default: return 0;
  }
}

// Work items: MAXPOOL / EPI -> one float4 channel group of one output pixel;
// COPYCH -> one channel of one pixel (a0/a1 need not be 4-aligned);
// SOFTMAX -> one warp per pixel (work counted in warps * 32 lanes).
// Each block walks one contiguous chunk of the launch's work items, so a
// thread finds its descriptor once (binary search) and then only advances it
// as its items cross into the next descriptor; per-descriptor item indices
// are 32-bit (tobf_ew_prepare checks the bound). Round 1 binary-searched the
// descriptors for every item and divided in 64 bits: the headline step's
// maxpool launches ran at a fraction of HBM bandwidth.
__global__ void ew_grouped_kernel(const tobf_ew_desc* __restrict__ descs, int n, int64_t total) {
  const int64_t chunk = ((total + gridDim.x - 1) / gridDim.x + blockDim.x - 1) / blockDim.x * blockDim.x;
  const int64_t w0 = blockIdx.x * chunk, w1 = min(total, w0 + chunk);
  int di = -1, dwork = 0;
  int64_t next_start = 0;  // work_start of descriptor di + 1 (or total)
  for (int64_t w = w0 + threadIdx.x; w < w1; w += blockDim.x) {
    if (w >= next_start) {
      di = di < 0 ? find_desc(descs, n, w) : di + 1;
      while (di + 1 < n && descs[di + 1].work_start <= w) ++di;
      next_start = di + 1 < n ? descs[di + 1].work_start : total;
      dwork = (int)ew_work(descs[di]);
    }
    const tobf_ew_desc& d = descs[di];
    const int local = (int)(w - d.work_start);
    if (local >= dwork) continue;  // padding to the warp boundary (tobf_ew_prepare)
    switch (d.op) {
      case TOBF_OP_MAXPOOL: {
        const int groups = d.Cpo >> 2;
        const int pix = local / groups;
        const int g = local - pix * groups;
        const int hw = d.Ho * d.Wo;
        const int n_img = pix / hw;
        const int rem = pix - n_img * hw;
        const int yo = rem / d.Wo, xo = rem - (rem / d.Wo) * d.Wo;
        const int win = d.a0, st = d.a1;
        const float* base = d.x + ((int64_t)n_img * d.H * d.W) * d.ldx + g * 4;
        float4 m = make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY);
        for (int u = 0; u < win; ++u) {
          const float* row = base + ((int64_t)(yo * st + u) * d.W) * d.ldx;
          for (int v = 0; v < win; ++v) {
            const float4 q = __ldg(reinterpret_cast<const float4*>(row + (int64_t)(xo * st + v) * d.ldx));
            m.x = fmaxf(m.x, q.x); m.y = fmaxf(m.y, q.y); m.z = fmaxf(m.z, q.z); m.w = fmaxf(m.w, q.w);
          }
        }
        *reinterpret_cast<float4*>(d.y + (int64_t)pix * d.ldy + g * 4) = m;
        break;
      }
      case TOBF_OP_EPI: {
        const int groups = d.Cpo >> 2;
        const int pix = local / groups;
        const int g = local - pix * groups;
        const float4 q = __ldg(reinterpret_cast<const float4*>(d.x + (int64_t)pix * d.ldx + g * 4));
        const int hw = d.H * d.W;
        int period = 1;
        for (int s = 0; s < d.nepi; ++s)
          if (d.epi[s].op == TOBF_EPI_ADD_CONST) period = d.epi[s].aux;
        const int n_img = pix / hw;
        const int64_t cbase = ((int64_t)(n_img % period) * hw + (pix - n_img * hw)) * d.Cpo;
        const int c = g * 4;
        float o[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) o[e] = (c + e < d.C) ? ew_epi(o[e], d, pix, c + e, cbase) : 0.0f;
        *reinterpret_cast<float4*>(d.y + (int64_t)pix * d.ldy + c) = make_float4(o[0], o[1], o[2], o[3]);
        break;
      }
      case TOBF_OP_COPYCH: {
        // channels [0, C) copied; channels [a0+C, Cpo) of the output zero-filled
        const int span = d.Cpo - d.a0;  // >= C
        const int pix = local / span;
        const int c = local - pix * span;
        const float v = c < d.C ? __ldg(d.x + (int64_t)pix * d.ldx + d.a1 + c) : 0.0f;
        d.y[(int64_t)pix * d.ldy + d.a0 + c] = v;
        break;
      }
      case TOBF_OP_SOFTMAX: {
        const int pix = local >> 5;
        const int lane = local & 31;
        const float* xr = d.x + (int64_t)pix * d.ldx;
        float mx = -INFINITY;
        for (int c = lane; c < d.C; c += 32) mx = fmaxf(mx, xr[c]);
        for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        float sum = 0.0f;
        for (int c = lane; c < d.C; c += 32) sum += expf(xr[c] - mx);
        for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
        float* yr = d.y + (int64_t)pix * d.ldy;
        for (int c = lane; c < d.Cpo; c += 32) yr[c] = c < d.C ? expf(xr[c] - mx) / sum : 0.0f;
        break;
      }
      default:
        break;
    }
  }
}

// ---------------------------------------------------------------- verdict
__global__ void equiv_kernel(const float* const* __restrict__ a_list, const float* const* __restrict__ b_list,
                             int64_t pixels, int C, int ld, float tol, float* __restrict__ worst,
                             int32_t* __restrict__ ok) {
  const int p = blockIdx.y;
  const float* a = a_list[p];
  const float* b = b_list[p];
  float wmax = 0.0f;
  int good = 1;
  const int64_t total = pixels * C;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t pix = i / C;
    const int c = (int)(i - pix * C);
    const float av = a[pix * ld + c], bv = b[pix * ld + c];
    const float diff = fabsf(av - bv);        // np.abs(a - b)            (float32)
    const float den = 1.0f + fabsf(bv);       // 1.0 + np.abs(b)          (float32)
    const float rel = diff / den;             // IEEE division            (float32)
    wmax = fmaxf(wmax, rel);
    if (!(diff <= tol * den)) good = 0;       // |a-b| <= tol*(1+|b|)      (float32)
  }
  for (int o = 16; o; o >>= 1) {
    wmax = fmaxf(wmax, __shfl_xor_sync(0xffffffffu, wmax, o));
    good &= __shfl_xor_sync(0xffffffffu, good, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMax(reinterpret_cast<int*>(worst + p), __float_as_int(wmax));  // non-negative floats order as ints
    if (!good) atomicAnd(ok + p, 0);
  }
}

__global__ void init_verdict_kernel(float* worst, int32_t* ok, int pairs) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < pairs) {
    worst[i] = 0.0f;
    ok[i] = 1;
  }
}

__global__ void nhwc_to_nchw_kernel(const float* __restrict__ x, float* __restrict__ y, int B, int C, int H, int W,
                                    int ld) {
  const int64_t total = (int64_t)B * C * H * W;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t w_ = i % W;
    const int64_t h = (i / W) % H;
    const int64_t c = (i / ((int64_t)W * H)) % C;
    const int64_t b = i / ((int64_t)W * H * C);
    y[i] = x[((b * H + h) * W + w_) * ld + c];
  }
}

__global__ void nchw_to_nhwc_kernel(const float* __restrict__ x, float* __restrict__ y, int B, int C, int H, int W,
                                    int ld) {
  const int64_t total = (int64_t)B * H * W * ld;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = i % ld;
    const int64_t pix = i / ld;
    const int64_t w_ = pix % W;
    const int64_t h = (pix / W) % H;
    const int64_t b = pix / ((int64_t)W * H);
    y[i] = c < C ? x[((b * C + c) * H + h) * W + w_] : 0.0f;
  }
}

static unsigned grid_for(int64_t work, int threads) {
  const int64_t blocks = (work + threads - 1) / threads;
  return (unsigned)std::min<int64_t>(std::max<int64_t>(blocks, 1), 148 * 32);
}

}  // namespace tobf

using namespace tobf;

extern "C" int tobf_ew_prepare(tobf_ew_desc* descs, int n, int64_t* total_work) {
  if (n < 0 || (n > 0 && !descs) || !total_work) return tobf_fail(TOBF_E_INVALID, "tobf_ew_prepare: bad arguments");
  int64_t acc = 0;
  for (int i = 0; i < n; ++i) {
    tobf_ew_desc& d = descs[i];
    switch (d.op) {
      case TOBF_OP_MAXPOOL:
        if (d.Cpo % 4 || d.ldx % 4 || d.ldy % 4 || d.a0 < 1 || d.a1 < 1)
          return tobf_fail(TOBF_E_INVALID, "ew desc %d: bad maxpool geometry", i);
        break;
      case TOBF_OP_EPI:
        if (d.Cpo % 4 || d.ldx % 4 || d.ldy % 4 || d.nepi < 0 || d.nepi > TOBF_MAX_EPI)
          return tobf_fail(TOBF_E_INVALID, "ew desc %d: bad epilogue op", i);
        break;
      case TOBF_OP_COPYCH:
        if (d.Cpo < d.a0 + d.C) return tobf_fail(TOBF_E_INVALID, "ew desc %d: bad channel copy", i);
        break;
      case TOBF_OP_SOFTMAX:
        break;
      default:
        return tobf_fail(TOBF_E_INVALID, "ew desc %d: unknown op %d", i, d.op);
    }
    const int64_t work = ew_work(d);
    if (work >= ((int64_t)1 << 31) - 32) return tobf_fail(TOBF_E_INVALID, "ew desc %d: more than 2^31 work items", i);
    d.work_start = acc;
    acc += (work + 31) & ~int64_t(31);  // warp-aligned descriptor ranges
  }
  *total_work = acc;
  return TOBF_OK;
}

extern "C" int tobf_ew_grouped(const tobf_ew_desc* d_descs, int n, int64_t total_work, void* stream) {
  if (n <= 0 || total_work <= 0) return TOBF_OK;
  if (!d_descs) return tobf_fail(TOBF_E_INVALID, "tobf_ew_grouped: null descriptors");
  ew_grouped_kernel<<<grid_for(total_work, 256), 256, 0, (cudaStream_t)stream>>>(d_descs, n, total_work);
  return tobf_cuda_check("tobf_ew_grouped");
}

extern "C" int tobf_equiv_compare(const float* const* a_list, const float* const* b_list, int pairs, int64_t pixels,
                                  int32_t C, int32_t ld, float tol, float* worst, int32_t* ok, void* stream) {
  if (pairs <= 0) return TOBF_OK;
  if (!a_list || !b_list || !worst || !ok || C < 1 || ld < C)
    return tobf_fail(TOBF_E_INVALID, "tobf_equiv_compare: bad arguments");
  cudaStream_t st = (cudaStream_t)stream;
  init_verdict_kernel<<<(pairs + 127) / 128, 128, 0, st>>>(worst, ok, pairs);
  const int64_t total = pixels * C;
  dim3 grid((unsigned)std::min<int64_t>((total + 255) / 256, 64), (unsigned)pairs);
  equiv_kernel<<<grid, 256, 0, st>>>(a_list, b_list, pixels, C, ld, tol, worst, ok);
  return tobf_cuda_check("tobf_equiv_compare");
}

extern "C" int tobf_nhwc_to_nchw(const float* x, float* y, int32_t B, int32_t C, int32_t H, int32_t W, int32_t ld,
                                 void* stream) {
  if (!x || !y || ld < C) return tobf_fail(TOBF_E_INVALID, "tobf_nhwc_to_nchw: bad arguments");
  const int64_t total = (int64_t)B * C * H * W;
  nhwc_to_nchw_kernel<<<grid_for(total, 256), 256, 0, (cudaStream_t)stream>>>(x, y, B, C, H, W, ld);
  return tobf_cuda_check("tobf_nhwc_to_nchw");
}

extern "C" int tobf_nchw_to_nhwc(const float* x, float* y, int32_t B, int32_t C, int32_t H, int32_t W, int32_t ld,
                                 void* stream) {
  if (!x || !y || ld < C) return tobf_fail(TOBF_E_INVALID, "tobf_nchw_to_nhwc: bad arguments");
  const int64_t total = (int64_t)B * H * W * ld;
  nchw_to_nhwc_kernel<<<grid_for(total, 256), 256, 0, (cudaStream_t)stream>>>(x, y, B, C, H, W, ld);
  return tobf_cuda_check("tobf_nchw_to_nhwc");
}

// Input im2col (the executor's stem path, executor.py `input_im2col`): for a
// conv reading the graph input with few channels (c % 32 != 0: no TMA
// im2col), the K = k1*k2*c elements of every output pixel, in the weights'
// (u, v, c) order, zero-padded to Kp (a multiple of 32), as one NHWC-like
// matrix out[n][yo][xo][Kp]. Built once per staged input and shared by every
// candidate whose conv reads it; the conv becomes a 1x1 GEMM over it fed by
// the TMA path (RN18 stem: 7x7x3 -> Kp 160 = 5 K blocks instead of 7 padded
// 7x7x4 blocks gathered with cp.async). One thread per 4 output columns.
__global__ void im2col_kernel(const float* __restrict__ x, int B, int H, int W, int ldx, int c, int k1, int k2,
                              int stride, int pad, int Ho, int Wo, int Kp, float* __restrict__ out) {
  // per K element: its tap offsets and channel (-1: padding past K), decoded
  // once per block instead of three integer divisions per element
  extern __shared__ int4 ktab[];
  const int K = k1 * k2 * c;
  for (int k = threadIdx.x; k < Kp; k += blockDim.x) {
    const int uv = k / c, cc = k - uv * c, u = uv / k2;
    ktab[k] = k < K ? make_int4(u, uv - u * k2, cc, 0) : make_int4(0, 0, -1, 0);
  }
  __syncthreads();
  const unsigned kq4 = Kp / 4;
  const unsigned quads = (unsigned)B * Ho * Wo * kq4;  // < 2^31 (checked by the caller): 32-bit divisions
  for (unsigned q = blockIdx.x * blockDim.x + threadIdx.x; q < quads; q += gridDim.x * blockDim.x) {
    const unsigned pix = q / kq4;
    const int kq = (int)(q - pix * kq4);
    const unsigned r = pix / (unsigned)Wo;
    const int xo = (int)(pix - r * Wo);
    const unsigned n_ = r / (unsigned)Ho;
    const int yo = (int)(r - n_ * Ho);
    const int n = (int)n_;
    const int y0 = yo * stride - pad, x0 = xo * stride - pad;
    const float* xn = x + (int64_t)n * H * W * ldx;
    float v[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int4 t = ktab[kq * 4 + e];
      const int yi = y0 + t.x, xi = x0 + t.y;
      v[e] = (t.z >= 0 && (unsigned)yi < (unsigned)H && (unsigned)xi < (unsigned)W)
                 ? __ldg(xn + ((int64_t)yi * W + xi) * ldx + t.z) : 0.0f;
    }
    *reinterpret_cast<float4*>(out + (int64_t)pix * Kp + kq * 4) = make_float4(v[0], v[1], v[2], v[3]);
  }
}

extern "C" int tobf_im2col(const float* x, int32_t B, int32_t H, int32_t W, int32_t ldx, int32_t c, int32_t k1,
                           int32_t k2, int32_t stride, int32_t pad, int32_t Ho, int32_t Wo, int32_t Kp, float* out,
                           void* stream) {
  if (!x || !out || B < 1 || H < 1 || W < 1 || c < 1 || ldx < c || k1 < 1 || k2 < 1 || stride < 1 || pad < 0 ||
      Ho < 1 || Wo < 1 || Kp % 4 || Kp < k1 * k2 * c)
    return tobf_fail(TOBF_E_INVALID, "tobf_im2col: bad arguments");
  const int64_t quads = (int64_t)B * Ho * Wo * (Kp / 4);
  if ((size_t)Kp * sizeof(int4) > 48 * 1024 || quads >= ((int64_t)1 << 31))
    return tobf_fail(TOBF_E_INVALID, "tobf_im2col: Kp or the matrix too large");
  im2col_kernel<<<grid_for(quads, 256), 256, (size_t)Kp * sizeof(int4), (cudaStream_t)stream>>>(
      x, B, H, W, ldx, c, k1, k2, stride, pad, Ho, Wo, Kp, out);
  return tobf_cuda_check("tobf_im2col");
}
