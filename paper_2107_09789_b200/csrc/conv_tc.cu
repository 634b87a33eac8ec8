// Grouped implicit-GEMM convolution on sm_100a tensor cores (tcgen05 + TMEM),
// fp32-faithful via 3xTF32 (a*b ~= a_hi*b_hi + a_hi*b_lo + a_lo*b_hi).
//
// Replaces interpreter.py:22-30 (conv2d: np.pad + sliding_window_view +
// einsum -> OpenBLAS sgemm) and the Linear of interpreter.py:48-51 (expressed
// as a full-extent convolution), plus the injective ops the executor fuses
// into the epilogue (BatchNorm interpreter.py:54-56 folded to an affine,
// ReLU :52, Add :59-65 incl. residual operands and dummy constants).
//
// One CTA computes a 128 x BN output tile of one problem of the group:
//   warps 0-3 : im2col gather of the A tile (NHWC fp32, float4 per lane,
//               8 lanes per 128-B row => coalesced), tf32 hi/lo split,
//               128B-swizzled st.shared; then the epilogue (TMEM -> regs ->
//               fused BN/ReLU/Add chain -> NHWC float4 stores)
//   warp 4    : TMEM allocator + bulk-copy producer of the pre-packed,
//               pre-split, pre-swizzled weight image (one UBLKCP per stage)
//   warp 5    : single-thread tcgen05.mma issuer (M=128, N=BN, K=8 per MMA)
// Stages are a ring of {A_hi, A_lo, B_hi, B_lo} guarded by full/empty
// mbarriers; MMA completion frees a stage through tcgen05.commit.
#include "ptx.cuh"
#include "tobf_internal.h"

namespace tobf {

constexpr int kBM = 128;
constexpr int kBK = 32;           // fp32 elements per K block = one 128-B swizzle row
constexpr int kRowBytes = 128;
constexpr int kABytes = kBM * kRowBytes;  // 16 KB

template <int BN>
struct ConvCfg {
  static constexpr int kBBytes = BN * kRowBytes;
  static constexpr int kStageBytes = 2 * kABytes + 2 * kBBytes;
  static constexpr int kStages = BN >= 128 ? 3 : 4;
  static constexpr int kSmem = kStages * kStageBytes + 1024 /*align*/ + 256 /*barriers*/;
  // [0,BN): correction terms (a_lo*b_hi + a_hi*b_lo), whole K;
  // [BN,3BN): ping-pong main accumulators (a_hi*b_hi), one K chunk each
  static constexpr int kTmemCols = 4 * BN;
};

// K blocks accumulated in TMEM before the main partial sum is drained into
// fp32 registers. The tensor-core accumulator loses ~2^-24 relative per MMA
// step (error grows linearly with K, measured in scripts/gpu_acc_probe.py):
// short chains on the main term, the 2^-11-smaller correction terms in their
// own accumulator, and round-to-nearest fp32 adds keep the conv
// fp32-faithful (error at OpenBLAS-sgemm level).
constexpr int kChunkKB = 4;

struct EpiRegs {
  int nepi;
  int op[TOBF_MAX_EPI];
  int aux[TOBF_MAX_EPI];
  const float* ptr[TOBF_MAX_EPI];
};

__device__ __forceinline__ float epi_apply(float v, const EpiRegs& e, int64_t m, int c, int64_t cidx) {
#pragma unroll
  for (int s = 0; s < TOBF_MAX_EPI; ++s) {
    if (s >= e.nepi) break;
    switch (e.op[s]) {
      case TOBF_EPI_AFFINE:
        v = v * __ldg(e.ptr[s] + c) + __ldg(e.ptr[s] + e.aux[s] + c);
        break;
      case TOBF_EPI_RELU:
        v = fmaxf(v, 0.0f);
        break;
      case TOBF_EPI_ADD_TENSOR:
        v = v + __ldg(e.ptr[s] + m * e.aux[s] + c);
        break;
      case TOBF_EPI_ADD_CONST:
        v = v + __ldg(e.ptr[s] + cidx + c);
        break;
      default:
        break;
    }
  }
  return v;
}

// Warp roles (320 threads):
//   0-3  A producer (im2col gather, tf32 split, swizzled st.shared)
//   4    TMEM allocator + B producer (bulk copy of the packed weight image)
//   5    MMA issuer
//   6-9  accumulator drain + epilogue (TMEM lanes 32*(warp%4) ...)
template <int BN>
__global__ void __launch_bounds__(320, 1)
    conv_tf32x3_kernel(const tobf_conv_desc* __restrict__ descs, int nprob) {
  using Cfg = ConvCfg<BN>;
  constexpr int STAGES = Cfg::kStages;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + STAGES * Cfg::kStageBytes);
  uint64_t* empty_bar = full_bar + STAGES;
  uint64_t* acc_full = empty_bar + STAGES;   // [2] MMA -> drain
  uint64_t* acc_empty = acc_full + 2;        // [2] drain -> MMA
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);
  int* s_prob = reinterpret_cast<int*>(tmem_slot + 1);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    int lo = 0, hi = nprob - 1;
    const int b = blockIdx.x;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (__ldg(&descs[mid].tile_start) <= b) lo = mid; else hi = mid - 1;
    }
    *s_prob = lo;
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full_bar[s], 128 + 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&acc_full[s], 1);
      mbar_init(&acc_empty[s], 128);
    }
    fence_mbar_init();
  }
  if (warp == 4) tmem_alloc(tmem_slot, Cfg::kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const tobf_conv_desc& d = descs[*s_prob];

  const int tile = blockIdx.x - d.tile_start;
  const int m_tile = tile / d.ntiles;
  const int n_tile = tile - m_tile * d.ntiles;
  const int m0 = m_tile * kBM;
  const int HWo = d.Ho * d.Wo;
  const int M = d.batch * HWo;
  const int kblocks = d.kblocks;
  const int nchunks = (kblocks + kChunkKB - 1) / kChunkKB;

  if (warp < 4) {
    // ---------------------------------------------------------- A producer
    const int t = threadIdx.x;
    const int chunk = t & 7;
    const int rsub = t >> 3;
    int pixbase[8], ybase[8], xbase[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int m = m0 + rsub + 16 * i;
      if (m < M) {
        const int n = m / HWo;
        const int rem = m - n * HWo;
        const int yo = rem / d.Wo;
        const int xo = rem - yo * d.Wo;
        pixbase[i] = n * d.H * d.W;
        ybase[i] = yo * d.stride - d.pad;
        xbase[i] = xo * d.stride - d.pad;
      } else {
        pixbase[i] = 0;
        ybase[i] = -(1 << 28);  // forces the bounds test to fail
        xbase[i] = -(1 << 28);
      }
    }
    const int Cp = d.Cp, k1 = d.k1, k2 = d.k2;
    int u = 0, v = 0, c0 = chunk * 4;
    while (c0 >= Cp) {
      c0 -= Cp;
      if (++v == k2) { v = 0; ++u; }
    }
    const float* __restrict__ x = d.x;
    const int H = d.H, W = d.W, ldx = d.ldx;
    int stage = 0;
    uint32_t phase = 0;
    for (int kb = 0; kb < kblocks; ++kb) {
      const bool kvalid = u < k1;
      float4 vals[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int yi = ybase[i] + u;
        const int xi = xbase[i] + v;
        if (kvalid && (unsigned)yi < (unsigned)H && (unsigned)xi < (unsigned)W) {
          vals[i] = ldg_nc4(x + (int64_t)(pixbase[i] + yi * W + xi) * ldx + c0);
        } else {
          vals[i] = make_float4(0.f, 0.f, 0.f, 0.f);
        }
      }
      mbar_wait(&empty_bar[stage], phase ^ 1, 0x101);
      const uint32_t a_hi = smem_u32(smem + stage * Cfg::kStageBytes);
      const uint32_t a_lo = a_hi + kABytes;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int r = rsub + 16 * i;
        const uint32_t off = sw128_off(r, chunk);
        float4 h, l;
        h.x = __uint_as_float(to_tf32_rna(vals[i].x)); l.x = vals[i].x - h.x;
        h.y = __uint_as_float(to_tf32_rna(vals[i].y)); l.y = vals[i].y - h.y;
        h.z = __uint_as_float(to_tf32_rna(vals[i].z)); l.z = vals[i].z - h.z;
        h.w = __uint_as_float(to_tf32_rna(vals[i].w)); l.w = vals[i].w - h.w;
        sts128(a_hi + off, h);
        sts128(a_lo + off, l);
      }
      fence_proxy_async_smem();
      mbar_arrive(&full_bar[stage]);
      c0 += kBK;
      while (c0 >= Cp) {
        c0 -= Cp;
        if (++v == k2) { v = 0; ++u; }
      }
      if (++stage == STAGES) { stage = 0; phase ^= 1; }
    }
  } else if (warp == 4) {
    // ---------------------------------------------------------- B producer
    if (lane == 0) {
      const uint8_t* wimg = reinterpret_cast<const uint8_t*>(d.wimg) +
                            (int64_t)n_tile * kblocks * (2 * Cfg::kBBytes);
      int stage = 0;
      uint32_t phase = 0;
      for (int kb = 0; kb < kblocks; ++kb) {
        mbar_wait(&empty_bar[stage], phase ^ 1, 0x104);
        uint8_t* dst = smem + stage * Cfg::kStageBytes + 2 * kABytes;
        mbar_arrive_expect_tx(&full_bar[stage], 2 * Cfg::kBBytes);
        bulk_g2s(dst, wimg + (int64_t)kb * (2 * Cfg::kBBytes), 2 * Cfg::kBBytes, &full_bar[stage]);
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp == 5) {
    // ---------------------------------------------------------- MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc = idesc_make(2u /*tf32*/, kBM, BN);
      int stage = 0;
      uint32_t phase = 0;
      int kb = 0;
      const uint32_t acc_small = tmem_base;
      for (int ch = 0; ch < nchunks; ++ch) {
        const int buf = ch & 1;
        const uint32_t acc = tmem_base + BN + buf * BN;
        mbar_wait(&acc_empty[buf], ((ch >> 1) & 1) ^ 1, 0x106);
        tc_fence_after();
        const int kend = min(kblocks, kb + kChunkKB);
        for (int kc = 0; kb < kend; ++kb, ++kc) {
          mbar_wait(&full_bar[stage], phase, 0x105);
          tc_fence_after();
          const uint32_t a_hi = smem_u32(smem + stage * Cfg::kStageBytes);
          const uint32_t a_lo = a_hi + kABytes;
          const uint32_t b_hi = a_hi + 2 * kABytes;
          const uint32_t b_lo = b_hi + Cfg::kBBytes;
#pragma unroll
          for (int kk = 0; kk < kBK / 8; ++kk) {
            const uint32_t koff = kk * 32;  // 8 tf32 = 32 bytes along the swizzled row
            const uint64_t dah = sdesc_k128(a_hi + koff), dal = sdesc_k128(a_lo + koff);
            const uint64_t dbh = sdesc_k128(b_hi + koff), dbl = sdesc_k128(b_lo + koff);
            mma_tf32(acc_small, dal, dbh, idesc, (kb | kk) != 0);
            mma_tf32(acc_small, dah, dbl, idesc, 1u);
            mma_tf32(acc, dah, dbh, idesc, (kc | kk) != 0);
          }
          mma_commit(&empty_bar[stage]);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        mma_commit(&acc_full[buf]);
      }
    }
  } else {
    // ---------------------------------------------------------- drain + epilogue
    const int lq = warp & 3;  // TMEM lane quarter this warp may access
    float sum[BN];
#pragma unroll
    for (int i = 0; i < BN; ++i) sum[i] = 0.0f;
    for (int ch = 0; ch < nchunks; ++ch) {
      const int buf = ch & 1;
      mbar_wait(&acc_full[buf], (ch >> 1) & 1, 0x103);
      tc_fence_after();
      const uint32_t taddr = tmem_base + (static_cast<uint32_t>(lq * 32) << 16) + BN + buf * BN;
#pragma unroll
      for (int cc = 0; cc < BN / 16; ++cc) {
        float part[16];
        tmem_ld16(taddr + cc * 16, part);
#pragma unroll
        for (int i = 0; i < 16; ++i) sum[cc * 16 + i] += part[i];
      }
      tc_fence_before();
      mbar_arrive(&acc_empty[buf]);
    }
    {
      // the last acc_full commit covered every MMA, so the correction
      // accumulator is complete as well
      const uint32_t taddr = tmem_base + (static_cast<uint32_t>(lq * 32) << 16);
#pragma unroll
      for (int cc = 0; cc < BN / 16; ++cc) {
        float part[16];
        tmem_ld16(taddr + cc * 16, part);
#pragma unroll
        for (int i = 0; i < 16; ++i) sum[cc * 16 + i] += part[i];
      }
    }
    // Stage the tile's fp32 sums in shared memory (the operand ring is idle:
    // every K block has been consumed), 16-B chunks XOR-swizzled by row so
    // the row-per-thread writes are bank-conflict free.
    {
      const int row = lq * 32 + lane;
      float* srow = reinterpret_cast<float*>(smem) + row * BN;
#pragma unroll
      for (int g = 0; g < BN / 4; ++g) {
        const int gs = g ^ (row & (BN / 4 - 1));
        *reinterpret_cast<float4*>(srow + gs * 4) =
            make_float4(sum[g * 4], sum[g * 4 + 1], sum[g * 4 + 2], sum[g * 4 + 3]);
      }
    }
    asm volatile("bar.sync 1, 128;" ::: "memory");
    EpiRegs e;
    e.nepi = d.nepi;
#pragma unroll
    for (int s = 0; s < TOBF_MAX_EPI; ++s) {
      e.op[s] = d.epi[s].op;
      e.aux[s] = d.epi[s].aux;
      e.ptr[s] = d.epi[s].ptr;
    }
    int cperiod = 1;
    for (int s = 0; s < e.nepi; ++s)
      if (e.op[s] == TOBF_EPI_ADD_CONST) cperiod = e.aux[s];
    // Row-per-warp-iteration epilogue: lanes cover 4 consecutive channels
    // each, so residual / constant reads and output writes are coalesced.
    constexpr int kLanesPerRow = BN / 4;            // 32 (BN=128) or 16 (BN=64)
    constexpr int kRowsPerIter = 32 / kLanesPerRow;  // 1 or 2
    const int sub = lane / kLanesPerRow;
    const int g = lane % kLanesPerRow;
    const int c = n_tile * BN + g * 4;
    const int Cpo = d.Cpo, j = d.j;
    const int ew = warp - 6;  // 0..3
#pragma unroll 1
    for (int r0 = ew * kRowsPerIter; r0 < kBM; r0 += 4 * kRowsPerIter) {
      const int row = r0 + sub;
      const int m = m0 + row;
      if (m >= M || c >= Cpo) continue;
      const float* srow = reinterpret_cast<const float*>(smem) + row * BN;
      const float4 a = *reinterpret_cast<const float4*>(srow + ((g ^ (row & (BN / 4 - 1))) * 4));
      const int n_img = m / HWo;
      const int pix = m - n_img * HWo;
      const int64_t cidx = ((int64_t)(n_img % cperiod) * HWo + pix) * Cpo;
      float o[4] = {a.x, a.y, a.z, a.w};
#pragma unroll
      for (int q = 0; q < 4; ++q) o[q] = (c + q < j) ? epi_apply(o[q], e, m, c + q, cidx) : 0.0f;
      *reinterpret_cast<float4*>(d.y + (int64_t)m * d.ldy + c) = make_float4(o[0], o[1], o[2], o[3]);
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 4) {
    tc_fence_after();
    tmem_dealloc(tmem_base, Cfg::kTmemCols);
  }
}

// ------------------------------------------------------------ weight packing
// Image layout: [ntiles][kblocks][hi|lo][BN rows][128 B swizzled], element
// (k, n) of the GEMM B operand (k = (u*k2 + v)*Cp + c) in row n%BN, column k%32.
__global__ void pack_weights_kernel(const float* __restrict__ w, int k1, int k2, int c_real, int Cp, int j,
                                    int64_t su, int64_t sv, int64_t sc, int64_t sn, int BN, int kblocks,
                                    int ntiles, float* __restrict__ img) {
  const int64_t total = (int64_t)ntiles * kblocks * BN * 8;  // 16-B chunks of the hi plane
  const int K = k1 * k2 * Cp;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < total;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int chunk = q & 7;
    const int64_t rowq = q >> 3;
    const int r = rowq % BN;
    const int64_t tk = rowq / BN;
    const int kb = tk % kblocks;
    const int nt = tk / kblocks;
    const int n = nt * BN + r;
    float hv[4], lv[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int k = kb * 32 + chunk * 4 + e;
      float val = 0.f;
      if (n < j && k < K) {
        const int uv = k / Cp;
        const int c = k - uv * Cp;
        const int uu = uv / k2;
        const int vv = uv - uu * k2;
        if (c < c_real) val = w[uu * su + vv * sv + c * sc + n * sn];
      }
      hv[e] = __uint_as_float(to_tf32_rna(val));
      lv[e] = val - hv[e];
    }
    const int64_t plane = (int64_t)BN * 32;  // floats per hi (or lo) plane
    float* base = img + ((int64_t)nt * kblocks + kb) * 2 * plane;
    const uint32_t off = sw128_off(r, chunk) / 4;
    *reinterpret_cast<float4*>(base + off) = make_float4(hv[0], hv[1], hv[2], hv[3]);
    *reinterpret_cast<float4*>(base + plane + off) = make_float4(lv[0], lv[1], lv[2], lv[3]);
  }
}

}  // namespace tobf

using namespace tobf;

extern "C" int tobf_conv_prepare(tobf_conv_desc* descs, int n, int block_n, int64_t* total_tiles) {
  if (n < 0 || (block_n != 64 && block_n != 128) || (n > 0 && !descs)) {
    return tobf_fail(TOBF_E_INVALID, "tobf_conv_prepare: bad arguments");
  }
  int64_t acc = 0;
  for (int i = 0; i < n; ++i) {
    tobf_conv_desc& d = descs[i];
    if (d.Cp % 4 || d.Cpo % 4 || d.ldx % 4 || d.ldy % 4 || d.j < 1 || d.j > d.Cpo || d.k1 < 1 || d.k2 < 1 ||
        d.batch < 1 || d.Ho < 1 || d.Wo < 1 || d.nepi < 0 || d.nepi > TOBF_MAX_EPI) {
      return tobf_fail(TOBF_E_INVALID, "tobf_conv_prepare: descriptor %d violates layout invariants", i);
    }
    d.K = d.k1 * d.k2 * d.Cp;
    d.kblocks = (d.K + kBK - 1) / kBK;
    const int64_t M = (int64_t)d.batch * d.Ho * d.Wo;
    d.mtiles = (int)((M + kBM - 1) / kBM);
    d.ntiles = (d.j + block_n - 1) / block_n;
    d.tile_start = (int)acc;
    acc += (int64_t)d.mtiles * d.ntiles;
  }
  if (acc >= (int64_t)1 << 31) return tobf_fail(TOBF_E_INVALID, "tobf_conv_prepare: too many tiles");
  *total_tiles = acc;
  return TOBF_OK;
}

extern "C" int64_t tobf_wimg_bytes(int32_t k1, int32_t k2, int32_t Cp, int32_t j, int32_t block_n) {
  const int64_t K = (int64_t)k1 * k2 * Cp;
  const int64_t kblocks = (K + kBK - 1) / kBK;
  const int64_t ntiles = (j + block_n - 1) / block_n;
  return ntiles * kblocks * 2 * block_n * kRowBytes;
}

extern "C" int tobf_pack_weights(const float* w, int32_t k1, int32_t k2, int32_t c_real, int32_t Cp, int32_t j,
                                 int64_t su, int64_t sv, int64_t sc, int64_t sn, int32_t block_n, void* wimg,
                                 void* stream) {
  if (!w || !wimg || Cp % 4 || c_real > Cp || (block_n != 64 && block_n != 128)) {
    return tobf_fail(TOBF_E_INVALID, "tobf_pack_weights: bad arguments");
  }
  const int K = k1 * k2 * Cp;
  const int kblocks = (K + kBK - 1) / kBK;
  const int ntiles = (j + block_n - 1) / block_n;
  const int64_t chunks = (int64_t)ntiles * kblocks * block_n * 8;
  const int threads = 256;
  const int64_t blocks = std::min<int64_t>((chunks + threads - 1) / threads, 148 * 16);
  pack_weights_kernel<<<(unsigned)blocks, threads, 0, (cudaStream_t)stream>>>(
      w, k1, k2, c_real, Cp, j, su, sv, sc, sn, block_n, kblocks, ntiles, static_cast<float*>(wimg));
  return tobf_cuda_check("tobf_pack_weights");
}

template <int BN>
static int launch_conv(const tobf_conv_desc* d_descs, int n, int64_t total_tiles, cudaStream_t st) {
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(conv_tf32x3_kernel<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         ConvCfg<BN>::kSmem);
    if (e != cudaSuccess) return tobf_fail(TOBF_E_CUDA, "cudaFuncSetAttribute: %s", cudaGetErrorString(e));
    configured = true;
  }
  conv_tf32x3_kernel<BN><<<(unsigned)total_tiles, 320, ConvCfg<BN>::kSmem, st>>>(d_descs, n);
  return tobf_cuda_check("tobf_conv_grouped");
}

extern "C" int tobf_conv_grouped(const tobf_conv_desc* d_descs, int n, int64_t total_tiles, int block_n,
                                 void* stream) {
  if (n <= 0 || total_tiles <= 0) return TOBF_OK;
  if (!d_descs) return tobf_fail(TOBF_E_INVALID, "tobf_conv_grouped: null descriptors");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (block_n == 128) return launch_conv<128>(d_descs, n, total_tiles, st);
  if (block_n == 64) return launch_conv<64>(d_descs, n, total_tiles, st);
  return tobf_fail(TOBF_E_INVALID, "tobf_conv_grouped: block_n must be 64 or 128");
}

extern "C" int tobf_check_fault(void* stream) {
  int h = 0;
  cudaError_t e = cudaMemcpyFromSymbolAsync(&h, g_tobf_fault, sizeof(int), 0, cudaMemcpyDeviceToHost,
                                            static_cast<cudaStream_t>(stream));
  if (e == cudaSuccess) e = cudaStreamSynchronize(static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return tobf_fail(TOBF_E_CUDA, "tobf_check_fault: %s", cudaGetErrorString(e));
  if (h != 0) {
    const int zero = 0;
    cudaMemcpyToSymbol(g_tobf_fault, &zero, sizeof(int));
    return tobf_fail(TOBF_E_FAULT, "device pipeline wait timed out (code 0x%x)", h);
  }
  return TOBF_OK;
}
