// Grouped implicit-GEMM convolution on sm_100a tensor cores (tcgen05 + TMEM),
// in two precisions (PREC template parameter):
//   0  fp32-faithful via 3xTF32 (a*b ~= a_hi*b_hi + a_hi*b_lo + a_lo*b_hi),
//      kind::tf32 — the 1e-4 contract of the fp32 mode;
//   1  bf16 mode: bf16 weight image; activations enter tensor memory as a
//      bf16 pair a = a_hi + a_lo (a_lo = bf16(a - a_hi)), two kind::f16 MMAs
//      per 16 K (a_hi*b, a_lo*b), fp32 accumulation in TMEM — the 2e-2
//      contract of BASELINE's bf16 mode (cfg4). Rounding the activations too
//      (one MMA) doubles the error: a bf16 emulation of the config-1 stack
//      gives 3.0e-2 max relative error vs fp32, the pair 1.7e-2 (weights'
//      rounding only), so the pair is what keeps the contract on every
//      fixture, at 1/3 of the tensor work of 3xTF32.
//
// Replaces interpreter.py:22-30 (conv2d: np.pad + sliding_window_view +
// einsum -> OpenBLAS sgemm) and the Linear of interpreter.py:48-51 (expressed
// as a full-extent convolution), plus the injective ops the executor fuses
// into the epilogue (BatchNorm interpreter.py:54-56 folded to an affine,
// ReLU :52, Add :59-65 incl. residual operands and dummy constants).
//
// One CTA computes 128 x BN output tiles of the group's problems (persistent,
// warp-specialised; roles below). Operands: A (im2col of the NHWC fp32
// activations) is gathered by cp.async into a shared staging ring, split
// hi/lo per row and written to tensor memory; B (weights) is a pre-packed,
// pre-split, 128B-swizzled image bulk-copied into shared memory. Each K step
// issues three tcgen05.mma kind::tf32 with A from TMEM and B from SMEM.
#include <cuda.h>
#include "ptx.cuh"
#include "tobf_internal.h"

namespace tobf {

// 1 (default): tf32 correction products in their own per-tile TMEM
// accumulator. 0 (measured, reverted): into the chunk's main accumulator —
// 3 tf32 accumulates per K step into one buffer lose enough (the obfuscated
// RN18 logits' error reached 1.4e-4 against the fp32 oracle's 4.5e-5) to
// break the 1e-4 contract, for a 1.5 % faster conv.
#ifndef TOBF_CONV_SPLIT_CORR
#define TOBF_CONV_SPLIT_CORR 1
#endif

// A staging ring depth (K blocks the cp.async gather / TMA im2col loads run
// ahead of the split into TMEM), per BN.
// TMA A staging (fp32 mode): release a slot after the whole split (1)
// instead of as soon as its rows have landed (0); bf16 mode always releases
// after the split
#ifndef TOBF_CONV_RELEASE_LATE
#define TOBF_CONV_RELEASE_LATE 0
#endif
// drain / epilogue arithmetic two lanes per instruction (FADD2 / FFMA2)
// fp32 A stage: hi and lo as one 32-column tcgen05.st each (1) or two x16 (0)
#ifndef TOBF_A_ST32
#define TOBF_A_ST32 1
#endif
#ifndef TOBF_DRAIN_FADD2
#define TOBF_DRAIN_FADD2 1
#endif
// drain: tcgen05.ld x16 loads in flight per wait::ld, per BN
#ifndef TOBF_TMEM_GROUP64
#define TOBF_TMEM_GROUP64 4
#endif
#ifndef TOBF_TMEM_GROUP128
#define TOBF_TMEM_GROUP128 2
#endif
// A producer: load the next staging block's row right after the current
// block's split when it has already landed (1) instead of at the top of the
// next iteration (0), per precision. Measured (RN18 step conv, same box):
// bf16 7.77 -> 7.43 ms; fp32 10.75 -> 10.92 ms (the extra live row spills in
// the fp32 split), so off there
// fp32 A split: hi = the raw fp32 (truncated by the tensor core), lo = a -
// trunc(a) (1), or hi = rna(a), lo = a - hi (0)
#ifndef TOBF_CONV_RAWHI
#define TOBF_CONV_RAWHI 1
#endif
// launches with >= TOBF_CONV_CLAIM_MIN tiles per SM claim TOBF_CONV_CLAIM
// consecutive tiles per atomic
#ifndef TOBF_CONV_CLAIM
#define TOBF_CONV_CLAIM 4
#endif
#ifndef TOBF_CONV_CLAIM_MIN
#define TOBF_CONV_CLAIM_MIN 16
#endif
// tiles the scheduler may hold claimed ahead of the A producer in launches of
// many short tiles (1 = claim only once the A warps took the previous tile).
// 2 measured equal (RN18 step conv 8.84 / 7.26 ms fp32 / bf16 either way):
// the A warps' info_full waits are not the claim gating
#ifndef TOBF_CONV_LOOK
#define TOBF_CONV_LOOK 1
#endif
#ifndef TOBF_CONV_APF_F32
#define TOBF_CONV_APF_F32 1
#endif
#ifndef TOBF_CONV_APF_BF16
#define TOBF_CONV_APF_BF16 1
#endif
#ifndef TOBF_CONV_SD64
#define TOBF_CONV_SD64 4
#endif
#ifndef TOBF_CONV_SD128
#define TOBF_CONV_SD128 4
#endif

// problems whose tile_start the scheduler keeps in shared memory (the rest
// are read from the descriptors)
#ifndef TOBF_CONV_TAB
#define TOBF_CONV_TAB 1024
#endif
#ifndef TOBF_CONV_ST64
#define TOBF_CONV_ST64 4
#endif

#ifndef TOBF_CONV_INFO_SLOTS
#define TOBF_CONV_INFO_SLOTS 4
#endif
constexpr int kBM = 128;
constexpr int kBK = 32;           // fp32 elements per K block = one 128-B swizzle row
constexpr int kRowBytes = 128;
constexpr int kABytes = kBM * kRowBytes;  // 16 KB

template <int BN, int PREC>
struct ConvCfg {
  static constexpr bool kBf16 = PREC == 1;
  // A K block = kStgPerKB staging blocks of 32 fp32 per row; its GEMM K
  // extent is kBKe (tf32: 32 elements = one 128-B row; bf16: 64 = one 128-B
  // bf16 row of the B image, two fp32 staging blocks of A)
  static constexpr int kStgPerKB = kBf16 ? 2 : 1;
  static constexpr int kBKe = kBK * kStgPerKB;
  // The A tile (hi/lo) lives in tensor memory (tcgen05.st by the producer, A
  // operand read from TMEM by the MMA); shared memory carries only B, whose
  // three MMA reads per K step are what the tensor pipe pulls from it.
  static constexpr int kBBytes = BN * kRowBytes;
  static constexpr int kStageBytes = kBf16 ? kBBytes : 2 * kBBytes;  // B (tf32: hi, lo)
  static constexpr int kStages = kBf16 ? 4 : (BN >= 128 ? 2 : TOBF_CONV_ST64);
  // fp32 A blocks land here by cp.async (coalesced, zero-filled padding)
  // kStagingKB blocks ahead of the split into TMEM
  static constexpr int kStagingKB = BN >= 128 ? TOBF_CONV_SD128 : TOBF_CONV_SD64;
  static constexpr int kStagingOff = kStages * kStageBytes;
  static constexpr int kEpiOff = kStagingOff + kStagingKB * kABytes;
  static constexpr int kEpiBytes = kBM * BN * 4;  // fp32 tile staged for the coalesced epilogue
  static constexpr int kInfoBytes = TOBF_CONV_INFO_SLOTS * 256;  // tile-info ring (descriptor copies)
  static_assert(sizeof(tobf_conv_desc) <= 256, "a descriptor fills at most one 256-B ring slot (32 lanes x 8 B)");
  static constexpr int kBarOff = kEpiOff + kEpiBytes + kInfoBytes;
  static constexpr int kTabOff = kBarOff + 512;   // scheduler's copy of the problems' tile_start (kSchedTab ints)
  static constexpr int kSmem = kTabOff + 4 * TOBF_CONV_TAB + 1024 /*align*/;
  // TMEM columns (512 allocated):
  //   [0, kCorrSlots*BN)           (TOBF_CONV_SPLIT_CORR=1 only) correction accumulators
  //                                (a_lo*b_hi + a_hi*b_lo), one per tile slot
  //   next kMainBufs*BN            main accumulators, one K chunk each, round robin
  //   kTmemACol + 64*s             A stage s: 32 hi + 32 lo columns
  // With TOBF_CONV_SPLIT_CORR=0 the two tf32 correction products would go
  // into the chunk's main accumulator and the freed columns give 3 (BN=128) /
  // 4 (BN=64) chunk buffers (too lossy: see the macro). bf16: the tile
  // accumulates in one buffer (no chunked drain: bf16 rounding dominates),
  // two buffers so tile i+1's MMAs overlap tile i's drain.
  static constexpr bool kSplitCorr = !kBf16 && TOBF_CONV_SPLIT_CORR;
  static constexpr int kCorrSlots = kSplitCorr ? (BN >= 128 ? 1 : 2) : 0;
  static constexpr int kMainBufsRaw = (512 - 64 * kStages) / BN;
  static constexpr int kMainBufs = (kSplitCorr || kBf16) ? 2 : (kMainBufsRaw > 4 ? 4 : kMainBufsRaw);
  static constexpr int kTmemMainCol = kCorrSlots * BN;
  static constexpr int kTmemACol = kTmemMainCol + kMainBufs * BN;
  static constexpr int kAStageCols = 64;  // tf32: 32 hi + 32 lo; bf16: 64 K as 32 hi + 32 lo bf16x2 columns
  static constexpr int kTmemCols = 512;
  static_assert(kTmemACol + kAStageCols * kStages <= 512, "TMEM budget");
  static_assert(kSmem <= 227 * 1024, "shared memory budget");
};

// K blocks accumulated in TMEM before the main partial sum is drained into
// fp32 registers. The tensor-core accumulator loses ~2^-24 relative per MMA
// step (error grows linearly with K, measured in scripts/gpu_acc_probe.py):
// short chains on the main term, the 2^-11-smaller correction terms in their
// own accumulator, and round-to-nearest fp32 adds keep the conv
// fp32-faithful (error at OpenBLAS-sgemm level).
#ifndef TOBF_CONV_CHUNK_KB
#define TOBF_CONV_CHUNK_KB 4
#endif
constexpr int kChunkKB = TOBF_CONV_CHUNK_KB;

// Persistent: one CTA per SM walks tiles blockIdx.x, +gridDim.x, ... of the
// group (problems sorted by K descending, so long tiles go first). Every role
// runs the same tile sequence; the operand ring, the chunk accumulators and
// the tile-slot correction accumulators carry their phases across tiles, so
// tile i+1's loads and MMAs overlap tile i's drain and epilogue.
// Warp roles (384 threads = 3 warpgroups; registers rebalanced with setmaxnreg):
//   WG0 warps 0-3   A producer (cp.async im2col gather into the staging ring,
//                   tf32 hi/lo split, tcgen05.st into the TMEM A stage)
//   WG1 warp 4      TMEM allocator + B producer (bulk copy of the packed weight image)
//       warp 5      MMA issuer
//       warp 6      tile scheduler: resolves tile -> problem and copies the
//                   descriptor into a 4-slot shared-memory ring ahead of use
//       warp 7      idle
//   WG2 warps 8-11  accumulator drain + fused epilogue (TMEM lanes 32*(warp%4) ...)
constexpr int kThreads = 384;
constexpr int kRegsProducer = 152, kRegsControl = 56, kRegsDrain = 256;

#ifdef TOBF_CONV_PROF
// Debug-only role timing: per-role wait / busy cycle counters summed over CTAs.
__device__ unsigned long long g_conv_prof[32];
#define PROF_T0() const long long _p0 = clock64()
#define PROF_ADD(slot) atomicAdd(&g_conv_prof[slot], (unsigned long long)(clock64() - _p0))
#define PROF_WAIT(slot, expr) do { const long long _w0 = clock64(); expr; _pacc[slot] += clock64() - _w0; } while (0)
#define PROF_DECL long long _pacc[8] = {0, 0, 0, 0, 0, 0, 0, 0}
#define PROF_FLUSH(base) do { for (int _i = 0; _i < 8; ++_i) atomicAdd(&g_conv_prof[(base) + _i], (unsigned long long)_pacc[_i]); } while (0)
#else
#define PROF_T0()
#define PROF_ADD(slot)
#define PROF_WAIT(slot, expr) expr
#define PROF_DECL
#define PROF_FLUSH(base)
#endif

// Tile-info ring depth: how many tiles the scheduler warp may claim ahead of
// the drain. Tiles are claimed dynamically (atomic counter): an idle SM takes
// the next tile instead of a pre-assigned one waiting behind a long tile
// elsewhere. Must be >= 4: the A producer issues cp.async up to
// kStagingKB-1 = 3 K blocks ahead of its split, which for 1-K-block tiles is
// 3 tiles ahead, while a slot frees only when its tile is fully drained.
constexpr int kInfoSlots = TOBF_CONV_INFO_SLOTS;
// Dynamic tile counters: [0] next tile (beyond the first gridDim.x), [1] CTAs
// exited; the last CTA to exit resets both, so consecutive launches (stream
// ordered: every conv of the executor runs on its engine stream) start at 0.
__device__ int g_conv_sched[2][2][2];  // [PREC][BN>=128]: fallback when the caller passes none
constexpr int kInfoConsumers = 4 /*A warps*/ + 1 /*B*/ + 1 /*MMA*/ + 4 /*drain warps*/;

__device__ __forceinline__ int find_problem(const tobf_conv_desc* __restrict__ descs, int lo, int nprob, int tile) {
  int hi = nprob - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (__ldg(&descs[mid].tile_start) <= tile) lo = mid; else hi = mid - 1;
  }
  return lo;
}


// sum[i] += TMEM column i of this thread's lane (i < BN), G x16 loads in
// flight per tcgen05.wait::ld (TOBF_TMEM_GROUP; 1 = a wait after every load)
template <int BN>
__device__ __forceinline__ void tmem_add_cols(uint32_t taddr, float (&sum)[BN]) {
  constexpr int kG0 = BN >= 128 ? TOBF_TMEM_GROUP128 : TOBF_TMEM_GROUP64;
  constexpr int kG = kG0 < BN / 16 ? kG0 : BN / 16;
#pragma unroll
  for (int c0 = 0; c0 < BN / 16; c0 += kG) {
    uint32_t r[kG][16];
#pragma unroll
    for (int g = 0; g < kG; ++g) tmem_ld16_nw(taddr + (c0 + g) * 16, r[g]);
    tmem_wait_ld();
#pragma unroll
    for (int g = 0; g < kG; ++g) {
      reg_fence16(r[g]);
#if TOBF_DRAIN_FADD2
      // two columns per FADD2 (the same round-to-nearest adds, half the
      // instructions: drain warps share their SMSPs with the A producers)
#pragma unroll
      for (int i = 0; i < 16; i += 2) {
        float* sp = &sum[(c0 + g) * 16 + i];
        f32x2_split(add_f32x2(f32x2(sp[0], sp[1]), f32x2(__uint_as_float(r[g][i]), __uint_as_float(r[g][i + 1]))),
                    sp[0], sp[1]);
      }
#else
#pragma unroll
      for (int i = 0; i < 16; ++i) sum[(c0 + g) * 16 + i] += __uint_as_float(r[g][i]);
#endif
    }
  }
}

// ---------------------------------------------------------------- epilogue
struct EpiArgs {
  uint32_t epi_s;          // shared address of the staged fp32 tile
  int m0, M, c, j, ldy, ldr;
  bool cvalid;
  float* y;
  const float* res0;       // tensor operands of a simple chain (<= 2)
  const float* res1;
  int ldr1;
  float4 sc, sh;           // the (single) folded BatchNorm of a simple chain
};

__device__ __forceinline__ float4 lds_tile(uint32_t epi_s, int row, int g, int bn) {
  return lds128(epi_s + row * bn * 4 + ((g ^ (row & (bn / 4 - 1))) * 16));
}

// Compile-time specialised chain: PROG packs one TOBF_EPI op per nibble.
// Lanes own 4 consecutive channels; a warp covers 32/(BN/4) rows per step,
// kEpiUnroll steps are issued before any is consumed (loads in flight),
// row addresses are linear in the row index (no divisions).
constexpr int kEpiUnroll = 8;
// rows per batch of operand-free full tiles: 16 measured slower than 8
// (RN18 step conv 8.27 vs 8.21 ms fp32, 6.72 vs 6.66 bf16)
#ifndef TOBF_EPI_U0
#define TOBF_EPI_U0 8
#endif

// L1 prefetch of the epilogue's BatchNorm vectors at the drain's tile start:
// measured slower (RN18 step conv 8.50 -> 8.72 ms fp32, 6.87 -> 7.07 bf16), off
#ifndef TOBF_EPI_PREFETCH
#define TOBF_EPI_PREFETCH 0
#endif
// full-tile epilogue rows specialised on the number of tensor operands
#ifndef TOBF_EPI_NT
#define TOBF_EPI_NT 1
#endif
#ifndef TOBF_EPI_FULL
#define TOBF_EPI_FULL 1
#endif
// kFull: every row of the tile is inside M (all but a problem's last M tile),
// so the row loop carries no per-row bounds branches (the stem / 1x1 levels
// are epilogue-bound and their row loop was branch-issue bound)
// NT >= 0: the number of tensor operands fixed at compile time (full tiles)
template <int BN, bool kFull, int NT = -1>
__device__ __forceinline__ void epi_rows(const EpiArgs ea, uint32_t prog, int nsteps, int nt_rt, int ew, int lane) {
  const int nt = NT >= 0 ? NT : nt_rt;
  // full tiles without tensor operands keep twice the rows' stores in flight
  constexpr int kU = (kFull && NT == 0) ? TOBF_EPI_U0 : kEpiUnroll;
  constexpr int kLanesPerRow = BN / 4;
  constexpr int kRowsPerIter = 32 / kLanesPerRow;
  constexpr int kRowStep = 4 * kRowsPerIter;
  const int sub = lane / kLanesPerRow;
  const int g = lane % kLanesPerRow;
  const int c = ea.c;
  if (!ea.cvalid) return;
  const bool cfull = c + 3 < ea.j;
#pragma unroll 1
  for (int r0 = ew * kRowsPerIter + sub; r0 < kBM; r0 += kRowStep * kU) {
    float o[kU][4], ta[kU][4], tb[kU][4];
    int mrow[kU];
#pragma unroll
    for (int q = 0; q < kU; ++q) {
      const int row = r0 + q * kRowStep;
      mrow[q] = ea.m0 + row;
      const bool ok = kFull || (row < kBM && mrow[q] < ea.M);  // row < kBM holds by construction
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f), t0 = v, t1 = v;
      if (ok) {
        v = lds_tile(ea.epi_s, row, g, BN);
        if (nt > 0) t0 = ldg_nc4(ea.res0 + (int64_t)mrow[q] * ea.ldr + c);
        if (nt > 1) t1 = ldg_nc4(ea.res1 + (int64_t)mrow[q] * ea.ldr1 + c);
      } else {
        mrow[q] = -1;
      }
      o[q][0] = v.x; o[q][1] = v.y; o[q][2] = v.z; o[q][3] = v.w;
      ta[q][0] = t0.x; ta[q][1] = t0.y; ta[q][2] = t0.z; ta[q][3] = t0.w;
      tb[q][0] = t1.x; tb[q][1] = t1.y; tb[q][2] = t1.z; tb[q][3] = t1.w;
    }
    const float av[4] = {ea.sc.x, ea.sc.y, ea.sc.z, ea.sc.w};
    const float bv[4] = {ea.sh.x, ea.sh.y, ea.sh.z, ea.sh.w};
    // one warp-uniform branch per step for the whole batch of rows
    int ti = 0;
#pragma unroll 1
    for (int s = 0; s < nsteps; ++s) {
      const uint32_t op = (prog >> (4 * s)) & 7u;
      if (op == TOBF_EPI_AFFINE) {
#if TOBF_DRAIN_FADD2
#pragma unroll
        for (int q = 0; q < kU; ++q)
#pragma unroll
          for (int e = 0; e < 4; e += 2)
            f32x2_split(fma_f32x2(f32x2(o[q][e], o[q][e + 1]), f32x2(av[e], av[e + 1]), f32x2(bv[e], bv[e + 1])),
                        o[q][e], o[q][e + 1]);
#else
#pragma unroll
        for (int q = 0; q < kU; ++q)
#pragma unroll
          for (int e = 0; e < 4; ++e) o[q][e] = o[q][e] * av[e] + bv[e];
#endif
      } else if (op == TOBF_EPI_RELU) {
#pragma unroll
        for (int q = 0; q < kU; ++q)
#pragma unroll
          for (int e = 0; e < 4; ++e) o[q][e] = fmaxf(o[q][e], 0.0f);
      } else if (op == TOBF_EPI_ADD_TENSOR) {
        if (ti == 0) {
#pragma unroll
          for (int q = 0; q < kU; ++q)
#pragma unroll
            for (int e = 0; e < 4; ++e) o[q][e] += ta[q][e];
        } else {
#pragma unroll
          for (int q = 0; q < kU; ++q)
#pragma unroll
            for (int e = 0; e < 4; ++e) o[q][e] += tb[q][e];
        }
        ++ti;
      }
    }
#pragma unroll
    for (int q = 0; q < kU; ++q) {
      if (!kFull && mrow[q] < 0) continue;
#pragma unroll
      for (int e = 0; e < 4; ++e) o[q][e] = (cfull || c + e < ea.j) ? o[q][e] : 0.0f;
      stg128(ea.y + (int64_t)mrow[q] * ea.ldy + c, make_float4(o[q][0], o[q][1], o[q][2], o[q][3]));
    }
  }
}

// Chains with dummy-add constants, 3-4 tensor / constant operands or two
// folded BatchNorms (dimension-mode candidates: a layer with n dummies is
// Conv -> Add(const) x n -> BN -> ReLU, fused): like epi_rows, U rows per
// batch with EVERY step's operands loaded (16-B vectors) before the chain
// runs in step order, so a batch pays one memory latency, not one per step.
// Round 1 ran these through the per-element interpreter below: scalar loads,
// one latency per step per row — the VGG-16 stem level with dummies took
// 8.9 ms of a 54 ms bf16 population forward.
#ifndef TOBF_EPI_OPS
#define TOBF_EPI_OPS 1
#endif
struct EpiOps {
  const float* ptr[4];
  int aux[4];        // tensor: channel stride; const: batch period
  int is_const[4];
  float4 sc[2], sh[2];
  int HWo, Cpo;
};

template <int BN, int U, bool kFull>
__device__ __forceinline__ void epi_rows_ops(const EpiArgs ea, const EpiOps& eo, uint32_t prog, int nsteps, int ew,
                                             int lane) {
  constexpr int kLanesPerRow = BN / 4;
  constexpr int kRowsPerIter = 32 / kLanesPerRow;
  constexpr int kRowStep = 4 * kRowsPerIter;
  const int sub = lane / kLanesPerRow;
  const int g = lane % kLanesPerRow;
  const int c = ea.c;
  if (!ea.cvalid) return;
  const bool cfull = c + 3 < ea.j;
#pragma unroll 1
  for (int r0 = ew * kRowsPerIter + sub; r0 < kBM; r0 += kRowStep * U) {
    float4 o[U], opnd[4][U];
    int mrow[U];
#pragma unroll
    for (int q = 0; q < U; ++q) {
      const int row = r0 + q * kRowStep;
      mrow[q] = ea.m0 + row;
      const bool ok = kFull || (row < kBM && mrow[q] < ea.M);  // row < kBM holds by construction
      o[q] = ok ? lds_tile(ea.epi_s, row, g, BN) : make_float4(0.f, 0.f, 0.f, 0.f);
      int pix = 0, img = 0;
      if (ok) {
        img = mrow[q] / eo.HWo;
        pix = mrow[q] - img * eo.HWo;
      } else {
        mrow[q] = -1;
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        opnd[k][q] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (ok && eo.ptr[k] != nullptr) {
          const int64_t base = eo.is_const[k] ? ((int64_t)(img % eo.aux[k]) * eo.HWo + pix) * eo.Cpo
                                              : (int64_t)mrow[q] * eo.aux[k];
          opnd[k][q] = ldg_nc4(eo.ptr[k] + base + c);
        }
      }
    }
#pragma unroll 1
    for (int s = 0; s < nsteps; ++s) {
      const uint32_t f = (prog >> (5 * s)) & 31u;
      const uint32_t op = f & 7u, slot = f >> 3;
      if (op == TOBF_EPI_AFFINE) {
        const float4 a = slot ? eo.sc[1] : eo.sc[0], b = slot ? eo.sh[1] : eo.sh[0];
#pragma unroll
        for (int q = 0; q < U; ++q) {
          o[q].x = o[q].x * a.x + b.x; o[q].y = o[q].y * a.y + b.y;
          o[q].z = o[q].z * a.z + b.z; o[q].w = o[q].w * a.w + b.w;
        }
      } else if (op == TOBF_EPI_RELU) {
#pragma unroll
        for (int q = 0; q < U; ++q) {
          o[q].x = fmaxf(o[q].x, 0.0f); o[q].y = fmaxf(o[q].y, 0.0f);
          o[q].z = fmaxf(o[q].z, 0.0f); o[q].w = fmaxf(o[q].w, 0.0f);
        }
      } else {  // ADD_TENSOR / ADD_CONST: operand `slot`
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          if (k != (int)slot) continue;
#pragma unroll
          for (int q = 0; q < U; ++q) {
            o[q].x += opnd[k][q].x; o[q].y += opnd[k][q].y; o[q].z += opnd[k][q].z; o[q].w += opnd[k][q].w;
          }
        }
      }
    }
#pragma unroll
    for (int q = 0; q < U; ++q) {
      if (!kFull && mrow[q] < 0) continue;
      o[q].x = (cfull || c + 0 < ea.j) ? o[q].x : 0.0f;
      o[q].y = (cfull || c + 1 < ea.j) ? o[q].y : 0.0f;
      o[q].z = (cfull || c + 2 < ea.j) ? o[q].z : 0.0f;
      o[q].w = (cfull || c + 3 < ea.j) ? o[q].w : 0.0f;
      stg128(ea.y + (int64_t)mrow[q] * ea.ldy + c, o[q]);
    }
  }
}

// Anything else (more than 4 operands or 2 BatchNorms): a per-element
// interpreter of the descriptor's steps.
template <int BN>
__device__ __forceinline__ void epi_rows_generic(const EpiArgs ea, const tobf_conv_desc& d, int ew, int lane,
                                              int HWo) {
  constexpr int kLanesPerRow = BN / 4;
  constexpr int kRowsPerIter = 32 / kLanesPerRow;
  constexpr int kRowStep = 4 * kRowsPerIter;
  const int sub = lane / kLanesPerRow;
  const int g = lane % kLanesPerRow;
  const int c = ea.c;
  if (!ea.cvalid) return;
  const int nepi = d.nepi;
#pragma unroll 1
  for (int row = ew * kRowsPerIter + sub; row < kBM; row += kRowStep) {
    const int m = ea.m0 + row;
    if (m >= ea.M) break;
    const float4 v = lds_tile(ea.epi_s, row, g, BN);
    float o[4] = {v.x, v.y, v.z, v.w};
#pragma unroll 1
    for (int s = 0; s < nepi; ++s) {
      const tobf_epi_step st = d.epi[s];
      int64_t base = 0;
      if (st.op == TOBF_EPI_ADD_TENSOR) base = (int64_t)m * st.aux;
      if (st.op == TOBF_EPI_ADD_CONST) {
        const int n_img = m / HWo;
        base = ((int64_t)(n_img % st.aux) * HWo + (m - n_img * HWo)) * d.Cpo;
      }
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int ce = c + e;
        switch (st.op) {
          case TOBF_EPI_RELU: o[e] = fmaxf(o[e], 0.0f); break;
          case TOBF_EPI_AFFINE: o[e] = o[e] * __ldg(st.ptr + ce) + __ldg(st.ptr + st.aux + ce); break;
          case TOBF_EPI_ADD_TENSOR:
          case TOBF_EPI_ADD_CONST: o[e] += __ldg(st.ptr + base + ce); break;
          default: break;
        }
      }
    }
#pragma unroll
    for (int e = 0; e < 4; ++e)
      if (c + e >= ea.j) o[e] = 0.0f;
    stg128(ea.y + (int64_t)m * ea.ldy + c, make_float4(o[0], o[1], o[2], o[3]));
  }
}

// AM: A-operand mode of the launch — 0 cp.async gather only, 1 mixed (per
// problem: TMA im2col where tobf_conv_desc.tma != 0, else cp.async), 2 TMA
// only (the gather code is compiled out: a smaller A loop, fewer registers)
template <int BN, int PREC, int AM>
__global__ void __launch_bounds__(kThreads, 1)
    conv_tc_kernel(const tobf_conv_desc* __restrict__ descs, int nprob, int total_tiles, int* __restrict__ sched,
                   int claim) {
  using Cfg = ConvCfg<BN, PREC>;
  constexpr bool TMA = AM != 0;
  constexpr bool kAllTma = AM == 2;
  constexpr int STAGES = Cfg::kStages;
  constexpr bool kBf16 = Cfg::kBf16;
  constexpr int kChunk = kBf16 ? (1 << 30) : kChunkKB;  // K blocks per main-accumulator drain
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  float* epi_buf = reinterpret_cast<float*>(smem + Cfg::kEpiOff);
  tobf_conv_desc* info = reinterpret_cast<tobf_conv_desc*>(smem + Cfg::kEpiOff + Cfg::kEpiBytes);
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + Cfg::kBarOff);
  uint64_t* empty_bar = full_bar + STAGES;
  constexpr int NB = Cfg::kMainBufs;
  uint64_t* acc_full = empty_bar + STAGES;   // [NB <= 4] MMA -> drain (one K chunk)
  uint64_t* acc_empty = acc_full + 4;        // [NB] drain -> MMA
  uint64_t* small_empty = acc_empty + 4;     // [2] drain -> MMA (tile-slot correction accumulator)
  uint64_t* info_full = small_empty + 2;     // [kInfoSlots] scheduler -> roles
  uint64_t* info_empty = info_full + kInfoSlots;  // [kInfoSlots] roles -> scheduler
  uint64_t* a_took = info_empty + kInfoSlots;     // [2] A producer took tile k's descriptor (a_took[k&1], phase k>>1)
  uint64_t* stg_full = a_took + 2;                // [kStagingKB] TMA im2col -> A warps (TMA mode)
  uint64_t* stg_empty = stg_full + Cfg::kStagingKB;  // [kStagingKB] A warps -> TMA issuer
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(stg_empty + Cfg::kStagingKB);
  volatile int* info_tile = reinterpret_cast<volatile int*>(tmem_slot + 1);  // [kInfoSlots], -1 = no more tiles
  volatile int* split_last = info_tile + kInfoSlots;  // drain: this unit completes its split-K tile
  // launch-wide tile counters: the caller's pair, else this variant's module pair
  if (sched == nullptr) sched = g_conv_sched[PREC][BN >= 128 ? 1 : 0];

#ifdef TOBF_CONV_PROF
  const unsigned long long _cta_t0 = globaltimer_ns();
  if (threadIdx.x == 0) {
    atomicMax(&g_conv_prof[28], _cta_t0);
    atomicMax(&g_conv_prof[29], ~_cta_t0);
  }
#endif
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full_bar[s], 128 + 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int s = 0; s < NB; ++s) {
      mbar_init(&acc_full[s], 1);
      mbar_init(&acc_empty[s], 128);
    }
    for (int s = 0; s < 2; ++s) mbar_init(&small_empty[s], 128);
    for (int s = 0; s < kInfoSlots; ++s) {
      mbar_init(&info_full[s], 1);
      mbar_init(&info_empty[s], kInfoConsumers + (TMA ? 1 : 0));  // + the TMA issuer warp
    }
    // the scheduler claims tile k+1 once the A warps' issue cursor took tile k
    mbar_init(&a_took[0], 4);
    mbar_init(&a_took[1], 4);
    for (int s = 0; s < Cfg::kStagingKB; ++s) {
      mbar_init(&stg_full[s], 1);
      mbar_init(&stg_empty[s], 4);
    }
    fence_mbar_init();
  }
  if (warp == 4) tmem_alloc(tmem_slot, Cfg::kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp < 4) {
    // ------------------------------------------ A producer (A in tensor memory)
    // Two cursors over this CTA's sequence of K blocks (across tiles):
    //  issue:   lane (chunk = lane&7, rsub = lane>>3) cp.async's 16-B chunk
    //           `chunk` of rows 32*warp + rsub + 4i (i < 8) into staging slot
    //           (block % kStagingKB), zero-filling padding taps — 4 rows x
    //           128 B per instruction, coalesced; kStagingKB-1 blocks ahead;
    //  consume: thread t reads its row t (= TMEM lane t) from the slot,
    //           splits hi/lo and tcgen05.st's 32 + 32 columns of the stage.
    // A warp only reads rows it copied itself, so __syncwarp orders the two.
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kRegsProducer));
    constexpr int SD = Cfg::kStagingKB;
    // measured (RN18 step, same box): fp32 9.42 ms released on landing vs
    // 9.55 after the split; bf16 8.11 vs 7.74 — the other way round
    constexpr bool kReleaseLate = kBf16 || TOBF_CONV_RELEASE_LATE;
    const int t = threadIdx.x;
    const int chunk = lane & 7;
    const int rsub = lane >> 3;
    const uint32_t stg_s = smem_u32(smem + Cfg::kStagingOff);
    PROF_DECL;
    PROF_T0();
    // ---- issue cursor state (current tile of the issue side)
    int iit = 0, ikb = 0, ikblocks = 0;
    bool adone = false;
    const float* x = nullptr;
    const float* rowp[8];
    int yb[8], xb[8];
    int Cp = 32, k1 = 1, k2 = 1, H = 1, W = 1, ldx = 0;
    bool itma = false;                 // issue cursor's tile: A by TMA
    int isb0 = 0, insb = 0;            // its first staging block, the problem's staging blocks within K
    uint32_t tma_bits = 0, zero_bits = 0;  // per staging slot (TMA launches)
    int u = 0, v = 0, c0 = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) { rowp[i] = nullptr; yb[i] = xb[i] = -(1 << 28); }
    auto ensure = [&]() -> bool {  // a K block is ready to issue (fetches the next tile's descriptor)
      while (ikb == ikblocks) {
        if (adone) return false;
        const int islot = iit % kInfoSlots;
        PROF_WAIT(0, mbar_wait(&info_full[islot], (iit / kInfoSlots) & 1, 0x110));
        const int itile = info_tile[islot];
        if (itile < 0) {
          adone = true;
          return false;
        }
        const tobf_conv_desc& d = info[islot];
        const int lt = itile - d.tile_start;
        const int t2 = lt / d.ksplit;             // tile within the problem
        const int kb0 = (lt - t2 * d.ksplit) * d.kper;  // first K block of this work unit
        const int m0 = (t2 / d.ntiles) * kBM + 32 * warp + rsub;
        const int HWo = d.Ho * d.Wo;
        const int M = d.batch * HWo;
        ikblocks = Cfg::kStgPerKB * min(d.kper, d.kblocks - kb0);  // staging blocks
        Cp = d.Cp; k1 = d.k1; k2 = d.k2; H = d.H; W = d.W; ldx = d.ldx;
        x = d.x;
        itma = kAllTma || (TMA && d.tma != 0);             // this tile's A blocks come by TMA (warp 7)
        isb0 = kb0 * Cfg::kStgPerKB;
        insb = d.K / kBK;
#pragma unroll
        for (int i = 0; i < 8 && !itma; ++i) {
          const int m = m0 + 4 * i;
          if (m < M) {
            const int n = m / HWo;
            const int rem = m - n * HWo;
            const int yo = rem / d.Wo;
            const int xo = rem - yo * d.Wo;
            yb[i] = yo * d.stride - d.pad;
            xb[i] = xo * d.stride - d.pad;
            rowp[i] = x + (int64_t)(n * H * W + yb[i] * W + xb[i]) * ldx;
          } else {
            yb[i] = xb[i] = -(1 << 28);  // fails every bounds test
            rowp[i] = x;
          }
        }
        if (!itma) {  // cursor at K element kb0*kBKe + chunk*4 = ((u*k2 + v)*Cp + c0)
          const int k0 = kb0 * Cfg::kBKe + chunk * 4;
          const int tap = k0 / Cp;
          c0 = k0 - tap * Cp;
          u = tap / k2;
          v = tap - u * k2;
        }
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(&info_empty[islot]);  // descriptor fully read into registers
          mbar_arrive(&a_took[iit & 1]);    // the scheduler may claim a further tile
        }
        ikb = 0;
        ++iit;
      }
      return true;
    };
    int issued = 0;
    auto issue = [&]() {
      if (TMA) {
        // per slot: block mode (TMA or cp.async) and "wholly past K" (zeros)
        const uint32_t bit = 1u << (issued % SD);
        // (kAllTma: constant, so the all-TMA variant carries no gather code)
        const bool blk_tma = kAllTma || itma;
        tma_bits = blk_tma ? (tma_bits | bit) : (tma_bits & ~bit);
        zero_bits = (blk_tma && isb0 + ikb >= insb) ? (zero_bits | bit) : (zero_bits & ~bit);
        if (blk_tma) {  // warp 7 loads this block
          ++ikb;
          ++issued;
          return;
        }
      }
      const uint32_t slot = stg_s + (issued % SD) * kABytes;
      const int uq = u < k1 ? u : (1 << 28);  // K tail beyond k1*k2*Cp reads zeros
      const int toff = (u * W + v) * ldx + c0;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int r = 32 * warp + rsub + 4 * i;
        const bool ok = (unsigned)(yb[i] + uq) < (unsigned)H && (unsigned)(xb[i] + v) < (unsigned)W;
        cp_async16(slot + r * kRowBytes + ((chunk ^ (r & 7)) << 4), ok ? rowp[i] + toff : x, ok ? 16u : 0u);
      }
      if (Cp >= kBK) {          // Cp % 32 == 0 or a single wrap
        c0 += kBK;
        if (c0 >= Cp) {
          c0 -= Cp;
          if (++v == k2) { v = 0; ++u; }
        }
      } else {                  // Cp in {4, 8, 16, ...}: step 32/Cp filter taps
        c0 += kBK;
        const int adv = c0 / Cp;
        c0 -= adv * Cp;
        v += adv;
        if (v >= k2) {
          u += v / k2;
          v -= (v / k2) * k2;
        }
      }
      ++ikb;
      ++issued;
    };
#pragma unroll 1
    for (int q = 0; q < SD - 1; ++q) {
      if (ensure()) issue();
      cp_async_commit();
    }
    int stage = 0;
    uint32_t phase = 0;
    // one staged block of this thread's row (32 fp32 of K, = TMEM lane t)
    // -> its A stage in tensor memory (tf32 hi/lo split, or the bf16 pair)
    auto to_tmem = [&](const float4 (&row)[8], int g, auto&& release) {
      if constexpr (kBf16) {
        // 32 fp32 -> 16 hi + 16 lo bf16x2 columns (round to nearest even),
        // element k in the low half of column k/2; two staging blocks fill
        // one 64-K stage (hi columns [0,32), lo columns [32,64))
        uint32_t pk[16], pl[16];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const float4 a = row[q];
          pk[2 * q] = pack_bf16x2(a.x, a.y);
          pk[2 * q + 1] = pack_bf16x2(a.z, a.w);
          pl[2 * q] = pack_bf16x2(a.x - bf16lo_f(pk[2 * q]), a.y - bf16hi_f(pk[2 * q]));
          pl[2 * q + 1] = pack_bf16x2(a.z - bf16lo_f(pk[2 * q + 1]), a.w - bf16hi_f(pk[2 * q + 1]));
        }
        release();  // every loaded value is consumed: the staging slot may be refilled
        const int half = g & 1;
        if (half == 0) {
          PROF_WAIT(1, mbar_wait(&empty_bar[stage], phase ^ 1, 0x101));
          tc_fence_after();
        }
        const uint32_t ta = tmem_base + (static_cast<uint32_t>(warp * 32) << 16) + Cfg::kTmemACol +
                            stage * Cfg::kAStageCols + half * 16;
        tmem_st16u(ta, pk);
        tmem_st16u(ta + 32, pl);
        if (half == 1) {
          PROF_WAIT(3, tmem_wait_st());
          tc_fence_before();
          mbar_arrive(&full_bar[stage]);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        return;
      }
      // split hi/lo BEFORE waiting for the free TMEM stage: after the MMAs
      // release it only the four tcgen05.st are left on the critical path
      float hh[2][16], ll[2][16];
#pragma unroll
      for (int half = 0; half < 2; ++half) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float4 a = row[half * 4 + q];
          float* h = &hh[half][4 * q];
          float* l = &ll[half][4 * q];
#if TOBF_CONV_RAWHI
          // the tensor core reads a tf32 operand by truncation (low 13 bits
          // ignored; scripts/tf32_trunc_probe.cu, both A from TMEM and B from
          // SMEM), so the raw fp32 IS the truncated hi and lo = a - trunc(a)
          // (exact): no rounding ops for hi
          h[0] = a.x; h[1] = a.y; h[2] = a.z; h[3] = a.w;
          const float t0 = __uint_as_float(__float_as_uint(a.x) & 0xFFFFE000u);
          const float t1 = __uint_as_float(__float_as_uint(a.y) & 0xFFFFE000u);
          const float t2 = __uint_as_float(__float_as_uint(a.z) & 0xFFFFE000u);
          const float t3 = __uint_as_float(__float_as_uint(a.w) & 0xFFFFE000u);
          f32x2_split(sub_f32x2(f32x2(a.x, a.y), f32x2(t0, t1)), l[0], l[1]);
          f32x2_split(sub_f32x2(f32x2(a.z, a.w), f32x2(t2, t3)), l[2], l[3]);
          continue;
#endif
          h[0] = tf32_rna_finite(a.x);
          h[1] = tf32_rna_finite(a.y);
          h[2] = tf32_rna_finite(a.z);
          h[3] = tf32_rna_finite(a.w);
          // lo = a - hi, two per FADD2 (the same round-to-nearest subtractions;
          // RN18 conv 9.97 -> 9.88 ms; the bf16 pair split measured slower with it)
          f32x2_split(sub_f32x2(f32x2(a.x, a.y), f32x2(h[0], h[1])), l[0], l[1]);
          f32x2_split(sub_f32x2(f32x2(a.z, a.w), f32x2(h[2], h[3])), l[2], l[3]);
        }
      }
      release();  // every loaded value is consumed: the staging slot may be refilled
      PROF_WAIT(1, mbar_wait(&empty_bar[stage], phase ^ 1, 0x101));
      tc_fence_after();
      const uint32_t ta = tmem_base + (static_cast<uint32_t>(warp * 32) << 16) + Cfg::kTmemACol + stage * 64;
#if TOBF_A_ST32
      tmem_st32(ta, reinterpret_cast<const float(&)[32]>(hh));
      tmem_st32(ta + 32, reinterpret_cast<const float(&)[32]>(ll));
#else
#pragma unroll
      for (int half = 0; half < 2; ++half) {
        tmem_st16(ta + half * 16, hh[half]);
        tmem_st16(ta + 32 + half * 16, ll[half]);
      }
#endif
      PROF_WAIT(3, tmem_wait_st());
      tc_fence_before();
      mbar_arrive(&full_bar[stage]);
      if (++stage == STAGES) { stage = 0; phase ^= 1; }
    };
    // A row of staging block h (this thread's 32 fp32 of K): waits until the
    // block has landed (TMA: stg_full; cp.async: the warp's group h, with
    // `pend` groups issued after it still allowed in flight), then ld.shared
    auto load_row = [&](int h, float4 (&r)[8], auto pend) {
      const uint32_t sbit = 1u << (h % SD);
      const bool blk_tma = kAllTma || (TMA && (tma_bits & sbit));
      // TMA launches: EVERY block passes stg_full (warp 7 arrives for
      // cp.async blocks too), so the A warps can never run SD blocks ahead of
      // warp 7 and complete two phases of a slot's stg_empty before it waits
      // on the first (a mixed cp.async / TMA launch hung or faulted that way)
      if (TMA) PROF_WAIT(2, mbar_wait(&stg_full[h % SD], (h / SD) & 1, 0x11a));
      if (!blk_tma) PROF_WAIT(2, cp_async_wait<decltype(pend)::value>(); __syncwarp());
      const uint32_t src = stg_s + (h % SD) * kABytes + t * kRowBytes;
      if (TMA && (zero_bits & sbit)) {
#pragma unroll
        for (int q = 0; q < 8; ++q) r[q] = make_float4(0.f, 0.f, 0.f, 0.f);
      } else {
#pragma unroll
        for (int q = 0; q < 8; ++q) r[q] = lds128(src + ((q ^ (t & 7)) << 4));
      }
    };
    constexpr bool kApf = TMA && (kBf16 ? TOBF_CONV_APF_BF16 : TOBF_CONV_APF_F32);
    float4 row[8];
    bool have_row = false;  // row already holds block g (loaded during block g-1's split)
#pragma unroll 1
    for (int g = 0;; ++g) {
      __syncwarp();  // every lane is done reading the slot about to be refilled
#ifdef TOBF_CONV_DIAG_NOA
      // diagnostic build: no A gather/split (wrong results; isolates the MMA/B/drain side)
      if (ensure()) { ++ikb; ++issued; }
      cp_async_commit();
      if (g >= issued) break;
      if (g % Cfg::kStgPerKB == Cfg::kStgPerKB - 1) {
        PROF_WAIT(1, mbar_wait(&empty_bar[stage], phase ^ 1, 0x101));
        mbar_arrive(&full_bar[stage]);
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
      continue;
#endif
      PROF_WAIT(4, if (ensure()) issue());
      if (!kAllTma) cp_async_commit();  // one group per block (empty past the end): group g holds block g
      if (g >= issued) break;
      if (!kApf || !have_row) load_row(g, row, std::integral_constant<int, SD - 1>{});
      // TMA launches: release the slot to warp 7 (every block: keeps its
      // phases) only once the row has LANDED: ld.shared results may still be
      // in flight when a following arrive executes, and warp 7's next TMA
      // load into the slot then overwrote rows not yet read — a rare wrong A
      // block (one candidate's forward in ~10 population runs, found by
      // scripts/race_probe.py; never on the cp.async path, whose refills
      // follow the consuming split in program order). A branch on a value
      // that depends on all eight loads makes the warp wait for them (cheaper
      // than releasing after the whole split: TOBF_CONV_RELEASE_LATE=1).
#ifdef TOBF_CONV_PROF
      const long long _l0 = clock64();
#endif
      if (TMA && !kReleaseLate) {
        // an OR tree (LOP3) over one word of each load; the branch is
        // practically never taken and harmless when it is (adds 0)
        const uint32_t lb = ((__float_as_uint(row[0].x) | __float_as_uint(row[1].x) | __float_as_uint(row[2].x)) |
                             (__float_as_uint(row[3].x) | __float_as_uint(row[4].x) | __float_as_uint(row[5].x))) |
                            (__float_as_uint(row[6].x) | __float_as_uint(row[7].x));
        if (lb == 0x7fbfe001u) atomicAdd(&g_tobf_fault, 0);
        __syncwarp();
        if (lane == 0) mbar_arrive(&stg_empty[g % SD]);
      }
#ifdef TOBF_CONV_PROF
      _pacc[5] += clock64() - _l0;  // A.lds: the row's loads landing (+ release)
#endif
      // row is consumed (split into registers): if block g+1 has already
      // landed by TMA (a non-blocking test: waiting for it here would put the
      // next block's arrival on this block's critical path — measured 9.3 ->
      // 12.0 ms), load its row now so the shared-memory latency overlaps this
      // block's TMEM stores (bf16: right after the split; fp32: after the
      // stores, where the split's 64 registers are free again)
      auto prefetch = [&]() {
        if constexpr (kApf) {
          have_row = false;
          if (g + 1 < issued) {
            const int h = g + 1;
            const uint32_t hbit = 1u << (h % SD);
            if ((kAllTma || (tma_bits & hbit)) && !(zero_bits & hbit) &&
                mbar_test_wait(smem_u32(&stg_full[h % SD]), (h / SD) & 1)) {
              const uint32_t src = stg_s + (h % SD) * kABytes + t * kRowBytes;
#pragma unroll
              for (int q = 0; q < 8; ++q) row[q] = lds128(src + ((q ^ (t & 7)) << 4));
              have_row = true;
            }
          }
          have_row = __all_sync(0xffffffffu, have_row);  // warp-uniform (lanes test independently)
        }
      };
      to_tmem(row, g, [&]() {
        if (TMA && kReleaseLate) {
          __syncwarp();
          if (lane == 0) mbar_arrive(&stg_empty[g % SD]);
        }
        if constexpr (kBf16) prefetch();
      });
#ifdef TOBF_CONV_PROF
      const long long _p6 = clock64();
#endif
      if constexpr (!kBf16) prefetch();
#ifdef TOBF_CONV_PROF
      _pacc[6] += clock64() - _p6;  // A.sts: the fp32 prefetch test + issue
#endif
    }
    cp_async_wait<0>();
#ifdef TOBF_CONV_PROF
    if (t == 0) { PROF_FLUSH(0); PROF_ADD(7); }
#endif
  } else if (warp < 8) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kRegsControl));
  }
  if (TMA && warp == 7) {
    // ---------------------------------------------------------- TMA im2col issuer
    // Per tile: the first output pixel (n, yo, xo) of the M tile gives the
    // im2col base (xo*s - pad, yo*s - pad, n); each 32-channel K block is one
    // filter tap (u, v) — the load's im2col offsets — and a channel offset c0.
    // The tensor map's pixel box walks the tile's 128 output pixels (wrapping
    // rows and images, zero-filling the padding) with the conv stride.
    constexpr int SD = Cfg::kStagingKB;
    const uint32_t stg_s = smem_u32(smem + Cfg::kStagingOff);
    int g = 0;
    for (int it = 0;; ++it) {
      const int islot = it % kInfoSlots;
      mbar_wait(&info_full[islot], (it / kInfoSlots) & 1, 0x119);
      const int tile = info_tile[islot];
      if (tile < 0) break;
      const tobf_conv_desc& d = info[islot];
      const int lt = tile - d.tile_start;
      const int t2 = lt / d.ksplit;
      const int kb0 = (lt - t2 * d.ksplit) * d.kper;
      const int nsb = Cfg::kStgPerKB * min(d.kper, d.kblocks - kb0);
      const int sb0 = kb0 * Cfg::kStgPerKB, K = d.K;
      const bool tile_tma = kAllTma || d.tma != 0;
      const int m0 = (t2 / d.ntiles) * kBM;
      const int HWo = d.Ho * d.Wo;
      const int n0 = m0 / HWo;
      const int rem = m0 - n0 * HWo;
      const int yo = rem / d.Wo;
      const int xo = rem - yo * d.Wo;
      const int w0 = xo * d.stride - d.pad, h0 = yo * d.stride - d.pad;
      const int Cp = d.Cp, k2 = d.k2;
      const void* tmap = d.tmap;
      __syncwarp();
      if (lane == 0) mbar_arrive(&info_empty[islot]);
      for (int j = 0; j < nsb; ++j, ++g) {
        const int slot = g % SD;
        mbar_wait(&stg_empty[slot], ((g / SD) & 1) ^ 1, 0x11b);
        if (lane == 0) {
          const int kk = (sb0 + j) * kBK;
          if (tile_tma && kk < K) {
            const int tap = kk / Cp;
            const int c0 = kk - tap * Cp;
            const int u = tap / k2, v = tap - (tap / k2) * k2;
            mbar_arrive_expect_tx(&stg_full[slot], kABytes);
            tma_im2col_4d(stg_s + slot * kABytes, tmap, c0, w0, h0, n0, (uint16_t)v, (uint16_t)u,
                          &stg_full[slot]);
          } else {
            // a cp.async tile's block (the A warps load it), or wholly past K
            // (zeros): keep every slot's phase in step
            mbar_arrive(&stg_full[slot]);
          }
        }
        __syncwarp();
      }
    }
  }
  if (warp == 4) {
    // ---------------------------------------------------------- B producer
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      PROF_DECL;
      PROF_T0();
      for (;; ++it) {
        const int islot = it % kInfoSlots;
        PROF_WAIT(0, mbar_wait(&info_full[islot], (it / kInfoSlots) & 1, 0x111));
        const int tile = info_tile[islot];
        if (tile < 0) break;
        const tobf_conv_desc& d = info[islot];
        const int lt = tile - d.tile_start;
        const int t2 = lt / d.ksplit;
        const int kb0 = (lt - t2 * d.ksplit) * d.kper;
        const int n_tile = t2 - (t2 / d.ntiles) * d.ntiles;
        const int kblocks = min(d.kper, d.kblocks - kb0);
        const uint8_t* wimg = reinterpret_cast<const uint8_t*>(d.wimg) +
                              ((int64_t)n_tile * d.kblocks + kb0) * Cfg::kStageBytes;
        mbar_arrive(&info_empty[islot]);
        for (int kb = 0; kb < kblocks; ++kb) {
          PROF_WAIT(1, mbar_wait(&empty_bar[stage], phase ^ 1, 0x104));
          uint8_t* dst = smem + stage * Cfg::kStageBytes;
#ifdef TOBF_CONV_DIAG_NOB
          (void)dst;  // diagnostic build: no B stream (wrong results)
          mbar_arrive(&full_bar[stage]);
#else
          mbar_arrive_expect_tx(&full_bar[stage], Cfg::kStageBytes);
          bulk_g2s(dst, wimg + (int64_t)kb * Cfg::kStageBytes, Cfg::kStageBytes, &full_bar[stage]);
#endif
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
#ifdef TOBF_CONV_PROF
      PROF_FLUSH(24); PROF_ADD(31);
#endif
    }
  } else if (warp == 5) {
    // ---------------------------------------------------------- MMA issuer
    // The whole warp runs the schedule so stage addresses, descriptors and
    // TMEM addresses are warp-uniform (uniform registers: no per-MMA
    // register->uniform broadcast loop); one elected lane issues.
    constexpr uint32_t idesc = idesc_make(kBf16 ? 1u /*bf16*/ : 2u /*tf32*/, kBM, BN);
    const uint32_t tb = __shfl_sync(0xffffffffu, tmem_base, 0);
    const uint32_t sbase = __shfl_sync(0xffffffffu, smem_u32(smem), 0);
    int stage = 0;
    uint32_t phase = 0;
    int gc = 0;  // global chunk counter (main accumulator ping-pong)
    int it = 0;  // local tile counter (correction accumulator slot)
    PROF_DECL;
    PROF_T0();
    for (;; ++it) {
      const int islot = it % kInfoSlots;
      PROF_WAIT(0, mbar_wait(&info_full[islot], (it / kInfoSlots) & 1, 0x112));
      const int mtile = info_tile[islot];
      if (mtile < 0) break;
      int kblocks;
      {
        const tobf_conv_desc& d = info[islot];
        const int lt = mtile - d.tile_start;
        const int kb0 = (lt % d.ksplit) * d.kper;
        kblocks = min(d.kper, d.kblocks - kb0);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&info_empty[islot]);
      const int slot = Cfg::kSplitCorr ? it % (Cfg::kSplitCorr ? Cfg::kCorrSlots : 1) : 0;
      const uint32_t acc_small = tb + slot * BN;
      if constexpr (Cfg::kSplitCorr) {
        PROF_WAIT(1, mbar_wait(&small_empty[slot], ((it / Cfg::kCorrSlots) & 1) ^ 1, 0x107));
        tc_fence_after();
      }
      for (int kb0 = 0; kb0 < kblocks; kb0 += kChunk, ++gc) {
        const int buf = gc % NB;
        const uint32_t acc = tb + Cfg::kTmemMainCol + buf * BN;
        PROF_WAIT(2, mbar_wait(&acc_empty[buf], ((gc / NB) & 1) ^ 1, 0x106));
        tc_fence_after();
        const int kend = kblocks - kb0 > kChunk ? kb0 + kChunk : kblocks;
        for (int kb = kb0; kb < kend; ++kb) {
          PROF_WAIT(3, mbar_wait(&full_bar[stage], phase, 0x105));
          tc_fence_after();
          const uint32_t b_hi = sbase + stage * Cfg::kStageBytes;
          const uint32_t b_lo = b_hi + Cfg::kBBytes;
          const uint32_t ta = tb + Cfg::kTmemACol + stage * Cfg::kAStageCols;  // tf32: A hi, lo at +32
          if constexpr (kBf16) {
            if (elect_one()) {
#pragma unroll
              for (int kk = 0; kk < Cfg::kBKe / 16; ++kk) {  // 16 bf16 = 32 B of the B row, 8 A columns
                const uint64_t db = sdesc_k128(b_hi + kk * 32);
                mma_bf16_ts(acc, ta + kk * 8, db, idesc, (kb - kb0 | kk) != 0);  // a_hi * b
                mma_bf16_ts(acc, ta + 32 + kk * 8, db, idesc, 1u);               // a_lo * b
              }
              mma_commit(&empty_bar[stage]);
            }
          } else if (elect_one()) {
#pragma unroll
            for (int kk = 0; kk < kBK / 8; ++kk) {
              const uint32_t koff = kk * 32;  // 8 tf32 = 32 bytes along the swizzled row
              const uint64_t dbh = sdesc_k128(b_hi + koff), dbl = sdesc_k128(b_lo + koff);
              if constexpr (Cfg::kSplitCorr) {
                mma_tf32_ts(acc_small, ta + 32 + kk * 8, dbh, idesc, (kb | kk) != 0);
                mma_tf32_ts(acc_small, ta + kk * 8, dbl, idesc, 1u);
                mma_tf32_ts(acc, ta + kk * 8, dbh, idesc, (kb - kb0 | kk) != 0);
              } else {
                mma_tf32_ts(acc, ta + kk * 8, dbh, idesc, (kb - kb0 | kk) != 0);  // a_hi * b_hi
                mma_tf32_ts(acc, ta + kk * 8, dbl, idesc, 1u);                    // a_hi * b_lo
                mma_tf32_ts(acc, ta + 32 + kk * 8, dbh, idesc, 1u);               // a_lo * b_hi
              }
            }
            mma_commit(&empty_bar[stage]);
          }
          __syncwarp();
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        if (elect_one()) mma_commit(&acc_full[buf]);
        __syncwarp();
      }
    }
#ifdef TOBF_CONV_PROF
    if (lane == 0) { PROF_FLUSH(8); PROF_ADD(15); }
#endif
  } else if (warp >= 8) {
    // ---------------------------------------------------------- drain + epilogue
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kRegsDrain));
    const int lq = warp & 3;  // TMEM lane quarter this warp may access
    const int ew = warp - 8;  // 0..3
    int gc = 0, it = 0;
    PROF_DECL;
    PROF_T0();
    for (;; ++it) {
      const int islot = it % kInfoSlots;
      // one drain warp polls, the other three sleep in the named barrier
      // (polling warps take issue slots from the producers on their SMSPs)
      if (ew == 0) PROF_WAIT(0, mbar_wait(&info_full[islot], (it / kInfoSlots) & 1, 0x113));
      asm volatile("bar.sync 2, 128;" ::: "memory");
      const int tile = info_tile[islot];
      if (tile < 0) break;
      const tobf_conv_desc& d = info[islot];
      const int lt = tile - d.tile_start;
      const int t2 = lt / d.ksplit;
      const int ks = lt - t2 * d.ksplit;
      const int m_tile = t2 / d.ntiles;
      const int n_tile = t2 - m_tile * d.ntiles;
      const int m0 = m_tile * kBM;
      const int HWo = d.Ho * d.Wo;
      const int M = d.batch * HWo;
      const int kblocks = min(d.kper, d.kblocks - ks * d.kper);
#if TOBF_EPI_PREFETCH
      {
        // the epilogue's folded-BatchNorm vectors into L1 now, so the setup's
        // loads after the drain hit L1 instead of paying an L2 round trip
        const int cpf = n_tile * BN + (lane % (BN / 4)) * 4;
        if (cpf < d.Cpo) {
#pragma unroll
          for (int s = 0; s < TOBF_MAX_EPI; ++s) {
            if (s < d.nepi && d.epi[s].op == TOBF_EPI_AFFINE) {
              // a paired problem's upper half reads its own vectors (aff2)
              const bool up = d.pair != 0 && cpf >= 64;
              const float* ap = up ? d.aff2 : d.epi[s].ptr;
              const int cc = up ? cpf - 64 : cpf;
              prefetch_l1(ap + cc);
              prefetch_l1(ap + d.epi[s].aux + cc);
            }
          }
        }
      }
#endif
      const int slot = Cfg::kSplitCorr ? it % (Cfg::kSplitCorr ? Cfg::kCorrSlots : 1) : 0;
      float sum[BN];
#pragma unroll
      for (int i = 0; i < BN; ++i) sum[i] = 0.0f;
      for (int kb0 = 0; kb0 < kblocks; kb0 += kChunk, ++gc) {
        const int buf = gc % NB;
        if (ew == 0) PROF_WAIT(1, mbar_wait(&acc_full[buf], (gc / NB) & 1, 0x103));
        asm volatile("bar.sync 2, 128;" ::: "memory");
        tc_fence_after();
        const uint32_t taddr = tmem_base + (static_cast<uint32_t>(lq * 32) << 16) + Cfg::kTmemMainCol + buf * BN;
#ifndef TOBF_CONV_DIAG_NOD  // diagnostic build: no drain / epilogue (wrong results)
        tmem_add_cols<BN>(taddr, sum);
#endif
        tc_fence_before();
        mbar_arrive(&acc_empty[buf]);
      }
      if constexpr (Cfg::kSplitCorr) {
        // the tile's last acc_full commit covered every MMA of the tile, so the
        // correction accumulator of this slot is complete as well
        const uint32_t taddr = tmem_base + (static_cast<uint32_t>(lq * 32) << 16) + slot * BN;
        tmem_add_cols<BN>(taddr, sum);
        tc_fence_before();
        mbar_arrive(&small_empty[slot]);
      }
      // Stage the tile's fp32 sums in the epilogue buffer, 16-B chunks
      // XOR-swizzled by row so the row-per-thread writes are conflict free.
      const uint32_t epi_s = smem_u32(epi_buf);  // explicit shared-space addressing
      {
        const int row = lq * 32 + lane;
        const uint32_t srow = epi_s + row * BN * 4;
#pragma unroll
        for (int g = 0; g < BN / 4; ++g) {
          const int gs = g ^ (row & (BN / 4 - 1));
          sts128(srow + gs * 16, make_float4(sum[g * 4], sum[g * 4 + 1], sum[g * 4 + 2], sum[g * 4 + 3]));
        }
      }
#ifdef TOBF_CONV_PROF
      const long long _e0 = clock64();
#endif
      asm volatile("bar.sync 1, 128;" ::: "memory");
#ifdef TOBF_CONV_PROF
      const long long _e1 = clock64();
      long long _e2 = _e1;
      _pacc[3] += _e1 - _e0;
#endif
#ifdef TOBF_CONV_DIAG_NOD
      bool run_epi = false;
      if (false) {
#else
      bool run_epi = true;
      if (d.ksplit > 1) {
#endif
        // ---- split-K: publish this unit's partial tile (coalesced rows), count
        // arrivals; the last unit of the tile sums all partials in unit order
        // (deterministic whichever unit arrives last) back into the staging
        // buffer and runs the epilogue. Partials stay L2-resident.
        constexpr int kLPR = BN / 4, kRPI = 32 / kLPR;
        const int sub = lane / kLPR, g = lane % kLPR;
        const int S = d.ksplit;
        float* part0 = d.ws + (int64_t)t2 * S * (kBM * BN);
        float* mine = part0 + (int64_t)ks * (kBM * BN);
#pragma unroll 4
        for (int row = ew * kRPI + sub; row < kBM; row += 4 * kRPI)
          __stcg(reinterpret_cast<float4*>(mine + row * BN + g * 4), lds_tile(epi_s, row, g, BN));
        __threadfence();
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (ew == 0 && lane == 0) *split_last = atomicAdd(d.cnt + t2, 1) == S - 1 ? 1 : 0;
        asm volatile("bar.sync 1, 128;" ::: "memory");
        run_epi = *split_last != 0;
        if (run_epi) {
          __threadfence();
#pragma unroll 2
          for (int row = ew * kRPI + sub; row < kBM; row += 4 * kRPI) {
            const float* src = part0 + row * BN + g * 4;
            float4 acc = __ldcg(reinterpret_cast<const float4*>(src));
            for (int q = 1; q < S; ++q) {
              const float4 p = __ldcg(reinterpret_cast<const float4*>(src + (int64_t)q * (kBM * BN)));
              acc.x += p.x; acc.y += p.y; acc.z += p.z; acc.w += p.w;
            }
            sts128(epi_s + row * BN * 4 + ((g ^ (row & (BN / 4 - 1))) << 4), acc);
          }
          if (ew == 0 && lane == 0) atomicExch(d.cnt + t2, 0);  // ready for the next launch
          asm volatile("bar.sync 1, 128;" ::: "memory");
        }
      }

      if (run_epi) {
      // ---- fused epilogue over the staged tile -----------------------------
      const int nepi = d.nepi;
      int eop[TOBF_MAX_EPI], eaux[TOBF_MAX_EPI];
      const float* eptr[TOBF_MAX_EPI];
      int naff = 0, nld = 0, nconst = 0;
      uint32_t prog = 0;
#pragma unroll
      for (int s = 0; s < TOBF_MAX_EPI; ++s) {
        eop[s] = s < nepi ? d.epi[s].op : TOBF_EPI_NONE;
        eaux[s] = d.epi[s].aux;
        eptr[s] = d.epi[s].ptr;
        int slot = 0;
        if (eop[s] == TOBF_EPI_AFFINE) slot = naff++;
        if (eop[s] == TOBF_EPI_ADD_TENSOR) slot = nld++;
        if (eop[s] == TOBF_EPI_ADD_CONST) ++nconst;
        prog |= (uint32_t)((eop[s] & 7) | ((slot & 1) << 3)) << (4 * s);
      }
      EpiArgs ea;
      ea.epi_s = epi_s;
      ea.m0 = m0;
      ea.M = M;
      ea.c = n_tile * BN + (lane % (BN / 4)) * 4;
      ea.cvalid = ea.c < d.Cpo;
      ea.j = d.j;
      ea.y = d.y;
      ea.ldy = d.ldy;
      // a paired problem (two 64-channel halves, tobf_conv_desc.pair): the
      // upper half's lanes write y2 with their own folded BatchNorm
      const bool upper = d.pair != 0 && ea.c >= 64;
      if (d.pair != 0) {
        ea.j = 64;
        if (upper) {
          ea.c -= 64;
          ea.y = d.y2;
        }
        ea.cvalid = ea.c < 64;
      }
      ea.sc = ea.sh = make_float4(0.f, 0.f, 0.f, 0.f);
      ea.res0 = ea.res1 = nullptr;
      ea.ldr = ea.ldr1 = 0;
      {
        int ti = 0;
#pragma unroll
        for (int s = 0; s < TOBF_MAX_EPI; ++s) {
          if (eop[s] == TOBF_EPI_AFFINE && ea.cvalid) {
            const float* ap = upper ? d.aff2 : eptr[s];
            ea.sc = __ldg(reinterpret_cast<const float4*>(ap + ea.c));
            ea.sh = __ldg(reinterpret_cast<const float4*>(ap + eaux[s] + ea.c));
          }
          if (eop[s] == TOBF_EPI_ADD_TENSOR) {
            if (ti == 0) { ea.res0 = eptr[s]; ea.ldr = eaux[s]; } else { ea.res1 = eptr[s]; ea.ldr1 = eaux[s]; }
            ++ti;
          }
        }
      }
#ifdef TOBF_CONV_PROF
      _e2 = clock64();
      _pacc[4] += _e2 - _e1;
#endif
      // Simple chains (<= 1 folded BN, <= 2 tensor operands, no dummy
      // constant) cover > 95% of the output volume the lowering emits for
      // RN18 sequence candidates; chains with constants / up to 4 operands /
      // 2 BNs take epi_rows_ops; anything else the per-element interpreter.
      if (naff <= 1 && nld <= 2 && nconst == 0) {
        if (TOBF_EPI_FULL && m0 + kBM <= M) {
#if TOBF_EPI_NT
          if (nld == 0) epi_rows<BN, true, 0>(ea, prog, nepi, nld, ew, lane);
          else if (nld == 1) epi_rows<BN, true, 1>(ea, prog, nepi, nld, ew, lane);
          else epi_rows<BN, true, 2>(ea, prog, nepi, nld, ew, lane);
#else
          epi_rows<BN, true>(ea, prog, nepi, nld, ew, lane);
#endif
        } else {
          epi_rows<BN, false>(ea, prog, nepi, nld, ew, lane);
        }
      } else if (TOBF_EPI_OPS && naff <= 2 && nld + nconst <= 4) {
        EpiOps eo;
        uint32_t prog5 = 0;
        int na = 0, nk = 0;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          eo.ptr[k] = nullptr;
          eo.aux[k] = 1;
          eo.is_const[k] = 0;
        }
        eo.sc[0] = eo.sc[1] = eo.sh[0] = eo.sh[1] = make_float4(0.f, 0.f, 0.f, 0.f);
        eo.HWo = HWo;
        eo.Cpo = d.Cpo;
#pragma unroll
        for (int s = 0; s < TOBF_MAX_EPI; ++s) {
          uint32_t slot = 0;
          if (eop[s] == TOBF_EPI_AFFINE) {
            slot = na;
            if (ea.cvalid) {
              const float4 a = __ldg(reinterpret_cast<const float4*>(eptr[s] + ea.c));
              const float4 b = __ldg(reinterpret_cast<const float4*>(eptr[s] + eaux[s] + ea.c));
              if (na == 0) { eo.sc[0] = a; eo.sh[0] = b; } else { eo.sc[1] = a; eo.sh[1] = b; }
            }
            ++na;
          } else if (eop[s] == TOBF_EPI_ADD_TENSOR || eop[s] == TOBF_EPI_ADD_CONST) {
            slot = nk;
#pragma unroll
            for (int k = 0; k < 4; ++k)
              if (k == nk) {
                eo.ptr[k] = eptr[s];
                eo.aux[k] = max(eaux[s], 1);
                eo.is_const[k] = eop[s] == TOBF_EPI_ADD_CONST;
              }
            ++nk;
          }
          prog5 |= (uint32_t)((eop[s] & 7) | (slot << 3)) << (5 * s);
        }
        if (TOBF_EPI_FULL && m0 + kBM <= M) epi_rows_ops<BN, 4, true>(ea, eo, prog5, nepi, ew, lane);
        else epi_rows_ops<BN, 4, false>(ea, eo, prog5, nepi, ew, lane);
      } else {
        epi_rows_generic<BN>(ea, d, ew, lane, HWo);
      }
      }  // run_epi
#ifdef TOBF_CONV_PROF
      const long long _e3 = clock64();
      _pacc[5] += _e3 - _e2;
#endif
      asm volatile("bar.sync 1, 128;" ::: "memory");  // epilogue buffer free for the next tile
#ifdef TOBF_CONV_PROF
      _pacc[6] += clock64() - _e3;
#endif
      if (lane == 0) mbar_arrive(&info_empty[islot]);
#ifdef TOBF_CONV_PROF
      _pacc[2] += clock64() - _e0;
#endif
    }
#ifdef TOBF_CONV_PROF
    if (ew == 0 && lane == 0) { PROF_FLUSH(16); PROF_ADD(23); }
#endif
  } else if (warp == 6) {
    // ---------------------------------------------------------- tile scheduler
    // Claims tiles in batches of `claim` consecutive tiles: the CTA's first
    // batch is [blockIdx.x*claim, +claim), every further one comes from the
    // launch-wide counter (tiles are in longest-K-first order, so greedy
    // claiming is an LPT schedule; launches of many short tiles claim 4 at a
    // time so the atomic's latency is paid once per 4 tiles). The problem of a
    // tile is found in a shared-memory copy of the descriptors' tile_start
    // (forward scan: a CTA's tiles only increase), and a tile of the previous
    // tile's problem copies its descriptor from the previous ring slot — the
    // round-1 global binary search + 224-B global copy per tile cost a few
    // microseconds of latency on every tile, longer than a 1x1 conv tile.
    constexpr int kTab = TOBF_CONV_TAB;
    int* s_tstart = reinterpret_cast<int*>(smem + Cfg::kTabOff);
    for (int i = lane; i < nprob && i < kTab; i += 32) s_tstart[i] = __ldg(&descs[i].tile_start);
    __syncwarp();
    auto tstart = [&](int i) { return i < kTab ? s_tstart[i] : __ldg(&descs[i].tile_start); };
    int prob = 0, prev_slot = -1;
    int bnext = 0, bend = 0;
    const int look = claim > 1 ? TOBF_CONV_LOOK : 1;
    for (int it = 0;; ++it) {
      const int islot = it % kInfoSlots;
#ifdef TOBF_SCHED_NOBACKOFF
      mbar_wait(&info_empty[islot], ((it / kInfoSlots) & 1) ^ 1, 0x114);
#else
      mbar_wait_backoff(&info_empty[islot], ((it / kInfoSlots) & 1) ^ 1, 0x114);
#endif
      // claim lazily: only once the A producer has taken tile it-look, so a
      // CTA holds at most `look` claimed-but-unstarted tiles and the launch's
      // tail stays balanced (the info ring would otherwise let it claim 3 ahead)
      // launches of many short tiles (claim > 1) may keep TOBF_CONV_LOOK
      // tiles claimed ahead; two alternating barriers, so a wait never
      // targets a phase two behind
      if (it >= look) {
        const int k = it - look;
        mbar_wait(&a_took[k & 1], (k >> 1) & 1, 0x118);
      }
      if (bnext == bend) {
        int first = 0;
        if (lane == 0) first = it == 0 ? (int)blockIdx.x * claim : (int)gridDim.x * claim + atomicAdd(&sched[0], claim);
        bnext = __shfl_sync(0xffffffffu, first, 0);
        bend = bnext + claim;
      }
      int tile = bnext++;
      if (tile >= total_tiles) tile = -1;
      if (tile >= 0) {
        const int p0 = prob;
        while (prob + 1 < nprob && tstart(prob + 1) <= tile) ++prob;
        uint64_t* dst = reinterpret_cast<uint64_t*>(info + islot);
        constexpr int kWords = sizeof(tobf_conv_desc) / 8;
        if (prob == p0 && prev_slot >= 0) {
          const uint64_t* src = reinterpret_cast<const uint64_t*>(info + prev_slot);
          if (lane < kWords) dst[lane] = src[lane];
        } else {
          const uint64_t* src = reinterpret_cast<const uint64_t*>(descs + prob);
          if (lane < kWords) dst[lane] = __ldg(src + lane);
        }
        prev_slot = islot;
      }
      if (lane == 0) info_tile[islot] = tile;
      __syncwarp();
      if (lane == 0) mbar_arrive(&info_full[islot]);
      if (tile < 0) break;
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 4) {
    tc_fence_after();
    tmem_dealloc(tmem_base, Cfg::kTmemCols);
  }
#ifdef TOBF_CONV_PROF
  if (threadIdx.x == 0) {
    const unsigned long long _cta_t1 = globaltimer_ns();
    atomicMax(&g_conv_prof[30], _cta_t1);
    atomicAdd(&g_conv_prof[26], _cta_t1 - _cta_t0);
  }
#endif
  if (threadIdx.x == 0) {
    // every claim of this CTA happened before the barrier above; the last CTA
    // out resets the counters for the next launch
    __threadfence();
    if (atomicAdd(&sched[1], 1) == (int)gridDim.x - 1) {
      atomicExch(&sched[0], 0);
      atomicExch(&sched[1], 0);
    }
  }
}

// ------------------------------------------------------------ weight packing
// Image layout: [ntiles][kblocks][plane][BN rows][128 B swizzled] with, per
// precision, element (k, n) of the GEMM B operand (k = (u*k2 + v)*Cp + c) in
// row n%BN of K block k / kBKe:
//   tf32x3  planes hi | lo, column k%32 as fp32 (tf32-rounded hi, exact lo)
//   bf16    one plane, column k%64 as bf16 (round to nearest even)
// maps (optional, knob-derived weights, derived.py): [mu(k1) | mv(k2) | mc(c_real) | mn(j)]
// source indices into the vanilla array (-1 = zero) and scales [sc(c_real) | sn(j)]:
// element (u, v, c, n) = w[mu[u]*su + mv[v]*sv + mc[c]*sc + mn[n]*sn] * sc[c] * sn[n].
__device__ __forceinline__ float weight_at(const float* __restrict__ w, int k, int n, int k1, int k2, int c_real,
                                           int Cp, int j, int K, int64_t su, int64_t sv, int64_t sc, int64_t sn,
                                           const int32_t* __restrict__ maps, const float* __restrict__ scales) {
  if (n >= j || k >= K) return 0.f;
  const int uv = k / Cp;
  const int c = k - uv * Cp;
  const int uu = uv / k2;
  const int vv = uv - uu * k2;
  if (c >= c_real) return 0.f;
  if (maps == nullptr) return w[uu * su + vv * sv + c * sc + n * sn];
  const int mu = __ldg(maps + uu), mv = __ldg(maps + k1 + vv);
  const int mc = __ldg(maps + k1 + k2 + c), mn = __ldg(maps + k1 + k2 + c_real + n);
  if ((mu | mv | mc | mn) < 0) return 0.f;
  return w[mu * su + mv * sv + mc * sc + mn * sn] * __ldg(scales + c) * __ldg(scales + c_real + n);
}

template <int PREC>
__global__ void pack_weights_kernel(const float* __restrict__ w, int k1, int k2, int c_real, int Cp, int j,
                                    int64_t su, int64_t sv, int64_t sc, int64_t sn, int BN, int kblocks,
                                    int ntiles, float* __restrict__ img, const int32_t* __restrict__ maps,
                                    const float* __restrict__ scales) {
  const int64_t total = (int64_t)ntiles * kblocks * BN * 8;  // 16-B chunks of one plane
  const int K = k1 * k2 * Cp;
  constexpr int kPer = PREC ? 8 : 4;       // elements per 16-B chunk
  constexpr int kBKe = PREC ? 64 : 32;     // elements per K block
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < total;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int chunk = q & 7;
    const int64_t rowq = q >> 3;
    const int r = rowq % BN;
    const int64_t tk = rowq / BN;
    const int kb = tk % kblocks;
    const int nt = tk / kblocks;
    const int n = nt * BN + r;
    float v[kPer];
#pragma unroll
    for (int e = 0; e < kPer; ++e)
      v[e] = weight_at(w, kb * kBKe + chunk * kPer + e, n, k1, k2, c_real, Cp, j, K, su, sv, sc, sn, maps, scales);
    const uint32_t off = sw128_off(r, chunk) / 4;  // in floats
    if constexpr (PREC == 1) {
      const int64_t plane = (int64_t)BN * 32;  // floats (= 128-B rows) per plane
      float* base = img + ((int64_t)nt * kblocks + kb) * plane;
      uint4 pk;
      pk.x = pack_bf16x2(v[0], v[1]);
      pk.y = pack_bf16x2(v[2], v[3]);
      pk.z = pack_bf16x2(v[4], v[5]);
      pk.w = pack_bf16x2(v[6], v[7]);
      *reinterpret_cast<uint4*>(base + off) = pk;
    } else {
      float hv[4], lv[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        hv[e] = __uint_as_float(to_tf32_rna(v[e]));
        lv[e] = v[e] - hv[e];
      }
      const int64_t plane = (int64_t)BN * 32;  // floats per hi (or lo) plane
      float* base = img + ((int64_t)nt * kblocks + kb) * 2 * plane;
      *reinterpret_cast<float4*>(base + off) = make_float4(hv[0], hv[1], hv[2], hv[3]);
      *reinterpret_cast<float4*>(base + plane + off) = make_float4(lv[0], lv[1], lv[2], lv[3]);
    }
  }
}

}  // namespace tobf

using namespace tobf;

static inline int prec_kbk(int prec) { return prec == TOBF_PREC_BF16 ? 64 : 32; }
static inline bool prec_ok(int prec) { return prec == TOBF_PREC_TF32X3 || prec == TOBF_PREC_BF16; }

extern "C" int tobf_conv_prepare_ex(tobf_conv_desc* descs, int n, int block_n, int prec, int64_t* total_tiles) {
  if (n < 0 || (block_n != 64 && block_n != 128) || (n > 0 && !descs) || !prec_ok(prec) || !total_tiles) {
    return tobf_fail(TOBF_E_INVALID, "tobf_conv_prepare: bad arguments");
  }
  const int kbk = prec_kbk(prec);
  int64_t acc = 0;
  for (int i = 0; i < n; ++i) {
    tobf_conv_desc& d = descs[i];
    if (d.Cp % 4 || d.Cpo % 4 || d.ldx % 4 || d.ldy % 4 || d.j < 1 || d.j > d.Cpo || d.k1 < 1 || d.k2 < 1 ||
        d.batch < 1 || d.Ho < 1 || d.Wo < 1 || d.nepi < 0 || d.nepi > TOBF_MAX_EPI) {
      return tobf_fail(TOBF_E_INVALID, "tobf_conv_prepare: descriptor %d violates layout invariants", i);
    }
    d.K = d.k1 * d.k2 * d.Cp;
    d.kblocks = (d.K + kbk - 1) / kbk;
    const int64_t M = (int64_t)d.batch * d.Ho * d.Wo;
    d.mtiles = (int)((M + kBM - 1) / kBM);
    d.ntiles = (d.j + block_n - 1) / block_n;
    d.tile_start = (int)acc;
    d.ksplit = 1;
    d.kper = d.kblocks;
    d.ws = nullptr;
    d.cnt = nullptr;
    acc += (int64_t)d.mtiles * d.ntiles;
  }
  if (acc >= (int64_t)1 << 31) return tobf_fail(TOBF_E_INVALID, "tobf_conv_prepare: too many tiles");
  *total_tiles = acc;
  return TOBF_OK;
}

extern "C" int tobf_conv_prepare(tobf_conv_desc* descs, int n, int block_n, int64_t* total_tiles) {
  return tobf_conv_prepare_ex(descs, n, block_n, TOBF_PREC_TF32X3, total_tiles);
}

#ifndef TOBF_SPLIT_TILES_PER_SM
#define TOBF_SPLIT_TILES_PER_SM 2
#endif
// Split policy: a group with fewer than 2 tiles per SM leaves SMs idle behind
// its longest tiles; cut the K loop of tiles clearly longer than ~1/4 of an
// SM's share of the group's work into units of U >= 16 K blocks (the partial
// write + read of a 128 x BN fp32 tile costs about as much as 3-4 K blocks of
// MMAs, hence the floor). Measured: splitting also in groups of 2-8 tiles per
// SM cost more in partial traffic than it won in balance (10.8 vs 10.6 ms).
extern "C" int tobf_conv_prepare_split_ex(tobf_conv_desc* descs, int n, int block_n, int prec, int sms,
                                          int max_split, float* ws_base, int32_t* cnt_base, int64_t* total_units,
                                          int64_t* ws_floats, int64_t* cnt_count) {
  int64_t tiles = 0;
  int rc = tobf_conv_prepare_ex(descs, n, block_n, prec, &tiles);
  if (rc != TOBF_OK) return rc;
  if (sms < 1 || max_split < 1 || !total_units || !ws_floats || !cnt_count)
    return tobf_fail(TOBF_E_INVALID, "tobf_conv_prepare_split: bad arguments");
  *ws_floats = 0;
  *cnt_count = 0;
  int64_t work = 0;
  for (int i = 0; i < n; ++i) work += (int64_t)descs[i].mtiles * descs[i].ntiles * descs[i].kblocks;
  // unit size: ~1/4 of one SM's share of the group's work (>= 16 K blocks), so
  // no single unit is long enough to leave the other SMs idle at the tail of
  // the greedy (longest-first) claim order; shorter tiles stay whole
  const int64_t per_unit = std::max<int64_t>(16, (work + 4 * (int64_t)sms - 1) / (4 * (int64_t)sms));
  const int64_t threshold = per_unit * 3 / 2;  // only clearly-too-long tiles are cut
  int64_t longest = 0;
  for (int i = 0; i < n; ++i) longest = std::max<int64_t>(longest, descs[i].kblocks);
  if (tiles >= TOBF_SPLIT_TILES_PER_SM * (int64_t)sms || longest <= threshold || max_split == 1) {
    *total_units = tiles;
    return TOBF_OK;
  }
  int64_t acc = 0, wsf = 0, cnts = 0;
  for (int i = 0; i < n; ++i) {
    tobf_conv_desc& d = descs[i];
    int s = d.kblocks > threshold ? (int)std::min<int64_t>(max_split, (d.kblocks + per_unit - 1) / per_unit) : 1;
    s = std::max(s, 1);
    const int kper = (d.kblocks + s - 1) / s;
    s = (d.kblocks + kper - 1) / kper;  // no empty unit
    const int64_t t = (int64_t)d.mtiles * d.ntiles;
    d.tile_start = (int)acc;
    d.ksplit = s;
    d.kper = kper;
    if (s > 1) {  // NULL bases: byte offsets, for the caller to rebase
      d.ws = reinterpret_cast<float*>(reinterpret_cast<uintptr_t>(ws_base) + wsf * sizeof(float));
      d.cnt = reinterpret_cast<int32_t*>(reinterpret_cast<uintptr_t>(cnt_base) + cnts * sizeof(int32_t));
      wsf += t * s * kBM * block_n;
      cnts += t;
    }
    acc += t * s;
  }
  if (acc >= (int64_t)1 << 31) return tobf_fail(TOBF_E_INVALID, "tobf_conv_prepare_split: too many units");
  *total_units = acc;
  *ws_floats = wsf;
  *cnt_count = cnts;
  return TOBF_OK;
}

extern "C" int tobf_conv_prepare_split(tobf_conv_desc* descs, int n, int block_n, int sms, int max_split,
                                       float* ws_base, int32_t* cnt_base, int64_t* total_units,
                                       int64_t* ws_floats, int64_t* cnt_count) {
  return tobf_conv_prepare_split_ex(descs, n, block_n, TOBF_PREC_TF32X3, sms, max_split, ws_base, cnt_base,
                                    total_units, ws_floats, cnt_count);
}

extern "C" int64_t tobf_wimg_bytes_ex(int32_t k1, int32_t k2, int32_t Cp, int32_t j, int32_t block_n, int32_t prec) {
  if (!prec_ok(prec)) return -1;
  const int kbk = prec_kbk(prec);
  const int64_t K = (int64_t)k1 * k2 * Cp;
  const int64_t kblocks = (K + kbk - 1) / kbk;
  const int64_t ntiles = (j + block_n - 1) / block_n;
  return ntiles * kblocks * (prec == TOBF_PREC_BF16 ? 1 : 2) * block_n * kRowBytes;
}

extern "C" int64_t tobf_wimg_bytes(int32_t k1, int32_t k2, int32_t Cp, int32_t j, int32_t block_n) {
  return tobf_wimg_bytes_ex(k1, k2, Cp, j, block_n, TOBF_PREC_TF32X3);
}

extern "C" int tobf_pack_weights_ex(const float* w, int32_t k1, int32_t k2, int32_t c_real, int32_t Cp, int32_t j,
                                    int64_t su, int64_t sv, int64_t sc, int64_t sn, const int32_t* maps,
                                    const float* scales, int32_t block_n, int32_t prec, void* wimg, void* stream) {
  if (!w || !wimg || Cp % 4 || c_real > Cp || (block_n != 64 && block_n != 128) || !prec_ok(prec) ||
      (maps == nullptr) != (scales == nullptr)) {
    return tobf_fail(TOBF_E_INVALID, "tobf_pack_weights: bad arguments");
  }
  const int kbk = prec_kbk(prec);
  const int K = k1 * k2 * Cp;
  const int kblocks = (K + kbk - 1) / kbk;
  const int ntiles = (j + block_n - 1) / block_n;
  const int64_t chunks = (int64_t)ntiles * kblocks * block_n * 8;
  const int threads = 256;
  const int64_t blocks = std::min<int64_t>((chunks + threads - 1) / threads, 148 * 16);
  if (prec == TOBF_PREC_BF16)
    pack_weights_kernel<1><<<(unsigned)blocks, threads, 0, (cudaStream_t)stream>>>(
        w, k1, k2, c_real, Cp, j, su, sv, sc, sn, block_n, kblocks, ntiles, static_cast<float*>(wimg), maps, scales);
  else
    pack_weights_kernel<0><<<(unsigned)blocks, threads, 0, (cudaStream_t)stream>>>(
        w, k1, k2, c_real, Cp, j, su, sv, sc, sn, block_n, kblocks, ntiles, static_cast<float*>(wimg), maps, scales);
  return tobf_cuda_check("tobf_pack_weights");
}

extern "C" int tobf_pack_weights(const float* w, int32_t k1, int32_t k2, int32_t c_real, int32_t Cp, int32_t j,
                                 int64_t su, int64_t sv, int64_t sc, int64_t sn, int32_t block_n, void* wimg,
                                 void* stream) {
  return tobf_pack_weights_ex(w, k1, k2, c_real, Cp, j, su, sv, sc, sn, nullptr, nullptr, block_n,
                              TOBF_PREC_TF32X3, wimg, stream);
}

extern "C" int tobf_pack_weights_gather(const float* w, int32_t k1, int32_t k2, int32_t c_real, int32_t Cp,
                                        int32_t j, int64_t su, int64_t sv, int64_t sc, int64_t sn,
                                        const int32_t* maps, const float* scales, int32_t block_n, void* wimg,
                                        void* stream) {
  if (!maps || !scales) return tobf_fail(TOBF_E_INVALID, "tobf_pack_weights_gather: null maps");
  return tobf_pack_weights_ex(w, k1, k2, c_real, Cp, j, su, sv, sc, sn, maps, scales, block_n, TOBF_PREC_TF32X3,
                              wimg, stream);
}

// ------------------------------------------------------------ TMA im2col maps
// cuTensorMapEncodeIm2col through the runtime's driver entry point (no link
// dependency on libcuda).
typedef CUresult (*EncodeIm2colFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const int*, const int*, cuuint32_t, cuuint32_t,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeIm2colFn encode_im2col_fn() {
  static EncodeIm2colFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return reinterpret_cast<EncodeIm2colFn>(p);
  }();
  return fn;
}

extern "C" int tobf_conv_tmaps(tobf_conv_desc* descs, int n, void* tmap_host, uint64_t tmap_dev, int* n_tma) {
  if (n < 0 || (n > 0 && (!descs || !tmap_host)) || (tmap_dev & 127) || !n_tma)
    return tobf_fail(TOBF_E_INVALID, "tobf_conv_tmaps: bad arguments");
  const EncodeIm2colFn enc = encode_im2col_fn();
  int count = 0;
  for (int i = 0; i < n; ++i) {
    tobf_conv_desc& d = descs[i];
    d.tma = 0;
    d.tmap = nullptr;
    // one load = 32 channels of one filter tap x 128 pixels (128-B rows,
    // 128B swizzle: the cp.async staging layout), so Cp % 32 == 0 only. A
    // variant loading 16/8/4-channel pieces for the other Cp was measured
    // slower than the cp.async gather for them (RN18 step conv 11.5 vs
    // 10.1 ms: the stem's 8 loads of 16-B rows per K block), so those
    // problems keep cp.async, in the SAME launch (per-tile A mode).
    const int cpp = 32;
    const bool ok = enc && d.Cp % cpp == 0 && d.k1 <= 256 && d.k2 <= 256 && d.stride >= 1 && d.stride <= 8 &&
                    d.pad <= 127 && d.pad - (d.k1 - 1) >= -128 && d.pad - (d.k2 - 1) >= -128 &&
                    (reinterpret_cast<uintptr_t>(d.x) & 15) == 0 && d.ldx % 4 == 0;
    if (!ok) continue;
    CUtensorMap* map = reinterpret_cast<CUtensorMap*>(static_cast<uint8_t*>(tmap_host) + 128 * (size_t)i);
    const cuuint64_t dims[4] = {(cuuint64_t)d.Cp, (cuuint64_t)d.W, (cuuint64_t)d.H, (cuuint64_t)d.batch};
    const cuuint64_t strides[3] = {(cuuint64_t)d.ldx * 4, (cuuint64_t)d.ldx * 4 * d.W,
                                   (cuuint64_t)d.ldx * 4 * d.W * d.H};
    const int lower[2] = {-d.pad, -d.pad};                              // (w, h)
    const int upper[2] = {d.pad - (d.k2 - 1), d.pad - (d.k1 - 1)};      // (w, h)
    const cuuint32_t estr[4] = {1, (cuuint32_t)d.stride, (cuuint32_t)d.stride, 1};
    const CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<float*>(d.x), dims, strides, lower,
                           upper, (cuuint32_t)cpp /*channels per pixel*/, kBM /*pixels per column*/, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE,
                           cpp == 32 ? CU_TENSOR_MAP_SWIZZLE_128B : cpp == 16 ? CU_TENSOR_MAP_SWIZZLE_64B
                           : cpp == 8 ? CU_TENSOR_MAP_SWIZZLE_32B : CU_TENSOR_MAP_SWIZZLE_NONE,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) continue;
    d.tmap = reinterpret_cast<const void*>(tmap_dev + 128 * (uint64_t)i);
    d.tma = cpp;
    ++count;
  }
  *n_tma = count;
  return TOBF_OK;
}

// Per-device launch state of one kernel variant: SM count and the one-time
// dynamic shared-memory opt-in (a context may drive several devices).
template <int BN, int PREC, int AM>
static int launch_conv(const tobf_conv_desc* d_descs, int n, int64_t total_tiles, int32_t* sched, cudaStream_t st) {
  constexpr int kMaxDev = 64;
  static int sms[kMaxDev] = {0};
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess || dev < 0 || dev >= kMaxDev)
    return tobf_fail(TOBF_E_CUDA, "tobf_conv_grouped: no current device");
  if (sms[dev] == 0) {
    int count = 0;
    cudaDeviceGetAttribute(&count, cudaDevAttrMultiProcessorCount, dev);
    e = cudaFuncSetAttribute(conv_tc_kernel<BN, PREC, AM>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             ConvCfg<BN, PREC>::kSmem);
    if (e != cudaSuccess || count < 1) return tobf_fail(TOBF_E_CUDA, "cudaFuncSetAttribute: %s", cudaGetErrorString(e));
    sms[dev] = count;
  }
  // claim 4 tiles at a time when there are many (short-tile levels: the stem,
  // 1x1 convs); one at a time otherwise (few long tiles: LPT balance)
  const int claim = total_tiles >= TOBF_CONV_CLAIM_MIN * (int64_t)sms[dev] ? TOBF_CONV_CLAIM : 1;
  const int grid = (int)std::min<int64_t>((total_tiles + claim - 1) / claim, sms[dev]);
  conv_tc_kernel<BN, PREC, AM><<<grid, kThreads, ConvCfg<BN, PREC>::kSmem, st>>>(d_descs, n, (int)total_tiles,
                                                                                sched, claim);
  return tobf_cuda_check("tobf_conv_grouped");
}

template <int AM>
static int launch_variant(const tobf_conv_desc* d_descs, int n, int64_t total_tiles, int block_n, int prec,
                          int32_t* sched, cudaStream_t st) {
  if (prec == TOBF_PREC_TF32X3) {
    if (block_n == 128) return launch_conv<128, 0, AM>(d_descs, n, total_tiles, sched, st);
    if (block_n == 64) return launch_conv<64, 0, AM>(d_descs, n, total_tiles, sched, st);
  } else if (prec == TOBF_PREC_BF16) {
    if (block_n == 128) return launch_conv<128, 1, AM>(d_descs, n, total_tiles, sched, st);
    if (block_n == 64) return launch_conv<64, 1, AM>(d_descs, n, total_tiles, sched, st);
  }
  return tobf_fail(TOBF_E_INVALID, "tobf_conv_grouped: block_n must be 64 or 128, prec 0 or 1");
}

extern "C" int tobf_conv_grouped_ex(const tobf_conv_desc* d_descs, int n, int64_t total_tiles, int block_n,
                                    int prec, int32_t* sched, void* stream) {
  if (n <= 0 || total_tiles <= 0) return TOBF_OK;
  if (!d_descs) return tobf_fail(TOBF_E_INVALID, "tobf_conv_grouped: null descriptors");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  // the A-operand mode of a launch is that of its problems (tobf_conv_tmaps);
  // block_n | TOBF_CONV_TMA marks a TMA-capable launch, | TOBF_CONV_TMA_ALL
  // one whose problems all take A by TMA
  const int am = (block_n & TOBF_CONV_TMA_ALL) ? 2 : (block_n & TOBF_CONV_TMA) ? 1 : 0;
  block_n &= 0xFF;
  if (prec == TOBF_PREC_TF32X3 || prec == TOBF_PREC_BF16) {
    if (am == 2) return launch_variant<2>(d_descs, n, total_tiles, block_n, prec, sched, st);
    return am == 1 ? launch_variant<1>(d_descs, n, total_tiles, block_n, prec, sched, st)
                   : launch_variant<0>(d_descs, n, total_tiles, block_n, prec, sched, st);
  } else {
    return tobf_fail(TOBF_E_INVALID, "tobf_conv_grouped: unknown precision %d", prec);
  }
  return tobf_fail(TOBF_E_INVALID, "tobf_conv_grouped: block_n must be 64 or 128");
}

extern "C" int tobf_conv_grouped(const tobf_conv_desc* d_descs, int n, int64_t total_tiles, int block_n,
                                 void* stream) {
  return tobf_conv_grouped_ex(d_descs, n, total_tiles, block_n, TOBF_PREC_TF32X3, nullptr, stream);
}

#ifdef TOBF_CONV_PROF
extern "C" int tobf_conv_prof_read(unsigned long long* out, int reset) {
  cudaMemcpyFromSymbol(out, g_conv_prof, sizeof(unsigned long long) * 32);
  if (reset) {
    unsigned long long z[32] = {0};
    cudaMemcpyToSymbol(g_conv_prof, z, sizeof(z));
  }
  return 0;
}
#endif

extern "C" int tobf_fault_async(int* host, void* stream) {
  if (host == nullptr) return tobf_fail(TOBF_E_INVALID, "tobf_fault_async: null host word");
  const cudaError_t e = cudaMemcpyFromSymbolAsync(host, g_tobf_fault, sizeof(int), 0, cudaMemcpyDeviceToHost,
                                                  static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return tobf_fail(TOBF_E_CUDA, "tobf_fault_async: %s", cudaGetErrorString(e));
  return TOBF_OK;
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
