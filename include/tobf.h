/*
 * tobf.h — C ABI of libtobf.so, the sm_100a engine behind the
 * paper_2107_09789_b200 drop-in for traceobf's candidate-evaluation path
 * (NeurObfuscator, arXiv 2107.09789).
 *
 * Every entry point is extern "C", takes plain pointers / sizes, never throws,
 * and returns 0 on success or a negative TOBF_E* code; tobf_last_error()
 * returns a thread-local message for the most recent failure. Device pointers
 * are caller-owned; `stream` is a cudaStream_t passed as void* (NULL = legacy
 * default stream). All launches are asynchronous on `stream`.
 *
 * Reference interfaces each group replaces (paths relative to the reference
 * package pkg/src/traceobf/):
 *   executor     interpreter.py:22-30 conv2d, :33-35 maxpool, :38-41 softmax,
 *                :44-72 _eval_node, :75-90 execute
 *   verdict      interpreter.py:93-118 equivalence_check (compare + reduce)
 *   trace        fusion.py:159-180 default_schedule, :141-156 candidate_triples,
 *                costmodel.py:166-232 profile_kernel, :96-98 Trace.total_latency
 *   fitness      SPEC.md:471-486 levenshtein/ler, PAPER.md:425,432 LSTM+CTC,
 *                PAPER.md:487 / SPEC.md:563-571 Eq. 10 fitness (no reference code)
 */
#ifndef TOBF_H_
#define TOBF_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TOBF_OK 0
#define TOBF_E_INVALID -1
#define TOBF_E_CUDA -2
#define TOBF_E_FAULT -3 /* device-side protocol timeout (see tobf_check_fault) */

/* ------------------------------------------------------------------ executor */

/* Epilogue step applied to each conv output element, in order. */
#define TOBF_EPI_NONE 0
#define TOBF_EPI_AFFINE 1     /* v = v*ptr[c] + ptr[ldc + c]   (folded BatchNorm); aux = ldc */
#define TOBF_EPI_RELU 2       /* v = max(v, 0) */
#define TOBF_EPI_ADD_TENSOR 3 /* v += ptr[pixel*aux + c]       (residual / branch sum); aux = channel stride */
#define TOBF_EPI_ADD_CONST 4  /* v += ptr[((n % aux)*HoWo + p)*Cpo + c] (dummy-add constant); aux = batch period */
#define TOBF_MAX_EPI 6

typedef struct tobf_epi_step {
  int32_t op;
  int32_t aux;
  const float* ptr;
} tobf_epi_step;

/* One implicit-GEMM convolution problem (a Conv2D, or a Linear expressed as a
 * full-extent convolution). Activations are NHWC float32 with the channel
 * count padded to a multiple of 4 (pad channels hold zeros). GEMM view:
 * M = batch*Ho*Wo output pixels, N = j output channels, K = k1*k2*Cp. */
typedef struct tobf_conv_desc {
  const float* x;    /* input view, first channel of the view */
  const float* wimg; /* packed weight image from tobf_pack_weights */
  float* y;          /* output view, first channel of the view */
  int32_t batch, H, W, Cp;   /* input geometry; Cp = padded channels of the view */
  int32_t Ho, Wo, Cpo, j;    /* output geometry; Cpo = roundup(j,4) channels written */
  int32_t k1, k2, stride, pad;
  int32_t K, kblocks, mtiles, ntiles; /* filled by tobf_conv_prepare */
  int32_t tile_start, nepi, ldx, ldy; /* ldx/ldy = channel stride of the x/y buffers */
  tobf_epi_step epi[TOBF_MAX_EPI];
  /* split-K (filled by tobf_conv_prepare / tobf_conv_prepare_split): a tile's
   * K blocks are cut into `ksplit` work units of `kper` blocks; units write
   * fp32 partial tiles to `ws` and the last unit of a tile (per-tile arrival
   * counter in `cnt`, zero between launches) sums them in unit order and runs
   * the epilogue. ksplit = 1: no workspace. */
  float* ws;
  int32_t* cnt;
  int32_t ksplit, kper;
  /* A operand by TMA im2col (filled by tobf_conv_tmaps): `tmap` = DEVICE
   * address of this problem's 128-B CUtensorMap (im2col mode, NHWC fp32,
   * 32 channels x 128 output pixels per load, 128B swizzle), tma = 32.
   * tma = 0: the A operand is gathered with cp.async. */
  const void* tmap;
  int32_t tma;
  /* Paired problem (executor stem pairing): two 64-channel problems reading
   * the same A (the input's im2col matrix) with the same weights, run as ONE
   * 128-channel problem: columns [0, 64) are written to `y`, [64, 128) to
   * `y2` (same ldy), each half's folded BatchNorm (the chain's AFFINE step)
   * read from its own array (`aff2` for the upper half). 0 = unpaired. */
  int32_t pair;
  float* y2;
  const float* aff2;
} tobf_conv_desc;

/* Conv arithmetic (the `prec` argument of the *_ex entry points):
 *   TOBF_PREC_TF32X3  fp32-faithful 3xTF32 tcgen05 kind::tf32 (the 1e-4 fp32
 *                     contract of interpreter.py:93-118's comparisons)
 *   TOBF_PREC_BF16    bf16 operands (activations rounded on the way into
 *                     tensor memory, bf16 weight image), kind::f16, fp32
 *                     accumulation (BASELINE's 2e-2 bf16 mode, cfg4)
 * A weight image, a prepared descriptor group and a launch must agree on it. */
#define TOBF_PREC_TF32X3 0
#define TOBF_PREC_BF16 1

/* Fill K/kblocks/mtiles/ntiles/tile_start for a group of descriptors (host
 * memory) for the given N tile width (64 or 128); returns total tile count
 * (no split-K: ksplit = 1). */
int tobf_conv_prepare(tobf_conv_desc* descs, int n, int block_n, int64_t* total_tiles);

int tobf_conv_prepare_ex(tobf_conv_desc* descs, int n, int block_n, int prec, int64_t* total_tiles);

/* As tobf_conv_prepare, and, in groups with fewer than 2 tiles per SM, split
 * the K loop of tiles longer than ~1/4 of one SM's share of the group's work
 * (work units of >= 16 K blocks, <= max_split units per tile). `tile_start` then counts work units. `ws` /
 * `cnt` of split problems are set to ws_base / cnt_base plus their offsets
 * (NULL bases: the byte offsets themselves, for the caller to rebase);
 * *ws_floats and *cnt_count return the workspace (floats) and counter
 * (int32, zero-initialised by the caller) extents this group needs. A group
 * may share the workspace with any other group launched on the same stream. */
int tobf_conv_prepare_split(tobf_conv_desc* descs, int n, int block_n, int sms, int max_split, float* ws_base,
                            int32_t* cnt_base, int64_t* total_units, int64_t* ws_floats, int64_t* cnt_count);

int tobf_conv_prepare_split_ex(tobf_conv_desc* descs, int n, int block_n, int prec, int sms, int max_split,
                               float* ws_base, int32_t* cnt_base, int64_t* total_units, int64_t* ws_floats,
                               int64_t* cnt_count);

/* Bytes of the packed weight image for a conv with the given geometry. */
int64_t tobf_wimg_bytes(int32_t k1, int32_t k2, int32_t Cp, int32_t j, int32_t block_n);
int64_t tobf_wimg_bytes_ex(int32_t k1, int32_t k2, int32_t Cp, int32_t j, int32_t block_n, int32_t prec);

/* Pack a float32 weight tensor into the tile-major, tf32 hi/lo split,
 * 128B-swizzled operand image the conv kernel streams with bulk copies.
 * Weight element (u,v,c,n) is read at w[u*su + v*sv + c*sc + n*sn] for
 * c < c_real (zero for c_real <= c < Cp). HWIO conv weights (k1,k2,c,j):
 * su=k2*c*j, sv=c*j, sc=j, sn=1. */
int tobf_pack_weights(const float* w, int32_t k1, int32_t k2, int32_t c_real, int32_t Cp, int32_t j,
                      int64_t su, int64_t sv, int64_t sc, int64_t sn, int32_t block_n, void* wimg,
                      void* stream);

/* As tobf_pack_weights for a knob-derived weight (widen / kernel-widen /
 * branch, transforms.py:115-335) that is never materialised: element
 * (u,v,c,n) = w[mu[u]*su + mv[v]*sv + mc[c]*sc + mn[n]*sn] * s_c[c] * s_n[n],
 * 0 where any map entry is -1. `maps` (device) = [mu(k1) | mv(k2) | mc(c_real)
 * | mn(j)] int32, `scales` (device) = [s_c(c_real) | s_n(j)] float32. */
int tobf_pack_weights_gather(const float* w, int32_t k1, int32_t k2, int32_t c_real, int32_t Cp, int32_t j,
                             int64_t su, int64_t sv, int64_t sc, int64_t sn, const int32_t* maps,
                             const float* scales, int32_t block_n, void* wimg, void* stream);

/* Either precision; `maps`/`scales` both NULL (plain) or both set (gather). */
int tobf_pack_weights_ex(const float* w, int32_t k1, int32_t k2, int32_t c_real, int32_t Cp, int32_t j,
                         int64_t su, int64_t sv, int64_t sc, int64_t sn, const int32_t* maps, const float* scales,
                         int32_t block_n, int32_t prec, void* wimg, void* stream);

/* Grouped 3xTF32 tcgen05 implicit-GEMM convolution over `n` problems whose
 * descriptors live in DEVICE memory (prepared with tobf_conv_prepare). */
int tobf_conv_grouped(const tobf_conv_desc* d_descs, int n, int64_t total_tiles, int block_n, void* stream);

/* TMA im2col tensor maps: for every descriptor (host memory, pointers
 * already final) with Cp % 32 == 0 (a 32-channel K block never straddles
 * two filter taps), k1, k2 <= 256, stride <= 8 and pad <= 127, encode its
 * CUtensorMap into tmap_host + 128*i and set descs[i].tmap = tmap_dev +
 * 128*i, tma = 32; every other descriptor gets tma = 0 (its A operand is
 * gathered with cp.async, also inside a TMA-capable launch). tmap_host /
 * tmap_dev must hold 128*n bytes, tmap_dev 128-B aligned; the caller copies
 * tmap_host to tmap_dev before the launch. *n_tma returns the count of
 * tma != 0 descriptors. */
int tobf_conv_tmaps(tobf_conv_desc* descs, int n, void* tmap_host, uint64_t tmap_dev, int* n_tma);

/* Either precision. `sched`: two int32 of DEVICE memory, zero before the
 * first launch, the launch-wide tile-claim counters (the launch's last CTA
 * re-zeroes them); give every stream that may run conv launches concurrently
 * its own pair. NULL: a module-global pair per kernel variant (launches of
 * one variant must then be stream-ordered). */
int tobf_conv_grouped_ex(const tobf_conv_desc* d_descs, int n, int64_t total_tiles, int block_n, int prec,
                         int32_t* sched, void* stream);
/* block_n | TOBF_CONV_TMA: a TMA-capable launch — problems with tma != 0
 * get their A operand by TMA im2col (cp.async.bulk.tensor.4d...im2col, one
 * load per 32-channel K block of 128 output pixels, issued by a dedicated
 * warp), the others by the cp.async gather. Without the flag every problem
 * uses cp.async (tma ignored). */
#define TOBF_CONV_TMA 0x100
/* block_n | TOBF_CONV_TMA | TOBF_CONV_TMA_ALL: every problem of the launch
 * has tma != 0 (the kernel variant without the cp.async gather). */
#define TOBF_CONV_TMA_ALL 0x200

/* Generic fused element-wise / pooling / copy ops (one op per descriptor). */
#define TOBF_OP_MAXPOOL 1  /* y = maxpool(x, window=a0, stride=a1) */
#define TOBF_OP_EPI 2      /* y = epilogue-chain(x) (standalone BN / ReLU / Add) */
#define TOBF_OP_COPYCH 3   /* y[..., a0:a0+C] = x[..., a1:a1+C] channel copy (Concat / Slice) */
#define TOBF_OP_SOFTMAX 4  /* y = softmax over channels (spatial 1x1 or per pixel) */

typedef struct tobf_ew_desc {
  const float* x;
  float* y;
  int32_t op, batch, H, W;   /* input geometry */
  int32_t C, ldx, Ho, Wo;    /* C = channels processed; ldx = input channel stride */
  int32_t ldy, a0, a1, nepi; /* ldy = output channel stride */
  int64_t work_start;        /* prefix of work items, each range padded to a multiple of 32 (tobf_ew_prepare) */
  int32_t Cpo, pad_;         /* output channels to write (zero-fill C..Cpo) */
  tobf_epi_step epi[TOBF_MAX_EPI];
} tobf_ew_desc;

int tobf_ew_prepare(tobf_ew_desc* descs, int n, int64_t* total_work);
int tobf_ew_grouped(const tobf_ew_desc* d_descs, int n, int64_t total_work, void* stream);

/* Equivalence verdict pieces (interpreter.py:114-117), bit-exact fp32:
 * for each pair p: worst[p] = max |a-b|/(1+|b|), ok[p] = all(|a-b| <= tol*(1+|b|)).
 * a/b are NHWC-padded buffers of `pairs` outputs each `count` pixels x C channels
 * (ld = channel stride); `b_list[p]`, `a_list[p]` are device pointer arrays. */
int tobf_equiv_compare(const float* const* a_list, const float* const* b_list, int pairs, int64_t pixels,
                       int32_t C, int32_t ld, float tol, float* worst, int32_t* ok, void* stream);

/* NHWC(padded) -> NCHW (dense) output unpacking. */
int tobf_nhwc_to_nchw(const float* x, float* y, int32_t batch, int32_t C, int32_t H, int32_t W, int32_t ld,
                      void* stream);
/* NCHW (dense) -> NHWC(padded) input packing, pad channels zeroed. */
int tobf_nchw_to_nhwc(const float* x, float* y, int32_t batch, int32_t C, int32_t H, int32_t W, int32_t ld,
                      void* stream);

/* im2col of a staged NHWC(padded) input for a k1 x k2 conv (stride, pad)
 * over its first c channels: out[b][yo][xo][Kp], element k = (u*k2 + v)*c + ch
 * (the weights' (u, v, c) order), zero past K = k1*k2*c and outside the image.
 * The executor's path for convs reading the graph input with c % 32 != 0
 * (interpreter.py:22-30's conv2d as a 1x1 GEMM over the shared matrix). */
int tobf_im2col(const float* x, int32_t batch, int32_t H, int32_t W, int32_t ldx, int32_t c, int32_t k1, int32_t k2,
                int32_t stride, int32_t pad, int32_t Ho, int32_t Wo, int32_t Kp, float* out, void* stream);

/* ------------------------------------------------------------------ trace */

/* One kernel of a compiled graph, reduced to the exact integers the cost
 * model reads (costmodel.py:166-232). */
typedef struct tobf_kern_desc {
  int64_t work, fused_work, fused_bytes;
  int64_t in_bytes, w_bytes, out_bytes;
  int32_t tiled;        /* anchor is Conv2D or MaxPool */
  int32_t is_conv;      /* Conv2D (else MaxPool) when tiled */
  int32_t c, k1, k2, s; /* conv: c,k1,k2,stride; pool: c=channels, k1=k2=window, s=stride */
  int32_t H, W, channel_like;  /* out height/width; attrs j (or channels) */
  int32_t reuse_x_stream;      /* non-tiled: Linear j else 1 */
  int32_t ty[3], tx[3];        /* schedule factor triples (input for profile, output of search) */
  int32_t unroll, label;       /* label: OperatorKind code or -1 */
  int32_t has_shape;           /* 0 -> degenerate zero step */
  int32_t strategy;            /* schedule strategy k (fusion.py:124-134), 0 = none */
  int32_t sig_index;           /* row of the signature table holding this kernel's default schedule */
  int32_t resolved;            /* signature table rows: 1 = schedule known (memo hit), skip the search */
} tobf_kern_desc;

typedef struct tobf_device_profile {
  int64_t macs_per_cycle, launch_overhead, l1_bytes, l2_bytes, sm_count;
} tobf_device_profile;

/* Brute-force default_schedule for `n` kernels (DEVICE descriptor array):
 * writes the lexicographic-argmin (ty, tx) into d_descs[i].ty/tx. */
int tobf_schedule_search(tobf_kern_desc* d_descs, int n, const tobf_device_profile* prof, void* stream);

/* Per kernel: (ty, tx) := d_sigs[sig_index].(ty, tx), then modify_schedule
 * with the kernel's strategy (fusion.py:105-134) — the memoised default
 * schedule lookup of compile_graph (costmodel.py:276-284) on the device. */
int tobf_resolve_schedules(tobf_kern_desc* d_kern, int n, const tobf_kern_desc* d_sigs, void* stream);

/* profile_kernel for every kernel: feats[i*9 + f] in FEATURE_NAMES order
 * (cycles, dram_read, dram_write, l1_tx, l1_util, l1_hit, l2_tx, l2_util, l2_hit). */
int tobf_profile_kernels(const tobf_kern_desc* d_descs, int n, const tobf_device_profile* prof, double* feats,
                         void* stream);

/* Per-candidate CPython-3.12 (Neumaier) sum of cycles: candidate c owns
 * kernels [offsets[c], offsets[c+1]). */
int tobf_trace_totals(const double* feats, const int32_t* offsets, int ncand, double* totals, void* stream);

/* ------------------------------------------------------------------ fitness */

/* Batched single-layer LSTM sequence predictor + linear head + greedy CTC.
 * Trace b owns feature rows [offsets[b], offsets[b+1]) of `feats` (fp64,
 * 9 columns in FEATURE_NAMES order, as written by tobf_profile_kernels); the
 * first F columns are normalised x = (float)log1p(v) on the fly.
 * Weights (fp32, gate order i,f,g,o): w_ihT [F][4H], w_hhT [H][4H], b [4H],
 * w_out [NC][H], b_out [NC]. Output: tokens [B][T_max] int8 decoded labels
 * (argmax, collapse repeats, drop blank 0), ntok[B]. T_max >= longest trace. */
int tobf_lstm_ctc(const double* feats, const int32_t* offsets, int32_t B, int32_t F, int32_t H, int32_t NC,
                  const float* w_ihT, const float* w_hhT, const float* b, const float* w_out, const float* b_out,
                  int8_t* tokens, int32_t T_max, int32_t* ntok, void* stream);

/* Unit-cost Levenshtein distance, one warp per pair, against a single truth.
 * pred: [B][T_max] int8 with lengths ntok; truth[tlen]. ed[B], ler[B] = ed/tlen. */
int tobf_levenshtein(const int8_t* pred, const int32_t* ntok, int32_t B, int32_t T_max, const int8_t* truth,
                     int32_t tlen, int32_t* ed, double* ler, void* stream);

/* Eq. 10 reward per candidate: R = mean_i(ler[i*ncand + c]) / (eps + ((T-(1+budget)T*)/T*)^2),
 * 0 where feasible[c] == 0. */
int tobf_fitness_eq10(const double* ler, int32_t npred, int32_t ncand, const double* T, const int32_t* feasible,
                      double Tstar, double budget, double eps, double* R, double* mean_ler, void* stream);

/* Dimension attacker (no reference code): R bagged
 * random-forest regressors (forest 2r predicts c, 2r+1 predicts j) on the
 * feature rows (F fp64 per kernel step, compared as float32) of each
 * candidate's Conv2D steps conv_rows[cand_off[c] .. cand_off[c+1]); forests
 * are flat CART node tables (left < 0 = leaf), trees of forest f are
 * tree_root[forest_off[f] .. forest_off[f+1]); a forest predicts
 * max(1, floor(mean of its trees' leaf values, summed in tree order, + 0.5)).
 * pred: (R, ncand, n_layers, 2) int32; der[r*ncand + c] = mean over layers of
 * |c-c*|/c* + |j-j*|/j* against truth (n_layers x 2: c*, j*), or -1 when the
 * candidate's conv step count != n_layers. */
int tobf_forest_der(const double* feats, int32_t F, const int32_t* conv_rows, const int32_t* cand_off,
                    int32_t ncand, int32_t n_layers, const int32_t* truth, const int32_t* node_feat,
                    const double* node_thr, const int32_t* node_left, const int32_t* node_right,
                    const double* node_value, const int32_t* tree_root, const int32_t* forest_off, int32_t R,
                    int32_t* pred, double* der, void* stream);

/* ------------------------------------------------------------------ misc */
const char* tobf_last_error(void);
int tobf_version(void);
/* Reads and clears the device fault word; returns TOBF_E_FAULT if a bounded
 * wait timed out since the last check. */
int tobf_check_fault(void* stream);
/* Enqueues a read of that fault word into ``host`` (pinned, 4 bytes) on
 * ``stream`` without synchronising: a batch's results and its fault word come
 * back together behind its last kernel; a nonzero word is then raised (and
 * cleared) by tobf_check_fault. */
int tobf_fault_async(int* host, void* stream);
int tobf_device_sync(void);

#ifdef __cplusplus
}
#endif
#endif /* TOBF_H_ */
