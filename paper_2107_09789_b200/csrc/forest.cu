// Dimension attacker (PAPER §V-B): bagged random-
// forest regressors predict each Conv2D step's (c, j) from its trace features,
// and the dimension error rate DER = |c - c*|/c* + |j - j*|/j* (eq:DER) is
// averaged over the vanilla graph's conv layers — the metric the GA maximises
// in dimension mode, in place of LER.
//
// Forests are flat node tables (CART, sklearn layout): node n splits on
// feature[n] at threshold[n] (x <= t goes left), leaves have left[n] < 0 and
// carry value[n]. A tree's prediction is its leaf value; a forest's is the
// tree values summed in tree order in fp64 and divided by the tree count
// (sklearn's RandomForestRegressor.predict with n_jobs=1), rounded to the
// nearest positive integer. Features are compared as float32 (sklearn casts
// X to float32 before the traversal).
//
// Latency-bound pointer chasing over a few MB of node tables that sit in L2:
// one warp per (regressor, candidate, conv layer, target), its lanes walking
// 32 trees at once; the leaf values are summed in tree order (the fp64 sum
// order is part of the contract); a second tiny kernel folds the layers into
// DER in layer order.
#include <cmath>
#include <cstdint>

#include "tobf_internal.h"

namespace {

__global__ void __launch_bounds__(128) forest_predict_kernel(
    const double* __restrict__ feats, int32_t F, const int32_t* __restrict__ conv_rows,
    const int32_t* __restrict__ cand_off, int32_t ncand, int32_t n_layers, const int32_t* __restrict__ node_feat,
    const double* __restrict__ node_thr, const int32_t* __restrict__ node_left, const int32_t* __restrict__ node_right,
    const double* __restrict__ node_value, const int32_t* __restrict__ tree_root,
    const int32_t* __restrict__ forest_off, int32_t R, int32_t* __restrict__ pred) {
  // one warp per (regressor, candidate, layer, target); the lanes walk 32
  // trees at a time, then every lane sums the 32 leaf values in tree order
  // (shuffles), so the fp64 sum order is the sequential one
  const int lane = threadIdx.x & 31;
  const int64_t total = (int64_t)R * ncand * n_layers * 2;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t t = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); t < total; t += warps) {
    const int target = (int)(t & 1);  // 0: c, 1: j
    int64_t q = t >> 1;
    const int layer = (int)(q % n_layers);
    q /= n_layers;
    const int cand = (int)(q % ncand);
    const int r = (int)(q / ncand);
    const int32_t lo = cand_off[cand], hi = cand_off[cand + 1];
    if (hi - lo != n_layers) {  // conv steps do not line up with the vanilla layers
      if (lane == 0) pred[t] = 0;
      continue;
    }
    const double* x = feats + (int64_t)conv_rows[lo + layer] * F;
    const int f = 2 * r + target;
    const int32_t t0 = forest_off[f], t1 = forest_off[f + 1];
    double sum = 0.0;
    for (int32_t base = t0; base < t1; base += 32) {
      double leaf = 0.0;
      if (base + lane < t1) {
        int32_t n = tree_root[base + lane];
        while (node_left[n] >= 0) {
          const double v = (double)(float)__ldg(x + node_feat[n]);
          n = v <= node_thr[n] ? node_left[n] : node_right[n];
        }
        leaf = node_value[n];
      }
      const int cnt = min(32, (int)(t1 - base));
      for (int k = 0; k < cnt; ++k) sum += __shfl_sync(0xffffffffu, leaf, k);
    }
    if (lane == 0) pred[t] = (int32_t)fmax(1.0, floor(sum / (double)(t1 - t0) + 0.5));
  }
}

__global__ void der_kernel(const int32_t* __restrict__ pred, const int32_t* __restrict__ truth, int32_t ncand,
                           int32_t n_layers, int32_t R, double* __restrict__ der) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;  // r * ncand + cand
  if (i >= (int64_t)R * ncand) return;
  const int32_t* p = pred + i * n_layers * 2;
  if (p[0] == 0) {  // unaligned candidate (see forest_predict_kernel)
    der[i] = -1.0;
    return;
  }
  double s = 0.0;
  for (int l = 0; l < n_layers; ++l) {
    const double c0 = truth[2 * l], j0 = truth[2 * l + 1];
    s += fabs((double)p[2 * l] - c0) / c0 + fabs((double)p[2 * l + 1] - j0) / j0;
  }
  der[i] = s / (double)n_layers;
}

}  // namespace

extern "C" int tobf_forest_der(const double* feats, int32_t F, const int32_t* conv_rows, const int32_t* cand_off,
                               int32_t ncand, int32_t n_layers, const int32_t* truth, const int32_t* node_feat,
                               const double* node_thr, const int32_t* node_left, const int32_t* node_right,
                               const double* node_value, const int32_t* tree_root, const int32_t* forest_off,
                               int32_t R, int32_t* pred, double* der, void* stream) {
  if (ncand <= 0) return TOBF_OK;
  if (!feats || !conv_rows || !cand_off || !truth || !node_feat || !node_thr || !node_left || !node_right ||
      !node_value || !tree_root || !forest_off || !pred || !der || F < 1 || n_layers < 1 || R < 1)
    return tobf_fail(TOBF_E_INVALID, "tobf_forest_der: bad arguments");
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t outputs = (int64_t)R * ncand * n_layers * 2;  // one warp each, 4 warps per CTA
  const int grid = (int)std::min<int64_t>((outputs + 3) / 4, 148 * 16);
  forest_predict_kernel<<<grid, 128, 0, st>>>(feats, F, conv_rows, cand_off, ncand, n_layers, node_feat, node_thr,
                                              node_left, node_right, node_value, tree_root, forest_off, R, pred);
  der_kernel<<<(int)(((int64_t)R * ncand + 127) / 128), 128, 0, st>>>(pred, truth, ncand, n_layers, R, der);
  return tobf_cuda_check("tobf_forest_der");
}
