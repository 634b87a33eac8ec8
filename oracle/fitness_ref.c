/*
 * fitness_ref.c — CPU restatement of the fitness stage (TEST ORACLE ONLY).
 *
 * The reference package has no attacker / fitness code; the behaviour is
 * restated from the paper and spec:
 *   - LSTM sequence predictor + CTC ("single-layer LSTM ... CTC",
 *     :432 hidden sizes, :623 bagging of 3 case-C predictors H=128/256/512);
 *   - greedy CTC decode (argmax per step, collapse repeats, drop blank);
 *   - Levenshtein / LER (LER = ED/|L*|);
 *   - Eq. 10 reward (eps = 0.05 SPEC.md:590).
 * Numerics contract: fixed-order fmaf
 * accumulation, transcendentals from IEEE-only operations, compiled with
 * -ffp-contract=off, so the GPU kernels can be bit-exact against this file.
 *
 * Build: gcc -O2 -ffp-contract=off -fPIC -shared (oracle/build.py).
 */
#include <math.h>
#include <stdint.h>
#include <string.h>

static float f_from_bits(uint32_t u) {
  float f;
  memcpy(&f, &u, sizeof f);
  return f;
}

/* exp: clamp, n = rint(x*log2e), Cody-Waite r = x - n*ln2 (hi/lo), degree-7
 * Taylor via fmaf Horner, scale by 2^n through the exponent field. */
static float ref_expf(float x) {
  float n, r, p, scale;
  if (x > 88.0f) x = 88.0f;
  if (x < -87.0f) x = -87.0f;
  n = rintf(x * 1.44269504088896341f);
  r = fmaf(n, -0.693145751953125f, x);
  r = fmaf(n, -1.428606765330187045e-06f, r);
  p = 1.98412698412698413e-04f;
  p = fmaf(p, r, 1.38888888888888889e-03f);
  p = fmaf(p, r, 8.33333333333333333e-03f);
  p = fmaf(p, r, 4.16666666666666667e-02f);
  p = fmaf(p, r, 1.66666666666666667e-01f);
  p = fmaf(p, r, 0.5f);
  p = fmaf(p, r, 1.0f);
  p = fmaf(p, r, 1.0f);
  scale = f_from_bits((uint32_t)((int)n + 127) << 23);
  return p * scale;
}

static float ref_sigmoid(float x) { return 1.0f / (1.0f + ref_expf(-x)); }

static float ref_tanh(float x) {
  float e = ref_expf(-2.0f * fabsf(x));
  float t = (1.0f - e) / (1.0f + e);
  return x < 0.0f ? -t : t;
}

/* log(1+v), v >= 0: y = m*2^e, m folded into [sqrt(1/2), sqrt(2)],
 * log m = 2s(1 + s^2/3 + ... + s^22/23), s = (m-1)/(m+1). */
static double ref_log1p(double v) {
  double y = 1.0 + v, m, f, s, s2, p;
  uint64_t bits;
  int e;
  memcpy(&bits, &y, 8);
  e = (int)((bits >> 52) & 0x7ff) - 1023;
  bits = (bits & 0x000fffffffffffffULL) | 0x3ff0000000000000ULL;
  memcpy(&m, &bits, 8);
  if (m > 1.4142135623730951) {
    m = m * 0.5;
    e += 1;
  }
  f = m - 1.0;
  s = f / (2.0 + f);
  s2 = s * s;
  p = 1.0 / 23.0;
  p = fma(p, s2, 1.0 / 21.0);
  p = fma(p, s2, 1.0 / 19.0);
  p = fma(p, s2, 1.0 / 17.0);
  p = fma(p, s2, 1.0 / 15.0);
  p = fma(p, s2, 1.0 / 13.0);
  p = fma(p, s2, 1.0 / 11.0);
  p = fma(p, s2, 1.0 / 9.0);
  p = fma(p, s2, 1.0 / 7.0);
  p = fma(p, s2, 1.0 / 5.0);
  p = fma(p, s2, 1.0 / 3.0);
  p = fma(p, s2, 1.0);
  return fma((double)e, 0.6931471805599453, 2.0 * s * p);
}

/* Output-head dot product in the lane-partition + xor-butterfly order:
 * lane l accumulates k = l, l+32, ... with fmaf from 0; then for
 * off = 16,8,4,2,1: p[l] = p[l] + p[l ^ off]; result = p[0]. */
static float head_dot(const float* w, const float* h, int H) {
  float p[32], q[32];
  int l, k, off;
  for (l = 0; l < 32; ++l) {
    float acc = 0.0f;
    for (k = l; k < H; k += 32) acc = fmaf(w[k], h[k], acc);
    p[l] = acc;
  }
  for (off = 16; off; off >>= 1) {
    for (l = 0; l < 32; ++l) q[l] = p[l] + p[l ^ off];
    memcpy(p, q, sizeof p);
  }
  return p[0];
}

/*
 * One trace: rows[t*9 + k] fp64 features (t < T), first F used.
 * Weights: w_ihT [F][4H], w_hhT [H][4H], b [4H], w_out [NC][H], b_out [NC].
 * Scratch: h [H], c [H], g [4H], hn [H].
 * Returns the number of decoded tokens written to tokens[].
 */
int ref_lstm_ctc_one(const double* rows, int T, int F, int H, int NC, const float* w_ihT, const float* w_hhT,
                     const float* b, const float* w_out, const float* b_out, float* h, float* c, float* g,
                     float* hn, int8_t* tokens) {
  int t, j, k, q, ntok = 0, prev = 0;
  const int G = 4 * H;
  float x[16], logit[8];
  for (j = 0; j < H; ++j) h[j] = c[j] = 0.0f;
  for (t = 0; t < T; ++t) {
    for (k = 0; k < F; ++k) x[k] = (float)ref_log1p(rows[(int64_t)t * 9 + k]);
    for (q = 0; q < G; ++q) g[q] = b[q];
    for (k = 0; k < F; ++k)
      for (q = 0; q < G; ++q) g[q] = fmaf(w_ihT[(int64_t)k * G + q], x[k], g[q]);
    for (k = 0; k < H; ++k)
      for (q = 0; q < G; ++q) g[q] = fmaf(w_hhT[(int64_t)k * G + q], h[k], g[q]);
    for (j = 0; j < H; ++j) {
      float ig = ref_sigmoid(g[j]);
      float fg = ref_sigmoid(g[H + j]);
      float gg = ref_tanh(g[2 * H + j]);
      float og = ref_sigmoid(g[3 * H + j]);
      c[j] = fmaf(fg, c[j], ig * gg);
      hn[j] = og * ref_tanh(c[j]);
    }
    memcpy(h, hn, sizeof(float) * H);
    for (q = 0; q < NC; ++q) logit[q] = b_out[q] + head_dot(w_out + (int64_t)q * H, h, H);
    {
      int best = 0;
      for (q = 1; q < NC; ++q)
        if (logit[q] > logit[best]) best = q;
      if (best != 0 && best != prev) tokens[ntok++] = (int8_t)best;
      prev = best;
    }
  }
  return ntok;
}

/* Unit-cost edit distance, two-row dynamic programme. */
int ref_levenshtein(const int8_t* a, int n, const int8_t* b, int m, int* row0, int* row1) {
  int i, j;
  for (j = 0; j <= m; ++j) row0[j] = j;
  for (i = 1; i <= n; ++i) {
    row1[0] = i;
    for (j = 1; j <= m; ++j) {
      int del = row0[j] + 1, ins = row1[j - 1] + 1, sub = row0[j - 1] + (a[i - 1] != b[j - 1]);
      int v = del < ins ? del : ins;
      row1[j] = v < sub ? v : sub;
    }
    memcpy(row0, row1, sizeof(int) * (m + 1));
  }
  return row0[m];
}

/* CPython 3.12 float sum(): Neumaier compensation, applied at the end only
 * when non-zero and finite. */
double ref_py_sum(const double* v, int n, int stride) {
  double s = 0.0, comp = 0.0;
  int i;
  for (i = 0; i < n; ++i) {
    double x = v[(int64_t)i * stride], t = s + x;
    if (fabs(s) >= fabs(x)) comp += (s - t) + x;
    else comp += (x - t) + s;
    s = t;
  }
  if (comp != 0.0 && isfinite(comp)) s += comp;
  return s;
}

/* Eq. 10: R = mean(LER) / (eps + ((T - (1+B)T*)/T*)^2), 0 if infeasible. */
double ref_eq10(const double* lers, int npred, double T, int feasible, double Tstar, double budget, double eps,
                double* mean_out) {
  double mean = ref_py_sum(lers, npred, 1) / (double)npred, dev;
  *mean_out = mean;
  if (!feasible) return 0.0;
  dev = (T - (1.0 + budget) * Tstar) / Tstar;
  return mean / (eps + dev * dev);
}
