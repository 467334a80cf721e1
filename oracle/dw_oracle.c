/*
 * dw_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * The plain, slow, obviously-correct CPU oracle for the depthwise-convolution
 * training layer of arXiv 1803.09926 ("Diagonalwise Refactorization").  Only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * leg may load it.  It shares no code, header, table or helper with the CUDA
 * path (paper_1803_09926_b200/csrc); neither includes the other.
 *
 * Everything is double precision, nested loops in definition order, no
 * blocking, no fusion, single-threaded by default.  For the
 * all-cores CPU baseline oracle_set_threads(t > 1) splits
 * the OUTER loops (images x channels for a1/a2, output channels for a3) over t
 * OpenMP threads; each output element is still summed by one thread in the same
 * order, so results are bitwise identical to the single-thread run (tested).  Every product of two
 * fp32 (or bf16) inputs is exact in double, so the only error is the double
 * summation, <= (n-1) * 2^-53 * sum|t|.  Each function also
 * returns, per output element, the sum of |terms| that the parity tolerance is
 * stated in (BASELINE.json north_star "1e-5 * sum|terms|").
 *
 * What the paper defines and where (PAPER.md = P):
 *  - depthwise convolution: "a depthwise convolution filter (kernel) is applied
 *    to one input channel with its own set of weights" (Sec. II);
 *    "a K x K block from the input feature map X is convolved with the weights
 *    w(i) of the same channel to compute one pixel".
 *  - the diagonalwise refactorization W (Eq. 1), mask A (Eq. 2,
 *    P:272-280), Z = (W (.) A) (x) X (Eq. 3) and the masked weight
 *    gradient dL/dW = dL/dW^ (.) A (Eq. 4).  The dense functions
 *    below exist only so tests can check Eqs. 1-4 against the depthwise ones.
 *
 * Readings where the paper is silent (DESIGN.md §3 lists them all):
 *  R1 cross-correlation (no kernel flip), as im2col + GEMM;
 *  R2 symmetric zero padding p, Ho = floor((H + 2p - K)/s) + 1;
 *  R5 dw is the SUM over the batch and is overwritten;
 *  R6 channel multiplier m: output channel o = c*m + j (j < m);
 *  R7 weights [C*m][kh][kw] for both activation layouts;
 *  R8 activations NCHW (layout 0) or NHWC (layout 1).
 */
#include <math.h>
#include <stddef.h>
#include <stdint.h>
#include <string.h>

#define ORACLE_NCHW 0
#define ORACLE_NHWC 1

/* Threads for the outer loops (1 = the plain sequential oracle). */
static int oracle_nthreads = 1;
void oracle_set_threads(int t) { oracle_nthreads = t < 1 ? 1 : t; }
int oracle_get_threads(void) { return oracle_nthreads; }

/* Flat offset of logical element (n, c, h, w) of a tensor with C channels and
 * H x W spatial size in the given layout. */
static size_t at(int layout, int64_t C, int64_t H, int64_t W,
                 int64_t n, int64_t c, int64_t h, int64_t w) {
  if (layout == ORACLE_NCHW) return (size_t)(((n * C + c) * H + h) * W + w);
  return (size_t)(((n * H + h) * W + w) * C + c);
}

/* Output spatial size (reading R2); returns 0 when the kernel exceeds the
 * padded input ("kernel exceeds padded input"). */
int oracle_out_size(int64_t in, int k, int s, int p, int64_t* out) {
  int64_t num = in + 2 * (int64_t)p - k;
  if (k < 1 || s < 1 || p < 0 || num < 0) { *out = 0; return 0; }
  *out = num / s + 1;
  return 1;
}

/* a1: forward.  y[n, c*m+j, oh, ow] = sum_{i<kh, jj<kw}
 *       w[c*m+j, i, jj] * x[n, c, oh*sh - ph + i, ow*sw - pw + jj],
 * x taken as 0 outside [0,H) x [0,W) (out-of-range taps are skipped). */
void oracle_dw_fwd(const double* x, const double* wt, double* y, double* abs_y,
                   int64_t N, int64_t C, int64_t H, int64_t W, int m,
                   int kh, int kw, int sh, int sw, int ph, int pw, int layout) {
  int64_t Ho, Wo;
  if (!oracle_out_size(H, kh, sh, ph, &Ho) || !oracle_out_size(W, kw, sw, pw, &Wo)) return;
  int64_t Co = C * m;
#pragma omp parallel for collapse(2) schedule(dynamic, 1) num_threads(oracle_nthreads) if (oracle_nthreads > 1)
  for (int64_t n = 0; n < N; ++n)
    for (int64_t c = 0; c < C; ++c)
      for (int j = 0; j < m; ++j) {
        int64_t o = c * m + j;
        for (int64_t oh = 0; oh < Ho; ++oh)
          for (int64_t ow = 0; ow < Wo; ++ow) {
            double acc = 0.0, sabs = 0.0;
            for (int i = 0; i < kh; ++i)
              for (int jj = 0; jj < kw; ++jj) {
                int64_t ih = oh * sh - ph + i, iw = ow * sw - pw + jj;
                if (ih < 0 || ih >= H || iw < 0 || iw >= W) continue;
                double t = x[at(layout, C, H, W, n, c, ih, iw)] *
                           wt[((size_t)o * kh + i) * kw + jj];
                acc += t;
                sabs += fabs(t);
              }
            size_t e = at(layout, Co, Ho, Wo, n, o, oh, ow);
            y[e] = acc;
            if (abs_y) abs_y[e] = sabs;
          }
      }
}

/* a2: input gradient, the adjoint of a1 (reading R9: the paper delegates it to
 * the framework).  dx[n, c, ih, iw] = sum_{j<m} sum_{i, jj}
 *   w[c*m+j, i, jj] * dy[n, c*m+j, (ih+ph-i)/sh, (iw+pw-jj)/sw]
 * over taps whose source is an integer output position inside [0,Ho) x [0,Wo). */
void oracle_dw_bwd_data(const double* dy, const double* wt, double* dx, double* abs_dx,
                        int64_t N, int64_t C, int64_t H, int64_t W, int m,
                        int kh, int kw, int sh, int sw, int ph, int pw, int layout) {
  int64_t Ho, Wo;
  if (!oracle_out_size(H, kh, sh, ph, &Ho) || !oracle_out_size(W, kw, sw, pw, &Wo)) return;
  int64_t Co = C * m;
#pragma omp parallel for collapse(2) schedule(dynamic, 1) num_threads(oracle_nthreads) if (oracle_nthreads > 1)
  for (int64_t n = 0; n < N; ++n)
    for (int64_t c = 0; c < C; ++c)
      for (int64_t ih = 0; ih < H; ++ih)
        for (int64_t iw = 0; iw < W; ++iw) {
          double acc = 0.0, sabs = 0.0;
          for (int j = 0; j < m; ++j) {
            int64_t o = c * m + j;
            for (int i = 0; i < kh; ++i)
              for (int jj = 0; jj < kw; ++jj) {
                int64_t th = ih + ph - i, tw = iw + pw - jj;
                if (th < 0 || tw < 0 || th % sh != 0 || tw % sw != 0) continue;
                int64_t oh = th / sh, ow = tw / sw;
                if (oh >= Ho || ow >= Wo) continue;
                double t = dy[at(layout, Co, Ho, Wo, n, o, oh, ow)] *
                           wt[((size_t)o * kh + i) * kw + jj];
                acc += t;
                sabs += fabs(t);
              }
          }
          size_t e = at(layout, C, H, W, n, c, ih, iw);
          dx[e] = acc;
          if (abs_dx) abs_dx[e] = sabs;
        }
}

/* a3: filter gradient = the diagonal kept by Eq. 4, summed over the
 * batch (reading R5).  dw[c*m+j, i, jj] = sum_n sum_{oh, ow}
 *   x[n, c, oh*sh-ph+i, ow*sw-pw+jj] * dy[n, c*m+j, oh, ow]  (in-bounds taps). */
void oracle_dw_bwd_filter(const double* x, const double* dy, double* dw, double* abs_dw,
                          int64_t N, int64_t C, int64_t H, int64_t W, int m,
                          int kh, int kw, int sh, int sw, int ph, int pw, int layout) {
  int64_t Ho, Wo;
  if (!oracle_out_size(H, kh, sh, ph, &Ho) || !oracle_out_size(W, kw, sw, pw, &Wo)) return;
  int64_t Co = C * m;
#pragma omp parallel for collapse(2) schedule(dynamic, 1) num_threads(oracle_nthreads) if (oracle_nthreads > 1)
  for (int64_t c = 0; c < C; ++c)
    for (int j = 0; j < m; ++j) {
      int64_t o = c * m + j;
      for (int i = 0; i < kh; ++i)
        for (int jj = 0; jj < kw; ++jj) {
          double acc = 0.0, sabs = 0.0;
          for (int64_t n = 0; n < N; ++n)
            for (int64_t oh = 0; oh < Ho; ++oh)
              for (int64_t ow = 0; ow < Wo; ++ow) {
                int64_t ih = oh * sh - ph + i, iw = ow * sw - pw + jj;
                if (ih < 0 || ih >= H || iw < 0 || iw >= W) continue;
                double t = x[at(layout, C, H, W, n, c, ih, iw)] *
                           dy[at(layout, Co, Ho, Wo, n, o, oh, ow)];
                acc += t;
                sabs += fabs(t);
              }
          size_t e = ((size_t)o * kh + i) * kw + jj;
          dw[e] = acc;
          if (abs_dw) abs_dw[e] = sabs;
        }
    }
}

/* ---------------------------------------------------------------------------
 * Dense (standard) convolution, NCHW, used ONLY to check Eqs. 1-4.
 * Standard convolution = im2col + GEMM Z = W C (Fig. 2); written
 * here as the equivalent five loops (SPEC.md oracle_conv).
 * wd is [Co][Ci][kh][kw].
 * ------------------------------------------------------------------------- */
void oracle_dense_fwd(const double* x, const double* wd, double* y,
                      int64_t N, int64_t Ci, int64_t H, int64_t W, int64_t Co,
                      int kh, int kw, int sh, int sw, int ph, int pw) {
  int64_t Ho, Wo;
  if (!oracle_out_size(H, kh, sh, ph, &Ho) || !oracle_out_size(W, kw, sw, pw, &Wo)) return;
  for (int64_t n = 0; n < N; ++n)
    for (int64_t o = 0; o < Co; ++o)
      for (int64_t oh = 0; oh < Ho; ++oh)
        for (int64_t ow = 0; ow < Wo; ++ow) {
          double acc = 0.0;
          for (int64_t ci = 0; ci < Ci; ++ci)
            for (int i = 0; i < kh; ++i)
              for (int jj = 0; jj < kw; ++jj) {
                int64_t ih = oh * sh - ph + i, iw = ow * sw - pw + jj;
                if (ih < 0 || ih >= H || iw < 0 || iw >= W) continue;
                acc += x[((n * Ci + ci) * H + ih) * W + iw] *
                       wd[((o * Ci + ci) * kh + i) * kw + jj];
              }
          y[((n * Co + o) * Ho + oh) * Wo + ow] = acc;
        }
}

/* Dense input gradient: dx[n,ci,ih,iw] = sum_o sum_{i,jj} wd[o,ci,i,jj] dy[n,o,oh,ow]. */
void oracle_dense_bwd_data(const double* dy, const double* wd, double* dx,
                           int64_t N, int64_t Ci, int64_t H, int64_t W, int64_t Co,
                           int kh, int kw, int sh, int sw, int ph, int pw) {
  int64_t Ho, Wo;
  if (!oracle_out_size(H, kh, sh, ph, &Ho) || !oracle_out_size(W, kw, sw, pw, &Wo)) return;
  for (int64_t n = 0; n < N; ++n)
    for (int64_t ci = 0; ci < Ci; ++ci)
      for (int64_t ih = 0; ih < H; ++ih)
        for (int64_t iw = 0; iw < W; ++iw) {
          double acc = 0.0;
          for (int64_t o = 0; o < Co; ++o)
            for (int i = 0; i < kh; ++i)
              for (int jj = 0; jj < kw; ++jj) {
                int64_t th = ih + ph - i, tw = iw + pw - jj;
                if (th < 0 || tw < 0 || th % sh != 0 || tw % sw != 0) continue;
                int64_t oh = th / sh, ow = tw / sw;
                if (oh >= Ho || ow >= Wo) continue;
                acc += dy[((n * Co + o) * Ho + oh) * Wo + ow] *
                       wd[((o * Ci + ci) * kh + i) * kw + jj];
              }
          dx[((n * Ci + ci) * H + ih) * W + iw] = acc;
        }
}

/* Dense weight gradient G = dL/dW^ (every entry, before Eq. 4's mask):
 * G[o,ci,i,jj] = sum_n sum_{oh,ow} x[n,ci,oh*sh-ph+i,ow*sw-pw+jj] dy[n,o,oh,ow]. */
void oracle_dense_bwd_filter(const double* x, const double* dy, double* g,
                             int64_t N, int64_t Ci, int64_t H, int64_t W, int64_t Co,
                             int kh, int kw, int sh, int sw, int ph, int pw) {
  int64_t Ho, Wo;
  if (!oracle_out_size(H, kh, sh, ph, &Ho) || !oracle_out_size(W, kw, sw, pw, &Wo)) return;
  for (int64_t o = 0; o < Co; ++o)
    for (int64_t ci = 0; ci < Ci; ++ci)
      for (int i = 0; i < kh; ++i)
        for (int jj = 0; jj < kw; ++jj) {
          double acc = 0.0;
          for (int64_t n = 0; n < N; ++n)
            for (int64_t oh = 0; oh < Ho; ++oh)
              for (int64_t ow = 0; ow < Wo; ++ow) {
                int64_t ih = oh * sh - ph + i, iw = ow * sw - pw + jj;
                if (ih < 0 || ih >= H || iw < 0 || iw >= W) continue;
                acc += x[((n * Ci + ci) * H + ih) * W + iw] *
                       dy[((n * Co + o) * Ho + oh) * Wo + ow];
              }
          g[((o * Ci + ci) * kh + i) * kw + jj] = acc;
        }
}

/* Eq. 1, generalised to a channel multiplier m: the C*m depthwise
 * filters placed on the block diagonal of a dense [C*m][C][kh][kw] weight,
 * wd[o, c', :, :] = w[o, :, :] if c' == o / m, else 0. */
void oracle_expand_weights(const double* wt, double* wd, int64_t C, int m, int kh, int kw) {
  int64_t Co = C * m;
  for (int64_t o = 0; o < Co; ++o)
    for (int64_t ci = 0; ci < C; ++ci)
      for (int i = 0; i < kh; ++i)
        for (int jj = 0; jj < kw; ++jj)
          wd[((o * C + ci) * kh + i) * kw + jj] =
              (ci == o / m) ? wt[((size_t)o * kh + i) * kw + jj] : 0.0;
}

/* Eq. 2: mask A, a 1_{1 x K*K} block on the (generalised) diagonal. */
void oracle_mask(double* a, int64_t C, int m, int kh, int kw) {
  int64_t Co = C * m;
  for (int64_t o = 0; o < Co; ++o)
    for (int64_t ci = 0; ci < C; ++ci)
      for (int i = 0; i < kh * kw; ++i)
        a[(o * C + ci) * kh * kw + i] = (ci == o / m) ? 1.0 : 0.0;
}

/* Elementwise product (the (.) of Eqs. 3-4). */
void oracle_hadamard(const double* a, const double* b, double* out, int64_t count) {
  for (int64_t i = 0; i < count; ++i) out[i] = a[i] * b[i];
}

/* Storage rounding of a double result (reading R10): one round-to-nearest-even
 * step to the storage precision.  dtype 0 = fp32 (C's double->float conversion
 * rounds to nearest even), dtype 1 = bf16 (8 significant bits, fp32 exponent
 * range, subnormals at the fp32 subnormal grid 2^-133, overflow to inf). */
void oracle_round(const double* in, double* out, int64_t count, int dtype) {
  for (int64_t i = 0; i < count; ++i) {
    double v = in[i];
    if (dtype == 0) {
      out[i] = (double)(float)v;
    } else {
      if (v == 0.0 || !isfinite(v)) { out[i] = v; continue; }
      int e = ilogb(v);            /* v = f * 2^e, 1 <= |f| < 2 */
      if (e < -126) e = -126;      /* subnormal grid of bf16 */
      double q = ldexp(nearbyint(ldexp(v, 7 - e)), e - 7);
      /* largest finite bf16 = (2 - 2^-7) * 2^127 */
      if (fabs(q) > ldexp(255.0, 127 - 7)) q = copysign(INFINITY, v);
      out[i] = q;
    }
  }
}
