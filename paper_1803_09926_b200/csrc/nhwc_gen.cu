// nhwc_gen.cu -- NHWC depthwise passes for the shapes the 3x3 / m = 1 NHWC families
// do not cover: K x K kernels (K = 3, 5, 7), symmetric padding (K-1)/2, stride 1 or
// 2, channel multiplier M in {1, 2, 4}, C % 4 == 0 (SURVEY §8(d) d.2 configs[3]:
// m = 2/4, 5x5 and 7x7, stride 2 on 56x56x512).
//
//   fwd  (Eq. 3):
//     y[n, oh, ow, c*M+j] = sum_{i,jj} w[c*M+j, i, jj] * x[n, oh*S-P+i, ow*S-P+jj, c]
//   bwd_data (the adjoint, R9):
//     dx[n, ih, iw, c] = sum_j sum_{i,jj} w[c*M+j, i, jj] * dy[n, (ih+P-i)/S, (iw+P-jj)/S, c*M+j]
//   bwd_filter (Eq. 4 diagonal, batch sum, R5):
//     dw[c*M+j, i, jj] = sum_{n,oh,ow} x[n, oh*S-P+i, ow*S-P+jj, c] * dy[n, oh, ow, c*M+j]
//
// A thread owns a vector of 4 consecutive input channels (16-B fp32 / 8-B bf16
// loads; consecutive lanes take consecutive vectors, so a warp reads a contiguous
// run of a pixel's channels) and their 4*M output channels (contiguous in NHWC).
//
//  * fwd / bwd_data: a CTA = a block of CVB channel vectors x tile slots; its
//    weights are converted once to fp32 and transposed to [tap][channel*M] in
//    shared memory (K*K*4*M values per vector -- too many for registers at K = 7).
//    A thread computes a TH x TW output tile: it walks the (TH-1)*S+K input rows of
//    its window one row at a time ((TW-1)*S+K vectors in registers, zero outside
//    the plane) and applies every tap of that row to every output of the tile that
//    uses it (compile-time tap indices; bwd_data is the polyphase form with tiles
//    aligned to the stride, tap i = ta + P - S*(D0 + r)).  Packed FFMA2 over
//    channel (M = 1) or multiplier (M > 1) pairs.
//  * bwd_filter: a CTA = (block of CVB channel vectors, slice of the N*Ho output
//    rows); thread = (channel vector, tap row i, pixel set).  Along an output row it
//    takes U output pixels per step: their M dy vectors and the U*S new x vectors of
//    tap row i's sliding window are loaded together, then 4*M*K*U FMAs (FFMA2);
//    per-row sums (<= 64 terms) -> running
//    sum over the thread's rows -> pixel sets in order -> per-slice partial ->
//    the last CTA of each group of 32 slices and then of the channel block sums the
//    partials pairwise in slice order (integer tickets; nchw::finalize_two_level):
//    no float atomics, bitwise reproducible, max_chain reported.
#include <cuda.h>

#include <algorithm>

#include "kernels.h"
#include "nchw_common.cuh"

namespace dwk {
namespace nhwcg {

using nchw::VecIO;
constexpr int VC = 4;
constexpr int kFdThreads = 256;

struct FArgs {
  const void* in;
  const void* w;
  void* out;
  int N, C, H, W, Ho, Wo;     // x dims (C input channels) and y dims
  int CVB, ncb, slots;        // channel vectors per CTA block, blocks, tile slots per CTA
  int OHB, OWB;               // tiles along the output rows / columns
  int64_t tiles;              // N * OHB * OWB
  int ctas_per_cb;
};

struct BArgs {
  const void* x;
  const void* dy;
  float* dw;
  float* part;                // [nslices][Co*K*K]
  float* l2;                  // [ngrp][Co*K*K]
  unsigned* t1;               // [ncb][ngrp]
  unsigned* t2;               // [ncb]
  int N, C, H, W, Ho, Wo;
  int CVB, ncb, PS;           // channel vectors per block, blocks, pixel sets
  int nslices, rps;           // slices of the N*Ho output rows, rows per slice
};

template <class T, int K, int S, int M, int TH, int TW, bool BWD>
__global__ void __launch_bounds__(kFdThreads, 2) gen_fd_kernel(const FArgs a) {
  constexpr int P = (K - 1) / 2, KK = K * K, QM = VC * M;  // QM: output channels per fwd thread
  constexpr int D0 = BWD ? floor_div(P - K + 1, S) : 0;
  constexpr int NWR = BWD ? floor_div(TH - 1 + P, S) - D0 + 1 : (TH - 1) * S + K;
  constexpr int NWC = BWD ? floor_div(TW - 1 + P, S) - D0 + 1 : (TW - 1) * S + K;
  static_assert(!BWD || (TH % S == 0 && TW % S == 0), "bwd_data tiles are stride aligned");
  extern __shared__ float ws[];  // [KK][CVB * QM]
  const T* __restrict__ in = static_cast<const T*>(a.in);
  const T* __restrict__ wt = static_cast<const T*>(a.w);
  T* __restrict__ out = static_cast<T*>(a.out);
  const int C = a.C;
  const int cb = blockIdx.x % a.ncb;
  const int cv = threadIdx.x % a.CVB, slot = threadIdx.x / a.CVB;
  const int c0 = (cb * a.CVB + cv) * VC;
  const int nq = a.CVB * QM;
  griddep_wait();
  for (int e = threadIdx.x; e < KK * nq; e += blockDim.x) {
    const int tap = e / nq, q = e - tap * nq;
    const int o = cb * a.CVB * QM + q;  // output channel c*M + j
    ws[e] = (o < C * M) ? Elem<T>::ldg(wt + (int64_t)o * KK + tap) : 0.f;
  }
  __syncthreads();
  if (slot >= a.slots || c0 >= C) return;
  const float* wsv = ws + cv * QM;
  const int IH = BWD ? a.Ho : a.H, IW = BWD ? a.Wo : a.W;  // window plane
  const int OH = BWD ? a.H : a.Ho, OW = BWD ? a.W : a.Wo;  // output plane
  const int CI = BWD ? C * M : C, CO = BWD ? C : C * M;    // channels of the input / output tensors
  const int ci0 = BWD ? c0 * M : c0, co0 = BWD ? c0 : c0 * M;
  constexpr int NIN = BWD ? QM : VC;    // input values per window position
  constexpr int NACC = BWD ? VC : QM;   // outputs per pixel
  const int64_t step = (int64_t)(gridDim.x / a.ncb) * a.slots;
  for (int64_t t = (int64_t)(blockIdx.x / a.ncb) * a.slots + slot; t < a.tiles; t += step) {
    const int64_t r2 = t / a.OWB;
    const int owb = (int)(t - r2 * a.OWB);
    const int64_t n = r2 / a.OHB;
    const int ohb = (int)(r2 - n * a.OHB);
    const int oh0 = ohb * TH, ow0 = owb * TW;
    const int wr0 = BWD ? oh0 / S + D0 : oh0 * S - P;
    const int wc0 = BWD ? ow0 / S + D0 : ow0 * S - P;
    float2 acc[TH][TW][NACC / 2];
#pragma unroll
    for (int i = 0; i < TH; ++i)
#pragma unroll
      for (int j = 0; j < TW; ++j)
#pragma unroll
        for (int v = 0; v < NACC / 2; ++v) acc[i][j][v] = make_float2(0.f, 0.f);
    const T* base = in + (n * IH) * (int64_t)IW * CI + ci0;
#pragma unroll 1
    for (int r = 0; r < NWR; ++r) {
      const int ir = wr0 + r;
      const bool rv = (unsigned)ir < (unsigned)IH;
      float xv[NWC][NIN];
#pragma unroll
      for (int cc = 0; cc < NWC; ++cc) {
        const int ic = wc0 + cc;
        if (rv && (unsigned)ic < (unsigned)IW) {
          VecIO<T, NIN>::load(base + ((int64_t)ir * IW + ic) * CI, xv[cc]);
        } else {
#pragma unroll
          for (int v = 0; v < NIN; ++v) xv[cc][v] = 0.f;
        }
      }
      if constexpr (!BWD) {
#pragma unroll
        for (int ta = 0; ta < TH; ++ta) {
          const int i = r - ta * S;  // runtime r: taps checked at run time (loop kept rolled over rows)
          if (i < 0 || i >= K) continue;
#pragma unroll
          for (int jj = 0; jj < K; ++jj) {
            float wv[QM];
            const float* wp = wsv + (i * K + jj) * nq;
#pragma unroll
            for (int q = 0; q < QM; q += 4) {
              const float4 f = *reinterpret_cast<const float4*>(wp + q);
              wv[q] = f.x; wv[q + 1] = f.y; wv[q + 2] = f.z; wv[q + 3] = f.w;
            }
#pragma unroll
            for (int tb = 0; tb < TW; ++tb) {
              const int cc = tb * S + jj;
#pragma unroll
              for (int k2 = 0; k2 < QM / 2; ++k2) {
                const int q = 2 * k2, v = q / M;
                const float2 xp = (M == 1) ? make_float2(xv[cc][q], xv[cc][q + 1]) : make_float2(xv[cc][v], xv[cc][v]);
                acc[ta][tb][k2] = __ffma2_rn(xp, make_float2(wv[q], wv[q + 1]), acc[ta][tb][k2]);
              }
            }
          }
        }
      } else {
        // dx[ta][tb][v] += sum_j w[(c0+v)*M + j, i, jj] * dy[(c0+v)*M + j], i = ta + P - S*(D0 + r)
#pragma unroll
        for (int ta = 0; ta < TH; ++ta) {
          const int i = ta + P - S * (D0 + r);
          if (i < 0 || i >= K) continue;
#pragma unroll
          for (int tb = 0; tb < TW; ++tb) {
#pragma unroll
            for (int cc = 0; cc < NWC; ++cc) {
              const int jj = tb + P - S * (D0 + cc);
              if (jj < 0 || jj >= K) continue;
              const float* wp = wsv + (i * K + jj) * nq;
              float wv[QM];
#pragma unroll
              for (int q = 0; q < QM; q += 4) {
                const float4 f = *reinterpret_cast<const float4*>(wp + q);
                wv[q] = f.x; wv[q + 1] = f.y; wv[q + 2] = f.z; wv[q + 3] = f.w;
              }
#pragma unroll
              for (int j = 0; j < M; ++j) {
                acc[ta][tb][0] = __ffma2_rn(make_float2(xv[cc][0 * M + j], xv[cc][1 * M + j]),
                                            make_float2(wv[0 * M + j], wv[1 * M + j]), acc[ta][tb][0]);
                acc[ta][tb][1] = __ffma2_rn(make_float2(xv[cc][2 * M + j], xv[cc][3 * M + j]),
                                            make_float2(wv[2 * M + j], wv[3 * M + j]), acc[ta][tb][1]);
              }
            }
          }
        }
      }
    }
    T* obase = out + (n * OH) * (int64_t)OW * CO + co0;
#pragma unroll
    for (int ta = 0; ta < TH; ++ta) {
      const int oh = oh0 + ta;
      if (oh >= OH) continue;
#pragma unroll
      for (int tb = 0; tb < TW; ++tb) {
        const int ow = ow0 + tb;
        if (ow >= OW) continue;
        float o[NACC];
#pragma unroll
        for (int k2 = 0; k2 < NACC / 2; ++k2) { o[2 * k2] = acc[ta][tb][k2].x; o[2 * k2 + 1] = acc[ta][tb][k2].y; }
        VecIO<T, NACC>::store(obase + ((int64_t)oh * OW + ow) * CO, o);
      }
    }
  }
  griddep_launch_dependents();
}

// bwd_filter: thread = (channel vector cv, tap row i, pixel set ps)
template <class T, int K, int S, int M>
__global__ void __launch_bounds__(256, (M >= 4 ? 1 : 2)) gen_bf_kernel(const BArgs a) {
  constexpr int P = (K - 1) / 2, QM = VC * M, SEG = 64;
  constexpr int U = (M >= 4 && K >= 7) ? 1 : 2, NXW = (U - 1) * S + K;  // pixels per step, x vectors per step
  extern __shared__ float red[];  // [PS][CVB*K][QM*K] per-thread partials, reduced over ps in order
  __shared__ unsigned s_flag;
  const T* __restrict__ x = static_cast<const T*>(a.x);
  const T* __restrict__ dy = static_cast<const T*>(a.dy);
  const int C = a.C, Co = C * M;
  const int cb = blockIdx.x % a.ncb, sl = blockIdx.x / a.ncb;
  const int cv = threadIdx.x % a.CVB;
  const int rest = threadIdx.x / a.CVB;
  const int i = rest % K, ps = rest / K;
  const int c0 = (cb * a.CVB + cv) * VC;
  const bool live = c0 < C && ps < a.PS;
  const int H = a.H, W = a.W, Ho = a.Ho, Wo = a.Wo;
  griddep_wait();
  float2 run[K][QM / 2];  // pairs: channel pairs (M = 1) or multiplier pairs (M > 1), packed FFMA2
#pragma unroll
  for (int jj = 0; jj < K; ++jj)
#pragma unroll
    for (int k2 = 0; k2 < QM / 2; ++k2) run[jj][k2] = make_float2(0.f, 0.f);
  if (live) {
    const int64_t r0 = (int64_t)sl * a.rps;
    const int64_t r1 = std::min<int64_t>((int64_t)a.N * Ho, r0 + a.rps);
    for (int64_t r = r0 + ps; r < r1; r += a.PS) {
      const int64_t n = r / Ho;
      const int oh = (int)(r - n * Ho);
      const int ih = oh * S - P + i;
      if ((unsigned)ih >= (unsigned)H) continue;
      const T* xr = x + ((n * H + ih) * (int64_t)W) * C + c0;
      const T* dr = dy + ((n * Ho + oh) * (int64_t)Wo) * Co + (int64_t)c0 * M;
      for (int s0 = 0; s0 < Wo; s0 += SEG) {
        const int s1 = min(Wo, s0 + SEG);
        float2 loc[K][QM / 2];
#pragma unroll
        for (int jj = 0; jj < K; ++jj)
#pragma unroll
          for (int k2 = 0; k2 < QM / 2; ++k2) loc[jj][k2] = make_float2(0.f, 0.f);
        // x window of tap row i: columns ow0*S - P + cc, cc < NXW; the K - S columns the next
        // U pixels share with these are carried, U*S new ones loaded per step
        float xw[NXW][VC];
        auto ldx = [&](int ic, float* v) {
          if ((unsigned)ic < (unsigned)W) VecIO<T, VC>::load(xr + (int64_t)ic * C, v);
          else
#pragma unroll
            for (int q = 0; q < VC; ++q) v[q] = 0.f;
        };
#pragma unroll
        for (int cc = 0; cc < K - S; ++cc) ldx(s0 * S - P + cc, xw[cc]);
        // software pipeline: the next step's U dy vectors and U*S new x vectors are loaded
        // while this step's FMAs run (ncu: without it the compiler sinks each load next to
        // its first use and the loop waits one L2 round trip per load)
        float dn[U][QM], xn[U * S][VC];
        // running pointers (no per-load 64-bit index math): next dy pixel, next new x column
        const T* dnext = dr + (int64_t)s0 * Co;
        const T* xnext = xr + (int64_t)(s0 * S - P + K - S) * C;
        int cnext = s0 * S - P + K - S, onext = s0;
        auto load_step = [&](int) {
#pragma unroll
          for (int u = 0; u < U; ++u) {
            if (onext + u < s1) VecIO<T, QM>::load(dnext + u * Co, dn[u]);
            else
#pragma unroll
              for (int q = 0; q < QM; ++q) dn[u][q] = 0.f;
          }
#pragma unroll
          for (int cc = 0; cc < U * S; ++cc) {
            if ((unsigned)(cnext + cc) < (unsigned)W) VecIO<T, VC>::load(xnext + cc * C, xn[cc]);
            else
#pragma unroll
              for (int q = 0; q < VC; ++q) xn[cc][q] = 0.f;
          }
          dnext += U * Co;
          xnext += U * S * C;
          cnext += U * S;
          onext += U;
        };
        load_step(s0);
#pragma unroll 2
        for (int ow0 = s0; ow0 < s1; ow0 += U) {
          float d[U][QM];
#pragma unroll
          for (int u = 0; u < U; ++u)
#pragma unroll
            for (int q = 0; q < QM; ++q) d[u][q] = dn[u][q];
#pragma unroll
          for (int cc = 0; cc < U * S; ++cc)
#pragma unroll
            for (int q = 0; q < VC; ++q) xw[K - S + cc][q] = xn[cc][q];
          if (ow0 + U < s1) load_step(ow0 + U);
#pragma unroll
          for (int u = 0; u < U; ++u)
#pragma unroll
            for (int jj = 0; jj < K; ++jj)
#pragma unroll
              for (int k2 = 0; k2 < QM / 2; ++k2) {
                const int q = 2 * k2, v = q / M;
                const float* xc = xw[u * S + jj];
                const float2 xp = (M == 1) ? make_float2(xc[q], xc[q + 1]) : make_float2(xc[v], xc[v]);
                loc[jj][k2] = __ffma2_rn(xp, make_float2(d[u][q], d[u][q + 1]), loc[jj][k2]);
              }
#pragma unroll
          for (int cc = 0; cc < K - S; ++cc)
#pragma unroll
            for (int q = 0; q < VC; ++q) xw[cc][q] = xw[cc + U * S][q];
        }
#pragma unroll
        for (int jj = 0; jj < K; ++jj)
#pragma unroll
          for (int k2 = 0; k2 < QM / 2; ++k2) {
            run[jj][k2].x += loc[jj][k2].x;
            run[jj][k2].y += loc[jj][k2].y;
          }
      }
    }
  }
  // pixel sets in order -> this CTA's slice partial of (cv, i): dw[(c0*M + q), i, jj]
  const int nthr = a.CVB * K;
  const int tslot = cv * K + i;
  if (ps < a.PS) {
    float* mine = red + ((size_t)ps * nthr + tslot) * (QM * K);
#pragma unroll
    for (int jj = 0; jj < K; ++jj)
#pragma unroll
      for (int k2 = 0; k2 < QM / 2; ++k2) {
        mine[(2 * k2) * K + jj] = run[jj][k2].x;
        mine[(2 * k2 + 1) * K + jj] = run[jj][k2].y;
      }
  }
  __syncthreads();
  const int64_t sstride = (int64_t)Co * K * K;
  if (ps == 0 && c0 < C) {
    float* dst = a.part + (int64_t)sl * sstride;
    for (int e = 0; e < QM * K; ++e) {
      float v = red[(size_t)tslot * (QM * K) + e];
      for (int p2 = 1; p2 < a.PS; ++p2) v += red[((size_t)p2 * nthr + tslot) * (QM * K) + e];
      const int q = e / K, jj = e - q * K;
      const int o = c0 * M + q;
      __stcg(dst + ((int64_t)o * K + i) * K + jj, v);
    }
  }
  __threadfence();
  __syncthreads();
  const int64_t e0 = (int64_t)cb * a.CVB * VC * M * K * K;
  const int nvals = (int)std::min<int64_t>((int64_t)a.CVB * VC * M * K * K, sstride - e0);
  nchw::finalize_two_level(a.part, a.l2, a.t1, a.t2, cb, sl, a.nslices, sstride, e0, nvals, a.dw, &s_flag);
  griddep_launch_dependents();
}

// ---------------------------------------------------------------------------
// bwd_filter, TMA-staged (the default where the tensors are 16-B aligned): CTA =
// (block of CB channels = 64 B per pixel, slice of TR-row output bands).  A producer
// lane stages each band's x rows [oh0*S-P, oh0*S-P+(TR-1)*S+K) x all columns (4-D
// tensor-map box, zero-filled halo and tail) and its dy rows into a 2-stage ring;
// consumer thread = (channel pair cp, column set cs, tap row i) walks its columns of
// every band row with a K-wide sliding x window in registers read from shared memory
// (S new pairs + M dy values per output pixel, K*M packed FFMA2).  Row sums (<= 64
// terms) -> running sum over the slice's rows -> column sets in order -> slice
// partial -> the two-level ticketed finalize (deterministic, no float atomics).
struct TArgs {
  float* dw;
  float* part;
  float* l2;
  unsigned* t1;
  unsigned* t2;
  int C, Ho, Wo;
  int CB, NCP, NCS, CW, TR, XR, BWX;
  int ncb, bpi, units, nslices, ups;     // bands per image, band units, slices, units per slice
  uint32_t x_bytes, dy_bytes, dy_off, stage_bytes;  // dy_off: x region rounded up to 128 B (TMA destination)
};

__device__ __forceinline__ void tma4(void* dst, const CUtensorMap* tm, int c0, int c1, int c2, int c3,
                                     uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];"
      ::"r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(tm)), "r"(c0), "r"(c1), "r"(c2), "r"(c3),
      "r"(smem_u32(bar))
      : "memory");
}

template <class T>
__device__ __forceinline__ float2 ld_pair(const T* p) {
  if constexpr (sizeof(T) == 4) {
    return *reinterpret_cast<const float2*>(p);
  } else {
    const uint32_t w = *reinterpret_cast<const uint32_t*>(p);
    return make_float2(nchw::bf_lo(w), nchw::bf_hi(w));
  }
}

template <class T, int K, int S, int M>
__global__ void __launch_bounds__(288) gen_bft_kernel(const __grid_constant__ CUtensorMap tmx,
                                                      const __grid_constant__ CUtensorMap tmd, const TArgs a) {
  constexpr int P = (K - 1) / 2, NS = 2;
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ unsigned s_flag;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  uint64_t* empty = full + NS;
  unsigned char* ring = smem + 128;
  const int tid = threadIdx.x;
  const int ncw = (blockDim.x - 32) >> 5;  // consumer warps
  const int cb = blockIdx.x % a.ncb, sl = blockIdx.x / a.ncb;
  const int u0 = sl * a.ups, u1 = min(a.units, u0 + a.ups);
  if (tid == 0) {
    for (int i = 0; i < NS; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], ncw);
    }
    fence_mbar_init();
  }
  __syncthreads();
  griddep_wait();
  const int ctid = tid - 32;
  const int cp = ctid % a.NCP, rest = ctid / a.NCP;
  const int cs = rest % a.NCS, i = rest / a.NCS;
  const bool live = ctid >= 0 && i < K;
  float2 run[K][M];
#pragma unroll
  for (int jj = 0; jj < K; ++jj)
#pragma unroll
    for (int j = 0; j < M; ++j) run[jj][j] = make_float2(0.f, 0.f);
  if (tid < 32) {
    if (tid == 0) {  // producer
      int st = 0;
      uint32_t ph = 0;
      for (int u = u0, it = 0; u < u1; ++u, ++it) {
        if (it >= NS) mbar_wait(&empty[st], ph ^ 1);
        const int n = u / a.bpi, oh0 = (u - n * a.bpi) * a.TR;
        unsigned char* sx = ring + (size_t)st * a.stage_bytes;
        mbar_arrive_expect_tx(&full[st], a.x_bytes + a.dy_bytes);
        tma4(sx, &tmx, cb * a.CB, -P, oh0 * S - P, n, &full[st]);
        tma4(sx + a.dy_off, &tmd, cb * a.CB * M, 0, oh0, n, &full[st]);
        if (++st == NS) { st = 0; ph ^= 1; }
      }
    }
  } else {
    int st = 0;
    uint32_t ph = 0;
    const int c_lo = cs * a.CW, c_hi = min(a.Wo, c_lo + a.CW);
    for (int u = u0; u < u1; ++u) {
      mbar_wait(&full[st], ph);
      if (live) {
        const int n = u / a.bpi, oh0 = (u - n * a.bpi) * a.TR;
        const T* sx = reinterpret_cast<const T*>(ring + (size_t)st * a.stage_bytes);
        const T* sd = reinterpret_cast<const T*>(ring + (size_t)st * a.stage_bytes + a.dy_off);
        const int rows = min(a.TR, a.Ho - oh0);
        for (int r = 0; r < rows; ++r) {
          const T* xr = sx + ((size_t)(r * S + i) * a.BWX) * a.CB + 2 * cp;  // x row of tap row i
          const T* dr = sd + ((size_t)r * a.Wo) * (a.CB * M) + 2 * cp * M;
          float2 loc[K][M];
#pragma unroll
          for (int jj = 0; jj < K; ++jj)
#pragma unroll
            for (int j = 0; j < M; ++j) loc[jj][j] = make_float2(0.f, 0.f);
          float2 xw[K];
#pragma unroll
          for (int jj = 0; jj < K - S; ++jj) xw[jj] = ld_pair<T>(xr + (size_t)(c_lo * S + jj) * a.CB);
          // unrolled so the window's register rotation costs moves only once per 8 pixels
#pragma unroll 8
          for (int ow = c_lo; ow < c_hi; ++ow) {
#pragma unroll
            for (int u2 = 0; u2 < S; ++u2) xw[K - S + u2] = ld_pair<T>(xr + (size_t)(ow * S + K - S + u2) * a.CB);
            float dv[2 * M];  // dy[c0*M .. c0*M + 2M): channel c0 -> [0, M), c0+1 -> [M, 2M)
#pragma unroll
            for (int q = 0; q < M; ++q) {
              const float2 v = ld_pair<T>(dr + (size_t)ow * (a.CB * M) + 2 * q);
              dv[2 * q] = v.x;
              dv[2 * q + 1] = v.y;
            }
#pragma unroll
            for (int jj = 0; jj < K; ++jj)
#pragma unroll
              for (int j = 0; j < M; ++j)
                loc[jj][j] = __ffma2_rn(xw[jj], make_float2(dv[j], dv[M + j]), loc[jj][j]);
#pragma unroll
            for (int jj = 0; jj < K - S; ++jj) xw[jj] = xw[jj + S];
          }
#pragma unroll
          for (int jj = 0; jj < K; ++jj)
#pragma unroll
            for (int j = 0; j < M; ++j) {
              run[jj][j].x += loc[jj][j].x;
              run[jj][j].y += loc[jj][j].y;
            }
        }
      }
      __syncwarp();
      if ((tid & 31) == 0) mbar_arrive(&empty[st]);
      if (++st == NS) { st = 0; ph ^= 1; }
    }
  }
  griddep_launch_dependents();
  __syncthreads();  // the ring is idle: reuse it for the column-set reduction
  float* red = reinterpret_cast<float*>(ring);  // [cs][cp][i][2][M][K]
  const int per = 2 * M * K;
  if (live) {
    float* mine = red + ((size_t)(cs * a.NCP + cp) * K + i) * per;
#pragma unroll
    for (int jj = 0; jj < K; ++jj)
#pragma unroll
      for (int j = 0; j < M; ++j) {
        mine[(0 * M + j) * K + jj] = run[jj][j].x;
        mine[(1 * M + j) * K + jj] = run[jj][j].y;
      }
  }
  __syncthreads();
  const int64_t sstride = (int64_t)a.C * M * K * K;
  if (live && cs == 0) {
    float* dst = a.part + (int64_t)sl * sstride;
    for (int e = 0; e < per; ++e) {
      float v = red[((size_t)(0 * a.NCP + cp) * K + i) * per + e];
      for (int c2 = 1; c2 < a.NCS; ++c2) v += red[((size_t)(c2 * a.NCP + cp) * K + i) * per + e];
      const int h = e / (M * K), j = (e / K) % M, jj = e % K;
      const int o = (cb * a.CB + 2 * cp + h) * M + j;
      __stcg(dst + ((int64_t)o * K + i) * K + jj, v);
    }
  }
  __threadfence();
  __syncthreads();
  const int64_t e0 = (int64_t)cb * a.CB * M * K * K;
  nchw::finalize_two_level(a.part, a.l2, a.t1, a.t2, cb, sl, a.nslices, sstride, e0, a.CB * M * K * K, a.dw,
                           &s_flag);
}

using BftFn = void (*)(const CUtensorMap, const CUtensorMap, const TArgs);
template <class T, int K, int S>
BftFn bft_m(int M) {
  switch (M) {
    case 1: return gen_bft_kernel<T, K, S, 1>;
    case 2: return gen_bft_kernel<T, K, S, 2>;
    case 4: return gen_bft_kernel<T, K, S, 4>;
    default: return nullptr;
  }
}
template <class T>
BftFn bft_k(int K, int S, int M) {
  if (S != 1 && S != 2) return nullptr;
  switch (K) {
    case 3: return S == 1 ? bft_m<T, 3, 1>(M) : bft_m<T, 3, 2>(M);
    case 5: return S == 1 ? bft_m<T, 5, 1>(M) : bft_m<T, 5, 2>(M);
    case 7: return S == 1 ? bft_m<T, 7, 1>(M) : bft_m<T, 7, 2>(M);
    default: return nullptr;
  }
}
BftFn bft_kernel(int dtype, int K, int S, int M) {
  return dtype == DWCONV_F32 ? bft_k<float>(K, S, M) : bft_k<__nv_bfloat16>(K, S, M);
}

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeFn encode_fn() {
  static EncodeFn fn = []() -> EncodeFn {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return nullptr;
    return reinterpret_cast<EncodeFn>(ptr);
  }();
  return fn;
}

using FdFn = void (*)(const FArgs);
using BfFn = void (*)(const BArgs);

// tile shapes: TH x TW = 2 x 4 at stride 1, 2 x 2 at stride 2 and where the 4*M accumulators per pixel
// would spill (M = 4; M = 2 with K >= 5); bwd_data tiles aligned to S
constexpr int tile_w(int K, int S, int M) { return (M == 4 || S == 2 || (M == 2 && K >= 5)) ? 2 : 4; }
template <class T, int K, int S, int M, bool BWD>
FdFn fd_pick() {
  return gen_fd_kernel<T, K, S, M, 2, tile_w(K, S, M), BWD>;
}
template <class T, int K, int S>
FdFn fd_m(int M, bool bwd) {
  switch (M) {
    case 1: return bwd ? fd_pick<T, K, S, 1, true>() : fd_pick<T, K, S, 1, false>();
    case 2: return bwd ? fd_pick<T, K, S, 2, true>() : fd_pick<T, K, S, 2, false>();
    case 4: return bwd ? fd_pick<T, K, S, 4, true>() : fd_pick<T, K, S, 4, false>();
    default: return nullptr;
  }
}
template <class T, int K>
FdFn fd_s(int S, int M, bool bwd) {
  return S == 1 ? fd_m<T, K, 1>(M, bwd) : (S == 2 ? fd_m<T, K, 2>(M, bwd) : nullptr);
}
template <class T>
FdFn fd_k(int K, int S, int M, bool bwd) {
  switch (K) {
    case 3: return fd_s<T, 3>(S, M, bwd);
    case 5: return fd_s<T, 5>(S, M, bwd);
    case 7: return fd_s<T, 7>(S, M, bwd);
    default: return nullptr;
  }
}
FdFn fd_kernel(int dtype, int K, int S, int M, bool bwd) {
  return dtype == DWCONV_F32 ? fd_k<float>(K, S, M, bwd) : fd_k<__nv_bfloat16>(K, S, M, bwd);
}

template <class T, int K, int S>
BfFn bf_m(int M) {
  switch (M) {
    case 1: return gen_bf_kernel<T, K, S, 1>;
    case 2: return gen_bf_kernel<T, K, S, 2>;
    case 4: return gen_bf_kernel<T, K, S, 4>;
    default: return nullptr;
  }
}
template <class T>
BfFn bf_k(int K, int S, int M) {
  if (S != 1 && S != 2) return nullptr;
  switch (K) {
    case 3: return S == 1 ? bf_m<T, 3, 1>(M) : bf_m<T, 3, 2>(M);
    case 5: return S == 1 ? bf_m<T, 5, 1>(M) : bf_m<T, 5, 2>(M);
    case 7: return S == 1 ? bf_m<T, 7, 1>(M) : bf_m<T, 7, 2>(M);
    default: return nullptr;
  }
}
BfFn bf_kernel(int dtype, int K, int S, int M) {
  return dtype == DWCONV_F32 ? bf_k<float>(K, S, M) : bf_k<__nv_bfloat16>(K, S, M);
}

cudaError_t launch_ex(const void* fn, int grid, int block, int smem, cudaStream_t st, void** args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3((unsigned)block);
  cfg.dynamicSmemBytes = (size_t)smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelExC(&cfg, fn, args);
}

}  // namespace nhwcg

// the TMA-staged bwd_filter (gen_bft_kernel) where its boxes fit; false -> the direct kernel
static bool plan_staged_bf(const Geom& g, int num_sms, int smem_optin, NhwcGenPlan* p) {
  using namespace nhwcg;
  const int K = g.kh, S = g.sh, M = g.m;
  const int eb = g.dtype == DWCONV_F32 ? 4 : 2;
  const int CB = 64 / eb;
  if (g.C % CB != 0 || !bft_kernel(g.dtype, K, S, M) || !encode_fn()) return false;
  const int64_t BWX = (g.Wo - 1) * S + K;
  if (BWX > 256 || g.Wo > 256 || CB * M > 256 || g.N >= (1 << 24)) return false;
  const int NCP = CB / 2;
  int NCS = std::max(1, 256 / (NCP * K));
  NCS = std::min<int>(NCS, (int)std::max<int64_t>(1, g.Wo / 4));
  const int CW = (int)((g.Wo + NCS - 1) / NCS);
  if (CW > 64) return false;
  const int consumers = NCP * NCS * K;
  const int threads = 32 + (consumers + 31) / 32 * 32;
  if (threads > 288) return false;
  int TR = 0;
  uint32_t xb = 0, db = 0, stb = 0;
  for (int tr : {4, 2, 1}) {
    const int XR = (tr - 1) * S + K;
    xb = (uint32_t)(XR * BWX * CB * eb);
    db = (uint32_t)(tr * g.Wo * CB * M * eb);
    stb = (((xb + 127) & ~127u) + db + 127) & ~127u;
    const size_t red = (size_t)NCS * NCP * K * 2 * M * K * 4;
    if (128 + 2 * (size_t)stb <= (size_t)std::min(smem_optin, 112 * 1024) && red <= 2 * (size_t)stb) {
      TR = tr;
      break;
    }
  }
  if (TR == 0) return false;
  p->tma = true;
  p->CB = CB; p->NCP = NCP; p->NCS = NCS; p->CW = CW; p->TR = TR; p->XR = (TR - 1) * S + K; p->BWX = (int)BWX;
  p->x_bytes = xb; p->dy_bytes = db; p->stage_bytes = stb;
  p->ncb = (int)(g.C / CB);
  p->bpi = (int)((g.Ho + TR - 1) / TR);
  p->units = (int)(g.N * p->bpi);
  p->threads = threads;
  p->smem = 128 + 2 * (int)stb;
  // about two waves of CTAs; each thread adds at most 48 row sums into its running sum
  const int ups_max = std::max(1, 48 / TR);
  int64_t ns = std::max<int64_t>(1, (int64_t)num_sms * 4 / p->ncb);
  ns = std::max<int64_t>(ns, (p->units + ups_max - 1) / ups_max);
  ns = std::min<int64_t>(ns, p->units);
  p->ups = (int)((p->units + ns - 1) / ns);
  p->nslices = (p->units + p->ups - 1) / p->ups;
  p->grid = p->ncb * p->nslices;
  const int64_t sstride = g.C * g.m * K * K;
  const int ngrp = (p->nslices + 31) / 32;
  int lg2 = 0;
  while ((1 << lg2) < ngrp) ++lg2;
  p->max_chain = CW + p->ups * TR + (NCS - 1) + 5 + lg2 + 1;
  p->part_off = 0;
  p->l2_off = (size_t)p->nslices * sstride * 4;
  p->t1_off = p->l2_off + (size_t)ngrp * sstride * 4;
  p->t2_off = p->t1_off + (size_t)p->ncb * ngrp * 4;
  p->ws_bytes = (p->t2_off + (size_t)p->ncb * 4 + 15) & ~(size_t)15;
  return p->max_chain <= 160;
}

bool plan_nhwc_gen(const Geom& g, int pass, int num_sms, int smem_optin, NhwcGenPlan* p) {
  using namespace nhwcg;
  if (g.layout != DWCONV_NHWC || g.kh != g.kw || g.sh != g.sw || g.ph != g.pw || g.ph != (g.kh - 1) / 2)
    return false;
  const int K = g.kh, S = g.sh, M = g.m;
  if ((K != 3 && K != 5 && K != 7) || (S != 1 && S != 2) || (M != 1 && M != 2 && M != 4) || g.C % VC != 0)
    return false;
  if (g.N * g.H * g.W * g.C >= (1ll << 40)) return false;
  *p = NhwcGenPlan{};
  p->K = K; p->S = S; p->M = M; p->pass = pass;
  const int cvt = (int)(g.C / VC);
  p->CVB = std::min(32, cvt);
  p->ncb = (cvt + p->CVB - 1) / p->CVB;
  if (pass == DWCONV_PASS_FWD || pass == DWCONV_PASS_BWD_DATA) {
    const bool bwd = pass == DWCONV_PASS_BWD_DATA;
    if (!fd_kernel(g.dtype, K, S, M, bwd)) return false;
    const int TW = tile_w(K, S, M), TH = 2;
    const int64_t OH = bwd ? g.H : g.Ho, OW = bwd ? g.W : g.Wo;
    p->TH = TH; p->TW = TW;
    p->OHB = (int)((OH + TH - 1) / TH);
    p->OWB = (int)((OW + TW - 1) / TW);
    p->tiles = g.N * (int64_t)p->OHB * p->OWB;
    p->threads = kFdThreads;
    p->slots = kFdThreads / p->CVB;
    p->smem = K * K * p->CVB * VC * M * 4;
    if (p->smem > smem_optin) return false;
    const int64_t want = std::max<int64_t>(1, (int64_t)num_sms * 6 / p->ncb);
    const int64_t need = (p->tiles + p->slots - 1) / p->slots;
    p->ctas_per_cb = (int)std::max<int64_t>(1, std::min(want, need));
    p->grid = p->ncb * p->ctas_per_cb;
    return true;
  }
  if (pass != DWCONV_PASS_BWD_FILTER || !bf_kernel(g.dtype, K, S, M)) return false;
  if (plan_staged_bf(g, num_sms, smem_optin, p)) return true;
  const int64_t rows = g.N * g.Ho;
  p->PS = std::max(1, 256 / (p->CVB * K));
  if (p->PS > 4) p->PS = 4;
  p->threads = p->CVB * K * p->PS;
  // several waves of CTAs (the per-thread loop is load-latency bound: ncu shows 14% warps
  // active at ~2 CTAs per SM); every thread adds at most 48 row sums into its running sum
  const int segs = (int)((g.Wo + 63) / 64);
  int64_t ns = std::max<int64_t>(1, (int64_t)num_sms * 8 / p->ncb);
  const int64_t cap_rows = std::max<int64_t>(1, 48 / segs) * p->PS;  // rows per slice so each thread adds <= 48
  ns = std::max(ns, (rows + cap_rows - 1) / cap_rows);
  ns = std::min<int64_t>(ns, std::max<int64_t>(1, rows));
  p->rps = (int)((rows + ns - 1) / ns);
  p->nslices = (int)((rows + p->rps - 1) / p->rps);
  p->grid = p->ncb * p->nslices;
  p->smem = p->PS * p->CVB * K * VC * M * K * 4;
  if (p->smem > smem_optin) return false;
  const int64_t sstride = g.C * g.m * K * K;
  const int ngrp = (p->nslices + 31) / 32;
  const int64_t per_thread_rows = ((int64_t)p->rps + p->PS - 1) / p->PS;
  int lg = 0;
  while ((1 << lg) < 32) ++lg;
  int lg2 = 0;
  while ((1 << lg2) < ngrp) ++lg2;
  p->max_chain = (int)(std::min<int64_t>(64, g.Wo) + per_thread_rows * segs + (p->PS - 1) + lg + lg2 + 1);
  p->part_off = 0;
  p->l2_off = (size_t)p->nslices * sstride * 4;
  p->t1_off = p->l2_off + (size_t)ngrp * sstride * 4;
  p->t2_off = p->t1_off + (size_t)p->ncb * ngrp * 4;
  p->ws_bytes = (p->t2_off + (size_t)p->ncb * 4 + 15) & ~(size_t)15;
  return true;
}

cudaError_t launch_nhwc_gen_fd(const Geom& g, const NhwcGenPlan& p, const void* in, const void* w, void* out,
                               cudaStream_t st) {
  using namespace nhwcg;
  FdFn fn = fd_kernel(g.dtype, p.K, p.S, p.M, p.pass == DWCONV_PASS_BWD_DATA);
  if (!fn) return cudaErrorNotSupported;
  FArgs a{};
  a.in = in; a.w = w; a.out = out;
  a.N = (int)g.N; a.C = (int)g.C; a.H = (int)g.H; a.W = (int)g.W; a.Ho = (int)g.Ho; a.Wo = (int)g.Wo;
  a.CVB = p.CVB; a.ncb = p.ncb; a.slots = p.slots;
  a.OHB = p.OHB; a.OWB = p.OWB; a.tiles = p.tiles; a.ctas_per_cb = p.ctas_per_cb;
  if (p.smem > 48 * 1024 &&
      cudaFuncSetAttribute(reinterpret_cast<const void*>(fn), cudaFuncAttributeMaxDynamicSharedMemorySize, p.smem) !=
          cudaSuccess)
    return cudaErrorInvalidValue;
  void* args[] = {&a};
  return launch_ex(reinterpret_cast<const void*>(fn), p.grid, p.threads, p.smem, st, args);
}

cudaError_t launch_nhwc_gen_bf(const Geom& g, const NhwcGenPlan& p, const void* x, const void* dy, float* dw,
                               void* ws, cudaStream_t st) {
  using namespace nhwcg;
  if (p.tma) {
    BftFn fn = bft_kernel(g.dtype, p.K, p.S, p.M);
    EncodeFn enc = encode_fn();
    if (!fn || !enc) return cudaErrorNotSupported;
    const int eb = g.dtype == DWCONV_F32 ? 4 : 2;
    const CUtensorMapDataType dt = g.dtype == DWCONV_F32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
    CUtensorMap tmx, tmd;
    const cuuint32_t es[4] = {1, 1, 1, 1};
    {
      const cuuint64_t dims[4] = {(cuuint64_t)g.C, (cuuint64_t)g.W, (cuuint64_t)g.H, (cuuint64_t)g.N};
      const cuuint64_t str[3] = {(cuuint64_t)(g.C * eb), (cuuint64_t)(g.W * g.C * eb), (cuuint64_t)(g.H * g.W * g.C * eb)};
      const cuuint32_t box[4] = {(cuuint32_t)p.CB, (cuuint32_t)p.BWX, (cuuint32_t)p.XR, 1};
      if (enc(&tmx, dt, 4, const_cast<void*>(x), dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
              CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) !=
          CUDA_SUCCESS)
        return cudaErrorInvalidValue;
    }
    {
      const int64_t Co = g.C * g.m;
      const cuuint64_t dims[4] = {(cuuint64_t)Co, (cuuint64_t)g.Wo, (cuuint64_t)g.Ho, (cuuint64_t)g.N};
      const cuuint64_t str[3] = {(cuuint64_t)(Co * eb), (cuuint64_t)(g.Wo * Co * eb), (cuuint64_t)(g.Ho * g.Wo * Co * eb)};
      const cuuint32_t box[4] = {(cuuint32_t)(p.CB * g.m), (cuuint32_t)g.Wo, (cuuint32_t)p.TR, 1};
      if (enc(&tmd, dt, 4, const_cast<void*>(dy), dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
              CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) !=
          CUDA_SUCCESS)
        return cudaErrorInvalidValue;
    }
    unsigned char* b = static_cast<unsigned char*>(ws);
    TArgs a{};
    a.dw = dw;
    a.part = reinterpret_cast<float*>(b + p.part_off);
    a.l2 = reinterpret_cast<float*>(b + p.l2_off);
    a.t1 = reinterpret_cast<unsigned*>(b + p.t1_off);
    a.t2 = reinterpret_cast<unsigned*>(b + p.t2_off);
    a.C = (int)g.C; a.Ho = (int)g.Ho; a.Wo = (int)g.Wo;
    a.CB = p.CB; a.NCP = p.NCP; a.NCS = p.NCS; a.CW = p.CW; a.TR = p.TR; a.XR = p.XR; a.BWX = p.BWX;
    a.ncb = p.ncb; a.bpi = p.bpi; a.units = p.units; a.nslices = p.nslices; a.ups = p.ups;
    a.x_bytes = p.x_bytes; a.dy_bytes = p.dy_bytes; a.stage_bytes = p.stage_bytes;
    a.dy_off = (p.x_bytes + 127) & ~127u;
    if (p.smem > 48 * 1024 &&
        cudaFuncSetAttribute(reinterpret_cast<const void*>(fn), cudaFuncAttributeMaxDynamicSharedMemorySize,
                             p.smem) != cudaSuccess)
      return cudaErrorInvalidValue;
    void* args[] = {&tmx, &tmd, &a};
    return launch_ex(reinterpret_cast<const void*>(fn), p.grid, p.threads, p.smem, st, args);
  }
  BfFn fn = bf_kernel(g.dtype, p.K, p.S, p.M);
  if (!fn) return cudaErrorNotSupported;
  unsigned char* b = static_cast<unsigned char*>(ws);
  BArgs a{};
  a.x = x; a.dy = dy; a.dw = dw;
  a.part = reinterpret_cast<float*>(b + p.part_off);
  a.l2 = reinterpret_cast<float*>(b + p.l2_off);
  a.t1 = reinterpret_cast<unsigned*>(b + p.t1_off);
  a.t2 = reinterpret_cast<unsigned*>(b + p.t2_off);
  a.N = (int)g.N; a.C = (int)g.C; a.H = (int)g.H; a.W = (int)g.W; a.Ho = (int)g.Ho; a.Wo = (int)g.Wo;
  a.CVB = p.CVB; a.ncb = p.ncb; a.PS = p.PS; a.nslices = p.nslices; a.rps = p.rps;
  if (p.smem > 48 * 1024 &&
      cudaFuncSetAttribute(reinterpret_cast<const void*>(fn), cudaFuncAttributeMaxDynamicSharedMemorySize, p.smem) !=
          cudaSuccess)
    return cudaErrorInvalidValue;
  void* args[] = {&a};
  return launch_ex(reinterpret_cast<const void*>(fn), p.grid, p.threads, p.smem, st, args);
}

}  // namespace dwk
