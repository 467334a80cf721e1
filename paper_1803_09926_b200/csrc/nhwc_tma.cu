// nhwc_tma.cu -- NHWC fwd and bwd_data from tensor-map TMA tiles (sm_100a),
// multiplier m = 1, 3x3, pad 1, S in {1, 2}.
//
//   fwd (Eq. 3):
//     y[n, oh, ow, c] = sum_{i,j} w[c, i, j] * x[n, oh*S-1+i, ow*S-1+j, c]
//   bwd_data (the adjoint, reading R9):
//     dx[n, ih, iw, c] = sum_{i,j: (ih+1-i) % S == 0, (iw+1-j) % S == 0} w[c, i, j] * dy[n, (ih+1-i)/S, (iw+1-j)/S, c]
//
// A tile is TH x TW output pixels x CB channels (CB * eb = 128 B, or all of C
// when C is smaller).  Its input window is ONE 4-D tensor-map box
// {CB, box_w, box_h, 1} of the NHWC tensor (cp.async.bulk.tensor.4d -> UTMALDG):
// the box starts one pixel above/left of the tile, and the TMA unit fills the
// out-of-bounds halo with zeros, so the stencil has no bounds checks at all.
// Warp 0 is the producer (one lane issues the boxes into a ring of `ns` stages
// with full/empty mbarriers); the other warps are consumers.  A consumer thread
// owns VC = 4 channels (a 16-B fp32 / 8-B bf16 vector; consecutive lanes take
// consecutive vectors, so every shared-memory wavefront is a contiguous 128 B)
// and one output column of the tile, walks its TH rows with a sliding window in
// registers (stride 1: 3 new vectors per output row; stride 2: 6), accumulates
// in fp32 with packed FFMA2 over channel pairs, and stores straight to global
// memory (coalesced: the lanes of a pixel write its contiguous channel run).
//
//   * bwd_data, stride 1: the forward stencil over dy with the kernel rotated
//     by 180 degrees (w'[i][j] = w[2-i][2-j]).
//   * bwd_data, stride 2 (polyphase): a thread owns a dx column PAIR (2b, 2b+1)
//     and walks dx row pairs (2a, 2a+1); every dx value is 1, 2 or 4 taps of the
//     dy 2x2 neighbourhood (a..a+1, b..b+1); the dy box starts at (oh0/2, ow0/2).
#include <cuda.h>

#include <mutex>
#include <vector>

#include "kernels.h"
#include "nchw_common.cuh"

namespace dwk {
namespace nhwct {

using nchw::VecIO;
constexpr int VC = 4;
constexpr int kMaxConsumers = 256;

enum Mode { kFwd1 = 0, kFwd2 = 1, kBd1 = 2, kBd2 = 3 };

struct TArgs {
  void* out;
  const void* w;
  int N, C, OH, OW;        // output tensor dims (y for fwd, dx for bwd_data)
  int CB, NCV;             // channels per tile, channel vectors per tile
  int TW;                  // output columns per tile (TH is the template parameter)
  int tiles_h, tiles_w, ncb;
  int64_t ntiles;
  int BW;                  // box width (pixels)
  uint32_t box_bytes, stage_bytes;
  int ns, cons;            // ring depth, consumer threads
  int early_pdl;
};

__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* tm, int c0, int c1, int c2, int c3,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];"
      ::"r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(tm)), "r"(c0), "r"(c1), "r"(c2), "r"(c3),
      "r"(smem_u32(bar))
      : "memory");
}

struct Tile { int n, cb, oh0, ow0; };

__device__ __forceinline__ Tile decode(const TArgs& a, int64_t t64) {  // ntiles < 2^31 (planner)
  Tile k;
  uint32_t t = (uint32_t)t64;
  const uint32_t t1 = t / (uint32_t)a.tiles_w;
  const int tw = (int)(t - t1 * (uint32_t)a.tiles_w);
  const uint32_t t2 = t1 / (uint32_t)a.tiles_h;
  const int th = (int)(t1 - t2 * (uint32_t)a.tiles_h);
  k.cb = (int)(t2 / (uint32_t)a.N);
  k.n = (int)(t2 - (uint32_t)k.cb * (uint32_t)a.N);
  k.oh0 = th;  // scaled by TH in the kernel
  k.ow0 = tw * a.TW;
  return k;
}

template <class T>
__device__ __forceinline__ void ld4(const T* p, float2& lo, float2& hi) {
  float v[4];
  VecIO<T, 4>::load(p, v);
  lo = make_float2(v[0], v[1]);
  hi = make_float2(v[2], v[3]);
}

template <class T, int MODE, int TH>
__global__ void __launch_bounds__(kMaxConsumers + 32) nhwc_tma_kernel(const __grid_constant__ CUtensorMap tm,
                                                                       const TArgs a) {
  constexpr int S = (MODE == kFwd2 || MODE == kBd2) ? 2 : 1;
  static_assert(MODE != kBd2 || TH % 2 == 0, "stride-2 dx tiles have whole row pairs");
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  uint64_t* empty = reinterpret_cast<uint64_t*>(smem + 64);
  const int nwarps_c = (a.cons + 31) >> 5;
  if (threadIdx.x == 0) {
    for (int i = 0; i < a.ns; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], nwarps_c);
    }
    fence_mbar_init();
  }
  __syncthreads();
  griddep_wait();
  auto stage = [&](int s) { return reinterpret_cast<T*>(smem + 128 + (size_t)s * a.stage_bytes); };

  if (threadIdx.x < 32) {
    // ------------------------------------------------------------ producer
    if (threadIdx.x == 0) {
      int s = 0;
      uint32_t ph = 0;
      int it = 0;
      for (int64_t t = blockIdx.x; t < a.ntiles; t += gridDim.x, ++it) {
        if (it >= a.ns) mbar_wait(&empty[s], ph ^ 1);
        const Tile k = decode(a, t);
        const int oh0 = k.oh0 * TH;
        int x0, y0;
        if constexpr (MODE == kBd2) { x0 = k.ow0 / 2; y0 = oh0 / 2; }
        else { x0 = k.ow0 * S - 1; y0 = oh0 * S - 1; }
        mbar_arrive_expect_tx(&full[s], a.box_bytes);
        tma_load_4d(stage(s), &tm, k.cb * a.CB, x0, y0, k.n, &full[s]);
        if (++s == a.ns) { s = 0; ph ^= 1; }
      }
      if (a.early_pdl) griddep_launch_dependents();
    }
    return;
  }
  // -------------------------------------------------------------- consumers
  const int ctid = threadIdx.x - 32;
  const int cv = ctid % a.NCV;
  const int col = ctid / a.NCV;  // output column (kBd2: column pair)
  const int ncols = (MODE == kBd2) ? a.TW / 2 : a.TW;
  const bool live = ctid < a.cons && col < ncols;
  const T* __restrict__ wt = static_cast<const T*>(a.w);
  T* __restrict__ out = static_cast<T*>(a.out);
  const int C = a.C, CB = a.CB, BW = a.BW;
  float2 w2[9][2];
  int wcb = -1;
  int s = 0;
  uint32_t ph = 0;
  for (int64_t t = blockIdx.x; t < a.ntiles; t += gridDim.x) {
    const Tile k = decode(a, t);
    const int oh0 = k.oh0 * TH;
    const int c0 = k.cb * CB + cv * VC;
    if (live && k.cb != wcb) {
      wcb = k.cb;
#pragma unroll
      for (int q = 0; q < 9; ++q) {
        const int qs = (MODE == kBd1) ? 8 - q : q;  // 180-degree rotation for the stride-1 adjoint
        float wv[VC];
#pragma unroll
        for (int v = 0; v < VC; ++v) wv[v] = Elem<T>::ldg(wt + (int64_t)(c0 + v) * 9 + qs);
        w2[q][0] = make_float2(wv[0], wv[1]);
        w2[q][1] = make_float2(wv[2], wv[3]);
      }
    }
    mbar_wait(&full[s], ph);
    if (live) {
      // running pointers only (no per-access index arithmetic): smem rows step by
      // rowS elements, window columns by CB; output rows by OW * C
      const int rowS = BW * CB;
      const int64_t orow = (int64_t)a.OW * C;
      if constexpr (MODE == kBd2) {
        const int b = col;  // dy box columns b, b+1 -> dx columns 2b, 2b+1
        const T* pr = stage(s) + cv * VC + b * CB;
        float2 d0[2][2], d1[2][2];  // [column][channel pair] of dy rows a (d0) and a+1 (d1)
        ld4<T>(pr, d0[0][0], d0[0][1]);
        ld4<T>(pr + CB, d0[1][0], d0[1][1]);
        const int ow = k.ow0 + 2 * b;
        const bool ok0 = ow < a.OW, ok1 = ow + 1 < a.OW;
        const int rmax = a.OH - oh0;  // dx rows of this tile inside the tensor
        T* po = out + (((int64_t)k.n * a.OH + oh0) * a.OW + ow) * C + c0;
#pragma unroll
        for (int ap = 0; ap < TH / 2; ++ap) {
          pr += rowS;
          ld4<T>(pr, d1[0][0], d1[0][1]);
          ld4<T>(pr + CB, d1[1][0], d1[1][1]);
          float2 o[4][2];  // (even,even) (even,odd) (odd,even) (odd,odd)
#pragma unroll
          for (int v = 0; v < 2; ++v) {
            o[0][v] = __fmul2_rn(w2[4][v], d0[0][v]);
            o[1][v] = __ffma2_rn(w2[5][v], d0[0][v], __fmul2_rn(w2[3][v], d0[1][v]));
            o[2][v] = __ffma2_rn(w2[7][v], d0[0][v], __fmul2_rn(w2[1][v], d1[0][v]));
            o[3][v] = __ffma2_rn(w2[8][v], d0[0][v],
                                 __ffma2_rn(w2[6][v], d0[1][v],
                                            __ffma2_rn(w2[2][v], d1[0][v], __fmul2_rn(w2[0][v], d1[1][v]))));
          }
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int rr = 2 * ap + (u >> 1);
            if (rr < rmax && ((u & 1) ? ok1 : ok0)) {
              const float ov[4] = {o[u][0].x, o[u][0].y, o[u][1].x, o[u][1].y};
              VecIO<T, 4>::store(po + (u >> 1) * orow + (u & 1) * C, ov);
            }
          }
          po += 2 * orow;
#pragma unroll
          for (int cc = 0; cc < 2; ++cc)
#pragma unroll
            for (int v = 0; v < 2; ++v) d0[cc][v] = d1[cc][v];
        }
      } else {
        // window rows held: stride 1 keeps 2 rows and loads 1 per output row; stride 2 keeps 1 and loads 2
        const T* pr = stage(s) + cv * VC + col * S * CB;  // box row 0, first window column
        float2 xw[3][3][2];  // [row][column][channel pair]
#pragma unroll
        for (int r = 0; r < 3 - S; ++r) {
#pragma unroll
          for (int j = 0; j < 3; ++j) ld4<T>(pr + j * CB, xw[r][j][0], xw[r][j][1]);
          pr += rowS;
        }
        const int ow = k.ow0 + col;
        const int rmax = (ow < a.OW) ? a.OH - oh0 : 0;
        T* po = out + (((int64_t)k.n * a.OH + oh0) * a.OW + ow) * C + c0;
#pragma unroll
        for (int r = 0; r < TH; ++r) {
#pragma unroll
          for (int rr = 3 - S; rr < 3; ++rr) {
#pragma unroll
            for (int j = 0; j < 3; ++j) ld4<T>(pr + j * CB, xw[rr][j][0], xw[rr][j][1]);
            pr += rowS;
          }
          // two partial chains per channel pair (taps 0-4, 5-8): shorter FFMA2 dependency
          float2 acc[2], acc2[2];
#pragma unroll
          for (int v = 0; v < 2; ++v) {
            acc[v] = __fmul2_rn(w2[0][v], xw[0][0][v]);
            acc2[v] = __fmul2_rn(w2[5][v], xw[1][2][v]);
#pragma unroll
            for (int q = 1; q < 5; ++q) acc[v] = __ffma2_rn(w2[q][v], xw[q / 3][q % 3][v], acc[v]);
#pragma unroll
            for (int q = 6; q < 9; ++q) acc2[v] = __ffma2_rn(w2[q][v], xw[q / 3][q % 3][v], acc2[v]);
            acc[v] = __fadd2_rn(acc[v], acc2[v]);
          }
          if (r < rmax) {
            const float ov[4] = {acc[0].x, acc[0].y, acc[1].x, acc[1].y};
            VecIO<T, 4>::store(po, ov);
          }
          po += orow;
#pragma unroll
          for (int rr = 0; rr < 3 - S; ++rr)
#pragma unroll
            for (int j = 0; j < 3; ++j)
#pragma unroll
              for (int v = 0; v < 2; ++v) xw[rr][j][v] = xw[rr + S][j][v];
        }
      }
    }
    __syncwarp();
    if ((threadIdx.x & 31) == 0) mbar_arrive(&empty[s]);
    if (++s == a.ns) { s = 0; ph ^= 1; }
  }
  if (!a.early_pdl) griddep_launch_dependents();
}

// ---------------------------------------------------------------- bwd_filter
// dw[c, i, j] = sum_{n, oh, ow} x[n, oh*S-1+i, ow*S-1+j, c] * dy[n, oh, ow, c]
// (the block diagonal Eq. 4 keeps, summed over the batch:
// reading R5).  A stage holds the tile's x box (zero-filled halo) and its dy box
// (zero-filled past the edges, so ragged tiles add exact zeros).  CTA = (channel
// block, slice of the block's tiles); consumer thread = (channel vector, tile
// column), walking the TH rows with the forward's sliding x window.
// Deterministic reduction, fixed order everywhere:
//   per tile (TH terms, FFMA2) -> running sum over the CTA's tiles (<= 64)
//   -> tile columns pairwise -> per-slice partial in the workspace; the last CTA
//   of the channel block (integer ticket) sums the slices pairwise in slice
//   order and re-zeroes the workspace.  No float atomics.
struct BArgs {
  float* dw;
  float* ws_part;
  unsigned* ws_ticket;
  int N, C, CB, NCV, TW;
  int tiles_h, tiles_w, ncb, nslices, tps;
  int tiles_per_cb;
  int BW, DBW;  // x box width, dy box width (pixels)
  uint32_t x_bytes, dy_bytes, dy_off, stage_bytes;
  int ns, cons;
  int early_pdl;
};

template <class T, int S, int TH>
__global__ void __launch_bounds__(kMaxConsumers + 32) nhwc_tma_bf_kernel(const __grid_constant__ CUtensorMap tmx,
                                                                          const __grid_constant__ CUtensorMap tmd,
                                                                          const BArgs a) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ unsigned s_last;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  uint64_t* empty = reinterpret_cast<uint64_t*>(smem + 64);
  const int nwarps_c = (a.cons + 31) >> 5;
  if (threadIdx.x == 0) {
    for (int i = 0; i < a.ns; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], nwarps_c);
    }
    fence_mbar_init();
  }
  __syncthreads();
  griddep_wait();
  const int g = blockIdx.x % a.ncb;
  const int sl = blockIdx.x / a.ncb;
  const int t0 = sl * a.tps;
  const int t1 = min(a.tiles_per_cb, t0 + a.tps);
  auto sx = [&](int s) { return reinterpret_cast<T*>(smem + 128 + (size_t)s * a.stage_bytes); };
  auto sd = [&](int s) { return reinterpret_cast<T*>(smem + 128 + (size_t)s * a.stage_bytes + a.dy_off); };
  auto dec = [&](int t, int* n, int* oh0, int* ow0) {
    const int q1 = t / a.tiles_w;
    *ow0 = (t - q1 * a.tiles_w) * a.TW;
    const int q2 = q1 / a.tiles_h;
    *oh0 = (q1 - q2 * a.tiles_h) * TH;
    *n = q2;
  };
  const int ctid = (int)threadIdx.x - 32;
  const int cv = ctid % a.NCV;
  const int col = ctid / a.NCV;
  const bool live = ctid >= 0 && ctid < a.cons && col < a.TW;
  float2 run[9][2];
#pragma unroll
  for (int q = 0; q < 9; ++q) run[q][0] = run[q][1] = make_float2(0.f, 0.f);

  if (threadIdx.x < 32) {
    if (threadIdx.x == 0) {  // producer
      int s = 0, it = 0;
      uint32_t ph = 0;
      for (int t = t0; t < t1; ++t, ++it) {
        if (it >= a.ns) mbar_wait(&empty[s], ph ^ 1);
        int n, oh0, ow0;
        dec(t, &n, &oh0, &ow0);
        mbar_arrive_expect_tx(&full[s], a.x_bytes + a.dy_bytes);
        tma_load_4d(sx(s), &tmx, g * a.CB, ow0 * S - 1, oh0 * S - 1, n, &full[s]);
        tma_load_4d(sd(s), &tmd, g * a.CB, ow0, oh0, n, &full[s]);
        if (++s == a.ns) { s = 0; ph ^= 1; }
      }
      if (a.early_pdl) griddep_launch_dependents();
    }
  } else {
    int s = 0;
    uint32_t ph = 0;
    const int rowS = a.BW * a.CB, drowS = a.DBW * a.CB, CB = a.CB;
    for (int t = t0; t < t1; ++t) {
      mbar_wait(&full[s], ph);
      if (live) {
        const T* pr = sx(s) + cv * VC + col * S * CB;
        const T* pd = sd(s) + cv * VC + col * CB;
        float2 xw[3][3][2];
#pragma unroll
        for (int r = 0; r < 3 - S; ++r) {
#pragma unroll
          for (int j = 0; j < 3; ++j) ld4<T>(pr + j * CB, xw[r][j][0], xw[r][j][1]);
          pr += rowS;
        }
        float2 loc[9][2];
#pragma unroll
        for (int r = 0; r < TH; ++r) {
#pragma unroll
          for (int rr = 3 - S; rr < 3; ++rr) {
#pragma unroll
            for (int j = 0; j < 3; ++j) ld4<T>(pr + j * CB, xw[rr][j][0], xw[rr][j][1]);
            pr += rowS;
          }
          float2 dv[2];
          ld4<T>(pd, dv[0], dv[1]);
          pd += drowS;
#pragma unroll
          for (int q = 0; q < 9; ++q)
#pragma unroll
            for (int v = 0; v < 2; ++v)
              loc[q][v] = (r == 0) ? __fmul2_rn(xw[q / 3][q % 3][v], dv[v])
                                   : __ffma2_rn(xw[q / 3][q % 3][v], dv[v], loc[q][v]);
#pragma unroll
          for (int rr = 0; rr < 3 - S; ++rr)
#pragma unroll
            for (int j = 0; j < 3; ++j)
#pragma unroll
              for (int v = 0; v < 2; ++v) xw[rr][j][v] = xw[rr + S][j][v];
        }
#pragma unroll
        for (int q = 0; q < 9; ++q)
#pragma unroll
          for (int v = 0; v < 2; ++v) run[q][v] = __fadd2_rn(run[q][v], loc[q][v]);
      }
      __syncwarp();
      if ((threadIdx.x & 31) == 0) mbar_arrive(&empty[s]);
      if (++s == a.ns) { s = 0; ph ^= 1; }
    }
  }
  if (!a.early_pdl) griddep_launch_dependents();
  // ---- every stage has been consumed (no TMA write is pending): reuse the ring
  __syncthreads();
  float* red = reinterpret_cast<float*>(smem + 128);  // [col][cv][q*4 + ch]
  if (live) {
#pragma unroll
    for (int q = 0; q < 9; ++q) {
      float* d = red + ((int64_t)col * a.NCV + cv) * 36 + q * 4;
      d[0] = run[q][0].x; d[1] = run[q][0].y; d[2] = run[q][1].x; d[3] = run[q][1].y;
    }
  }
  __syncthreads();
  const int C = a.C;
  float* part = a.ws_part + (int64_t)sl * C * 9;
  for (int e = threadIdx.x; e < a.NCV * 36; e += blockDim.x) {
    const int cvv = e / 36, rem = e - cvv * 36;
    const int q = rem >> 2, ch = rem & 3;
    float stk[8];
    int top = 0;
    for (int c2 = 0; c2 < a.TW; ++c2) {  // tile columns pairwise (binary counter)
      float cur = red[((int64_t)c2 * a.NCV + cvv) * 36 + rem];
      int bits = c2;
      while (bits & 1) { cur = stk[--top] + cur; bits >>= 1; }
      stk[top++] = cur;
    }
    float tot = stk[--top];
    while (top > 0) tot = stk[--top] + tot;
    part[(int64_t)(g * a.CB + cvv * VC + ch) * 9 + q] = tot;
  }
  __threadfence();
  __syncthreads();
  const int ngrp = (a.nslices + 31) / 32;
  nchw::finalize_two_level(a.ws_part, a.ws_part + (int64_t)a.nslices * C * 9, a.ws_ticket, a.ws_ticket + a.ncb * ngrp,
                           g, sl, a.nslices, (int64_t)C * 9, (int64_t)g * a.CB * 9, a.CB * 9, a.dw, &s_last);
}

using BKernelFn = void (*)(const CUtensorMap, const CUtensorMap, const BArgs);
BKernelFn bf_kernel_for(int dtype, int S, int TH) {
  if (S == 1 && TH == 14)  // two-strip tiles (stride 1)
    return dtype == DWCONV_F32 ? nhwc_tma_bf_kernel<float, 1, 14> : nhwc_tma_bf_kernel<__nv_bfloat16, 1, 14>;
  if (dtype == DWCONV_F32) {
    if (S == 1) return TH == 7 ? nhwc_tma_bf_kernel<float, 1, 7> : nhwc_tma_bf_kernel<float, 1, 8>;
    return TH == 7 ? nhwc_tma_bf_kernel<float, 2, 7> : nhwc_tma_bf_kernel<float, 2, 8>;
  }
  using B = __nv_bfloat16;
  if (S == 1) return TH == 7 ? nhwc_tma_bf_kernel<B, 1, 7> : nhwc_tma_bf_kernel<B, 1, 8>;
  return TH == 7 ? nhwc_tma_bf_kernel<B, 2, 7> : nhwc_tma_bf_kernel<B, 2, 8>;
}

using TKernelFn = void (*)(const CUtensorMap, const TArgs);

template <class T, int MODE>
TKernelFn pick_th(int TH) {
  if constexpr (MODE == kBd2) {
    return TH == 14 ? nhwc_tma_kernel<T, MODE, 14> : (TH == 8 ? nhwc_tma_kernel<T, MODE, 8> : nullptr);
  } else {
    if constexpr (MODE == kFwd1 || MODE == kBd1)  // stride 1 also has two-strip (14-row) tiles
      if (TH == 14) return nhwc_tma_kernel<T, MODE, 14>;
    return TH == 7 ? nhwc_tma_kernel<T, MODE, 7> : (TH == 8 ? nhwc_tma_kernel<T, MODE, 8> : nullptr);
  }
}
template <class T>
TKernelFn pick_mode(int mode, int TH) {
  switch (mode) {
    case kFwd1: return pick_th<T, kFwd1>(TH);
    case kFwd2: return pick_th<T, kFwd2>(TH);
    case kBd1: return pick_th<T, kBd1>(TH);
    case kBd2: return pick_th<T, kBd2>(TH);
    default: return nullptr;
  }
}
TKernelFn kernel_for(int dtype, int mode, int TH) {
  return dtype == DWCONV_F32 ? pick_mode<float>(mode, TH) : pick_mode<__nv_bfloat16>(mode, TH);
}

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn encode_fn() {
  static EncodeFn fn = []() -> EncodeFn {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return nullptr;
    return reinterpret_cast<EncodeFn>(p);
  }();
  return fn;
}

// Opt a kernel in to the largest dynamic shared memory it can use (the opt-in
// limit minus its static shared memory), once: the attribute is per function, so
// every plan of that kernel must fit under the same setting.
bool allow_max_smem(const void* fn, int smem_optin) {
  static std::mutex mu;
  static std::vector<const void*> done;
  std::lock_guard<std::mutex> lk(mu);
  for (const void* f : done)
    if (f == fn) return true;
  cudaFuncAttributes fa{};
  if (cudaFuncGetAttributes(&fa, fn) != cudaSuccess) return false;
  if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_optin - (int)fa.sharedSizeBytes) !=
      cudaSuccess)
    return false;
  done.push_back(fn);
  return true;
}

int env_int(const char* name, int dflt, int lo, int hi) {
  const char* e = dev_knob(name);
  const int v = e ? std::atoi(e) : dflt;
  return (v >= lo && v <= hi) ? v : dflt;
}

}  // namespace nhwct

// Plan: mode, channel block, tile, box, ring depth, grid.  false = not eligible.
bool plan_nhwc_tma(const Geom& g, int pass, int num_sms, int smem_optin, NhwcTmaPlan* p, int tw_max, int stages,
                   int th) {
  using namespace nhwct;
  static const int on = env_int("DWCONV_NHWC_TMA", 1, 0, 1);
  if (!on || g.layout != DWCONV_NHWC || g.m != 1 || g.kh != 3 || g.kw != 3 || g.ph != 1 || g.pw != 1) return false;
  if (pass != DWCONV_PASS_FWD && pass != DWCONV_PASS_BWD_DATA) return false;
  const int S = g.sh;
  if (g.sw != S || (S != 1 && S != 2)) return false;
  if (!encode_fn()) return false;
  const int64_t eb = (g.dtype == DWCONV_F32) ? 4 : 2;
  if ((g.C * eb) % 16 != 0 || g.C % VC != 0) return false;  // tensor-map strides: 16-B multiples
  if (g.N > INT32_MAX || g.H > 65535 || g.W > 65535) return false;
  *p = NhwcTmaPlan{};
  const bool fwd = pass == DWCONV_PASS_FWD;
  p->mode = fwd ? (S == 1 ? kFwd1 : kFwd2) : (S == 1 ? kBd1 : kBd2);
  const int64_t OH = fwd ? g.Ho : g.H, OW = fwd ? g.Wo : g.W;
  // channel block: one 128-B run per pixel (or all of C), dividing C
  int64_t CB = std::min<int64_t>(g.C, 128 / eb);
  while (CB > VC && (g.C % CB != 0 || CB % VC != 0)) CB -= VC;
  if (g.C % CB != 0 || (CB * eb) % 16 != 0) return false;
  const int NCV = (int)(CB / VC);
  // tile: TH rows (7 when it divides the output height), TW columns (largest
  // divisor of the output width <= the CTA's thread budget)
  int TH = (OH % 7 == 0) ? 7 : 8;
  if (p->mode == kBd2) TH = (OH % 14 == 0) ? 14 : 8;
  if (th == 14 && (p->mode == kFwd1 || p->mode == kBd1)) {
    if (OH % 14 != 0) return false;
    TH = 14;
  }
  static const int tw_max_env0 = env_int("DWCONV_NHWC_TW", 16, 1, 64);
  const int tw_max_env = tw_max > 0 ? tw_max : tw_max_env0;
  const int per_col = (p->mode == kBd2) ? 2 : 1;  // dx columns per consumer thread
  int tw_cap = std::min<int>(tw_max_env * per_col, (kMaxConsumers / NCV) * per_col);
  int TW = 0;
  for (int t = (int)std::min<int64_t>(OW, tw_cap); t >= 1; --t) {
    if (p->mode == kBd2 && (t % 2)) continue;
    if (OW % t == 0) { TW = t; break; }
  }
  if (TW == 0 || (TW < tw_cap / 2 && OW > tw_cap)) TW = (p->mode == kBd2) ? (tw_cap & ~1) : tw_cap;  // ragged last tile
  if (TW < 1) return false;
  auto box_of = [&](int tw, int* bw, int* bh) {
    if (p->mode == kBd2) { *bw = tw / 2 + 1; *bh = TH / 2 + 1; }
    else { *bw = (tw - 1) * S + 3; *bh = (TH - 1) * S + 3; }
  };
  int BW, BH;
  box_of(TW, &BW, &BH);
  // keep the ring of a CTA <= ~100 KB so two or more CTAs share an SM (stride-2
  // forward boxes are 4x the tile): narrower tiles, still dividing the width
  static const int ns_env = env_int("DWCONV_NHWC_STAGES", 4, 2, 8);
  const int ns_want = stages > 0 ? stages : ns_env;
  while ((int64_t)ns_want * CB * BW * BH * eb > 100 * 1024 && TW > 4) {
    int t = TW - 1;
    while (t > 4 && (OW % t != 0 || (p->mode == kBd2 && (t % 2)))) --t;
    TW = t;
    box_of(TW, &BW, &BH);
  }
  if (BW > 256 || BH > 256) return false;
  p->TH = TH; p->TW = TW; p->CB = (int)CB; p->NCV = NCV; p->BW = BW; p->BH = BH;
  p->cons = NCV * (TW / per_col);
  p->box_bytes = (uint32_t)(CB * BW * BH * eb);
  p->stage_bytes = (p->box_bytes + 127u) & ~127u;
  p->tiles_h = (int)((OH + TH - 1) / TH);
  p->tiles_w = (int)((OW + TW - 1) / TW);
  p->ncb = (int)(g.C / CB);
  p->ntiles = g.N * p->tiles_h * p->tiles_w * p->ncb;
  if (p->ntiles >= ((int64_t)1 << 31)) return false;
  p->ns = ns_want;
  while (p->ns > 2 && 128 + (int64_t)p->ns * p->stage_bytes > smem_optin) --p->ns;
  p->smem = (int)(128 + p->ns * p->stage_bytes);
  if (p->smem > smem_optin - 1024) return false;
  TKernelFn fn = kernel_for(g.dtype, p->mode, TH);
  if (!fn) return false;
  p->threads = 32 + ((p->cons + 31) / 32) * 32;
  if (!allow_max_smem(reinterpret_cast<const void*>(fn), smem_optin)) return false;
  int occ = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, p->threads, p->smem) != cudaSuccess || occ < 1)
    return false;
  p->grid = (int)std::min<int64_t>(p->ntiles, (int64_t)occ * num_sms);
  return p->ntiles > 0;
}

cudaError_t launch_nhwc_tma(const Geom& g, const NhwcTmaPlan& p, const void* in, const void* w, void* out,
                            cudaStream_t st) {
  using namespace nhwct;
  const bool bd = p.mode == kBd1 || p.mode == kBd2;
  // the box source: x (fwd) or dy (bwd_data), NHWC, dims innermost first {C, W, H, N}
  const int64_t IH = bd ? g.Ho : g.H, IW = bd ? g.Wo : g.W;
  const int64_t eb = (g.dtype == DWCONV_F32) ? 4 : 2;
  CUtensorMap tm;
  const cuuint64_t dims[4] = {(cuuint64_t)g.C, (cuuint64_t)IW, (cuuint64_t)IH, (cuuint64_t)g.N};
  const cuuint64_t strides[3] = {(cuuint64_t)(g.C * eb), (cuuint64_t)(g.C * IW * eb), (cuuint64_t)(g.C * IW * IH * eb)};
  const cuuint32_t box[4] = {(cuuint32_t)p.CB, (cuuint32_t)p.BW, (cuuint32_t)p.BH, 1};
  const cuuint32_t es[4] = {1, 1, 1, 1};
  EncodeFn enc = encode_fn();
  if (!enc) return cudaErrorNotSupported;
  const CUresult r = enc(&tm, g.dtype == DWCONV_F32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16,
                         4, const_cast<void*>(in), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return cudaErrorInvalidValue;
  TArgs a{};
  a.out = out; a.w = w;
  a.N = (int)g.N; a.C = (int)g.C;
  a.OH = (int)(bd ? g.H : g.Ho); a.OW = (int)(bd ? g.W : g.Wo);
  a.CB = p.CB; a.NCV = p.NCV; a.TW = p.TW;
  a.tiles_h = p.tiles_h; a.tiles_w = p.tiles_w; a.ncb = p.ncb; a.ntiles = p.ntiles;
  a.BW = p.BW; a.box_bytes = p.box_bytes; a.stage_bytes = p.stage_bytes;
  a.ns = p.ns; a.cons = p.cons;
  static const int early = env_int("DWCONV_EARLY_PDL", 1, 0, 1);
  a.early_pdl = early;
  TKernelFn fn = kernel_for(g.dtype, p.mode, p.TH);
  if (!fn) return cudaErrorInvalidValue;
  static const bool pdl = env_int("DWCONV_PDL", 1, 0, 1) == 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)p.grid);
  cfg.blockDim = dim3((unsigned)p.threads);
  cfg.dynamicSmemBytes = (size_t)p.smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, fn, tm, a);
}

bool plan_nhwc_tma_bf(const Geom& g, int num_sms, int smem_optin, NhwcTmaPlan* p, int tw_max, int stages,
                      int th) {
  using namespace nhwct;
  static const int on = env_int("DWCONV_NHWC_TMA", 1, 0, 1);
  if (!on || g.layout != DWCONV_NHWC || g.m != 1 || g.kh != 3 || g.kw != 3 || g.ph != 1 || g.pw != 1) return false;
  const int S = g.sh;
  if (g.sw != S || (S != 1 && S != 2)) return false;
  if (!encode_fn()) return false;
  const int64_t eb = (g.dtype == DWCONV_F32) ? 4 : 2;
  if ((g.C * eb) % 16 != 0 || g.C % VC != 0) return false;
  if (g.N > INT32_MAX || g.H > 65535 || g.W > 65535) return false;
  *p = NhwcTmaPlan{};
  p->mode = 4 + S;  // bwd_filter
  int64_t CB = std::min<int64_t>(g.C, 128 / eb);
  while (CB > VC && (g.C % CB != 0 || CB % VC != 0)) CB -= VC;
  if (g.C % CB != 0 || (CB * eb) % 16 != 0) return false;
  const int NCV = (int)(CB / VC);
  int TH = (g.Ho % 7 == 0) ? 7 : 8;
  if (th == 14) {
    if (S != 1 || g.Ho % 14 != 0) return false;
    TH = 14;
  }
  static const int tw_env0 = env_int("DWCONV_NHWC_TW", 16, 1, 64);
  const int tw_env = tw_max > 0 ? tw_max : tw_env0;
  const int tw_cap = std::max(1, std::min(tw_env, kMaxConsumers / NCV));
  int TW = 0;
  for (int t = (int)std::min<int64_t>(g.Wo, tw_cap); t >= 1; --t)
    if (g.Wo % t == 0) { TW = t; break; }
  if (TW < tw_cap / 2 && g.Wo > tw_cap) TW = tw_cap;
  static const int ns_env = env_int("DWCONV_NHWC_STAGES", 4, 2, 8);
  const int ns_want = stages > 0 ? stages : ns_env;
  auto sizes = [&](int tw, int* bw, int* bh, uint32_t* xb, uint32_t* db) {
    *bw = (tw - 1) * S + 3; *bh = (TH - 1) * S + 3;
    *xb = (uint32_t)(CB * *bw * *bh * eb);
    *db = (uint32_t)(CB * tw * TH * eb);
  };
  int BW, BH;
  uint32_t xb, db;
  sizes(TW, &BW, &BH, &xb, &db);
  // a shallower ring before narrower tiles (consumer threads = NCV x TW): keep
  // the CTA's ring <= ~100 KB so two CTAs share an SM
  int ns_fit = ns_want;
  while (ns_fit > 2 && (int64_t)ns_fit * (xb + db) > 100 * 1024) --ns_fit;
  while ((int64_t)ns_fit * (xb + db) > 100 * 1024 && TW > 4) {
    int t = TW - 1;
    while (t > 4 && g.Wo % t != 0) --t;
    TW = t;
    sizes(TW, &BW, &BH, &xb, &db);
  }
  if (BW > 256 || BH > 256 || TW > 256) return false;
  p->TH = TH; p->TW = TW; p->CB = (int)CB; p->NCV = NCV; p->BW = BW; p->BH = BH;
  p->cons = NCV * TW;
  p->box_bytes = xb;
  p->dy_bytes = db;
  p->dy_off = (xb + 127u) & ~127u;
  p->stage_bytes = (p->dy_off + db + 127u) & ~127u;
  p->tiles_h = (int)((g.Ho + TH - 1) / TH);
  p->tiles_w = (int)((g.Wo + TW - 1) / TW);
  p->ncb = (int)(g.C / CB);
  const int64_t tpc = g.N * p->tiles_h * p->tiles_w;
  if (tpc >= ((int64_t)1 << 31) || tpc < 1) return false;
  p->tiles_per_cb = (int)tpc;
  p->ns = ns_fit;
  const uint32_t red_bytes = (uint32_t)(TW * NCV * 36 * 4);
  while (p->ns > 2 && 128 + (int64_t)p->ns * p->stage_bytes > smem_optin) --p->ns;
  p->smem = (int)(128 + std::max<uint32_t>(p->ns * p->stage_bytes, red_bytes));
  if (p->smem > smem_optin - 1024) return false;
  BKernelFn fn = bf_kernel_for(g.dtype, S, TH);
  p->threads = 32 + ((p->cons + 31) / 32) * 32;
  if (!allow_max_smem(reinterpret_cast<const void*>(fn), smem_optin)) return false;
  int occ = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, p->threads, p->smem) != cudaSuccess || occ < 1)
    return false;
  // slices: one full wave of CTAs, <= 64 tiles per CTA (running-sum chain), <= 1024 slices
  int64_t nsl = std::max<int64_t>(1, ((int64_t)occ * num_sms) / p->ncb);
  nsl = std::max<int64_t>(nsl, (tpc + 63) / 64);
  nsl = std::min<int64_t>(nsl, std::min<int64_t>(tpc, 1024));
  int64_t tps = (tpc + nsl - 1) / nsl;
  nsl = (tpc + tps - 1) / tps;
  if (tps > 64) return false;
  p->nslices = (int)nsl;
  p->tps = (int)tps;
  p->grid = (int)(p->ncb * nsl);
  int lt = 0;
  while ((1 << lt) < TW) ++lt;
  int ls = 0;
  while ((1ll << ls) < nsl) ++ls;
  p->max_chain = TH + (int)tps + lt + 2 * ls + 1;
  // workspace: level-1 tickets [ncb][groups of 32 slices] + level-2 tickets [ncb],
  // slice partials [nslices][C][9], group partials [groups][C][9]
  const int64_t ngrp = (nsl + 31) / 32;
  const size_t tick = ((size_t)(p->ncb * ngrp + p->ncb) * 4 + 15) / 16 * 16;
  p->ws_bytes = tick + (size_t)(nsl + ngrp) * g.C * 9 * 4;
  return p->max_chain <= 160;
}

cudaError_t launch_nhwc_tma_bf(const Geom& g, const NhwcTmaPlan& p, const void* x, const void* dy, float* dw,
                               void* ws, cudaStream_t st) {
  using namespace nhwct;
  const int64_t eb = (g.dtype == DWCONV_F32) ? 4 : 2;
  EncodeFn enc = encode_fn();
  if (!enc) return cudaErrorNotSupported;
  const CUtensorMapDataType dt = g.dtype == DWCONV_F32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
  CUtensorMap tmx, tmd;
  const cuuint32_t es[4] = {1, 1, 1, 1};
  {
    const cuuint64_t dims[4] = {(cuuint64_t)g.C, (cuuint64_t)g.W, (cuuint64_t)g.H, (cuuint64_t)g.N};
    const cuuint64_t str[3] = {(cuuint64_t)(g.C * eb), (cuuint64_t)(g.C * g.W * eb), (cuuint64_t)(g.C * g.W * g.H * eb)};
    const cuuint32_t box[4] = {(cuuint32_t)p.CB, (cuuint32_t)p.BW, (cuuint32_t)p.BH, 1};
    if (enc(&tmx, dt, 4, const_cast<void*>(x), dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) !=
        CUDA_SUCCESS)
      return cudaErrorInvalidValue;
  }
  {
    const cuuint64_t dims[4] = {(cuuint64_t)g.C, (cuuint64_t)g.Wo, (cuuint64_t)g.Ho, (cuuint64_t)g.N};
    const cuuint64_t str[3] = {(cuuint64_t)(g.C * eb), (cuuint64_t)(g.C * g.Wo * eb),
                               (cuuint64_t)(g.C * g.Wo * g.Ho * eb)};
    const cuuint32_t box[4] = {(cuuint32_t)p.CB, (cuuint32_t)p.TW, (cuuint32_t)p.TH, 1};
    if (enc(&tmd, dt, 4, const_cast<void*>(dy), dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) !=
        CUDA_SUCCESS)
      return cudaErrorInvalidValue;
  }
  BArgs a{};
  a.dw = dw;
  const int64_t ngrp = (p.nslices + 31) / 32;
  const size_t tick = ((size_t)(p.ncb * ngrp + p.ncb) * 4 + 15) / 16 * 16;
  a.ws_ticket = static_cast<unsigned*>(ws);
  a.ws_part = reinterpret_cast<float*>(static_cast<char*>(ws) + tick);
  a.N = (int)g.N; a.C = (int)g.C; a.CB = p.CB; a.NCV = p.NCV; a.TW = p.TW;
  a.tiles_h = p.tiles_h; a.tiles_w = p.tiles_w; a.ncb = p.ncb; a.nslices = p.nslices; a.tps = p.tps;
  a.tiles_per_cb = p.tiles_per_cb;
  a.BW = p.BW; a.DBW = p.TW;
  a.x_bytes = p.box_bytes; a.dy_bytes = p.dy_bytes; a.dy_off = p.dy_off; a.stage_bytes = p.stage_bytes;
  a.ns = p.ns; a.cons = p.cons;
  static const int early = env_int("DWCONV_EARLY_PDL", 1, 0, 1);
  a.early_pdl = early;
  BKernelFn fn = bf_kernel_for(g.dtype, (int)g.sh, p.TH);
  static const bool pdl = env_int("DWCONV_PDL", 1, 0, 1) == 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)p.grid);
  cfg.blockDim = dim3((unsigned)p.threads);
  cfg.dynamicSmemBytes = (size_t)p.smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, fn, tmx, tmd, a);
}

}  // namespace dwk
