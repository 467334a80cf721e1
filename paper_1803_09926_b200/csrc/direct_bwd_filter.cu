// direct_bwd_filter.cu -- dwconv_bwd_filter for NCHW, K = 3, straight from HBM
// into registers (no shared-memory staging).
//
// dw[o, i, jj] = sum_n sum_{oh,ow} x[n, c, oh*S-1+i, ow*S-1+jj] * dy[n, o, oh, ow],
// c = o / m -- the block diagonal that Eq. 4 keeps, summed
// over the batch (reading R5).
//
// Layout of the work: a "row set" is L = Wo / V consecutive lanes of a warp, lane
// li owning output columns [li*V, li*V + V); a warp holds 32 / L row sets.  A
// task is (image n, strip of R dy rows) of one output channel: the set loads the
// R dy rows and the (R-1)*S + 3 x rows it needs with coalesced vector loads
// (all of them issued before any arithmetic, so one warp keeps ~R*(1+S)*V*eb*32
// bytes in flight), fetches the one-column left halo from the neighbour lane
// with a shuffle (and, at stride 1, the right halo), and accumulates the K*K
// taps in registers (packed FFMA2 at stride 1).  CTA = (group of P output
// channels, batch slice); each channel owns `spc` row sets that stride over its
// tasks.  The x rows shared by adjacent strips are re-read from L2, not HBM.
//
// Deterministic reduction, fixed order everywhere:
//   per task (R*V/2 + 1 deep) -> running sum over the set's tasks
//   -> lanes of a set (sequential, L) -> sets of a channel (sequential, spc)
//   -> per-slice partial in the workspace; the last CTA of the group (integer
//      ticket) sums the slices pairwise in slice order and re-zeroes the
//      workspace (same protocol as nchw_bwd_filter.cu).
#include "nchw_common.cuh"

namespace dwk {
namespace direct {

using nchw::VecIO;

template <class T, int S, int V, int R>
__global__ void __launch_bounds__(256) dbf_kernel(const DArgs a) {
  constexpr int K = 3, KK = 9;
  constexpr int NRows = (R - 1) * S + K;  // x rows of a strip
  constexpr int NX = S * V;               // x columns a lane loads
  constexpr bool kPacked = (S == 1 && V % 2 == 0);
  __shared__ float red[256 * KK];
  __shared__ unsigned s_last;
  const T* __restrict__ x = static_cast<const T*>(a.x);
  const T* __restrict__ dy = static_cast<const T*>(a.dy);
  const int H = a.H, W = a.W, Ho = a.Ho, Wo = a.Wo;

  const int g = blockIdx.x % a.groups;
  const int sl = blockIdx.x / a.groups;
  const int64_t n0 = (int64_t)sl * a.nps;
  const int nimg = (int)(min((int64_t)a.N, n0 + a.nps) - n0);
  const int ntask = nimg * a.nsb;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int siw = lane / a.L;             // row set within the warp
  const int li = lane - siw * a.L;        // lane within the set
  const int gset = warp * a.SPW + siw;    // row set within the CTA
  const int ch = gset / a.spc;            // channel of this set within the group
  const int sidx = gset - ch * a.spc;     // set index within the channel
  const int o = g * a.P + ch;
  const bool live = siw < a.SPW && ch < a.P && o < a.Co;
  const int cin = live ? o / a.m : 0;
  const int c0 = li * V;                  // first output column of the lane
  const bool first = (li == 0), last = (li == a.L - 1);

  griddep_wait();
  float run[KK];
#pragma unroll
  for (int q = 0; q < KK; ++q) run[q] = 0.f;
  const int kmax = (ntask + a.spc - 1) / a.spc;  // warp-uniform trip count (shuffles stay converged)
  // L2 prefetch of a task's x rows and dy rows (one bulk prefetch each, issued by
  // the set's first lane): the register loads of that task then hit L2, so the
  // memory-level parallelism is not bounded by the registers holding them.
  auto prefetch = [&](int kp) {
    const int t = sidx + kp * a.spc;
    if (!(live && first && a.pf && t < ntask)) return;
    const int nn = t / a.nsb, sb = t - nn * a.nsb;
    const int64_t n = n0 + nn;
    const int r0 = sb * R, r1 = min(r0 + R, Ho);
    const int x0 = max(0, r0 * S - 1), x1 = min(H, (r1 - 1) * S + 2);
    const char* px = reinterpret_cast<const char*>(x + ((n * a.C + cin) * H + x0) * (int64_t)W);
    const char* pd = reinterpret_cast<const char*>(dy + ((n * a.Co + o) * Ho + r0) * (int64_t)Wo);
    bulk_prefetch_l2(px, (uint32_t)((x1 - x0) * W * sizeof(T)));
    bulk_prefetch_l2(pd, (uint32_t)((r1 - r0) * Wo * sizeof(T)));
  };
  prefetch(0);
  prefetch(1);
  for (int k = 0; k < kmax; ++k) {
    prefetch(k + 2);
    const int t = sidx + k * a.spc;
    const bool tv = live && t < ntask;
    const int nn = tv ? t / a.nsb : 0;
    const int sb = tv ? t - nn * a.nsb : 0;
    const int64_t n = n0 + nn;
    const int oh0 = sb * R;
    const T* dyp = dy + (((n * a.Co + o) * Ho) + oh0) * (int64_t)Wo + c0;
    const T* xp = x + (((n * a.C + cin) * H) + (int64_t)oh0 * S - 1) * (int64_t)W + (int64_t)S * c0;
    float dv[R][V];
    float xv[NRows][NX];
#pragma unroll
    for (int tt = 0; tt < R; ++tt) {
      if (tv && oh0 + tt < Ho) VecIO<T, V>::load(dyp + (int64_t)tt * Wo, dv[tt]);
      else
#pragma unroll
        for (int u = 0; u < V; ++u) dv[tt][u] = 0.f;
    }
#pragma unroll
    for (int rr = 0; rr < NRows; ++rr) {
      const int ih = oh0 * S - 1 + rr;
      if (tv && (unsigned)ih < (unsigned)H) VecIO<T, NX>::load(xp + (int64_t)rr * W, xv[rr]);
      else
#pragma unroll
        for (int u = 0; u < NX; ++u) xv[rr][u] = 0.f;
    }
    float2 loc2[kPacked ? KK : 1];
    float loc[kPacked ? 1 : KK];
#pragma unroll
    for (int q = 0; q < (kPacked ? KK : 1); ++q) loc2[q] = make_float2(0.f, 0.f);
#pragma unroll
    for (int q = 0; q < (kPacked ? 1 : KK); ++q) loc[q] = 0.f;
#pragma unroll
    for (int rr = 0; rr < NRows; ++rr) {
      // window of the row: x[S*c0 - 1 .. S*c0 + NX] (left halo, own NX, right halo at S = 1)
      float xw[NX + 2];
      const float lft = __shfl_up_sync(0xffffffffu, xv[rr][NX - 1], 1);
      const float rgt = __shfl_down_sync(0xffffffffu, xv[rr][0], 1);
      xw[0] = first ? 0.f : lft;
#pragma unroll
      for (int u = 0; u < NX; ++u) xw[1 + u] = xv[rr][u];
      xw[NX + 1] = (last || S * c0 + NX >= W) ? 0.f : rgt;
#pragma unroll
      for (int tt = 0; tt < R; ++tt) {
        const int i = rr - tt * S;
        if (i >= 0 && i < K) {
#pragma unroll
          for (int jj = 0; jj < K; ++jj) {
            if constexpr (kPacked) {
#pragma unroll
              for (int u = 0; u < V; u += 2)
                loc2[i * K + jj] = __ffma2_rn(make_float2(xw[u + jj], xw[u + 1 + jj]),
                                              make_float2(dv[tt][u], dv[tt][u + 1]), loc2[i * K + jj]);
            } else {
#pragma unroll
              for (int u = 0; u < V; ++u) loc[i * K + jj] = fmaf(xw[S * u + jj], dv[tt][u], loc[i * K + jj]);
            }
          }
        }
      }
    }
#pragma unroll
    for (int q = 0; q < KK; ++q) run[q] += kPacked ? (loc2[q].x + loc2[q].y) : loc[q];
  }
  griddep_launch_dependents();

  // ---- reduce: lanes of a set (sequential), then sets of a channel (sequential)
#pragma unroll
  for (int q = 0; q < KK; ++q) red[threadIdx.x * KK + q] = run[q];
  __syncthreads();
  float* part = a.ws_part + ((int64_t)sl * a.Co + (int64_t)g * a.P) * KK;
  const int nch = min(a.P, a.Co - g * a.P);
  for (int pq = threadIdx.x; pq < nch * KK; pq += blockDim.x) {
    const int c = pq / KK, q = pq - c * KK;
    float tot = 0.f;
    for (int s = 0; s < a.spc; ++s) {
      const int gs = c * a.spc + s;
      const int w = gs / a.SPW, si = gs - w * a.SPW;
      const float* src = red + (w * 32 + si * a.L) * KK + q;
      float v = src[0];
      for (int l = 1; l < a.L; ++l) v += src[l * KK];
      tot = (s == 0) ? v : tot + v;
    }
    part[pq] = tot;
  }
  __threadfence();
  __syncthreads();
  {  // two-level slice finalize (nchw_common.cuh)
    const int ngrp = (a.nslices + 31) / 32;
    nchw::finalize_two_level(a.ws_part, a.ws_part + (int64_t)a.nslices * a.Co * KK, a.ws_ticket,
                             a.ws_ticket + (int64_t)a.groups * ngrp, g, sl, a.nslices, (int64_t)a.Co * KK,
                             (int64_t)g * a.P * KK, nch * KK, a.dw, &s_last);
  }
}

template <class T, int S, int R>
DKernelFn pick_v(int V) {
  switch (V) {
    case 1: return dbf_kernel<T, S, 1, R>;
    case 2: return dbf_kernel<T, S, 2, R>;
    case 4: return dbf_kernel<T, S, 4, R>;
    case 8: return std::is_same<T, float>::value ? nullptr : dbf_kernel<T, S, 8, R>;
    default: return nullptr;
  }
}

template <class T>
DKernelFn pick_t(int S, int R, int V) {
  if (S == 1) return R == 7 ? pick_v<T, 1, 7>(V) : pick_v<T, 1, 8>(V);
  if (S == 2) return R == 7 ? pick_v<T, 2, 7>(V) : pick_v<T, 2, 8>(V);
  return nullptr;
}

DKernelFn bwd_filter_kernel(int dtype, int S, int R, int V) {
  return dtype == DWCONV_F32 ? pick_t<float>(S, R, V) : pick_t<__nv_bfloat16>(S, R, V);
}

}  // namespace direct
}  // namespace dwk
