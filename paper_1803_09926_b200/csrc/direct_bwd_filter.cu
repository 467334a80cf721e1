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

// ---------------------------------------------------------------- streaming bf16
// bf16 variant for large planes: a task is (image, band of BR dy rows); the set
// walks the band's x rows top to bottom, each x row loaded once (one 16-B vector
// per lane, halo columns from the neighbour lanes by shuffles) and widened once
// into interleaved pairs (lanes = output columns u, u + V/2; nchw_common.cuh), and
// every dy row is widened once at its first use and kept while the next K x rows
// need it (K/S + 1 dy rows live).  Raw words of the next row are loaded one row
// ahead; the whole next-but-one task is prefetched into L2 by bulk copies.
// Per-task chains are BR*V/2 + 1 deep; reduction as dbf_kernel.
template <int S, int V, int BR>
__global__ void __launch_bounds__(256, 2) sdbf_kernel(const DArgs a) {
  using B = __nv_bfloat16;
  constexpr int K = 3, KK = 9;
  constexpr int NRows = (BR - 1) * S + K;  // x rows of a band
  constexpr int NX = S * V;                // own x columns
  constexpr int NWX = NX / 2, NWD = V / 2;  // 32-bit words per x / dy row
  constexpr int H2 = S * V / 2;            // pair lane distance in the x window
  constexpr int NP = S * (V / 2 - 1) + K;  // operand pairs per x row
  static_assert(V >= 4 && V % 2 == 0, "interleaved pairs need V >= 4");
  __shared__ float red[256 * KK];
  __shared__ unsigned s_last;
  const B* __restrict__ x = static_cast<const B*>(a.x);
  const B* __restrict__ dy = static_cast<const B*>(a.dy);
  const int H = a.H, W = a.W, Ho = a.Ho, Wo = a.Wo;

  const int g = blockIdx.x % a.groups;
  const int sl = blockIdx.x / a.groups;
  // slice sl = tasks [t0, t0 + ntask) of the channel's N * nsb (image, band) list (a.nps = tasks per slice)
  const int64_t t0 = (int64_t)sl * a.nps;
  const int ntask = (int)(min((int64_t)a.N * a.nsb, t0 + a.nps) - t0);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int siw = lane / a.L;
  const int li = lane - siw * a.L;
  const int gset = warp * a.SPW + siw;
  const int ch = gset / a.spc;
  const int sidx = gset - ch * a.spc;
  const int o = g * a.P + ch;
  const bool live = siw < a.SPW && ch < a.P && o < a.Co;
  const int cin = live ? o / a.m : 0;
  const int c0 = li * V;
  const bool first = (li == 0), last = (li == a.L - 1);

  griddep_wait();
  float run[KK];
#pragma unroll
  for (int q = 0; q < KK; ++q) run[q] = 0.f;
  const int kmax = (ntask + a.spc - 1) / a.spc;  // warp-uniform trip count (shuffles stay converged)
  auto prefetch = [&](int kp) {
    const int t = sidx + kp * a.spc;
    if (!(live && first && a.pf && t < ntask)) return;
    const int64_t tg = t0 + t;
    const int64_t n = tg / a.nsb;
    const int sb = (int)(tg - n * a.nsb);
    const int r0 = sb * BR, r1 = min(r0 + BR, Ho);
    const int x0 = max(0, r0 * S - 1), x1 = min(H, (r1 - 1) * S + 2);
    bulk_prefetch_l2(x + ((n * a.C + cin) * H + x0) * (int64_t)W, (uint32_t)((x1 - x0) * W * sizeof(B)));
    bulk_prefetch_l2(dy + ((n * a.Co + o) * Ho + r0) * (int64_t)Wo, (uint32_t)((r1 - r0) * Wo * sizeof(B)));
  };
  prefetch(0);
  prefetch(1);
  for (int k = 0; k < kmax; ++k) {
    prefetch(k + 2);
    const int t = sidx + k * a.spc;
    const bool tv = live && t < ntask;
    const int64_t tg = tv ? t0 + t : 0;
    const int64_t n = tg / a.nsb;
    const int sb = (int)(tg - n * a.nsb);
    const int oh0 = sb * BR;
    const int ih0 = oh0 * S - 1;
    const B* dyp = dy + (((n * a.Co + o) * Ho) + oh0) * (int64_t)Wo + c0;
    const B* xp = x + ((n * a.C + cin) * H) * (int64_t)W + (int64_t)S * c0;
    auto ldx = [&](int rr, uint32_t* w) {
      const int ih = ih0 + rr;
      if (tv && (unsigned)ih < (unsigned)H) {
        nchw::load_words<NWX>(xp + (int64_t)ih * W, w);
      } else {
#pragma unroll
        for (int q = 0; q < NWX; ++q) w[q] = 0u;
      }
    };
    auto ldd = [&](int tt, uint32_t* w) {
      if (tv && oh0 + tt < Ho) {
        nchw::load_words<NWD>(dyp + (int64_t)tt * Wo, w);
      } else {
#pragma unroll
        for (int q = 0; q < NWD; ++q) w[q] = 0u;
      }
    };
    float2 loc2[KK];
#pragma unroll
    for (int q = 0; q < KK; ++q) loc2[q] = make_float2(0.f, 0.f);
    uint32_t xw_cur[NWX], xw_nxt[NWX];
    uint32_t dw_raw[BR][NWD];
    float2 dv2[BR][V / 2];
    ldx(0, xw_cur);
    ldd(0, dw_raw[0]);
#pragma unroll
    for (int rr = 0; rr < NRows; ++rr) {
      // issue the loads of the next x row and of the dy row first used there
      if (rr + 1 < NRows) ldx(rr + 1, xw_nxt);
#pragma unroll
      for (int tt = 1; tt < BR; ++tt)
        if (rr + 1 == tt * S) ldd(tt, dw_raw[tt]);
      // widen the dy row first used at this x row
#pragma unroll
      for (int tt = 0; tt < BR; ++tt) {
        if (rr == tt * S) {
#pragma unroll
          for (int u = 0; u < V / 2; ++u) {
            const int qa = u, qb = u + V / 2;
            dv2[tt][u] = make_float2((qa & 1) ? nchw::bfw_hi(dw_raw[tt][qa >> 1]) : nchw::bfw_lo(dw_raw[tt][qa >> 1]),
                                     (qb & 1) ? nchw::bfw_hi(dw_raw[tt][qb >> 1]) : nchw::bfw_lo(dw_raw[tt][qb >> 1]));
          }
        }
      }
      // x window: left halo (neighbour's last element), own NX, right halo at S = 1
      const uint32_t lw = __shfl_up_sync(0xffffffffu, xw_cur[NWX - 1], 1);
      uint32_t rw = 0u;
      if constexpr (S == 1) rw = __shfl_down_sync(0xffffffffu, xw_cur[0], 1);
      const uint32_t lwv = first ? 0u : lw;
      const uint32_t rwv = last ? 0u : rw;
      auto val = [&](int kx) -> float {
        if (kx == 0) return nchw::bfw_hi(lwv);
        if (kx <= NX) {
          const int q = kx - 1;
          return (q & 1) ? nchw::bfw_hi(xw_cur[q >> 1]) : nchw::bfw_lo(xw_cur[q >> 1]);
        }
        return nchw::bfw_lo(rwv);
      };
      float2 X2[NP];
#pragma unroll
      for (int kx = 0; kx < NP; ++kx) X2[kx] = make_float2(val(kx), val(kx + H2));
#pragma unroll
      for (int tt = 0; tt < BR; ++tt) {
        const int i = rr - tt * S;
        if (i >= 0 && i < K) {
#pragma unroll
          for (int jj = 0; jj < K; ++jj)
#pragma unroll
            for (int u = 0; u < V / 2; ++u) loc2[i * K + jj] = __ffma2_rn(X2[S * u + jj], dv2[tt][u], loc2[i * K + jj]);
        }
      }
#pragma unroll
      for (int q = 0; q < NWX; ++q) xw_cur[q] = xw_nxt[q];
    }
#pragma unroll
    for (int q = 0; q < KK; ++q) run[q] += loc2[q].x + loc2[q].y;
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
  {
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

// Streaming bf16 variant: BR dy rows per task (8 or 16), V in {4, 8}.
DKernelFn bwd_filter_stream_kernel(int dtype, int S, int BR, int V) {
  if (dtype != DWCONV_BF16) return nullptr;
#define DW_SB(S_, BR_) \
  return V == 4 ? sdbf_kernel<S_, 4, BR_> : (V == 8 ? sdbf_kernel<S_, 8, BR_> : nullptr)
  if (S == 1 && BR == 8) DW_SB(1, 8);
  if (S == 1 && BR == 16) DW_SB(1, 16);
  if (S == 2 && BR == 8) DW_SB(2, 8);
  return nullptr;
#undef DW_SB
}

}  // namespace direct
}  // namespace dwk
