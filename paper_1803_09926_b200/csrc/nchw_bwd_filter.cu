// nchw_bwd_filter.cu -- dwconv_bwd_filter for NCHW on sm_100a (see nchw_common.cuh).
//
// dw[c*m+j, i, jj] = sum_n sum_{oh,ow} x[n, c, oh*S-PAD+i, ow*S-PAD+jj] * dy[n, c*m+j, oh, ow]
// -- the block diagonal that Eq. 4 keeps, summed over the
// batch (reading R5).  CTA = (channel group of P channels, batch slice); groups
// of `tpg` consecutive threads own one dy plane.  Deterministic reduction:
//   thread strip (R rows x V cols, fp32 / packed fp32x2 FMA)   chain <= 64
//   -> running sum over the CTA's chunks                        chain <= 32
//   -> fixed-order sum over the tpg threads of a plane            <= 32 or tpg/32 + 5
//   -> per-slice partial in the workspace; the last CTA of the group (integer
//      ticket) sums the slices pairwise in slice order and re-zeroes the
//      workspace.                                               depth 2*log2(slices)
// No float atomics; the worst-case chain is reported by dwconv_plan (max_chain).
#include "nchw_common.cuh"

namespace dwk {
namespace nchw {
namespace {

// FUSED (S = 1, m = 1): the fused backward.  The dy planes are
// staged with PAD halo rows, and every thread strip also computes the matching
// R x V strip of dx -- the forward stencil over the staged dy with the flipped
// kernel (reading R9) -- and stores it, so dy is read from HBM once for both
// gradients: 3|x| + 2|y| per layer instead of 3|x| + 3|y|.
template <class T, int K, int S, int R, int V, bool PADDED, bool FUSED = false>
__global__ void __launch_bounds__(kThreads + 32) nchw_bwd_filter_kernel(const NArgs a) {
  constexpr int PAD = (K - 1) / 2, KK = K * K;
  constexpr int NRows = (R - 1) * S + K;
  // bf16, V >= 4: interleaved pairs (lanes = columns u, u + V/2; nchw_common.cuh), FFMA2 at any stride
  constexpr bool kIl = std::is_same<T, __nv_bfloat16>::value && V >= 4 && kBf16Interleave;
  constexpr bool kPacked = kIl || (S == 1 && V % 2 == 0);  // float2 accumulators, FFMA2
  using Wd = Win<K, S, V>;
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem);
  unsigned* s_last = reinterpret_cast<unsigned*>(smem + 64);
  const T* __restrict__ x = static_cast<const T*>(a.in);
  const T* __restrict__ dy = static_cast<const T*>(a.in2);
  const int W = a.W, Wo = a.Wo, m = a.m, H = a.H, Ho = a.Ho;
  const T* zrow = reinterpret_cast<const T*>(smem + a.zrow_off);

  const int g = blockIdx.x % a.groups;
  const int sl = blockIdx.x / a.groups;
  const int c0ch = g * a.P;
  const int np = min(a.P, (int)(a.C - c0ch));
  const int64_t n0 = (int64_t)sl * a.nps;
  const int64_t n1 = min(a.N, n0 + a.nps);
  const int iters = (int)(n1 - n0) * a.nbands;

  // Warp-specialised: warp 0 is the producer (its lane 0 refills stage st once every
  // consumer warp has arrived on empty[st]); warps 1.. compute.  Consumers never wait
  // for each other inside the loop, and all ns stages stay in flight.
  uint64_t* empty = reinterpret_cast<uint64_t*>(smem + 72);  // <= 7 stages below the zero row at 128
  const int ncw = (int)(blockDim.x >> 5) - 1;  // consumer warps
  const int nct = 32 * ncw;
  const int ctid = (int)threadIdx.x - 32;     // consumer thread index (< 0: producer warp)
  if (threadIdx.x == 0)
    for (int i = 0; i < a.ns; ++i) mbar_init(&empty[i], ncw);
  prologue(smem, bars, a);
  auto sx_of = [&](int st) { return reinterpret_cast<T*>(smem + a.in0_off + 128 + st * a.in_stage); };
  auto sdy_of = [&](int st) { return reinterpret_cast<T*>(smem + a.in0_off + a.in2_off + st * a.in_stage); };

  struct Rows { int64_t n; int r0, r1, lo, hi, dlo, dhi; };  // dy rows [r0,r1) staged as [dlo,dhi); x rows [lo,hi)
  auto rows_of = [&](int kk) {
    Rows r;
    const int nn = kk / a.nbands;
    const int b = kk - nn * a.nbands;
    r.n = n0 + nn;
    if (a.nbands == 1) { r.r0 = 0; r.r1 = Ho; r.lo = 0; r.hi = H; }
    else {
      r.r0 = b * a.BR;
      r.r1 = min(r.r0 + a.BR, Ho);
      r.lo = max(0, r.r0 * S - PAD);
      r.hi = min(H, (r.r1 - 1) * S - PAD + K);
    }
    r.dlo = FUSED ? max(0, r.r0 - PAD) : r.r0;  // fused: dy halo rows for the dx stencil
    r.dhi = FUSED ? min(Ho, r.r1 + PAD) : r.r1;
    return r;
  };
  auto x_src = [&](const Rows& r) { return x + ((r.n * a.C + c0ch) * H + r.lo) * W; };
  auto dy_src = [&](const Rows& r) { return dy + (((r.n * a.C + c0ch) * m) * Ho + r.dlo) * Wo; };
  auto x_spec = [&](const Rows& r) {
    StageSpec sp;
    sp.cnt = (int64_t)(r.hi - r.lo) * W;
    sp.gstride = (int64_t)H * W;
    sp.npl = np;
    sp.pitch = PADDED ? a.pitch : (int)sp.cnt;
    sp.zbe = PADDED ? a.zbe : 0;
    return sp;
  };
  auto dy_spec = [&](const Rows& r) {  // dy needs no halo: planes back to back
    StageSpec sp;
    sp.cnt = (int64_t)(r.dhi - r.dlo) * Wo;
    sp.gstride = (int64_t)Ho * Wo;
    sp.npl = np * m;
    sp.pitch = (int)sp.cnt;
    sp.zbe = 0;
    return sp;
  };
  auto chunk_bulk = [&](const Rows& r) {
    return stage_bulk_ok<T>(x_src(r), x_spec(r)) && stage_bulk_ok<T>(dy_src(r), dy_spec(r));
  };
  auto issue = [&](int kk, int st) {
    const Rows r = rows_of(kk);
    if constexpr (PADDED) {
      if (a.nbands > 1 && r.hi == H) {  // zero rows under the last band of every plane (read unchecked)
        const StageSpec xs = x_spec(r);
        for (int pl = 0; pl < np; ++pl)
          zero_bytes16(sx_of(st) + pl * xs.pitch + xs.zbe + xs.cnt, (uint32_t)(PAD * W * sizeof(T) + 15) & ~15u, 0, 1);
      }
    }
    if (chunk_bulk(r)) {
      const StageSpec xs = x_spec(r), ds = dy_spec(r);
      mbar_arrive_expect_tx(&bars[st], stage_bytes<T>(xs) + stage_bytes<T>(ds));
      stage_copy<T>(sx_of(st), x_src(r), xs, &bars[st]);
      stage_copy<T>(sdy_of(st), dy_src(r), ds, &bars[st]);
    } else {
      mbar_arrive(&bars[st]);
    }
  };

  const int gp = ctid >= 0 ? ctid / a.tpg : 0;  // dy plane of this thread within the group
  const int lane_g = ctid - gp * a.tpg;
  const bool active = ctid >= 0 && gp < np * m;
  const int ncg = (int)a.div_ncg.d;
  float run[KK];
#pragma unroll
  for (int q = 0; q < KK; ++q) run[q] = 0.f;
  float wf[FUSED ? KK : 1];  // fused: this plane's kernel, flipped (dx = forward stencil of dy)
  if constexpr (FUSED) {
    const T* wt = static_cast<const T*>(a.w);
    const int o = c0ch * m + (active ? gp : 0);
#pragma unroll
    for (int q = 0; q < KK; ++q) wf[q] = Elem<T>::ldg(wt + (int64_t)o * KK + (KK - 1 - q));
  }

  if (ctid < 0) {
    // ------------------------------------------------------------ producer warp
    if (threadIdx.x == 0) {
      int st = 0;
      uint32_t par = 0;
      for (int kk = 0; kk < iters; ++kk) {
        if (kk >= a.ns) mbar_wait(&empty[st], par ^ 1);  // every consumer warp is done with the stage
        issue(kk, st);
        if (++st == a.ns) { st = 0; par ^= 1; }
      }
    }
  } else {
  // ------------------------------------------------------------ consumers
  int st = 0;
  uint32_t par = 0;
  for (int kk = 0; kk < iters; ++kk) {
    const Rows r = rows_of(kk);
    const int cur = st;
    T* sx = sx_of(st);
    T* sdy = sdy_of(st);
    mbar_wait(&bars[st], par);
    if (++st == a.ns) { st = 0; par ^= 1; }
    const StageSpec xs = x_spec(r);
    const bool bulk = chunk_bulk(r);
    const bool zbot = false;  // issue() zeroes the rows under the last band of every plane
    if (!bulk || zbot) {  // uniform over the consumers
      if (!bulk) {
        stage_coop_n<T>(sx, x_src(r), xs, ctid, nct);
        stage_coop_n<T>(sdy, dy_src(r), dy_spec(r), ctid, nct);
      }
      consumer_sync(nct);
    }
    if (active) {
      const int rows_x = r.hi - r.lo;
      const int rows_dy = r.dhi - r.dlo;
      const T* s_x = sx + (gp / m) * xs.pitch + xs.zbe - r.lo * W;  // row ih at s_x + ih * W
      const T* s_dy = sdy + gp * rows_dy * Wo - r.dlo * Wo;  // row oh at s_dy + oh * Wo
      float2 loc2[kPacked ? KK : 1];
      float loc[kPacked ? 1 : KK];
#pragma unroll
      for (int q = 0; q < (kPacked ? KK : 1); ++q) loc2[q] = make_float2(0.f, 0.f);
#pragma unroll
      for (int q = 0; q < (kPacked ? 1 : KK); ++q) loc[q] = 0.f;
      const int ntl = a.nsb * ncg;
      for (int t = lane_g; t < ntl; t += a.tpg) {
        const int sb = (int)fdiv((uint32_t)t, a.div_ncg);
        const int c0 = (t - sb * ncg) * V;
        const int oh0 = r.r0 + sb * R;
        const int b0 = S * c0;
        bool lok[Wd::NL > 0 ? Wd::NL : 1], rok[Wd::NR > 0 ? Wd::NR : 1];
#pragma unroll
        for (int l = 0; l < Wd::NL; ++l) lok[l] = b0 - Wd::NL + l >= 0;
#pragma unroll
        for (int q = 0; q < Wd::NR; ++q) rok[q] = b0 + Wd::NV + q < W;
        const int ih0 = oh0 * S - PAD;
        if constexpr (kIl) {
          // dy row tt is loaded at its first use (input row tt*S): at most K/S + 1 rows live
          float2 dv2[R][V / 2];
#pragma unroll
          for (int rr = 0; rr < NRows; ++rr) {
#pragma unroll
            for (int tt = 0; tt < R; ++tt) {
              if (rr == tt * S) {
                if (oh0 + tt < r.r1) {
                  load_vec_bf2<V>(reinterpret_cast<const __nv_bfloat16*>(s_dy + (oh0 + tt) * Wo + c0), dv2[tt]);
                } else {
#pragma unroll
                  for (int u = 0; u < V / 2; ++u) dv2[tt][u] = make_float2(0.f, 0.f);
                }
              }
            }
            const int ih = ih0 + rr;
            const bool rv = PADDED || (unsigned)(ih - r.lo) < (unsigned)rows_x;
            const T* p = (rv ? s_x + ih * W : zrow) + b0;
            float2 X2[Win2<K, S, V>::NP];
            load_window_bf2<K, S, V>(reinterpret_cast<const __nv_bfloat16*>(p), lok, rok, X2);
#pragma unroll
            for (int tt = 0; tt < R; ++tt) {
              const int i = rr - tt * S;
              if (i >= 0 && i < K) {
#pragma unroll
                for (int jj = 0; jj < K; ++jj)
#pragma unroll
                  for (int u = 0; u < V / 2; ++u)
                    loc2[i * K + jj] = __ffma2_rn(X2[S * u + jj], dv2[tt][u], loc2[i * K + jj]);
              }
            }
          }
        } else {
        // dy row tt is loaded at its first use (input row tt*S): at most K/S + 1 rows live
        float dv[R][V];
#pragma unroll
        for (int rr = 0; rr < NRows; ++rr) {
#pragma unroll
          for (int tt = 0; tt < R; ++tt) {
            if (rr == tt * S) {
              if (oh0 + tt < r.r1) {
                VecIO<T, V>::load(s_dy + (oh0 + tt) * Wo + c0, dv[tt]);
              } else {
#pragma unroll
                for (int u = 0; u < V; ++u) dv[tt][u] = 0.f;
              }
            }
          }
          const int ih = ih0 + rr;
          const bool rv = PADDED || (unsigned)(ih - r.lo) < (unsigned)rows_x;
          const T* p = (rv ? s_x + ih * W : zrow) + b0;
          float xw[Wd::N];
          load_window<T, K, S, V>(p, lok, rok, xw);
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
        }
        if constexpr (FUSED) {  // dx strip at the same rows / columns (S = 1: H = Ho, W = Wo)
          float acc[R][V];
#pragma unroll
          for (int tt = 0; tt < R; ++tt)
#pragma unroll
            for (int u = 0; u < V; ++u) acc[tt][u] = 0.f;
          stencil_strip<T, K, 1, R, V, false>(s_dy, zrow, Wo, r.dlo, rows_dy, oh0 - PAD, c0, wf, acc);
          T* xo = static_cast<T*>(a.out) + ((r.n * a.C + c0ch + gp) * (int64_t)H + oh0) * W + c0;
#pragma unroll
          for (int tt = 0; tt < R; ++tt)
            if (oh0 + tt < r.r1) VecIO<T, V>::store(xo + (int64_t)tt * W, acc[tt]);
        }
      }
#pragma unroll
      for (int q = 0; q < KK; ++q) run[q] += kPacked ? (loc2[q].x + loc2[q].y) : loc[q];
    }
    __syncwarp();
    if ((threadIdx.x & 31) == 0) mbar_arrive(&empty[cur]);  // this warp is done with the stage
  }
  }
  __syncthreads();  // all warps are done with the stages before the sums are parked in them

  griddep_launch_dependents();
  // ---- reduce over the tpg threads of each dy plane: every thread parks its sums
  // in shared memory (the input stages are all consumed), then one warp per
  // (plane, tap) adds the tpg values -- a strided fixed-order sum per lane and a
  // fixed shuffle tree across lanes.
  float* red = reinterpret_cast<float*>(smem + a.in0_off);
  if (ctid >= 0)
#pragma unroll
    for (int q = 0; q < KK; ++q) red[ctid * KK + q] = run[q];
  __syncthreads();
  const int Co = a.Co;
  float* part = a.ws_part + ((int64_t)sl * Co + (int64_t)c0ch * m) * KK;
  const int nplanes = np * m;
  if (a.tpg <= 32) {  // one thread per (plane, tap): fixed-order sum of tpg values
    for (int pq = threadIdx.x; pq < nplanes * KK; pq += (int)blockDim.x) {
      const int p = pq / KK, q = pq - p * KK;
      const float* src = red + (p * a.tpg) * KK + q;
      float v = src[0];
      for (int u = 1; u < a.tpg; ++u) v += src[u * KK];
      part[pq] = v;
    }
  } else {  // one warp per (plane, tap): strided fixed-order lane sums + shuffle tree
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = (int)(blockDim.x >> 5);
    for (int pq = warp; pq < nplanes * KK; pq += nwarps) {
      const int p = pq / KK, q = pq - p * KK;
      float v = 0.f;
      for (int u = lane; u < a.tpg; u += 32) v += red[(p * a.tpg + u) * KK + q];
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
      if (lane == 0) part[pq] = v;
    }
  }
  __threadfence();
  __syncthreads();
  {  // two-level slice finalize (nchw_common.cuh): groups of 32 slices, then groups
    const int ngrp = (a.nslices + 31) / 32;
    finalize_two_level(a.ws_part, a.ws_part + (int64_t)a.nslices * Co * KK, a.ws_ticket,
                       a.ws_ticket + (int64_t)a.groups * ngrp, g, sl, a.nslices, (int64_t)Co * KK,
                       (int64_t)c0ch * m * KK, np * m * KK, a.dw, s_last);
  }
}

// V = 8 (one 16-B row load per window) exists for bf16 3x3 only.
template <class T, int K, int S, int R, bool PD>
KernelFn v8_kernel() {
  if constexpr (std::is_same<T, __nv_bfloat16>::value && K == 3 && PD) return nchw_bwd_filter_kernel<T, K, S, R, 8, PD>;
  else return nullptr;
}

template <class T, int K, int S, bool PD>
KernelFn pick_rv(int RI, int VI) {
  constexpr int R0 = rows_bf(K, 0), R1 = rows_bf(K, 1);
#define DW_V(R)                                                     \
  switch (VI) {                                                     \
    case 0: return nchw_bwd_filter_kernel<T, K, S, R, 1, PD>;       \
    case 1: return nchw_bwd_filter_kernel<T, K, S, R, 2, PD>;       \
    case 2: return PD ? nchw_bwd_filter_kernel<T, K, S, R, 4, PD> : nullptr; \
    case 3: return v8_kernel<T, K, S, R, PD>();                 \
    default: return nullptr;                                        \
  }
  if (RI == 0) { DW_V(R0) } else { DW_V(R1) }
#undef DW_V
}

template <class T, bool PD>
KernelFn pick_t(int K, int S, int RI, int VI) {
  if (K == 3 && S == 1) return pick_rv<T, 3, 1, PD>(RI, VI);
  if (K == 3 && S == 2) return pick_rv<T, 3, 2, PD>(RI, VI);
  if (K == 5 && S == 1) return pick_rv<T, 5, 1, PD>(RI, VI);
  if (K == 5 && S == 2) return pick_rv<T, 5, 2, PD>(RI, VI);
  if (K == 7 && S == 1) return pick_rv<T, 7, 1, PD>(RI, VI);
  if (K == 7 && S == 2) return pick_rv<T, 7, 2, PD>(RI, VI);
  return nullptr;
}

}  // namespace

// Fused backward (3x3, S = 1, m = 1): V in {1, 2, 4}.
template <class T, bool PD>
KernelFn pick_fused(int RI, int VI) {
  constexpr int R0 = rows_bf(3, 0), R1 = rows_bf(3, 1);
  switch (VI) {
    case 0: return RI == 0 ? nchw_bwd_filter_kernel<T, 3, 1, R0, 1, PD, true> : nchw_bwd_filter_kernel<T, 3, 1, R1, 1, PD, true>;
    case 1: return RI == 0 ? nchw_bwd_filter_kernel<T, 3, 1, R0, 2, PD, true> : nchw_bwd_filter_kernel<T, 3, 1, R1, 2, PD, true>;
    case 2:
      if constexpr (PD)
        return RI == 0 ? nchw_bwd_filter_kernel<T, 3, 1, R0, 4, PD, true> : nchw_bwd_filter_kernel<T, 3, 1, R1, 4, PD, true>;
      else
        return nullptr;
    case 3:
      if constexpr (PD && std::is_same<T, __nv_bfloat16>::value)
        return RI == 0 ? nchw_bwd_filter_kernel<T, 3, 1, R0, 8, PD, true> : nchw_bwd_filter_kernel<T, 3, 1, R1, 8, PD, true>;
      else
        return nullptr;
    default: return nullptr;
  }
}

KernelFn bwd_fused_kernel(int dtype, int K, int S, int RI, int VI, bool padded) {
  if (K != 3 || S != 1) return nullptr;
  if (dtype == DWCONV_F32) return padded ? pick_fused<float, true>(RI, VI) : pick_fused<float, false>(RI, VI);
  return padded ? pick_fused<__nv_bfloat16, true>(RI, VI) : pick_fused<__nv_bfloat16, false>(RI, VI);
}

KernelFn bwd_filter_kernel(int dtype, int K, int S, int RI, int VI, bool padded) {
  if (dtype == DWCONV_F32) return padded ? pick_t<float, true>(K, S, RI, VI) : pick_t<float, false>(K, S, RI, VI);
  return padded ? pick_t<__nv_bfloat16, true>(K, S, RI, VI) : pick_t<__nv_bfloat16, false>(K, S, RI, VI);
}

}  // namespace nchw
}  // namespace dwk
