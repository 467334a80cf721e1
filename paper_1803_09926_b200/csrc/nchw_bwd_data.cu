// nchw_bwd_data.cu -- dwconv_bwd_data for NCHW on sm_100a (see nchw_common.cuh).
//
// dx[n,c,ih,iw] = sum_{j<m} sum_{i,jj} w[c*m+j,i,jj] * dy[n,c*m+j,(ih+PAD-i)/S,(iw+PAD-jj)/S]
// over exact divisions in range -- the adjoint of the forward pass (DESIGN.md
// reading R9; the paper delegates it to the framework).
//  * S = 1: the forward stencil on dy with the kernel flipped (weights are staged
//    flipped on read), strip = R dx rows x V dx columns, packed FFMA2.
//  * S = 2: polyphase tile of R dx rows x S dx columns aligned to the stride so
//    the tap -> dy mapping is static.
// Per-j partial sums keep each serial chain at K*K (R5 iii).  Same warp-
// specialised structure as nchw_fwd.cu: a producer warp stages dy planes (TMA
// ring) and the flipped weights; consumer warps store dx from registers.
#include "nchw_common.cuh"

namespace dwk {
namespace nchw {
namespace {

template <int K, int S>
__device__ __forceinline__ ChunkRows bd_rows(const NArgs& a, int64_t c) {
  constexpr int PAD = (K - 1) / 2;
  ChunkRows k;
  if (a.nbands == 1) {
    k.q0 = c * a.P;
    k.np = (int)min((int64_t)a.P, a.Q - k.q0);
    k.r0 = 0; k.r1 = a.H; k.lo = 0; k.hi = a.Ho;
  } else {
    k.q0 = (int64_t)fdiv((uint32_t)c, a.div_nb);
    const int b = (int)(c - k.q0 * a.nbands);
    k.np = 1;
    k.r0 = b * a.BR;
    k.r1 = min(k.r0 + a.BR, (int)a.H);
    // dy rows reaching dx rows [r0, r1): ceil((r0+PAD-K+1)/S) .. floor((r1-1+PAD)/S)
    k.lo = max(0, -floor_div(-(k.r0 + PAD - K + 1), S));
    k.hi = min(a.Ho, floor_div(k.r1 - 1 + PAD, S) + 1);
  }
  return k;
}

// PAIR (bf16, m = 1): tiles of two dx planes at once, FFMA2 lanes = planes --
// S = 1 through stencil_strip_pair (flipped kernels), S = 2 polyphase.
// M1: compiled for m = 1 (the per-j partial then is the output strip itself: one
// accumulator set instead of two -- 163 -> ~116 registers for bf16 3x3 s1 V = 8)
template <class T, int K, int S, int R, int V, bool PADDED, bool PAIR = false, bool M1 = false>
__global__ void __launch_bounds__(kThreads + 32) nchw_bwd_data_kernel(const NArgs a) {
  constexpr int PAD = (K - 1) / 2, KK = K * K;
  constexpr int D0 = floor_div(PAD - K + 1, S);
  constexpr int NRY = floor_div(R - 1 + PAD, S) - D0 + 1;
  constexpr int TW = (S == 1) ? V : S * V;  // dx columns per thread tile (stride aligned)
  constexpr int NCY = floor_div(TW - 1 + PAD, S) - D0 + 1;
  static_assert(R % S == 0, "dx strip must be stride aligned");
  // bf16 3x3 stride 2, m = 1: streaming polyphase strip (see below)
  constexpr bool kStream = std::is_same<T, __nv_bfloat16>::value && K == 3 && S == 2 && V >= 2 && kBf16Interleave;
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  uint64_t* empty = reinterpret_cast<uint64_t*>(smem + 64);
  const T* __restrict__ dy = static_cast<const T*>(a.in);
  T* __restrict__ dx = static_cast<T*>(a.out);
  const T* __restrict__ wt = static_cast<const T*>(a.w);
  const int W = a.W, Wo = a.Wo, m = M1 ? 1 : a.m, H = a.H;
  const T* zrow = reinterpret_cast<const T*>(smem + a.zrow_off);
  const int nct = (int)blockDim.x - 32;  // consumer threads

  prologue_ws(smem, a, nct >> 5, 2);  // full: TMA arrival + weights arrival
  auto sin_of = [&](int st) { return reinterpret_cast<T*>(smem + a.in0_off + 128 + st * a.in_stage); };
  auto sw_of = [&](int st) { return reinterpret_cast<float*>(smem + a.in0_off + a.in2_off + st * a.in_stage); };
  // input staging of a chunk: the m dy planes of each dx plane (rows [lo, hi))
  auto src_of = [&](const ChunkRows& k) { return dy + ((k.q0 * m) * a.Ho + k.lo) * Wo; };
  auto spec_of = [&](const ChunkRows& k) {
    StageSpec sp;
    sp.cnt = (int64_t)(k.hi - k.lo) * Wo;
    sp.gstride = (int64_t)a.Ho * Wo;
    sp.npl = k.np * m;
    sp.pitch = PADDED ? a.pitch : (int)sp.cnt;
    sp.zbe = PADDED ? a.zbe : 0;
    return sp;
  };

  if (threadIdx.x < 32) {
    // ------------------------------------------------------------ producer warp
    int s = 0;
    uint32_t ph = 0;
    int it = 0;
    for (int64_t c = blockIdx.x; c < a.nchunks; c += gridDim.x, ++it) {
      if (it >= a.ns) mbar_wait(&empty[s], ph ^ 1);  // consumers released the stage
      const ChunkRows k = bd_rows<K, S>(a, c);
      const WeightWin ww = weight_win<T, KK>(a, k.q0, k.np);
      if constexpr (PADDED) {
        if (a.nbands > 1 && k.hi == a.Ho) {  // zero rows under the last band's dy rows (read unchecked)
          const StageSpec sp = spec_of(k);
          for (int j = 0; j < m; ++j)
            zero_bytes16(sin_of(s) + j * sp.pitch + sp.zbe + sp.cnt, (uint32_t)(PAD * Wo * sizeof(T) + 15) & ~15u,
                         threadIdx.x, 32);
          __syncwarp();
        }
      }
      if (threadIdx.x == 0) {
        const StageSpec sp = spec_of(k);
        const bool xb = stage_bulk_ok<T>(src_of(k), sp);  // else consumers copy this chunk themselves
        const uint32_t tx = (xb ? stage_bytes<T>(sp) : 0u) + (ww.tma ? ww.bytes : 0u);
        if (tx) {
          mbar_arrive_expect_tx(&full[s], tx);
          if (xb) stage_copy<T>(sin_of(s), src_of(k), sp, &full[s]);
          if (ww.tma) bulk_g2s(sw_of(s), wt + ww.a0, ww.bytes, &full[s]);
        } else {
          mbar_arrive(&full[s]);
        }
      }
      if (!ww.tma) {  // fallback: the producer warp writes the weights as an fp32 table (flipped for S == 1)
        __syncwarp();
        const int cbase = (int)(k.q0 % a.C) * m;
        float* sw = sw_of(s);
        for (int idx = threadIdx.x; idx < k.np * m * KK; idx += 32) {
          const int pl = idx / KK, q = idx - pl * KK;
          const uint32_t ov = (uint32_t)(cbase + pl);
          const int o = (int)(ov - fdiv(ov, a.div_co) * (uint32_t)a.Co);
          sw[idx] = Elem<T>::ldg(wt + (int64_t)o * KK + ((S == 1) ? (KK - 1 - q) : q));
        }
        __syncwarp();
      }
      if (threadIdx.x == 0) mbar_arrive(&full[s]);  // second arrival: the weight table is written
      if (++s == a.ns) { s = 0; ph ^= 1; }
    }
    // every load of this CTA is issued: let the next kernel on the stream launch
    // and run its prologue on free SM resources (it still waits for this grid to
    // complete in griddepcontrol.wait before touching global memory)
    if (a.early_pdl) griddep_launch_dependents();
  } else {
    // ------------------------------------------------------------ consumers
    const int ctid = threadIdx.x - 32;
    const int ncg = (int)a.div_ncg.d;
    int s = 0;
    uint32_t ph = 0;
    for (int64_t c = blockIdx.x; c < a.nchunks; c += gridDim.x) {
      const ChunkRows k = bd_rows<K, S>(a, c);
      const StageSpec sp = spec_of(k);
      T* sin = sin_of(s);
      mbar_wait(&full[s], ph);
      const bool coop = !stage_bulk_ok<T>(src_of(k), sp);
      const bool zbot = false;  // the producer zeroes the rows under the last band's dy rows
      if (coop || zbot) {
        if (coop) stage_coop_n<T>(sin, src_of(k), sp, ctid, nct);
        if (zbot)
          for (int j = 0; j < m; ++j) zero_elems_n(sin + j * sp.pitch + sp.zbe + sp.cnt, PAD * Wo, ctid, nct);
        consumer_sync(nct);
      }
      const float* swc = sw_of(s);
      const WeightWin ww = weight_win<T, KK>(a, k.q0, k.np);
      const T* swr = reinterpret_cast<const T*>(swc) + ww.off;  // raw rows (ww.tma), flipped on read for S == 1
      const int rows_dy = k.hi - k.lo;
      if constexpr (PAIR) {  // m == 1: dy plane pp feeds dx plane pp
        const int npair = (k.np + 1) >> 1;
        const int ntp = npair * a.nsb * ncg;
        for (int t = ctid; t < ntp; t += nct) {
          const int t2 = (int)fdiv((uint32_t)t, a.div_ncg);
          const int cb = t - t2 * ncg;
          const int pp2 = (int)fdiv((uint32_t)t2, a.div_nsb);
          const int sb = t2 - pp2 * a.nsb;
          const int ppa = 2 * pp2;
          const bool hasb = ppa + 1 < k.np;
          const int ppb = hasb ? ppa + 1 : ppa;
          const int ih0 = k.r0 + sb * R;
          const int iw0 = cb * TW;
          float2 wp[KK];
          if (ww.tma) {
#pragma unroll
            for (int q = 0; q < KK; ++q) {
              const int qq = (S == 1) ? (KK - 1 - q) : q;
              wp[q] = make_float2(Elem<T>::load(swr + ppa * KK + qq), Elem<T>::load(swr + ppb * KK + qq));
            }
          } else {
#pragma unroll
            for (int q = 0; q < KK; ++q) wp[q] = make_float2(swc[ppa * KK + q], swc[ppb * KK + q]);
          }
          float2 acc[R][TW];
#pragma unroll
          for (int tt = 0; tt < R; ++tt)
#pragma unroll
            for (int u = 0; u < TW; ++u) acc[tt][u] = make_float2(0.f, 0.f);
          const T* base = sin + sp.zbe - k.lo * Wo;
          if constexpr (S == 1) {
            stencil_strip_pair<K, 1, R, V, PADDED>(base + ppa * sp.pitch, base + ppb * sp.pitch, zrow, Wo, k.lo,
                                                   rows_dy, ih0 - PAD, iw0, wp, acc);
          } else {  // polyphase, as in the scalar path below, with (plane A, plane B) lanes
            const int ohb = ih0 / S + D0;
            const int owb = iw0 / S + D0;
            bool cok[NCY];
#pragma unroll
            for (int cy = 0; cy < NCY; ++cy) cok[cy] = (unsigned)(owb + cy) < (unsigned)Wo;
            const T* spa = base + ppa * sp.pitch + owb;
            const T* spb = base + ppb * sp.pitch + owb;
#pragma unroll
            for (int ry = 0; ry < NRY; ++ry) {
              const int oh = ohb + ry;
              const bool rok = PADDED || (unsigned)(oh - k.lo) < (unsigned)rows_dy;
              const T* pa = rok ? spa + oh * Wo : zrow + owb;
              const T* pb = rok ? spb + oh * Wo : zrow + owb;
              float2 v[NCY];
#pragma unroll
              for (int cy = 0; cy < NCY; ++cy)
                v[cy] = cok[cy] ? make_float2(Elem<T>::load(pa + cy), Elem<T>::load(pb + cy)) : make_float2(0.f, 0.f);
#pragma unroll
              for (int tt = 0; tt < R; ++tt)
#pragma unroll
                for (int i = 0; i < K; ++i) {
                  const int th = tt + PAD - i;
                  if (pmod(th, S) == 0 && floor_div(th, S) - D0 == ry) {
#pragma unroll
                    for (int u = 0; u < TW; ++u)
#pragma unroll
                      for (int jj = 0; jj < K; ++jj) {
                        const int tw = u + PAD - jj;
                        if (pmod(tw, S) == 0) {
                          const int cy = floor_div(tw, S) - D0;
                          acc[tt][u] = __ffma2_rn(wp[i * K + jj], v[cy], acc[tt][u]);
                        }
                      }
                  }
                }
            }
          }
          T* xa = dx + (k.q0 + ppa) * (int64_t)H * W + iw0;
          T* xb = xa + (int64_t)H * W;
#pragma unroll
          for (int tt = 0; tt < R; ++tt) {
            if (ih0 + tt < k.r1) {
              float va[TW], vb[TW];
#pragma unroll
              for (int u = 0; u < TW; ++u) { va[u] = acc[tt][u].x; vb[u] = acc[tt][u].y; }
              if (S == 1 || W % TW == 0) {
                VecIO<T, TW>::store(xa + (int64_t)(ih0 + tt) * W, va);
                if (hasb) VecIO<T, TW>::store(xb + (int64_t)(ih0 + tt) * W, vb);
              } else {
#pragma unroll
                for (int u = 0; u < TW; ++u)
                  if (iw0 + u < W) {
                    Elem<T>::store(xa + (int64_t)(ih0 + tt) * W + u, va[u]);
                    if (hasb) Elem<T>::store(xb + (int64_t)(ih0 + tt) * W + u, vb[u]);
                  }
              }
            }
          }
        }
      }
      const int ntiles = PAIR ? 0 : k.np * a.nsb * ncg;
      for (int t = ctid; t < ntiles; t += nct) {
        const int t2 = (int)fdiv((uint32_t)t, a.div_ncg);
        const int cb = t - t2 * ncg;
        const int pp = (int)fdiv((uint32_t)t2, a.div_nsb);
        const int sb = t2 - pp * a.nsb;
        const int ih0 = k.r0 + sb * R;  // multiple of S
        const int iw0 = cb * TW;
        if constexpr (kStream) {
          if (m == 1) {
            // dx rows stream down the strip: even dx row ih0+2s takes dy row a0+s (tap row 1), odd
            // row ih0+2s+1 takes dy rows a0+s (tap row 2) and a0+s+1 (tap row 0); columns alike
            // (dx column iw0+2b: dy column c0+b, tap 1; iw0+2b+1: c0+b+1, tap 0 and c0+b, tap 2).
            // FFMA2 lanes = dx columns (u, u+V), so the operand pairs are P[k] = (dy[c0+k], dy[c0+k+V/2]),
            // widened once per dy row (nchw_common.cuh interleaved pairs); 2 dy rows live.
            float wr[KK];
            if (ww.tma) {
#pragma unroll
              for (int q = 0; q < KK; ++q) wr[q] = Elem<T>::load(swr + pp * KK + q);
            } else {
#pragma unroll
              for (int q = 0; q < KK; ++q) wr[q] = swc[pp * KK + q];
            }
            const int a0 = ih0 / 2, c0 = iw0 / 2;
            const T* splane = sin + pp * sp.pitch + sp.zbe - k.lo * Wo;  // dy row oh at splane + oh * Wo
            const bool hok = c0 + V < Wo;
            auto load_pairs = [&](int oh, float2* P) {
              const bool rok = PADDED || (unsigned)(oh - k.lo) < (unsigned)rows_dy;
              const __nv_bfloat16* p = reinterpret_cast<const __nv_bfloat16*>((rok ? splane + oh * Wo : zrow) + c0);
              uint32_t wv[V / 2];
              load_words<V / 2>(p, wv);
              const uint32_t h = hok ? (uint32_t)reinterpret_cast<const unsigned short*>(p)[V] : 0u;
              auto val = [&](int q) -> float { return q < V ? ((q & 1) ? bfw_hi(wv[q >> 1]) : bfw_lo(wv[q >> 1])) : bfw_lo(h); };
#pragma unroll
              for (int kk = 0; kk <= V / 2; ++kk) P[kk] = make_float2(val(kk), val(kk + V / 2));
            };
            auto put_row = [&](int ih, const float2* e) {
              if (ih >= k.r1) return;
              float v[TW];
#pragma unroll
              for (int u = 0; u < V; ++u) { v[u] = e[u].x; v[u + V] = e[u].y; }
              T* row = dx + (k.q0 + pp) * (int64_t)H * W + (int64_t)ih * W + iw0;
              if (W % TW == 0) {
                VecIO<T, TW>::store(row, v);
              } else {
#pragma unroll
                for (int u = 0; u < TW; ++u)
                  if (iw0 + u < W) Elem<T>::store(row + u, v[u]);
              }
            };
            auto f2 = [](float w) { return make_float2(w, w); };
            float2 Pc[V / 2 + 1], Pn[V / 2 + 1];
            load_pairs(a0, Pc);
#pragma unroll
            for (int s2 = 0; s2 < R / 2; ++s2) {
              float2 e[V];
#pragma unroll
              for (int b = 0; b < V / 2; ++b) {
                e[2 * b] = __fmul2_rn(f2(wr[4]), Pc[b]);
                e[2 * b + 1] = __ffma2_rn(f2(wr[5]), Pc[b], __fmul2_rn(f2(wr[3]), Pc[b + 1]));
              }
              put_row(ih0 + 2 * s2, e);
              load_pairs(a0 + s2 + 1, Pn);
#pragma unroll
              for (int b = 0; b < V / 2; ++b) {
                e[2 * b] = __ffma2_rn(f2(wr[7]), Pc[b], __fmul2_rn(f2(wr[1]), Pn[b]));
                float2 o = __fmul2_rn(f2(wr[0]), Pn[b + 1]);
                o = __ffma2_rn(f2(wr[2]), Pn[b], o);
                o = __ffma2_rn(f2(wr[6]), Pc[b + 1], o);
                e[2 * b + 1] = __ffma2_rn(f2(wr[8]), Pc[b], o);
              }
              put_row(ih0 + 2 * s2 + 1, e);
#pragma unroll
              for (int kk = 0; kk <= V / 2; ++kk) Pc[kk] = Pn[kk];
            }
            continue;
          }
        }
        if constexpr (M1 && S == 1 && std::is_same<T, __nv_bfloat16>::value && V >= 4 && kBf16Interleave) {
          // bf16, m = 1: the flipped forward stencil with rows stored as they complete (3 live rows)
          float wr[KK];
          if (ww.tma) {
#pragma unroll
            for (int q = 0; q < KK; ++q) wr[q] = Elem<T>::load(swr + pp * KK + (KK - 1 - q));
          } else {
#pragma unroll
            for (int q = 0; q < KK; ++q) wr[q] = swc[pp * KK + q];
          }
          T* xo = dx + (k.q0 + pp) * (int64_t)H * W + iw0;
          stencil_strip_bf2_stream<K, 1, R, V, PADDED>(
              reinterpret_cast<const __nv_bfloat16*>(sin + pp * sp.pitch + sp.zbe - k.lo * Wo),
              reinterpret_cast<const __nv_bfloat16*>(zrow), Wo, k.lo, rows_dy, ih0 - PAD, iw0, wr,
              [&](int tt, const float* v) {
                if (ih0 + tt < k.r1) VecIO<T, V>::store(xo + (int64_t)(ih0 + tt) * W, v);
              });
          continue;
        }
        if constexpr (!(kStream && V >= 8)) {
        float acc[R][TW];
#pragma unroll
        for (int tt = 0; tt < R; ++tt)
#pragma unroll
          for (int u = 0; u < TW; ++u) acc[tt][u] = 0.f;
        for (int j = 0; j < m; ++j) {
          float wr[KK];
          if (ww.tma) {
            const T* wp = swr + (pp * m + j) * KK;
#pragma unroll
            for (int q = 0; q < KK; ++q) wr[q] = Elem<T>::load(wp + ((S == 1) ? (KK - 1 - q) : q));
          } else {
            const float* wp = swc + (pp * m + j) * KK;
#pragma unroll
            for (int q = 0; q < KK; ++q) wr[q] = wp[q];
          }
          float part[R][TW];
#pragma unroll
          for (int tt = 0; tt < R; ++tt)
#pragma unroll
            for (int u = 0; u < TW; ++u) part[tt][u] = 0.f;
          const T* splane = sin + (pp * m + j) * sp.pitch + sp.zbe;
          if constexpr (S == 1) {
            // forward stencil with the flipped kernel: dx[ih][iw] = sum wf[a][b] dy[ih-PAD+a][iw-PAD+b]
            stencil_strip<T, K, 1, R, V, PADDED>(splane - k.lo * Wo, zrow, Wo, k.lo, rows_dy, ih0 - PAD, iw0, wr,
                                                 part);
          } else {
            const int ohb = ih0 / S + D0;
            const int owb = iw0 / S + D0;
            bool cok[NCY];
#pragma unroll
            for (int cy = 0; cy < NCY; ++cy) cok[cy] = (unsigned)(owb + cy) < (unsigned)Wo;
            const T* spl = splane - k.lo * Wo + owb;
            const T* zp = zrow + owb;
#pragma unroll
            for (int ry = 0; ry < NRY; ++ry) {
              const int oh = ohb + ry;
              const bool rok = PADDED || (unsigned)(oh - k.lo) < (unsigned)rows_dy;
              const T* p = rok ? spl + oh * Wo : zp;
              float v[NCY];
#pragma unroll
              for (int cy = 0; cy < NCY; ++cy) v[cy] = cok[cy] ? Elem<T>::load(p + cy) : 0.f;
#pragma unroll
              for (int tt = 0; tt < R; ++tt)
#pragma unroll
                for (int i = 0; i < K; ++i) {
                  const int th = tt + PAD - i;  // relative to ih0
                  if (pmod(th, S) == 0 && floor_div(th, S) - D0 == ry) {
#pragma unroll
                    for (int u = 0; u < TW; ++u)
#pragma unroll
                      for (int jj = 0; jj < K; ++jj) {
                        const int tw = u + PAD - jj;
                        if (pmod(tw, S) == 0) {
                          const int cy = floor_div(tw, S) - D0;
                          part[tt][u] = fmaf(wr[i * K + jj], v[cy], part[tt][u]);
                        }
                      }
                  }
                }
            }
          }
#pragma unroll
          for (int tt = 0; tt < R; ++tt)
#pragma unroll
            for (int u = 0; u < TW; ++u) acc[tt][u] = (j == 0) ? part[tt][u] : acc[tt][u] + part[tt][u];
        }
        T* xo = dx + (k.q0 + pp) * (int64_t)H * W + iw0;
        if constexpr (S == 1) {
#pragma unroll
          for (int tt = 0; tt < R; ++tt)
            if (ih0 + tt < k.r1) VecIO<T, V>::store(xo + (int64_t)(ih0 + tt) * W, acc[tt]);
        } else {
          const bool whole = (W % TW == 0);  // the tile's columns fit and are TW-element aligned
#pragma unroll
          for (int tt = 0; tt < R; ++tt) {
            if (ih0 + tt >= k.r1) continue;
            T* row = xo + (int64_t)(ih0 + tt) * W;
            if (whole) {
              VecIO<T, TW>::store(row, acc[tt]);
            } else {
#pragma unroll
              for (int u = 0; u < TW; ++u)
                if (iw0 + u < W) Elem<T>::store(row + u, acc[tt][u]);
            }
          }
        }
        }
      }
      __syncwarp();
      if ((threadIdx.x & 31) == 0) mbar_arrive(&empty[s]);
      if (++s == a.ns) { s = 0; ph ^= 1; }
    }
  }
  griddep_launch_dependents();
}

// V = 8 (one 16-B row load per window) exists for bf16 3x3 only.
template <class T, int K, int S, int R, bool PD, bool M1 = false>
KernelFn v8_kernel() {
  if constexpr (std::is_same<T, __nv_bfloat16>::value && K == 3 && PD)
    return nchw_bwd_data_kernel<T, K, S, R, 8, PD, false, M1>;
  else return nullptr;
}

template <class T, int K, int S, bool PD, bool M1 = false>
KernelFn pick_rv(int RI, int VI) {
  constexpr int R0 = rows_bd(K, S, 0), R1 = rows_bd(K, S, 1);
  if constexpr (S == 1) {
#define DW_V(R)                                                   \
  switch (VI) {                                                   \
    case 0: return nchw_bwd_data_kernel<T, K, S, R, 1, PD, false, M1>;       \
    case 1: return nchw_bwd_data_kernel<T, K, S, R, 2, PD, false, M1>;       \
    case 2: return PD ? nchw_bwd_data_kernel<T, K, S, R, 4, PD, false, M1> : nullptr; \
    case 3: return v8_kernel<T, K, S, R, PD, M1>();                 \
    default: return nullptr;                                      \
  }
    if (RI == 0) { DW_V(R0) } else { DW_V(R1) }
#undef DW_V
  } else {  // stride 2: tiles of R rows x 2V columns
    switch (VI) {
      case 0: return RI == 0 ? nchw_bwd_data_kernel<T, K, S, R0, 1, PD, false, M1> : nchw_bwd_data_kernel<T, K, S, R1, 1, PD, false, M1>;
      case 1: return RI == 0 ? nchw_bwd_data_kernel<T, K, S, R0, 2, PD, false, M1> : nchw_bwd_data_kernel<T, K, S, R1, 2, PD, false, M1>;
      case 2:
        if constexpr (K == 3) return RI == 0 ? nchw_bwd_data_kernel<T, K, S, R0, 4, PD, false, M1> : nchw_bwd_data_kernel<T, K, S, R1, 4, PD, false, M1>;
        else return nullptr;
      case 3:  // bf16 3x3 streaming strips (m = 1), 16 dx columns
        if constexpr (K == 3 && PD && std::is_same<T, __nv_bfloat16>::value)
          return RI == 0 ? nchw_bwd_data_kernel<T, K, S, R0, 8, PD, false, M1> : nchw_bwd_data_kernel<T, K, S, R1, 8, PD, false, M1>;
        else return nullptr;
      default: return nullptr;
    }
  }
}

template <class T, bool PD>
KernelFn pick_t_m1(int K, int S, int RI, int VI) {  // m = 1
  if (S == 1) {
    if (K == 3) return pick_rv<T, 3, 1, PD, true>(RI, VI);
    if (K == 5) return pick_rv<T, 5, 1, PD, true>(RI, VI);
    if (K == 7) return pick_rv<T, 7, 1, PD, true>(RI, VI);
  } else if (S == 2) {
    if (K == 3) return pick_rv<T, 3, 2, PD, true>(RI, VI);
    if (K == 5) return pick_rv<T, 5, 2, PD, true>(RI, VI);
    if (K == 7) return pick_rv<T, 7, 2, PD, true>(RI, VI);
  }
  return nullptr;
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

// bf16 plane-pair kernels (S = 1, 3x3): V even.
template <int R, bool PD>
KernelFn pick_pair_v(int VI) {
  using B = __nv_bfloat16;
  switch (VI) {
    case 1: return nchw_bwd_data_kernel<B, 3, 1, R, 2, PD, true>;
    case 2: if constexpr (PD) return nchw_bwd_data_kernel<B, 3, 1, R, 4, PD, true>; else return nullptr;
    case 3: if constexpr (PD) return nchw_bwd_data_kernel<B, 3, 1, R, 8, PD, true>; else return nullptr;
    default: return nullptr;
  }
}

KernelFn bwd_data_kernel(int dtype, int K, int S, int RI, int VI, bool padded, bool pair, bool m1) {
  if (!pair && m1 && (S == 1 || S == 2)) {
    if (dtype == DWCONV_F32) return padded ? pick_t_m1<float, true>(K, S, RI, VI) : pick_t_m1<float, false>(K, S, RI, VI);
    return padded ? pick_t_m1<__nv_bfloat16, true>(K, S, RI, VI) : pick_t_m1<__nv_bfloat16, false>(K, S, RI, VI);
  }
  if (pair) {
    if (dtype != DWCONV_BF16 || K != 3) return nullptr;
    if (S == 2) {  // polyphase pair tiles, 2V columns
      using B = __nv_bfloat16;
      constexpr int R0 = rows_bd(3, 2, 0), R1 = rows_bd(3, 2, 1);
      switch (VI) {
        case 0: return RI == 0 ? (padded ? nchw_bwd_data_kernel<B, 3, 2, R0, 1, true, true> : nchw_bwd_data_kernel<B, 3, 2, R0, 1, false, true>)
                               : (padded ? nchw_bwd_data_kernel<B, 3, 2, R1, 1, true, true> : nchw_bwd_data_kernel<B, 3, 2, R1, 1, false, true>);
        case 1: return RI == 0 ? (padded ? nchw_bwd_data_kernel<B, 3, 2, R0, 2, true, true> : nchw_bwd_data_kernel<B, 3, 2, R0, 2, false, true>)
                               : (padded ? nchw_bwd_data_kernel<B, 3, 2, R1, 2, true, true> : nchw_bwd_data_kernel<B, 3, 2, R1, 2, false, true>);
        case 2: return RI == 0 ? (padded ? nchw_bwd_data_kernel<B, 3, 2, R0, 4, true, true> : nchw_bwd_data_kernel<B, 3, 2, R0, 4, false, true>)
                               : (padded ? nchw_bwd_data_kernel<B, 3, 2, R1, 4, true, true> : nchw_bwd_data_kernel<B, 3, 2, R1, 4, false, true>);
        default: return nullptr;
      }
    }
    constexpr int R0 = rows_bd(3, 1, 0), R1 = rows_bd(3, 1, 1);
    if (RI == 0) return padded ? pick_pair_v<R0, true>(VI) : pick_pair_v<R0, false>(VI);
    return padded ? pick_pair_v<R1, true>(VI) : pick_pair_v<R1, false>(VI);
  }
  if (dtype == DWCONV_F32) return padded ? pick_t<float, true>(K, S, RI, VI) : pick_t<float, false>(K, S, RI, VI);
  return padded ? pick_t<__nv_bfloat16, true>(K, S, RI, VI) : pick_t<__nv_bfloat16, false>(K, S, RI, VI);
}

}  // namespace nchw
}  // namespace dwk
