// nchw_fwd.cu -- dwconv_fwd for NCHW on sm_100a (see nchw_common.cuh).
//
// y[n, c*m+j, oh, ow] = sum_{i,jj} w[c*m+j, i, jj] * x[n, c, oh*S-PAD+i, ow*S-PAD+jj]
// (Eq. 3).
//
// Warp-specialised persistent kernel.  Warp 0 is the producer: one lane walks
// the CTA's chunks (P whole x planes, or a band of one plane) and stages each
// into a ring of `ns` shared-memory stages with 1-D TMA bulk copies
// (cp.async.bulk -> UBLKCP), completing on the stage's "full" mbarrier; before
// refilling a stage it waits on the stage's "empty" mbarrier.  The other warps
// are consumers: they wait "full", compute strips of R output rows x V output
// columns (LDS.64/128 windows, packed FFMA2 for stride 1) and store the outputs
// straight from registers with coalesced vector stores, then arrive "empty".
// No CTA-wide barrier inside the loop, so fast warps run ahead into the next
// staged chunk and the ring keeps ns loads in flight per CTA.
#include "nchw_common.cuh"

namespace dwk {
namespace nchw {
namespace {

template <int K, int S>
__device__ __forceinline__ ChunkRows fwd_rows(const NArgs& a, int64_t c) {
  constexpr int PAD = (K - 1) / 2;
  ChunkRows k;
  if (a.nbands == 1) {
    k.q0 = c * a.P;
    k.np = (int)min((int64_t)a.P, a.Q - k.q0);
    k.r0 = 0; k.r1 = a.Ho; k.lo = 0; k.hi = a.H;
  } else {
    k.q0 = (int64_t)fdiv((uint32_t)c, a.div_nb);
    const int b = (int)(c - k.q0 * a.nbands);
    k.np = 1;
    k.r0 = b * a.BR;
    k.r1 = min(k.r0 + a.BR, a.Ho);
    k.lo = max(0, k.r0 * S - PAD);
    k.hi = min(a.H, (k.r1 - 1) * S - PAD + K);
  }
  return k;
}

// PAIR (bf16): consumers compute strips of two output planes at once
// (stencil_strip_pair): FFMA2 lanes = planes, no pair-forming moves.
template <class T, int K, int S, int R, int V, bool PADDED, bool PAIR = false>
__global__ void __launch_bounds__(kThreads + 32) nchw_fwd_kernel(const NArgs a) {
  constexpr int PAD = (K - 1) / 2, KK = K * K;
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  uint64_t* empty = reinterpret_cast<uint64_t*>(smem + 64);
  const T* __restrict__ x = static_cast<const T*>(a.in);
  T* __restrict__ y = static_cast<T*>(a.out);
  const T* __restrict__ wt = static_cast<const T*>(a.w);
  const int W = a.W, Wo = a.Wo, m = a.m;
  const T* zrow = reinterpret_cast<const T*>(smem + a.zrow_off);
  const int nct = (int)blockDim.x - 32;  // consumer threads

  prologue_ws(smem, a, nct >> 5, 2);  // full: TMA arrival + weights arrival
  auto sin_of = [&](int st) { return reinterpret_cast<T*>(smem + a.in0_off + 128 + st * a.in_stage); };
  auto sw_of = [&](int st) { return reinterpret_cast<float*>(smem + a.in0_off + a.in2_off + st * a.in_stage); };
  auto spec_of = [&](const ChunkRows& k) {  // x planes of the chunk, rows [lo, hi)
    StageSpec sp;
    sp.cnt = (int64_t)(k.hi - k.lo) * W;
    sp.gstride = (int64_t)a.H * W;
    sp.npl = k.np;
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
      const ChunkRows k = fwd_rows<K, S>(a, c);
      const WeightWin ww = weight_win<T, KK>(a, k.q0, k.np);
      if constexpr (PADDED) {
        if (a.nbands > 1 && k.hi == a.H) {  // zero rows under the plane's last band (read unchecked)
          const StageSpec sp = spec_of(k);
          zero_bytes16(sin_of(s) + sp.zbe + sp.cnt, (uint32_t)(PAD * W * sizeof(T) + 15) & ~15u, threadIdx.x, 32);
          __syncwarp();
        }
      }
      if (threadIdx.x == 0) {
        const T* src = x + (k.q0 * a.H + k.lo) * W;
        const StageSpec sp = spec_of(k);
        const bool xb = stage_bulk_ok<T>(src, sp);  // else consumers copy this chunk themselves
        const uint32_t tx = (xb ? stage_bytes<T>(sp) : 0u) + (ww.tma ? ww.bytes : 0u);
        if (tx) {
          mbar_arrive_expect_tx(&full[s], tx);
          if (xb) stage_copy<T>(sin_of(s), src, sp, &full[s]);
          if (ww.tma) bulk_g2s(sw_of(s), wt + ww.a0, ww.bytes, &full[s]);
        } else {
          mbar_arrive(&full[s]);
        }
      }
      if (!ww.tma) {  // fallback: the producer warp writes the chunk's weights as an fp32 table
        __syncwarp();
        const int cbase = (int)(k.q0 % a.C) * m;
        float* sw = sw_of(s);
        for (int idx = threadIdx.x; idx < k.np * m * KK; idx += 32) {
          const int pl = idx / KK, q = idx - pl * KK;
          const uint32_t ov = (uint32_t)(cbase + pl);
          const int o = (int)(ov - fdiv(ov, a.div_co) * (uint32_t)a.Co);
          sw[idx] = Elem<T>::ldg(wt + (int64_t)o * KK + q);
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
      const ChunkRows k = fwd_rows<K, S>(a, c);
      const StageSpec sp = spec_of(k);
      T* sin = sin_of(s);
      mbar_wait(&full[s], ph);
      const T* src = x + (k.q0 * a.H + k.lo) * W;
      const bool coop = !stage_bulk_ok<T>(src, sp);
      const bool zbot = false;  // the producer zeroes the rows under a plane's last band
      if (coop || zbot) {  // uniform over the consumers
        if (coop) stage_coop_n<T>(sin, src, sp, ctid, nct);
        if (zbot) zero_elems_n(sin + sp.zbe + sp.cnt, PAD * W, ctid, nct);
        consumer_sync(nct);
      }
      const int rows_in = k.hi - k.lo;
      const int npl = k.np * m;
      const float* swc = sw_of(s);
      const WeightWin ww = weight_win<T, KK>(a, k.q0, k.np);
      const T* swr = reinterpret_cast<const T*>(swc) + ww.off;  // raw rows (ww.tma)
      if constexpr (PAIR) {
        const int npair = (npl + 1) >> 1;
        const int ntp = npair * a.nsb * ncg;
        for (int t = ctid; t < ntp; t += nct) {
          const int t2 = (int)fdiv((uint32_t)t, a.div_ncg);
          const int c0 = (t - t2 * ncg) * V;
          const int pp2 = (int)fdiv((uint32_t)t2, a.div_nsb);
          const int sb = t2 - pp2 * a.nsb;
          const int ppa = 2 * pp2;
          const bool hasb = ppa + 1 < npl;
          const int ppb = hasb ? ppa + 1 : ppa;
          const int pina = (int)fdiv((uint32_t)ppa, a.div_m), pinb = (int)fdiv((uint32_t)ppb, a.div_m);
          const int oh0 = k.r0 + sb * R;
          float2 wp[KK];
          if (ww.tma) {
#pragma unroll
            for (int q = 0; q < KK; ++q) wp[q] = make_float2(Elem<T>::load(swr + ppa * KK + q), Elem<T>::load(swr + ppb * KK + q));
          } else {
#pragma unroll
            for (int q = 0; q < KK; ++q) wp[q] = make_float2(swc[ppa * KK + q], swc[ppb * KK + q]);
          }
          float2 acc[R][V];
#pragma unroll
          for (int tt = 0; tt < R; ++tt)
#pragma unroll
            for (int u = 0; u < V; ++u) acc[tt][u] = make_float2(0.f, 0.f);
          const T* base = sin + sp.zbe - k.lo * W;
          stencil_strip_pair<K, S, R, V, PADDED>(base + pina * sp.pitch, base + pinb * sp.pitch, zrow, W, k.lo, rows_in,
                                                 oh0 * S - PAD, c0, wp, acc);
          T* yoa = y + ((k.q0 * m + ppa) * a.Ho + oh0) * Wo + c0;
          T* yob = yoa + (int64_t)a.Ho * Wo;
#pragma unroll
          for (int tt = 0; tt < R; ++tt) {
            if (oh0 + tt < k.r1) {
              float va[V], vb[V];
#pragma unroll
              for (int u = 0; u < V; ++u) { va[u] = acc[tt][u].x; vb[u] = acc[tt][u].y; }
              VecIO<T, V>::store(yoa + tt * Wo, va);
              if (hasb) VecIO<T, V>::store(yob + tt * Wo, vb);
            }
          }
        }
      }
      const int ntiles = PAIR ? 0 : npl * a.nsb * ncg;
      for (int t = ctid; t < ntiles; t += nct) {
        const int t2 = (int)fdiv((uint32_t)t, a.div_ncg);
        const int c0 = (t - t2 * ncg) * V;
        const int pp = (int)fdiv((uint32_t)t2, a.div_nsb);
        const int sb = t2 - pp * a.nsb;
        const int pin = (int)fdiv((uint32_t)pp, a.div_m);
        const int oh0 = k.r0 + sb * R;
        float wr[KK];
        if (ww.tma) {
#pragma unroll
          for (int q = 0; q < KK; ++q) wr[q] = Elem<T>::load(swr + pp * KK + q);
        } else {
#pragma unroll
          for (int q = 0; q < KK; ++q) wr[q] = swc[pp * KK + q];
        }
        T* yo = y + ((k.q0 * m + pp) * a.Ho + oh0) * Wo + c0;
        if constexpr (std::is_same<T, __nv_bfloat16>::value && S == 1 && V >= 4 && kBf16Interleave) {
          // bf16 stride 1: rows leave as soon as they are complete (3 live rows instead of R;
          // measured slower at stride 2, which keeps the whole strip)
          stencil_strip_bf2_stream<K, S, R, V, PADDED>(
              reinterpret_cast<const __nv_bfloat16*>(sin + pin * sp.pitch + sp.zbe - k.lo * W),
              reinterpret_cast<const __nv_bfloat16*>(zrow), W, k.lo, rows_in, oh0 * S - PAD, c0, wr,
              [&](int tt, const float* v) {
                if (oh0 + tt < k.r1) VecIO<T, V>::store(yo + tt * Wo, v);
              });
        } else {
        float acc[R][V];
#pragma unroll
        for (int tt = 0; tt < R; ++tt)
#pragma unroll
          for (int u = 0; u < V; ++u) acc[tt][u] = 0.f;
        stencil_strip<T, K, S, R, V, PADDED>(sin + pin * sp.pitch + sp.zbe - k.lo * W, zrow, W, k.lo, rows_in,
                                             oh0 * S - PAD, c0, wr, acc);
#pragma unroll
        for (int tt = 0; tt < R; ++tt)
          if (oh0 + tt < k.r1) VecIO<T, V>::store(yo + tt * Wo, acc[tt]);
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
template <class T, int K, int S, int R, bool PD>
KernelFn v8_kernel() {
  if constexpr (std::is_same<T, __nv_bfloat16>::value && K == 3 && PD) return nchw_fwd_kernel<T, K, S, R, 8, PD>;
  else return nullptr;
}

template <class T, int K, int S, bool PD>
KernelFn pick_rv(int RI, int VI) {
  constexpr int R0 = rows_fwd(K, 0), R1 = rows_fwd(K, 1);
#define DW_V(R)                                              \
  switch (VI) {                                              \
    case 0: return nchw_fwd_kernel<T, K, S, R, 1, PD>;       \
    case 1: return nchw_fwd_kernel<T, K, S, R, 2, PD>;       \
    case 2: return PD ? nchw_fwd_kernel<T, K, S, R, 4, PD> : nullptr; \
    case 3: return v8_kernel<T, K, S, R, PD>();                 \
    default: return nullptr;                                 \
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

// bf16 plane-pair kernels: S*V even (whole 32-bit words per window), 3x3.
template <int S, int R, bool PD>
KernelFn pick_pair_v(int VI) {
  using B = __nv_bfloat16;
  switch (VI) {
    case 0: if constexpr (S == 2) return nchw_fwd_kernel<B, 3, S, R, 1, PD, true>; else return nullptr;
    case 1: return nchw_fwd_kernel<B, 3, S, R, 2, PD, true>;
    case 2: if constexpr (PD) return nchw_fwd_kernel<B, 3, S, R, 4, PD, true>; else return nullptr;
    case 3: if constexpr (PD) return nchw_fwd_kernel<B, 3, S, R, 8, PD, true>; else return nullptr;
    default: return nullptr;
  }
}
template <bool PD>
KernelFn pick_pair(int S, int RI, int VI) {
  constexpr int R0 = rows_fwd(3, 0), R1 = rows_fwd(3, 1);
  if (S == 1) return RI == 0 ? pick_pair_v<1, R0, PD>(VI) : pick_pair_v<1, R1, PD>(VI);
  return RI == 0 ? pick_pair_v<2, R0, PD>(VI) : pick_pair_v<2, R1, PD>(VI);
}

KernelFn fwd_kernel(int dtype, int K, int S, int RI, int VI, bool padded, bool pair) {
  if (pair) {
    if (dtype != DWCONV_BF16 || K != 3) return nullptr;
    return padded ? pick_pair<true>(S, RI, VI) : pick_pair<false>(S, RI, VI);
  }
  if (dtype == DWCONV_F32) return padded ? pick_t<float, true>(K, S, RI, VI) : pick_t<float, false>(K, S, RI, VI);
  return padded ? pick_t<__nv_bfloat16, true>(K, S, RI, VI) : pick_t<__nv_bfloat16, false>(K, S, RI, VI);
}

}  // namespace nchw
}  // namespace dwk
