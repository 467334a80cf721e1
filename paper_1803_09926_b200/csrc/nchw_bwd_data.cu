// nchw_bwd_data.cu -- dwconv_bwd_data for NCHW on sm_100a (see nchw_common.cuh).
//
// dx[n,c,ih,iw] = sum_{j<m} sum_{i,jj} w[c*m+j,i,jj] * dy[n,c*m+j,(ih+PAD-i)/S,(iw+PAD-jj)/S]
// over exact divisions in range -- the adjoint of the forward pass (DESIGN.md
// reading R9; the paper delegates it to the framework).
//  * S = 1: the forward stencil on dy with the kernel flipped (weights are staged
//    flipped), strip = R dx rows x V dx columns, packed FFMA2.
//  * S = 2: polyphase tile of R dx rows x S dx columns aligned to the stride so
//    the tap -> dy mapping is static.
// Per-j partial sums keep each serial chain at K*K (R5 iii).
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
    k.q0 = c / a.nbands;
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

template <class T, int K, int S, int R, int V, bool PADDED>
__global__ void __launch_bounds__(kThreads) nchw_bwd_data_kernel(const NArgs a) {
  constexpr int PAD = (K - 1) / 2, KK = K * K;
  constexpr int kWPT = 4;  // weights per thread per chunk (host keeps P*m*K*K <= 4*256)
  constexpr int D0 = floor_div(PAD - K + 1, S);
  constexpr int NRY = floor_div(R - 1 + PAD, S) - D0 + 1;
  constexpr int NCY = floor_div(S - 1 + PAD, S) - D0 + 1;
  constexpr int TW = (S == 1) ? V : S;  // dx columns per thread tile
  static_assert(R % S == 0, "dx strip must be stride aligned");
  static_assert(S == 1 || V == 1, "stride-2 tiles are scalar");
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem);
  const T* __restrict__ dy = static_cast<const T*>(a.in);
  T* __restrict__ dx = static_cast<T*>(a.out);
  const T* __restrict__ wt = static_cast<const T*>(a.w);
  const int W = a.W, Wo = a.Wo, m = a.m, H = a.H;
  const T* zrow = reinterpret_cast<const T*>(smem + a.zrow_off);

  prologue(smem, bars, a);
  auto sin_of = [&](int st) { return reinterpret_cast<T*>(smem + a.in0_off + 128 + st * a.in_stage); };
  auto sout_of = [&](int st) { return reinterpret_cast<T*>(smem + a.out0_off + st * a.out_stage); };
  float* sw = reinterpret_cast<float*>(smem + a.w_off);
  // Staged fp32 weights, double-buffered: sw[0..] for even iterations, sw[wstride..] for odd.
  // Each thread holds up to kWPT weights of the next chunk in registers.
  const int wstride = a.P * m * KK;
  float wnext[kWPT];
  auto load_w = [&](int64_t c, float* wreg) {
    const ChunkRows k = bd_rows<K, S>(a, c);
    const int cbase = (int)(k.q0 % a.C) * m;
    const int nw = k.np * m * KK;
#pragma unroll
    for (int q = 0; q < kWPT; ++q) {
      const int idx = threadIdx.x + q * (int)blockDim.x;
      if (idx < nw) {
        const int pl = idx / KK, qq = idx - pl * KK;
        const uint32_t ov = (uint32_t)(cbase + pl);
        const int o = (int)(ov - fdiv(ov, a.div_co) * (uint32_t)a.Co);
        wreg[q] = Elem<T>::ldg(wt + (int64_t)o * KK + ((S == 1) ? (KK - 1 - qq) : qq));
      }
    }
  };
  auto store_w = [&](float* dst, const float* wreg) {
#pragma unroll
    for (int q = 0; q < kWPT; ++q) {
      const int idx = threadIdx.x + q * (int)blockDim.x;
      if (idx < wstride) dst[idx] = wreg[q];
    }
  };

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
  auto issue = [&](int64_t c, int st) {
    const ChunkRows k = bd_rows<K, S>(a, c);
    const StageSpec sp = spec_of(k);
    if (stage_bulk_ok<T>(src_of(k), sp)) {
      mbar_arrive_expect_tx(&bars[st], stage_bytes<T>(sp));
      stage_copy<T>(sin_of(st), src_of(k), sp, &bars[st]);
    } else {
      mbar_arrive(&bars[st]);
    }
  };

  if (threadIdx.x == 0)
    for (int i = 0; i < a.ns - 1; ++i)
      if (blockIdx.x + (int64_t)i * gridDim.x < a.nchunks) issue(blockIdx.x + (int64_t)i * gridDim.x, i);
  if (blockIdx.x < a.nchunks) {  // first chunk's weights (LDG latency overlaps the TMA issue above)
    load_w(blockIdx.x, wnext);
    store_w(sw, wnext);
  }
  int it = 0, st = 0;
  uint32_t par = 0;
  for (int64_t c = blockIdx.x; c < a.nchunks; c += gridDim.x, ++it) {
    if (threadIdx.x == 0) {
      const int64_t cn = c + (int64_t)(a.ns - 1) * gridDim.x;
      if (cn < a.nchunks) issue(cn, st == 0 ? a.ns - 1 : st - 1);
      bulk_wait_read<1>();
    }
    const ChunkRows k = bd_rows<K, S>(a, c);
    T* sin = sin_of(st);
    T* sout = sout_of(it & 1);
    const float* swc = sw + (it & 1) * wstride;
    // weights of the NEXT chunk: loads in flight now, stored to smem after compute
    if (c + gridDim.x < a.nchunks) load_w(c + gridDim.x, wnext);
    mbar_wait(&bars[st], par);
    if (++st == a.ns) { st = 0; par ^= 1; }
    const StageSpec sp = spec_of(k);
    if (!stage_bulk_ok<T>(src_of(k), sp)) stage_coop<T>(sin, src_of(k), sp);
    if (PADDED && a.nbands > 1 && k.hi == a.Ho)  // zero rows under the last band's dy rows
      for (int j = 0; j < m; ++j) zero_elems(sin + j * sp.pitch + sp.zbe + sp.cnt, PAD * Wo);
    __syncthreads();

    const int rows_dy = k.hi - k.lo;
    const int rows_dx = k.r1 - k.r0;
    const int ncg = (int)a.div_ncg.d;
    const int ntiles = k.np * a.nsb * ncg;
    for (int t = threadIdx.x; t < ntiles; t += (int)blockDim.x) {
      const int t2 = (int)fdiv((uint32_t)t, a.div_ncg);
      const int cb = t - t2 * ncg;
      const int pp = (int)fdiv((uint32_t)t2, a.div_nsb);
      const int sb = t2 - pp * a.nsb;
      const int ih0 = k.r0 + sb * R;  // multiple of S
      const int iw0 = cb * TW;
      float acc[R][TW];
#pragma unroll
      for (int tt = 0; tt < R; ++tt)
#pragma unroll
        for (int u = 0; u < TW; ++u) acc[tt][u] = 0.f;
      for (int j = 0; j < m; ++j) {
        const float* wp = swc + (pp * m + j) * KK;
        float wr[KK];
#pragma unroll
        for (int q = 0; q < KK; ++q) wr[q] = wp[q];
        float part[R][TW];
#pragma unroll
        for (int tt = 0; tt < R; ++tt)
#pragma unroll
          for (int u = 0; u < TW; ++u) part[tt][u] = 0.f;
        const T* splane = sin + (pp * m + j) * sp.pitch + sp.zbe;
        if constexpr (S == 1) {
          // forward stencil with the flipped kernel: dx[ih][iw] = sum wf[a][b] dy[ih-PAD+a][iw-PAD+b]
          stencil_strip<T, K, 1, R, V, PADDED>(splane - k.lo * Wo, zrow, Wo, k.lo, rows_dy, ih0 - PAD, iw0, wr, part);
        } else {
          const int ohb = ih0 / S + D0;
          const int owb = cb + D0;
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
                  for (int u = 0; u < S; ++u)
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
      T* so = sout + (pp * rows_dx - k.r0) * W;
      if constexpr (S == 1) {
#pragma unroll
        for (int tt = 0; tt < R; ++tt)
          if (ih0 + tt < k.r1) VecIO<T, V>::store(so + (ih0 + tt) * W + iw0, acc[tt]);
      } else {
#pragma unroll
        for (int tt = 0; tt < R; ++tt)
#pragma unroll
          for (int u = 0; u < S; ++u) {
            const int ih = ih0 + tt, iw = iw0 + u;
            if (ih < k.r1 && iw < W) Elem<T>::store(so + ih * W + iw, acc[tt][u]);
          }
      }
    }
    store_w(sw + ((it + 1) & 1) * wstride, wnext);
    fence_proxy_async_smem();
    __syncthreads();

    T* dst = dx + (k.q0 * H + k.r0) * W;
    const int64_t ocnt = (int64_t)k.np * rows_dx * W;
    if (bulk_ok(dst, ocnt, 0)) {
      if (threadIdx.x == 0) bulk_s2g(dst, sout, (uint32_t)(ocnt * sizeof(T)));
    } else {
      coop_copy(dst, (const T*)sout, ocnt);
    }
    if (threadIdx.x == 0) bulk_commit();
  }
  griddep_launch_dependents();
  if (threadIdx.x == 0) bulk_wait_read<0>();  // smem must outlive the stores' reads
}

template <class T, int K, int S, bool PD>
KernelFn pick_rv(int RI, int VI) {
  constexpr int R0 = rows_bd(K, S, 0), R1 = rows_bd(K, S, 1);
  if constexpr (S == 1) {
#define DW_V(R)                                                   \
  switch (VI) {                                                   \
    case 0: return nchw_bwd_data_kernel<T, K, S, R, 1, PD>;       \
    case 1: return nchw_bwd_data_kernel<T, K, S, R, 2, PD>;       \
    case 2: return PD ? nchw_bwd_data_kernel<T, K, S, R, 4, PD> : nullptr; \
    default: return nullptr;                                      \
  }
    if (RI == 0) { DW_V(R0) } else { DW_V(R1) }
#undef DW_V
  } else {
    if (VI != 0) return nullptr;
    return RI == 0 ? nchw_bwd_data_kernel<T, K, S, R0, 1, PD> : nchw_bwd_data_kernel<T, K, S, R1, 1, PD>;
  }
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

KernelFn bwd_data_kernel(int dtype, int K, int S, int RI, int VI, bool padded) {
  if (dtype == DWCONV_F32) return padded ? pick_t<float, true>(K, S, RI, VI) : pick_t<float, false>(K, S, RI, VI);
  return padded ? pick_t<__nv_bfloat16, true>(K, S, RI, VI) : pick_t<__nv_bfloat16, false>(K, S, RI, VI);
}

}  // namespace nchw
}  // namespace dwk
