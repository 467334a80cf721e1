// nchw_fwd.cu -- dwconv_fwd for NCHW on sm_100a (see nchw_common.cuh).
//
// y[n, c*m+j, oh, ow] = sum_{i,jj} w[c*m+j, i, jj] * x[n, c, oh*S-PAD+i, ow*S-PAD+jj]
// (Eq. 3).  Persistent grid; each
// chunk is P whole x planes or one band of one plane; thread strip = R output
// rows x V output columns of one output plane.
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
    k.q0 = c / a.nbands;
    const int b = (int)(c - k.q0 * a.nbands);
    k.np = 1;
    k.r0 = b * a.BR;
    k.r1 = min(k.r0 + a.BR, a.Ho);
    k.lo = max(0, k.r0 * S - PAD);
    k.hi = min(a.H, (k.r1 - 1) * S - PAD + K);
  }
  return k;
}

template <class T, int K, int S, int R, int V, bool PADDED>
__global__ void __launch_bounds__(kThreads) nchw_fwd_kernel(const NArgs a) {
  constexpr int PAD = (K - 1) / 2, KK = K * K;
  constexpr int kWPT = 4;  // weights per thread per chunk (host keeps P*m*K*K <= 4*256)
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem);
  const T* __restrict__ x = static_cast<const T*>(a.in);
  T* __restrict__ y = static_cast<T*>(a.out);
  const T* __restrict__ wt = static_cast<const T*>(a.w);
  const int W = a.W, Wo = a.Wo, m = a.m;
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
    const ChunkRows k = fwd_rows<K, S>(a, c);
    const int cbase = (int)(k.q0 % a.C) * m;
    const int nw = k.np * m * KK;
#pragma unroll
    for (int q = 0; q < kWPT; ++q) {
      const int idx = threadIdx.x + q * (int)blockDim.x;
      if (idx < nw) {
        const int pl = idx / KK, qq = idx - pl * KK;
        const uint32_t ov = (uint32_t)(cbase + pl);
        const int o = (int)(ov - fdiv(ov, a.div_co) * (uint32_t)a.Co);
        wreg[q] = Elem<T>::ldg(wt + (int64_t)o * KK + qq);
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

  // input staging of a chunk: its x planes (rows [lo, hi) of each)
  auto spec_of = [&](const ChunkRows& k) {
    StageSpec sp;
    sp.cnt = (int64_t)(k.hi - k.lo) * W;
    sp.gstride = (int64_t)a.H * W;
    sp.npl = k.np;
    sp.pitch = PADDED ? a.pitch : (int)sp.cnt;
    sp.zbe = PADDED ? a.zbe : 0;
    return sp;
  };
  auto issue = [&](int64_t c, int st) {  // thread 0
    const ChunkRows k = fwd_rows<K, S>(a, c);
    const T* src = x + (k.q0 * a.H + k.lo) * W;
    const StageSpec sp = spec_of(k);
    if (stage_bulk_ok<T>(src, sp)) {
      mbar_arrive_expect_tx(&bars[st], stage_bytes<T>(sp));
      stage_copy<T>(sin_of(st), src, sp, &bars[st]);
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
      const int64_t cn = c + (int64_t)(a.ns - 1) * gridDim.x;  // into the stage freed last iteration
      if (cn < a.nchunks) issue(cn, st == 0 ? a.ns - 1 : st - 1);
      bulk_wait_read<1>();  // the bulk store issued two iterations ago has read sout[it & 1]
    }
    const ChunkRows k = fwd_rows<K, S>(a, c);
    T* sin = sin_of(st);
    T* sout = sout_of(it & 1);
    const int npl = k.np * m;
    const float* swc = sw + (it & 1) * wstride;
    // weights of the NEXT chunk: loads in flight now, stored to smem after compute
    if (c + gridDim.x < a.nchunks) load_w(c + gridDim.x, wnext);
    mbar_wait(&bars[st], par);
    if (++st == a.ns) { st = 0; par ^= 1; }
    const StageSpec sp = spec_of(k);
    {
      const T* src = x + (k.q0 * a.H + k.lo) * W;
      if (!stage_bulk_ok<T>(src, sp)) stage_coop<T>(sin, src, sp);
      // band mode: the padding rows under the last band are zero rows
      if (PADDED && a.nbands > 1 && k.hi == a.H) zero_elems(sin + sp.zbe + sp.cnt, PAD * W);
    }
    __syncthreads();

    const int rows_in = k.hi - k.lo;
    (void)rows_in;
    const int rows_out = k.r1 - k.r0;
    const int ncg = (int)a.div_ncg.d;
    const int ntiles = npl * a.nsb * ncg;
    for (int t = threadIdx.x; t < ntiles; t += (int)blockDim.x) {
      const int t2 = (int)fdiv((uint32_t)t, a.div_ncg);
      const int c0 = (t - t2 * ncg) * V;
      const int pp = (int)fdiv((uint32_t)t2, a.div_nsb);
      const int sb = t2 - pp * a.nsb;
      const int pin = (int)fdiv((uint32_t)pp, a.div_m);
      const int oh0 = k.r0 + sb * R;
      float wr[KK];
#pragma unroll
      for (int q = 0; q < KK; ++q) wr[q] = swc[pp * KK + q];
      float acc[R][V];
#pragma unroll
      for (int tt = 0; tt < R; ++tt)
#pragma unroll
        for (int u = 0; u < V; ++u) acc[tt][u] = 0.f;
      stencil_strip<T, K, S, R, V, PADDED>(sin + pin * sp.pitch + sp.zbe - k.lo * W, zrow, W, k.lo, rows_in,
                                           oh0 * S - PAD, c0, wr, acc);
      T* so = sout + (pp * rows_out + (oh0 - k.r0)) * Wo + c0;
#pragma unroll
      for (int tt = 0; tt < R; ++tt)
        if (oh0 + tt < k.r1) VecIO<T, V>::store(so + tt * Wo, acc[tt]);
    }
    store_w(sw + ((it + 1) & 1) * wstride, wnext);
    fence_proxy_async_smem();
    __syncthreads();

    // ---- store: one contiguous range (whole planes) or m ranges (band mode)
    const int nranges = (rows_out == a.Ho) ? 1 : m;
    const int64_t rcnt = (rows_out == a.Ho) ? (int64_t)npl * a.Ho * Wo : (int64_t)rows_out * Wo;
    bool ok = true;
    for (int j = 0; j < nranges; ++j) {
      T* dst = y + ((k.q0 * m + j) * a.Ho + k.r0) * Wo;
      ok = ok && bulk_ok(dst, rcnt, (uint32_t)(j * rcnt * sizeof(T)));
    }
    if (ok) {
      if (threadIdx.x == 0) {
        for (int j = 0; j < nranges; ++j)
          bulk_s2g(y + ((k.q0 * m + j) * a.Ho + k.r0) * Wo, sout + j * rcnt, (uint32_t)(rcnt * sizeof(T)));
      }
    } else {
      for (int j = 0; j < nranges; ++j)
        coop_copy(y + ((k.q0 * m + j) * a.Ho + k.r0) * Wo, (const T*)(sout + j * rcnt), rcnt);
    }
    if (threadIdx.x == 0) bulk_commit();
  }
  griddep_launch_dependents();
  if (threadIdx.x == 0) bulk_wait_read<0>();  // smem must outlive the stores' reads
}

template <class T, int K, int S, bool PD>
KernelFn pick_rv(int RI, int VI) {
  constexpr int R0 = rows_fwd(K, 0), R1 = rows_fwd(K, 1);
#define DW_V(R)                                              \
  switch (VI) {                                              \
    case 0: return nchw_fwd_kernel<T, K, S, R, 1, PD>;       \
    case 1: return nchw_fwd_kernel<T, K, S, R, 2, PD>;       \
    case 2: return PD ? nchw_fwd_kernel<T, K, S, R, 4, PD> : nullptr; \
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

KernelFn fwd_kernel(int dtype, int K, int S, int RI, int VI, bool padded) {
  if (dtype == DWCONV_F32) return padded ? pick_t<float, true>(K, S, RI, VI) : pick_t<float, false>(K, S, RI, VI);
  return padded ? pick_t<__nv_bfloat16, true>(K, S, RI, VI) : pick_t<__nv_bfloat16, false>(K, S, RI, VI);
}

}  // namespace nchw
}  // namespace dwk
