// nchw_chunk.cu -- NCHW depthwise fwd / bwd_data / bwd_filter for sm_100a.
//
// The depthwise layer is a memory-bound stencil ("memory
// access takes more execution time than computation"), so the
// design moves every byte of x, y, dy, dx exactly once between HBM and the SM:
//
//  * In NCHW every (n, c) plane is contiguous and consecutive planes are
//    contiguous, so a "chunk" -- P whole planes, or a band of rows of one large
//    plane plus its halo rows -- is ONE contiguous global range.  It is staged
//    into shared memory with a 1-D TMA bulk copy (cp.async.bulk, SASS UBLKCP)
//    completing on an mbarrier, double-buffered so chunk i+1 streams in while
//    chunk i is computed.
//  * Each thread computes a register-blocked strip of outputs (R rows x 1 or S
//    columns) from shared memory; lanes map to consecutive columns so shared
//    loads are conflict-free for stride 1.  Padding is a predicate, not data.
//  * Results are written to a shared output tile and leave with a bulk
//    shared->global copy (bulk_group), so stores are also full-line TMA traffic.
//  * Grids are persistent (min(chunks, resident CTAs x 148 SMs)) for fwd and
//    bwd_data; bwd_filter runs one CTA per (channel group, batch slice) and
//    reduces deterministically: per-chunk chains of <= 64 products, a running
//    sum over <= 32 chunks, a fixed shuffle/shared-memory tree over the threads
//    of a plane, then the last CTA of a channel group (integer ticket) sums the
//    per-slice partials in a fixed pairwise order.  No float atomics.
//
// This is the paper's "specialized kernel" family re-designed for
// B200, not the diagonalwise GEMM: no weight scatter, no C-fold
// extra multiply-adds.
#include <algorithm>
#include <cstdlib>
#include <mutex>

#include "common.cuh"
#include "kernels.h"

namespace dwk {
namespace {

constexpr int kThreads = 256;

struct NArgs {
  const void* in;     // fwd: x; bwd_data: dy; bwd_filter: x
  const void* in2;    // bwd_filter: dy
  void* out;          // fwd: y; bwd_data: dx
  const void* w;      // [C*m][K][K] storage dtype
  float* dw;          // bwd_filter output
  float* ws_part;     // bwd_filter per-slice partials [nslices][Co][K*K]
  unsigned* ws_ticket;// bwd_filter tickets [groups]
  int64_t N, C, Q;    // Q: planes iterated (fwd: N*C x planes, bwd_data: N*C dx planes)
  int m, Co, H, W, Ho, Wo;
  int P, nbands, BR, nsb;
  int64_t nchunks;
  uint32_t in_bytes, in2_bytes, out_bytes;
  int groups, nslices, nps, tpg;
  FastDiv div_wo, div_nsb, div_m, div_ncb, div_tiles;
};

__host__ __device__ constexpr int pmod(int a, int b) { return ((a % b) + b) % b; }

template <class T>
__device__ __forceinline__ bool bulk_ok(const T* gptr, int64_t count, uint32_t smem_off_bytes) {
  return ((reinterpret_cast<uintptr_t>(gptr) | (uintptr_t)(count * (int64_t)sizeof(T)) | smem_off_bytes) & 15u) == 0;
}

// ============================================================================
// Forward.  Output strip: R consecutive output rows of one output plane at one
// column.  Input rows are streamed: each input row's K taps are loaded once and
// applied to every output row of the strip that uses it.
// ============================================================================
template <int K, int S>
struct FwdCfg {
  static constexpr int PAD = (K - 1) / 2;
  static constexpr int R = (K == 7) ? 4 : ((S == 1) ? 8 : 4);
  static constexpr int NR = (R - 1) * S + K;
};

struct ChunkRows {
  int64_t q0;  // first input plane (fwd/bwd_filter: x plane; bwd_data: dx plane)
  int np;      // planes in chunk
  int r0, r1;  // output rows [r0, r1)
  int lo, hi;  // rows of the input held in smem [lo, hi)
};

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

template <class T, int K, int S>
__global__ void __launch_bounds__(kThreads) nchw_fwd_kernel(const NArgs a) {
  using Cfg = FwdCfg<K, S>;
  constexpr int R = Cfg::R, PAD = Cfg::PAD, NR = Cfg::NR;
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem);
  const uint32_t stage = a.in_bytes + a.out_bytes;
  const T* __restrict__ x = static_cast<const T*>(a.in);
  T* __restrict__ y = static_cast<T*>(a.out);
  const T* __restrict__ wt = static_cast<const T*>(a.w);
  const int W = a.W, Wo = a.Wo, m = a.m;

  if (threadIdx.x == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    fence_mbar_init();
  }
  __syncthreads();

  auto sin_of = [&](int st) { return reinterpret_cast<T*>(smem + 128 + st * stage); };
  auto sout_of = [&](int st) { return reinterpret_cast<T*>(smem + 128 + st * stage + a.in_bytes); };

  auto issue = [&](int64_t c, int st) {  // thread 0
    const ChunkRows k = fwd_rows<K, S>(a, c);
    const T* src = x + (k.q0 * a.H + k.lo) * W;
    const int64_t cnt = (int64_t)k.np * (k.hi - k.lo) * W;
    if (bulk_ok(src, cnt, 0)) {
      mbar_arrive_expect_tx(&bars[st], (uint32_t)(cnt * sizeof(T)));
      bulk_g2s(sin_of(st), src, (uint32_t)(cnt * sizeof(T)), &bars[st]);
    } else {
      mbar_arrive(&bars[st]);
    }
  };

  int it = 0;
  int64_t c = blockIdx.x;
  if (threadIdx.x == 0 && c < a.nchunks) issue(c, 0);
  for (; c < a.nchunks; c += gridDim.x, ++it) {
    const int st = it & 1;
    const int64_t cn = c + gridDim.x;
    if (threadIdx.x == 0) {
      if (cn < a.nchunks) issue(cn, st ^ 1);
      bulk_wait_read<1>();  // the bulk store issued two iterations ago has read sout[st]
    }
    const ChunkRows k = fwd_rows<K, S>(a, c);
    T* sin = sin_of(st);
    T* sout = sout_of(st);
    mbar_wait(&bars[st], (it >> 1) & 1);
    {
      const T* src = x + (k.q0 * a.H + k.lo) * W;
      const int64_t cnt = (int64_t)k.np * (k.hi - k.lo) * W;
      if (!bulk_ok(src, cnt, 0)) coop_copy(sin, src, cnt);
    }
    __syncthreads();

    const int rows_in = k.hi - k.lo;
    const int rows_out = k.r1 - k.r0;
    const int npl = k.np * m;
    const int ntiles = npl * a.nsb * Wo;
    int cached_pp = -1;
    const int cbase = (int)(k.q0 % a.C) * m;
    float wr[K * K];
    for (int t = threadIdx.x; t < ntiles; t += kThreads) {
      const int t2 = (int)fdiv((uint32_t)t, a.div_wo);
      const int ow = t - t2 * Wo;
      const int pp = (int)fdiv((uint32_t)t2, a.div_nsb);
      const int sb = t2 - pp * a.nsb;
      const int pin = (int)fdiv((uint32_t)pp, a.div_m);
      if (pp != cached_pp) {
        cached_pp = pp;
        const int o = (cbase + pp) % a.Co;
#pragma unroll
        for (int q = 0; q < K * K; ++q) wr[q] = Elem<T>::ldg(wt + (int64_t)o * (K * K) + q);
      }
      const T* s = sin + pin * rows_in * W;
      const int oh0 = k.r0 + sb * R;
      const int ih0 = oh0 * S - PAD;
      const int iw0 = ow * S - PAD;
      float acc[R];
#pragma unroll
      for (int tt = 0; tt < R; ++tt) acc[tt] = 0.f;
#pragma unroll
      for (int r = 0; r < NR; ++r) {
        const int ih = ih0 + r;
        const bool rok = (ih >= k.lo) && (ih < k.hi);
        const T* srow = s + (ih - k.lo) * W;
        float v[K];
#pragma unroll
        for (int jj = 0; jj < K; ++jj) {
          const int iw = iw0 + jj;
          v[jj] = (rok && iw >= 0 && iw < W) ? Elem<T>::load(srow + iw) : 0.f;
        }
#pragma unroll
        for (int tt = 0; tt < R; ++tt) {
          const int i = r - tt * S;
          if (i >= 0 && i < K) {
#pragma unroll
            for (int jj = 0; jj < K; ++jj) acc[tt] = fmaf(wr[i * K + jj], v[jj], acc[tt]);
          }
        }
      }
      T* so = sout + (pp * rows_out + (oh0 - k.r0)) * Wo + ow;
#pragma unroll
      for (int tt = 0; tt < R; ++tt)
        if (oh0 + tt < k.r1) Elem<T>::store(so + tt * Wo, acc[tt]);
    }
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
  if (threadIdx.x == 0) bulk_wait<0>();
}

// ============================================================================
// Input gradient.  Output tile: R dx rows x S dx columns, aligned to the stride
// so that which taps reach which dy element is static (polyphase form).  dy
// rows are streamed; per-j partial sums keep the serial chain at K*K (R5 iii).
// ============================================================================
template <int K, int S>
struct BdCfg {
  static constexpr int PAD = (K - 1) / 2;
  static constexpr int R = (K == 7) ? 4 : 8;  // multiple of S
  static constexpr int D0 = floor_div(PAD - K + 1, S);
  static constexpr int NRY = floor_div(R - 1 + PAD, S) - D0 + 1;
  static constexpr int NCY = floor_div(S - 1 + PAD, S) - D0 + 1;
};

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

template <class T, int K, int S>
__global__ void __launch_bounds__(kThreads) nchw_bwd_data_kernel(const NArgs a) {
  using Cfg = BdCfg<K, S>;
  constexpr int R = Cfg::R, PAD = Cfg::PAD, D0 = Cfg::D0, NRY = Cfg::NRY, NCY = Cfg::NCY;
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem);
  const uint32_t stage = a.in_bytes + a.out_bytes;
  const T* __restrict__ dy = static_cast<const T*>(a.in);
  T* __restrict__ dx = static_cast<T*>(a.out);
  const T* __restrict__ wt = static_cast<const T*>(a.w);
  const int W = a.W, Wo = a.Wo, m = a.m, H = a.H;

  if (threadIdx.x == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    fence_mbar_init();
  }
  __syncthreads();
  auto sin_of = [&](int st) { return reinterpret_cast<T*>(smem + 128 + st * stage); };
  auto sout_of = [&](int st) { return reinterpret_cast<T*>(smem + 128 + st * stage + a.in_bytes); };

  // input ranges: whole planes -> one range of np*m planes; band -> m ranges
  auto in_src = [&](const ChunkRows& k, int j) -> const T* {
    return dy + ((k.q0 * m + j) * a.Ho + k.lo) * Wo;
  };
  auto in_cnt = [&](const ChunkRows& k) -> int64_t {
    return (a.nbands == 1) ? (int64_t)k.np * m * a.Ho * Wo : (int64_t)(k.hi - k.lo) * Wo;
  };
  auto in_n = [&]() { return (a.nbands == 1) ? 1 : m; };
  auto chunk_bulk = [&](const ChunkRows& k) {
    const int64_t cnt = in_cnt(k);
    bool ok = true;
    for (int j = 0; j < in_n(); ++j) ok = ok && bulk_ok(in_src(k, j), cnt, (uint32_t)(j * cnt * sizeof(T)));
    return ok;
  };
  auto issue = [&](int64_t c, int st) {
    const ChunkRows k = bd_rows<K, S>(a, c);
    const int64_t cnt = in_cnt(k);
    if (chunk_bulk(k)) {
      mbar_arrive_expect_tx(&bars[st], (uint32_t)(in_n() * cnt * sizeof(T)));
      for (int j = 0; j < in_n(); ++j)
        bulk_g2s(sin_of(st) + j * cnt, in_src(k, j), (uint32_t)(cnt * sizeof(T)), &bars[st]);
    } else {
      mbar_arrive(&bars[st]);
    }
  };

  int it = 0;
  int64_t c = blockIdx.x;
  if (threadIdx.x == 0 && c < a.nchunks) issue(c, 0);
  for (; c < a.nchunks; c += gridDim.x, ++it) {
    const int st = it & 1;
    const int64_t cn = c + gridDim.x;
    if (threadIdx.x == 0) {
      if (cn < a.nchunks) issue(cn, st ^ 1);
      bulk_wait_read<1>();
    }
    const ChunkRows k = bd_rows<K, S>(a, c);
    T* sin = sin_of(st);
    T* sout = sout_of(st);
    mbar_wait(&bars[st], (it >> 1) & 1);
    if (!chunk_bulk(k)) {
      const int64_t cnt = in_cnt(k);
      for (int j = 0; j < in_n(); ++j) coop_copy(sin + j * cnt, in_src(k, j), cnt);
    }
    __syncthreads();

    const int rows_dy = k.hi - k.lo;
    const int rows_dx = k.r1 - k.r0;
    const int ncb = (int)a.div_ncb.d;
    const int ntiles = k.np * a.nsb * ncb;
    for (int t = threadIdx.x; t < ntiles; t += kThreads) {
      const int t2 = (int)fdiv((uint32_t)t, a.div_ncb);
      const int cb = t - t2 * ncb;
      const int pp = (int)fdiv((uint32_t)t2, a.div_nsb);
      const int sb = t2 - pp * a.nsb;
      const int ch = (int)((k.q0 % a.C + pp) % a.C);
      const int ih0 = k.r0 + sb * R;  // multiple of S
      const int iw0 = cb * S;
      const int ohb = ih0 / S + D0;
      const int owb = cb + D0;
      float acc[R][S];
#pragma unroll
      for (int tt = 0; tt < R; ++tt)
#pragma unroll
        for (int u = 0; u < S; ++u) acc[tt][u] = 0.f;
      for (int j = 0; j < m; ++j) {
        const int o = ch * m + j;
        float wr[K * K];
#pragma unroll
        for (int q = 0; q < K * K; ++q) wr[q] = Elem<T>::ldg(wt + (int64_t)o * (K * K) + q);
        const T* s = sin + (pp * m + j) * rows_dy * Wo;
        float part[R][S];
#pragma unroll
        for (int tt = 0; tt < R; ++tt)
#pragma unroll
          for (int u = 0; u < S; ++u) part[tt][u] = 0.f;
#pragma unroll
        for (int ry = 0; ry < NRY; ++ry) {
          const int oh = ohb + ry;
          const bool rok = (oh >= k.lo) && (oh < k.hi);
          const T* srow = s + (oh - k.lo) * Wo;
          float v[NCY];
#pragma unroll
          for (int cy = 0; cy < NCY; ++cy) {
            const int ow = owb + cy;
            v[cy] = (rok && ow >= 0 && ow < Wo) ? Elem<T>::load(srow + ow) : 0.f;
          }
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
#pragma unroll
        for (int tt = 0; tt < R; ++tt)
#pragma unroll
          for (int u = 0; u < S; ++u) acc[tt][u] = (j == 0) ? part[tt][u] : acc[tt][u] + part[tt][u];
      }
      T* so = sout + pp * rows_dx * W;
#pragma unroll
      for (int tt = 0; tt < R; ++tt)
#pragma unroll
        for (int u = 0; u < S; ++u) {
          const int ih = ih0 + tt, iw = iw0 + u;
          if (ih < k.r1 && iw < W) Elem<T>::store(so + (ih - k.r0) * W + iw, acc[tt][u]);
        }
    }
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
  if (threadIdx.x == 0) bulk_wait<0>();
}

// ============================================================================
// Filter gradient.  CTA = (channel group g of P channels, batch slice sl).
// Thread groups of `tpg` consecutive threads own one dy plane (o = c*m + j).
// ============================================================================
template <class T, int K, int S>
__global__ void __launch_bounds__(kThreads) nchw_bwd_filter_kernel(const NArgs a) {
  using Cfg = FwdCfg<K, S>;
  constexpr int R = Cfg::R, PAD = Cfg::PAD, NR = Cfg::NR, KK = K * K;
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem);
  unsigned* s_last = reinterpret_cast<unsigned*>(smem + 64);
  const uint32_t stage = a.in_bytes + a.in2_bytes;
  const T* __restrict__ x = static_cast<const T*>(a.in);
  const T* __restrict__ dy = static_cast<const T*>(a.in2);
  const int W = a.W, Wo = a.Wo, m = a.m, H = a.H, Ho = a.Ho;

  const int g = blockIdx.x % a.groups;
  const int sl = blockIdx.x / a.groups;
  const int c0 = g * a.P;
  const int np = min(a.P, (int)(a.C - c0));
  const int64_t n0 = (int64_t)sl * a.nps;
  const int64_t n1 = min(a.N, n0 + a.nps);
  const int iters = (int)(n1 - n0) * a.nbands;

  if (threadIdx.x == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    fence_mbar_init();
  }
  __syncthreads();
  auto sx_of = [&](int st) { return reinterpret_cast<T*>(smem + 128 + st * stage); };
  auto sdy_of = [&](int st) { return reinterpret_cast<T*>(smem + 128 + st * stage + a.in_bytes); };

  struct Rows { int64_t n; int r0, r1, lo, hi; };
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
    return r;
  };
  auto x_src = [&](const Rows& r) { return x + ((r.n * a.C + c0) * H + r.lo) * W; };
  auto x_cnt = [&](const Rows& r) { return (int64_t)np * (r.hi - r.lo) * W; };
  auto dy_src = [&](const Rows& r, int j) { return dy + (((r.n * a.C + c0) * m + j) * Ho + r.r0) * Wo; };
  auto dy_cnt = [&](const Rows& r) {
    return (a.nbands == 1) ? (int64_t)np * m * Ho * Wo : (int64_t)(r.r1 - r.r0) * Wo;
  };
  auto dy_n = [&]() { return (a.nbands == 1) ? 1 : m; };
  auto chunk_bulk = [&](const Rows& r) {
    bool ok = bulk_ok(x_src(r), x_cnt(r), 0);
    const int64_t dc = dy_cnt(r);
    for (int j = 0; j < dy_n(); ++j) ok = ok && bulk_ok(dy_src(r, j), dc, (uint32_t)(j * dc * sizeof(T)));
    return ok;
  };
  auto issue = [&](int kk, int st) {
    const Rows r = rows_of(kk);
    if (chunk_bulk(r)) {
      const int64_t xc = x_cnt(r), dc = dy_cnt(r);
      mbar_arrive_expect_tx(&bars[st], (uint32_t)((xc + dy_n() * dc) * sizeof(T)));
      bulk_g2s(sx_of(st), x_src(r), (uint32_t)(xc * sizeof(T)), &bars[st]);
      for (int j = 0; j < dy_n(); ++j)
        bulk_g2s(sdy_of(st) + j * dc, dy_src(r, j), (uint32_t)(dc * sizeof(T)), &bars[st]);
    } else {
      mbar_arrive(&bars[st]);
    }
  };

  const int gp = threadIdx.x / a.tpg;       // dy plane of this thread within the group
  const int lane_g = threadIdx.x - gp * a.tpg;
  const bool active = gp < np * m;
  float run[KK];
#pragma unroll
  for (int q = 0; q < KK; ++q) run[q] = 0.f;

  if (threadIdx.x == 0 && iters > 0) issue(0, 0);
  for (int kk = 0; kk < iters; ++kk) {
    const int st = kk & 1;
    if (threadIdx.x == 0 && kk + 1 < iters) issue(kk + 1, st ^ 1);
    const Rows r = rows_of(kk);
    T* sx = sx_of(st);
    T* sdy = sdy_of(st);
    mbar_wait(&bars[st], (kk >> 1) & 1);
    if (!chunk_bulk(r)) {
      coop_copy(sx, x_src(r), x_cnt(r));
      const int64_t dc = dy_cnt(r);
      for (int j = 0; j < dy_n(); ++j) coop_copy(sdy + j * dc, dy_src(r, j), dc);
    }
    __syncthreads();
    if (active) {
      const int rows_x = r.hi - r.lo;
      const int rows_dy = r.r1 - r.r0;
      const T* s_x = sx + (gp / m) * rows_x * W;
      const T* s_dy = sdy + gp * rows_dy * Wo;
      float loc[KK];
#pragma unroll
      for (int q = 0; q < KK; ++q) loc[q] = 0.f;
      const int ntl = a.nsb * Wo;
      for (int t = lane_g; t < ntl; t += a.tpg) {
        const int sb = (int)fdiv((uint32_t)t, a.div_wo);
        const int ow = t - sb * Wo;
        const int oh0 = r.r0 + sb * R;
        float dv[R];
#pragma unroll
        for (int tt = 0; tt < R; ++tt)
          dv[tt] = (oh0 + tt < r.r1) ? Elem<T>::load(s_dy + (oh0 + tt - r.r0) * Wo + ow) : 0.f;
        const int ih0 = oh0 * S - PAD, iw0 = ow * S - PAD;
#pragma unroll
        for (int rr = 0; rr < NR; ++rr) {
          const int ih = ih0 + rr;
          const bool rok = (ih >= r.lo) && (ih < r.hi);
          const T* srow = s_x + (ih - r.lo) * W;
          float v[K];
#pragma unroll
          for (int jj = 0; jj < K; ++jj) {
            const int iw = iw0 + jj;
            v[jj] = (rok && iw >= 0 && iw < W) ? Elem<T>::load(srow + iw) : 0.f;
          }
#pragma unroll
          for (int tt = 0; tt < R; ++tt) {
            const int i = rr - tt * S;
            if (i >= 0 && i < K) {
#pragma unroll
              for (int jj = 0; jj < K; ++jj) loc[i * K + jj] = fmaf(v[jj], dv[tt], loc[i * K + jj]);
            }
          }
        }
      }
#pragma unroll
      for (int q = 0; q < KK; ++q) run[q] += loc[q];
    }
    __syncthreads();  // stage st may be refilled by the next-next issue
  }

  // ---- reduce over the tpg threads of each dy plane (fixed tree)
  float* red = reinterpret_cast<float*>(smem + 128);  // reuse stage memory (all loads consumed)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int span = min(a.tpg, 32);
#pragma unroll
  for (int q = 0; q < KK; ++q)
    for (int off = span >> 1; off > 0; off >>= 1) run[q] += __shfl_xor_sync(0xffffffffu, run[q], off);
  const int Co = a.Co;
  float* part = a.ws_part + ((int64_t)sl * Co + (int64_t)c0 * m) * KK;
  if (a.tpg <= 32) {
    if (active && lane_g == 0) {
#pragma unroll
      for (int q = 0; q < KK; ++q) part[gp * KK + q] = run[q];
    }
  } else {
    if (lane == 0) {
#pragma unroll
      for (int q = 0; q < KK; ++q) red[warp * KK + q] = run[q];
    }
    __syncthreads();
    const int wpg = a.tpg >> 5;  // warps per plane
    const int nplanes = np * m;
    for (int idx = threadIdx.x; idx < nplanes * KK; idx += kThreads) {
      const int p = idx / KK, q = idx - p * KK;
      float* base = red + (p * wpg) * KK + q;
      for (int stride = 1; stride < wpg; stride <<= 1)
        for (int u = 0; u + stride < wpg; u += 2 * stride) base[u * KK] += base[(u + stride) * KK];
      part[p * KK + q] = base[0];
    }
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned prev = atomicAdd(&a.ws_ticket[g], 1u);
    *s_last = (prev == (unsigned)(a.nslices - 1)) ? 1u : 0u;
  }
  __syncthreads();
  if (*s_last) {
    __threadfence();
    const int nvals = np * m * KK;
    const float* base = a.ws_part + (int64_t)c0 * m * KK;
    const int64_t sstride = (int64_t)Co * KK;
    for (int idx = threadIdx.x; idx < nvals; idx += kThreads) {
      // pairwise (binary-counter) summation over slices in slice order
      float stk[8];
      int top = 0;
      for (int s = 0; s < a.nslices; ++s) {
        float* slot = const_cast<float*>(base) + s * sstride + idx;
        float cur = __ldcg(slot);
        __stcg(slot, 0.f);  // hand the workspace back zero-filled
        int bits = s;
        while (bits & 1) { cur = stk[--top] + cur; bits >>= 1; }
        stk[top++] = cur;
      }
      float tot = stk[--top];
      while (top > 0) tot = stk[--top] + tot;
      a.dw[(int64_t)c0 * m * KK + idx] = tot;
    }
    if (threadIdx.x == 0) a.ws_ticket[g] = 0u;  // leave the workspace zeroed
  }
}

// ============================================================================
// Host side: kernel tables, planning, launch.
// ============================================================================
using KernelFn = void (*)(NArgs);

template <template <class, int, int> class KT>
struct Table;

template <class T, int K, int S>
struct FwdK { static constexpr KernelFn fn = nchw_fwd_kernel<T, K, S>; };
template <class T, int K, int S>
struct BdK { static constexpr KernelFn fn = nchw_bwd_data_kernel<T, K, S>; };
template <class T, int K, int S>
struct BfK { static constexpr KernelFn fn = nchw_bwd_filter_kernel<T, K, S>; };

template <template <class, int, int> class KT>
KernelFn pick(int dtype, int K, int S) {
#define DW_PICK(T, KV, SV) \
  if (K == KV && S == SV) return KT<T, KV, SV>::fn;
  if (dtype == DWCONV_F32) {
    DW_PICK(float, 3, 1) DW_PICK(float, 3, 2) DW_PICK(float, 5, 1) DW_PICK(float, 5, 2)
    DW_PICK(float, 7, 1) DW_PICK(float, 7, 2)
  } else {
    DW_PICK(__nv_bfloat16, 3, 1) DW_PICK(__nv_bfloat16, 3, 2) DW_PICK(__nv_bfloat16, 5, 1)
    DW_PICK(__nv_bfloat16, 5, 2) DW_PICK(__nv_bfloat16, 7, 1) DW_PICK(__nv_bfloat16, 7, 2)
  }
#undef DW_PICK
  return nullptr;
}

KernelFn kernel_for(int pass, int dtype, int K, int S) {
  if (pass == DWCONV_PASS_FWD) return pick<FwdK>(dtype, K, S);
  if (pass == DWCONV_PASS_BWD_DATA) return pick<BdK>(dtype, K, S);
  return pick<BfK>(dtype, K, S);
}

int tile_rows(int pass, int K, int S) {
  if (pass == DWCONV_PASS_BWD_DATA) return (K == 7) ? 4 : 8;
  return (K == 7) ? 4 : ((S == 1) ? 8 : 4);
}

uint32_t round128(uint64_t b) { return (uint32_t)((b + 127) & ~uint64_t(127)); }

int64_t gcd64(int64_t a, int64_t b) {
  while (b) { int64_t t = a % b; a = b; b = t; }
  return a;
}

int stage_budget() {
  static int kb = [] {
    const char* e = std::getenv("DWCONV_STAGE_KB");
    int v = e ? std::atoi(e) : 0;
    return (v >= 8 && v <= 110) ? v : 48;
  }();
  return kb * 1024;
}

int occupancy(KernelFn fn, int smem) {
  static std::mutex mu;
  static bool attr_set[64] = {};
  static KernelFn fns[64] = {};
  {
    std::lock_guard<std::mutex> lk(mu);
    int slot = -1;
    for (int i = 0; i < 64; ++i) {
      if (fns[i] == fn) { slot = i; break; }
      if (!fns[i]) { fns[i] = fn; slot = i; break; }
    }
    if (slot >= 0 && !attr_set[slot]) {
      int dev = 0;
      cudaGetDevice(&dev);
      int optin = 0;
      cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
      cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, optin);
      attr_set[slot] = true;
    }
  }
  int blocks = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, fn, kThreads, smem) != cudaSuccess) return 0;
  return blocks;
}

int ilog2_ceil(int64_t v) {
  int l = 0;
  while ((1ll << l) < v) ++l;
  return l;
}

}  // namespace

bool plan_nchw(const Geom& g, int pass, int num_sms, int max_smem_optin, ChunkPlan* p) {
  if (g.layout != DWCONV_NCHW) return false;
  const int K = g.kh;
  if (g.kw != K || (K != 3 && K != 5 && K != 7)) return false;
  const int S = g.sh;
  if (g.sw != S || (S != 1 && S != 2)) return false;
  if (g.ph != (K - 1) / 2 || g.pw != (K - 1) / 2) return false;
  if (g.m < 1 || g.m > 8) return false;
  if (g.H > 32767 || g.W > 32767 || g.Ho * g.Wo * (int64_t)g.m > (1 << 24)) return false;
  if (g.N * g.C > (int64_t)1 << 40) return false;
  *p = ChunkPlan{};
  p->threads = kThreads;
  const int64_t eb = (g.dtype == DWCONV_F32) ? 4 : 2;
  const int budget = stage_budget();
  const int R = tile_rows(pass, K, S);
  const int64_t Q = g.N * g.C;
  const int m = g.m;
  const int64_t x_plane = g.H * g.W * eb;
  const int64_t y_plane = (int64_t)m * g.Ho * g.Wo * eb;  // the m output planes of one input plane
  const int PAD = (K - 1) / 2;
  KernelFn fn = kernel_for(pass, g.dtype, K, S);
  if (!fn) return false;

  if (pass == DWCONV_PASS_FWD || pass == DWCONV_PASS_BWD_DATA) {
    const bool fwd = pass == DWCONV_PASS_FWD;
    const int64_t in_plane = fwd ? x_plane : y_plane;
    const int64_t out_plane = fwd ? y_plane : x_plane;
    const int64_t per = in_plane + out_plane;
    const int out_rows_total = fwd ? (int)g.Ho : (int)g.H;
    if (per <= budget) {
      int64_t P = budget / per;
      const int64_t a1 = 16 / gcd64(in_plane, 16), a2 = 16 / gcd64(out_plane, 16);
      const int64_t al = a1 / gcd64(a1, a2) * a2;
      const int64_t want_chunks = (int64_t)num_sms * 2 * 4;  // ~4 chunks per resident CTA
      const int64_t p_bal = (Q + want_chunks - 1) / want_chunks;
      const int64_t p_min = std::max<int64_t>(1, (8 * 1024) / per);
      P = std::min(P, std::max(p_bal, p_min));
      if (P >= al) P = P / al * al;
      else if (al * per <= 2 * budget) P = al;
      P = std::max<int64_t>(1, std::min(P, Q));
      p->P = (int)P;
      p->nbands = 1;
      p->band_rows = out_rows_total;
      p->nchunks = (Q + P - 1) / P;
      p->in_bytes = round128(P * in_plane);
      p->out_bytes = round128(P * out_plane);
    } else {
      // band mode: BR output rows (multiple of R); input rows needed per band
      auto in_rows = [&](int br) -> int64_t {
        if (fwd) return std::min<int64_t>(g.H, (int64_t)(br - 1) * S + K);
        return std::min<int64_t>(g.Ho, (br + K - 1 + S - 1) / S + 1);
      };
      auto bytes = [&](int br) -> int64_t {
        if (fwd) return in_rows(br) * g.W * eb + (int64_t)m * br * g.Wo * eb;
        return (int64_t)m * in_rows(br) * g.Wo * eb + (int64_t)br * g.W * eb;
      };
      int br = R;
      if (bytes(br) > budget) return false;
      while (br + R <= out_rows_total && bytes(br + R) <= budget) br += R;
      const int nb = (out_rows_total + br - 1) / br;
      int br2 = (out_rows_total + nb - 1) / nb;
      br2 = (br2 + R - 1) / R * R;
      p->P = 1;
      p->nbands = (out_rows_total + br2 - 1) / br2;
      p->band_rows = br2;
      p->nchunks = Q * p->nbands;
      if (fwd) {
        p->in_bytes = round128(in_rows(br2) * g.W * eb);
        p->out_bytes = round128((int64_t)m * br2 * g.Wo * eb);
      } else {
        p->in_bytes = round128((int64_t)m * in_rows(br2) * g.Wo * eb);
        p->out_bytes = round128((int64_t)br2 * g.W * eb);
      }
    }
    p->smem_bytes = 128 + 2 * (int)(p->in_bytes + p->out_bytes);
    if (p->smem_bytes > max_smem_optin) return false;
    const int occ = occupancy(fn, p->smem_bytes);
    if (occ < 1) return false;
    p->grid = (int)std::min<int64_t>(p->nchunks, (int64_t)occ * num_sms);
    (void)PAD;
    return true;
  }

  // ---------------- bwd_filter
  const int64_t per = x_plane + y_plane;
  int P = 1;
  int nb = 1, br = (int)g.Ho;
  if (kThreads % m != 0) return false;  // thread groups need m | 256 (m in {1,2,4,8})
  if (per <= budget) {
    while (2 * P * per <= budget && 2 * P * m <= kThreads && 2 * P <= g.C) P *= 2;
    // keep enough channel groups x slices to fill the machine
    while (P > 1 && ((g.C + P - 1) / P) * std::min<int64_t>(g.N, 128) < (int64_t)num_sms * 2) P /= 2;
  } else {
    auto x_rows = [&](int b) { return std::min<int64_t>(g.H, (int64_t)(b - 1) * S + K); };
    auto bytes = [&](int b) { return x_rows(b) * g.W * eb + (int64_t)m * b * g.Wo * eb; };
    br = R;
    if (bytes(br) > budget) return false;
    while (br + R <= g.Ho && bytes(br + R) <= budget) br += R;
    nb = (int)((g.Ho + br - 1) / br);
    br = (int)((g.Ho + nb - 1) / nb);
    br = (br + R - 1) / R * R;
    nb = (int)((g.Ho + br - 1) / br);
  }
  p->P = P;
  p->nbands = nb;
  p->band_rows = br;
  p->groups = (int)((g.C + P - 1) / P);
  p->tpg = kThreads / (P * m);
  if (nb == 1) {
    p->in_bytes = round128(P * x_plane);
    p->in2_bytes = round128(P * y_plane);
  } else {
    p->in_bytes = round128(std::min<int64_t>(g.H, (int64_t)(br - 1) * S + K) * g.W * eb);
    p->in2_bytes = round128((int64_t)m * br * g.Wo * eb);
  }
  p->out_bytes = 0;
  p->smem_bytes = 128 + 2 * (int)(p->in_bytes + p->in2_bytes);
  const int KK = K * K;
  // the cross-warp reduction reuses stage memory: needs (256/32) * KK floats
  p->smem_bytes = std::max<int>(p->smem_bytes, 128 + (kThreads / 32) * KK * 4);
  if (p->smem_bytes > max_smem_optin) return false;
  const int occ = occupancy(fn, p->smem_bytes);
  if (occ < 1) return false;
  // batch slices: fill ~2 waves, keep <= 32 chunks per CTA (running-sum chain) and <= 128 slices
  const int64_t N = std::max<int64_t>(g.N, 1);
  int64_t ns = ((int64_t)num_sms * occ * 2 + p->groups - 1) / p->groups;
  ns = std::max<int64_t>(ns, (N * nb + 31) / 32);
  ns = std::min<int64_t>(ns, std::min<int64_t>(N, 128));
  ns = std::max<int64_t>(ns, 1);
  int64_t nps = (N + ns - 1) / ns;
  ns = (N + nps - 1) / nps;
  p->nslices = (int)ns;
  p->n_per_slice = (int)nps;
  p->grid = (int)(p->groups * ns);
  p->nchunks = (int64_t)p->grid;
  const int nsb = (br + R - 1) / R;
  const int64_t tiles_per_thread = ((int64_t)nsb * g.Wo + p->tpg - 1) / p->tpg;
  p->max_chain = (int)(tiles_per_thread * R + nps * nb + ilog2_ceil(p->tpg) + 2 * ilog2_ceil(ns) + 1);
  const size_t tick = ((size_t)p->groups * 4 + 15) / 16 * 16;
  p->ws_bytes = tick + (size_t)ns * g.C * m * KK * 4;
  return ns <= 128;
}

static NArgs base_args(const Geom& g, const ChunkPlan& p, int pass) {
  NArgs a{};
  a.N = g.N; a.C = g.C; a.Q = g.N * g.C;
  a.m = g.m; a.Co = (int)(g.C * g.m);
  a.H = (int)g.H; a.W = (int)g.W; a.Ho = (int)g.Ho; a.Wo = (int)g.Wo;
  a.P = p.P; a.nbands = p.nbands; a.BR = p.band_rows;
  const int R = tile_rows(pass, g.kh, g.sh);
  a.nsb = (p.band_rows + R - 1) / R;
  a.nchunks = p.nchunks;
  a.in_bytes = p.in_bytes; a.in2_bytes = p.in2_bytes; a.out_bytes = p.out_bytes;
  a.groups = p.groups; a.nslices = p.nslices; a.nps = p.n_per_slice; a.tpg = p.tpg;
  a.div_wo = make_fastdiv((uint32_t)g.Wo);
  a.div_nsb = make_fastdiv((uint32_t)a.nsb);
  a.div_m = make_fastdiv((uint32_t)g.m);
  a.div_ncb = make_fastdiv((uint32_t)((g.W + g.sw - 1) / g.sw));
  return a;
}

cudaError_t launch_nchw_fwd(const Geom& g, const ChunkPlan& p, const void* x, const void* w, void* y,
                            cudaStream_t st) {
  NArgs a = base_args(g, p, DWCONV_PASS_FWD);
  a.in = x; a.w = w; a.out = y;
  KernelFn fn = kernel_for(DWCONV_PASS_FWD, g.dtype, g.kh, g.sh);
  fn<<<p.grid, p.threads, p.smem_bytes, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_nchw_bwd_data(const Geom& g, const ChunkPlan& p, const void* dy, const void* w, void* dx,
                                 cudaStream_t st) {
  NArgs a = base_args(g, p, DWCONV_PASS_BWD_DATA);
  a.in = dy; a.w = w; a.out = dx;
  KernelFn fn = kernel_for(DWCONV_PASS_BWD_DATA, g.dtype, g.kh, g.sh);
  fn<<<p.grid, p.threads, p.smem_bytes, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_nchw_bwd_filter(const Geom& g, const ChunkPlan& p, const void* x, const void* dy, float* dw,
                                   void* ws, cudaStream_t st) {
  NArgs a = base_args(g, p, DWCONV_PASS_BWD_FILTER);
  a.in = x; a.in2 = dy; a.dw = dw;
  const size_t tick = ((size_t)p.groups * 4 + 15) / 16 * 16;
  a.ws_ticket = static_cast<unsigned*>(ws);
  a.ws_part = reinterpret_cast<float*>(static_cast<char*>(ws) + tick);
  KernelFn fn = kernel_for(DWCONV_PASS_BWD_FILTER, g.dtype, g.kh, g.sh);
  fn<<<p.grid, p.threads, p.smem_bytes, st>>>(a);
  return cudaGetLastError();
}

}  // namespace dwk
