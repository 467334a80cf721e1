// nchw_small.cu -- NCHW kernels for small square planes (W = H in {7, 14, 28}),
// 3x3, pad 1, stride 1, m = 1: the 28x28 / 14x14 / 7x7 MobileNet layers.
//
//   fwd       y[n,c,oh,ow] = sum_{i,j} w[c,i,j] * x[n,c,oh-1+i,ow-1+j]      (Eq. 3)
//   bwd_data  dx = the same stencil over dy with w rotated by 180 degrees   (adjoint at s = 1, reading R9)
//   bwd_filter dw[c,i,j] = sum_{n,oh,ow} x[n,c,oh-1+i,ow-1+j] * dy[n,c,oh,ow] (Eq. 4 diagonal; R5)
//
// The chunk kernels (nchw_fwd.cu ...) spend most of their instructions on
// per-strip index arithmetic when a plane is only 7-28 wide.  Here the unit of
// work is a WARP TASK of 4 consecutive planes (one contiguous range of x, and of
// dy for bwd_filter): lane l of the warp owns plane l / 7 and the V = W / 7
// columns [V*(l%7), V*(l%7)+V) of it (28 of 32 lanes busy), and walks all W rows
// with a 3-row sliding window, so a row costs 1 vector LDS + 2 halo LDS and
// 9*V FFMA.  Every warp is independent: lane 0 bulk-copies the warp's next
// tasks into a private ring of `ns` shared-memory slots (cp.async.bulk ->
// UBLKCP, one mbarrier per slot); there is no CTA-wide synchronisation in the
// loop.  fwd / bwd_data store straight from registers (STG.64/.128 along the
// row).  bwd_filter: CTA = (group of 4 channels, batch slice), warps split the
// slice's images; deterministic reduction: rows x V columns per lane (<= 28
// terms) -> per-image partials added to a running sum (<= 32 images per warp)
// -> the 7 lanes of a plane in order -> the warps in order -> per-slice partial
// in the workspace -> last CTA of the group (integer ticket) sums the slices
// pairwise in slice order and re-zeroes the workspace (as nchw_bwd_filter.cu).
#include "kernels.h"
#include "nchw_common.cuh"

namespace dwk {
namespace small {

using nchw::VecIO;

struct SArgs {
  const void* in;    // fwd: x, bwd_data: dy, bwd_filter: x
  const void* in2;   // bwd_filter: dy
  void* out;         // fwd: y, bwd_data: dx
  const void* w;
  float* dw;
  float* ws_part;
  unsigned* ws_ticket;
  int64_t ntasks;    // fwd / bwd_data: Q / 4
  int C, N;
  int ns;            // ring slots per warp
  uint32_t slot_bytes;
  int groups, nslices, nps;  // bwd_filter
  // band bwd_filter (band_bf_kernel)
  int H, W, Ho, Wo, nbands, cpg;  // cpg: channels per group (one per warp)
  int early_pdl;                   // trigger the dependent launch once the ring is primed
};

// one row of the window: the lane's V columns and the two halo columns
template <class T, int W, int V>
__device__ __forceinline__ void load_row(const T* row, int c0, bool lft, bool rgt, float* xv) {
  float v[V];
  VecIO<T, V>::load(row + c0, v);
#pragma unroll
  for (int u = 0; u < V; ++u) xv[1 + u] = v[u];
  xv[0] = lft ? Elem<T>::load(row + c0 - 1) : 0.f;
  xv[V + 1] = rgt ? Elem<T>::load(row + c0 + V) : 0.f;
}

// the same row with the halo columns taken from the neighbouring lanes (warp
// shuffles; every lane of the warp must call it)
template <class T, int W, int V>
__device__ __forceinline__ void load_row_shfl(const T* row, int c0, bool lft, bool rgt, float* xv) {
  float v[V];
  VecIO<T, V>::load(row + c0, v);
#pragma unroll
  for (int u = 0; u < V; ++u) xv[1 + u] = v[u];
  const float l = __shfl_up_sync(0xffffffffu, v[V - 1], 1), r = __shfl_down_sync(0xffffffffu, v[0], 1);
  xv[0] = lft ? l : 0.f;
  xv[V + 1] = rgt ? r : 0.f;
}

// MODE 0 fwd, 1 bwd_data (rotated kernel)
template <class T, int W, int MODE>
__global__ void __launch_bounds__(256) small_fd_kernel(const SArgs a) {
  constexpr int V = W / 7, HW = W * W;
  extern __shared__ __align__(128) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nwarps = blockDim.x >> 5;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem) + warp * 8;
  T* ring = reinterpret_cast<T*>(smem + 64 * nwarps + (size_t)warp * a.ns * a.slot_bytes);
  const int pl = min(lane / 7, 3), cg = (lane < 28) ? lane - (lane / 7) * 7 : 6;  // plane, column group
  const bool live = lane < 28;  // lanes 28-31 shadow lane 27 (shuffle partners only)
  const int c0 = cg * V;
  const T* __restrict__ in = static_cast<const T*>(a.in);
  T* __restrict__ out = static_cast<T*>(a.out);
  const T* __restrict__ wt = static_cast<const T*>(a.w);
  if (lane == 0) {
    for (int i = 0; i < a.ns; ++i) mbar_init(&bars[i], 1);
    fence_mbar_init();
  }
  __syncwarp();
  griddep_wait();
  const int64_t gw = (int64_t)blockIdx.x * nwarps + warp;
  const int64_t stride = (int64_t)gridDim.x * nwarps;
  const uint32_t task_bytes = 4u * HW * (uint32_t)sizeof(T);
  auto slot = [&](int s) { return ring + (size_t)s * (a.slot_bytes / sizeof(T)); };
  auto issue = [&](int64_t t, int s) {
    if (lane == 0 && t < a.ntasks) {
      mbar_arrive_expect_tx(&bars[s], task_bytes);
      bulk_g2s(slot(s), in + t * 4 * HW, task_bytes, &bars[s]);
    }
  };
  for (int i = 0; i < a.ns; ++i) issue(gw + i * stride, i);
  if (a.early_pdl) griddep_launch_dependents();  // grid is one wave: let the next kernel's CTAs queue
  int s = 0;
  uint32_t ph = 0;
  for (int64_t t = gw; t < a.ntasks; t += stride) {
    const int64_t q = t * 4 + pl;  // plane
    const int c = (int)(q % a.C);
    float wr[9];
#pragma unroll
    for (int k = 0; k < 9; ++k) wr[k] = Elem<T>::ldg(wt + (int64_t)c * 9 + (MODE == 1 ? 8 - k : k));
    mbar_wait(&bars[s], ph);
    {
      const T* pln = slot(s) + pl * HW;
      const bool lft = c0 > 0, rgt = c0 + V < W;
      float xw[3][V + 2];
#pragma unroll
      for (int u = 0; u < V + 2; ++u) xw[0][u] = 0.f;  // row -1
      load_row_shfl<T, W, V>(pln, c0, lft, rgt, xw[1]);
      T* po = out + q * HW + c0;
#pragma unroll
      for (int r = 0; r < W; ++r) {
        if (r + 1 < W) load_row_shfl<T, W, V>(pln + (r + 1) * W, c0, lft, rgt, xw[2]);
        else
#pragma unroll
          for (int u = 0; u < V + 2; ++u) xw[2][u] = 0.f;  // row W
        float o[V];
#pragma unroll
        for (int u = 0; u < V; ++u) {
          float acc = wr[0] * xw[0][u];
#pragma unroll
          for (int k = 1; k < 9; ++k) acc = fmaf(wr[k], xw[k / 3][u + k % 3], acc);
          o[u] = acc;
        }
        if (live) VecIO<T, V>::store(po + r * W, o);
#pragma unroll
        for (int u = 0; u < V + 2; ++u) { xw[0][u] = xw[1][u]; xw[1][u] = xw[2][u]; }
      }
    }
    __syncwarp();
    issue(t + a.ns * stride, s);  // the slot is free: every lane is past it
    if (++s == a.ns) { s = 0; ph ^= 1; }
  }
  if (!a.early_pdl) griddep_launch_dependents();
}

// FUSED: also dx = the forward stencil over the staged dy with the rotated kernel
// (the fused backward): x and dy leave HBM once for both gradients.
template <class T, int W, bool FUSED = false>
__global__ void __launch_bounds__(256) small_bf_kernel(const SArgs a) {
  constexpr int V = W / 7, HW = W * W;
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ unsigned s_last;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nwarps = blockDim.x >> 5;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem) + warp * 8;
  T* ring = reinterpret_cast<T*>(smem + 64 * nwarps + (size_t)warp * a.ns * a.slot_bytes);
  const int pl = min(lane / 7, 3), cg = (lane < 28) ? lane - (lane / 7) * 7 : 6;
  const bool live = lane < 28;  // lanes 28-31 shadow lane 27 (shuffle partners only)
  const int c0 = cg * V;
  const int g = blockIdx.x % a.groups, sl = blockIdx.x / a.groups;
  const int cb = g * 4;  // first channel of the group
  const int n0 = sl * a.nps, n1 = min(a.N, n0 + a.nps);
  const T* __restrict__ x = static_cast<const T*>(a.in);
  const T* __restrict__ dy = static_cast<const T*>(a.in2);
  if (lane == 0) {
    for (int i = 0; i < a.ns; ++i) mbar_init(&bars[i], 1);
    fence_mbar_init();
  }
  __syncwarp();
  griddep_wait();
  const uint32_t task_bytes = 4u * HW * (uint32_t)sizeof(T);
  auto slot = [&](int s) { return ring + (size_t)s * (a.slot_bytes / sizeof(T)); };
  auto issue = [&](int n, int s) {
    if (lane == 0 && n < n1) {
      const int64_t off = ((int64_t)n * a.C + cb) * HW;
      mbar_arrive_expect_tx(&bars[s], 2 * task_bytes);
      bulk_g2s(slot(s), x + off, task_bytes, &bars[s]);
      bulk_g2s(slot(s) + 4 * HW, dy + off, task_bytes, &bars[s]);
    }
  };
  for (int i = 0; i < a.ns; ++i) issue(n0 + warp + i * nwarps, i);
  if (a.early_pdl) griddep_launch_dependents();  // grid is one wave: let the next kernel's CTAs queue
  float wf[FUSED ? 9 : 1];  // rotated kernel of this lane's channel (fused dx)
  if constexpr (FUSED) {
    const T* __restrict__ wt = static_cast<const T*>(a.w);
#pragma unroll
    for (int k = 0; k < 9; ++k) wf[k] = Elem<T>::ldg(wt + (int64_t)(cb + (live ? pl : 0)) * 9 + 8 - k);
  }
  T* __restrict__ dxo = static_cast<T*>(a.out);
  float run[9];
#pragma unroll
  for (int k = 0; k < 9; ++k) run[k] = 0.f;
  int s = 0;
  uint32_t ph = 0;
  for (int n = n0 + warp; n < n1; n += nwarps) {
    mbar_wait(&bars[s], ph);
    {
      const T* pln = slot(s) + pl * HW;
      const T* pd = slot(s) + 4 * HW + pl * HW;
      const bool lft = c0 > 0, rgt = c0 + V < W;
      float xw[3][V + 2];
#pragma unroll
      for (int u = 0; u < V + 2; ++u) xw[0][u] = 0.f;
      load_row_shfl<T, W, V>(pln, c0, lft, rgt, xw[1]);
      float loc[9];
      float dw3[FUSED ? 3 : 1][V + 2];  // dy window (fused dx)
      T* po = dxo + ((int64_t)n * a.C + cb + pl) * HW + c0;
      if constexpr (FUSED) {
#pragma unroll
        for (int u = 0; u < V + 2; ++u) dw3[0][u] = 0.f;
        load_row_shfl<T, W, V>(pd, c0, lft, rgt, dw3[1]);
      }
#pragma unroll
      for (int r = 0; r < W; ++r) {
        if (r + 1 < W) load_row_shfl<T, W, V>(pln + (r + 1) * W, c0, lft, rgt, xw[2]);
        else
#pragma unroll
          for (int u = 0; u < V + 2; ++u) xw[2][u] = 0.f;
        float d[V];
        if constexpr (FUSED) {
          if (r + 1 < W) load_row_shfl<T, W, V>(pd + (r + 1) * W, c0, lft, rgt, dw3[2]);
          else
#pragma unroll
            for (int u = 0; u < V + 2; ++u) dw3[2][u] = 0.f;
          float o[V];
#pragma unroll
          for (int u = 0; u < V; ++u) {
            d[u] = dw3[1][u + 1];
            float acc = wf[0] * dw3[0][u];
#pragma unroll
            for (int k = 1; k < 9; ++k) acc = fmaf(wf[k], dw3[k / 3][u + k % 3], acc);
            o[u] = acc;
          }
          if (live) VecIO<T, V>::store(po + r * W, o);
#pragma unroll
          for (int u = 0; u < V + 2; ++u) { dw3[0][u] = dw3[1][u]; dw3[1][u] = dw3[2][u]; }
        } else {
          VecIO<T, V>::load(pd + r * W + c0, d);
        }
#pragma unroll
        for (int k = 0; k < 9; ++k)
#pragma unroll
          for (int u = 0; u < V; ++u)
            loc[k] = (r == 0 && u == 0) ? xw[k / 3][u + k % 3] * d[u] : fmaf(xw[k / 3][u + k % 3], d[u], loc[k]);
#pragma unroll
        for (int u = 0; u < V + 2; ++u) { xw[0][u] = xw[1][u]; xw[1][u] = xw[2][u]; }
      }
      if (live) {
#pragma unroll
        for (int k = 0; k < 9; ++k) run[k] += loc[k];
      }
    }
    __syncwarp();
    issue(n + a.ns * nwarps, s);
    if (++s == a.ns) { s = 0; ph ^= 1; }
  }
  if (!a.early_pdl) griddep_launch_dependents();
  // ---- lanes of a plane in order, then warps in order -> the slice partial
  __syncthreads();
  float* red = reinterpret_cast<float*>(smem + 64 * nwarps);  // [warp][lane][9]; the ring is idle now
  if (live) {
#pragma unroll
    for (int k = 0; k < 9; ++k) red[(warp * 32 + lane) * 9 + k] = run[k];
  }
  __syncthreads();
  float* part = a.ws_part + (int64_t)sl * a.C * 9;
  for (int e = threadIdx.x; e < 4 * 9; e += blockDim.x) {
    const int p = e / 9, k = e - p * 9;
    float tot = 0.f;
    for (int wv = 0; wv < nwarps; ++wv) {
      float v = red[(wv * 32 + p * 7) * 9 + k];
      for (int l = 1; l < 7; ++l) v += red[(wv * 32 + p * 7 + l) * 9 + k];
      tot = (wv == 0) ? v : tot + v;
    }
    part[(int64_t)(cb + p) * 9 + k] = tot;
  }
  __threadfence();
  __syncthreads();
  {
    const int ngrp = (a.nslices + 31) / 32;
    nchw::finalize_two_level(a.ws_part, a.ws_part + (int64_t)a.nslices * a.C * 9, a.ws_ticket,
                             a.ws_ticket + (int64_t)a.groups * ngrp, g, sl, a.nslices, (int64_t)a.C * 9,
                             (int64_t)cb * 9, 36, a.dw, &s_last);
  }
}

// ------------------------------------------------------------ band bwd_filter
// Large planes (output width Wo = 28 V, V in {1,2,4}; the 112/56/28 MobileNet
// layers at stride 1 and 2): warp task = (image, band of R dy rows) of ONE
// channel -- x rows [R*b*S - 1, (R*b + R - 1)*S + 1] and the R dy rows are two
// contiguous ranges, bulk-copied by lane 0 into the warp's ring slot.  Lane l
// (< 28) owns dy columns [V*l, V*l + V) and walks the band's rows with a sliding
// x window (stride 1: one new x row per dy row, stride 2: two), 9*V FFMA per
// dy row.  CTA = (group of `cpg` channels, one per warp; batch slice).
// Deterministic reduction: R*V terms per task -> running sum over the warp's
// tasks -> xor-shuffle tree over the 32 lanes -> per-slice partial -> ticketed
// pairwise finalize over slices (as above).
template <class T, int S, int V, int R, int PPW = 1>
__global__ void __launch_bounds__(256) band_bf_kernel(const SArgs a) {
  // PPW planes (consecutive channels) per warp: lanes [16p, 16p + Wo/V) own plane p
  // when PPW = 2 (Wo = 14 V), lanes [0, 28) when PPW = 1 (Wo = 28 V)
  constexpr int NX = S * V;  // own x columns per lane (stride 2: + the left halo only)
  constexpr int LPP = 32 / PPW;
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ unsigned s_last;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nwarps = blockDim.x >> 5;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem) + warp * 8;
  T* ring = reinterpret_cast<T*>(smem + 64 * nwarps + (size_t)warp * a.ns * a.slot_bytes);
  const int g = blockIdx.x % a.groups, sl = blockIdx.x / a.groups;
  const int cw = g * a.cpg + warp * PPW;  // first channel of this warp
  const int pl = lane / LPP, li = lane - pl * LPP;
  const int c = cw + pl;                  // this lane's channel
  const int np_w = max(0, min(PPW, min(a.cpg - warp * PPW, a.C - cw)));  // live planes of the warp
  const bool wlive = np_w > 0;
  const int H = a.H, W = a.W, Ho = a.Ho, Wo = a.Wo;
  const bool live = pl < np_w && li * V < Wo;
  const int n0 = sl * a.nps, n1 = min(a.N, n0 + a.nps);
  const int ntask = (n1 - n0) * a.nbands;
  const T* __restrict__ x = static_cast<const T*>(a.in);
  const T* __restrict__ dy = static_cast<const T*>(a.in2);
  const uint32_t xcap = (uint32_t)(((R - 1) * S + 3) * W * sizeof(T) + 15) & ~15u;  // x part of a plane's slot
  const uint32_t dcap = (uint32_t)(R * Wo * sizeof(T) + 15) & ~15u;
  if (lane == 0) {
    for (int i = 0; i < a.ns; ++i) mbar_init(&bars[i], 1);
    fence_mbar_init();
  }
  __syncwarp();
  griddep_wait();
  auto slot = [&](int s) { return reinterpret_cast<unsigned char*>(ring) + (size_t)s * a.slot_bytes; };
  auto rows_of = [&](int t, int* n, int* r0, int* r1, int* lo, int* hi) {
    const int nn = t / a.nbands, b = t - nn * a.nbands;
    *n = n0 + nn;
    *r0 = b * R;
    *r1 = min(*r0 + R, Ho);
    *lo = max(0, *r0 * S - 1);
    *hi = min(H, (*r1 - 1) * S + 2);
  };
  auto issue = [&](int t, int s) {
    if (lane == 0 && wlive && t < ntask) {
      int n, r0, r1, lo, hi;
      rows_of(t, &n, &r0, &r1, &lo, &hi);
      const uint32_t xb = (uint32_t)((hi - lo) * W * sizeof(T)), db = (uint32_t)((r1 - r0) * Wo * sizeof(T));
      mbar_arrive_expect_tx(&bars[s], (uint32_t)np_w * (xb + db));
      for (int p = 0; p < np_w; ++p) {
        unsigned char* sp = slot(s) + (size_t)p * (xcap + dcap);
        bulk_g2s(sp, x + (((int64_t)n * a.C + cw + p) * H + lo) * W, xb, &bars[s]);
        bulk_g2s(sp + xcap, dy + (((int64_t)n * a.C + cw + p) * Ho + r0) * Wo, db, &bars[s]);
      }
    }
  };
  for (int i = 0; i < a.ns; ++i) issue(i, i);
  if (a.early_pdl) griddep_launch_dependents();  // grid is one wave: let the next kernel's CTAs queue
  const int c0 = li * V;
  float run[9];
#pragma unroll
  for (int k = 0; k < 9; ++k) run[k] = 0.f;
  int s = 0;
  uint32_t ph = 0;
  for (int t = 0; t < (wlive ? ntask : 0); ++t) {
    mbar_wait(&bars[s], ph);
    if (live) {
      int n, r0, r1, lo, hi;
      rows_of(t, &n, &r0, &r1, &lo, &hi);
      const unsigned char* sp = slot(s) + (size_t)pl * (xcap + dcap);
      const T* xs = reinterpret_cast<const T*>(sp) - (int64_t)lo * W;  // x row ih at xs + ih*W (ih in [lo,hi))
      const T* ds = reinterpret_cast<const T*>(sp + xcap) - (int64_t)r0 * Wo;
      // window rows: x row ih = r*S - 1 + i, i = 0..2; columns S*c0 - 1 .. S*c0 + NX (+1 at S = 1)
      float xw[3][NX + 2];
      auto ldx = [&](int ih, float* v) {
        if (ih >= lo && ih < hi) {
          const T* row = xs + (int64_t)ih * W;
          float o[NX];
          VecIO<T, NX>::load(row + S * c0, o);
#pragma unroll
          for (int u = 0; u < NX; ++u) v[1 + u] = o[u];
          v[0] = (c0 > 0) ? Elem<T>::load(row + S * c0 - 1) : 0.f;
          v[NX + 1] = (S == 1 && c0 + V < W) ? Elem<T>::load(row + c0 + V) : 0.f;
        } else {
#pragma unroll
          for (int u = 0; u < NX + 2; ++u) v[u] = 0.f;
        }
      };
#pragma unroll
      for (int i = 0; i < 3 - S; ++i) ldx(r0 * S - 1 + i, xw[i]);
      float loc[9];
#pragma unroll
      for (int k = 0; k < 9; ++k) loc[k] = 0.f;
#pragma unroll
      for (int rr = 0; rr < R; ++rr) {
        const int r = r0 + rr;
        if (r < r1) {
#pragma unroll
          for (int i = 3 - S; i < 3; ++i) ldx(r * S - 1 + i, xw[i]);
          float d[V];
          VecIO<T, V>::load(ds + (int64_t)r * Wo + c0, d);
#pragma unroll
          for (int k = 0; k < 9; ++k)
#pragma unroll
            for (int u = 0; u < V; ++u) loc[k] = fmaf(xw[k / 3][S * u + k % 3], d[u], loc[k]);
#pragma unroll
          for (int i = 0; i < 3 - S; ++i)
#pragma unroll
            for (int u = 0; u < NX + 2; ++u) xw[i][u] = xw[i + S][u];
        }
      }
#pragma unroll
      for (int k = 0; k < 9; ++k) run[k] += loc[k];
    }
    __syncwarp();
    issue(t + a.ns, s);
    if (++s == a.ns) { s = 0; ph ^= 1; }
  }
  if (!a.early_pdl) griddep_launch_dependents();
  // ---- lanes: fixed xor tree (lanes >= 28 hold zeros) -> the warp's channel partial
#pragma unroll
  for (int k = 0; k < 9; ++k) {
#pragma unroll
    for (int off = LPP / 2; off > 0; off >>= 1) run[k] += __shfl_xor_sync(0xffffffffu, run[k], off);
  }
  float* part = a.ws_part + (int64_t)sl * a.C * 9;
  if (pl < np_w && li < 9) {
    float v = run[0];
#pragma unroll
    for (int k = 1; k < 9; ++k) v = (li == k) ? run[k] : v;
    part[(int64_t)c * 9 + li] = v;
  }
  __threadfence();
  __syncthreads();
  {
    const int ngrp = (a.nslices + 31) / 32;
    nchw::finalize_two_level(a.ws_part, a.ws_part + (int64_t)a.nslices * a.C * 9, a.ws_ticket,
                             a.ws_ticket + (int64_t)a.groups * ngrp, g, sl, a.nslices, (int64_t)a.C * 9,
                             (int64_t)g * a.cpg * 9, min(a.cpg, a.C - g * a.cpg) * 9, a.dw, &s_last);
  }
}

// ------------------------------------------------------------ stride 2
// Input planes W x W (W in {14, 28}), output Wo = W / 2 = 7 V.  Lane (plane l/7,
// column group) owns V output columns = 2V input columns + the left halo;
// each output row consumes two new input rows (the window keeps row 2r-1).
template <class T, int V>
__device__ __forceinline__ void load_row2(const T* row, int c0, float* xv) {  // x[2c0-1 .. 2c0+2V-1]
  float v[2 * V];
  VecIO<T, 2 * V>::load(row + 2 * c0, v);
#pragma unroll
  for (int u = 0; u < 2 * V; ++u) xv[1 + u] = v[u];
  // the left halo is the previous lane's last column (every lane of the warp calls this)
  const float l = __shfl_up_sync(0xffffffffu, v[2 * V - 1], 1);
  xv[0] = (c0 > 0) ? l : 0.f;
}

// bf16 plane pairs (stride 1): a warp task is 8 planes; lane (p, column group)
// owns two planes and runs their stencils together with packed FFMA2 (lanes of
// the float2 = the two planes), halving the FMA instructions per output of the
// bf16 kernels, which are instruction-bound.
//
// Which two planes, and where they sit in shared memory, is chosen against bank
// conflicts (ncu, W = 14: 74% of the shared-load wavefronts were conflicts with
// planes p and p + 4 packed back to back -- the four planes one load touches sat
// 2 banks apart).  W = 7: planes p, p + 4, packed (already conflict-free).
// W = 14 / 28: ADJACENT planes 2p, 2p + 1 (pair p); W = 14 stages each pair by its
// own bulk copy at a pitch of 400 elements (200 words = 8 banks, so the four
// pairs' rows land on disjoint banks: one wavefront per load instead of four);
// W = 28 keeps one copy (a pair is 784 words = 16 banks apart).
template <int W> struct PairLayout {
  static constexpr int HW = W * W;
  static constexpr bool ADJ = W != 7;                  // planes (2p, 2p+1) instead of (p, p+4)
  static constexpr int QP = (W == 14) ? 400 : 2 * HW;  // pair pitch in elements (ADJ)
  static constexpr bool SPLIT = ADJ && QP != 2 * HW;   // one bulk copy per pair
  static constexpr int REGION = ADJ ? 4 * QP : 8 * HW;  // elements of one 8-plane task in the slot
  __host__ __device__ static constexpr int plane_a(int p) { return ADJ ? 2 * p : p; }
  __host__ __device__ static constexpr int plane_b(int p) { return ADJ ? 2 * p + 1 : p + 4; }
  __host__ __device__ static constexpr int off(int plane) { return ADJ ? (plane >> 1) * QP + (plane & 1) * HW : plane * HW; }
};

// stage the 8 planes starting at src (contiguous in global) into a slot region
template <int W>
__device__ __forceinline__ void stage_pairs(__nv_bfloat16* dst, const __nv_bfloat16* src, uint64_t* bar) {
  using L = PairLayout<W>;
  if constexpr (L::SPLIT) {
#pragma unroll
    for (int q = 0; q < 4; ++q) bulk_g2s(dst + q * L::QP, src + q * 2 * L::HW, 2u * L::HW * 2u, bar);
  } else {
    bulk_g2s(dst, src, 8u * L::HW * 2u, bar);
  }
}
template <int W, int MODE>
__global__ void __launch_bounds__(256) small_fd_pair_kernel(const SArgs a) {
  using T = __nv_bfloat16;
  constexpr int V = W / 7, HW = W * W;
  extern __shared__ __align__(128) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nwarps = blockDim.x >> 5;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem) + warp * 8;
  T* ring = reinterpret_cast<T*>(smem + 64 * nwarps + (size_t)warp * a.ns * a.slot_bytes);
  const int pl = min(lane / 7, 3), cg = (lane < 28) ? lane - (lane / 7) * 7 : 6;  // lanes 28-31 shadow lane 27
  const bool live = lane < 28;
  const int c0 = cg * V;
  const T* __restrict__ in = static_cast<const T*>(a.in);
  T* __restrict__ out = static_cast<T*>(a.out);
  const T* __restrict__ wt = static_cast<const T*>(a.w);
  if (lane == 0) {
    for (int i = 0; i < a.ns; ++i) mbar_init(&bars[i], 1);
    fence_mbar_init();
  }
  __syncwarp();
  griddep_wait();
  const int64_t gw = (int64_t)blockIdx.x * nwarps + warp;
  const int64_t stride = (int64_t)gridDim.x * nwarps;
  const uint32_t task_bytes = 8u * HW * (uint32_t)sizeof(T);
  auto slot = [&](int s) { return ring + (size_t)s * (a.slot_bytes / sizeof(T)); };
  auto issue = [&](int64_t t, int s) {
    if (lane == 0 && t < a.ntasks) {
      mbar_arrive_expect_tx(&bars[s], task_bytes);
      stage_pairs<W>(slot(s), in + t * 8 * HW, &bars[s]);
    }
  };
  for (int i = 0; i < a.ns; ++i) issue(gw + i * stride, i);
  if (a.early_pdl) griddep_launch_dependents();
  const bool lft = c0 > 0, rgt = c0 + V < W;
  // the halo columns come from the neighbouring lanes of the same plane (warp
  // shuffles instead of two more shared-memory loads per plane and row)
  auto ldrow = [&](const T* ra, const T* rb, float2* xv) {  // .x plane A, .y plane B
    float va[V], vb[V];
    VecIO<T, V>::load(ra + c0, va);
    VecIO<T, V>::load(rb + c0, vb);
#pragma unroll
    for (int u = 0; u < V; ++u) xv[1 + u] = make_float2(va[u], vb[u]);
    const float la = __shfl_up_sync(0xffffffffu, va[V - 1], 1), lb = __shfl_up_sync(0xffffffffu, vb[V - 1], 1);
    const float ra2 = __shfl_down_sync(0xffffffffu, va[0], 1), rb2 = __shfl_down_sync(0xffffffffu, vb[0], 1);
    xv[0] = lft ? make_float2(la, lb) : make_float2(0.f, 0.f);
    xv[V + 1] = rgt ? make_float2(ra2, rb2) : make_float2(0.f, 0.f);
  };
  int s = 0;
  uint32_t ph = 0;
  using L = PairLayout<W>;
  for (int64_t t = gw; t < a.ntasks; t += stride) {
    const int64_t qa = t * 8 + L::plane_a(pl), qb = t * 8 + L::plane_b(pl);
    const int ca = (int)(qa % a.C), cb2 = (int)(qb % a.C);
    float2 w2[9];
#pragma unroll
    for (int k = 0; k < 9; ++k) {
      const int kk = (MODE == 1) ? 8 - k : k;
      w2[k] = make_float2(Elem<T>::ldg(wt + (int64_t)ca * 9 + kk), Elem<T>::ldg(wt + (int64_t)cb2 * 9 + kk));
    }
    mbar_wait(&bars[s], ph);
    {  // every lane runs the loop (shuffles); lanes 28-31 recompute lane 27's columns and store nothing
      const T* pa = slot(s) + L::off(L::plane_a(pl));
      const T* pb = slot(s) + L::off(L::plane_b(pl));
      float2 xw[3][V + 2];
#pragma unroll
      for (int u = 0; u < V + 2; ++u) xw[0][u] = make_float2(0.f, 0.f);
      ldrow(pa, pb, xw[1]);
      T* poa = out + qa * HW + c0;
      T* pob = out + qb * HW + c0;
#pragma unroll
      for (int r = 0; r < W; ++r) {
        if (r + 1 < W) ldrow(pa + (r + 1) * W, pb + (r + 1) * W, xw[2]);
        else
#pragma unroll
          for (int u = 0; u < V + 2; ++u) xw[2][u] = make_float2(0.f, 0.f);
        float oa[V], ob[V];
#pragma unroll
        for (int u = 0; u < V; ++u) {
          float2 acc = __fmul2_rn(w2[0], xw[0][u]);
#pragma unroll
          for (int k = 1; k < 9; ++k) acc = __ffma2_rn(w2[k], xw[k / 3][u + k % 3], acc);
          oa[u] = acc.x;
          ob[u] = acc.y;
        }
        if (live) {
          VecIO<T, V>::store(poa + r * W, oa);
          VecIO<T, V>::store(pob + r * W, ob);
        }
#pragma unroll
        for (int u = 0; u < V + 2; ++u) { xw[0][u] = xw[1][u]; xw[1][u] = xw[2][u]; }
      }
    }
    __syncwarp();
    issue(t + a.ns * stride, s);
    if (++s == a.ns) { s = 0; ph ^= 1; }
  }
  if (!a.early_pdl) griddep_launch_dependents();
}

// bf16 plane-pair bwd_filter (stride 1): CTA = (group of 8 channels, batch
// slice); lane (p, column group) owns channels cb + p and cb + p + 4 and
// accumulates both with FFMA2 (float2 lanes = the two channels).  Reduction as
// small_bf_kernel, per channel.
template <int W>
__global__ void __launch_bounds__(256) small_bf_pair_kernel(const SArgs a) {
  using T = __nv_bfloat16;
  constexpr int V = W / 7, HW = W * W;
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ unsigned s_last;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nwarps = blockDim.x >> 5;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem) + warp * 8;
  T* ring = reinterpret_cast<T*>(smem + 64 * nwarps + (size_t)warp * a.ns * a.slot_bytes);
  const int pl = min(lane / 7, 3), cg = (lane < 28) ? lane - (lane / 7) * 7 : 6;  // lanes 28-31 shadow lane 27
  const bool live = lane < 28;
  const int c0 = cg * V;
  const int g = blockIdx.x % a.groups, sl = blockIdx.x / a.groups;
  const int cb = g * 8;
  const int n0 = sl * a.nps, n1 = min(a.N, n0 + a.nps);
  const T* __restrict__ x = static_cast<const T*>(a.in);
  const T* __restrict__ dy = static_cast<const T*>(a.in2);
  if (lane == 0) {
    for (int i = 0; i < a.ns; ++i) mbar_init(&bars[i], 1);
    fence_mbar_init();
  }
  __syncwarp();
  griddep_wait();
  const uint32_t task_bytes = 8u * HW * (uint32_t)sizeof(T);
  auto slot = [&](int s) { return ring + (size_t)s * (a.slot_bytes / sizeof(T)); };
  using L = PairLayout<W>;
  auto issue = [&](int n, int s) {
    if (lane == 0 && n < n1) {
      const int64_t off = ((int64_t)n * a.C + cb) * HW;
      mbar_arrive_expect_tx(&bars[s], 2 * task_bytes);
      stage_pairs<W>(slot(s), x + off, &bars[s]);
      stage_pairs<W>(slot(s) + L::REGION, dy + off, &bars[s]);
    }
  };
  for (int i = 0; i < a.ns; ++i) issue(n0 + warp + i * nwarps, i);
  if (a.early_pdl) griddep_launch_dependents();
  const bool lft = c0 > 0, rgt = c0 + V < W;
  auto ldrow = [&](const T* ra, const T* rb, float2* xv) {  // halos by warp shuffles (all lanes call this)
    float va[V], vb[V];
    VecIO<T, V>::load(ra + c0, va);
    VecIO<T, V>::load(rb + c0, vb);
#pragma unroll
    for (int u = 0; u < V; ++u) xv[1 + u] = make_float2(va[u], vb[u]);
    const float la = __shfl_up_sync(0xffffffffu, va[V - 1], 1), lb = __shfl_up_sync(0xffffffffu, vb[V - 1], 1);
    const float ra2 = __shfl_down_sync(0xffffffffu, va[0], 1), rb2 = __shfl_down_sync(0xffffffffu, vb[0], 1);
    xv[0] = lft ? make_float2(la, lb) : make_float2(0.f, 0.f);
    xv[V + 1] = rgt ? make_float2(ra2, rb2) : make_float2(0.f, 0.f);
  };
  float2 run[9];
#pragma unroll
  for (int k = 0; k < 9; ++k) run[k] = make_float2(0.f, 0.f);
  int s = 0;
  uint32_t ph = 0;
  for (int n = n0 + warp; n < n1; n += nwarps) {
    mbar_wait(&bars[s], ph);
    {  // every lane runs the loop (shuffles); lanes 28-31 duplicate lane 27 and are left out of the sums
      const T* pa = slot(s) + L::off(L::plane_a(pl));
      const T* pb = slot(s) + L::off(L::plane_b(pl));
      const T* da = slot(s) + L::REGION + L::off(L::plane_a(pl));
      const T* db = slot(s) + L::REGION + L::off(L::plane_b(pl));
      float2 xw[3][V + 2];
#pragma unroll
      for (int u = 0; u < V + 2; ++u) xw[0][u] = make_float2(0.f, 0.f);
      ldrow(pa, pb, xw[1]);
      float2 loc[9];
#pragma unroll
      for (int r = 0; r < W; ++r) {
        if (r + 1 < W) ldrow(pa + (r + 1) * W, pb + (r + 1) * W, xw[2]);
        else
#pragma unroll
          for (int u = 0; u < V + 2; ++u) xw[2][u] = make_float2(0.f, 0.f);
        float dva[V], dvb[V];
        VecIO<T, V>::load(da + r * W + c0, dva);
        VecIO<T, V>::load(db + r * W + c0, dvb);
#pragma unroll
        for (int k = 0; k < 9; ++k)
#pragma unroll
          for (int u = 0; u < V; ++u) {
            const float2 dv = make_float2(dva[u], dvb[u]);
            loc[k] = (r == 0 && u == 0) ? __fmul2_rn(xw[k / 3][u + k % 3], dv)
                                        : __ffma2_rn(xw[k / 3][u + k % 3], dv, loc[k]);
          }
#pragma unroll
        for (int u = 0; u < V + 2; ++u) { xw[0][u] = xw[1][u]; xw[1][u] = xw[2][u]; }
      }
      if (live) {
#pragma unroll
        for (int k = 0; k < 9; ++k) run[k] = __fadd2_rn(run[k], loc[k]);
      }
    }
    __syncwarp();
    issue(n + a.ns * nwarps, s);
    if (++s == a.ns) { s = 0; ph ^= 1; }
  }
  if (!a.early_pdl) griddep_launch_dependents();
  __syncthreads();
  float* red = reinterpret_cast<float*>(smem + 64 * nwarps);  // [warp][lane][18]; the ring is idle now
  if (live) {
#pragma unroll
    for (int k = 0; k < 9; ++k) {
      red[(warp * 32 + lane) * 18 + k] = run[k].x;
      red[(warp * 32 + lane) * 18 + 9 + k] = run[k].y;
    }
  }
  __syncthreads();
  float* part = a.ws_part + (int64_t)sl * a.C * 9;
  for (int e = threadIdx.x; e < 8 * 9; e += blockDim.x) {
    const int ch = e / 9, k = e - ch * 9;  // channel cb + ch = plane_a(p) (hi 0) or plane_b(p) (hi 1)
    const int p = L::ADJ ? ch >> 1 : ch & 3, hi = L::ADJ ? ch & 1 : ch >> 2;
    float tot = 0.f;
    for (int wv = 0; wv < nwarps; ++wv) {
      float v = red[(wv * 32 + p * 7) * 18 + hi * 9 + k];
      for (int l = 1; l < 7; ++l) v += red[(wv * 32 + p * 7 + l) * 18 + hi * 9 + k];
      tot = (wv == 0) ? v : tot + v;
    }
    part[(int64_t)(cb + ch) * 9 + k] = tot;
  }
  __threadfence();
  __syncthreads();
  {
    const int ngrp = (a.nslices + 31) / 32;
    nchw::finalize_two_level(a.ws_part, a.ws_part + (int64_t)a.nslices * a.C * 9, a.ws_ticket,
                             a.ws_ticket + (int64_t)a.groups * ngrp, g, sl, a.nslices, (int64_t)a.C * 9,
                             (int64_t)cb * 9, 72, a.dw, &s_last);
  }
}

template <class T, int W>
__global__ void __launch_bounds__(256) small_fwd2_kernel(const SArgs a) {
  constexpr int Wo = W / 2, V = Wo / 7, HW = W * W, HWo = Wo * Wo, NXW = 2 * V + 1;
  extern __shared__ __align__(128) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nwarps = blockDim.x >> 5;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem) + warp * 8;
  T* ring = reinterpret_cast<T*>(smem + 64 * nwarps + (size_t)warp * a.ns * a.slot_bytes);
  const int pl = min(lane / 7, 3), cg = (lane < 28) ? lane - (lane / 7) * 7 : 6;  // lanes 28-31 shadow lane 27
  const bool live = lane < 28;
  const int c0 = cg * V;
  const T* __restrict__ in = static_cast<const T*>(a.in);
  T* __restrict__ out = static_cast<T*>(a.out);
  const T* __restrict__ wt = static_cast<const T*>(a.w);
  if (lane == 0) {
    for (int i = 0; i < a.ns; ++i) mbar_init(&bars[i], 1);
    fence_mbar_init();
  }
  __syncwarp();
  griddep_wait();
  const int64_t gw = (int64_t)blockIdx.x * nwarps + warp;
  const int64_t stride = (int64_t)gridDim.x * nwarps;
  const uint32_t task_bytes = 4u * HW * (uint32_t)sizeof(T);
  auto slot = [&](int s) { return ring + (size_t)s * (a.slot_bytes / sizeof(T)); };
  auto issue = [&](int64_t t, int s) {
    if (lane == 0 && t < a.ntasks) {
      mbar_arrive_expect_tx(&bars[s], task_bytes);
      bulk_g2s(slot(s), in + t * 4 * HW, task_bytes, &bars[s]);
    }
  };
  for (int i = 0; i < a.ns; ++i) issue(gw + i * stride, i);
  if (a.early_pdl) griddep_launch_dependents();  // grid is one wave: let the next kernel's CTAs queue
  int s = 0;
  uint32_t ph = 0;
  for (int64_t t = gw; t < a.ntasks; t += stride) {
    const int64_t q = t * 4 + pl;
    const int c = (int)(q % a.C);
    float wr[9];
#pragma unroll
    for (int k = 0; k < 9; ++k) wr[k] = Elem<T>::ldg(wt + (int64_t)c * 9 + k);
    mbar_wait(&bars[s], ph);
    {  // every lane runs the loop (halo shuffles); only live lanes store / accumulate
      const T* pln = slot(s) + pl * HW;
      float xw[3][NXW];
#pragma unroll
      for (int u = 0; u < NXW; ++u) xw[0][u] = 0.f;  // input row -1
      T* po = out + q * HWo + c0;
#pragma unroll
      for (int r = 0; r < Wo; ++r) {
        load_row2<T, V>(pln + (2 * r) * W, c0, xw[1]);
        if (2 * r + 1 < W) load_row2<T, V>(pln + (2 * r + 1) * W, c0, xw[2]);
        else
#pragma unroll
          for (int u = 0; u < NXW; ++u) xw[2][u] = 0.f;
        float o[V];
#pragma unroll
        for (int u = 0; u < V; ++u) {
          float acc = wr[0] * xw[0][2 * u];
#pragma unroll
          for (int k = 1; k < 9; ++k) acc = fmaf(wr[k], xw[k / 3][2 * u + k % 3], acc);
          o[u] = acc;
        }
        if (live) VecIO<T, V>::store(po + r * Wo, o);
#pragma unroll
        for (int u = 0; u < NXW; ++u) xw[0][u] = xw[2][u];
      }
    }
    __syncwarp();
    issue(t + a.ns * stride, s);
    if (++s == a.ns) { s = 0; ph ^= 1; }
  }
  if (!a.early_pdl) griddep_launch_dependents();
}

// stride-2 input gradient (polyphase): dx plane W x W from the dy plane Wo = W/2.
// With pad 1, dx[ih, iw] = sum_{i,j} w[i,j] dy[(ih+1-i)/2, (iw+1-j)/2] over exact
// divisions (reading R9), so per dy position (a, b):
//   dx[2a,   2b  ] = w11 dy[a,b]
//   dx[2a,   2b+1] = w10 dy[a,b+1] + w12 dy[a,b]
//   dx[2a+1, 2b  ] = w01 dy[a+1,b] + w21 dy[a,b]
//   dx[2a+1, 2b+1] = w00 dy[a+1,b+1] + w02 dy[a+1,b] + w20 dy[a,b+1] + w22 dy[a,b]
// (dy = 0 past the plane).  Warp task = TP dy planes (one bulk copy; TP = 8 when 4
// planes are not a 16-B multiple: bf16 7x7); lane (plane, column group) owns V dy
// columns and the 2V dx columns they feed, walks the dy rows with a 2-row window
// (the right halo column from the next lane by shuffle) and stores two dx rows
// per dy row straight from registers; TP = 8 runs the lanes over two plane quads.
template <class T, int W, int TP = 4>
__global__ void __launch_bounds__(256) small_bd2_kernel(const SArgs a) {
  constexpr int Wo = W / 2, V = Wo / 7, HWo = Wo * Wo, HW = W * W;
  extern __shared__ __align__(128) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nwarps = blockDim.x >> 5;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem) + warp * 8;
  T* ring = reinterpret_cast<T*>(smem + 64 * nwarps + (size_t)warp * a.ns * a.slot_bytes);
  const int pl = min(lane / 7, 3), cg = (lane < 28) ? lane - (lane / 7) * 7 : 6;  // lanes 28-31 shadow lane 27
  const bool live = lane < 28;
  const int c0 = cg * V;
  const bool rgt = c0 + V < Wo;
  const T* __restrict__ in = static_cast<const T*>(a.in);
  T* __restrict__ out = static_cast<T*>(a.out);
  const T* __restrict__ wt = static_cast<const T*>(a.w);
  if (lane == 0) {
    for (int i = 0; i < a.ns; ++i) mbar_init(&bars[i], 1);
    fence_mbar_init();
  }
  __syncwarp();
  griddep_wait();
  const int64_t gw = (int64_t)blockIdx.x * nwarps + warp;
  const int64_t stride = (int64_t)gridDim.x * nwarps;
  const uint32_t task_bytes = (uint32_t)TP * HWo * (uint32_t)sizeof(T);
  auto slot = [&](int s) { return ring + (size_t)s * (a.slot_bytes / sizeof(T)); };
  auto issue = [&](int64_t t, int s) {
    if (lane == 0 && t < a.ntasks) {
      mbar_arrive_expect_tx(&bars[s], task_bytes);
      bulk_g2s(slot(s), in + t * TP * HWo, task_bytes, &bars[s]);
    }
  };
  for (int i = 0; i < a.ns; ++i) issue(gw + i * stride, i);
  if (a.early_pdl) griddep_launch_dependents();  // grid is one wave: let the next kernel's CTAs queue
  // one dy row: the lane's V columns and the next lane's first column (all lanes call this)
  auto ldrow = [&](const T* row, float* d) {
    float v[V];
    VecIO<T, V>::load(row + c0, v);
#pragma unroll
    for (int u = 0; u < V; ++u) d[u] = v[u];
    const float r = __shfl_down_sync(0xffffffffu, v[0], 1);
    d[V] = rgt ? r : 0.f;
  };
  int s = 0;
  uint32_t ph = 0;
  for (int64_t t = gw; t < a.ntasks; t += stride) {
    mbar_wait(&bars[s], ph);
#pragma unroll 1
    for (int quad = 0; quad < TP / 4; ++quad) {  // every lane runs the loop (shuffles); only live lanes store
      const int64_t q = t * TP + quad * 4 + pl;
      const int c = (int)(q % a.C);
      float w[9];
#pragma unroll
      for (int k = 0; k < 9; ++k) w[k] = Elem<T>::ldg(wt + (int64_t)c * 9 + k);
      const T* pln = slot(s) + (quad * 4 + pl) * HWo;
      T* po = out + q * HW + 2 * c0;
      float cur[V + 1], nxt[V + 1];
      ldrow(pln, cur);
#pragma unroll
      for (int r = 0; r < Wo; ++r) {
        if (r + 1 < Wo) ldrow(pln + (r + 1) * Wo, nxt);
        else
#pragma unroll
          for (int u = 0; u <= V; ++u) nxt[u] = 0.f;
        float e0[2 * V], e1[2 * V];
#pragma unroll
        for (int u = 0; u < V; ++u) {
          const float d00 = cur[u], d01 = cur[u + 1], d10 = nxt[u], d11 = nxt[u + 1];
          e0[2 * u] = w[4] * d00;
          e0[2 * u + 1] = fmaf(w[5], d00, w[3] * d01);
          e1[2 * u] = fmaf(w[7], d00, w[1] * d10);
          e1[2 * u + 1] = fmaf(w[8], d00, fmaf(w[6], d01, fmaf(w[2], d10, w[0] * d11)));
        }
        if (live) {
          VecIO<T, 2 * V>::store(po + (2 * r) * W, e0);
          VecIO<T, 2 * V>::store(po + (2 * r + 1) * W, e1);
        }
#pragma unroll
        for (int u = 0; u <= V; ++u) cur[u] = nxt[u];
      }
    }
    __syncwarp();
    issue(t + a.ns * stride, s);
    if (++s == a.ns) { s = 0; ph ^= 1; }
  }
  if (!a.early_pdl) griddep_launch_dependents();
}

template <class T, int W, int TP = 4>  // TP channels per group (8: bf16 7x7 dy planes, 4 x 98 B is not a 16-B multiple)
__global__ void __launch_bounds__(256) small_bf2_kernel(const SArgs a) {
  constexpr int Wo = W / 2, V = Wo / 7, HW = W * W, HWo = Wo * Wo, NXW = 2 * V + 1, NQ = TP / 4;
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ unsigned s_last;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nwarps = blockDim.x >> 5;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem) + warp * 8;
  T* ring = reinterpret_cast<T*>(smem + 64 * nwarps + (size_t)warp * a.ns * a.slot_bytes);
  const int pl = min(lane / 7, 3), cg = (lane < 28) ? lane - (lane / 7) * 7 : 6;  // lanes 28-31 shadow lane 27
  const bool live = lane < 28;
  const int c0 = cg * V;
  const int g = blockIdx.x % a.groups, sl = blockIdx.x / a.groups;
  const int cb = g * TP;
  const int n0 = sl * a.nps, n1 = min(a.N, n0 + a.nps);
  const T* __restrict__ x = static_cast<const T*>(a.in);
  const T* __restrict__ dy = static_cast<const T*>(a.in2);
  if (lane == 0) {
    for (int i = 0; i < a.ns; ++i) mbar_init(&bars[i], 1);
    fence_mbar_init();
  }
  __syncwarp();
  griddep_wait();
  const uint32_t xbytes = (uint32_t)TP * HW * (uint32_t)sizeof(T), dbytes = (uint32_t)TP * HWo * (uint32_t)sizeof(T);
  auto slot = [&](int s) { return ring + (size_t)s * (a.slot_bytes / sizeof(T)); };
  auto issue = [&](int n, int s) {
    if (lane == 0 && n < n1) {
      mbar_arrive_expect_tx(&bars[s], xbytes + dbytes);
      bulk_g2s(slot(s), x + ((int64_t)n * a.C + cb) * HW, xbytes, &bars[s]);
      bulk_g2s(slot(s) + TP * HW, dy + ((int64_t)n * a.C + cb) * HWo, dbytes, &bars[s]);
    }
  };
  for (int i = 0; i < a.ns; ++i) issue(n0 + warp + i * nwarps, i);
  if (a.early_pdl) griddep_launch_dependents();  // grid is one wave: let the next kernel's CTAs queue
  float run[NQ][9];
#pragma unroll
  for (int qd = 0; qd < NQ; ++qd)
#pragma unroll
    for (int k = 0; k < 9; ++k) run[qd][k] = 0.f;
  int s = 0;
  uint32_t ph = 0;
  for (int n = n0 + warp; n < n1; n += nwarps) {
    mbar_wait(&bars[s], ph);
#pragma unroll
    for (int qd = 0; qd < NQ; ++qd) {  // every lane runs the loop (halo shuffles); only live lanes accumulate
      const T* pln = slot(s) + (qd * 4 + pl) * HW;
      const T* pd = slot(s) + TP * HW + (qd * 4 + pl) * HWo;
      float xw[3][NXW];
#pragma unroll
      for (int u = 0; u < NXW; ++u) xw[0][u] = 0.f;
      float loc[9];
#pragma unroll
      for (int k = 0; k < 9; ++k) loc[k] = 0.f;
#pragma unroll
      for (int r = 0; r < Wo; ++r) {
        load_row2<T, V>(pln + (2 * r) * W, c0, xw[1]);
        if (2 * r + 1 < W) load_row2<T, V>(pln + (2 * r + 1) * W, c0, xw[2]);
        else
#pragma unroll
          for (int u = 0; u < NXW; ++u) xw[2][u] = 0.f;
        float d[V];
        VecIO<T, V>::load(pd + r * Wo + c0, d);
#pragma unroll
        for (int k = 0; k < 9; ++k)
#pragma unroll
          for (int u = 0; u < V; ++u) loc[k] = fmaf(xw[k / 3][2 * u + k % 3], d[u], loc[k]);
#pragma unroll
        for (int u = 0; u < NXW; ++u) xw[0][u] = xw[2][u];
      }
      if (live) {
#pragma unroll
        for (int k = 0; k < 9; ++k) run[qd][k] += loc[k];
      }
    }
    __syncwarp();
    issue(n + a.ns * nwarps, s);
    if (++s == a.ns) { s = 0; ph ^= 1; }
  }
  if (!a.early_pdl) griddep_launch_dependents();
  __syncthreads();
  float* red = reinterpret_cast<float*>(smem + 64 * nwarps);  // [warp][lane][NQ*9]; the ring is idle now
  if (live) {
#pragma unroll
    for (int qd = 0; qd < NQ; ++qd)
#pragma unroll
      for (int k = 0; k < 9; ++k) red[(warp * 32 + lane) * (NQ * 9) + qd * 9 + k] = run[qd][k];
  }
  __syncthreads();
  float* part = a.ws_part + (int64_t)sl * a.C * 9;
  for (int e = threadIdx.x; e < TP * 9; e += blockDim.x) {
    const int ch = e / 9, k = e - ch * 9;  // channel cb + ch = quad ch / 4, lane group ch % 4
    const int qd = ch >> 2, p = ch & 3;
    float tot = 0.f;
    for (int wv = 0; wv < nwarps; ++wv) {
      float v = red[(wv * 32 + p * 7) * (NQ * 9) + qd * 9 + k];
      for (int l = 1; l < 7; ++l) v += red[(wv * 32 + p * 7 + l) * (NQ * 9) + qd * 9 + k];
      tot = (wv == 0) ? v : tot + v;
    }
    part[(int64_t)(cb + ch) * 9 + k] = tot;
  }
  __threadfence();
  __syncthreads();
  {
    const int ngrp = (a.nslices + 31) / 32;
    nchw::finalize_two_level(a.ws_part, a.ws_part + (int64_t)a.nslices * a.C * 9, a.ws_ticket,
                             a.ws_ticket + (int64_t)a.groups * ngrp, g, sl, a.nslices, (int64_t)a.C * 9,
                             (int64_t)cb * 9, TP * 9, a.dw, &s_last);
  }
}

// Band bwd_filter over channel PAIRS: every lane owns V dy columns of two
// consecutive channels (the task stages both planes' bands) and accumulates
// them as packed FFMA2 (float2 lanes = the two channels) -- half the FMA
// instructions of band_bf_kernel, for the instruction-bound bf16 case.
template <class T, int S, int V, int R>
__global__ void __launch_bounds__(256) band_bf_pair_kernel(const SArgs a) {
  constexpr int NX = S * V;
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ unsigned s_last;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nwarps = blockDim.x >> 5;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem) + warp * 8;
  T* ring = reinterpret_cast<T*>(smem + 64 * nwarps + (size_t)warp * a.ns * a.slot_bytes);
  const int g = blockIdx.x % a.groups, sl = blockIdx.x / a.groups;
  const int cw = g * a.cpg + warp * 2;  // channels cw, cw + 1
  const int np_w = max(0, min(2, min(a.cpg - warp * 2, a.C - cw)));
  const bool wlive = np_w > 0;
  const int H = a.H, W = a.W, Ho = a.Ho, Wo = a.Wo;
  const bool live = wlive && lane * V < Wo;
  const int n0 = sl * a.nps, n1 = min(a.N, n0 + a.nps);
  const int ntask = (n1 - n0) * a.nbands;
  const T* __restrict__ x = static_cast<const T*>(a.in);
  const T* __restrict__ dy = static_cast<const T*>(a.in2);
  const uint32_t xcap = (uint32_t)(((R - 1) * S + 3) * W * sizeof(T) + 15) & ~15u;
  const uint32_t dcap = (uint32_t)(R * Wo * sizeof(T) + 15) & ~15u;
  if (lane == 0) {
    for (int i = 0; i < a.ns; ++i) mbar_init(&bars[i], 1);
    fence_mbar_init();
  }
  __syncwarp();
  griddep_wait();
  auto slot = [&](int s) { return reinterpret_cast<unsigned char*>(ring) + (size_t)s * a.slot_bytes; };
  auto rows_of = [&](int t, int* n, int* r0, int* r1, int* lo, int* hi) {
    const int nn = t / a.nbands, b = t - nn * a.nbands;
    *n = n0 + nn;
    *r0 = b * R;
    *r1 = min(*r0 + R, Ho);
    *lo = max(0, *r0 * S - 1);
    *hi = min(H, (*r1 - 1) * S + 2);
  };
  auto issue = [&](int t, int s) {
    if (lane == 0 && wlive && t < ntask) {
      int n, r0, r1, lo, hi;
      rows_of(t, &n, &r0, &r1, &lo, &hi);
      const uint32_t xb = (uint32_t)((hi - lo) * W * sizeof(T)), db = (uint32_t)((r1 - r0) * Wo * sizeof(T));
      mbar_arrive_expect_tx(&bars[s], (uint32_t)np_w * (xb + db));
      for (int p = 0; p < np_w; ++p) {
        unsigned char* sp = slot(s) + (size_t)p * (xcap + dcap);
        bulk_g2s(sp, x + (((int64_t)n * a.C + cw + p) * H + lo) * W, xb, &bars[s]);
        bulk_g2s(sp + xcap, dy + (((int64_t)n * a.C + cw + p) * Ho + r0) * Wo, db, &bars[s]);
      }
    }
  };
  for (int i = 0; i < a.ns; ++i) issue(i, i);
  if (a.early_pdl) griddep_launch_dependents();
  const int c0 = lane * V;
  float2 run[9];
#pragma unroll
  for (int k = 0; k < 9; ++k) run[k] = make_float2(0.f, 0.f);
  int s = 0;
  uint32_t ph = 0;
  for (int t = 0; t < (wlive ? ntask : 0); ++t) {
    mbar_wait(&bars[s], ph);
    if (live) {
      int n, r0, r1, lo, hi;
      rows_of(t, &n, &r0, &r1, &lo, &hi);
      const unsigned char* spa = slot(s);
      const unsigned char* spb = slot(s) + (np_w > 1 ? (xcap + dcap) : 0);  // a lone last channel pairs with itself
      const T* xa = reinterpret_cast<const T*>(spa) - (int64_t)lo * W;
      const T* xb2 = reinterpret_cast<const T*>(spb) - (int64_t)lo * W;
      const T* dsa = reinterpret_cast<const T*>(spa + xcap) - (int64_t)r0 * Wo;
      const T* dsb = reinterpret_cast<const T*>(spb + xcap) - (int64_t)r0 * Wo;
      float2 xw[3][NX + 2];
      auto ldx = [&](int ih, float2* v) {
        if (ih >= lo && ih < hi) {
          const T* ra = xa + (int64_t)ih * W;
          const T* rb = xb2 + (int64_t)ih * W;
          float oa[NX], ob[NX];
          VecIO<T, NX>::load(ra + S * c0, oa);
          VecIO<T, NX>::load(rb + S * c0, ob);
#pragma unroll
          for (int u = 0; u < NX; ++u) v[1 + u] = make_float2(oa[u], ob[u]);
          v[0] = (c0 > 0) ? make_float2(Elem<T>::load(ra + S * c0 - 1), Elem<T>::load(rb + S * c0 - 1))
                          : make_float2(0.f, 0.f);
          v[NX + 1] = (S == 1 && c0 + V < W) ? make_float2(Elem<T>::load(ra + c0 + V), Elem<T>::load(rb + c0 + V))
                                             : make_float2(0.f, 0.f);
        } else {
#pragma unroll
          for (int u = 0; u < NX + 2; ++u) v[u] = make_float2(0.f, 0.f);
        }
      };
#pragma unroll
      for (int i = 0; i < 3 - S; ++i) ldx(r0 * S - 1 + i, xw[i]);
      float2 loc[9];
#pragma unroll
      for (int k = 0; k < 9; ++k) loc[k] = make_float2(0.f, 0.f);
#pragma unroll
      for (int rr = 0; rr < R; ++rr) {
        const int r = r0 + rr;
        if (r < r1) {
#pragma unroll
          for (int i = 3 - S; i < 3; ++i) ldx(r * S - 1 + i, xw[i]);
          float da[V], db[V];
          VecIO<T, V>::load(dsa + (int64_t)r * Wo + c0, da);
          VecIO<T, V>::load(dsb + (int64_t)r * Wo + c0, db);
#pragma unroll
          for (int k = 0; k < 9; ++k)
#pragma unroll
            for (int u = 0; u < V; ++u)
              loc[k] = __ffma2_rn(xw[k / 3][S * u + k % 3], make_float2(da[u], db[u]), loc[k]);
#pragma unroll
          for (int i = 0; i < 3 - S; ++i)
#pragma unroll
            for (int u = 0; u < NX + 2; ++u) xw[i][u] = xw[i + S][u];
        }
      }
#pragma unroll
      for (int k = 0; k < 9; ++k) run[k] = __fadd2_rn(run[k], loc[k]);
    }
    __syncwarp();
    issue(t + a.ns, s);
    if (++s == a.ns) { s = 0; ph ^= 1; }
  }
  if (!a.early_pdl) griddep_launch_dependents();
  // ---- lanes: fixed xor tree per channel -> the warp's two channel partials
#pragma unroll
  for (int k = 0; k < 9; ++k) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      run[k].x += __shfl_xor_sync(0xffffffffu, run[k].x, off);
      run[k].y += __shfl_xor_sync(0xffffffffu, run[k].y, off);
    }
  }
  float* part = a.ws_part + (int64_t)sl * a.C * 9;
  if (lane < 9 * np_w) {
    const int p = lane / 9, kk = lane - p * 9;
    float v = 0.f;
#pragma unroll
    for (int k = 0; k < 9; ++k) v = (kk == k) ? (p ? run[k].y : run[k].x) : v;
    part[(int64_t)(cw + p) * 9 + kk] = v;
  }
  __threadfence();
  __syncthreads();
  {
    const int ngrp = (a.nslices + 31) / 32;
    nchw::finalize_two_level(a.ws_part, a.ws_part + (int64_t)a.nslices * a.C * 9, a.ws_ticket,
                             a.ws_ticket + (int64_t)a.groups * ngrp, g, sl, a.nslices, (int64_t)a.C * 9,
                             (int64_t)g * a.cpg * 9, min(a.cpg, a.C - g * a.cpg) * 9, a.dw, &s_last);
  }
}

// ---------------------------------------------------------------- lane-per-plane kernels
// W in {7, 14}, 3x3, stride 1, pad 1, m = 1.  A warp task is 32 consecutive planes
// (one bulk copy); lane l computes plane l end to end -- no shuffles, no per-strip
// index arithmetic -- with a 3-row window in registers and FFMA2 over interleaved
// column pairs (u, u + H2), H2 = ceil(W / 2): the operand pair of tap j is
// X2[u + j] = (xw[u + j], xw[u + j + H2]), xw = the row with its zero halo, so
// bf16 values are widened straight into pair halves (PRMT / LOP3) and no pair is
// formed by moves.  fwd / bwd_data write each output row back over the staged
// input row (every input row is read into registers before the output row above
// the next one is written), then lane 0 bulk-stores the 32 planes
// (cp.async.bulk shared -> global) and refills the slot once the store has read it.
// bwd_filter: CTA = (32 channels, batch slice), lane = channel; warps take the
// slice's images in turn; the same windows with dy rows as the second operand.
namespace lanek {
template <class T, int W>
struct Row {
  static constexpr int H2 = (W + 1) / 2;
  static constexpr int NP = H2 + 2;  // operand pairs per row
  // raw words of one row: bf16 W even -> W/2 words; bf16 W odd -> W halfwords; fp32 -> W words
  static constexpr int NR = (sizeof(T) == 2 && W % 2 == 0) ? W / 2 : W;
  uint32_t r[NR];
  __device__ __forceinline__ void load(const T* p) {
    if constexpr (sizeof(T) == 2 && W % 2 == 0) {
#pragma unroll
      for (int q = 0; q < NR; ++q) r[q] = reinterpret_cast<const uint32_t*>(p)[q];
    } else if constexpr (sizeof(T) == 2) {
#pragma unroll
      for (int q = 0; q < NR; ++q) r[q] = reinterpret_cast<const unsigned short*>(p)[q];
    } else if constexpr (W % 2 == 0) {
#pragma unroll
      for (int q = 0; q < NR / 2; ++q) {
        const uint2 v = reinterpret_cast<const uint2*>(p)[q];
        r[2 * q] = v.x; r[2 * q + 1] = v.y;
      }
    } else {
#pragma unroll
      for (int q = 0; q < NR; ++q) r[q] = reinterpret_cast<const uint32_t*>(p)[q];
    }
  }
  __device__ __forceinline__ void zero() {
#pragma unroll
    for (int q = 0; q < NR; ++q) r[q] = 0u;
  }
  // element k of the row (0 <= k < W) as fp32
  __device__ __forceinline__ float val(int k) const {
    if constexpr (sizeof(T) == 2 && W % 2 == 0) return (k & 1) ? nchw::bfw_hi(r[k >> 1]) : nchw::bfw_lo(r[k >> 1]);
    else if constexpr (sizeof(T) == 2) return nchw::bfw_lo(r[k]);
    else return __uint_as_float(r[k]);
  }
  // xw[k]: the row with a zero column on each side (and zeros past it)
  __device__ __forceinline__ float xw(int k) const { return (k >= 1 && k <= W) ? val(k - 1) : 0.f; }
  __device__ __forceinline__ void pairs(float2* X2) const {
#pragma unroll
    for (int k = 0; k < NP; ++k) X2[k] = make_float2(xw(k), xw(k + H2));
  }
  // D2[u] = (v[u], v[u + H2]) of the row itself (dy operand of bwd_filter)
  __device__ __forceinline__ void dpairs(float2* D2) const {
#pragma unroll
    for (int u = 0; u < H2; ++u) D2[u] = make_float2(val(u), u + H2 < W ? val(u + H2) : 0.f);
  }
};
// store W values o[c] = c < H2 ? acc[c].x : acc[c - H2].y at p
template <class T, int W>
__device__ __forceinline__ void store_row(T* p, const float2* acc) {
  constexpr int H2 = (W + 1) / 2;
  auto o = [&](int c) { return c < H2 ? acc[c].x : acc[c - H2].y; };
  if constexpr (sizeof(T) == 2 && W % 2 == 0) {
#pragma unroll
    for (int q = 0; q < W / 2; ++q) reinterpret_cast<uint32_t*>(p)[q] = nchw::bf_pack(o(2 * q), o(2 * q + 1));
  } else if constexpr (sizeof(T) == 2) {
#pragma unroll
    for (int c = 0; c < W; ++c) p[c] = __float2bfloat16_rn(o(c));
  } else if constexpr (W % 2 == 0) {
#pragma unroll
    for (int q = 0; q < W / 2; ++q) reinterpret_cast<float2*>(p)[q] = make_float2(o(2 * q), o(2 * q + 1));
  } else {
#pragma unroll
    for (int c = 0; c < W; ++c) reinterpret_cast<float*>(p)[c] = o(c);
  }
}
}  // namespace lanek

// MODE 0 fwd, 1 bwd_data (kernel rotated by 180 degrees: reading R9)
template <class T, int W, int MODE>
__global__ void __launch_bounds__(256) lane_fd_kernel(const SArgs a) {
  using RowT = lanek::Row<T, W>;
  constexpr int HW = W * W, H2 = RowT::H2, NP = RowT::NP;
  extern __shared__ __align__(128) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nwarps = blockDim.x >> 5;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem) + warp * 8;
  T* ring = reinterpret_cast<T*>(smem + 64 * nwarps + (size_t)warp * a.ns * a.slot_bytes);
  const T* __restrict__ in = static_cast<const T*>(a.in);
  T* __restrict__ out = static_cast<T*>(a.out);
  const T* __restrict__ wt = static_cast<const T*>(a.w);
  if (lane == 0) {
    for (int i = 0; i < a.ns; ++i) mbar_init(&bars[i], 1);
    fence_mbar_init();
  }
  __syncwarp();
  griddep_wait();
  const int64_t gw = (int64_t)blockIdx.x * nwarps + warp;
  const int64_t stride = (int64_t)gridDim.x * nwarps;
  constexpr uint32_t task_bytes = 32u * HW * (uint32_t)sizeof(T);
  auto slot = [&](int s) { return ring + (size_t)s * (a.slot_bytes / sizeof(T)); };
  auto issue = [&](int64_t t, int s) {
    if (t < a.ntasks) {
      mbar_arrive_expect_tx(&bars[s], task_bytes);
      bulk_g2s(slot(s), in + t * 32 * HW, task_bytes, &bars[s]);
    }
  };
  if (lane == 0)
    for (int i = 0; i < a.ns; ++i) issue(gw + i * stride, i);
  int s = 0;
  uint32_t ph = 0;
  for (int64_t t = gw; t < a.ntasks; t += stride) {
    const int64_t q = t * 32 + lane;  // this lane's plane
    const int c = (int)(q % a.C);
    float wr[9];
#pragma unroll
    for (int k = 0; k < 9; ++k) wr[k] = Elem<T>::ldg(wt + (int64_t)c * 9 + (MODE == 1 ? 8 - k : k));
    mbar_wait(&bars[s], ph);
    T* pln = slot(s) + lane * HW;
    // operand pairs of input rows oh - 1, oh, oh + 1 (each row widened once)
    float2 X0[NP], X1[NP], X2[NP];
#pragma unroll
    for (int k = 0; k < NP; ++k) X0[k] = make_float2(0.f, 0.f);
    {
      RowT r;
      r.load(pln);
      r.pairs(X1);
    }
#pragma unroll
    for (int oh = 0; oh < W; ++oh) {
      if (oh + 1 < W) {
        RowT r;
        r.load(pln + (oh + 1) * W);
        r.pairs(X2);
      } else {
#pragma unroll
        for (int k = 0; k < NP; ++k) X2[k] = make_float2(0.f, 0.f);
      }
      float2 acc[H2];
#pragma unroll
      for (int u = 0; u < H2; ++u) {
        float2 v = __fmul2_rn(make_float2(wr[0], wr[0]), X0[u]);
#pragma unroll
        for (int j = 1; j < 3; ++j) v = __ffma2_rn(make_float2(wr[j], wr[j]), X0[u + j], v);
#pragma unroll
        for (int j = 0; j < 3; ++j) v = __ffma2_rn(make_float2(wr[3 + j], wr[3 + j]), X1[u + j], v);
#pragma unroll
        for (int j = 0; j < 3; ++j) v = __ffma2_rn(make_float2(wr[6 + j], wr[6 + j]), X2[u + j], v);
        acc[u] = v;
      }
      lanek::store_row<T, W>(pln + oh * W, acc);  // rows <= oh + 1 are already in registers
#pragma unroll
      for (int k = 0; k < NP; ++k) { X0[k] = X1[k]; X1[k] = X2[k]; }
    }
    fence_proxy_async_smem();  // the generic-proxy stores, before the bulk copy reads them
    __syncwarp();
    if (lane == 0) {
      bulk_s2g(out + t * 32 * HW, slot(s), task_bytes);
      bulk_commit();
      bulk_wait_read<0>();  // the slot has been read out: refill it
      issue(t + a.ns * stride, s);
    }
    if (++s == a.ns) { s = 0; ph ^= 1; }
  }
  if (lane == 0) bulk_wait<0>();
  griddep_launch_dependents();
}

// bwd_filter: CTA = (group of 32 channels, batch slice of nps images); warp w takes
// images n0 + w, n0 + w + warps, ...; lane = channel.  Reduction, fixed order:
// per image the window sums (W * H2 deep) -> a running sum over the warp's images
// -> the warps in order -> per-slice partial -> two-level slice finalize.
template <class T, int W>
__global__ void __launch_bounds__(256) lane_bf_kernel(const SArgs a) {
  using RowT = lanek::Row<T, W>;
  constexpr int HW = W * W, H2 = RowT::H2, NP = RowT::NP;
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ unsigned s_last;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nwarps = blockDim.x >> 5;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem) + warp * 8;
  T* ring = reinterpret_cast<T*>(smem + 64 * nwarps + (size_t)warp * a.ns * a.slot_bytes);
  const T* __restrict__ x = static_cast<const T*>(a.in);
  const T* __restrict__ dy = static_cast<const T*>(a.in2);
  const int g = blockIdx.x % a.groups;
  const int sl = blockIdx.x / a.groups;
  const int c0 = g * 32;
  const int64_t n0 = (int64_t)sl * a.nps;
  const int nimg = (int)(min((int64_t)a.N, n0 + a.nps) - n0);
  if (lane == 0) {
    for (int i = 0; i < a.ns; ++i) mbar_init(&bars[i], 1);
    fence_mbar_init();
  }
  __syncwarp();
  griddep_wait();
  constexpr uint32_t half = 32u * HW * (uint32_t)sizeof(T);
  auto slot = [&](int s) { return ring + (size_t)s * (a.slot_bytes / sizeof(T)); };
  auto issue = [&](int k, int s) {  // k-th image of this warp
    const int ni = warp + k * nwarps;
    if (ni < nimg) {
      const int64_t base = ((n0 + ni) * a.C + c0) * (int64_t)HW;
      mbar_arrive_expect_tx(&bars[s], 2 * half);
      bulk_g2s(slot(s), x + base, half, &bars[s]);
      bulk_g2s(slot(s) + 32 * HW, dy + base, half, &bars[s]);
    }
  };
  if (lane == 0)
    for (int i = 0; i < a.ns; ++i) issue(i, i);
  float run[9];
#pragma unroll
  for (int q = 0; q < 9; ++q) run[q] = 0.f;
  int s = 0;
  uint32_t ph = 0;
  for (int k = 0; warp + k * nwarps < nimg; ++k) {
    mbar_wait(&bars[s], ph);
    const T* px = slot(s) + lane * HW;
    const T* pd = slot(s) + 32 * HW + lane * HW;
    float2 loc[9];
#pragma unroll
    for (int q = 0; q < 9; ++q) loc[q] = make_float2(0.f, 0.f);
    // x row ih meets dy rows ih + 1 (tap row 0), ih (1), ih - 1 (2)
    float2 Dm[H2], D0[H2], Dp[H2];  // dy rows ih - 1, ih, ih + 1
    {
      RowT r;
      r.load(pd);
      r.dpairs(D0);
#pragma unroll
      for (int u = 0; u < H2; ++u) Dm[u] = make_float2(0.f, 0.f);
    }
#pragma unroll
    for (int ih = 0; ih < W; ++ih) {
      if (ih + 1 < W) {
        RowT r;
        r.load(pd + (ih + 1) * W);
        r.dpairs(Dp);
      }
      RowT rx;
      rx.load(px + ih * W);
      float2 X[NP];
      rx.pairs(X);
#pragma unroll
      for (int j = 0; j < 3; ++j)
#pragma unroll
        for (int u = 0; u < H2; ++u) {
          if (ih + 1 < W) loc[0 * 3 + j] = __ffma2_rn(X[u + j], Dp[u], loc[0 * 3 + j]);
          loc[1 * 3 + j] = __ffma2_rn(X[u + j], D0[u], loc[1 * 3 + j]);
          if (ih >= 1) loc[2 * 3 + j] = __ffma2_rn(X[u + j], Dm[u], loc[2 * 3 + j]);
        }
#pragma unroll
      for (int u = 0; u < H2; ++u) { Dm[u] = D0[u]; D0[u] = Dp[u]; }
    }
#pragma unroll
    for (int q = 0; q < 9; ++q) run[q] += loc[q].x + loc[q].y;
    __syncwarp();
    if (lane == 0) issue(k + a.ns, s);  // every lane is past the slot
    if (++s == a.ns) { s = 0; ph ^= 1; }
  }
  griddep_launch_dependents();
  // ---- reduce over the warps in order (ring slots are consumed: reuse the smem)
  __syncthreads();
  float* red = reinterpret_cast<float*>(smem + 64 * nwarps);
#pragma unroll
  for (int q = 0; q < 9; ++q) red[(warp * 32 + lane) * 9 + q] = run[q];
  __syncthreads();
  const int nch = min(32, a.C - c0);
  float* part = a.ws_part + ((int64_t)sl * a.C + c0) * 9;
  for (int e = threadIdx.x; e < nch * 9; e += blockDim.x) {
    float v = red[e];
    for (int w2 = 1; w2 < nwarps; ++w2) v += red[w2 * 32 * 9 + e];
    part[e] = v;
  }
  __threadfence();
  __syncthreads();
  {
    const int ngrp = (a.nslices + 31) / 32;
    nchw::finalize_two_level(a.ws_part, a.ws_part + (int64_t)a.nslices * a.C * 9, a.ws_ticket,
                             a.ws_ticket + (int64_t)a.groups * ngrp, g, sl, a.nslices, (int64_t)a.C * 9,
                             (int64_t)c0 * 9, nch * 9, a.dw, &s_last);
  }
}

using SKernelFn = void (*)(SArgs);

template <class T, int S, int R, int PPW>
SKernelFn band_pick_v(int V) {
  switch (V) {
    case 1: return PPW == 1 ? band_bf_kernel<T, S, 1, R, PPW> : nullptr;
    case 2: return band_bf_kernel<T, S, 2, R, PPW>;
    case 4: return (S == 1 || sizeof(T) == 2) ? band_bf_kernel<T, S, 4, R, PPW> : nullptr;
    default: return nullptr;
  }
}
template <class T, int PPW>
SKernelFn band_pick_sr(int S, int V, int R) {
  if (S == 1) return R == 7 ? band_pick_v<T, 1, 7, PPW>(V) : band_pick_v<T, 1, 14, PPW>(V);
  return R == 7 ? band_pick_v<T, 2, 7, PPW>(V) : band_pick_v<T, 2, 14, PPW>(V);
}
template <class T>
SKernelFn band_pair_pick(int S, int V, int R) {
  if (S == 1) {
    if (V == 1) return R == 7 ? band_bf_pair_kernel<T, 1, 1, 7> : band_bf_pair_kernel<T, 1, 1, 14>;
    if (V == 2) return R == 7 ? band_bf_pair_kernel<T, 1, 2, 7> : band_bf_pair_kernel<T, 1, 2, 14>;
    if (V == 4) return R == 7 ? band_bf_pair_kernel<T, 1, 4, 7> : band_bf_pair_kernel<T, 1, 4, 14>;
  } else {
    if (V == 1) return R == 7 ? band_bf_pair_kernel<T, 2, 1, 7> : band_bf_pair_kernel<T, 2, 1, 14>;
    if (V == 2) return R == 7 ? band_bf_pair_kernel<T, 2, 2, 7> : band_bf_pair_kernel<T, 2, 2, 14>;
  }
  return nullptr;
}
SKernelFn band_kernel_for(int dtype, int S, int V, int R, int PPW = 1) {
  if (PPW == 3) return dtype == DWCONV_F32 ? band_pair_pick<float>(S, V, R) : band_pair_pick<__nv_bfloat16>(S, V, R);
  if (dtype == DWCONV_F32) return PPW == 2 ? band_pick_sr<float, 2>(S, V, R) : band_pick_sr<float, 1>(S, V, R);
  using B = __nv_bfloat16;
  return PPW == 2 ? band_pick_sr<B, 2>(S, V, R) : band_pick_sr<B, 1>(S, V, R);
}

template <class T>
SKernelFn pick(int pass, int W) {
  switch (W) {
    case 7: return pass == 0 ? small_fd_kernel<T, 7, 0> : pass == 1 ? small_fd_kernel<T, 7, 1>
                 : pass == 2 ? small_bf_kernel<T, 7> : small_bf_kernel<T, 7, true>;
    case 14: return pass == 0 ? small_fd_kernel<T, 14, 0> : pass == 1 ? small_fd_kernel<T, 14, 1>
                  : pass == 2 ? small_bf_kernel<T, 14> : small_bf_kernel<T, 14, true>;
    case 28: return pass == 0 ? small_fd_kernel<T, 28, 0> : pass == 1 ? small_fd_kernel<T, 28, 1>
                  : pass == 2 ? small_bf_kernel<T, 28> : small_bf_kernel<T, 28, true>;
    default: return nullptr;
  }
}
template <class T>
SKernelFn pick2(int pass, int W) {  // stride 2: fwd, bwd_data, bwd_filter
  if (pass == 0) return W == 14 ? small_fwd2_kernel<T, 14> : W == 28 ? small_fwd2_kernel<T, 28> : nullptr;
  if (pass == 1) {  // bf16 7x7 dy planes: 8-plane tasks (4 x 98 B is not a 16-B multiple)
    if (W == 14) return sizeof(T) == 2 ? small_bd2_kernel<T, 14, 8> : small_bd2_kernel<T, 14, 4>;
    return W == 28 ? small_bd2_kernel<T, 28> : nullptr;
  }
  if (pass == 2) {
    if (W == 14) return sizeof(T) == 2 ? small_bf2_kernel<T, 14, 8> : small_bf2_kernel<T, 14, 4>;
    return W == 28 ? small_bf2_kernel<T, 28> : nullptr;
  }
  return nullptr;
}
SKernelFn pair_kernel_for(int pass, int W) {
  if (pass == 2) return W == 7 ? small_bf_pair_kernel<7> : W == 14 ? small_bf_pair_kernel<14>
                      : W == 28 ? small_bf_pair_kernel<28> : nullptr;
  if (pass == 0) return W == 7 ? small_fd_pair_kernel<7, 0> : W == 14 ? small_fd_pair_kernel<14, 0>
                      : W == 28 ? small_fd_pair_kernel<28, 0> : nullptr;
  if (pass == 1) return W == 7 ? small_fd_pair_kernel<7, 1> : W == 14 ? small_fd_pair_kernel<14, 1>
                      : W == 28 ? small_fd_pair_kernel<28, 1> : nullptr;
  return nullptr;
}
SKernelFn lane_kernel_for(int dtype, int pass, int W) {
  using B = __nv_bfloat16;
  if (W == 14) {
    if (dtype == DWCONV_F32) return pass == 0 ? lane_fd_kernel<float, 14, 0> : pass == 1 ? lane_fd_kernel<float, 14, 1>
                                  : pass == 2 ? lane_bf_kernel<float, 14> : nullptr;
    return pass == 0 ? lane_fd_kernel<B, 14, 0> : pass == 1 ? lane_fd_kernel<B, 14, 1> : pass == 2 ? lane_bf_kernel<B, 14> : nullptr;
  }
  if (W == 7) {
    if (dtype == DWCONV_F32) return pass == 0 ? lane_fd_kernel<float, 7, 0> : pass == 1 ? lane_fd_kernel<float, 7, 1>
                                  : pass == 2 ? lane_bf_kernel<float, 7> : nullptr;
    return pass == 0 ? lane_fd_kernel<B, 7, 0> : pass == 1 ? lane_fd_kernel<B, 7, 1> : pass == 2 ? lane_bf_kernel<B, 7> : nullptr;
  }
  return nullptr;
}
SKernelFn kernel_for(int dtype, int pass, int W, int S = 1) {
  if (S == 2) return dtype == DWCONV_F32 ? pick2<float>(pass, W) : pick2<__nv_bfloat16>(pass, W);
  return dtype == DWCONV_F32 ? pick<float>(pass, W) : pick<__nv_bfloat16>(pass, W);
}

int env_int(const char* name, int dflt, int lo, int hi) {
  const char* e = dev_knob(name);
  const int v = e ? std::atoi(e) : dflt;
  return (v >= lo && v <= hi) ? v : dflt;
}

}  // namespace small

// Eligibility + launch shape.  pass: 0 fwd, 1 bwd_data, 2 bwd_filter.
bool plan_nchw_small(const Geom& g, int pass, int num_sms, int smem_optin, SmallPlan* p, int warps, int stages,
                     int slices, bool pair) {
  using namespace small;
  static const int on = env_int("DWCONV_SMALL", 1, 0, 1);
  if (!on || g.layout != DWCONV_NCHW || g.m != 1 || g.kh != 3 || g.kw != 3 || g.ph != 1 || g.pw != 1) return false;
  const int S = g.sh;
  if (g.sw != S || g.H != g.W) return false;
  if (S == 1 && g.W != 7 && g.W != 14 && g.W != 28) return false;
  if (S == 2 && ((g.W != 14 && g.W != 28) || pass == 3)) return false;  // s2: fwd, bwd_data, bwd_filter
  if (S != 1 && S != 2) return false;
  if (g.C % 4 != 0 || g.N < 1) return false;
  const int64_t eb = (g.dtype == DWCONV_F32) ? 4 : 2;
  if (pair && (g.dtype != DWCONV_BF16 || S != 1 || pass > 2 || (g.N * g.C) % 8 != 0 || (pass == 2 && g.C % 8))) return false;
  // the staged planes: x (fwd, bwd_filter) or dy (bwd_data); stride-2 bf16 bwd_data on 14x14 takes
  // 8 dy planes per task (4 x 7x7 bf16 is not a 16-B multiple)
  const int tp = (pair || (S == 2 && (pass == 1 || pass == 2) && eb == 2 && g.W == 14)) ? 8 : 4;
  const int64_t task_bytes = tp * (pass == 1 ? g.Ho * g.Wo : g.H * g.W) * eb;
  const int64_t dy_bytes = tp * g.Ho * g.Wo * eb;
  if (task_bytes % 16 != 0 || (pass >= 2 && dy_bytes % 16 != 0)) return false;  // bulk copies: 16-B granules
  *p = SmallPlan{};
  static const int warps_env = env_int("DWCONV_SMALL_WARPS", 4, 1, 8);
  static const int ns_env = env_int("DWCONV_SMALL_STAGES", 3, 2, 6);
  p->warps = warps > 0 ? warps : warps_env;
  p->ns = stages > 0 ? stages : ns_env;
  const bool bf = pass >= 2;  // bwd_filter or the fused backward
  p->slot_bytes = (uint32_t)(task_bytes + (bf ? dy_bytes : 0));
  if (pair && g.W == 14) p->slot_bytes = (uint32_t)((bf ? 2 : 1) * PairLayout<14>::REGION * eb);  // padded pairs
  p->S = S;
  p->pair = pair;
  p->smem = 64 * p->warps + p->warps * p->ns * (int)p->slot_bytes;
  if (bf) p->smem = std::max(p->smem, 64 * p->warps + p->warps * 32 * (tp == 8 ? 18 : 9) * 4);
  if (p->smem > smem_optin - 1024) return false;
  SKernelFn fn = pair ? pair_kernel_for(pass, (int)g.W) : kernel_for(g.dtype, pass, (int)g.W, S);
  if (!fn) return false;
  cudaFuncAttributes fa{};
  if (cudaFuncGetAttributes(&fa, fn) != cudaSuccess) return false;
  if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_optin - (int)fa.sharedSizeBytes) !=
      cudaSuccess)
    return false;
  int occ = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, 32 * p->warps, p->smem) != cudaSuccess || occ < 1)
    return false;
  p->occ = occ;
  p->sms = num_sms;
  if (!bf) {
    if ((g.N * g.C) % tp != 0) return false;
    p->ntasks = g.N * g.C / tp;
    p->grid = (int)std::min<int64_t>((p->ntasks + p->warps - 1) / p->warps, (int64_t)occ * num_sms);
    if (slices > 0) {  // fwd / bwd_data: `slices` = tasks per warp (an even split: no partial last round)
      const int64_t g2 = (p->ntasks + (int64_t)p->warps * slices - 1) / ((int64_t)p->warps * slices);
      if (g2 > (int64_t)occ * num_sms) return false;
      p->grid = (int)g2;
    }
    p->max_chain = 9;
    return true;
  }
  // bwd_filter: groups of 4 (pair: 8) channels x batch slices, ~one wave, <= 32 images per warp
  if (g.C % tp != 0) return false;
  p->groups = (int)(g.C / tp);
  int64_t nsl = std::max<int64_t>(1, ((int64_t)occ * num_sms) / p->groups);
  nsl = std::max<int64_t>(nsl, (g.N + 32 * p->warps - 1) / (32 * p->warps));
  nsl = std::min<int64_t>(nsl, std::min<int64_t>(g.N, 128));
  if (slices > 0) nsl = std::max<int64_t>(std::min<int64_t>(slices, g.N), (g.N + 32 * p->warps - 1) / (32 * p->warps));
  int64_t nps = (g.N + nsl - 1) / nsl;
  nsl = (g.N + nps - 1) / nps;
  p->nslices = (int)nsl;
  p->nps = (int)nps;
  p->grid = (int)(p->groups * nsl);
  const int64_t per_warp = (nps + p->warps - 1) / p->warps;
  int ls = 0;
  while ((1ll << ls) < nsl) ++ls;
  p->max_chain = (int)(g.Wo * (g.Wo / 7) + per_warp + 7 + p->warps + 2 * ls + 1);
  p->ws_bytes = two_level_ws_bytes(p->groups, nsl, g.C);
  return p->max_chain <= 160;
}

// Lane-per-plane kernels: 32-plane warp tasks, W = H in {7, 14}, 3x3 s1 p1 m1, C % 32 == 0.
bool plan_nchw_lane(const Geom& g, int pass, int num_sms, int smem_optin, SmallPlan* p, int warps, int stages,
                    int slices) {
  using namespace small;
  if (g.layout != DWCONV_NCHW || g.m != 1 || g.kh != 3 || g.kw != 3 || g.ph != 1 || g.pw != 1) return false;
  if (g.sh != 1 || g.sw != 1 || g.H != g.W || (g.W != 7 && g.W != 14) || g.C % 32 != 0 || g.N < 1) return false;
  if (pass > 2 || warps < 1 || warps > 8 || stages < 2 || stages > 6) return false;
  if (g.N * g.C >= ((int64_t)1 << 31)) return false;
  const int64_t eb = (g.dtype == DWCONV_F32) ? 4 : 2;
  const int64_t plane = g.H * g.W * eb;
  const bool bf = pass == 2;
  *p = SmallPlan{};
  p->lane = true;
  p->S = 1;
  p->warps = warps;
  p->ns = stages;
  p->slot_bytes = (uint32_t)(((bf ? 2 : 1) * 32 * plane + 15) & ~(int64_t)15);
  p->smem = 64 * warps + warps * stages * (int)p->slot_bytes;
  if (bf) p->smem = std::max(p->smem, 64 * warps + warps * 32 * 9 * 4);
  if (p->smem > smem_optin - 1024) return false;
  SKernelFn fn = lane_kernel_for(g.dtype, pass, (int)g.W);
  if (!fn) return false;
  cudaFuncAttributes fa{};
  if (cudaFuncGetAttributes(&fa, fn) != cudaSuccess) return false;
  if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_optin - (int)fa.sharedSizeBytes) !=
      cudaSuccess)
    return false;
  int occ = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, 32 * warps, p->smem) != cudaSuccess || occ < 1)
    return false;
  p->occ = occ;
  p->sms = num_sms;
  if (!bf) {
    p->ntasks = g.N * g.C / 32;
    p->grid = (int)std::min<int64_t>((p->ntasks + warps - 1) / warps, (int64_t)occ * num_sms);
    p->max_chain = 9;
    return true;
  }
  // bwd_filter: groups of 32 channels x batch slices; the slice count whose busiest SM
  // (ceil(grid / SMs) CTAs of ceil(nps / warps) images per warp) is closest to the even share
  p->groups = (int)(g.C / 32);
  const int64_t N = g.N;
  int64_t nsl = 1;
  if (slices > 0) {
    nsl = std::min<int64_t>(slices, N);
  } else {
    double best = -1.0;
    const double ideal = (double)p->groups * N / ((double)num_sms * warps);
    for (int64_t t = 1; t <= std::min<int64_t>(N, 128); ++t) {
      const int64_t np_ = (N + t - 1) / t, ns_ = (N + np_ - 1) / np_;
      const int64_t grid = p->groups * ns_;
      if (grid > 2 * (int64_t)occ * num_sms && t > 1) break;
      const double sc = ideal / ((double)((grid + num_sms - 1) / num_sms) * ((np_ + warps - 1) / warps));
      if (sc > best + 1e-9) { best = sc; nsl = ns_; }  // ties: fewer CTAs (measured: the per-CTA reduction dominates)
    }
  }
  int64_t nps = (N + nsl - 1) / nsl;
  nsl = (N + nps - 1) / nps;
  p->nslices = (int)nsl;
  p->nps = (int)nps;
  p->grid = (int)(p->groups * nsl);
  int ls = 0;
  while ((1ll << ls) < nsl) ++ls;
  const int64_t H2 = (g.W + 1) / 2;
  p->max_chain = (int)(g.W * H2 + (nps + warps - 1) / warps + warps + 2 * ls + 1);
  p->ws_bytes = two_level_ws_bytes(p->groups, nsl, g.C);
  return p->max_chain <= 160;
}

// Band bwd_filter for large planes (band_bf_kernel): Wo = 28 V, V in {1, 2, 4}.
bool plan_nchw_band_bf(const Geom& g, int num_sms, int smem_optin, SmallPlan* p, int warps, int stages, int rows,
                       int ppw) {
  using namespace small;
  static const int on = env_int("DWCONV_BAND_BF", 1, 0, 1);
  if (!on || g.layout != DWCONV_NCHW || g.m != 1 || g.kh != 3 || g.kw != 3 || g.ph != 1 || g.pw != 1) return false;
  const int S = g.sh;
  if (ppw != 1 && ppw != 2 && ppw != 3) return false;
  const int lanes = (ppw == 2) ? 14 : 28;  // columns over 28 lanes (one plane / a channel pair) or 14 (two planes)
  if (g.sw != S || (S != 1 && S != 2) || g.Wo % lanes != 0 || g.W != S * g.Wo || g.N < 1) return false;
  const int V = (int)(g.Wo / lanes);
  const int64_t eb = (g.dtype == DWCONV_F32) ? 4 : 2;
  if ((g.W * eb) % 16 != 0 || (g.Wo * eb) % 16 != 0 || g.N * g.C >= ((int64_t)1 << 31)) return false;
  if (rows != 7 && rows != 14) return false;
  SKernelFn fn = band_kernel_for(g.dtype, S, V, rows, ppw);
  if (!fn) return false;
  *p = SmallPlan{};
  p->band = true;
  p->R = rows;
  p->V = V;
  p->ppw = ppw;
  p->warps = warps;
  p->ns = stages;
  const int64_t xcap = ((((int64_t)rows - 1) * S + 3) * g.W * eb + 15) & ~(int64_t)15;
  p->slot_bytes = (uint32_t)((ppw == 1 ? 1 : 2) * (xcap + (((int64_t)rows * g.Wo * eb + 15) & ~(int64_t)15)));
  p->smem = 64 * warps + warps * stages * (int)p->slot_bytes;
  if (p->smem > smem_optin - 1024) return false;
  cudaFuncAttributes fa{};
  if (cudaFuncGetAttributes(&fa, fn) != cudaSuccess) return false;
  if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_optin - (int)fa.sharedSizeBytes) !=
      cudaSuccess)
    return false;
  int occ = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, 32 * warps, p->smem) != cudaSuccess || occ < 1)
    return false;
  p->occ = occ;
  p->sms = num_sms;
  p->nbands = (int)((g.Ho + rows - 1) / rows);
  p->cpg = warps * (ppw == 1 ? 1 : 2);
  p->groups = (int)((g.C + p->cpg - 1) / p->cpg);
  // slices: about one wave, <= 64 tasks (image x band) per warp, <= 128 slices
  int64_t nsl = std::max<int64_t>(1, ((int64_t)occ * num_sms) / p->groups);
  nsl = std::max<int64_t>(nsl, (g.N * p->nbands + 63) / 64);
  nsl = std::min<int64_t>(nsl, std::min<int64_t>(g.N, 128));
  int64_t nps = (g.N + nsl - 1) / nsl;
  nsl = (g.N + nps - 1) / nps;
  if (nps * p->nbands > 64) return false;
  p->nslices = (int)nsl;
  p->nps = (int)nps;
  p->grid = (int)(p->groups * nsl);
  int ls = 0;
  while ((1ll << ls) < nsl) ++ls;
  p->max_chain = (int)(rows * V + nps * p->nbands + 5 + 2 * ls + 1);  // xor tree: <= 5 levels
  p->ws_bytes = two_level_ws_bytes(p->groups, nsl, g.C);
  return p->max_chain <= 160;
}

cudaError_t launch_nchw_small(const Geom& g, const SmallPlan& p, int pass, const void* in, const void* in2,
                              const void* w, void* out, float* dw, void* ws, cudaStream_t st) {
  using namespace small;
  SArgs a{};
  a.H = (int)g.H; a.W = (int)g.W; a.Ho = (int)g.Ho; a.Wo = (int)g.Wo;
  a.nbands = p.nbands; a.cpg = p.cpg;
  static const int early = env_int("DWCONV_SMALL_EARLY_PDL", 0, 0, 1);
  a.early_pdl = early && (int64_t)p.grid <= (int64_t)p.occ * p.sms;
  a.in = in; a.in2 = in2; a.out = out; a.w = w; a.dw = dw;
  a.ntasks = p.ntasks;
  a.C = (int)g.C; a.N = (int)g.N;
  a.ns = p.ns; a.slot_bytes = p.slot_bytes;
  a.groups = p.groups; a.nslices = p.nslices; a.nps = p.nps;
  if (pass >= 2) {
    const size_t tick = two_level_tick_bytes(p.groups, p.nslices);
    a.ws_ticket = static_cast<unsigned*>(ws);
    a.ws_part = reinterpret_cast<float*>(static_cast<char*>(ws) + tick);
  }
  SKernelFn fn = p.lane ? lane_kernel_for(g.dtype, pass, (int)g.W)
               : p.band ? band_kernel_for(g.dtype, (int)g.sh, p.V, p.R, p.ppw)
               : p.pair ? pair_kernel_for(pass, (int)g.W) : kernel_for(g.dtype, pass, (int)g.W, p.S);
  if (!fn) return cudaErrorInvalidValue;
  static const bool pdl = env_int("DWCONV_PDL", 1, 0, 1) == 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)p.grid);
  cfg.blockDim = dim3((unsigned)(32 * p.warps));
  cfg.dynamicSmemBytes = (size_t)p.smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, fn, a);
}

}  // namespace dwk
