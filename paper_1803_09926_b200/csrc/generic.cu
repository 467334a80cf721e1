// generic.cu -- the correctness net: any kernel size, stride, padding, multiplier,
// layout and alignment.  One thread per output element with plain global loads
// (fwd, bwd_data); one CTA per (output channel, tap) with a bounded-chain
// blocked summation and a fixed tree (bwd_filter).  Used when no fast family
// applies; never a CPU fallback.
//
// Definitions follow include/dwconv.h (PAPER.md P:173-176, P:235-236 forward;
// Eq. 4 P:295-301 filter gradient; reading R9 input gradient).
#include "common.cuh"
#include "kernels.h"

namespace dwk {
namespace {

__device__ __forceinline__ int64_t act_index(int layout, int64_t C, int64_t H, int64_t W, int64_t n, int64_t c,
                                             int64_t h, int64_t w) {
  return layout == DWCONV_NCHW ? ((n * C + c) * H + h) * W + w : ((n * H + h) * W + w) * C + c;
}

// Decompose a flat index of an activation tensor in its memory order.
__device__ __forceinline__ void act_coords(int layout, int64_t e, int64_t C, int64_t H, int64_t W, int64_t& n,
                                           int64_t& c, int64_t& h, int64_t& w) {
  if (layout == DWCONV_NCHW) {
    w = e % W; e /= W;
    h = e % H; e /= H;
    c = e % C; n = e / C;
  } else {
    c = e % C; e /= C;
    w = e % W; e /= W;
    h = e % H; n = e / H;
  }
}

template <class T>
__global__ void generic_fwd(const Geom g, const T* __restrict__ x, const T* __restrict__ wt, T* __restrict__ y) {
  const int64_t Co = g.C * g.m;
  const int64_t total = g.N * Co * g.Ho * g.Wo;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    int64_t n, o, oh, ow;
    act_coords(g.layout, e, Co, g.Ho, g.Wo, n, o, oh, ow);
    const int64_t c = o / g.m;
    float acc = 0.f;
    for (int i = 0; i < g.kh; ++i) {
      const int64_t ih = oh * g.sh - g.ph + i;
      if (ih < 0 || ih >= g.H) continue;
      for (int jj = 0; jj < g.kw; ++jj) {
        const int64_t iw = ow * g.sw - g.pw + jj;
        if (iw < 0 || iw >= g.W) continue;
        acc = fmaf(Elem<T>::ldg(wt + (o * g.kh + i) * g.kw + jj),
                   Elem<T>::ldg(x + act_index(g.layout, g.C, g.H, g.W, n, c, ih, iw)), acc);
      }
    }
    Elem<T>::store(y + e, acc);
  }
}

template <class T>
__global__ void generic_bwd_data(const Geom g, const T* __restrict__ dy, const T* __restrict__ wt,
                                 T* __restrict__ dx) {
  const int64_t Co = g.C * g.m;
  const int64_t total = g.N * g.C * g.H * g.W;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    int64_t n, c, ih, iw;
    act_coords(g.layout, e, g.C, g.H, g.W, n, c, ih, iw);
    float acc = 0.f;
    for (int j = 0; j < g.m; ++j) {  // per-j partial sums, then a chain of m adds (R5 iii)
      const int64_t o = c * g.m + j;
      float part = 0.f;
      for (int i = 0; i < g.kh; ++i) {
        const int64_t th = ih + g.ph - i;
        if (th < 0 || th % g.sh != 0) continue;
        const int64_t oh = th / g.sh;
        if (oh >= g.Ho) continue;
        for (int jj = 0; jj < g.kw; ++jj) {
          const int64_t tw = iw + g.pw - jj;
          if (tw < 0 || tw % g.sw != 0) continue;
          const int64_t ow = tw / g.sw;
          if (ow >= g.Wo) continue;
          part = fmaf(Elem<T>::ldg(wt + (o * g.kh + i) * g.kw + jj),
                      Elem<T>::ldg(dy + act_index(g.layout, Co, g.Ho, g.Wo, n, o, oh, ow)), part);
        }
      }
      acc = (j == 0) ? part : acc + part;
    }
    Elem<T>::store(dx + e, acc);
  }
}

// One CTA per (o, i, jj).  Each thread sums its positions in blocks of 64
// products (level 1), blocks into super-blocks of 64 (level 2), then a running
// level-3 sum; the CTA then combines threads with a fixed shuffle/smem tree.
template <class T>
__global__ void __launch_bounds__(256) generic_bwd_filter(const Geom g, const T* __restrict__ x,
                                                          const T* __restrict__ dy, float* __restrict__ dw) {
  const int64_t Co = g.C * g.m;
  const int k2 = g.kh * g.kw;
  const int64_t o = blockIdx.x / k2;
  const int tap = blockIdx.x % k2;
  const int i = tap / g.kw, jj = tap % g.kw;
  const int64_t c = o / g.m;
  const int64_t npos = g.N * g.Ho * g.Wo;
  float l1 = 0.f, l2 = 0.f, l3 = 0.f;
  int c1 = 0, c2 = 0;
  for (int64_t pidx = threadIdx.x; pidx < npos; pidx += blockDim.x) {
    const int64_t ow = pidx % g.Wo;
    const int64_t t = pidx / g.Wo;
    const int64_t oh = t % g.Ho;
    const int64_t n = t / g.Ho;
    const int64_t ih = oh * g.sh - g.ph + i, iw = ow * g.sw - g.pw + jj;
    if (ih >= 0 && ih < g.H && iw >= 0 && iw < g.W) {
      l1 = fmaf(Elem<T>::ldg(x + act_index(g.layout, g.C, g.H, g.W, n, c, ih, iw)),
                Elem<T>::ldg(dy + act_index(g.layout, Co, g.Ho, g.Wo, n, o, oh, ow)), l1);
    }
    if (++c1 == 64) {
      l2 += l1; l1 = 0.f; c1 = 0;
      if (++c2 == 64) { l3 += l2; l2 = 0.f; c2 = 0; }
    }
  }
  float v = l3 + (l2 + l1);
  for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  __shared__ float red[32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) red[warp] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    int nw = blockDim.x >> 5;
    // fixed pairwise tree over warps
    for (int stride = 1; stride < nw; stride <<= 1)
      for (int a = 0; a + stride < nw; a += 2 * stride) red[a] += red[a + stride];
    dw[o * k2 + tap] = red[0];
  }
}

template <class T>
cudaError_t fwd_t(const Geom& g, const void* x, const void* w, void* y, cudaStream_t st) {
  const int64_t total = g.N * g.C * g.m * g.Ho * g.Wo;
  if (total == 0) return cudaSuccess;
  const int threads = 256;
  const int64_t blocks = (total + threads - 1) / threads;
  const int grid = (int)(blocks < 148 * 64 ? blocks : 148 * 64);
  generic_fwd<T><<<grid, threads, 0, st>>>(g, (const T*)x, (const T*)w, (T*)y);
  return cudaGetLastError();
}
template <class T>
cudaError_t bwd_data_t(const Geom& g, const void* dy, const void* w, void* dx, cudaStream_t st) {
  const int64_t total = g.N * g.C * g.H * g.W;
  if (total == 0) return cudaSuccess;
  const int threads = 256;
  const int64_t blocks = (total + threads - 1) / threads;
  const int grid = (int)(blocks < 148 * 64 ? blocks : 148 * 64);
  generic_bwd_data<T><<<grid, threads, 0, st>>>(g, (const T*)dy, (const T*)w, (T*)dx);
  return cudaGetLastError();
}
template <class T>
cudaError_t bwd_filter_t(const Geom& g, const void* x, const void* dy, float* dw, cudaStream_t st) {
  const int64_t blocks = g.C * g.m * g.kh * g.kw;
  generic_bwd_filter<T><<<(unsigned)blocks, 256, 0, st>>>(g, (const T*)x, (const T*)dy, dw);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_generic_fwd(const Geom& g, const void* x, const void* w, void* y, cudaStream_t st) {
  return g.dtype == DWCONV_F32 ? fwd_t<float>(g, x, w, y, st) : fwd_t<__nv_bfloat16>(g, x, w, y, st);
}
cudaError_t launch_generic_bwd_data(const Geom& g, const void* dy, const void* w, void* dx, cudaStream_t st) {
  return g.dtype == DWCONV_F32 ? bwd_data_t<float>(g, dy, w, dx, st) : bwd_data_t<__nv_bfloat16>(g, dy, w, dx, st);
}
cudaError_t launch_generic_bwd_filter(const Geom& g, const void* x, const void* dy, float* dw, cudaStream_t st) {
  return g.dtype == DWCONV_F32 ? bwd_filter_t<float>(g, x, dy, dw, st)
                               : bwd_filter_t<__nv_bfloat16>(g, x, dy, dw, st);
}

}  // namespace dwk
