// nhwc.cu -- the three depthwise passes for NHWC activations ([N][H][W][C]) on
// sm_100a, multiplier m = 1, 3x3 kernels, symmetric padding 1, S in {1,2}
// (other NHWC shapes take the generic kernels).
//
// In NHWC the channels of a pixel are contiguous, so a thread owns a vector of
// VC = 4 consecutive channels (16-B loads for fp32, 8-B for bf16) and consecutive
// lanes own consecutive channel vectors: every warp load is a coalesced run of
// pixels x channels, and the k x k window of a channel vector is k*k vector loads
// whose neighbours are shared by adjacent outputs through L1.  The per-channel
// weights never change along a thread's grid-stride walk when VC*blockDim*grid is
// a multiple of C, so each thread loads its 4 x K*K weights once (transposed to
// [tap][channel] in registers).  Channel pairs go through packed FFMA2 -- the
// operands are naturally aligned pairs, no shuffling.
//
//  * fwd (Eq. 3): thread tile of TH x TW output pixels;
//    the (TH-1)*S+K window rows are loaded one row at a time.
//  * bwd_data (adjoint, reading R9): polyphase tile of TH x TW dx
//    pixels aligned to the stride; the dy window and every tap index are
//    compile-time (tap i = a + PAD - S*(D0 + r)).
//  * bwd_filter (Eq. 4 diagonal, summed over the batch, reading R5): CTA =
//    (group of CVB channel vectors, slice of (n, oh) output rows); PSET pixel
//    sets per channel vector each walk rows in TW-wide blocks.  Deterministic:
//    per block (TW terms) -> running sum over the thread's blocks -> pixel sets
//    pairwise in order -> per-slice partials -> last CTA of the group sums
//    slices pairwise in slice order (integer ticket) and re-zeroes the workspace.
#include <algorithm>
#include <cstdlib>

#include "kernels.h"
#include "nchw_common.cuh"

namespace dwk {
namespace nhwc {

using nchw::VecIO;
constexpr int VC = 4;

struct HArgs {
  const void* in;   // fwd: x, bwd_data: dy, bwd_filter: x
  const void* in2;  // bwd_filter: dy
  const void* w;
  void* out;        // fwd: y, bwd_data: dx
  float* dw;
  float* ws_part;
  unsigned* ws_ticket;
  int N, C, H, W, Ho, Wo;  // x dims and y dims
  int CV;                  // channel vectors per pixel
  int OHB, OWB;            // fwd / bwd_data: tiles along the output rows / columns
  int64_t items;           // fwd / bwd_data: N * OHB * OWB * CV
  // bwd_filter
  int CVB, PSET, groups, nslices, rps;  // channel vectors per CTA, pixel sets, groups, slices, rows per slice
};

template <class T>
__device__ __forceinline__ void load_w(const T* w, int c0, int KK, int q, float* wv) {
#pragma unroll
  for (int v = 0; v < VC; ++v) wv[v] = Elem<T>::ldg(w + (int64_t)(c0 + v) * KK + q);
}

// fwd (BWD = false) and bwd_data (BWD = true)
template <class T, int K, int S, int TH, int TW, bool BWD>
__global__ void __launch_bounds__(256, 2) nhwc_fd_kernel(const HArgs a) {
  constexpr int PAD = (K - 1) / 2, KK = K * K;
  constexpr int D0 = BWD ? floor_div(PAD - K + 1, S) : 0;
  constexpr int NWR = BWD ? floor_div(TH - 1 + PAD, S) - D0 + 1 : (TH - 1) * S + K;
  constexpr int NWC = BWD ? floor_div(TW - 1 + PAD, S) - D0 + 1 : (TW - 1) * S + K;
  static_assert(!BWD || (TH % S == 0 && TW % S == 0), "bwd_data tiles are stride aligned");
  const T* __restrict__ in = static_cast<const T*>(a.in);
  const T* __restrict__ wt = static_cast<const T*>(a.w);
  T* __restrict__ out = static_cast<T*>(a.out);
  const int C = a.C;
  const int IH = BWD ? a.Ho : a.H, IW = BWD ? a.Wo : a.W;  // input (window) plane
  const int OH = BWD ? a.H : a.Ho, OW = BWD ? a.W : a.Wo;  // output plane
  griddep_wait();
  float2 wr[KK][VC / 2];
  int wcv = -1;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < a.items; idx += stride) {
    int64_t rest = idx / a.CV;
    const int cv = (int)(idx - rest * a.CV);
    const int64_t r2 = rest / a.OWB;
    const int owb = (int)(rest - r2 * a.OWB);
    const int64_t n = r2 / a.OHB;
    const int ohb = (int)(r2 - n * a.OHB);
    const int c0 = cv * VC;
    if (cv != wcv) {  // weights of this channel vector, [tap][channel pair]
      wcv = cv;
#pragma unroll
      for (int q = 0; q < KK; ++q) {
        float wv[VC];
        load_w<T>(wt, c0, KK, q, wv);
#pragma unroll
        for (int v = 0; v < VC / 2; ++v) wr[q][v] = make_float2(wv[2 * v], wv[2 * v + 1]);
      }
    }
    const int oh0 = ohb * TH, ow0 = owb * TW;
    const int wr0 = BWD ? oh0 / S + D0 : oh0 * S - PAD;
    const int wc0 = BWD ? ow0 / S + D0 : ow0 * S - PAD;
    float2 acc[TH][TW][VC / 2];
#pragma unroll
    for (int i = 0; i < TH; ++i)
#pragma unroll
      for (int j = 0; j < TW; ++j)
#pragma unroll
        for (int v = 0; v < VC / 2; ++v) acc[i][j][v] = make_float2(0.f, 0.f);
    const T* base = in + (n * IH) * (int64_t)IW * C + c0;
#pragma unroll
    for (int r = 0; r < NWR; ++r) {
      const int ir = wr0 + r;
      const bool rv = (unsigned)ir < (unsigned)IH;
      float xv[NWC][VC];
#pragma unroll
      for (int cc = 0; cc < NWC; ++cc) {
        const int ic = wc0 + cc;
        if (rv && (unsigned)ic < (unsigned)IW) VecIO<T, VC>::load(base + ((int64_t)ir * IW + ic) * C, xv[cc]);
        else
#pragma unroll
          for (int v = 0; v < VC; ++v) xv[cc][v] = 0.f;
      }
#pragma unroll
      for (int ta = 0; ta < TH; ++ta) {
        const int i = BWD ? ta + PAD - S * (D0 + r) : r - ta * S;
        if (i < 0 || i >= K) continue;
#pragma unroll
        for (int tb = 0; tb < TW; ++tb)
#pragma unroll
          for (int cc = 0; cc < NWC; ++cc) {
            const int jj = BWD ? tb + PAD - S * (D0 + cc) : cc - tb * S;
            if (jj < 0 || jj >= K) continue;
#pragma unroll
            for (int v = 0; v < VC / 2; ++v)
              acc[ta][tb][v] = __ffma2_rn(wr[i * K + jj][v], make_float2(xv[cc][2 * v], xv[cc][2 * v + 1]),
                                          acc[ta][tb][v]);
          }
      }
    }
    T* obase = out + (n * OH) * (int64_t)OW * C + c0;
#pragma unroll
    for (int ta = 0; ta < TH; ++ta)
#pragma unroll
      for (int tb = 0; tb < TW; ++tb) {
        const int oh = oh0 + ta, ow = ow0 + tb;
        if (oh < OH && ow < OW) {
          float o[VC];
#pragma unroll
          for (int v = 0; v < VC / 2; ++v) { o[2 * v] = acc[ta][tb][v].x; o[2 * v + 1] = acc[ta][tb][v].y; }
          VecIO<T, VC>::store(obase + ((int64_t)oh * OW + ow) * C, o);
        }
      }
  }
  griddep_launch_dependents();
}

// bwd_filter
template <class T, int K, int S, int TW>
__global__ void __launch_bounds__(256, 2) nhwc_bf_kernel(const HArgs a) {
  constexpr int PAD = (K - 1) / 2, KK = K * K;
  constexpr int NXC = (TW - 1) * S + K;  // x columns of a TW block
  extern __shared__ __align__(16) float red[];  // [256][KK * VC]
  __shared__ unsigned s_last;
  const T* __restrict__ x = static_cast<const T*>(a.in);
  const T* __restrict__ dy = static_cast<const T*>(a.in2);
  const int C = a.C, H = a.H, W = a.W, Ho = a.Ho, Wo = a.Wo;
  const int g = blockIdx.x % a.groups;
  const int sl = blockIdx.x / a.groups;
  const int cvl = threadIdx.x % a.CVB;
  const int ps = threadIdx.x / a.CVB;
  const int cv = g * a.CVB + cvl;
  const bool live = ps < a.PSET && cv < a.CV;
  const int c0 = (live ? cv : 0) * VC;
  const int64_t row0 = (int64_t)sl * a.rps;
  const int64_t row1 = min((int64_t)a.N * Ho, row0 + a.rps);
  const int owblocks = (Wo + TW - 1) / TW;
  griddep_wait();
  float2 run[KK][VC / 2];
#pragma unroll
  for (int q = 0; q < KK; ++q)
#pragma unroll
    for (int v = 0; v < VC / 2; ++v) run[q][v] = make_float2(0.f, 0.f);
  if (live) {
    for (int64_t rr = row0 + ps; rr < row1; rr += a.PSET) {
      const int64_t n = rr / Ho;
      const int oh = (int)(rr - n * Ho);
      for (int ob = 0; ob < owblocks; ++ob) {
        const int ow0 = ob * TW;
        float dv[TW][VC];
#pragma unroll
        for (int tb = 0; tb < TW; ++tb) {
          if (ow0 + tb < Wo) VecIO<T, VC>::load(dy + (((n * Ho + oh) * (int64_t)Wo) + ow0 + tb) * C + c0, dv[tb]);
          else
#pragma unroll
            for (int v = 0; v < VC; ++v) dv[tb][v] = 0.f;
        }
        float2 loc[KK][VC / 2];
#pragma unroll
        for (int q = 0; q < KK; ++q)
#pragma unroll
          for (int v = 0; v < VC / 2; ++v) loc[q][v] = make_float2(0.f, 0.f);
#pragma unroll
        for (int i = 0; i < K; ++i) {
          const int ih = oh * S - PAD + i;
          const bool rv = (unsigned)ih < (unsigned)H;
          float xv[NXC][VC];
#pragma unroll
          for (int cc = 0; cc < NXC; ++cc) {
            const int iw = ow0 * S - PAD + cc;
            if (rv && (unsigned)iw < (unsigned)W) VecIO<T, VC>::load(x + (((n * H + ih) * (int64_t)W) + iw) * C + c0, xv[cc]);
            else
#pragma unroll
              for (int v = 0; v < VC; ++v) xv[cc][v] = 0.f;
          }
#pragma unroll
          for (int tb = 0; tb < TW; ++tb)
#pragma unroll
            for (int jj = 0; jj < K; ++jj)
#pragma unroll
              for (int v = 0; v < VC / 2; ++v)
                loc[i * K + jj][v] = __ffma2_rn(make_float2(xv[tb * S + jj][2 * v], xv[tb * S + jj][2 * v + 1]),
                                                make_float2(dv[tb][2 * v], dv[tb][2 * v + 1]), loc[i * K + jj][v]);
        }
#pragma unroll
        for (int q = 0; q < KK; ++q)
#pragma unroll
          for (int v = 0; v < VC / 2; ++v) {
            run[q][v].x += loc[q][v].x;
            run[q][v].y += loc[q][v].y;
          }
      }
    }
  }
  griddep_launch_dependents();
  // ---- pixel sets of a channel vector, in order; then the slice partial
#pragma unroll
  for (int q = 0; q < KK; ++q)
#pragma unroll
    for (int v = 0; v < VC / 2; ++v) {
      red[threadIdx.x * KK * VC + q * VC + 2 * v] = run[q][v].x;
      red[threadIdx.x * KK * VC + q * VC + 2 * v + 1] = run[q][v].y;
    }
  __syncthreads();
  const int nvec = min(a.CVB, a.CV - g * a.CVB);
  float* part = a.ws_part + (int64_t)sl * C * KK;
  for (int e = threadIdx.x; e < nvec * VC * KK; e += blockDim.x) {
    const int cl = e / (VC * KK);       // channel vector within the group
    const int rem = e - cl * VC * KK;   // q * VC + v
    const int q = rem / VC, v = rem - q * VC;
    // pixel sets in order, pairwise (binary counter): depth log2(PSET)
    float stk[10];
    int top = 0;
    for (int p = 0; p < a.PSET; ++p) {
      float cur = red[(p * a.CVB + cl) * KK * VC + rem];
      int bits = p;
      while (bits & 1) { cur = stk[--top] + cur; bits >>= 1; }
      stk[top++] = cur;
    }
    float s = stk[--top];
    while (top > 0) s = stk[--top] + s;
    part[(int64_t)((g * a.CVB + cl) * VC + v) * KK + q] = s;  // dw layout [c][tap]
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned prev = atomicAdd(&a.ws_ticket[g], 1u);
    s_last = (prev == (unsigned)(a.nslices - 1)) ? 1u : 0u;
  }
  __syncthreads();
  if (s_last) {
    __threadfence();
    const int64_t e0 = (int64_t)g * a.CVB * VC * KK;
    const int nvals = nvec * VC * KK;
    const int64_t sstride = (int64_t)C * KK;
    for (int idx = threadIdx.x; idx < nvals; idx += blockDim.x) {
      float stk[16];
      int top = 0;
      for (int s0 = 0; s0 < a.nslices; s0 += 32) {  // 32 loads in flight per thread
        float vals[32];
#pragma unroll
        for (int u = 0; u < 32; ++u)
          vals[u] = (s0 + u < a.nslices) ? __ldcg(a.ws_part + (s0 + u) * sstride + e0 + idx) : 0.f;
#pragma unroll
        for (int u = 0; u < 32; ++u)
          if (s0 + u < a.nslices) __stcg(a.ws_part + (s0 + u) * sstride + e0 + idx, 0.f);
#pragma unroll
        for (int u = 0; u < 32; ++u) {
          const int s = s0 + u;
          if (s < a.nslices) {
            float cur = vals[u];
            int bits = s;
            while (bits & 1) { cur = stk[--top] + cur; bits >>= 1; }
            stk[top++] = cur;
          }
        }
      }
      float tot = stk[--top];
      while (top > 0) tot = stk[--top] + tot;
      a.dw[e0 + idx] = tot;
    }
    if (threadIdx.x == 0) a.ws_ticket[g] = 0u;
  }
}

using HKernelFn = void (*)(HArgs);

template <class T, int K, int S>
HKernelFn fd_pick(bool bwd) {
  // fwd tile TH x TW; bwd_data tiles are stride aligned
  if (bwd) return S == 1 ? nhwc_fd_kernel<T, K, 1, 2, 4, true> : nhwc_fd_kernel<T, K, 2, 2, 2, true>;
  return S == 1 ? nhwc_fd_kernel<T, K, 1, 2, 4, false> : nhwc_fd_kernel<T, K, 2, 1, 4, false>;
}
template <class T>
HKernelFn fd_pick_k(int K, int S, bool bwd) {
  if (K == 3) return S == 1 ? fd_pick<T, 3, 1>(bwd) : fd_pick<T, 3, 2>(bwd);
  return nullptr;  // K = 5, 7: the per-thread tap tables do not fit in registers; generic kernels
}
constexpr int kBfTW = 4;
template <class T>
HKernelFn bf_pick_k(int K, int S) {
  if (K == 3) return S == 1 ? nhwc_bf_kernel<T, 3, 1, kBfTW> : nhwc_bf_kernel<T, 3, 2, kBfTW>;
  return nullptr;
}

static cudaError_t launch(HKernelFn fn, int grid, int smem, cudaStream_t st, const HArgs& a) {
  static const bool pdl = []() {
    const char* e = dev_knob("DWCONV_PDL");
    return !(e && e[0] == '0');
  }();
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(256u);
  cfg.dynamicSmemBytes = (size_t)smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, fn, a);
}

static HArgs base(const Geom& g) {
  HArgs a{};
  a.N = (int)g.N; a.C = (int)g.C; a.H = (int)g.H; a.W = (int)g.W; a.Ho = (int)g.Ho; a.Wo = (int)g.Wo;
  a.CV = (int)(g.C / VC);
  return a;
}

}  // namespace nhwc

bool plan_nhwc(const Geom& g, int pass, int num_sms, NhwcPlan* p) {
  using namespace nhwc;
  if (g.layout != DWCONV_NHWC || g.m != 1) return false;
  const int K = g.kh;
  if (g.kw != K || K != 3) return false;
  if (g.sw != g.sh || (g.sh != 1 && g.sh != 2) || g.ph != (K - 1) / 2 || g.pw != (K - 1) / 2) return false;
  if (g.C % VC != 0 || g.C > (1 << 20) || g.N * g.H * g.W > ((int64_t)1 << 40)) return false;
  *p = NhwcPlan{};
  const int S = g.sh;
  const int KK = K * K;
  if (pass != DWCONV_PASS_BWD_FILTER) {
    const bool bwd = pass == DWCONV_PASS_BWD_DATA;
    const int TH = bwd ? 2 : (S == 1 ? 2 : 1);
    const int TW = bwd ? (S == 1 ? 4 : 2) : 4;
    const int64_t OH = bwd ? g.H : g.Ho, OW = bwd ? g.W : g.Wo;
    const int64_t OHB = (OH + TH - 1) / TH, OWB = (OW + TW - 1) / TW;
    p->TH = TH; p->TW = TW;
    p->OHB = (int)OHB; p->OWB = (int)OWB;
    p->items = g.N * OHB * OWB * (g.C / VC);
    HKernelFn fn = (g.dtype == DWCONV_F32) ? fd_pick_k<float>(K, S, bwd) : fd_pick_k<__nv_bfloat16>(K, S, bwd);
    if (!fn) return false;
    int occ = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, 256, 0) != cudaSuccess || occ < 1) return false;
    int64_t grid = std::min<int64_t>((p->items + 255) / 256, (int64_t)occ * num_sms);
    // keep each thread on one channel vector: threads in the grid a multiple of C / VC
    const int64_t cv = g.C / VC;
    if ((256 % cv) != 0 && cv % 256 == 0) {
      // grid * 256 is a multiple of cv iff grid is a multiple of cv / 256
      const int64_t q = cv / 256;
      grid = std::max<int64_t>(q, grid / q * q);
    }
    p->grid = (int)std::max<int64_t>(1, grid);
    p->threads = 256;
    p->smem = 0;
    p->max_chain = KK;
    return true;
  }
  // bwd_filter
  // a CTA owns CVB <= 8 channel vectors (<= 128 B of every pixel) and PSET pixel
  // sets each: groups run in parallel and each group's finalize stays small
  const int64_t CV = g.C / VC;
  const int CVB = (int)std::min<int64_t>(CV, 8);
  const int PSET = 256 / CVB;
  const int64_t groups = (CV + CVB - 1) / CVB;
  const int TW = kBfTW;
  const int64_t rows = g.N * g.Ho;
  const int64_t bpr = (g.Wo + TW - 1) / TW;  // blocks per row
  HKernelFn fn = (g.dtype == DWCONV_F32) ? bf_pick_k<float>(K, S) : bf_pick_k<__nv_bfloat16>(K, S);
  if (!fn) return false;
  const int smem = 256 * KK * VC * 4;
  static bool attr_set[2][3][2] = {};
  bool& done = attr_set[g.dtype == DWCONV_F32 ? 0 : 1][0][S - 1];
  if (!done) {
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    done = true;
  }
  int occ = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, 256, smem) != cudaSuccess || occ < 1) return false;
  // slices: ~one wave of CTAs (measured best: each CTA's epilogue is a fixed cost),
  // and <= 120 blocks per thread (running-sum chain)
  static const int waves = []() { const char* e = dev_knob("DWCONV_NHWC_BF_WAVES"); return e ? std::max(1, std::atoi(e)) : 1; }();
  int64_t nsl = std::max<int64_t>(1, ((int64_t)waves * occ * num_sms + groups - 1) / groups);
  nsl = std::max<int64_t>(nsl, (rows * bpr + (int64_t)PSET * 120 - 1) / ((int64_t)PSET * 120));
  nsl = std::min<int64_t>(nsl, std::min<int64_t>(rows, 256));
  const int64_t rps = (rows + nsl - 1) / nsl;
  nsl = (rows + rps - 1) / rps;
  const int64_t bpt = ((rps + PSET - 1) / PSET) * bpr;  // blocks per thread
  p->threads = 256;
  p->smem = smem;
  p->TW = TW;
  p->CVB = CVB; p->PSET = PSET; p->groups = (int)groups; p->nslices = (int)nsl; p->rps = (int)rps;
  p->grid = (int)(groups * nsl);
  int lg = 0;
  while ((1ll << lg) < nsl) ++lg;
  int lp = 0;
  while ((1 << lp) < PSET) ++lp;
  p->max_chain = (int)(TW + bpt + lp + 2 * lg + 1);
  const size_t tick = ((size_t)groups * 4 + 15) / 16 * 16;
  p->ws_bytes = tick + (size_t)nsl * g.C * KK * 4;
  return p->max_chain <= 160 && p->grid > 0;
}

cudaError_t launch_nhwc_fd(const Geom& g, const NhwcPlan& p, int pass, const void* in, const void* w, void* out,
                           cudaStream_t st) {
  using namespace nhwc;
  const bool bwd = pass == DWCONV_PASS_BWD_DATA;
  HKernelFn fn = (g.dtype == DWCONV_F32) ? fd_pick_k<float>(g.kh, g.sh, bwd) : fd_pick_k<__nv_bfloat16>(g.kh, g.sh, bwd);
  HArgs a = base(g);
  a.in = in; a.w = w; a.out = out;
  a.OHB = p.OHB; a.OWB = p.OWB; a.items = p.items;
  return launch(fn, p.grid, 0, st, a);
}

cudaError_t launch_nhwc_bwd_filter(const Geom& g, const NhwcPlan& p, const void* x, const void* dy, float* dw,
                                   void* ws, cudaStream_t st) {
  using namespace nhwc;
  HKernelFn fn = (g.dtype == DWCONV_F32) ? bf_pick_k<float>(g.kh, g.sh) : bf_pick_k<__nv_bfloat16>(g.kh, g.sh);
  HArgs a = base(g);
  a.in = x; a.in2 = dy; a.dw = dw;
  const size_t tick = ((size_t)p.groups * 4 + 15) / 16 * 16;
  a.ws_ticket = static_cast<unsigned*>(ws);
  a.ws_part = reinterpret_cast<float*>(static_cast<char*>(ws) + tick);
  a.CVB = p.CVB; a.PSET = p.PSET; a.groups = p.groups; a.nslices = p.nslices; a.rps = p.rps;
  return launch(fn, p.grid, p.smem, st, a);
}

}  // namespace dwk
