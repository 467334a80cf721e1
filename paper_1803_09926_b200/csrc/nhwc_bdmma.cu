// nhwc_bdmma.cu -- the paper's diagonalwise refactorization executed on the
// 5th-generation tensor cores: a MEASURED variant, NHWC bf16,
// m = 1, stride 1, K in {3, 5, 7}, group size S in {16, 32, 64}.
//
// The paper (§III-A, Eqs. 1-3) scatters the depthwise weights
// of a group of S channels into a block-diagonal S x S matrix per tap, so that a
// standard convolution -- a GEMM -- computes the depthwise result with S-fold
// redundant multiply-adds (grouping, §III-B; the group-size
// sweep, Fig. 5).  Here the standard convolution is an implicit GEMM
// on tcgen05:
//
//   for every tap (i, j):  D[p, o] += sum_{c in group} X[p + i*BW + j, c] * Wdiag_{ij}[o, c]
//
//   * A (M = 128 rows = flat output positions p, K = channels): the NHWC input box
//     staged by ONE 4-D TMA load in the SWIZZLE_128B layout -- one 128-B row per
//     pixel (64 bf16 channels), BW = 32 pixels per staged row.  Output position p
//     = r * BW + c reads input pixel p + i*BW + j of the box, so the tap's A
//     operand is the same staged box with its descriptor start shifted by
//     (i*BW + j) rows: no data movement per tap.  Flat positions with c >= TW =
//     BW - K + 1 are computed and discarded (the implicit-GEMM "ragged columns").
//   * B (N = S output channels, K = 16 input channels per MMA): diag_S(w[:, i, j])
//     in the K-major no-swizzle layout, built once per CTA in shared memory for the
//     CTA's 64-channel block (every tap, every group, every 16-channel K chunk).
//   * D: fp32 in TMEM, 64 columns per accumulator (group g owns columns g*S ..);
//     4 accumulators so the epilogue of one M tile overlaps the MMAs of the next.
//
// Per tap and 64 channels the MMAs perform 128 * 64 * S multiply-adds of which
// 128 * 64 are useful: the S-fold redundancy the paper trades for GEMM
// efficiency.  bf16 x bf16 products are exact in the fp32 accumulator, so the
// parity contract (R13) is unchanged; the summation order differs from
// the stencil's (tensor-core accumulation), which R13 allows.
//
// Warp roles (192 threads): warp 0 lane 0 = TMA producer (ring of 2 input
// stages, full/empty mbarriers); warp 1 = TMEM allocator + lane 0 issues every
// tcgen05.mma and commits (tcgen05.commit -> mbarrier) the accumulator to the
// epilogue and the stage back to the producer; warps 2-5 = epilogue (warp w reads
// TMEM lanes 32*(w%4) .. +31 with tcgen05.ld.32x32b, packs bf16 and stores the
// pixel's 64 channels -- 128 contiguous bytes -- straight to HBM).
//
// bwd_data (stride 1) is the same GEMM over dy with the kernel rotated by 180
// degrees and padding K-1-p (reading R9).
#include <cuda.h>

#include <mutex>
#include <vector>

#include "common.cuh"
#include "kernels.h"

namespace dwk {
namespace bdmma {

constexpr int BW = 32;                 // staged box width in pixels = flat row pitch of the implicit GEMM
constexpr int NS = 2;                  // input ring stages
constexpr int kThreads = 224;            // producer, 2 MMA issuers, 4 epilogue warps
constexpr uint32_t kTmemCols = 256;    // accumulators: 2 stages x MT tiles x CB fp32 columns
// Channel block CB (16 / 32 / 64 bf16 = one 32 / 64 / 128-B swizzled row per pixel): the TMA
// box, the tensor core's A rows and the accumulator width.  TH output rows per tile keep a
// stage's box near the same size: TH * CB = 512, MT = TH * BW / 128 M tiles per tile.
template <int CB> struct Blk {
  static constexpr int TH = 512 / CB;
  static constexpr int MT = TH * BW / 128;
  static constexpr int NACC = 2 * MT;
  static constexpr int ROWB = CB * 2;                          // bytes per staged pixel
  static constexpr uint32_t LAYOUT = CB == 64 ? 2 : (CB == 32 ? 4 : 6);  // UMMA SWIZZLE_128B / 64B / 32B
  static_assert(NACC * CB == (int)kTmemCols, "TMEM budget");
};

struct Args {
  __nv_bfloat16* out;
  const __nv_bfloat16* w;
  int C, OH, OW, K, pad;
  int TW;                  // valid output columns per tile = BW - K + 1
  int tiles_h, tiles_w;    // tiles per image
  int tiles_per_cb;        // N * tiles_h * tiles_w
  int ctas_per_cb;
  uint32_t stage_bytes;    // (BH + 1) * BW * ROWB (one spare row: ragged flat columns read past the box)
  uint32_t box_bytes;      // BH * BW * ROWB
  uint32_t bw_bytes;       // diagonal weight tiles
  int flip;                // bwd_data: kernel rotated 180 degrees
};

__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* tm, int c0, int c1, int c2, int c3,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];"
      ::"r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(tm)), "r"(c0), "r"(c1), "r"(c2), "r"(c3),
      "r"(smem_u32(bar))
      : "memory");
}

// tcgen05 shared-memory matrix descriptor (sm_100 "version 1"): start, leading /
// stride byte offsets (16-B units), base offset of a start that is not aligned to
// the swizzle pattern, layout type (0 = none, 2 = SWIZZLE_128B).
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr, uint32_t lbo, uint32_t sbo, uint32_t layout,
                                              uint32_t base_off) {
  return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46) | ((uint64_t)(base_off & 7) << 49) |
         ((uint64_t)(layout & 7) << 61);
}

// kind::f16 instruction descriptor: D fp32, A and B bf16, both K-major, M x N.
__host__ __device__ constexpr uint32_t instr_desc(int M, int N) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void mma_bf16(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// 16 TMEM columns of this warp's 32 lanes -> 16 registers per thread.
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t* v) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ uint32_t pack_bf16(uint32_t lo, uint32_t hi) {
  __nv_bfloat162 h = __floats2bfloat162_rn(__uint_as_float(lo), __uint_as_float(hi));
  return *reinterpret_cast<uint32_t*>(&h);
}

template <int K, int S, int CB>
__global__ void __launch_bounds__(kThreads, 1) bdmma_kernel(const __grid_constant__ CUtensorMap tm, const Args a) {
  constexpr int G = CB / S;      // groups per channel block
  constexpr int KC = S / 16;     // 16-channel K chunks per group
  constexpr int TH = Blk<CB>::TH, MT = Blk<CB>::MT, NACC = Blk<CB>::NACC, ROWB = Blk<CB>::ROWB;
  constexpr uint32_t kIdesc = instr_desc(128, S);
  extern __shared__ unsigned char smem_raw[];
  // 1024-B alignment for the swizzled stages (the host adds 1 KB of slack)
  unsigned char* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  // [barriers + TMEM slot: 1 KB][stages (1024-B aligned)][diagonal weight tiles]
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem);
  unsigned char* stages = smem + 1024;
  unsigned char* bw = stages + NS * a.stage_bytes;
  uint64_t* full = bars;
  uint64_t* empty = bars + NS;
  uint64_t* tfull = bars + 2 * NS;
  uint64_t* tempty = bars + 2 * NS + NACC;
  uint32_t* tbase_slot = reinterpret_cast<uint32_t*>(bars + 2 * NS + 2 * NACC);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int cb = blockIdx.x / a.ctas_per_cb;
  const int local = blockIdx.x - cb * a.ctas_per_cb;

  if (tid == 0) {
    for (int i = 0; i < NS; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < NACC; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 4);
    }
    fence_mbar_init();
  }
  __syncthreads();  // barrier inits visible before any other shared-memory traffic (TMEM alloc included)
  if (warp == 3) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tbase_slot)),
                 "n"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  griddep_wait();  // w (and the input) may come from the previous kernel
  // B: diag_S(w[c0 + g*S + n, tap]) per (tap, group, K chunk): [S rows (n) x 16 K] bf16,
  // K-major interleave: core matrix (n/8, k/8) at ((n/8)*2 + k/8)*128 B, row n%8 at 16 B.
  {
    const int KK = K * K;
    uint4* z = reinterpret_cast<uint4*>(bw);
    for (uint32_t i = tid; i < a.bw_bytes / 16; i += kThreads) z[i] = make_uint4(0, 0, 0, 0);
    __syncthreads();
    const int c0 = cb * CB;
    for (int e = tid; e < KK * CB; e += kThreads) {
      const int tap = e / CB, ch = e - tap * CB;    // channel within the block
      const int g = ch / S, n = ch - g * S, kc = n >> 4, k = n & 15;
      const int src_tap = a.flip ? (KK - 1 - tap) : tap;
      const __nv_bfloat16 v = a.w[(size_t)(c0 + ch) * KK + src_tap];
      unsigned char* blk = bw + (size_t)(((tap * G + g) * KC + kc) * S * 32);
      *reinterpret_cast<__nv_bfloat16*>(blk + ((n >> 3) * 2 + (k >> 3)) * 128 + (n & 7) * 16 + (k & 7) * 2) = v;
    }
  }
  fence_proxy_async_smem();  // generic-proxy writes of B -> visible to the tensor core (async proxy)
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tbase_slot;
  const int per_img = a.tiles_h * a.tiles_w;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      int it = 0;
      for (int t = local; t < a.tiles_per_cb; t += a.ctas_per_cb, ++it) {
        const int s = it % NS;
        if (it >= NS) mbar_wait(&empty[s], ((it / NS) & 1) ^ 1);
        const int n = t / per_img, r = t - n * per_img;
        const int th = r / a.tiles_w, tw = r - th * a.tiles_w;
        mbar_arrive_expect_tx(&full[s], a.box_bytes);
        tma_load_4d(stages + (size_t)s * a.stage_bytes, &tm, cb * CB, tw * a.TW - a.pad, th * TH - a.pad, n,
                    &full[s]);
      }
    }
  } else if (warp == 1 || warp == 2) {
    // ------------------------------------------------------------ MMA issuers
    // Warp 1 issues the MMAs of the tiles in ring stage 0, warp 2 those of stage 1: the
    // tensor core runs the two instruction streams concurrently, while MMAs of one stream
    // execute one after another (measured: one stream keeps the tensor core's shared-memory
    // operand reads at ~1/3 of the SMEM bandwidth, ~110 clk per M=128 K=16 MMA).
    if (lane == 0) {
      const int s = warp - 1;
      const uint32_t st0 = smem_u32(stages), bw0 = smem_u32(bw);  // < 2^18: start field never carries
      const uint32_t sa = st0 + (uint32_t)s * a.stage_bytes;
      const uint64_t abase = smem_desc(sa, 16, 8 * ROWB, Blk<CB>::LAYOUT, 0);
      const uint64_t bbase = smem_desc(bw0, 128, 256, 0, 0);
      int it = s;
      for (int t = local + s * a.ctas_per_cb; t < a.tiles_per_cb; t += NS * a.ctas_per_cb, it += NS) {
        mbar_wait(&full[s], (it / NS) & 1);
        // this stage's MT accumulators: wait until the epilogue has drained each
        if (it >= NS)
          for (int mt = 0; mt < MT; ++mt) mbar_wait(&tempty[s * MT + mt], ((it / NS) & 1) ^ 1);
        tc_fence_after();
        // taps outer, M tiles inner: consecutive MMAs accumulate into different TMEM
        // accumulators (independent chains); descriptors advance by adding to the
        // start-address field (16-B units) of a base descriptor
#pragma unroll 1
        for (int tap = 0; tap < K * K; ++tap) {
          const int i = tap / K, j = tap - i * K;
          const uint32_t arow = (uint32_t)((i * BW + j) * ROWB);
#pragma unroll
          for (int mt = 0; mt < MT; ++mt) {
            const uint32_t d0 = tbase + (uint32_t)((s * MT + mt) * CB);
#pragma unroll
            for (int g = 0; g < G; ++g) {
#pragma unroll
              for (int kc = 0; kc < KC; ++kc) {
                // base offset 0 at ANY row shift: the swizzle XOR is taken from the absolute
                // shared-memory address, like the TMA write (tools/umma_probe.cu: every shift 0..127
                // exact with 0, wrong with (addr >> 7) & 7)
                const uint64_t ad = abase + ((arow + (uint32_t)(mt * 128 * ROWB + (g * S + kc * 16) * 2)) >> 4);
                const uint64_t bd = bbase + ((uint32_t)(((tap * G + g) * KC + kc) * S * 32) >> 4);
                mma_bf16(d0 + (uint32_t)(g * S), ad, bd, kIdesc, (tap | kc) != 0);
              }
            }
          }
        }
        for (int mt = 0; mt < MT; ++mt) mma_commit(&tfull[s * MT + mt]);
        mma_commit(&empty[s]);  // the stage is free once every MMA reading it has completed
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue
    const int q = warp & 3;  // TMEM lane quarter this warp may access (warps 3-6 cover all four)
    int acc_it = 0;
    for (int t = local; t < a.tiles_per_cb; t += a.ctas_per_cb) {
      const int n = t / per_img, r0 = t - n * per_img;
      const int th = r0 / a.tiles_w, tw = r0 - th * a.tiles_w;
      const int oh0 = th * TH, ow0 = tw * a.TW;
      for (int mt = 0; mt < MT; ++mt, ++acc_it) {
        const int ac = acc_it % NACC;
        mbar_wait(&tfull[ac], (acc_it / NACC) & 1);
        tc_fence_after();
        const int row = mt * 128 + q * 32 + lane;
        const int r = row / BW, c = row - r * BW;
        const uint32_t ta = tbase + ((uint32_t)(q * 32) << 16) + (uint32_t)(ac * CB);
        uint32_t v[CB];
#pragma unroll
        for (int u = 0; u < CB / 16; ++u) tmem_ld16(ta + 16 * u, &v[16 * u]);
        tmem_ld_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[ac]);
        const int oh = oh0 + r, ow = ow0 + c;
        if (c < a.TW && oh < a.OH && ow < a.OW) {
          uint4* dst = reinterpret_cast<uint4*>(a.out + (((size_t)n * a.OH + oh) * a.OW + ow) * a.C + cb * CB);
#pragma unroll
          for (int u = 0; u < CB / 8; ++u)
            dst[u] = make_uint4(pack_bf16(v[8 * u], v[8 * u + 1]), pack_bf16(v[8 * u + 2], v[8 * u + 3]),
                                pack_bf16(v[8 * u + 4], v[8 * u + 5]), pack_bf16(v[8 * u + 6], v[8 * u + 7]));
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  griddep_launch_dependents();
  if (warp == 3) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "n"(kTmemCols));
  }
}

using KernelFn = void (*)(const CUtensorMap, const Args);

// group size S (the block-diagonal weight's width) needs a channel block CB >= S; CB = 16 / 32
// also staged for S = 16 (the swizzled A rows the tensor core reads per MMA are CB*2 bytes)
template <int K>
KernelFn pick(int S, int CB) {
  if (S == 16 && CB == 16) return bdmma_kernel<K, 16, 16>;
  if (S == 16 && CB == 32) return bdmma_kernel<K, 16, 32>;
  if (S == 32 && CB == 32) return bdmma_kernel<K, 32, 32>;
  if (S == 16 && CB == 64) return bdmma_kernel<K, 16, 64>;
  if (S == 32 && CB == 64) return bdmma_kernel<K, 32, 64>;
  if (S == 64 && CB == 64) return bdmma_kernel<K, 64, 64>;
  return nullptr;
}
KernelFn kernel_for(int K, int S, int CB) {
  switch (K) {
    case 3: return pick<3>(S, CB);
    case 5: return pick<5>(S, CB);
    case 7: return pick<7>(S, CB);
    default: return nullptr;
  }
}

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn encode_fn() {
  static EncodeFn fn = []() -> EncodeFn {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return nullptr;
    return reinterpret_cast<EncodeFn>(p);
  }();
  return fn;
}

bool opt_in_smem(const void* fn, int bytes) {
  static std::mutex mu;
  static std::vector<std::pair<const void*, int>> done;
  std::lock_guard<std::mutex> lk(mu);
  for (auto& d : done)
    if (d.first == fn && d.second >= bytes) return true;
  if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes) != cudaSuccess) return false;
  done.push_back({fn, bytes});
  return true;
}

int th_of(int CB) { return 512 / CB; }

int smem_bytes(int K, int S, int CB) {
  const int BH = th_of(CB) + K - 1;
  const int nacc = 2 * (th_of(CB) * BW / 128);
  static_assert((2 * NS + 2 * 16) * 8 + 16 <= 1024, "barriers fit the 1 KB header");
  (void)nacc;
  return 1024 + 1024 + NS * (BH + 1) * BW * CB * 2 + K * K * (CB / S) * S * S * 2;
}

}  // namespace bdmma

bool plan_nhwc_bdmma(const Geom& g, int pass, int num_sms, int smem_optin, int S, int CB, BdmmaPlan* p) {
  using namespace bdmma;
  if (g.layout != DWCONV_NHWC || g.dtype != DWCONV_BF16 || g.m != 1 || g.kh != g.kw || g.sh != 1 || g.sw != 1 ||
      g.ph != g.pw || (pass != DWCONV_PASS_FWD && pass != DWCONV_PASS_BWD_DATA))
    return false;
  const int K = g.kh;
  if (K != 3 && K != 5 && K != 7) return false;
  KernelFn fn = kernel_for(K, S, CB);
  if (!fn || g.C % CB != 0) return false;
  const int pad = pass == DWCONV_PASS_FWD ? g.ph : K - 1 - g.ph;
  if (pad < 0 || pad > K - 1) return false;
  const int smem = smem_bytes(K, S, CB);
  if (smem > smem_optin) return false;
  const int64_t OH = pass == DWCONV_PASS_FWD ? g.Ho : g.H, OW = pass == DWCONV_PASS_FWD ? g.Wo : g.W;
  const int TW = BW - K + 1, TH = th_of(CB);
  p->K = K;
  p->S = S;
  p->CB = CB;
  p->pass = pass;
  p->TW = TW;
  p->tiles_h = (int)((OH + TH - 1) / TH);
  p->tiles_w = (int)((OW + TW - 1) / TW);
  const int64_t per_cb = g.N * (int64_t)p->tiles_h * p->tiles_w;
  if (per_cb >= (1ll << 30)) return false;
  p->tiles_per_cb = (int)per_cb;
  p->ncb = (int)(g.C / CB);
  // one wave: resident CTAs per SM (shared memory; TMEM: 256 columns each, so at most 2) x SMs,
  // every CTA on one channel block (its diagonal weight tiles are built once)
  if (!opt_in_smem(reinterpret_cast<const void*>(fn), smem)) return false;
  int dev = 0, sm_smem = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sm_smem, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
  const int occ = std::max(1, std::min(2, sm_smem / (smem + 1024)));  // TMEM: 256 columns each
  p->ctas_per_cb = (int)std::max<int64_t>(1, std::min<int64_t>(per_cb, (occ * num_sms) / p->ncb));
  p->grid = p->ncb * p->ctas_per_cb;
  p->smem = smem;
  p->pad = pad;
  return true;
}

cudaError_t launch_nhwc_bdmma(const Geom& g, const BdmmaPlan& p, const void* in, const void* w, void* out,
                              cudaStream_t st) {
  using namespace bdmma;
  KernelFn fn = kernel_for(p.K, p.S, p.CB);
  EncodeFn enc = encode_fn();
  if (!fn || !enc) return cudaErrorNotSupported;
  const bool fwd = p.pass == DWCONV_PASS_FWD;
  const int64_t IH = fwd ? g.H : g.Ho, IW = fwd ? g.W : g.Wo;
  const int BH = th_of(p.CB) + p.K - 1, ROWB = p.CB * 2;
  CUtensorMap tm;
  const cuuint64_t dims[4] = {(cuuint64_t)g.C, (cuuint64_t)IW, (cuuint64_t)IH, (cuuint64_t)g.N};
  const cuuint64_t strides[3] = {(cuuint64_t)g.C * 2, (cuuint64_t)(IW * g.C * 2), (cuuint64_t)(IH * IW * g.C * 2)};
  const cuuint32_t box[4] = {(cuuint32_t)p.CB, (cuuint32_t)BW, (cuuint32_t)BH, 1};
  const cuuint32_t es[4] = {1, 1, 1, 1};
  const CUtensorMapSwizzle sw = p.CB == 64 ? CU_TENSOR_MAP_SWIZZLE_128B
                                           : (p.CB == 32 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B);
  if (enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(in), dims, strides, box, es,
          CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return cudaErrorInvalidValue;
  Args a{};
  a.out = static_cast<__nv_bfloat16*>(out);
  a.w = static_cast<const __nv_bfloat16*>(w);
  a.C = (int)g.C;
  a.OH = (int)(fwd ? g.Ho : g.H);
  a.OW = (int)(fwd ? g.Wo : g.W);
  a.K = p.K;
  a.pad = p.pad;
  a.TW = p.TW;
  a.tiles_h = p.tiles_h;
  a.tiles_w = p.tiles_w;
  a.tiles_per_cb = p.tiles_per_cb;
  a.ctas_per_cb = p.ctas_per_cb;
  a.stage_bytes = (uint32_t)((BH + 1) * BW * ROWB);
  a.box_bytes = (uint32_t)(BH * BW * ROWB);
  a.bw_bytes = (uint32_t)(p.K * p.K * p.CB * p.S * 2);
  a.flip = fwd ? 0 : 1;
  if (!opt_in_smem(reinterpret_cast<const void*>(fn), p.smem)) return cudaErrorInvalidValue;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)p.grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = (size_t)p.smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, fn, tm, a);
}

}  // namespace dwk
