// nchw_common.cuh -- shared pieces of the NCHW chunk kernels (nchw_fwd.cu,
// nchw_bwd_data.cu, nchw_bwd_filter.cu) and their planner (nchw_plan.cu).
//
// Design: the depthwise layer is a memory-bound stencil
// (PAPER.md P:62-63).  In NCHW a chunk -- P whole planes, or a band
// of rows of one large plane plus halo rows -- is one contiguous global range,
// staged into shared memory by a 1-D TMA bulk copy (cp.async.bulk -> UBLKCP) on
// an mbarrier, `ns` stages deep.  Each thread computes a strip of R output rows x
// V adjacent output columns from shared memory with vector loads (LDS.64/128)
// and, for stride 1, packed fp32x2 FMAs (FFMA2).  Rows outside the staged range
// read a zero row; the PAD edge columns are predicated loads.  Results leave
// through a shared-memory tile and a bulk shared->global copy.
#pragma once

#include <cuda_bf16.h>

#include <type_traits>

#include "common.cuh"
#include "kernels.h"

namespace dwk {
namespace nchw {

constexpr int kThreads = 256;  // maximum CTA size (the planner picks <= 256)
constexpr int kZPad = 8;  // zero-row elements on each side of column 0..W-1

struct NArgs {
  const void* in;      // fwd: x; bwd_data: dy; bwd_filter: x
  const void* in2;     // bwd_filter: dy
  void* out;           // fwd: y; bwd_data: dx
  const void* w;       // [C*m][K][K] storage dtype
  float* dw;           // bwd_filter output
  float* ws_part;      // bwd_filter per-slice partials [nslices][Co][K*K]
  unsigned* ws_ticket; // bwd_filter tickets [groups]
  int64_t N, C, Q;     // Q: planes iterated (fwd: N*C x planes, bwd_data: N*C dx planes)
  int m, Co, H, W, Ho, Wo;
  int P, nbands, BR, nsb;
  int64_t nchunks;
  // shared-memory layout (bytes): [0,128) barriers | zero row | weights |
  // ns input stages (128 B zero slack | in | 128 B zero slack | in2) | 2 output stages
  uint32_t zrow_off, w_off;
  uint32_t in0_off, in_stage, in_bytes, in2_off, in2_bytes;
  uint32_t out0_off, out_stage, out_bytes;
  int pitch, zbe;      // PADDED input staging: elements between planes, zero elements above each plane
  int ns;
  int groups, nslices, nps, tpg;
  FastDiv div_ncg, div_nsb, div_m, div_co;
  FastDiv div_c, div_nb;  // channel of a plane index; chunk -> (plane, band)
  int wbulk;              // w is 16-B aligned with a 16-B multiple size: weight rows may be bulk-copied
  int early_pdl;          // persistent kernels: trigger the dependent launch once the producer is done
};

using KernelFn = void (*)(NArgs);

// Kernel tables (one per pass, each in its own translation unit).
// RI: strip-height variant, VI: column-vector variant (V = 1 << VI).
// PADDED: input planes staged with zero rows around them (see stage_issue).
KernelFn fwd_kernel(int dtype, int K, int S, int RI, int VI, bool padded, bool pair = false);
KernelFn bwd_data_kernel(int dtype, int K, int S, int RI, int VI, bool padded, bool pair = false, bool m1 = false);
KernelFn bwd_filter_kernel(int dtype, int K, int S, int RI, int VI, bool padded);
KernelFn bwd_fused_kernel(int dtype, int K, int S, int RI, int VI, bool padded);  // dx + dw in one pass

// Strip heights: index 0 = "7*2^k planes", index 1 = default.
__host__ __device__ constexpr int rows_fwd(int K, int RI) { return K == 3 ? (RI == 0 ? 7 : 8) : (K == 5 ? 8 : 4); }
__host__ __device__ constexpr int rows_bd(int K, int S, int RI) {
  return S == 1 ? rows_fwd(K, RI) : (K == 3 ? (RI == 0 ? 14 : 8) : (K == 5 ? 8 : 4));
}
__host__ __device__ constexpr int rows_bf(int K, int RI) { return K == 3 ? (RI == 0 ? 7 : 8) : (K == 5 ? 8 : 4); }

__host__ __device__ constexpr int pmod(int a, int b) { return ((a % b) + b) % b; }

template <class T>
__device__ __forceinline__ bool bulk_ok(const T* gptr, int64_t count, uint32_t smem_off_bytes) {
  return ((reinterpret_cast<uintptr_t>(gptr) | (uintptr_t)(count * (int64_t)sizeof(T)) | smem_off_bytes) & 15u) == 0;
}

struct ChunkRows {
  int64_t q0;  // first plane of the chunk (fwd/bwd_filter: x plane; bwd_data: dx plane)
  int np;      // planes in chunk
  int r0, r1;  // output rows [r0, r1)
  int lo, hi;  // rows of the input held in smem [lo, hi)
};

// Kernel prologue shared by the three kernels: thread 0 initialises the ring's
// mbarriers; all threads zero the zero row and the input stages (padding gaps
// must read as zero; everything else must at least be finite); the generic-proxy
// zero writes are ordered before the TMA writes that follow; then the grid waits
// for the kernels it depends on (programmatic dependent launch).  Kernels call
// griddep_launch_dependents() once their last chunk is in flight, so the next
// kernel's launch overlaps this one's tail without taking SM slots early.
__device__ __forceinline__ void prologue(unsigned char* smem, uint64_t* bars, const NArgs& a) {
  if (threadIdx.x == 0) {
    for (int i = 0; i < a.ns; ++i) mbar_init(&bars[i], 1);
    fence_mbar_init();
  }
  auto zero = [&](uint32_t off, uint32_t bytes) {
    uint4* p = reinterpret_cast<uint4*>(smem + off);
    for (uint32_t i = threadIdx.x; i < bytes / 16; i += blockDim.x) p[i] = make_uint4(0, 0, 0, 0);
  };
  zero(a.zrow_off - kZPad * 4, a.w_off - (a.zrow_off - kZPad * 4));
  zero(a.in0_off, a.ns * a.in_stage);
  fence_proxy_async_smem();
  griddep_wait();
  __syncthreads();
}

// Prologue of the warp-specialised kernels: "full" mbarriers at smem[0..64)
// (count 1: the producer's arrive + TMA bytes), "empty" mbarriers at
// smem[64..128) (count = consumer warps), zero row and input stages zeroed,
// ordered before the TMA writes, then the programmatic-dependent-launch wait.
__device__ __forceinline__ void prologue_ws(unsigned char* smem, const NArgs& a, int consumer_warps,
                                            int full_count = 1) {
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  uint64_t* empty = reinterpret_cast<uint64_t*>(smem + 64);
  if (threadIdx.x == 0) {
    for (int i = 0; i < a.ns; ++i) {
      mbar_init(&full[i], full_count);
      mbar_init(&empty[i], consumer_warps);
    }
    fence_mbar_init();
  }
  auto zero = [&](uint32_t off, uint32_t bytes) {
    uint4* p = reinterpret_cast<uint4*>(smem + off);
    for (uint32_t i = threadIdx.x; i < bytes / 16; i += blockDim.x) p[i] = make_uint4(0, 0, 0, 0);
  };
  zero(a.zrow_off - kZPad * 4, a.w_off - (a.zrow_off - kZPad * 4));
  zero(a.in0_off, a.ns * a.in_stage);
  fence_proxy_async_smem();
  griddep_wait();
  __syncthreads();
}

// Named barrier over the consumer warps only (warps 1..): barrier 1.
__device__ __forceinline__ void consumer_sync(int nthreads) {
  asm volatile("bar.sync 1, %0;" ::"r"(nthreads) : "memory");
}

// ------------------------------------------------------------------ vector I/O
// N consecutive elements at p (aligned to min(16, N * sizeof(T)) bytes) <-> floats.
template <class T, int N> struct VecIO;
template <int N> struct VecIO<float, N> {
  static __device__ __forceinline__ void load(const float* p, float* v) {
    if constexpr (N == 1) {
      v[0] = *p;
    } else if constexpr (N == 2) {
      const float2 a = *reinterpret_cast<const float2*>(p);
      v[0] = a.x; v[1] = a.y;
    } else {
#pragma unroll
      for (int q = 0; q < N / 4; ++q) {
        const float4 a = reinterpret_cast<const float4*>(p)[q];
        v[4 * q] = a.x; v[4 * q + 1] = a.y; v[4 * q + 2] = a.z; v[4 * q + 3] = a.w;
      }
    }
  }
  static __device__ __forceinline__ void store(float* p, const float* v) {
    if constexpr (N == 1) {
      *p = v[0];
    } else if constexpr (N == 2) {
      *reinterpret_cast<float2*>(p) = make_float2(v[0], v[1]);
    } else {
#pragma unroll
      for (int q = 0; q < N / 4; ++q)
        reinterpret_cast<float4*>(p)[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
    }
  }
};
__device__ __forceinline__ float bf_lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf_hi(uint32_t w) { return __uint_as_float(w & 0xffff0000u); }
__device__ __forceinline__ uint32_t bf_pack(float lo, float hi) {
  __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);  // round to nearest even
  return *reinterpret_cast<uint32_t*>(&h);
}
template <int N> struct VecIO<__nv_bfloat16, N> {
  static __device__ __forceinline__ void load(const __nv_bfloat16* p, float* v) {
    if constexpr (N == 1) {
      v[0] = __bfloat162float(*p);
    } else if constexpr (N == 2) {
      const uint32_t a = *reinterpret_cast<const uint32_t*>(p);
      v[0] = bf_lo(a); v[1] = bf_hi(a);
    } else if constexpr (N == 4) {
      const uint2 a = *reinterpret_cast<const uint2*>(p);
      v[0] = bf_lo(a.x); v[1] = bf_hi(a.x); v[2] = bf_lo(a.y); v[3] = bf_hi(a.y);
    } else {
#pragma unroll
      for (int q = 0; q < N / 8; ++q) {
        const uint4 a = reinterpret_cast<const uint4*>(p)[q];
        float* o = v + 8 * q;
        o[0] = bf_lo(a.x); o[1] = bf_hi(a.x); o[2] = bf_lo(a.y); o[3] = bf_hi(a.y);
        o[4] = bf_lo(a.z); o[5] = bf_hi(a.z); o[6] = bf_lo(a.w); o[7] = bf_hi(a.w);
      }
    }
  }
  static __device__ __forceinline__ void store(__nv_bfloat16* p, const float* v) {
    if constexpr (N == 1) {
      *p = __float2bfloat16_rn(v[0]);
    } else if constexpr (N == 2) {
      *reinterpret_cast<uint32_t*>(p) = bf_pack(v[0], v[1]);
    } else if constexpr (N == 4) {
      *reinterpret_cast<uint2*>(p) = make_uint2(bf_pack(v[0], v[1]), bf_pack(v[2], v[3]));
    } else {
#pragma unroll
      for (int q = 0; q < N / 8; ++q)
        reinterpret_cast<uint4*>(p)[q] = make_uint4(bf_pack(v[8 * q], v[8 * q + 1]), bf_pack(v[8 * q + 2], v[8 * q + 3]),
                                                    bf_pack(v[8 * q + 4], v[8 * q + 5]), bf_pack(v[8 * q + 6], v[8 * q + 7]));
    }
  }
};

// ------------------------------------------------------------------ input window
// One input row's window for V output columns at stride S: columns
// [S*c0 - PAD, S*c0 - PAD + (V-1)*S + K).  The S*V columns starting at S*c0 are
// one aligned vector load; the PAD columns on the left and K-PAD-S on the right
// are predicated scalar loads (zero outside the plane).
template <int K, int S, int V>
struct Win {
  static constexpr int PAD = (K - 1) / 2;
  static constexpr int NV = S * V;
  static constexpr int NL = PAD;
  static constexpr int NR = (K - PAD - S) > 0 ? (K - PAD - S) : 0;
  static constexpr int N = NL + NV + NR;
};

template <class T, int K, int S, int V>
__device__ __forceinline__ void load_window(const T* p /* at column S*c0 */, const bool* lok, const bool* rok,
                                            float* xw) {
  using Wd = Win<K, S, V>;
  if constexpr (V == 1) {  // V = 1 is the fallback for unaligned rows: scalar loads only
#pragma unroll
    for (int q = 0; q < Wd::NV; ++q) xw[Wd::NL + q] = Elem<T>::load(p + q);
  } else {
    VecIO<T, Wd::NV>::load(p, xw + Wd::NL);
  }
#pragma unroll
  for (int l = 0; l < Wd::NL; ++l) xw[l] = lok[l] ? Elem<T>::load(p - Wd::NL + l) : 0.f;
#pragma unroll
  for (int r = 0; r < Wd::NR; ++r) xw[Wd::NL + Wd::NV + r] = rok[r] ? Elem<T>::load(p + Wd::NV + r) : 0.f;
}

// ------------------------------------------------------------------ input staging
// A chunk's input is `npl` planes (cnt elements each: rows [lo, hi) of width Wr)
// whose global data start at src0 + p * gstride.  They land at
// base + p * pitch + zbe.  With pitch == gstride == cnt and zbe == 0 the planes
// are back to back and contiguous in global memory: ONE bulk copy.  Otherwise
// one bulk copy per plane; a PADDED plan leaves zbe zero elements above every
// plane (and below the last one), so strips need no row checks.
struct StageSpec {
  int64_t gstride, cnt;
  int npl, pitch, zbe;
};
template <class T>
__device__ __forceinline__ bool stage_contig(const StageSpec& s) {
  return s.gstride == s.cnt && s.pitch == s.cnt && s.zbe == 0;
}
template <class T>
__device__ __forceinline__ bool stage_bulk_ok(const T* src0, const StageSpec& s) {
  if (stage_contig<T>(s)) return ((reinterpret_cast<uintptr_t>(src0) | (uintptr_t)(s.cnt * s.npl * sizeof(T))) & 15u) == 0;
  return ((reinterpret_cast<uintptr_t>(src0) | (uintptr_t)(s.gstride * sizeof(T)) | (uintptr_t)(s.cnt * sizeof(T)) |
           (uintptr_t)(s.pitch * sizeof(T)) | (uintptr_t)(s.zbe * sizeof(T))) & 15u) == 0;
}
template <class T>
__device__ __forceinline__ uint32_t stage_bytes(const StageSpec& s) { return (uint32_t)(s.cnt * s.npl * sizeof(T)); }
// Thread 0, after the barrier is armed for all bytes: issue the copies.
template <class T>
__device__ __forceinline__ void stage_copy(T* base, const T* src0, const StageSpec& s, uint64_t* bar) {
  if (stage_contig<T>(s)) {
    bulk_g2s(base, src0, stage_bytes<T>(s), bar);
  } else {
    for (int p = 0; p < s.npl; ++p)
      bulk_g2s(base + p * s.pitch + s.zbe, src0 + p * s.gstride, (uint32_t)(s.cnt * sizeof(T)), bar);
  }
}
// All threads: cooperative copy (used when the stage was not bulk-eligible).
template <class T>
__device__ __forceinline__ void stage_coop(T* base, const T* src0, const StageSpec& s) {
  if (stage_contig<T>(s)) {
    coop_copy(base, src0, s.cnt * s.npl);
  } else {
    for (int p = 0; p < s.npl; ++p) coop_copy(base + p * s.pitch + s.zbe, src0 + p * s.gstride, s.cnt);
  }
}
// All threads: write zeros to n elements (band-mode bottom padding rows).
template <class T>
__device__ __forceinline__ void zero_elems(T* p, int n) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) p[i] = T(0.f);
}
// 16-B zero stores over [p, p + bytes) by thread t of nt (p and bytes 16-B multiples).
__device__ __forceinline__ void zero_bytes16(void* p, uint32_t bytes, int t, int nt) {
  uint4* q = reinterpret_cast<uint4*>(p);
  for (uint32_t i = t; i < bytes / 16; i += nt) q[i] = make_uint4(0u, 0u, 0u, 0u);
}
// Same over a subset of threads (thread t of nt).
template <class T>
__device__ __forceinline__ void zero_elems_n(T* p, int n, int t, int nt) {
  for (int i = t; i < n; i += nt) p[i] = T(0.f);
}
template <class T>
__device__ __forceinline__ void stage_coop_n(T* base, const T* src0, const StageSpec& s, int t, int nt) {
  if (stage_contig<T>(s)) {
    for (int64_t i = t; i < s.cnt * s.npl; i += nt) base[i] = src0[i];
  } else {
    for (int p = 0; p < s.npl; ++p)
      for (int64_t i = t; i < s.cnt; i += nt) base[p * s.pitch + s.zbe + i] = src0[p * s.gstride + i];
  }
}

// ------------------------------------------------------------------ chunk weights
// A chunk of planes [q0, q0+np) (plane q = n*C + c) needs the weight rows of the
// output channels [cb*m, (cb+np)*m), cb = q0 mod C: elements [e0, e1) of w.
// When that range does not wrap past channel C-1 and a.wbulk holds, the producer
// stages the 16-B aligned superset [a0, a1) raw (storage dtype) with one bulk
// copy on the stage's full barrier, and consumers read element e at
// table + off + (e - e0).  Otherwise the producer warp writes an fp32 table.
struct WeightWin {
  bool tma;
  int off;        // elements from the staged start a0 to e0
  int64_t a0;     // first staged element
  uint32_t bytes; // staged bytes
};
template <class T, int KK>
__device__ __forceinline__ WeightWin weight_win(const NArgs& a, int64_t q0, int np) {
  constexpr int64_t A = 16 / sizeof(T);
  WeightWin r;
  const int64_t cb = q0 - (int64_t)fdiv((uint32_t)q0, a.div_c) * a.C;
  r.tma = a.wbulk && cb + np <= a.C;
  const int64_t e0 = cb * a.m * KK, e1 = (cb + np) * a.m * KK;
  r.a0 = e0 & ~(A - 1);
  r.bytes = (uint32_t)((((e1 + A - 1) & ~(A - 1)) - r.a0) * (int64_t)sizeof(T));
  r.off = (int)(e0 - r.a0);
  return r;
}

// ------------------------------------------------------------------ bf16 interleaved windows
#ifndef DWCONV_BF16_IL
#define DWCONV_BF16_IL 1
#endif
constexpr bool kBf16Interleave = DWCONV_BF16_IL != 0;
template <int NW>
__device__ __forceinline__ void load_words(const __nv_bfloat16* p, uint32_t* w) {
  if constexpr (NW == 1) {
    w[0] = *reinterpret_cast<const uint32_t*>(p);
  } else if constexpr (NW == 2) {
    const uint2 v = *reinterpret_cast<const uint2*>(p);
    w[0] = v.x; w[1] = v.y;
  } else {
#pragma unroll
    for (int q = 0; q < NW / 4; ++q) {
      const uint4 v = reinterpret_cast<const uint4*>(p)[q];
      w[4 * q] = v.x; w[4 * q + 1] = v.y; w[4 * q + 2] = v.z; w[4 * q + 3] = v.w;
    }
  }
}
// bf16 strips of V >= 4 columns pair output column u with column u + V/2 in one
// FFMA2 (lanes = (u, u + V/2)), so the operand pair of tap jj is
//   X2[S*u + jj] = (xw[S*u + jj], xw[S*u + jj + S*V/2]),
// two window elements half a strip apart.  Every element has to be widened from
// bf16 anyway, so each pair half is widened straight into its register: no
// pair-forming moves (a (u, u+1) pairing needs them for every other tap, and
// they issue as IMAD.MOV on the FMA pipe this path is bound by), at any stride.
// The widening is PRMT / LOP3 (ALU pipe), kept out of IMAD by inline PTX.
__device__ __forceinline__ float bfw_lo(uint32_t w) {  // low bf16 of a word -> fp32 (exact)
  float r;
  asm volatile("prmt.b32 %0, %1, 0, 0x1054;" : "=f"(r) : "r"(w));
  return r;
}
__device__ __forceinline__ float bfw_hi(uint32_t w) {  // high bf16 of a word -> fp32 (exact)
  float r;
  asm volatile("and.b32 %0, %1, 0xffff0000;" : "=f"(r) : "r"(w));
  return r;
}
template <int K, int S, int V>
struct Win2 {
  static_assert(V >= 4 && V % 2 == 0, "interleaved pairs need V >= 4");
  static constexpr int H = S * V / 2;            // lane distance inside the window
  static constexpr int NP = S * (V / 2 - 1) + K;  // operand pairs per row
};
// Window of one row (as Win<K,S,V>) in interleaved pairs X2[k] = (xw[k], xw[k + H]).
template <int K, int S, int V>
__device__ __forceinline__ void load_window_bf2(const __nv_bfloat16* p /* at column S*c0 */, const bool* lok,
                                                const bool* rok, float2* X2) {
  using Wd = Win<K, S, V>;
  using W2 = Win2<K, S, V>;
  static_assert(Wd::NV % 2 == 0, "whole 32-bit words");
  constexpr int NW = Wd::NV / 2;
  uint32_t wv[NW];
  load_words<NW>(p, wv);
  const unsigned short* us = reinterpret_cast<const unsigned short*>(p);
  uint32_t hl[Wd::NL > 0 ? Wd::NL : 1], hr[Wd::NR > 0 ? Wd::NR : 1];
#pragma unroll
  for (int l = 0; l < Wd::NL; ++l) hl[l] = lok[l] ? (uint32_t)us[l - Wd::NL] : 0u;
#pragma unroll
  for (int r = 0; r < Wd::NR; ++r) hr[r] = rok[r] ? (uint32_t)us[Wd::NV + r] : 0u;
  auto val = [&](int k) -> float {  // xw[k]; k is a compile-time constant after unrolling
    if (k < Wd::NL) return bfw_lo(hl[k]);
    if (k < Wd::NL + Wd::NV) {
      const int q = k - Wd::NL;
      return (q & 1) ? bfw_hi(wv[q >> 1]) : bfw_lo(wv[q >> 1]);
    }
    return bfw_lo(hr[k - Wd::NL - Wd::NV]);
  };
#pragma unroll
  for (int k = 0; k < W2::NP; ++k) X2[k] = make_float2(val(k), val(k + W2::H));
}
// V bf16 values at p (16-B / 8-B aligned) as pairs D2[u] = (v[u], v[u + V/2]).
template <int V>
__device__ __forceinline__ void load_vec_bf2(const __nv_bfloat16* p, float2* D2) {
  uint32_t wv[V / 2];
  load_words<V / 2>(p, wv);
  auto val = [&](int q) -> float { return (q & 1) ? bfw_hi(wv[q >> 1]) : bfw_lo(wv[q >> 1]); };
#pragma unroll
  for (int u = 0; u < V / 2; ++u) D2[u] = make_float2(val(u), val(u + V / 2));
}
// The bf16 interleaved strip: same sums as stencil_strip (below), FFMA2 at any stride.
template <int K, int S, int R, int V, bool PADDED>
__device__ __forceinline__ void stencil_strip_bf2(const __nv_bfloat16* sp, const __nv_bfloat16* zp, int W, int lo,
                                                  int rows, int ih0, int c0, const float* wr, float (&acc)[R][V]) {
  using Wd = Win<K, S, V>;
  using W2 = Win2<K, S, V>;
  constexpr int NRows = (R - 1) * S + K;
  const int b0 = S * c0;
  bool lok[Wd::NL > 0 ? Wd::NL : 1], rok[Wd::NR > 0 ? Wd::NR : 1];
#pragma unroll
  for (int l = 0; l < Wd::NL; ++l) lok[l] = b0 - Wd::NL + l >= 0;
#pragma unroll
  for (int r = 0; r < Wd::NR; ++r) rok[r] = b0 + Wd::NV + r < W;
  float2 acc2[R][V / 2];
#pragma unroll
  for (int tt = 0; tt < R; ++tt)
#pragma unroll
    for (int u = 0; u < V / 2; ++u) acc2[tt][u] = make_float2(acc[tt][u], acc[tt][u + V / 2]);
  const __nv_bfloat16* prow = sp + ih0 * W + b0;
#pragma unroll
  for (int r = 0; r < NRows; ++r) {
    const __nv_bfloat16* p;
    if constexpr (PADDED) {
      p = prow + r * W;
    } else {
      const bool rv = (unsigned)(ih0 + r - lo) < (unsigned)rows;
      p = rv ? prow + r * W : zp + b0;
    }
    float2 X2[W2::NP];
    load_window_bf2<K, S, V>(p, lok, rok, X2);
#pragma unroll
    for (int tt = 0; tt < R; ++tt) {
      const int i = r - tt * S;
      if (i >= 0 && i < K) {
#pragma unroll
        for (int jj = 0; jj < K; ++jj) {
          const float w = wr[i * K + jj];
#pragma unroll
          for (int u = 0; u < V / 2; ++u) acc2[tt][u] = __ffma2_rn(make_float2(w, w), X2[S * u + jj], acc2[tt][u]);
        }
      }
    }
  }
#pragma unroll
  for (int tt = 0; tt < R; ++tt)
#pragma unroll
    for (int u = 0; u < V / 2; ++u) { acc[tt][u] = acc2[tt][u].x; acc[tt][u + V / 2] = acc2[tt][u].y; }
}

// The same strip with each output row handed to store(tt, v[V]) as soon as its
// last input row is in (row tt after input row tt*S + K - 1): only the K/S + 1 rows
// still accumulating are live, not all R -- fewer registers, more warps per SM.
template <int K, int S, int R, int V, bool PADDED, class StoreRow>
__device__ __forceinline__ void stencil_strip_bf2_stream(const __nv_bfloat16* sp, const __nv_bfloat16* zp, int W,
                                                         int lo, int rows, int ih0, int c0, const float* wr,
                                                         StoreRow&& store) {
  using Wd = Win<K, S, V>;
  using W2 = Win2<K, S, V>;
  constexpr int NRows = (R - 1) * S + K;
  const int b0 = S * c0;
  bool lok[Wd::NL > 0 ? Wd::NL : 1], rok[Wd::NR > 0 ? Wd::NR : 1];
#pragma unroll
  for (int l = 0; l < Wd::NL; ++l) lok[l] = b0 - Wd::NL + l >= 0;
#pragma unroll
  for (int r = 0; r < Wd::NR; ++r) rok[r] = b0 + Wd::NV + r < W;
  float2 acc2[R][V / 2];
#pragma unroll
  for (int tt = 0; tt < R; ++tt)
#pragma unroll
    for (int u = 0; u < V / 2; ++u) acc2[tt][u] = make_float2(0.f, 0.f);
  const __nv_bfloat16* prow = sp + ih0 * W + b0;
#pragma unroll
  for (int r = 0; r < NRows; ++r) {
    const __nv_bfloat16* p;
    if constexpr (PADDED) {
      p = prow + r * W;
    } else {
      const bool rv = (unsigned)(ih0 + r - lo) < (unsigned)rows;
      p = rv ? prow + r * W : zp + b0;
    }
    float2 X2[W2::NP];
    load_window_bf2<K, S, V>(p, lok, rok, X2);
#pragma unroll
    for (int tt = 0; tt < R; ++tt) {
      const int i = r - tt * S;
      if (i >= 0 && i < K) {
#pragma unroll
        for (int jj = 0; jj < K; ++jj) {
          const float w = wr[i * K + jj];
#pragma unroll
          for (int u = 0; u < V / 2; ++u) acc2[tt][u] = __ffma2_rn(make_float2(w, w), X2[S * u + jj], acc2[tt][u]);
        }
      }
      if (r == tt * S + K - 1) {
        float v[V];
#pragma unroll
        for (int u = 0; u < V / 2; ++u) { v[u] = acc2[tt][u].x; v[u + V / 2] = acc2[tt][u].y; }
        store(tt, v);
      }
    }
  }
}

// ------------------------------------------------------------------ stencil strip
// acc[tt][u] = sum_{i,jj} wr[i*K+jj] * X[oh0*S - PAD + tt*S + i][S*(c0+u) - PAD + jj]
// where input row ih lives at sp + ih*W.  PADDED: every row the strip touches is
// staged or a zero row.  DENSE: rows with (unsigned)(ih - lo) >= rows read the
// zero row zp.  Used by the forward pass and (with the kernel flipped) the
// stride-1 input gradient.
template <class T, int K, int S, int R, int V, bool PADDED>
__device__ __forceinline__ void stencil_strip(const T* sp, const T* zp, int W, int lo, int rows, int ih0, int c0,
                                              const float* wr, float (&acc)[R][V]) {
  if constexpr (std::is_same<T, __nv_bfloat16>::value && V >= 4 && (S * V) % 2 == 0) {
    if (kBf16Interleave) {
      stencil_strip_bf2<K, S, R, V, PADDED>(sp, zp, W, lo, rows, ih0, c0, wr, acc);
      return;
    }
  }
  using Wd = Win<K, S, V>;
  constexpr int NRows = (R - 1) * S + K;
  const int b0 = S * c0;
  bool lok[Wd::NL > 0 ? Wd::NL : 1], rok[Wd::NR > 0 ? Wd::NR : 1];
#pragma unroll
  for (int l = 0; l < Wd::NL; ++l) lok[l] = b0 - Wd::NL + l >= 0;
#pragma unroll
  for (int r = 0; r < Wd::NR; ++r) rok[r] = b0 + Wd::NV + r < W;
  const T* prow = sp + ih0 * W + b0;
#pragma unroll
  for (int r = 0; r < NRows; ++r) {
    const T* p;
    if constexpr (PADDED) {
      p = prow + r * W;
    } else {
      const int ih = ih0 + r;
      const bool rv = (unsigned)(ih - lo) < (unsigned)rows;
      p = rv ? prow + r * W : zp + b0;
    }
    float xw[Wd::N];
    load_window<T, K, S, V>(p, lok, rok, xw);
#pragma unroll
    for (int tt = 0; tt < R; ++tt) {
      const int i = r - tt * S;
      if (i >= 0 && i < K) {
#pragma unroll
        for (int jj = 0; jj < K; ++jj) {
          const float w = wr[i * K + jj];
          if constexpr (S == 1 && V % 2 == 0) {
#pragma unroll
            for (int u = 0; u < V; u += 2) {
              float2 a = make_float2(acc[tt][u], acc[tt][u + 1]);
              a = __ffma2_rn(make_float2(w, w), make_float2(xw[u + jj], xw[u + 1 + jj]), a);
              acc[tt][u] = a.x;
              acc[tt][u + 1] = a.y;
            }
          } else {
#pragma unroll
            for (int u = 0; u < V; ++u) acc[tt][u] = fmaf(w, xw[S * u + jj], acc[tt][u]);
          }
        }
      }
    }
  }
}

// ------------------------------------------------------------------ bf16 plane pairs
// bf16 strips of TWO planes at once: packed FFMA2 lanes = (plane A, plane B) at
// the same position, so every operand pair is built straight from the loaded
// 16-bit values (one shift or mask per element into the pair's register) and no
// column pair ever straddles registers -- no pair-forming moves, FFMA2 at any
// stride.  Window: columns [S*c0 - PAD, S*c0 - PAD + (V-1)*S + K), as Win<K,S,V>.
__device__ __forceinline__ float bf_bits_lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf_bits_hi(uint32_t w) { return __uint_as_float(w & 0xffff0000u); }
template <int K, int S, int V>
__device__ __forceinline__ void load_window_pair(const __nv_bfloat16* pa, const __nv_bfloat16* pb, const bool* lok,
                                                 const bool* rok, float2* xw) {
  using Wd = Win<K, S, V>;
  static_assert(Wd::NV % 2 == 0, "pair windows load whole 32-bit words");
  constexpr int NW = Wd::NV / 2;
  uint32_t wa[NW], wb[NW];
  load_words<NW>(pa, wa);
  load_words<NW>(pb, wb);
#pragma unroll
  for (int k = 0; k < NW; ++k) {
    xw[Wd::NL + 2 * k] = make_float2(bf_bits_lo(wa[k]), bf_bits_lo(wb[k]));
    xw[Wd::NL + 2 * k + 1] = make_float2(bf_bits_hi(wa[k]), bf_bits_hi(wb[k]));
  }
  const unsigned short* ua = reinterpret_cast<const unsigned short*>(pa);
  const unsigned short* ub = reinterpret_cast<const unsigned short*>(pb);
#pragma unroll
  for (int l = 0; l < Wd::NL; ++l)
    xw[l] = lok[l] ? make_float2(bf_bits_lo(ua[l - Wd::NL]), bf_bits_lo(ub[l - Wd::NL])) : make_float2(0.f, 0.f);
#pragma unroll
  for (int r = 0; r < Wd::NR; ++r)
    xw[Wd::NL + Wd::NV + r] =
        rok[r] ? make_float2(bf_bits_lo(ua[Wd::NV + r]), bf_bits_lo(ub[Wd::NV + r])) : make_float2(0.f, 0.f);
}
// acc[tt][u] = (plane A, plane B) sums of stencil_strip at the same position.
template <int K, int S, int R, int V, bool PADDED>
__device__ __forceinline__ void stencil_strip_pair(const __nv_bfloat16* spa, const __nv_bfloat16* spb,
                                                   const __nv_bfloat16* zp, int W, int lo, int rows, int ih0, int c0,
                                                   const float2* wp, float2 (&acc)[R][V]) {
  using Wd = Win<K, S, V>;
  constexpr int NRows = (R - 1) * S + K;
  const int b0 = S * c0;
  bool lok[Wd::NL > 0 ? Wd::NL : 1], rok[Wd::NR > 0 ? Wd::NR : 1];
#pragma unroll
  for (int l = 0; l < Wd::NL; ++l) lok[l] = b0 - Wd::NL + l >= 0;
#pragma unroll
  for (int r = 0; r < Wd::NR; ++r) rok[r] = b0 + Wd::NV + r < W;
  const __nv_bfloat16* pra = spa + ih0 * W + b0;
  const __nv_bfloat16* prb = spb + ih0 * W + b0;
#pragma unroll
  for (int r = 0; r < NRows; ++r) {
    const __nv_bfloat16 *pa, *pb;
    if constexpr (PADDED) {
      pa = pra + r * W;
      pb = prb + r * W;
    } else {
      const bool rv = (unsigned)(ih0 + r - lo) < (unsigned)rows;
      pa = rv ? pra + r * W : zp + b0;
      pb = rv ? prb + r * W : zp + b0;
    }
    float2 xw[Wd::N];
    load_window_pair<K, S, V>(pa, pb, lok, rok, xw);
#pragma unroll
    for (int tt = 0; tt < R; ++tt) {
      const int i = r - tt * S;
      if (i >= 0 && i < K) {
#pragma unroll
        for (int jj = 0; jj < K; ++jj)
#pragma unroll
          for (int u = 0; u < V; ++u) acc[tt][u] = __ffma2_rn(wp[i * K + jj], xw[S * u + jj], acc[tt][u]);
      }
    }
  }
}


// Two-level deterministic cross-CTA reduction of per-slice partials (no float
// atomics).  Every CTA of channel block `gid` has written its slice partial
// part[sl * sstride + e0 + i] (i < nvals), issued __threadfence() and
// __syncthreads(); then all its threads call this.  Level 1: the last CTA (integer
// ticket) of each group of 32 consecutive slices sums the group's partials
// pairwise in slice order into l2[sg]; level 2: the last group finisher sums
// l2[0..ngrp) pairwise in group order into dw.  Each level is <= 32 dependent
// loads deep instead of one flat pass over hundreds of slices.  Both levels hand
// back zeroed partials and tickets.
__device__ __forceinline__ float pairwise_sum_strided(float* base, int64_t stride, int count) {
  float stk[8];
  int top = 0;
  for (int s0 = 0; s0 < count; s0 += 16) {
    float vals[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) vals[u] = (s0 + u < count) ? __ldcg(base + (s0 + u) * stride) : 0.f;
#pragma unroll
    for (int u = 0; u < 16; ++u)
      if (s0 + u < count) __stcg(base + (s0 + u) * stride, 0.f);
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const int s2 = s0 + u;
      if (s2 < count) {
        float cur = vals[u];
        int bits = s2;
        while (bits & 1) { cur = stk[--top] + cur; bits >>= 1; }
        stk[top++] = cur;
      }
    }
  }
  float tot = stk[--top];
  while (top > 0) tot = stk[--top] + tot;
  return tot;
}

__device__ __forceinline__ void finalize_two_level(float* part, float* l2, unsigned* t1, unsigned* t2, int gid,
                                                   int sl, int nslices, int64_t sstride, int64_t e0, int nvals,
                                                   float* dw, unsigned* s_flag) {
  const int ngrp = (nslices + 31) / 32;
  const int sg = sl / 32;
  const int gsz = min(32, nslices - sg * 32);
  if (threadIdx.x == 0) {
    const unsigned prev = atomicAdd(&t1[(int64_t)gid * ngrp + sg], 1u);
    *s_flag = (prev == (unsigned)(gsz - 1)) ? 1u : 0u;
  }
  __syncthreads();
  if (!*s_flag) return;
  __threadfence();
  if (ngrp == 1) {  // <= 32 slices: one level, straight into dw
    for (int i = threadIdx.x; i < nvals; i += blockDim.x) dw[e0 + i] = pairwise_sum_strided(part + e0 + i, sstride, gsz);
    if (threadIdx.x == 0) t1[gid] = 0u;
    return;
  }
  for (int i = threadIdx.x; i < nvals; i += blockDim.x)
    __stcg(l2 + sg * sstride + e0 + i, pairwise_sum_strided(part + (int64_t)sg * 32 * sstride + e0 + i, sstride, gsz));
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    t1[(int64_t)gid * ngrp + sg] = 0u;
    const unsigned prev = atomicAdd(&t2[gid], 1u);
    *s_flag = (prev == (unsigned)(ngrp - 1)) ? 1u : 0u;
  }
  __syncthreads();
  if (!*s_flag) return;
  __threadfence();
  for (int i = threadIdx.x; i < nvals; i += blockDim.x) dw[e0 + i] = pairwise_sum_strided(l2 + e0 + i, sstride, ngrp);
  if (threadIdx.x == 0) t2[gid] = 0u;
}
}  // namespace nchw

namespace direct {
// Arguments of the register-direct bwd_filter kernels (direct_bwd_filter.cu).
struct DArgs {
  const void* x;
  const void* dy;
  float* dw;
  float* ws_part;       // per-slice partials [nslices][Co][9]
  unsigned* ws_ticket;  // [groups]
  int N, C, m, Co, H, W, Ho, Wo;
  int P;                // output channels per group
  int groups, nslices, nps;
  int L, SPW, spc;      // lanes per row set, row sets per warp, row sets per channel
  int nsb;              // dy strips per plane
  int pf;               // rows are 16-B multiples and bases aligned: bulk L2 prefetch allowed
};
using DKernelFn = void (*)(DArgs);
DKernelFn bwd_filter_kernel(int dtype, int S, int R, int V);
DKernelFn bwd_filter_stream_kernel(int dtype, int S, int BR, int V);  // bf16 streaming (sdbf_kernel)
}  // namespace direct
}  // namespace dwk
