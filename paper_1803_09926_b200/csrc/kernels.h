// kernels.h -- host-visible launch interface between host.cpp and the .cu files.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <vector>

#include "../../include/dwconv.h"

namespace dwk {

struct FastDiv;

// Geometry shared by every kernel (validated by host.cpp).
struct Geom {
  int64_t N, C, H, W, Ho, Wo;
  int m, kh, kw, sh, sw, ph, pw;
  int layout, dtype;
};

// ---- generic kernels (any shape, both layouts): generic.cu
cudaError_t launch_generic_fwd(const Geom& g, const void* x, const void* w, void* y, cudaStream_t st);
cudaError_t launch_generic_bwd_data(const Geom& g, const void* dy, const void* w, void* dx, cudaStream_t st);
cudaError_t launch_generic_bwd_filter(const Geom& g, const void* x, const void* dy, float* dw, cudaStream_t st);

// Workspace of the two-level slice finalize (nchw_common.cuh finalize_two_level):
// level-1 tickets [groups][ceil(slices/32)] + level-2 tickets [groups] (16-B
// rounded), then slice partials [slices][C][9] and group partials [ceil(slices/32)][C][9].
inline size_t two_level_tick_bytes(int64_t groups, int64_t slices) {
  const int64_t ngrp = (slices + 31) / 32;
  return ((size_t)(groups * ngrp + groups) * 4 + 15) / 16 * 16;
}
inline size_t two_level_ws_bytes(int64_t groups, int64_t slices, int64_t channels, int64_t taps = 9) {
  return two_level_tick_bytes(groups, slices) + (size_t)(slices + (slices + 31) / 32) * channels * taps * 4;
}

// ---- NCHW small-plane warp-task kernels (W = H in {7,14,28}, 3x3 s1 p1 m1): nchw_small.cu
struct SmallPlan {
  int warps, ns, grid, smem;
  uint32_t slot_bytes;
  int64_t ntasks;
  int groups, nslices, nps, max_chain;
  size_t ws_bytes;
  int S;  // stride of the small-plane kernels
  bool pair;  // bf16 plane-pair kernel (8-plane tasks, FFMA2 over plane pairs)
  int occ, sms;  // resident CTAs per SM, SMs (early PDL only when the grid is one wave)
  // band bwd_filter for large planes (band_bf_kernel)
  bool band;
  int R, V, nbands, cpg, ppw;
  bool lane;  // lane-per-plane kernels (lane_fd_kernel / lane_bf_kernel): 32-plane warp tasks
};
// lane-per-plane kernels (W = H in {7, 14}, s1): warps per CTA, ring slots per warp, batch slices (bwd_filter)
bool plan_nchw_lane(const Geom& g, int pass, int num_sms, int smem_optin, SmallPlan* plan, int warps, int stages,
                    int slices = 0);
bool plan_nchw_band_bf(const Geom& g, int num_sms, int smem_optin, SmallPlan* plan, int warps, int stages, int rows,
                       int ppw = 1);
// warps / stages: CTA size and per-warp ring depth (0 = the defaults, env DWCONV_SMALL_WARPS / _STAGES)
// slices (bwd_filter): batch slices per channel group (0 = about one wave of CTAs)
bool plan_nchw_small(const Geom& g, int pass, int num_sms, int smem_optin, SmallPlan* plan, int warps = 0,
                     int stages = 0, int slices = 0, bool pair = false);
cudaError_t launch_nchw_small(const Geom& g, const SmallPlan& p, int pass, const void* in, const void* in2,
                              const void* w, void* out, float* dw, void* ws, cudaStream_t st);

// ---- NCHW chunk kernels: nchw_chunk.cu
struct ChunkPlan {
  int threads;          // CTA size
  int grid;             // CTAs
  int smem_bytes;       // dynamic smem per CTA
  int ri;               // strip-height variant (template index)
  int R;                // strip height (output rows per thread strip)
  int vi, V;            // column-vector variant: V = 1 << vi output columns per thread strip
  bool padded;          // input planes staged with zero rows around them
  bool pair;            // fwd bf16: strips of two planes at once (FFMA2 lanes = planes)
  int pitch, zbe;       // padded staging: elements between planes, zero elements above a plane
  int ncg;              // column groups (strips across a row)
  int nsb;              // strips down a band
  int P;                // input planes per chunk (full-plane mode); 1 in band mode
  int nbands;           // bands per plane (1 => full-plane mode)
  int band_rows;        // output rows per band (fwd: y rows, bwd_data: dx rows, bwd_filter: dy rows)
  int64_t nchunks;      // fwd/bwd_data: chunks iterated by the persistent grid
  // shared-memory layout (bytes): barriers | zero row | weights | ns input stages | 2 output stages
  int ns;                       // input stages (TMA loads in flight = ns - 1)
  uint32_t zrow_off, w_off;
  uint32_t in0_off, in_stage;   // first input stage, stride between input stages
  uint32_t in_bytes;            // input buffer (x / dy) inside a stage, after 128 B of zero slack
  uint32_t in2_off, in2_bytes;  // bwd_filter: dy buffer inside a stage
  uint32_t out0_off, out_stage, out_bytes;  // output stages (y / dx)
  // bwd_filter only
  int groups;           // channel groups of P channels
  int nslices;          // batch slices per group
  int n_per_slice;      // images per slice
  int tpg;              // threads per dy plane
  int max_chain;        // worst-case serial depth of the dw sums
  size_t ws_bytes;      // workspace
  // bwd_filter register-direct variant (direct_bwd_filter.cu): no smem staging
  bool direct;
  int dL, dSPW, dspc;   // lanes per row set, row sets per warp, row sets per channel
  int dstream;          // > 0: bf16 streaming variant (sdbf_kernel) with bands of dstream dy rows
  // small-plane warp-task kernels (nchw_small.cu)
  bool small;
  SmallPlan sp;
};

constexpr int kPassBwdFused = DWCONV_PASS_BWD;  // plan_nchw pass id of the fused backward

// Returns false if the NCHW chunk family cannot handle the geometry.
// cands: optionally also the distinct candidate plans (default first, then by score),
// at most max_cands, for measurement-driven selection (dwconv_plan_candidates).
bool plan_nchw(const Geom& g, int pass, int num_sms, int max_smem_optin, ChunkPlan* plan,
               std::vector<ChunkPlan>* cands = nullptr, int max_cands = 0);
bool small_chunk_plan(const Geom& g, int pass, int num_sms, int smem_optin, ChunkPlan* plan, int warps = 0,
                      int stages = 0, int slices = 0, bool pair = false);
bool lane_chunk_plan(const Geom& g, int pass, int num_sms, int smem_optin, ChunkPlan* plan, int warps, int stages,
                     int slices = 0);
bool band_chunk_plan(const Geom& g, int num_sms, int smem_optin, ChunkPlan* plan, int warps, int stages, int rows,
                     int ppw = 1);
cudaError_t launch_nchw_fwd(const Geom& g, const ChunkPlan& p, const void* x, const void* w, void* y,
                            cudaStream_t st);
cudaError_t launch_nchw_bwd_data(const Geom& g, const ChunkPlan& p, const void* dy, const void* w, void* dx,
                                 cudaStream_t st);
cudaError_t launch_nchw_bwd_filter(const Geom& g, const ChunkPlan& p, const void* x, const void* dy, float* dw,
                                   void* ws, cudaStream_t st);
cudaError_t launch_nchw_bwd_fused(const Geom& g, const ChunkPlan& p, const void* x, const void* dy, const void* w,
                                  void* dx, float* dw, void* ws, cudaStream_t st);

// ---- NHWC kernels (m = 1, 3x3, pad 1, S in {1,2}): nhwc.cu
struct NhwcPlan {
  int threads, grid, smem;
  int TH, TW;             // fwd / bwd_data output tile; bwd_filter: dy columns per block
  int OHB, OWB;           // tiles along output rows / columns
  int64_t items;          // fwd / bwd_data work items (tile x channel vector)
  int CVB, PSET;          // bwd_filter: channel vectors per CTA, pixel sets per channel vector
  int groups, nslices, rps;
  int max_chain;
  size_t ws_bytes;
};
bool plan_nhwc(const Geom& g, int pass, int num_sms, NhwcPlan* plan);
cudaError_t launch_nhwc_fd(const Geom& g, const NhwcPlan& p, int pass, const void* in, const void* w, void* out,
                           cudaStream_t st);
cudaError_t launch_nhwc_bwd_filter(const Geom& g, const NhwcPlan& p, const void* x, const void* dy, float* dw,
                                   void* ws, cudaStream_t st);

// ---- NHWC fwd / bwd_data from tensor-map TMA tiles (m = 1, 3x3, pad 1, S in {1,2}): nhwc_tma.cu
struct NhwcTmaPlan {
  int mode;               // 0 fwd s1, 1 fwd s2, 2 bwd_data s1, 3 bwd_data s2
  int threads, grid, smem, ns;
  int TH, TW, CB, NCV, BW, BH, cons;
  int tiles_h, tiles_w, ncb;
  int64_t ntiles;
  uint32_t box_bytes, stage_bytes;
  // bwd_filter (mode 5 / 6 = stride 1 / 2)
  uint32_t dy_bytes, dy_off;
  int tiles_per_cb, nslices, tps, max_chain;
  size_t ws_bytes;
};
// tw_max / stages: tile-column cap and ring depth (0 = the defaults, env DWCONV_NHWC_TW / _STAGES)
bool plan_nhwc_tma(const Geom& g, int pass, int num_sms, int smem_optin, NhwcTmaPlan* plan, int tw_max = 0,
                   int stages = 0, int th = 0);
cudaError_t launch_nhwc_tma(const Geom& g, const NhwcTmaPlan& p, const void* in, const void* w, void* out,
                            cudaStream_t st);
bool plan_nhwc_tma_bf(const Geom& g, int num_sms, int smem_optin, NhwcTmaPlan* plan, int tw_max = 0,
                      int stages = 0, int th = 0);
cudaError_t launch_nhwc_tma_bf(const Geom& g, const NhwcTmaPlan& p, const void* x, const void* dy, float* dw,
                               void* ws, cudaStream_t st);

// ---- NHWC K x K (3/5/7), stride 1/2, multiplier 1/2/4 register-tile kernels: nhwc_gen.cu
struct NhwcGenPlan {
  int K, S, M, pass;
  int CVB, ncb, threads, grid, smem;
  int TH, TW, OHB, OWB, slots, ctas_per_cb;  // fwd / bwd_data
  int64_t tiles;
  int PS, nslices, rps, max_chain;            // bwd_filter
  size_t part_off, l2_off, t1_off, t2_off, ws_bytes;
  // bwd_filter staged through shared memory by tensor-map TMA (tma = true)
  bool tma;
  int CB, NCP, NCS, CW, TR, XR, BWX, bpi, units, ups;
  uint32_t x_bytes, dy_bytes, stage_bytes;
};
bool plan_nhwc_gen(const Geom& g, int pass, int num_sms, int smem_optin, NhwcGenPlan* plan);
cudaError_t launch_nhwc_gen_fd(const Geom& g, const NhwcGenPlan& p, const void* in, const void* w, void* out,
                               cudaStream_t st);
cudaError_t launch_nhwc_gen_bf(const Geom& g, const NhwcGenPlan& p, const void* x, const void* dy, float* dw,
                               void* ws, cudaStream_t st);

// ---- the paper's block-diagonal GEMM on tcgen05 (NHWC bf16, m = 1, stride 1, K in {3,5,7}): nhwc_bdmma.cu
struct BdmmaPlan {
  int K, S, CB, pass, pad, TW;
  int tiles_h, tiles_w, tiles_per_cb, ncb, ctas_per_cb;
  int grid, smem;
};
bool plan_nhwc_bdmma(const Geom& g, int pass, int num_sms, int smem_optin, int S, int CB, BdmmaPlan* plan);
cudaError_t launch_nhwc_bdmma(const Geom& g, const BdmmaPlan& p, const void* in, const void* w, void* out,
                              cudaStream_t st);

}  // namespace dwk
