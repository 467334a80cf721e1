// host.cpp -- the C ABI of include/dwconv.h: validation, kernel-family
// selection, launch.  No allocation, no synchronisation, no device switch.
#include <algorithm>
#include <array>
#include <atomic>
#include <map>
#include <climits>
#include <cstring>
#include <mutex>
#include <new>
#include <vector>

#include <cuda_runtime.h>

#include "../../include/dwconv.h"
#include "kernels.h"

namespace {

using dwk::ChunkPlan;
using dwk::Geom;
using dwk::NhwcPlan;

std::atomic<int> g_override{0};

struct DevInfo {
  int sms = 0, major = 0, minor = 0, smem_optin = 0;
  bool ok = false;
};

// Per-device attribute cache (attributes never change for a device).
bool dev_info(DevInfo* out) {
  static std::mutex mu;
  static DevInfo cache[64];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return false;
  std::lock_guard<std::mutex> lk(mu);
  DevInfo& d = cache[dev];
  if (!d.ok) {
    if (cudaDeviceGetAttribute(&d.sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return false;
    cudaDeviceGetAttribute(&d.major, cudaDevAttrComputeCapabilityMajor, dev);
    cudaDeviceGetAttribute(&d.minor, cudaDevAttrComputeCapabilityMinor, dev);
    cudaDeviceGetAttribute(&d.smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    d.ok = true;
  }
  *out = d;
  return true;
}

int out_size(int64_t in, int k, int s, int p, int64_t* o) {
  const int64_t num = in + 2 * (int64_t)p - k;
  if (num < 0) return 0;
  *o = num / s + 1;
  return 1;
}

// Validation shared by every entry point.  Fills g on success.
int validate(const dwconv_desc* d, Geom* g) {
  if (!d) return DWCONV_ERR_NULL_POINTER;
  if (d->n < 0 || d->c < 1 || d->h < 1 || d->w < 1) return DWCONV_ERR_BAD_DESCRIPTOR;
  if (d->multiplier < 1 || d->kh < 1 || d->kw < 1 || d->stride_h < 1 || d->stride_w < 1) return DWCONV_ERR_BAD_DESCRIPTOR;
  if (d->pad_h < 0 || d->pad_w < 0) return DWCONV_ERR_BAD_DESCRIPTOR;
  if (d->layout != DWCONV_NCHW && d->layout != DWCONV_NHWC) return DWCONV_ERR_BAD_DESCRIPTOR;
  if (d->dtype != DWCONV_F32 && d->dtype != DWCONV_BF16) return DWCONV_ERR_BAD_DESCRIPTOR;
  if (d->h > INT_MAX || d->w > INT_MAX || d->c > INT_MAX || d->n > INT_MAX) return DWCONV_ERR_BAD_DESCRIPTOR;
  if ((int64_t)d->kh > d->h + 2 * (int64_t)d->pad_h || (int64_t)d->kw > d->w + 2 * (int64_t)d->pad_w)
    return DWCONV_ERR_KERNEL_EXCEEDS_INPUT;
  int64_t ho = 0, wo = 0;
  if (!out_size(d->h, d->kh, d->stride_h, d->pad_h, &ho) || !out_size(d->w, d->kw, d->stride_w, d->pad_w, &wo) ||
      ho < 1 || wo < 1)
    return DWCONV_ERR_KERNEL_EXCEEDS_INPUT;
  // element counts must stay far from int64 overflow (2^62)
  const __int128 cm = (__int128)d->c * d->multiplier;
  const __int128 xs = (__int128)d->n * d->c * d->h * d->w;
  const __int128 ys = (__int128)d->n * cm * ho * wo;
  const __int128 ws = cm * d->kh * d->kw;
  const __int128 lim = (__int128)1 << 62;
  if (xs > lim || ys > lim || ws > INT_MAX || cm > INT_MAX) return DWCONV_ERR_BAD_DESCRIPTOR;
  g->N = d->n; g->C = d->c; g->H = d->h; g->W = d->w; g->Ho = ho; g->Wo = wo;
  g->m = d->multiplier; g->kh = d->kh; g->kw = d->kw; g->sh = d->stride_h; g->sw = d->stride_w;
  g->ph = d->pad_h; g->pw = d->pad_w; g->layout = d->layout; g->dtype = d->dtype;
  return DWCONV_OK;
}

int check_ptr(const void* p, int64_t elems, int eb) {
  if (elems == 0) return DWCONV_OK;
  if (!p) return DWCONV_ERR_NULL_POINTER;
  if (reinterpret_cast<uintptr_t>(p) % (uintptr_t)eb) return DWCONV_ERR_MISALIGNED;
  return DWCONV_OK;
}

int check_device(DevInfo* di) {
  if (!dev_info(di)) return DWCONV_ERR_CUDA;
  // the library carries only an sm_100a cubin (no PTX): other 10.x parts (sm_103)
  // cannot load it, so they are UNSUPPORTED rather than a later launch failure
  if (di->major != 10 || di->minor != 0) return DWCONV_ERR_UNSUPPORTED;
  return DWCONV_OK;
}

struct Plan {
  int variant = DWCONV_VARIANT_NONE;
  ChunkPlan chunk{};
  NhwcPlan nhwc{};
  dwk::NhwcTmaPlan tma{};
  dwk::BdmmaPlan bdmma{};
  dwk::NhwcGenPlan gen{};
};

// Choose the kernel family for a pass.  Pure host computation, memoised per
// (geometry, pass, device, override) because the planner searches many chunkings.
void make_plan_uncached(const Geom& g, int pass, const DevInfo& di, Plan* p);

using PlanKey = std::array<int64_t, 18>;
PlanKey plan_key(const Geom& g, int pass, const DevInfo& di) {
  int dev = 0;
  cudaGetDevice(&dev);
  return {g.N, g.C, g.H, g.W, g.m, g.kh, g.kw, g.sh, g.sw, g.ph, g.pw, g.layout, g.dtype, pass, dev,
          g_override.load(), di.sms, 0};
}

// Plans chosen by measurement (dwconv_plan_select) take precedence over the
// planner's own pick for the same geometry, pass and device.
std::mutex g_sel_mu;
std::map<PlanKey, Plan> g_selected;
std::map<PlanKey, std::vector<Plan>> g_candidates;

void make_plan(const Geom& g, int pass, const DevInfo& di, Plan* p) {
  static std::mutex mu;
  static std::map<PlanKey, Plan> cache;
  const PlanKey key = plan_key(g, pass, di);
  {
    std::lock_guard<std::mutex> lk(g_sel_mu);
    auto it = g_selected.find(key);
    if (it != g_selected.end()) { *p = it->second; return; }
  }
  {
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find(key);
    if (it != cache.end()) { *p = it->second; return; }
  }
  make_plan_uncached(g, pass, di, p);
  std::lock_guard<std::mutex> lk(mu);
  if (cache.size() > 4096) cache.clear();
  cache[key] = *p;
}

void make_plan_uncached(const Geom& g, int pass, const DevInfo& di, Plan* p) {
  p->variant = DWCONV_VARIANT_GENERIC;
  if (g.N == 0) { p->variant = DWCONV_VARIANT_NONE; return; }
  if (g_override.load() == DWCONV_VARIANT_GENERIC) return;
  if (g.layout == DWCONV_NCHW && dwk::plan_nchw(g, pass, di.sms, di.smem_optin, &p->chunk)) {
    if ((pass != DWCONV_PASS_BWD_FILTER && pass != DWCONV_PASS_BWD) || p->chunk.max_chain <= 160)
      p->variant = DWCONV_VARIANT_NCHW_CHUNK;
  }
  // small square planes: the warp-task kernels (nchw_small.cu) when eligible
  ChunkPlan sp;
  if (g.layout == DWCONV_NCHW && (pass != DWCONV_PASS_BWD || g.dtype == DWCONV_F32) &&
      dwk::small_chunk_plan(g, pass, di.sms, di.smem_optin, &sp)) {
    p->chunk = sp;
    p->variant = DWCONV_VARIANT_NCHW_CHUNK;
  }
  if (pass == DWCONV_PASS_BWD) {  // fused backward: NCHW chunk family, fp32 (bf16 measured slower fused)
    if (p->variant != DWCONV_VARIANT_NCHW_CHUNK || g.dtype != DWCONV_F32) p->variant = DWCONV_VARIANT_NONE;
    return;
  }
  if (g.layout == DWCONV_NHWC && pass == DWCONV_PASS_BWD_FILTER &&
      dwk::plan_nhwc_tma_bf(g, di.sms, di.smem_optin, &p->tma)) {
    p->variant = DWCONV_VARIANT_NHWC_TMA;
    if (!dwk::plan_nhwc(g, pass, di.sms, &p->nhwc)) p->nhwc = NhwcPlan{};  // for unaligned pointers
    return;
  }
  if (g.layout == DWCONV_NHWC && dwk::plan_nhwc_tma(g, pass, di.sms, di.smem_optin, &p->tma)) {
    p->variant = DWCONV_VARIANT_NHWC_TMA;
    if (!dwk::plan_nhwc(g, pass, di.sms, &p->nhwc)) p->nhwc = NhwcPlan{};  // for unaligned pointers
    return;
  }
  if (g.layout == DWCONV_NHWC && dwk::plan_nhwc(g, pass, di.sms, &p->nhwc)) {
    p->variant = DWCONV_VARIANT_NHWC_TILE;
    return;
  }
  // K = 5 / 7, m = 2 / 4, the rest of stride 1 / 2: the general NHWC register-tile kernels
  if (g.layout == DWCONV_NHWC && dwk::plan_nhwc_gen(g, pass, di.sms, di.smem_optin, &p->gen) &&
      (pass != DWCONV_PASS_BWD_FILTER || p->gen.max_chain <= 160))
    p->variant = DWCONV_VARIANT_NHWC_GEN;
}

int cuda_status(cudaError_t e) { return e == cudaSuccess ? DWCONV_OK : DWCONV_ERR_CUDA; }

// the NHWC kernels move 4-channel vectors: 16-B (fp32) / 8-B (bf16) aligned activations
// tensor-map base and 16-B vector stores (fp32) / 8-B (bf16)
bool tma_aligned(const void* in, const void* out) {
  return ((reinterpret_cast<uintptr_t>(in) | reinterpret_cast<uintptr_t>(out)) % 16) == 0;
}

bool nhwc_aligned(const Geom& g, const void* a, const void* b) {
  const uintptr_t al = (g.dtype == DWCONV_F32) ? 16 : 8;
  return ((reinterpret_cast<uintptr_t>(a) | reinterpret_cast<uintptr_t>(b)) % al) == 0;
}

}  // namespace

extern "C" {

int dwconv_abi_version(void) { return DWCONV_ABI_VERSION; }

const char* dwconv_status_string(int s) {
  switch (s) {
    case DWCONV_OK: return "ok";
    case DWCONV_ERR_NULL_POINTER: return "null pointer for a non-empty tensor";
    case DWCONV_ERR_BAD_DESCRIPTOR: return "bad descriptor";
    case DWCONV_ERR_KERNEL_EXCEEDS_INPUT: return "kernel exceeds padded input";
    case DWCONV_ERR_MISALIGNED: return "pointer not aligned to its element size";
    case DWCONV_ERR_WORKSPACE_TOO_SMALL: return "workspace too small";
    case DWCONV_ERR_UNSUPPORTED: return "unsupported device (needs sm_100)";
    case DWCONV_ERR_CUDA: return "CUDA error";
    default: return "unknown status";
  }
}

int dwconv_output_shape(const dwconv_desc* d, int64_t* ho, int64_t* wo) {
  Geom g;
  const int s = validate(d, &g);
  if (s != DWCONV_OK) return s;
  if (!ho || !wo) return DWCONV_ERR_NULL_POINTER;
  *ho = g.Ho;
  *wo = g.Wo;
  return DWCONV_OK;
}

int dwconv_set_variant_override(int v) {
  if (v != 0 && v != DWCONV_VARIANT_GENERIC) return DWCONV_ERR_BAD_DESCRIPTOR;
  g_override.store(v);
  return DWCONV_OK;
}

}  // extern "C"

namespace {

// ---- dispatch from a resolved (geometry, plan): shared by the descriptor calls
// (plan chosen per call: the planner's pick or a dwconv_plan_select selection)
// and the immutable plan handles (dwconv_plan_create).
int ptr_check_fd(const Geom& g, int pass, const void* in, const void* w, const void* out) {
  const int eb = g.dtype == DWCONV_F32 ? 4 : 2;
  const int64_t nx = g.N * g.C * g.H * g.W, ny = g.N * g.C * g.m * g.Ho * g.Wo;
  int s;
  if ((s = check_ptr(in, pass == DWCONV_PASS_FWD ? nx : ny, eb)) || (s = check_ptr(w, g.C * g.m * g.kh * g.kw, eb)) ||
      (s = check_ptr(out, pass == DWCONV_PASS_FWD ? ny : nx, eb)))
    return s;
  return DWCONV_OK;
}

int run_fwd(const Geom& g, const Plan& p, const void* x, const void* w, void* y, cudaStream_t st) {
  if (g.N == 0) return DWCONV_OK;
  // the NCHW kernels store y with V-wide vector stores straight from registers
  if (p.variant == DWCONV_VARIANT_NCHW_CHUNK && (reinterpret_cast<uintptr_t>(y) % 16) == 0 &&
      (!p.chunk.small || (reinterpret_cast<uintptr_t>(x) % 16) == 0))
    return cuda_status(dwk::launch_nchw_fwd(g, p.chunk, x, w, y, st));
  if (p.variant == DWCONV_VARIANT_NHWC_TMA && tma_aligned(x, y))
    return cuda_status(dwk::launch_nhwc_tma(g, p.tma, x, w, y, st));
  if (p.variant == DWCONV_VARIANT_NHWC_BDMMA && tma_aligned(x, y))
    return cuda_status(dwk::launch_nhwc_bdmma(g, p.bdmma, x, w, y, st));
  if (p.variant == DWCONV_VARIANT_NHWC_GEN && tma_aligned(x, y))
    return cuda_status(dwk::launch_nhwc_gen_fd(g, p.gen, x, w, y, st));
  if ((p.variant == DWCONV_VARIANT_NHWC_TILE || p.variant == DWCONV_VARIANT_NHWC_TMA) && p.nhwc.grid > 0 &&
      nhwc_aligned(g, x, y))
    return cuda_status(dwk::launch_nhwc_fd(g, p.nhwc, DWCONV_PASS_FWD, x, w, y, st));
  return cuda_status(dwk::launch_generic_fwd(g, x, w, y, st));
}

int run_bwd_data(const Geom& g, const Plan& p, const void* dy, const void* w, void* dx, cudaStream_t st) {
  if (g.N == 0) return DWCONV_OK;
  // the NCHW kernels store dx with vector stores straight from registers
  if (p.variant == DWCONV_VARIANT_NCHW_CHUNK && (reinterpret_cast<uintptr_t>(dx) % 16) == 0 &&
      (!p.chunk.small || (reinterpret_cast<uintptr_t>(dy) % 16) == 0))
    return cuda_status(dwk::launch_nchw_bwd_data(g, p.chunk, dy, w, dx, st));
  if (p.variant == DWCONV_VARIANT_NHWC_TMA && tma_aligned(dy, dx))
    return cuda_status(dwk::launch_nhwc_tma(g, p.tma, dy, w, dx, st));
  if (p.variant == DWCONV_VARIANT_NHWC_BDMMA && tma_aligned(dy, dx))
    return cuda_status(dwk::launch_nhwc_bdmma(g, p.bdmma, dy, w, dx, st));
  if (p.variant == DWCONV_VARIANT_NHWC_GEN && tma_aligned(dy, dx))
    return cuda_status(dwk::launch_nhwc_gen_fd(g, p.gen, dy, w, dx, st));
  if ((p.variant == DWCONV_VARIANT_NHWC_TILE || p.variant == DWCONV_VARIANT_NHWC_TMA) && p.nhwc.grid > 0 &&
      nhwc_aligned(g, dy, dx))
    return cuda_status(dwk::launch_nhwc_fd(g, p.nhwc, DWCONV_PASS_BWD_DATA, dy, w, dx, st));
  return cuda_status(dwk::launch_generic_bwd_data(g, dy, w, dx, st));
}

size_t bf_workspace_bytes(const Plan& p) {
  if (p.variant == DWCONV_VARIANT_NHWC_TILE) return p.nhwc.ws_bytes;
  if (p.variant == DWCONV_VARIANT_NHWC_GEN) return p.gen.ws_bytes;
  if (p.variant == DWCONV_VARIANT_NHWC_TMA)  // either NHWC kernel may run (pointer alignment)
    return std::max(p.tma.ws_bytes, p.nhwc.grid > 0 ? p.nhwc.ws_bytes : (size_t)0);
  return p.variant == DWCONV_VARIANT_NCHW_CHUNK ? p.chunk.ws_bytes : 0;
}

int ws_check(const void* ws, size_t have, size_t need) {
  if (have < need) return DWCONV_ERR_WORKSPACE_TOO_SMALL;
  if (need == 0) return DWCONV_OK;
  if (!ws) return DWCONV_ERR_NULL_POINTER;
  if (reinterpret_cast<uintptr_t>(ws) % 16) return DWCONV_ERR_MISALIGNED;
  return DWCONV_OK;
}

int run_bwd_filter(const Geom& g, const Plan& p, const void* x, const void* dy, float* dw, void* workspace,
                   size_t workspace_bytes, cudaStream_t st) {
  if (g.N == 0) return cuda_status(cudaMemsetAsync(dw, 0, (size_t)(g.C * g.m * g.kh * g.kw) * 4, st));
  int s;
  // the register-direct variant needs 16-B aligned x and dy (vector loads)
  const bool direct_ok = !(p.chunk.direct || p.chunk.small) ||
                         ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(dy)) % 16) == 0;
  if (p.variant == DWCONV_VARIANT_NCHW_CHUNK && direct_ok) {
    if ((s = ws_check(workspace, workspace_bytes, p.chunk.ws_bytes))) return s;
    return cuda_status(dwk::launch_nchw_bwd_filter(g, p.chunk, x, dy, dw, workspace, st));
  }
  if (p.variant == DWCONV_VARIANT_NHWC_TMA && tma_aligned(x, dy)) {
    if ((s = ws_check(workspace, workspace_bytes, p.tma.ws_bytes))) return s;
    return cuda_status(dwk::launch_nhwc_tma_bf(g, p.tma, x, dy, dw, workspace, st));
  }
  if ((p.variant == DWCONV_VARIANT_NHWC_TILE || p.variant == DWCONV_VARIANT_NHWC_TMA) && p.nhwc.grid > 0 &&
      nhwc_aligned(g, x, dy)) {
    if ((s = ws_check(workspace, workspace_bytes, p.nhwc.ws_bytes))) return s;
    return cuda_status(dwk::launch_nhwc_bwd_filter(g, p.nhwc, x, dy, dw, workspace, st));
  }
  if (p.variant == DWCONV_VARIANT_NHWC_GEN && tma_aligned(x, dy)) {
    if ((s = ws_check(workspace, workspace_bytes, p.gen.ws_bytes))) return s;
    return cuda_status(dwk::launch_nhwc_gen_bf(g, p.gen, x, dy, dw, workspace, st));
  }
  return cuda_status(dwk::launch_generic_bwd_filter(g, x, dy, dw, st));
}

// fused backward: pf = the PASS_BWD plan; pd / pb = the two-call fallback plans
int run_bwd(const Geom& g, const Plan& pf, const Plan& pd, const Plan& pb, const void* x, const void* dy,
            const void* w, void* dx, float* dw, void* workspace, size_t workspace_bytes, cudaStream_t st) {
  int s;
  // the fused kernel stores dx with vector stores straight from registers
  if (g.N > 0 && pf.variant == DWCONV_VARIANT_NCHW_CHUNK && (reinterpret_cast<uintptr_t>(dx) % 16) == 0 &&
      (!pf.chunk.small || ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(dy)) % 16) == 0)) {
    if ((s = ws_check(workspace, workspace_bytes, pf.chunk.ws_bytes))) return s;
    return cuda_status(dwk::launch_nchw_bwd_fused(g, pf.chunk, x, dy, w, dx, dw, workspace, st));
  }
  if ((s = run_bwd_data(g, pd, dy, w, dx, st))) return s;
  return run_bwd_filter(g, pb, x, dy, dw, workspace, workspace_bytes, st);
}

size_t bwd_workspace_bytes(const Plan& pf, const Plan& pb) {
  const size_t two = bf_workspace_bytes(pb);
  return pf.variant == DWCONV_VARIANT_NCHW_CHUNK ? std::max(pf.chunk.ws_bytes, two) : two;
}

}  // namespace

// Immutable launch plan: geometry, pass and the resolved kernel plan(s), fixed at
// creation; calls through it read nothing that any other call can change.
struct dwconv_plan_s {
  Geom g;
  int pass = 0;
  int device = 0;
  int candidate = -1;
  Plan p;       // the pass's plan (PASS_BWD: the fused plan)
  Plan pd, pb;  // PASS_BWD: the two-call fallback's bwd_data / bwd_filter plans (planner defaults)
};

extern "C" {

int dwconv_fwd(const dwconv_desc* d, const void* x, const void* w, void* y, dwconv_stream stream) {
  Geom g;
  int s = validate(d, &g);
  if (s != DWCONV_OK) return s;
  if ((s = ptr_check_fd(g, DWCONV_PASS_FWD, x, w, y))) return s;
  if (g.N == 0) return DWCONV_OK;
  DevInfo di;
  if ((s = check_device(&di))) return s;
  Plan p;
  make_plan(g, DWCONV_PASS_FWD, di, &p);
  return run_fwd(g, p, x, w, y, reinterpret_cast<cudaStream_t>(stream));
}

int dwconv_bwd_data(const dwconv_desc* d, const void* dy, const void* w, void* dx, dwconv_stream stream) {
  Geom g;
  int s = validate(d, &g);
  if (s != DWCONV_OK) return s;
  if ((s = ptr_check_fd(g, DWCONV_PASS_BWD_DATA, dy, w, dx))) return s;
  if (g.N == 0) return DWCONV_OK;
  DevInfo di;
  if ((s = check_device(&di))) return s;
  Plan p;
  make_plan(g, DWCONV_PASS_BWD_DATA, di, &p);
  return run_bwd_data(g, p, dy, w, dx, reinterpret_cast<cudaStream_t>(stream));
}

size_t dwconv_bwd_filter_workspace_bytes(const dwconv_desc* d) {
  Geom g;
  if (validate(d, &g) != DWCONV_OK) return 0;
  DevInfo di;
  if (check_device(&di) != DWCONV_OK) return 0;
  Plan p;
  make_plan(g, DWCONV_PASS_BWD_FILTER, di, &p);
  return bf_workspace_bytes(p);
}

static int ptr_check_bf(const Geom& g, const void* x, const void* dy, const float* dw) {
  const int eb = g.dtype == DWCONV_F32 ? 4 : 2;
  int s;
  if ((s = check_ptr(x, g.N * g.C * g.H * g.W, eb)) || (s = check_ptr(dy, g.N * g.C * g.m * g.Ho * g.Wo, eb)) ||
      (s = check_ptr(dw, g.C * g.m * g.kh * g.kw, 4)))
    return s;
  return DWCONV_OK;
}

int dwconv_bwd_filter(const dwconv_desc* d, const void* x, const void* dy, float* dw, void* workspace,
                      size_t workspace_bytes, dwconv_stream stream) {
  Geom g;
  int s = validate(d, &g);
  if (s != DWCONV_OK) return s;
  if ((s = ptr_check_bf(g, x, dy, dw))) return s;
  DevInfo di;
  if ((s = check_device(&di))) return s;
  Plan p;
  if (g.N > 0) make_plan(g, DWCONV_PASS_BWD_FILTER, di, &p);
  return run_bwd_filter(g, p, x, dy, dw, workspace, workspace_bytes, reinterpret_cast<cudaStream_t>(stream));
}

size_t dwconv_bwd_workspace_bytes(const dwconv_desc* d) {
  Geom g;
  if (validate(d, &g) != DWCONV_OK) return 0;
  DevInfo di;
  if (check_device(&di) != DWCONV_OK) return 0;
  Plan pf, pb;
  make_plan(g, DWCONV_PASS_BWD, di, &pf);
  make_plan(g, DWCONV_PASS_BWD_FILTER, di, &pb);
  return bwd_workspace_bytes(pf, pb);
}

int dwconv_bwd(const dwconv_desc* d, const void* x, const void* dy, const void* w, void* dx, float* dw,
               void* workspace, size_t workspace_bytes, dwconv_stream stream) {
  Geom g;
  int s = validate(d, &g);
  if (s != DWCONV_OK) return s;
  if ((s = ptr_check_bf(g, x, dy, dw)) || (s = ptr_check_fd(g, DWCONV_PASS_BWD_DATA, dy, w, dx))) return s;
  DevInfo di;
  if ((s = check_device(&di))) return s;
  Plan pf, pd, pb;
  if (g.N > 0) {
    make_plan(g, DWCONV_PASS_BWD, di, &pf);
    make_plan(g, DWCONV_PASS_BWD_DATA, di, &pd);
    make_plan(g, DWCONV_PASS_BWD_FILTER, di, &pb);
  }
  return run_bwd(g, pf, pd, pb, x, dy, w, dx, dw, workspace, workspace_bytes,
                 reinterpret_cast<cudaStream_t>(stream));
}

int dwconv_workspace_init(void* workspace, size_t workspace_bytes, dwconv_stream stream) {
  if (workspace_bytes == 0) return DWCONV_OK;
  if (!workspace) return DWCONV_ERR_NULL_POINTER;
  return cuda_status(cudaMemsetAsync(workspace, 0, workspace_bytes, reinterpret_cast<cudaStream_t>(stream)));
}

static void fill_info(const Geom& g, const Plan& p, int pass, dwconv_plan_info* info) {
  std::memset(info, 0, sizeof(*info));
  info->variant = p.variant;
  if (pass == DWCONV_PASS_BWD && p.variant != DWCONV_VARIANT_NCHW_CHUNK) {  // two-call fallback
    info->variant = DWCONV_VARIANT_NONE;
    info->launches = 2;
    return;
  }
  if (p.variant == DWCONV_VARIANT_NCHW_CHUNK) {
    const ChunkPlan& c = p.chunk;
    info->grid = c.grid; info->block = c.threads; info->smem_bytes = c.smem_bytes; info->launches = 1;
    info->work_units = c.nchunks; info->planes_per_chunk = c.P; info->rows_per_band = c.band_rows;
    info->batch_slices = c.nslices; info->max_chain = c.max_chain; info->workspace_bytes = (int64_t)c.ws_bytes;
    info->kernel_family = c.direct ? (c.dstream > 0 ? 4 : 3) : (c.small ? (c.sp.lane ? 5 : c.sp.band ? 2 : 1) : 0);
  } else if (p.variant == DWCONV_VARIANT_NHWC_TMA) {
    const dwk::NhwcTmaPlan& c = p.tma;
    info->grid = c.grid; info->block = c.threads; info->smem_bytes = c.smem; info->launches = 1;
    info->work_units = c.ntiles; info->rows_per_band = c.TH; info->planes_per_chunk = c.TW;
    if (pass == DWCONV_PASS_BWD_FILTER) {
      info->work_units = (int64_t)c.ncb * c.tiles_per_cb;
      info->batch_slices = c.nslices; info->max_chain = c.max_chain;
      info->workspace_bytes = (int64_t)std::max(c.ws_bytes, p.nhwc.grid > 0 ? p.nhwc.ws_bytes : (size_t)0);
    }
  } else if (p.variant == DWCONV_VARIANT_NHWC_GEN) {
    const dwk::NhwcGenPlan& c = p.gen;
    info->grid = c.grid; info->block = c.threads; info->smem_bytes = c.smem; info->launches = 1;
    if (pass == DWCONV_PASS_BWD_FILTER) {
      info->work_units = (int64_t)c.ncb * c.nslices; info->batch_slices = c.nslices;
      info->max_chain = c.max_chain; info->workspace_bytes = (int64_t)c.ws_bytes;
    } else {
      info->work_units = c.tiles * c.ncb; info->rows_per_band = c.TH; info->planes_per_chunk = c.TW;
    }
  } else if (p.variant == DWCONV_VARIANT_NHWC_BDMMA) {
    const dwk::BdmmaPlan& c = p.bdmma;
    info->grid = c.grid; info->block = 192; info->smem_bytes = c.smem; info->launches = 1;
    info->work_units = (int64_t)c.ncb * c.tiles_per_cb;
    info->planes_per_chunk = c.S;   // group size S of the block-diagonal weight
    info->rows_per_band = c.CB;     // staged channel block (A rows of CB*2 bytes)
  } else if (p.variant == DWCONV_VARIANT_NHWC_TILE) {
    const NhwcPlan& c = p.nhwc;
    info->grid = c.grid; info->block = c.threads; info->smem_bytes = c.smem; info->launches = 1;
    info->work_units = (pass == DWCONV_PASS_BWD_FILTER) ? (int64_t)c.groups * c.nslices : c.items;
    info->batch_slices = c.nslices; info->max_chain = c.max_chain; info->workspace_bytes = (int64_t)c.ws_bytes;
  } else if (p.variant == DWCONV_VARIANT_GENERIC) {
    info->block = 256; info->launches = 1;
    if (pass == DWCONV_PASS_BWD_FILTER) {
      info->grid = (int)(g.C * g.m * g.kh * g.kw);
      const int64_t per = (g.N * g.Ho * g.Wo + 255) / 256;
      info->max_chain = (int)(64 + 64 + per / 4096 + 2 + 8);
    }
  } else if (pass == DWCONV_PASS_BWD_FILTER) {
    info->launches = 1;  // memset of dw
  }
}

// NHWC candidates: the TMA family at several tile widths / ring depths, then the
// L1 register-tile kernels.
static void nhwc_candidates(const Geom& g, int pass, const DevInfo& di, std::vector<Plan>* cands) {
  // {tile-column cap, ring depth, tile rows (0 = 7/8; 14 = two 7-row strips, stride 1)}
  static const int shapes[][3] = {{16, 2, 0}, {16, 3, 0}, {16, 4, 0}, {8, 2, 0}, {8, 3, 0}, {8, 4, 0},
                                  {4, 3, 0},  {4, 4, 0},  {32, 2, 0}, {16, 2, 14}, {16, 3, 14}, {8, 3, 14},
                                  {8, 4, 14}};
  for (const auto& sh : shapes) {
    Plan v;
    v.variant = DWCONV_VARIANT_NHWC_TMA;
    const bool ok = (pass == DWCONV_PASS_BWD_FILTER)
                        ? dwk::plan_nhwc_tma_bf(g, di.sms, di.smem_optin, &v.tma, sh[0], sh[1], sh[2])
                        : dwk::plan_nhwc_tma(g, pass, di.sms, di.smem_optin, &v.tma, sh[0], sh[1], sh[2]);
    if (!ok) continue;
    if (!dwk::plan_nhwc(g, pass, di.sms, &v.nhwc)) v.nhwc = NhwcPlan{};
    bool dup = false;
    for (const Plan& o : *cands)
      dup = dup || (o.variant == v.variant && o.tma.TW == v.tma.TW && o.tma.TH == v.tma.TH && o.tma.ns == v.tma.ns &&
                    o.tma.grid == v.tma.grid);
    if (!dup) cands->push_back(v);
  }
  Plan t;
  if (dwk::plan_nhwc(g, pass, di.sms, &t.nhwc)) {
    t.variant = DWCONV_VARIANT_NHWC_TILE;
    cands->push_back(t);
  }
}

int dwconv_plan_candidates(const dwconv_desc* d, int pass, int max_candidates, dwconv_plan_info* infos,
                           int* count) {
  Geom g;
  int s = validate(d, &g);
  if (s != DWCONV_OK) return s;
  if (!count || (max_candidates > 0 && !infos)) return DWCONV_ERR_NULL_POINTER;
  if (pass < DWCONV_PASS_FWD || pass > DWCONV_PASS_BWD || max_candidates < 0) return DWCONV_ERR_BAD_DESCRIPTOR;
  DevInfo di;
  if ((s = check_device(&di))) return s;
  *count = 0;
  if (g.N == 0 || g_override.load() == DWCONV_VARIANT_GENERIC) return DWCONV_OK;
  if (g.layout == DWCONV_NHWC && pass == DWCONV_PASS_BWD) return DWCONV_OK;
  const PlanKey key = plan_key(g, pass, di);
  std::vector<Plan> all;
  {
    std::lock_guard<std::mutex> lk(g_sel_mu);
    auto it = g_candidates.find(key);
    if (it != g_candidates.end()) all = it->second;
  }
  if (all.empty() && g.layout == DWCONV_NHWC) {
    Plan dp;
    make_plan_uncached(g, pass, di, &dp);
    // the paper's block-diagonal tensor-core GEMM, group sizes S = 16 / 32 / 64 over channel
    // blocks CB >= S (where the diagonal weight tiles fit in shared memory): measured
    // candidates, never the default
    std::vector<Plan> mma;
    static const int sc[][2] = {{16, 16}, {16, 32}, {32, 32}, {16, 64}, {32, 64}, {64, 64}};  // {S, CB}
    for (const auto& q : sc) {
      Plan v;
      v.variant = DWCONV_VARIANT_NHWC_BDMMA;
      if (dwk::plan_nhwc_bdmma(g, pass, di.sms, di.smem_optin, q[0], q[1], &v.bdmma)) mma.push_back(v);
    }
    if ((dp.variant == DWCONV_VARIANT_GENERIC || dp.variant == DWCONV_VARIANT_NHWC_GEN) && !mma.empty()) {
      all.push_back(dp);
      all.insert(all.end(), mma.begin(), mma.end());
    }
    if (dp.variant == DWCONV_VARIANT_NHWC_TMA || dp.variant == DWCONV_VARIANT_NHWC_TILE) {
      all.push_back(dp);
      nhwc_candidates(g, pass, di, &all);
      // drop a later duplicate of the default
      for (size_t i = 1; i < all.size(); ++i)
        if (all[i].variant == dp.variant && all[i].tma.TW == dp.tma.TW && all[i].tma.ns == dp.tma.ns &&
            all[i].tma.grid == dp.tma.grid && all[i].nhwc.grid == dp.nhwc.grid) {
          all.erase(all.begin() + (long)i);
          break;
        }
      all.insert(all.end(), mma.begin(), mma.end());
    }
    if ((int)all.size() > DWCONV_MAX_CANDIDATES) all.resize(DWCONV_MAX_CANDIDATES);
    std::lock_guard<std::mutex> lk(g_sel_mu);
    g_candidates[key] = all;
  }
  if (g.layout == DWCONV_NHWC) {
    const int n = std::min<int>((int)all.size(), max_candidates);
    for (int i = 0; i < n; ++i) fill_info(g, all[i], pass, &infos[i]);
    *count = (max_candidates == 0) ? (int)all.size() : n;
    return DWCONV_OK;
  }
  std::vector<ChunkPlan> cands;
  for (const Plan& q : all) cands.push_back(q.chunk);
  if (cands.empty()) {
    // the planner's own pick (what an unselected call launches) leads the list
    Plan dp;
    make_plan_uncached(g, pass, di, &dp);
    // candidate 0 is the planner's own pick; when that is not a chunk-family plan
    // (generic kernel, or bf16 fused backward = the two separate calls) there is
    // no list (the header's "0 candidates"), so index 0 never names a plan the
    // planner rejected
    if (dp.variant != DWCONV_VARIANT_NCHW_CHUNK) return DWCONV_OK;
    cands.push_back(dp.chunk);
    if (pass == DWCONV_PASS_BWD_FILTER && g.dtype <= DWCONV_BF16) {
      // band bwd_filter for large planes: {warps, ring slots, band rows}
      // {warps, ring slots, band rows, planes per warp}
      static const int bshapes[][4] = {{4, 2, 7, 1}, {4, 3, 7, 1}, {8, 2, 7, 1}, {2, 3, 7, 1}, {4, 2, 14, 1},
                                       {8, 2, 14, 1}, {4, 2, 7, 2}, {4, 3, 7, 2}, {8, 2, 7, 2}, {4, 2, 14, 2},
                                       {4, 2, 7, 3}, {4, 3, 7, 3}, {8, 2, 7, 3}, {4, 2, 14, 3},
                                       {4, 4, 7, 1}, {2, 4, 7, 1}, {4, 4, 7, 2}, {2, 4, 14, 2}};
      for (const auto& sh : bshapes) {
        ChunkPlan v;
        if (dwk::band_chunk_plan(g, di.sms, di.smem_optin, &v, sh[0], sh[1], sh[2], sh[3])) cands.push_back(v);
      }
    }
    if (pass <= DWCONV_PASS_BWD_FILTER) {
      // lane-per-plane kernels (7x7 / 14x14, s1): {warps, ring slots}
      static const int lshapes[][2] = {{4, 2}, {4, 3}, {8, 2}, {2, 3}, {2, 4}, {6, 2}, {8, 3}};
      std::vector<ChunkPlan> lv;
      for (const auto& sh : lshapes) {
        ChunkPlan v;
        if (dwk::lane_chunk_plan(g, pass, di.sms, di.smem_optin, &v, sh[0], sh[1])) lv.push_back(v);
      }
      cands.insert(cands.begin() + std::min<size_t>(1, cands.size()), lv.begin(), lv.end());
    }
    std::vector<ChunkPlan> more;
    ChunkPlan scratch;
    if (g.dtype == DWCONV_BF16 && pass <= DWCONV_PASS_BWD_FILTER) {
      // bf16 plane-pair small-plane kernels: {warps, ring slots}
      static const int pshapes[][2] = {{4, 2}, {4, 3}, {8, 2}, {2, 3}, {2, 2}};
      for (const auto& sh : pshapes) {
        ChunkPlan v;
        if (dwk::small_chunk_plan(g, pass, di.sms, di.smem_optin, &v, sh[0], sh[1], 0, true)) cands.push_back(v);
      }
    }
    if (!cands.empty() && cands[0].small) {
      // other CTA sizes / ring depths of the small-plane kernel, then the chunk family's own pick
      // {warps, ring slots, batch slices (bwd_filter; 0 = about one wave)}
      // (fwd / bwd_data: the third entry is tasks per warp instead)
      static const int shapes[][3] = {{2, 2, 0}, {2, 3, 0}, {4, 2, 0}, {8, 2, 0}, {8, 3, 0}, {8, 4, 0},
                                      {8, 2, 1}, {8, 3, 1}, {8, 2, 2}, {4, 3, 2}, {4, 2, 2}, {4, 2, 3},
                                      {4, 3, 4}, {2, 2, 4}, {2, 3, 6}, {8, 2, 3}};
      for (const auto& sh : shapes) {
        ChunkPlan v;
        if (!dwk::small_chunk_plan(g, pass, di.sms, di.smem_optin, &v, sh[0], sh[1], sh[2])) continue;
        bool dup = false;
        for (const ChunkPlan& o : cands)
          dup = dup || (o.small && !o.sp.pair && !o.sp.lane && o.threads == v.threads && o.ns == v.ns && o.nslices == v.nslices &&
                        o.grid == v.grid);
        if (!dup) cands.push_back(v);
      }
      if (dwk::plan_nchw(g, pass, di.sms, di.smem_optin, &scratch) &&
          (pass < DWCONV_PASS_BWD_FILTER || scratch.max_chain <= 160))
        cands.push_back(scratch);
    }
    if (dwk::plan_nchw(g, pass, di.sms, di.smem_optin, &scratch, &more, DWCONV_MAX_CANDIDATES) || !more.empty()) {
      for (const ChunkPlan& c : more) {
        if ((int)cands.size() >= DWCONV_MAX_CANDIDATES) break;
        bool dup = false;
        for (const ChunkPlan& o : cands)
          dup = dup || (o.P == c.P && o.nbands == c.nbands && o.band_rows == c.band_rows && o.threads == c.threads &&
                        o.tpg == c.tpg && o.ns == c.ns && o.pair == c.pair && o.direct == c.direct &&
                        o.dstream == c.dstream && o.V == c.V && o.small == c.small && o.sp.band == c.sp.band && o.sp.ppw == c.sp.ppw && o.nslices == c.nslices &&
                        o.grid == c.grid);
        if (!dup) cands.push_back(c);
      }
    }
    if ((int)cands.size() > DWCONV_MAX_CANDIDATES) cands.resize(DWCONV_MAX_CANDIDATES);
    std::vector<Plan> wrapped;
    for (const ChunkPlan& c : cands) {
      Plan q;
      q.variant = DWCONV_VARIANT_NCHW_CHUNK;
      q.chunk = c;
      wrapped.push_back(q);
    }
    std::lock_guard<std::mutex> lk(g_sel_mu);
    g_candidates[key] = wrapped;
  }
  const int n = std::min<int>((int)cands.size(), max_candidates);
  for (int i = 0; i < n; ++i) {
    Plan q;
    q.variant = DWCONV_VARIANT_NCHW_CHUNK;
    q.chunk = cands[i];
    fill_info(g, q, pass, &infos[i]);
  }
  *count = (max_candidates == 0) ? (int)cands.size() : n;
  return DWCONV_OK;
}

int dwconv_plan_select(const dwconv_desc* d, int pass, int index) {
  Geom g;
  int s = validate(d, &g);
  if (s != DWCONV_OK) return s;
  if (pass < DWCONV_PASS_FWD || pass > DWCONV_PASS_BWD) return DWCONV_ERR_BAD_DESCRIPTOR;
  DevInfo di;
  if ((s = check_device(&di))) return s;
  const PlanKey key = plan_key(g, pass, di);
  std::lock_guard<std::mutex> lk(g_sel_mu);
  if (index < 0) { g_selected.erase(key); return DWCONV_OK; }
  auto it = g_candidates.find(key);
  if (it == g_candidates.end() || index >= (int)it->second.size()) return DWCONV_ERR_BAD_DESCRIPTOR;
  g_selected[key] = it->second[(size_t)index];
  return DWCONV_OK;
}

int dwconv_plan(const dwconv_desc* d, int pass, dwconv_plan_info* info) {
  Geom g;
  int s = validate(d, &g);
  if (s != DWCONV_OK) return s;
  if (!info) return DWCONV_ERR_NULL_POINTER;
  if (pass < 0 || pass > 3) return DWCONV_ERR_BAD_DESCRIPTOR;
  DevInfo di;
  if ((s = check_device(&di))) return s;
  Plan p;
  make_plan(g, pass, di, &p);
  fill_info(g, p, pass, info);
  return DWCONV_OK;
}

// ---- immutable plan handles
int dwconv_plan_create(const dwconv_desc* d, int pass, int candidate, dwconv_plan_t* out) {
  if (!out) return DWCONV_ERR_NULL_POINTER;
  *out = nullptr;
  Geom g;
  int s = validate(d, &g);
  if (s != DWCONV_OK) return s;
  if (pass < DWCONV_PASS_FWD || pass > DWCONV_PASS_BWD || candidate < -1) return DWCONV_ERR_BAD_DESCRIPTOR;
  DevInfo di;
  if ((s = check_device(&di))) return s;
  auto* h = new (std::nothrow) dwconv_plan_s;
  if (!h) return DWCONV_ERR_CUDA;
  h->g = g;
  h->pass = pass;
  h->candidate = candidate;
  cudaGetDevice(&h->device);
  if (g.N > 0) {
    if (candidate < 0) {
      make_plan_uncached(g, pass, di, &h->p);  // the planner's own pick, whatever dwconv_plan_select installed
    } else {
      int count = 0;
      if ((s = dwconv_plan_candidates(d, pass, 0, nullptr, &count))) { delete h; return s; }
      const PlanKey key = plan_key(g, pass, di);
      std::lock_guard<std::mutex> lk(g_sel_mu);
      auto it = g_candidates.find(key);
      if (it == g_candidates.end() || candidate >= (int)it->second.size()) {
        delete h;
        return DWCONV_ERR_BAD_DESCRIPTOR;
      }
      h->p = it->second[(size_t)candidate];
    }
    if (pass == DWCONV_PASS_BWD) {
      make_plan_uncached(g, DWCONV_PASS_BWD_DATA, di, &h->pd);
      make_plan_uncached(g, DWCONV_PASS_BWD_FILTER, di, &h->pb);
    }
  }
  *out = h;
  return DWCONV_OK;
}

void dwconv_plan_destroy(dwconv_plan_t plan) { delete plan; }

static int plan_ready(dwconv_plan_t h, int pass) {
  if (!h) return DWCONV_ERR_NULL_POINTER;
  if (h->pass != pass) return DWCONV_ERR_BAD_DESCRIPTOR;
  int dev = -1;
  if (cudaGetDevice(&dev) != cudaSuccess) return DWCONV_ERR_CUDA;
  return dev == h->device ? DWCONV_OK : DWCONV_ERR_UNSUPPORTED;
}

int dwconv_plan_describe(dwconv_plan_t h, dwconv_plan_info* info) {
  if (!h || !info) return DWCONV_ERR_NULL_POINTER;
  fill_info(h->g, h->p, h->pass, info);
  if (h->pass == DWCONV_PASS_BWD) info->workspace_bytes = (int64_t)bwd_workspace_bytes(h->p, h->pb);
  if (h->pass == DWCONV_PASS_BWD_FILTER) info->workspace_bytes = (int64_t)bf_workspace_bytes(h->p);
  return DWCONV_OK;
}

size_t dwconv_plan_workspace_bytes(dwconv_plan_t h) {
  if (!h) return 0;
  if (h->pass == DWCONV_PASS_BWD_FILTER) return bf_workspace_bytes(h->p);
  if (h->pass == DWCONV_PASS_BWD) return bwd_workspace_bytes(h->p, h->pb);
  return 0;
}

int dwconv_fwd_plan(dwconv_plan_t h, const void* x, const void* w, void* y, dwconv_stream stream) {
  int s;
  if ((s = plan_ready(h, DWCONV_PASS_FWD)) || (s = ptr_check_fd(h->g, DWCONV_PASS_FWD, x, w, y))) return s;
  return run_fwd(h->g, h->p, x, w, y, reinterpret_cast<cudaStream_t>(stream));
}

int dwconv_bwd_data_plan(dwconv_plan_t h, const void* dy, const void* w, void* dx, dwconv_stream stream) {
  int s;
  if ((s = plan_ready(h, DWCONV_PASS_BWD_DATA)) || (s = ptr_check_fd(h->g, DWCONV_PASS_BWD_DATA, dy, w, dx)))
    return s;
  return run_bwd_data(h->g, h->p, dy, w, dx, reinterpret_cast<cudaStream_t>(stream));
}

int dwconv_bwd_filter_plan(dwconv_plan_t h, const void* x, const void* dy, float* dw, void* workspace,
                           size_t workspace_bytes, dwconv_stream stream) {
  int s;
  if ((s = plan_ready(h, DWCONV_PASS_BWD_FILTER)) || (s = ptr_check_bf(h->g, x, dy, dw))) return s;
  return run_bwd_filter(h->g, h->p, x, dy, dw, workspace, workspace_bytes, reinterpret_cast<cudaStream_t>(stream));
}

int dwconv_bwd_plan(dwconv_plan_t h, const void* x, const void* dy, const void* w, void* dx, float* dw,
                    void* workspace, size_t workspace_bytes, dwconv_stream stream) {
  int s;
  if ((s = plan_ready(h, DWCONV_PASS_BWD)) || (s = ptr_check_bf(h->g, x, dy, dw)) ||
      (s = ptr_check_fd(h->g, DWCONV_PASS_BWD_DATA, dy, w, dx)))
    return s;
  return run_bwd(h->g, h->p, h->pd, h->pb, x, dy, w, dx, dw, workspace, workspace_bytes,
                 reinterpret_cast<cudaStream_t>(stream));
}

}  // extern "C"
