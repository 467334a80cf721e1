// nchw_plan.cu -- host planner and launchers for the NCHW chunk kernels.
//
// For each pass it picks: whole-plane chunks of P planes (or row bands of one
// plane when a plane does not fit), the strip height R (7 when it divides the
// plane height, else 8), the column vector V (4/2/1 by row alignment), the TMA
// ring depth, and for bwd_filter the channel groups x batch slices that fill the
// GPU while keeping every dw serial chain short (dwconv_plan reports max_chain).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <utility>
#include <vector>

#include "nchw_common.cuh"

namespace dwk {
namespace nchw {
namespace {

uint32_t round128(uint64_t b) { return (uint32_t)((b + 127) & ~uint64_t(127)); }

int64_t gcd64(int64_t a, int64_t b) {
  while (b) { int64_t t = a % b; a = b; b = t; }
  return a;
}

int env_int(const char* name, int dflt, int lo, int hi) {
  const char* e = dev_knob(name);
  const int v = e ? std::atoi(e) : dflt;
  return (v >= lo && v <= hi) ? v : dflt;
}

int chunk_budget() {  // target bytes of one chunk (input + output)
  static int kb = env_int("DWCONV_CHUNK_KB", 32, 4, 100);
  return kb * 1024;
}

int num_stages() {
  static int ns = env_int("DWCONV_STAGES", 2, 2, 7);  // bwd_filter keeps 7 empty barriers at smem[72..128)
  return ns;
}

int num_stages_ws() {  // ring depth of the warp-specialised kernels
  static int ns = env_int("DWCONV_WS_STAGES", 3, 2, 8);
  return ns;
}

int occupancy(KernelFn fn, int smem, int threads) {
  static std::mutex mu;
  static KernelFn fns[512] = {};
  {
    std::lock_guard<std::mutex> lk(mu);
    bool seen = false;
    int i = 0;
    for (; i < 512 && fns[i]; ++i)
      if (fns[i] == fn) { seen = true; break; }
    if (!seen && i < 512) {
      int dev = 0, optin = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
      cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, optin);
      fns[i] = fn;
    }
  }
  int blocks = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, fn, threads, smem) != cudaSuccess) return 0;
  return blocks;
}

int ilog2_ceil(int64_t v) {
  int l = 0;
  while ((1ll << l) < v) ++l;
  return l;
}

// Column-vector variant: V = 8 (bf16 3x3), 4, 2 or 1 output columns per thread.  Needs the
// output width divisible by V and the input rows aligned for the S*V vector load.
int pick_vi(int64_t out_w, int64_t in_w, int S, int64_t eb, int K) {
  static const int v8 = env_int("DWCONV_BF16_V8", 1, 0, 1);
  for (int vi = (eb == 2 && K == 3 && v8) ? 3 : 2; vi > 0; --vi) {
    const int64_t V = 1 << vi;
    const int64_t align = std::min<int64_t>(16, S * V * eb);
    if (out_w % V == 0 && (in_w * eb) % align == 0 && (out_w * eb) % std::min<int64_t>(16, V * eb) == 0) return vi;
  }
  return 0;
}

KernelFn kernel_for(int pass, int dtype, int K, int S, int RI, int VI, bool padded, bool pair = false, bool m1 = false) {
  if (pass == DWCONV_PASS_FWD) return fwd_kernel(dtype, K, S, RI, VI, padded, pair);
  if (pass == DWCONV_PASS_BWD_DATA) return bwd_data_kernel(dtype, K, S, RI, VI, padded, pair, m1);
  if (pass == kPassBwdFused) return bwd_fused_kernel(dtype, K, S, RI, VI, padded);
  return bwd_filter_kernel(dtype, K, S, RI, VI, padded);
}

int64_t round16(int64_t b) { return (b + 15) & ~int64_t(15); }

int rows_for(int pass, int K, int S, int RI) {
  if (pass == DWCONV_PASS_FWD) return rows_fwd(K, RI);
  if (pass == DWCONV_PASS_BWD_DATA) return rows_bd(K, S, RI);
  return rows_bf(K, RI);
}

// Finalise the shared-memory layout of a plan (bytes).
void layout_smem(ChunkPlan* p, int64_t W, int64_t eb, uint32_t w_bytes, int ns) {
  p->ns = ns;
  p->zrow_off = 128 + kZPad * 4;  // element 0 of the zero row (bf16 rows use less of it)
  const uint32_t zbytes = round128((uint64_t)(W + 2 * kZPad) * (uint64_t)eb + 64);
  p->w_off = 128 + zbytes;
  p->in0_off = p->w_off + round128(w_bytes);
  p->in2_off = 128 + p->in_bytes + 128;  // 128 B of zero slack on both sides of the input buffer
  p->in_stage = p->in2_off + p->in2_bytes;
  p->out0_off = p->in0_off + (uint32_t)ns * p->in_stage;
  p->out_stage = p->out_bytes;
  p->smem_bytes = (int)(p->out0_off + 2 * p->out_stage);
}

}  // namespace
}  // namespace nchw

using nchw::kThreads;

namespace {

// Resident CTAs per SM for a plan, from shared memory and threads (registers are
// <= 128/thread for every instantiation at 256 threads, so they do not bind first).
int est_ctas_per_sm(int smem_bytes, int threads) {
  const int by_smem = (228 * 1024) / (smem_bytes + 1024);
  const int by_threads = 2048 / threads;
  const int by_regs = 65536 / (96 * threads);  // the kernels use ~60-110 registers per thread
  return std::max(0, std::min(std::min(std::min(by_smem, by_threads), by_regs), 32));
}

// Score of a candidate chunking: fraction of issued thread-strip slots doing real
// work, discounted when chunks are tiny (per-chunk fixed costs) or the SM holds
// too few warps to hide shared-memory latency.
inline int64_t nps_guard(int64_t v) { return v < 1 ? 1 : v; }

double chunk_score(int64_t useful, int64_t slots, int64_t chunk_bytes, int smem, int threads) {
  static const double min_chunk = 1024.0 * nchw::env_int("DWCONV_MIN_CHUNK_KB", 32, 1, 64);
  static const double occ_warps = nchw::env_int("DWCONV_OCC_WARPS", 16, 4, 64);
  const double eff = (double)useful / (double)slots;
  const double size_f = std::min(1.0, std::sqrt((double)chunk_bytes / min_chunk));
  const int ctas = est_ctas_per_sm(smem, threads);
  if (ctas < 1) return -1.0;
  const double warps = (double)ctas * ((threads + 31) / 32);
  const double occ_f = std::min(1.0, warps / occ_warps);
  return eff * size_f * occ_f;
}

}  // namespace

// Candidate list for measurement-driven plan selection: the default pick first,
// then the best-scoring candidate of every distinct chunk shape (planes per
// chunk, bands, band rows, CTA size / threads per plane, ring depth), in score order.
template <class Fin>
static void collect_candidates(std::vector<std::pair<double, ChunkPlan>>& pool, const ChunkPlan* dflt, Fin finalize,
                               std::vector<ChunkPlan>* out, int max_cands) {
  std::stable_sort(pool.begin(), pool.end(),
                   [](const std::pair<double, ChunkPlan>& a, const std::pair<double, ChunkPlan>& b) {
                     return a.first > b.first;
                   });
  auto same = [](const ChunkPlan& a, const ChunkPlan& b) {
    return a.P == b.P && a.nbands == b.nbands && a.band_rows == b.band_rows && a.threads == b.threads &&
           a.tpg == b.tpg && a.ns == b.ns && a.pair == b.pair && a.direct == b.direct;
  };
  out->clear();
  if (dflt) out->push_back(*dflt);
  for (auto& e : pool) {
    if ((int)out->size() >= max_cands) break;
    bool dup = false;
    for (const ChunkPlan& o : *out) dup = dup || same(o, e.second);
    if (dup) continue;
    ChunkPlan c = e.second;
    if (finalize(&c)) out->push_back(c);
  }
}

// Register-direct bwd_filter (direct_bwd_filter.cu) for K = 3, pad 1: a row set
// of L = Wo / V lanes covers an output row, so Wo / V <= 32; rows must be
// aligned for the vector loads.  Work: P = row sets per warp output channels per
// CTA (8 row sets each), ~DWCONV_DBF_TASKS tasks (image x strip) per row set.
static bool plan_direct_bwd_filter(const Geom& g, int num_sms, ChunkPlan* p, int tasks_arg = 0, int max_wo_arg = 0) {
  static const bool on = nchw::env_int("DWCONV_DIRECT_BF", 1, 0, 1) == 1;
  static const int tasks_env = nchw::env_int("DWCONV_DBF_TASKS", 4, 1, 64);
  static const int max_wo_env = nchw::env_int("DWCONV_DBF_MAXWO", 8, 1, 4096);
  const int tasks = tasks_arg > 0 ? tasks_arg : tasks_env;
  const int max_wo = max_wo_arg > 0 ? max_wo_arg : max_wo_env;
  if (!on || g.kh != 3 || g.kw != 3 || g.ph != 1 || g.pw != 1 || g.Wo > max_wo) return false;
  const int S = g.sh;
  if (g.sw != S || (S != 1 && S != 2) || g.W != S * g.Wo) return false;
  const int64_t eb = (g.dtype == DWCONV_F32) ? 4 : 2;
  int V = 0;
  for (int v : {8, 4, 2, 1}) {
    if (v * eb > 16 || g.Wo % v != 0 || g.Wo / v > 32) continue;
    if (S == 2 && v * eb > 8) continue;  // 2*V columns of x per lane: keep the window in registers
    const int64_t nx = std::min<int64_t>(16, (int64_t)S * v * eb);
    if ((g.W * eb) % nx != 0 || (g.Wo * eb) % std::min<int64_t>(16, v * eb) != 0) continue;
    V = v;
    break;
  }
  if (V == 0) return false;
  const int R = (g.Ho % 7 == 0) ? 7 : 8;
  if (!direct::bwd_filter_kernel(g.dtype, S, R, V)) return false;
  const int L = (int)(g.Wo / V), SPW = 32 / L, P = SPW, spc = 8;
  const int Co = (int)(g.C * g.m);
  const int nsb = (int)((g.Ho + R - 1) / R);
  const int64_t N = std::max<int64_t>(g.N, 1);
  const int64_t groups = (Co + P - 1) / P;
  int64_t nps = std::min<int64_t>(N, std::max<int64_t>(1, ((int64_t)tasks * spc + nsb - 1) / nsb));
  nps = std::max<int64_t>(nps, (N + 127) / 128);
  while (nps > 1 && groups * ((N + nps - 1) / nps) < 2 * num_sms && (nps + 1) / 2 >= (N + 127) / 128) nps = (nps + 1) / 2;
  const int64_t nsl = (N + nps - 1) / nps;
  *p = ChunkPlan{};
  p->direct = true;
  p->threads = 256;
  p->smem_bytes = 0;
  p->R = R; p->V = V; p->ri = (R == 7) ? 0 : 1;
  p->P = P; p->nbands = 1; p->band_rows = (int)g.Ho; p->nsb = nsb; p->ncg = L;
  p->dL = L; p->dSPW = SPW; p->dspc = spc;
  p->groups = (int)groups; p->nslices = (int)nsl; p->n_per_slice = (int)nps; p->tpg = L;
  p->grid = (int)(groups * nsl);
  p->nchunks = p->grid;
  const bool packed = (S == 1 && V % 2 == 0);
  const int64_t per_task = (int64_t)R * (packed ? V / 2 : V) + (packed ? 1 : 0);
  const int64_t task_sum = (nps * nsb + spc - 1) / spc;
  p->max_chain = (int)(per_task + task_sum + L + spc + 2 * nchw::ilog2_ceil(nsl) + 1);
  p->ws_bytes = two_level_ws_bytes(groups, nsl, Co);
  return p->max_chain <= 160 && groups * nsl < (int64_t)1 << 31;
}

// Streaming bf16 register-direct bwd_filter (sdbf_kernel) for K = 3, pad 1 on
// planes whose rows split into L = Wo / V <= 32 lanes (MobileNet 112/56/28
// columns): task = (image, band of BR dy rows); nps images per batch slice.
static bool plan_stream_bwd_filter(const Geom& g, int num_sms, ChunkPlan* p, int V, int BR, int tps_arg) {
  if (g.dtype != DWCONV_BF16 || g.kh != 3 || g.kw != 3 || g.ph != 1 || g.pw != 1) return false;
  const int S = g.sh;
  if (g.sw != S || (S != 1 && S != 2) || g.W != S * g.Wo || g.Wo % V != 0 || g.Wo / V > 32) return false;
  if (!direct::bwd_filter_stream_kernel(g.dtype, S, BR, V)) return false;
  const int L = (int)(g.Wo / V), SPW = 32 / L, spc = 8, P = SPW;
  const int Co = (int)(g.C * g.m);
  const int nsb = (int)((g.Ho + BR - 1) / BR);
  const int64_t N = std::max<int64_t>(g.N, 1);
  const int64_t groups = (Co + P - 1) / P;
  const int64_t ntot = N * nsb;  // (image, band) tasks per channel, sliced into runs of tps
  const int64_t nps = std::min<int64_t>(ntot, std::max(1, tps_arg));
  const int64_t nsl = (ntot + nps - 1) / nps;
  *p = ChunkPlan{};
  p->direct = true;
  p->dstream = BR;
  p->threads = 256;
  p->smem_bytes = 0;
  p->R = BR; p->V = V; p->ri = 0;
  p->P = P; p->nbands = 1; p->band_rows = (int)g.Ho; p->nsb = nsb; p->ncg = L;
  p->dL = L; p->dSPW = SPW; p->dspc = spc;
  p->groups = (int)groups; p->nslices = (int)nsl; p->n_per_slice = (int)nps; p->tpg = L;
  p->grid = (int)(groups * nsl);
  p->nchunks = p->grid;
  const int64_t kmax = (nps + spc - 1) / spc;
  p->max_chain = (int)(BR * V / 2 + 1 + kmax + L + spc + 2 * nchw::ilog2_ceil(nsl) + 1);
  p->ws_bytes = two_level_ws_bytes(groups, nsl, Co);
  return p->max_chain <= 160 && groups * nsl < (int64_t)1 << 31;
}

// Tasks per slice for the streaming variant: `res` resident CTAs per SM; picks the
// slicing whose busiest SM (ceil(grid / SMs) CTAs of kmax set rounds each) is
// closest to the even share, preferring <= `waves` CTAs per resident slot.
static int stream_tps(const Geom& g, int num_sms, int V, int BR, int res, double waves) {
  const int L = (int)(g.Wo / V);
  if (L < 1 || L > 32) return 1;
  const int P = 32 / L, spc = 8;
  const int64_t groups = (g.C * g.m + P - 1) / P;
  const int64_t ntot = std::max<int64_t>(g.N, 1) * ((g.Ho + BR - 1) / BR);
  const double ideal = (double)groups * ntot / ((double)num_sms * spc);  // set rounds per SM, perfectly spread
  double best = -1.0;
  int64_t best_tps = ntot;
  const int64_t cap = std::max<int64_t>(1, (int64_t)(waves * res * num_sms));
  for (int64_t nsl = 1; nsl <= std::min<int64_t>(ntot, 128); ++nsl) {
    const int64_t tps = (ntot + nsl - 1) / nsl;
    const int64_t nsl2 = (ntot + tps - 1) / tps;
    const int64_t grid = groups * nsl2;
    if (grid > cap) break;
    const int64_t kmax = (tps + spc - 1) / spc;
    const double t = (double)((grid + num_sms - 1) / num_sms) * kmax;
    const double sc = ideal / t;
    if (sc > best + 1e-9) { best = sc; best_tps = tps; }
  }
  return (int)best_tps;
}

bool plan_nchw(const Geom& g, int pass, int num_sms, int max_smem_optin, ChunkPlan* p,
               std::vector<ChunkPlan>* cands, int max_cands) {
  using namespace nchw;
  // cands != nullptr: also return up to max_cands distinct chunk shapes, best
  // score first, for measurement-driven selection (dwconv_plan_candidates);
  // the search then spans chunk budgets up to 96 KB and both chunk modes.
  std::vector<std::pair<double, ChunkPlan>> pool;
  auto keep = [&](double sc, const ChunkPlan& c) { if (cands) pool.emplace_back(sc, c); };
  if (g.layout != DWCONV_NCHW) return false;
  const int K = g.kh;
  if (g.kw != K || (K != 3 && K != 5 && K != 7)) return false;
  const int S = g.sh;
  if (g.sw != S || (S != 1 && S != 2)) return false;
  if (g.ph != (K - 1) / 2 || g.pw != (K - 1) / 2) return false;
  if (g.m < 1 || g.m > 8) return false;
  if (g.H > 8192 || g.W > 8192 || g.Ho * g.Wo * (int64_t)g.m > (1 << 24)) return false;
  if (g.N * g.C >= (int64_t)1 << 31) return false;  // plane and chunk indices use 32-bit magic division
  // strided windows must stay inside the row (odd W with S = 2 goes to the generic path)
  if (pass != DWCONV_PASS_BWD_DATA && S * g.Wo > g.W) return false;
  *p = ChunkPlan{};
  const int64_t eb = (g.dtype == DWCONV_F32) ? 4 : 2;
  const int budget = cands ? 96 * 1024 : chunk_budget();
  const int64_t budget_max = std::max<int64_t>(budget, 48 * 1024);
  const int64_t Q = g.N * g.C;
  const int m = g.m;
  const int KK = K * K;
  const int ns = num_stages();
  const int64_t x_plane = g.H * g.W * eb;
  const int64_t y_plane = (int64_t)m * g.Ho * g.Wo * eb;  // the m output planes of one input plane
  static const int kT[] = {256, 224, 192, 160, 128, 96, 64};

  if (pass == DWCONV_PASS_FWD || pass == DWCONV_PASS_BWD_DATA) {
    const bool fwd = pass == DWCONV_PASS_FWD;
    const int64_t in_plane = fwd ? x_plane : y_plane;
    const int64_t out_plane = fwd ? y_plane : x_plane;
    const int64_t wpp = (int64_t)m * KK * 4;  // staged weights per input plane
    const int64_t per = in_plane + out_plane;
    const int PADr = (K - 1) / 2;
    const int64_t Win = fwd ? g.W : g.Wo, Hin = fwd ? g.H : g.Ho;
    const int64_t npi = fwd ? 1 : m;  // staged input planes per chunk plane
    const int64_t zbe_b = round16(PADr * Win * eb);
    // padded staging needs 16-B aligned planes (full mode) or rows (band mode)
    const bool pad_full = (Hin * Win * eb) % 16 == 0;
    const bool pad_band = (Win * eb) % 16 == 0;
    // bf16 3x3 stride-2 bwd_data with m = 1 runs the streaming polyphase strips (nchw_bwd_data.cu)
    int bd_stream_vi = 0;
    if (!fwd && S == 2 && K == 3 && m == 1 && g.dtype == DWCONV_BF16 && nchw::kBf16Interleave) {
      for (int vi = 3; vi > 0 && !bd_stream_vi; --vi) {
        const int64_t v = (int64_t)1 << vi;
        if (g.W % (2 * v) == 0 && g.Wo % v == 0 && (vi < 3 || (g.Wo * eb) % 16 == 0)) bd_stream_vi = vi;
      }
    }
    const bool bd_stream = bd_stream_vi > 0;
    const int out_rows_total = fwd ? (int)g.Ho : (int)g.H;
    p->ri = (out_rows_total % rows_for(pass, K, S, 0) == 0) ? 0 : 1;
    p->R = rows_for(pass, K, S, p->ri);
    if (fwd) p->vi = pick_vi(g.Wo, g.W, S, eb, K);
    else if (S == 1) p->vi = pick_vi(g.W, g.Wo, 1, eb, K);
    else {  // stride-2 dx tiles of 2V columns: rows must split into whole, aligned tiles
      p->vi = 0;
      static const int wide = env_int("DWCONV_BD_WIDE", 1, 0, 2);  // 1: 4-column tiles (measured best)
      for (int vi = std::min(wide, K == 3 ? 2 : 1); vi > 0; --vi) {
        const int64_t tw = (int64_t)S << vi;
        if (g.W % tw == 0 && (g.W * eb) % std::min<int64_t>(16, tw * eb) == 0) { p->vi = vi; break; }
      }
      if (bd_stream) p->vi = bd_stream_vi;  // bf16 3x3 m = 1: streaming strips of 2V dx columns
    }
    p->V = 1 << p->vi;
    p->ncg = fwd ? (int)(g.Wo / p->V) : (S == 1 ? (int)(g.W / p->V) : (int)((g.W + S * p->V - 1) / (S * p->V)));
    const int R = p->R;
    const int nsb_full = (out_rows_total + R - 1) / R;
    const int64_t tpp = (int64_t)nsb_full * p->ncg;  // thread strips per plane
    const int64_t a1 = 16 / gcd64(in_plane, 16), a2 = 16 / gcd64(out_plane, 16);
    const int64_t al = a1 / gcd64(a1, a2) * a2;  // planes per chunk keeping bulk copies 16-B aligned
    auto in_rows = [&](int br) -> int64_t {
      if (fwd) return std::min<int64_t>(g.H, (int64_t)(br - 1) * S + K);
      return std::min<int64_t>(g.Ho, (br + K - 1 + S - 1) / S + 1);
    };
    auto band_bytes = [&](int br, int64_t* inb, int64_t* outb) {
      if (fwd) { *inb = in_rows(br) * g.W * eb; *outb = (int64_t)m * br * g.Wo * eb; }
      else { *inb = (int64_t)m * in_rows(br) * g.Wo * eb; *outb = (int64_t)br * g.W * eb; }
    };
    double best = -1.0;
    ChunkPlan bestp = *p;
    const bool ws_design = true;  // warp-specialised: producer warp + direct stores
    // Score a candidate: thread-strip slots used inside a chunk x chunks spread
    // over the resident CTAs (tail) x pipeline fill (the first chunk of every CTA
    // is exposed latency) x occupancy x a small-chunk penalty.
    auto consider = [&](int T, int P, int nbands, int band_rows, int64_t tiles, int64_t nch, int64_t useful_total,
                        int64_t inb, int64_t outb, int64_t wb) {
      if (!ws_design && (int64_t)P * m * KK > 4 * T) return;  // bwd_data prefetches <= 4 weights per thread
      // tuning aid: DWCONV_FD_FORCE="T,P,band_rows" (band_rows 0 = whole planes) pins the chunk shape
      static const int* force = []() -> const int* {
        static int f[3];
        const char* e = dev_knob("DWCONV_FD_FORCE");
        if (!e || sscanf(e, "%d,%d,%d", &f[0], &f[1], &f[2]) != 3) return nullptr;
        return f;
      }();
      if (force && (T != force[0] || P != force[1] || (nbands == 1 ? 0 : band_rows) != force[2])) return;
      ChunkPlan c = *p;
      if (ws_design) { outb = 0; c.in2_bytes = round128(wb / 2 + 32); wb = 0; }  // per-stage weight table (+ bulk-copy alignment slack)
      c.threads = T + (ws_design ? 32 : 0); c.P = P; c.nbands = nbands; c.band_rows = band_rows;
      c.in_bytes = round128(inb); c.out_bytes = round128(outb);
      const int nst = ws_design ? num_stages_ws() : ns;
      layout_smem(&c, std::max(g.W, g.Wo), eb, (uint32_t)wb, nst);
      if (c.smem_bytes > max_smem_optin) layout_smem(&c, std::max(g.W, g.Wo), eb, (uint32_t)wb, 2);
      if (c.smem_bytes > max_smem_optin) return;
      KernelFn kf = kernel_for(pass, g.dtype, K, S, c.ri, c.vi, c.padded, c.pair, g.m == 1);
      const int ctas = kf ? occupancy(kf, c.smem_bytes, c.threads) : 0;  // resident CTAs per SM
      if (ctas < 1) return;
      const int64_t grid = std::min<int64_t>(nch, (int64_t)ctas * num_sms);
      const int64_t rounds_c = (nch + grid - 1) / grid;
      const int64_t rounds_t = (tiles + T - 1) / T;
      const double eff = (double)useful_total / (double)(grid * rounds_c * rounds_t * ((T + 31) / 32) * 32);
      const double pipe = (double)rounds_c / (rounds_c + 1.0);
      const double ctas_eff = (double)std::min<int64_t>(ctas, (nch + num_sms - 1) / num_sms);
      const double warps = ctas_eff * ((c.threads + 31) / 32);
      const double occ_f = std::min(1.0, warps / 16.0);
      const double size_f = std::min(1.0, std::sqrt((double)(inb + outb) / (4.0 * 1024)));
      // bytes in flight per SM: every resident CTA keeps its ring of input stages loading
      static const double fill_b = 1024.0 * env_int("DWCONV_FILL_KB", 160, 8, 228);
      const double fill_f = std::min(1.0, ctas_eff * c.ns * (double)c.in_bytes / fill_b);
      // SMs that get a chunk at all: tiny planes (4x4 .. 8x8, the width/resolution variants of
      // configs[2]) otherwise pick a few huge chunks (measured: 43 CTAs, 44 us for a 2 MB pass)
      const double sm_f = std::min(1.0, (double)nch / num_sms);
      const double sc = eff * pipe * occ_f * size_f * fill_f * sm_f;
      keep(sc, c);
      if (sc > best) { best = sc; bestp = c; }
    };
    if (per <= budget_max) {  // whole-plane chunks
      const int64_t pmax = std::min<int64_t>(Q, budget_max / per);
      for (int T : kT) {
        for (int64_t P = al; P <= std::max<int64_t>(pmax, al); P += al) {
          if (P > Q) break;
          // bf16 fwd, whole planes, m = 1: plane-pair strips (half the tiles, each twice the work)
          static const bool pair_env = env_int("DWCONV_BF16_PAIR", 1, 0, 1) == 1;
          p->pair = pair_env && !bd_stream && g.dtype == DWCONV_BF16 && K == 3 && m == 1 && P >= 2 &&
                    ((S * p->V) % 2 == 0) && kernel_for(pass, g.dtype, K, S, p->ri, p->vi, pad_full, true) != nullptr;
          const int64_t tiles = p->pair ? (P + 1) / 2 * tpp : P * tpp;
          const int64_t useful = p->pair ? (Q + 1) / 2 * tpp : Q * tpp;
          const int64_t nch = (Q + P - 1) / P;
          int64_t inb = P * in_plane;
          if (pad_full)  // zero rows above each plane, below the last, and strip overrun
            inb = P * npi * (zbe_b + round16(Hin * Win * eb)) + zbe_b + (int64_t)R * S * Win * eb;
          p->padded = pad_full;
          p->zbe = (int)(zbe_b / eb);
          p->pitch = (int)((zbe_b + round16(Hin * Win * eb)) / eb);
          consider(T, (int)P, 1, out_rows_total, tiles, nch, useful, inb, P * out_plane, 2 * P * wpp);
        }
      }
    }
    if (best < 0.0 || per > budget || cands) {  // row bands of one plane
      for (int nsb_b = 1; nsb_b <= nsb_full; ++nsb_b) {
        const int br = nsb_b * R;
        int64_t inb, outb;
        band_bytes(br, &inb, &outb);
        if (inb + outb > budget_max) break;
        const int nb = (nsb_full + nsb_b - 1) / nsb_b;
        for (int T : kT) {
          p->pair = false;
          const int64_t tiles = (int64_t)nsb_b * p->ncg;
          if (pad_band) {
            const int64_t rows_buf = (fwd ? (int64_t)(br - 1) * S + K : (br + K - 1 + S - 1) / S + 1) + PADr;
            inb = npi * (zbe_b + round16(rows_buf * Win * eb)) + zbe_b;
          }
          p->padded = pad_band;
          p->zbe = (int)(zbe_b / eb);
          if (pad_band) {
            const int64_t rows_buf = (fwd ? (int64_t)(br - 1) * S + K : (br + K - 1 + S - 1) / S + 1) + PADr;
            p->pitch = (int)((zbe_b + round16(rows_buf * Win * eb)) / eb);
          }
          consider(T, 1, nb, br, tiles, Q * nb, Q * tpp, inb, outb, 2 * wpp);
        }
      }
    }
    if (best < 0.0) return false;
    auto finalize = [&](ChunkPlan* c) -> bool {
      c->nchunks = (c->nbands == 1) ? (Q + c->P - 1) / c->P : Q * c->nbands;
      if (c->nchunks >= ((int64_t)1 << 31)) return false;
      c->nsb = (c->band_rows + R - 1) / R;
      KernelFn fn = kernel_for(pass, g.dtype, K, S, c->ri, c->vi, c->padded, c->pair, g.m == 1);
      if (!fn) return false;
      const int occ = occupancy(fn, c->smem_bytes, c->threads);
      if (occ < 1) return false;
      c->grid = (int)std::min<int64_t>(c->nchunks, (int64_t)occ * num_sms);
      return true;
    };
    *p = bestp;
    if (!finalize(p)) return false;
    if (cands) {
      collect_candidates(pool, p, finalize, cands, max_cands);
      if (!fwd && S == 1 && m == 1) {
        // stride-1 bwd_data is the forward stencil over dy (same staged shapes): the forward's
        // leading shapes join the list, behind the default (the score-ranked list is capped
        // and ranks the two passes' shapes differently; measured: bf16 dw2 fwd's 224-thread
        // whole-plane shape is absent from the bwd_data list)
        std::vector<ChunkPlan> fc;
        ChunkPlan fd;
        if (plan_nchw(g, DWCONV_PASS_FWD, num_sms, max_smem_optin, &fd, &fc, 12)) {
          std::vector<ChunkPlan> add;
          for (ChunkPlan c : fc) {
            if (c.pair || !finalize(&c)) continue;
            bool dup = false;
            for (const ChunkPlan& o : *cands)
              dup = dup || (o.P == c.P && o.nbands == c.nbands && o.band_rows == c.band_rows && o.threads == c.threads &&
                            o.ns == c.ns && o.pair == c.pair);
            if (!dup) add.push_back(c);
          }
          cands->insert(cands->begin() + std::min<size_t>(1, cands->size()), add.begin(), add.end());
          if ((int)cands->size() > max_cands) cands->resize((size_t)max_cands);
        }
      }
    }
    return true;
  }

  // ---------------- bwd_filter (and the fused backward: + dx from the same staged dy)
  const bool fused = pass == kPassBwdFused;
  if (fused && (g.m != 1 || S != 1 || K != 3)) return false;
  if (!fused && !cands && plan_direct_bwd_filter(g, num_sms, p)) return true;
  const int64_t per = x_plane + y_plane;
  p->ri = (g.Ho % rows_bf(K, 0) == 0) ? 0 : 1;
  p->R = rows_bf(K, p->ri);
  p->vi = pick_vi(g.Wo, g.W, S, eb, K);
  p->V = 1 << p->vi;
  p->ncg = (int)(g.Wo / p->V);
  const int R = p->R;
  const int nsb_full = (int)((g.Ho + R - 1) / R);
  double best = -1.0;
  ChunkPlan bestp = *p;
  const int PADr = (K - 1) / 2;
  const int64_t zbe_b = round16(PADr * g.W * eb);
  const bool pad_full = (g.H * g.W * eb) % 16 == 0;
  const bool pad_band = (g.W * eb) % 16 == 0;
  // tuning aid: DWCONV_BF_FORCE="P,tpg,nsb" pins the chunk shape (nsb = strip rows per band, 0 = whole planes)
  static const int* bf_force = []() -> const int* {
    static int f[3];
    const char* e = dev_knob("DWCONV_BF_FORCE");
    if (!e || sscanf(e, "%d,%d,%d", &f[0], &f[1], &f[2]) != 3) return nullptr;
    return f;
  }();
  auto consider = [&](int P, int tpg, int nb, int br, int64_t xb, int64_t dyb) {
    if (bf_force && (P != bf_force[0] || tpg != bf_force[1] || (nb == 1 ? 0 : (br + R - 1) / R) != bf_force[2])) return;
    if (nb == 1 ? pad_full : pad_band) {  // padded x staging
      const int64_t rows_buf = (nb == 1) ? g.H : (int64_t)(br - 1) * S + K + PADr;
      const int64_t pitch_b = zbe_b + round16(rows_buf * g.W * eb);
      xb = P * pitch_b + zbe_b + (int64_t)R * S * g.W * eb;
      p->padded = true;
      p->pitch = (int)(pitch_b / eb);
      p->zbe = (int)(zbe_b / eb);
    } else {
      p->padded = false;
    }
    const int T = P * m * tpg;
    if (T > kThreads || T < 64 || T % 32 != 0) return;  // whole warps: the reduction shuffles full warps
    ChunkPlan c = *p;
    c.threads = T + 32; c.P = P; c.tpg = tpg; c.nbands = nb; c.band_rows = br;  // + the producer warp
    c.in_bytes = round128(xb); c.in2_bytes = round128(dyb); c.out_bytes = 0;
    layout_smem(&c, g.W, eb, 0, ns);
    if (c.smem_bytes > max_smem_optin) layout_smem(&c, g.W, eb, 0, 2);
    // the final reduction parks T * KK floats in the input stages
    if ((uint32_t)c.ns * c.in_stage < (uint32_t)(T * KK * 4)) {
      c.in2_bytes += round128(T * KK * 4);
      layout_smem(&c, g.W, eb, 0, c.ns);
    }
    if (c.smem_bytes > max_smem_optin) return;
    const int nsb_b = (br + R - 1) / R;
    const int64_t strips = (int64_t)nsb_b * p->ncg;  // per plane per chunk
    const int64_t rounds = (strips + tpg - 1) / tpg;
    const int64_t useful = (int64_t)nsb_full * p->ncg * P * m;
    const int64_t slots = (int64_t)nb * rounds * ((T + 31) / 32) * 32;
    // fewer channel groups than ~SMs would need many batch slices: discount
    const int64_t groups = (g.C + P - 1) / P;
    const double grp_f = std::min(1.0, (double)groups * std::min<int64_t>(g.N, 32) / (2.0 * num_sms));
    const double sc = chunk_score(useful, slots, xb + dyb, c.smem_bytes, T) * grp_f;
    keep(sc, c);
    if (sc > best) { best = sc; bestp = c; }
  };
  if (per <= budget_max) {
    const int64_t a1 = 16 / gcd64(x_plane, 16), a2 = 16 / gcd64(y_plane, 16);
    const int64_t al = a1 / gcd64(a1, a2) * a2;
    for (int P = 1; P * m <= kThreads && P <= g.C && P * per <= budget_max; ++P) {
      if (P % al != 0 && P != g.C) continue;
      for (int tpg = 1; P * m * tpg <= kThreads; ++tpg) consider(P, tpg, 1, (int)g.Ho, P * x_plane, P * y_plane);
    }
  }
  if (best < 0.0 || per > budget || cands) {
    for (int nsb_b = 1; nsb_b <= nsb_full; ++nsb_b) {
      const int br = nsb_b * R;
      const int64_t xb = std::min<int64_t>(g.H, (int64_t)(br - 1) * S + K) * g.W * eb;
      const int64_t dyb = (int64_t)m * std::min<int64_t>(g.Ho, br + (fused ? 2 * PADr : 0)) * g.Wo * eb;
      if (xb + dyb > budget_max) break;
      const int nb = (nsb_full + nsb_b - 1) / nsb_b;
      for (int P = 1; P * m <= kThreads && P <= g.C && P * (xb + dyb) <= budget_max; ++P)  // P planes per band chunk
        for (int tpg = 1; P * m * tpg <= kThreads; ++tpg) consider(P, tpg, nb, br, P * xb, P * dyb);
    }
  }
  if (best < 0.0) return false;
  auto finalize = [&](ChunkPlan* c) -> bool {
    c->nsb = (c->band_rows + R - 1) / R;
    c->groups = (int)((g.C + c->P - 1) / c->P);
    KernelFn fn = kernel_for(pass, g.dtype, K, S, c->ri, c->vi, c->padded);
    if (!fn) return false;
    const int occ = occupancy(fn, c->smem_bytes, c->threads);
    if (occ < 1) return false;
    const int nb = c->nbands;
    // batch slices: ~one wave of CTAs, >= 2 chunks per CTA when the batch allows,
    // <= 32 chunks per CTA (running-sum chain) and <= 128 slices.
    const int64_t N = std::max<int64_t>(g.N, 1);
    int64_t nsl = ((int64_t)num_sms * occ + c->groups - 1) / c->groups;  // ~one wave
    nsl = std::min<int64_t>(nsl, std::max<int64_t>(1, N * nb / 2));
    nsl = std::max<int64_t>(nsl, (N * nb + 31) / 32);
    nsl = std::min<int64_t>(nsl, std::min<int64_t>(N, 128));
    nsl = std::max<int64_t>(nsl, 1);
    int64_t nps = (N + nsl - 1) / nsl;
    nsl = (N + nps - 1) / nps;
    c->nslices = (int)nsl;
    c->n_per_slice = (int)nps;
    c->grid = (int)(c->groups * nsl);
    c->nchunks = (int64_t)c->grid;
    const bool packed = (S == 1 && c->V % 2 == 0);
    const int64_t strips_per_thread = ((int64_t)c->nsb * c->ncg + c->tpg - 1) / c->tpg;
    const int64_t per_chunk = strips_per_thread * R * (packed ? c->V / 2 : c->V) + (packed ? 1 : 0);
    const int64_t thread_sum = (c->tpg <= 32) ? c->tpg : (c->tpg + 31) / 32 + 5;
    c->max_chain = (int)(per_chunk + nps * nb + thread_sum + 2 * ilog2_ceil(nsl) + 1);
    c->ws_bytes = two_level_ws_bytes(c->groups, nsl, g.C * m, KK);
    return nsl <= 128 && c->max_chain <= 160;
  };
  *p = bestp;
  const bool ok = finalize(p);
  if (cands) {
    collect_candidates(pool, ok ? p : nullptr, finalize, cands, max_cands);
    // fewer batch slices for the leading shapes: on small tensors (the width/resolution
    // variants of configs[2]: 1-2 MB per pass) one wave of CTAs leaves each with a few KB
    // and the cross-slice finalize dominates; the measured selection decides
    const size_t lead = std::min<size_t>(cands->size(), 4);
    std::vector<ChunkPlan> var_bal, var_div;  // balanced slice counts go right behind the default
    for (size_t ci = 0; ci < lead; ++ci) {
      // slice counts: fewer (1/2, 1/4, 1/8), and the count whose busiest SM (ceil(grid / SMs)
      // CTAs of nps images) comes closest to the even share within one / two waves of
      // resident CTAs (a grid just past a wave leaves most SMs idle while the last CTAs run)
      for (int div : {-1, -2, 2, 4, 8}) {
        ChunkPlan v = (*cands)[ci];
        if (v.direct || v.small) continue;
        if (div > 0 && v.nslices < 2 * div) continue;
        const int64_t N = std::max<int64_t>(g.N, 1);
        int64_t nsl = div > 0 ? v.nslices / div : v.nslices;
        if (div < 0) {
          KernelFn fn = kernel_for(pass, g.dtype, K, S, v.ri, v.vi, v.padded);
          const int occ = fn ? occupancy(fn, v.smem_bytes, v.threads) : 0;
          if (occ < 1) continue;
          const int64_t lo = std::max<int64_t>(1, (N * v.nbands + 31) / 32), hi = std::min<int64_t>(N, 128);
          const double ideal = (double)v.groups * N / num_sms;
          double best_sc = -1.0;
          for (int64_t t = lo; t <= hi; ++t) {
            const int64_t np_ = (N + t - 1) / t, ns_ = (N + np_ - 1) / np_;
            const int64_t grid = (int64_t)v.groups * ns_;
            if (grid > (int64_t)(-div) * occ * num_sms) break;
            const double sc = ideal / ((double)((grid + num_sms - 1) / num_sms) * np_);
            if (sc > best_sc + 1e-9) { best_sc = sc; nsl = ns_; }
          }
          if (nsl == v.nslices) continue;
        }
        int64_t nps = (N + nsl - 1) / nps_guard(nsl);
        nsl = (N + nps - 1) / nps;
        if (nps * v.nbands > 32) continue;  // running-sum chain, as finalize()
        const int64_t old_nps = v.n_per_slice, old_nsl = v.nslices;
        v.nslices = (int)nsl;
        v.n_per_slice = (int)nps;
        v.grid = (int)(v.groups * nsl);
        v.nchunks = v.grid;
        v.max_chain = v.max_chain - (int)(old_nps * v.nbands) + (int)(nps * v.nbands) -
                      2 * ilog2_ceil(old_nsl) + 2 * ilog2_ceil(nsl);
        v.ws_bytes = two_level_ws_bytes(v.groups, nsl, g.C * m, KK);
        if (v.max_chain > 160) continue;
        bool dup = false;
        auto same_v = [&](const ChunkPlan& o) {
          return o.P == v.P && o.tpg == v.tpg && o.nbands == v.nbands && o.band_rows == v.band_rows &&
                 o.nslices == v.nslices && o.threads == v.threads && o.direct == v.direct;
        };
        for (const ChunkPlan& o : *cands) dup = dup || same_v(o);
        for (const ChunkPlan& o : var_bal) dup = dup || same_v(o);
        for (const ChunkPlan& o : var_div) dup = dup || same_v(o);
        if (!dup) (div < 0 ? var_bal : var_div).push_back(v);
      }
    }
    const size_t at = std::min<size_t>(1, cands->size());
    cands->insert(cands->begin() + at, var_bal.begin(), var_bal.end());
    cands->insert(cands->end(), var_div.begin(), var_div.end());
    if (!fused) {  // register-direct variants (no smem staging) compete too
      for (int tasks : {2, 4}) {
        ChunkPlan d;
        if (plan_direct_bwd_filter(g, num_sms, &d, tasks, 4096)) cands->push_back(d);
      }
      // bf16 streaming variants right behind the default (the list is capped)
      std::vector<ChunkPlan> sv;
      for (int V : {8, 4})
        for (int BR : {16, 8})
          for (double waves : {1.0, 3.0}) {
            ChunkPlan d;
            if (plan_stream_bwd_filter(g, num_sms, &d, V, BR, stream_tps(g, num_sms, V, BR, 2, waves))) {
              bool dup = false;
              for (const ChunkPlan& o : sv) dup = dup || (o.V == d.V && o.dstream == d.dstream && o.nslices == d.nslices);
              if (!dup) sv.push_back(d);
            }
          }
      cands->insert(cands->begin() + std::min<size_t>(1, cands->size()), sv.begin(), sv.end());
      ChunkPlan d0;  // the default planner's pick leads the list
      if (plan_direct_bwd_filter(g, num_sms, &d0)) cands->insert(cands->begin(), d0);
    }
    if ((int)cands->size() > max_cands) cands->resize((size_t)max_cands);
  }
  return ok;
}

// Launch with programmatic dependent launch allowed (the kernels call
// griddepcontrol.wait before touching global memory), so a kernel's launch and
// prologue overlap the tail of the previous kernel on the stream.
static cudaError_t launch(nchw::KernelFn fn, const ChunkPlan& p, cudaStream_t st, const nchw::NArgs& a) {
  static const bool pdl = nchw::env_int("DWCONV_PDL", 1, 0, 1) == 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)p.grid);
  cfg.blockDim = dim3((unsigned)p.threads);
  cfg.dynamicSmemBytes = (size_t)p.smem_bytes;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, fn, a);
}

// Weight rows may be staged by bulk copy (16-B aligned base and total size).
static int weights_bulk_ok(const Geom& g, const void* w) {
  const int64_t eb = (g.dtype == DWCONV_F32) ? 4 : 2;
  const int64_t bytes = g.C * g.m * g.kh * g.kw * eb;
  return ((reinterpret_cast<uintptr_t>(w) & 15u) == 0 && bytes % 16 == 0) ? 1 : 0;
}

static nchw::NArgs base_args(const Geom& g, const ChunkPlan& p) {
  nchw::NArgs a{};
  a.N = g.N; a.C = g.C; a.Q = g.N * g.C;
  a.m = g.m; a.Co = (int)(g.C * g.m);
  a.H = (int)g.H; a.W = (int)g.W; a.Ho = (int)g.Ho; a.Wo = (int)g.Wo;
  a.P = p.P; a.nbands = p.nbands; a.BR = p.band_rows;
  a.nsb = p.nsb;
  a.nchunks = p.nchunks;
  a.zrow_off = p.zrow_off; a.w_off = p.w_off;
  a.in0_off = p.in0_off; a.in_stage = p.in_stage; a.in_bytes = p.in_bytes;
  a.in2_off = p.in2_off; a.in2_bytes = p.in2_bytes;
  a.out0_off = p.out0_off; a.out_stage = p.out_stage; a.out_bytes = p.out_bytes;
  a.ns = p.ns;
  a.pitch = p.pitch; a.zbe = p.zbe;
  a.groups = p.groups; a.nslices = p.nslices; a.nps = p.n_per_slice; a.tpg = p.tpg;
  a.div_ncg = make_fastdiv((uint32_t)p.ncg);
  a.div_nsb = make_fastdiv((uint32_t)p.nsb);
  a.div_m = make_fastdiv((uint32_t)g.m);
  a.div_co = make_fastdiv((uint32_t)a.Co);
  a.div_c = make_fastdiv((uint32_t)g.C);
  static const int early = nchw::env_int("DWCONV_EARLY_PDL", 1, 0, 1);
  a.early_pdl = early;
  a.div_nb = make_fastdiv((uint32_t)std::max(1, p.nbands));
  return a;
}

// A ChunkPlan that runs the small-plane warp-task kernels (nchw_small.cu).
bool small_chunk_plan(const Geom& g, int pass, int num_sms, int smem_optin, ChunkPlan* p, int warps, int stages,
                      int slices, bool pair) {
  SmallPlan sp;
  if (!plan_nchw_small(g, pass, num_sms, smem_optin, &sp, warps, stages, slices, pair)) return false;
  *p = ChunkPlan{};
  p->small = true;
  p->sp = sp;
  p->threads = 32 * sp.warps;
  p->grid = sp.grid;
  p->smem_bytes = sp.smem;
  p->P = sp.pair ? 8 : 4;
  p->nbands = 1;
  p->band_rows = (int)g.H;
  p->ns = sp.ns;
  p->nchunks = (pass >= DWCONV_PASS_BWD_FILTER) ? (int64_t)sp.groups * sp.nslices : sp.ntasks;
  p->groups = sp.groups;
  p->nslices = sp.nslices;
  p->n_per_slice = sp.nps;
  p->max_chain = sp.max_chain;
  p->ws_bytes = sp.ws_bytes;
  return true;
}

bool lane_chunk_plan(const Geom& g, int pass, int num_sms, int smem_optin, ChunkPlan* p, int warps, int stages,
                     int slices) {
  SmallPlan sp;
  if (!plan_nchw_lane(g, pass, num_sms, smem_optin, &sp, warps, stages, slices)) return false;
  *p = ChunkPlan{};
  p->small = true;
  p->sp = sp;
  p->threads = 32 * sp.warps;
  p->grid = sp.grid;
  p->smem_bytes = sp.smem;
  p->P = 32;
  p->nbands = 1;
  p->band_rows = (int)g.H;
  p->ns = sp.ns;
  p->nchunks = (pass >= DWCONV_PASS_BWD_FILTER) ? (int64_t)sp.groups * sp.nslices : sp.ntasks;
  p->groups = sp.groups;
  p->nslices = sp.nslices;
  p->n_per_slice = sp.nps;
  p->max_chain = sp.max_chain;
  p->ws_bytes = sp.ws_bytes;
  return true;
}
bool band_chunk_plan(const Geom& g, int num_sms, int smem_optin, ChunkPlan* p, int warps, int stages, int rows,
                     int ppw) {
  SmallPlan sp;
  if (!plan_nchw_band_bf(g, num_sms, smem_optin, &sp, warps, stages, rows, ppw)) return false;
  *p = ChunkPlan{};
  p->small = true;
  p->sp = sp;
  p->threads = 32 * sp.warps;
  p->grid = sp.grid;
  p->smem_bytes = sp.smem;
  p->P = (sp.ppw == 1) ? 1 : 2;
  p->nbands = sp.nbands;
  p->band_rows = sp.R;
  p->ns = sp.ns;
  p->nchunks = (int64_t)sp.groups * sp.nslices;
  p->groups = sp.groups;
  p->nslices = sp.nslices;
  p->n_per_slice = sp.nps;
  p->max_chain = sp.max_chain;
  p->ws_bytes = sp.ws_bytes;
  return true;
}

cudaError_t launch_nchw_fwd(const Geom& g, const ChunkPlan& p, const void* x, const void* w, void* y,
                            cudaStream_t st) {
  if (p.small) return launch_nchw_small(g, p.sp, 0, x, nullptr, w, y, nullptr, nullptr, st);
  nchw::NArgs a = base_args(g, p);
  a.in = x; a.w = w; a.out = y;
  a.wbulk = weights_bulk_ok(g, w);
  nchw::KernelFn fn = nchw::fwd_kernel(g.dtype, g.kh, g.sh, p.ri, p.vi, p.padded, p.pair);
  return launch(fn, p, st, a);
}

cudaError_t launch_nchw_bwd_data(const Geom& g, const ChunkPlan& p, const void* dy, const void* w, void* dx,
                                 cudaStream_t st) {
  if (p.small) return launch_nchw_small(g, p.sp, 1, dy, nullptr, w, dx, nullptr, nullptr, st);
  nchw::NArgs a = base_args(g, p);
  a.in = dy; a.w = w; a.out = dx;
  a.wbulk = weights_bulk_ok(g, w);
  nchw::KernelFn fn = nchw::bwd_data_kernel(g.dtype, g.kh, g.sh, p.ri, p.vi, p.padded, p.pair, g.m == 1);
  return launch(fn, p, st, a);
}

cudaError_t launch_nchw_bwd_filter(const Geom& g, const ChunkPlan& p, const void* x, const void* dy, float* dw,
                                   void* ws, cudaStream_t st) {
  if (p.small) return launch_nchw_small(g, p.sp, 2, x, dy, nullptr, nullptr, dw, ws, st);
  const size_t tk = two_level_tick_bytes(p.groups, p.nslices);
  if (p.direct) {
    direct::DArgs d{};
    d.x = x; d.dy = dy; d.dw = dw;
    d.ws_ticket = static_cast<unsigned*>(ws);
    d.ws_part = reinterpret_cast<float*>(static_cast<char*>(ws) + tk);
    d.N = (int)g.N; d.C = (int)g.C; d.m = g.m; d.Co = (int)(g.C * g.m);
    d.H = (int)g.H; d.W = (int)g.W; d.Ho = (int)g.Ho; d.Wo = (int)g.Wo;
    d.P = p.P; d.groups = p.groups; d.nslices = p.nslices; d.nps = p.n_per_slice;
    d.L = p.dL; d.SPW = p.dSPW; d.spc = p.dspc; d.nsb = p.nsb;
    static const int pf_env = nchw::env_int("DWCONV_DBF_PF", 1, 0, 1);
    const int64_t ebb = (g.dtype == DWCONV_F32) ? 4 : 2;
    d.pf = pf_env && (g.W * ebb) % 16 == 0 && (g.Wo * ebb) % 16 == 0 &&
           ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(dy)) & 15u) == 0;
    direct::DKernelFn fn = p.dstream > 0 ? direct::bwd_filter_stream_kernel(g.dtype, g.sh, p.dstream, p.V)
                                         : direct::bwd_filter_kernel(g.dtype, g.sh, p.R, p.V);
    static const bool pdl = nchw::env_int("DWCONV_PDL", 1, 0, 1) == 1;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)p.grid);
    cfg.blockDim = dim3((unsigned)p.threads);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, fn, d);
  }
  nchw::NArgs a = base_args(g, p);
  a.in = x; a.in2 = dy; a.dw = dw;
  const size_t tick = two_level_tick_bytes(p.groups, p.nslices);
  a.ws_ticket = static_cast<unsigned*>(ws);
  a.ws_part = reinterpret_cast<float*>(static_cast<char*>(ws) + tick);
  nchw::KernelFn fn = nchw::bwd_filter_kernel(g.dtype, g.kh, g.sh, p.ri, p.vi, p.padded);
  return launch(fn, p, st, a);
}

cudaError_t launch_nchw_bwd_fused(const Geom& g, const ChunkPlan& p, const void* x, const void* dy, const void* w,
                                  void* dx, float* dw, void* ws, cudaStream_t st) {
  if (p.small) return launch_nchw_small(g, p.sp, 3, x, dy, w, dx, dw, ws, st);
  nchw::NArgs a = base_args(g, p);
  a.in = x; a.in2 = dy; a.dw = dw; a.w = w; a.out = dx;
  const size_t tick = two_level_tick_bytes(p.groups, p.nslices);
  a.ws_ticket = static_cast<unsigned*>(ws);
  a.ws_part = reinterpret_cast<float*>(static_cast<char*>(ws) + tick);
  nchw::KernelFn fn = nchw::bwd_fused_kernel(g.dtype, g.kh, g.sh, p.ri, p.vi, p.padded);
  if (!fn) return cudaErrorInvalidValue;
  return launch(fn, p, st, a);
}

}  // namespace dwk
