/*
 * dwconv.h -- C ABI of the B200 (sm_100a) depthwise-convolution training layer.
 *
 * The three calls are the three passes of the depthwise layer in training that
 * arXiv 1803.09926 ("Diagonalwise Refactorization") accelerates:
 *
 *   dwconv_fwd         y = x (*) w            PAPER.md P:173-176 (Sec. II): "a
 *                      depthwise convolution filter (kernel) is applied to one
 *                      input channel with its own set of weights"; P:235-236:
 *                      "a K x K block from the input feature map X is convolved
 *                      with the weights w(i) of the same channel to compute one
 *                      pixel"; Eq. 3, Z = (W (.) A) (x) X.
 *   dwconv_bwd_data    dx = transposed depthwise conv of dy.  The paper leaves
 *                      this pass to the framework; it is the exact
 *                      adjoint of dwconv_fwd (reading R9).
 *   dwconv_bwd_filter  dw = per-channel correlation of x with dy, summed over
 *                      the batch and space: the block diagonal that Eq. 4
 *                       keeps, "redundant gradients are also
 *                      filtered out".
 *
 * Definitions (readings R1-R8 of DESIGN.md §3), with o = c*m + j, j < m:
 *   Ho = (H + 2*pad_h - kh)/stride_h + 1, Wo likewise (floor division).
 *   y [n,o,oh,ow] = sum_{i<kh,jj<kw} w[o,i,jj] * x[n,c,oh*sh-ph+i, ow*sw-pw+jj]
 *   dx[n,c,ih,iw] = sum_{j<m} sum_{i,jj} w[c*m+j,i,jj] * dy[n,c*m+j,(ih+ph-i)/sh,(iw+pw-jj)/sw]
 *                   over taps where the division is exact and the quotient is in range
 *   dw[o,i,jj]    = sum_n sum_{oh,ow} x[n,c,oh*sh-ph+i, ow*sw-pw+jj] * dy[n,o,oh,ow]
 * x is zero outside [0,H) x [0,W) (symmetric zero padding).  The operation is a
 * cross-correlation (no kernel flip), like im2col + GEMM.
 *
 * Layouts.  Activations x, y, dx, dy are dense row-major NCHW ([N][C][H][W]) or
 * NHWC ([N][H][W][C]) as the descriptor says; all four use the same layout.
 * Weights w are always [C*m][kh][kw] (PyTorch's [C*m,1,kh,kw]); the filter
 * gradient dw is always fp32 [C*m][kh][kw].
 *
 * Precision.  DWCONV_F32: fp32 storage.  DWCONV_BF16: x, w, y, dx, dy stored as
 * bfloat16.  Every sum is accumulated in fp32 and rounded once (round to
 * nearest even) on store; no fast-math, no flush-to-zero.
 *
 * Ownership and execution.  Every pointer is a DEVICE pointer owned by the
 * caller; the library never allocates, frees or keeps a pointer after the call
 * returns.  Calls only enqueue work on `stream` (no host synchronisation, no
 * device switch) and are safe to capture in a CUDA graph.  y, dx and dw are
 * fully overwritten.  Inputs and outputs must not overlap.  Results are bitwise
 * deterministic for a given descriptor, device and input (no float atomics).
 *
 * Errors.  Descriptor and pointer validation happens before anything is
 * enqueued; on error nothing is written and the status says why
 * (dwconv_status_string).  DWCONV_ERR_CUDA reports a failed launch; faults
 * inside a kernel surface at the caller's next synchronisation (CUDA rule).
 * The calls are thread-safe.
 */
#ifndef DWCONV_H_
#define DWCONV_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* 2 (round 3): dwconv_plan_info grew kernel_family (+ reserved), DWCONV_MAX_CANDIDATES 32 -> 48,
   DWCONV_VARIANT values unchanged.  A caller built against version 1 passes a smaller
   dwconv_plan_info and must not be linked against this library. */
#define DWCONV_ABI_VERSION 2

#if defined(__GNUC__)
#define DWCONV_API __attribute__((visibility("default")))
#else
#define DWCONV_API
#endif

typedef struct CUstream_st* dwconv_stream; /* == cudaStream_t; NULL = legacy default stream */

typedef enum {
  DWCONV_OK = 0,
  DWCONV_ERR_NULL_POINTER = 1,         /* a required pointer is NULL while its tensor is non-empty */
  DWCONV_ERR_BAD_DESCRIPTOR = 2,       /* n < 0; c,h,w < 1; kh,kw,stride,multiplier < 1; pad < 0;
                                          bad enum; an element count or extent exceeds 2^31 - 1 per
                                          plane dimension or 2^62 in total */
  DWCONV_ERR_KERNEL_EXCEEDS_INPUT = 3, /* Ho < 1 or Wo < 1 ("kernel exceeds padded input") */
  DWCONV_ERR_MISALIGNED = 4,           /* a pointer is not aligned to its element size */
  DWCONV_ERR_WORKSPACE_TOO_SMALL = 5,  /* workspace_bytes < dwconv_bwd_filter_workspace_bytes() */
  DWCONV_ERR_UNSUPPORTED = 6,          /* the current device is not an sm_100 part */
  DWCONV_ERR_CUDA = 7                  /* a CUDA runtime call or kernel launch failed */
} dwconv_status;

typedef enum { DWCONV_NCHW = 0, DWCONV_NHWC = 1 } dwconv_layout;
typedef enum { DWCONV_F32 = 0, DWCONV_BF16 = 1 } dwconv_dtype;

typedef struct {
  int64_t n, c, h, w;          /* input x, logical N, C, H, W (n may be 0)                */
  int32_t multiplier;          /* channel multiplier m >= 1: C*m output channels          */
  int32_t kh, kw;              /* kernel size                                             */
  int32_t stride_h, stride_w;  /* stride >= 1                                             */
  int32_t pad_h, pad_w;        /* symmetric zero padding, pad >= 0                        */
  int32_t layout;              /* dwconv_layout                                           */
  int32_t dtype;               /* dwconv_dtype                                            */
} dwconv_desc;

/* DWCONV_ABI_VERSION of the loaded library. */
DWCONV_API int dwconv_abi_version(void);

/* Static text for a status code (never NULL). */
DWCONV_API const char* dwconv_status_string(int status);

/* Output spatial size; validates the descriptor (no device access). */
DWCONV_API int dwconv_output_shape(const dwconv_desc* d, int64_t* ho, int64_t* wo);

/* y = dwconv(x, w).  x: input activations, w: [C*m][kh][kw], y: output
 * activations [N][C*m][Ho][Wo] (or NHWC).  N == 0 enqueues nothing. */
DWCONV_API int dwconv_fwd(const dwconv_desc* d, const void* x, const void* w, void* y, dwconv_stream stream);

/* dx = dwconv_transpose(dy, w).  dy: [N][C*m][Ho][Wo] (or NHWC), dx: [N][C][H][W]. */
DWCONV_API int dwconv_bwd_data(const dwconv_desc* d, const void* dy, const void* w, void* dx, dwconv_stream stream);

/* Workspace dwconv_bwd_filter needs for this descriptor on the CURRENT device
 * (per-CTA partial sums plus one 32-bit ticket per channel group).  0 is a valid
 * answer.  Returns 0 for an invalid descriptor. */
DWCONV_API size_t dwconv_bwd_filter_workspace_bytes(const dwconv_desc* d);

/* dw = sum over batch and space of x (*) dy, fp32 [C*m][kh][kw].
 * workspace: device memory of at least dwconv_bwd_filter_workspace_bytes(d)
 * bytes, 16-byte aligned, that MUST be zero-filled before its first use (see
 * dwconv_workspace_init); every call leaves it zero-filled again on completion,
 * so one workspace serves any number of consecutive calls on one stream.  Two
 * calls that may run concurrently need separate workspaces.  The cross-CTA
 * reduction has a fixed order (last-CTA finalisation by an integer ticket), so
 * dw is bitwise reproducible.  N == 0 writes dw = 0. */
DWCONV_API int dwconv_bwd_filter(const dwconv_desc* d, const void* x, const void* dy, float* dw,
                      void* workspace, size_t workspace_bytes, dwconv_stream stream);

/* Fused backward: dx = dwconv_transpose(dy, w) AND dw = sum of
 * x (*) dy, from one pass over x and dy where a fused kernel exists (NCHW, 3x3,
 * stride 1, pad 1, m = 1: dy is read from HBM once instead of twice, so the
 * backward moves 2|x| + |dy| + ... instead of 2|x| + 2|dy|).  Other shapes run
 * dwconv_bwd_data then dwconv_bwd_filter on the same stream.  Arguments as for
 * those two calls (dx, dy: activations; w: [C*m][kh][kw]; dw: fp32 [C*m][kh][kw]);
 * workspace: at least dwconv_bwd_workspace_bytes(d), same zero-fill contract as
 * dwconv_bwd_filter.  Results equal the two-call results up to fp32 rounding
 * order (dx is produced by the same stencil arithmetic; dw by the same fixed-order
 * reduction scheme); bitwise reproducible run to run. */
DWCONV_API size_t dwconv_bwd_workspace_bytes(const dwconv_desc* d);
DWCONV_API int dwconv_bwd(const dwconv_desc* d, const void* x, const void* dy, const void* w, void* dx, float* dw,
                          void* workspace, size_t workspace_bytes, dwconv_stream stream);

/* Enqueue a zero-fill of a workspace (cudaMemsetAsync); needed once per buffer. */
DWCONV_API int dwconv_workspace_init(void* workspace, size_t workspace_bytes, dwconv_stream stream);

/* Diagnostics: which kernel family and launch shape a pass would use. */
typedef enum {
  DWCONV_PASS_FWD = 0,
  DWCONV_PASS_BWD_DATA = 1,
  DWCONV_PASS_BWD_FILTER = 2,
  DWCONV_PASS_BWD = 3  /* fused backward (dwconv_bwd); variant NONE with launches = 2: two-call fallback */
} dwconv_pass;
typedef enum {
  DWCONV_VARIANT_NONE = 0,        /* empty batch: nothing to launch (bwd_filter: a memset)  */
  DWCONV_VARIANT_GENERIC = 1,     /* any shape: one thread per output element, global loads */
  DWCONV_VARIANT_NCHW_CHUNK = 2,  /* NCHW: whole planes / row bands staged by bulk TMA      */
  DWCONV_VARIANT_NHWC_TILE = 3,   /* NHWC: spatial x channel-vector register tiles, L1 loads */
  DWCONV_VARIANT_NHWC_TMA = 4,    /* NHWC: 4-D tensor-map TMA boxes with zero-filled halos  */
  DWCONV_VARIANT_NHWC_BDMMA = 5,  /* NHWC bf16: the paper's block-diagonal GEMM on tcgen05 tensor
                                     cores (Eqs. 1-3); group size S in planes_per_chunk,
                                     staged channel block in rows_per_band; a measured candidate
                                     only, never the default */
  DWCONV_VARIANT_NHWC_GEN = 6     /* NHWC: K x K (3/5/7) stride 1/2 multiplier 1/2/4 register
                                     tiles, weights staged in shared memory */
} dwconv_variant;
typedef struct {
  int32_t variant;            /* dwconv_variant */
  int32_t grid, block;        /* launch shape of the main kernel                           */
  int32_t smem_bytes;         /* dynamic shared memory per CTA                            */
  int32_t launches;           /* kernels the pass enqueues                                 */
  int64_t work_units;         /* chunks / tiles the kernel iterates over                    */
  int32_t planes_per_chunk;   /* NCHW: input planes per chunk (1 in band mode)             */
  int32_t rows_per_band;      /* NCHW: output rows per chunk                               */
  int32_t batch_slices;       /* bwd_filter: CTAs that share one channel group              */
  int32_t max_chain;          /* bwd_filter: worst-case serial-add depth of any dw element  */
  int64_t workspace_bytes;    /* bwd_filter workspace                                       */
  int32_t kernel_family;      /* NCHW chunk variant: 0 warp-specialised chunk, 1 small-plane
                                 warp tasks, 2 band bwd_filter, 3 register-direct bwd_filter,
                                 4 streaming bf16 bwd_filter, 5 lane-per-plane (7x7/14x14);
                                 0 for other variants                                       */
  int32_t reserved;
} dwconv_plan_info;
DWCONV_API int dwconv_plan(const dwconv_desc* d, int pass, dwconv_plan_info* info);

/* Measurement-driven plan selection (cf. a "find" step): the fast kernel families'
 * distinct launch shapes for (d, pass), the planner's default first, then by the
 * planner's score.  The caller times them on its own buffers and installs the
 * fastest with dwconv_plan_select; later calls with the same descriptor and pass
 * on the same device use it.  Selection changes only the launch shape (chunking,
 * CTA size, batch slices), never the arithmetic contract: every candidate meets
 * the parity rules of DESIGN.md §5, and a bwd_filter candidate may need a
 * different workspace size (dwconv_bwd_filter_workspace_bytes reflects the
 * selection; re-query after selecting, and zero-fill a new workspace).
 *   dwconv_plan_candidates: pass in {FWD, BWD_DATA, BWD_FILTER, BWD (fused backward, NCHW;
 *     dwconv_bwd_workspace_bytes reflects its selection)}; NCHW and NHWC; writes at most
 *     max_candidates entries to infos (caller-owned array) and the number written
 *     to *count; max_candidates = 0 only reports the total in *count.  N = 0, the
 *     generic override and shapes only the generic kernels cover report 0 candidates.
 *   dwconv_plan_select: index into the same list; -1 restores the planner's pick.
 *     Returns DWCONV_ERR_BAD_DESCRIPTOR if the list was not queried first or the
 *     index is out of range.  Both are host-only calls (no launches) and
 *     thread-safe; neither may be called during stream capture of the same pass.
 *     dwconv_plan_select changes process-wide behaviour for every later call with
 *     that descriptor; callers that must not see (or make) such changes use the
 *     immutable plan handles below (what tune.py and bench.py do). */
#define DWCONV_MAX_CANDIDATES 48
DWCONV_API int dwconv_plan_candidates(const dwconv_desc* d, int pass, int max_candidates, dwconv_plan_info* infos,
                                      int* count);
DWCONV_API int dwconv_plan_select(const dwconv_desc* d, int pass, int index);

/* Immutable launch plans (stateless alternative to dwconv_plan_select).
 *   dwconv_plan_create: resolve (d, pass) once on the host, for the CURRENT device:
 *     candidate = -1 -> the planner's own pick (ignoring any dwconv_plan_select
 *     selection), k >= 0 -> entry k of dwconv_plan_candidates(d, pass) (the list
 *     is computed if it was not queried yet; out of range -> BAD_DESCRIPTOR).
 *     *plan receives a heap object the caller owns (dwconv_plan_destroy frees it).
 *   dwconv_*_plan: the pass of the plan on caller-owned device buffers, same
 *     argument meaning, layout, workspace contract, asynchrony and error codes as
 *     the descriptor calls; the pass must match (else BAD_DESCRIPTOR) and the
 *     current device must be the plan's (else UNSUPPORTED).  A plan is read-only
 *     after creation: any number of threads may use one plan concurrently, and
 *     nothing another call does (dwconv_plan_select included) changes what a plan
 *     launches -- the calls are stateless and capture-safe.
 *   dwconv_plan_workspace_bytes: the workspace the plan's bwd_filter / bwd needs.
 *   dwconv_plan_describe: the plan's launch shape (dwconv_plan_info). */
typedef struct dwconv_plan_s* dwconv_plan_t;
DWCONV_API int dwconv_plan_create(const dwconv_desc* d, int pass, int candidate, dwconv_plan_t* plan);
DWCONV_API void dwconv_plan_destroy(dwconv_plan_t plan);
DWCONV_API int dwconv_plan_describe(dwconv_plan_t plan, dwconv_plan_info* info);
DWCONV_API size_t dwconv_plan_workspace_bytes(dwconv_plan_t plan);
DWCONV_API int dwconv_fwd_plan(dwconv_plan_t plan, const void* x, const void* w, void* y, dwconv_stream stream);
DWCONV_API int dwconv_bwd_data_plan(dwconv_plan_t plan, const void* dy, const void* w, void* dx,
                                    dwconv_stream stream);
DWCONV_API int dwconv_bwd_filter_plan(dwconv_plan_t plan, const void* x, const void* dy, float* dw, void* workspace,
                                      size_t workspace_bytes, dwconv_stream stream);
DWCONV_API int dwconv_bwd_plan(dwconv_plan_t plan, const void* x, const void* dy, const void* w, void* dx, float* dw,
                               void* workspace, size_t workspace_bytes, dwconv_stream stream);

/* Force a kernel family for testing: 0 = automatic (default), 1 = generic only. */
DWCONV_API int dwconv_set_variant_override(int variant);

#ifdef __cplusplus
}
#endif
#endif /* DWCONV_H_ */
