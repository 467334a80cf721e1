// umma_probe.cu -- development probe for the tcgen05 encodings the block-diagonal
// MMA kernel (csrc/nhwc_bdmma.cu) relies on; not part of the library.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/umma_probe tools/umma_probe.cu && /tmp/umma_probe
//
// A: 256 rows x 64 bf16 (128 B per row) in the TMA SWIZZLE_128B layout (16-B chunk
//    index XOR (row & 7)), read as a K-major SW128 operand starting at row `shift`
//    (any 0..127: the tap shift of the implicit GEMM), K chunk kc (32 B) inside the row.
// B: N x 16 bf16 per K chunk, K-major no-swizzle (8-row x 16-B core matrices).
// D: 128 x N fp32 in TMEM, read back with tcgen05.ld.32x32b.
// Checks D = sum_kc A[shift + r, kc*16 + k] * B_kc[n, k] exactly (small integers).
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <vector>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo, uint32_t layout, uint32_t base_off) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;                 // version 1 (sm_100)
  d |= (uint64_t)(base_off & 7) << 49;
  d |= (uint64_t)(layout & 7) << 61;
  return d;
}

template <int N>
__global__ void probe(const __nv_bfloat16* ga, const __nv_bfloat16* gb, float* gd, int shift, int use_base) {
  extern __shared__ __align__(1024) unsigned char smem[];
  unsigned char* A = smem;                        // 256 x 128 B, 1024-aligned
  unsigned char* B = smem + 256 * 128;            // 4 chunks x N x 32 B
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x;
  // A: row r, element k (0..63) -> chunk (k/8) ^ (r&7)
  for (int i = tid; i < 256 * 64; i += blockDim.x) {
    const int r = i / 64, k = i % 64;
    const int ch = (k / 8) ^ (r & 7);
    *reinterpret_cast<__nv_bfloat16*>(A + r * 128 + ch * 16 + (k % 8) * 2) = ga[i];
  }
  // B chunk kc: [N][16] K-major interleave: core (n/8, k/8) at ((n/8)*2 + k/8)*128, row n%8 at 16 B
  for (int i = tid; i < 4 * N * 16; i += blockDim.x) {
    const int kc = i / (N * 16), n = (i / 16) % N, k = i % 16;
    *reinterpret_cast<__nv_bfloat16*>(B + kc * N * 32 + ((n / 8) * 2 + k / 8) * 128 + (n % 8) * 16 + (k % 8) * 2) =
        gb[i];
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (tid < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(smem_u32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;");  // generic-proxy smem writes -> visible to the tensor core
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = tbase;
  if (tid == 0) {
    const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    for (int kc = 0; kc < 4; ++kc) {
      const uint32_t aaddr = smem_u32(A) + shift * 128 + kc * 32;
      const uint64_t ad = sdesc(aaddr, 16, 1024, 2, use_base ? ((aaddr >> 7) & 7) : 0);
      const uint64_t bd = sdesc(smem_u32(B) + kc * N * 32, 128, 256, 0, 0);
      const uint32_t acc = kc > 0;
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
          "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tm),
          "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
  }
  // wait phase 0
  asm volatile(
      "{\n\t.reg .pred P1;\n\tLAB_WAIT:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t"
      "@P1 bra DONE;\n\tbra LAB_WAIT;\n\tDONE:\n\t}" ::"r"(smem_u32(&bar)));
  asm volatile("tcgen05.fence::after_thread_sync;");
  const int warp = tid / 32, lane = tid % 32;
  const int row = warp * 32 + lane;
  for (int c0 = 0; c0 < N; c0 += 8) {
    uint32_t v[8];
    const uint32_t ta = tm + ((uint32_t)(warp * 32) << 16) + c0;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                 : "r"(ta));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    for (int j = 0; j < 8; ++j) gd[row * N + c0 + j] = __uint_as_float(v[j]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tm));
}

template <int N>
int run(int shift, int use_base) {
  std::vector<__nv_bfloat16> a(256 * 64), b(4 * N * 16);
  std::vector<float> af(a.size()), bf(b.size());
  srand(shift * 7 + N);
  for (size_t i = 0; i < a.size(); ++i) { af[i] = (float)(rand() % 7 - 3); a[i] = __float2bfloat16(af[i]); }
  for (size_t i = 0; i < b.size(); ++i) { bf[i] = (float)(rand() % 5 - 2); b[i] = __float2bfloat16(bf[i]); }
  __nv_bfloat16 *da, *db;
  float* dd;
  cudaMalloc(&da, a.size() * 2);
  cudaMalloc(&db, b.size() * 2);
  cudaMalloc(&dd, 128 * N * 4);
  cudaMemcpy(da, a.data(), a.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(db, b.data(), b.size() * 2, cudaMemcpyHostToDevice);
  cudaMemset(dd, 0xFF, 128 * N * 4);
  const int smem = 256 * 128 + 4 * N * 32;
  cudaFuncSetAttribute(probe<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  probe<N><<<1, 128, smem>>>(da, db, dd, shift, use_base);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("N=%d shift=%d base=%d: CUDA error %s\n", N, shift, use_base, cudaGetErrorString(e)); exit(1); }
  std::vector<float> d(128 * N);
  cudaMemcpy(d.data(), dd, d.size() * 4, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int r = 0; r < 128; ++r)
    for (int n = 0; n < N; ++n) {
      float ref = 0;
      for (int kc = 0; kc < 4; ++kc)
        for (int k = 0; k < 16; ++k) ref += af[(shift + r) * 64 + kc * 16 + k] * bf[kc * N * 16 + n * 16 + k];
      if (d[r * N + n] != ref) {
        if (bad < 3) printf("  mismatch r=%d n=%d got %g ref %g\n", r, n, d[r * N + n], ref);
        ++bad;
      }
    }
  printf("N=%d shift=%d base_offset=%s: %s (%d bad)\n", N, shift, use_base ? "addr" : "0", bad ? "FAIL" : "PASS", bad);
  cudaFree(da); cudaFree(db); cudaFree(dd);
  return bad;
}

int main() {
  int bad = 0;
  for (int base = 0; base < 2; ++base)
    for (int s : {0, 1, 3, 8, 13, 40, 127}) bad += run<16>(s, base) ? 1 : 0;
  for (int s : {0, 5, 33}) bad += run<32>(s, 0) ? 1 : 0;
  for (int s : {0, 7, 66}) bad += run<64>(s, 0) ? 1 : 0;
  printf("probe done, %d failing configs\n", bad);
  return 0;
}
