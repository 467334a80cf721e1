// fma_probe.cu -- development probe: FMA-pipe throughput of FFMA, FFMA2 and the
// mixed-precision FHFMA.BF16 (fma.rn.f32.bf16: bf16 x bf16 + fp32, operands read
// straight from the 16-bit halves of packed registers) on sm_100a.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o build/fma_probe tools/fma_probe.cu && build/fma_probe
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ITERS = 4096, NACC = 16;

__global__ void k_ffma(float* out, float a, float b) {
  float acc[NACC];
  for (int i = 0; i < NACC; ++i) acc[i] = threadIdx.x + i;
  for (int it = 0; it < ITERS; ++it)
#pragma unroll
    for (int i = 0; i < NACC; ++i) acc[i] = fmaf(acc[i], a, b);
  float s = 0;
  for (int i = 0; i < NACC; ++i) s += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_ffma2(float* out, float a, float b) {
  float2 acc[NACC / 2];
  for (int i = 0; i < NACC / 2; ++i) acc[i] = make_float2(threadIdx.x + i, i);
  const float2 a2 = make_float2(a, a), b2 = make_float2(b, b);
  for (int it = 0; it < ITERS; ++it)
#pragma unroll
    for (int i = 0; i < NACC / 2; ++i) acc[i] = __ffma2_rn(acc[i], a2, b2);
  float s = 0;
  for (int i = 0; i < NACC / 2; ++i) s += acc[i].x + acc[i].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_fhfma(float* out, unsigned xa, unsigned xb) {
  float acc[NACC];
  for (int i = 0; i < NACC; ++i) acc[i] = threadIdx.x + i;
  unsigned x = xa ^ threadIdx.x, y = xb;
  for (int it = 0; it < ITERS; ++it)
#pragma unroll
    for (int i = 0; i < NACC; i += 2)
      asm volatile("{.reg .b16 xl, xh, yl, yh;\n mov.b32 {xl, xh}, %2;\n mov.b32 {yl, yh}, %3;\n"
                   " fma.rn.f32.bf16 %0, xl, yl, %0;\n fma.rn.f32.bf16 %1, xh, yh, %1;}"
                   : "+f"(acc[i]), "+f"(acc[i + 1]) : "r"(x), "r"(y));
  float s = 0;
  for (int i = 0; i < NACC; ++i) s += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const int blocks = sms * 8, threads = 256;
  float* out;
  cudaMalloc(&out, (size_t)blocks * threads * 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const double fmas = (double)blocks * threads * ITERS * NACC;
  for (int rep = 0; rep < 2; ++rep)
    for (int which = 0; which < 3; ++which) {
      cudaEventRecord(e0);
      if (which == 0) k_ffma<<<blocks, threads>>>(out, 1.0001f, 0.5f);
      if (which == 1) k_ffma2<<<blocks, threads>>>(out, 1.0001f, 0.5f);
      if (which == 2) k_fhfma<<<blocks, threads>>>(out, 0x3f803f80u, 0x3f803f80u);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      if (rep == 1)
        printf("%-6s %8.3f ms  %7.2f T FMA/s  %6.1f FMA/clk/SM (clock %d MHz, %d SMs)\n",
               which == 0 ? "FFMA" : which == 1 ? "FFMA2" : "FHFMA", ms, fmas / ms / 1e9,
               fmas / (ms * 1e-3) / sms / (clk * 1e3), clk / 1000, sms);
    }
  return 0;
}
