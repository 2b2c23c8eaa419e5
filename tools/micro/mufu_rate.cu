// Dev microbenchmark: MUFU.EX2 and FFMA2 throughput per SM on this GPU.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mufu_rate mufu_rate.cu && ./mufu_rate
#include <cstdio>
#include <cstdint>
__global__ void ex2_kernel(float* out, int iters) {
  float a[8];
  for (int i = 0; i < 8; ++i) a[i] = -0.001f * (threadIdx.x + i);
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
  float s = 0;
  for (int i = 0; i < 8; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
// packed bf16 / f16 exp2: two results per lane per instruction
__global__ void ex2_bf16x2_kernel(float* out, int iters) {
  uint32_t a[8];
  for (int i = 0; i < 8; ++i) a[i] = 0xBC00BC00u - threadIdx.x - i;  // ~ -0.0078 (bf16 pairs)
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(a[i]));
  uint32_t s = 0;
  for (int i = 0; i < 8; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = (float)s;
}
__global__ void ex2_f16x2_kernel(float* out, int iters) {
  uint32_t a[8];
  for (int i = 0; i < 8; ++i) a[i] = 0xA000A000u - threadIdx.x - i;  // ~ -0.0078 (f16 pairs)
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(a[i]));
  uint32_t s = 0;
  for (int i = 0; i < 8; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = (float)s;
}
__global__ void ffma2_kernel(float* out, int iters) {
  uint64_t a[8];
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x + i;
  const uint64_t b = 0x3f8000003f800000ull;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("fma.rn.f32x2 %0, %0, %1, %1;" : "+l"(a[i]) : "l"(b));
  uint64_t s = 0;
  for (int i = 0; i < 8; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = (float)s;
}
int main() {
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  float* out;
  cudaMalloc(&out, sizeof(float) * sms * 1024);
  const int iters = 4096;
  const char* names[4] = {"EX2 f32", "FFMA2(pairs)", "EX2 bf16x2 (instructions)", "EX2 f16x2 (instructions)"};
  for (int k = 0; k < 4; ++k) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      if (k == 0) ex2_kernel<<<sms, 1024>>>(out, iters);
      else if (k == 1) ffma2_kernel<<<sms, 1024>>>(out, iters);
      else if (k == 2) ex2_bf16x2_kernel<<<sms, 1024>>>(out, iters);
      else ex2_f16x2_kernel<<<sms, 1024>>>(out, iters);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
    }
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double ops = double(sms) * 1024 * iters * 8;  // lane-ops (FFMA2: pairs)
    printf("%s: %.3f ms, %.1f lane-ops/clk/SM at %d MHz (max clock)\n", names[k],
           ms, ops / (ms * 1e-3) / sms / (clk * 1e3), clk / 1000);
  }
  return 0;
}
