// FP32 peak probe: scalar FFMA vs packed FFMA2 (fma.rn.f32x2) throughput on
// this GPU, CUDA-event timed.  Reports TFLOP/s (FMA = 2 FLOP).
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long f2u(float2 v) { return *reinterpret_cast<unsigned long long*>(&v); }
__device__ __forceinline__ float2 u2f(unsigned long long v) { return *reinterpret_cast<float2*>(&v); }

__global__ void ffma1(float* out, float b, float c, int iters) {
  float acc[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) acc[i] = threadIdx.x * 1e-3f + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) acc[i] = fmaf(acc[i], b, c);
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void ffma2(float* out, float b, float c, int iters) {
  unsigned long long acc[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) acc[i] = f2u(make_float2(threadIdx.x * 1e-3f + i, i + 0.5f));
  const unsigned long long bb = f2u(make_float2(b, b)), cc = f2u(make_float2(c, c));
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(acc[i]) : "l"(bb), "l"(cc));
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) { float2 v = u2f(acc[i]); s += v.x + v.y; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int threads = 256, blocks = sms * 8, iters = 1 << 16;
  float* out; cudaMalloc(&out, sizeof(float) * blocks * threads);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const double flops = 2.0 * 16 * (double)iters * blocks * threads;
  for (int rep = 0; rep < 2; ++rep) {
    ffma1<<<blocks, threads>>>(out, 0.999f, 1e-3f, iters / 8);
    cudaEventRecord(a); ffma1<<<blocks, threads>>>(out, 0.999f, 1e-3f, iters); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms1; cudaEventElapsedTime(&ms1, a, b);
    cudaEventRecord(a); ffma2<<<blocks, threads>>>(out, 0.999f, 1e-3f, iters); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms2; cudaEventElapsedTime(&ms2, a, b);
    printf("{\"ffma_tflops\": %.2f, \"ffma2_tflops\": %.2f, \"sms\": %d}\n", flops / ms1 / 1e9, flops / ms2 / 1e9, sms);
  }
  return 0;
}
