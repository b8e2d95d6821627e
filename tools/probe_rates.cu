// Microbenchmark: FP32 FFMA, FP64 DFMA, MUFU ex2 and rcp throughput on this GPU.
#include <cstdio>
#include <cuda_runtime.h>
template <typename T> __global__ void fma_loop(T* out, int iters, T a, T b) {
  T x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0+4, x5=x0+5, x6=x0+6, x7=x0+7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      x0 = x0 * a + b; x1 = x1 * a + b; x2 = x2 * a + b; x3 = x3 * a + b;
      x4 = x4 * a + b; x5 = x5 * a + b; x6 = x6 * a + b; x7 = x7 * a + b;
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
__global__ void ex2_loop(float* out, int iters) {
  float x0 = threadIdx.x * 1e-3f, x1 = x0 + .1f, x2 = x0 + .2f, x3 = x0 + .3f;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x0)); asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x1));
      asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x2)); asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x3));
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3;
}
int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  printf("%s SMs=%d cc=%d.%d clk=%d kHz\n", p.name, p.multiProcessorCount, p.major, p.minor, p.clockRate);
  int blocks = p.multiProcessorCount * 8, threads = 256, iters = 2000;
  float* of; double* od; cudaMalloc(&of, blocks*threads*8); cudaMalloc(&od, blocks*threads*8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1); float ms;
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0); fma_loop<float><<<blocks, threads>>>(of, iters, 1.0001f, 0.5f); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("FP32 FFMA: %.1f TFLOP/s\n", 2.0 * blocks * threads * iters * 16 * 8 / (ms * 1e-3) / 1e12);
    cudaEventRecord(e0); fma_loop<double><<<blocks, threads>>>(od, iters/4, 1.0001, 0.5); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("FP64 DFMA: %.2f TFLOP/s\n", 2.0 * blocks * threads * (iters/4) * 16 * 8 / (ms * 1e-3) / 1e12);
    cudaEventRecord(e0); ex2_loop<<<blocks, threads>>>(of, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("MUFU ex2: %.2f Tops/s\n", 1.0 * blocks * threads * iters * 16 * 4 / (ms * 1e-3) / 1e12);
  }
  return 0;
}
