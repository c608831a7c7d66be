// FP64 peak microbenchmarks for the roofline denominator (B200, sm_100a):
//   dfma  : independent DFMA chains per thread (vector FP64 pipe)
//   dmma  : mma.sync m8n8k4 f64 (FP64 tensor path)
// Timed with CUDA events after warm-up; prints one JSON line per kernel.
#include <cstdio>
#include <cuda_runtime.h>

template <int CHAINS>
__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double acc[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) acc[c] = threadIdx.x * 1e-9 + c;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) acc[c] = fma(acc[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += acc[c];
  if (s == 12345.678) out[0] = s;
}

__global__ void dmma_kernel(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i) { c[i][0] = 0; c[i][1] = 0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
}

int main() {
  cudaDeviceProp prop; cudaGetDeviceProperties(&prop, 0);
  int sms = prop.multiProcessorCount;
  double* out; cudaMalloc(&out, 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 20000;
  for (int tpb : {256, 512}) for (int bps : {2, 4, 8}) {
    int blocks = sms * bps;
    dfma_kernel<8><<<blocks, tpb>>>(out, 100, 1.0000001, 1e-7);
    cudaEventRecord(e0);
    dfma_kernel<8><<<blocks, tpb>>>(out, iters, 1.0000001, 1e-7);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 8 * iters * (double)blocks * tpb;
    printf("{\"kernel\":\"dfma\",\"tpb\":%d,\"blocks\":%d,\"tflops\":%.2f}\n", tpb, blocks, flops / ms / 1e9);
  }
  for (int tpb : {128, 256}) for (int bps : {2, 4, 8}) {
    int blocks = sms * bps;
    dmma_kernel<<<blocks, tpb>>>(out, 100);
    cudaEventRecord(e0);
    dmma_kernel<<<blocks, tpb>>>(out, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 8 * 8 * 4 * 4 * iters * (double)blocks * (tpb / 32);
    printf("{\"kernel\":\"dmma_m8n8k4\",\"tpb\":%d,\"blocks\":%d,\"tflops\":%.2f}\n", tpb, blocks, flops / ms / 1e9);
  }
  cudaError_t err = cudaGetLastError();
  printf("{\"sms\":%d,\"clock_khz\":%d,\"err\":\"%s\"}\n", sms, prop.clockRate, cudaGetErrorString(err));
  return 0;
}
