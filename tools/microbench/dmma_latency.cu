// DMMA (mma.sync.m8n8k4.f64) issue characteristics on B200: throughput per SM
// as a function of warps per SM and independent accumulator chains per warp.
// Prints one JSON line per (warps/SM, chains) point. Tuning aid for
// responses_mma.cu (how much ILP/TLP the FP64 tensor pipe needs).
#include <cstdio>
#include <cuda_runtime.h>

template <int C>
__global__ void chains(double* out, int iters) {
    double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
    double c[C][2];
#pragma unroll
    for (int i = 0; i < C; ++i) c[i][0] = c[i][1] = 0.0;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < C; ++i)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                         : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < C; ++i) s += c[i][0] + c[i][1];
    if (s == 12345.678) out[0] = s;
}

template <int C>
void run(int sms, int warps_per_sm, double* out) {
    const int iters = 4096;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    chains<C><<<sms, 32 * warps_per_sm>>>(out, 16);
    cudaEventRecord(e0);
    chains<C><<<sms, 32 * warps_per_sm>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    int khz;
    cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, 0);
    const double dmma = double(iters) * C * warps_per_sm;  // per SM
    const double clk = ms * 1e-3 * khz * 1e3;
    printf("{\"warps_per_sm\":%d,\"chains\":%d,\"clk_per_dmma_per_sm\":%.2f,\"tflops\":%.2f}\n", warps_per_sm, C,
           clk / dmma, 2.0 * 256 * dmma * sms / (ms * 1e-3) / 1e12);
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* out;
    cudaMalloc(&out, 8);
    for (int w : {4, 8, 16, 32}) {
        run<1>(sms, w, out);
        run<2>(sms, w, out);
        run<4>(sms, w, out);
        run<8>(sms, w, out);
    }
    return 0;
}
