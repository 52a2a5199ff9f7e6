// Microbenchmark: FP64 SIMT (DFMA) vs FP64 tensor (DMMA m8n8k4) throughput on B200.
// Decides the per-bin solver design ("K1 solver").
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}

__global__ void dmma_kernel(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[8][2];
#pragma unroll
  for (int t = 0; t < 8; ++t) { c[t][0] = 0; c[t][1] = 0; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[t][0]), "+d"(c[t][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int t = 0; t < 8; ++t) s += c[t][0] + c[t][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void sincos_kernel(double* out, int iters) {
  double x = threadIdx.x * 1e-3, s0 = 0, c0 = 0;
  for (int i = 0; i < iters; ++i) {
    double s, c;
    sincospi(x, &s, &c);
    s0 += s; c0 += c; x += 1e-7;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s0 + c0;
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double* out; cudaMalloc(&out, 1 << 26);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int blocksPerSM : {2, 4, 8}) {
    int threads = 256, blocks = sms * blocksPerSM, iters = 4096;
    dfma_kernel<<<blocks, threads>>>(out, 16, 1.0000001, 1e-9);
    cudaEventRecord(e0);
    dfma_kernel<<<blocks, threads>>>(out, iters, 1.0000001, 1e-9);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 64 * iters * (double)blocks * threads;
    printf("DFMA  blocks/SM=%d: %.2f TFLOP/s (%.3f ms)\n", blocksPerSM, flops / ms / 1e9, ms);
  }
  for (int blocksPerSM : {1, 2, 4, 8}) {
    int threads = 128, blocks = sms * blocksPerSM, iters = 2048;
    dmma_kernel<<<blocks, threads>>>(out, 16);
    cudaEventRecord(e0);
    dmma_kernel<<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 256 * 8 * iters * (double)blocks * (threads / 32);
    printf("DMMA  blocks/SM=%d: %.2f TFLOP/s (%.3f ms)\n", blocksPerSM, flops / ms / 1e9, ms);
  }
  {
    int threads = 256, blocks = sms * 8, iters = 1024;
    sincos_kernel<<<blocks, threads>>>(out, 16);
    cudaEventRecord(e0);
    sincos_kernel<<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("sincospi f64: %.2f Gop/s\n", (double)iters * blocks * threads / ms / 1e6);
  }
  printf("SMs=%d clock=%d kHz err=%s\n", sms, clk, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
