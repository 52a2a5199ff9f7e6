// Microbenchmark: FP32 throughput on B200 -- scalar FFMA (3-register form) vs
// packed FFMA2 (fma.rn.f32x2) with a broadcast scalar operand, the form the K3
// render tiles issue.  The FFMA2 number is the render roofline's denominator.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void ffma_kernel(float* out, int iters, float a, float b) {
  float x[16];
#pragma unroll
  for (int r = 0; r < 16; ++r) x[r] = threadIdx.x + r;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int r = 0; r < 16; ++r) x[r] = fmaf(x[r], a, b);
  }
  float s = 0;
#pragma unroll
  for (int r = 0; r < 16; ++r) s += x[r];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void ffma2_kernel(float* out, int iters, float a, float b) {
  unsigned long long x[16], bb;
  asm("mov.b64 %0, {%1, %1};" : "=l"(bb) : "f"(b));
#pragma unroll
  for (int r = 0; r < 16; ++r) {
    float lo = threadIdx.x + r, hi = lo + 0.5f;
    asm("mov.b64 %0, {%1, %2};" : "=l"(x[r]) : "f"(lo), "f"(hi));
  }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      unsigned long long aa;
      asm("mov.b64 %0, {%1, %1};" : "=l"(aa) : "f"(a));
      asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(x[r]) : "l"(aa), "l"(bb));
    }
  }
  float s = 0;
#pragma unroll
  for (int r = 0; r < 16; ++r) {
    float lo, hi;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(x[r]));
    s += lo + hi;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// all operands in ordinary (per-thread) registers, as in the render tiles
__global__ void ffma2_reg_kernel(float* out, int iters, float a, float b) {
  unsigned long long x[16], bb, aa;
  const float at = a + threadIdx.x * 1e-12f, bt = b + threadIdx.x * 1e-12f;
  asm("mov.b64 %0, {%1, %2};" : "=l"(bb) : "f"(bt), "f"(bt));
#pragma unroll
  for (int r = 0; r < 16; ++r) {
    float lo = threadIdx.x + r, hi = lo + 0.5f;
    asm("mov.b64 %0, {%1, %2};" : "=l"(x[r]) : "f"(lo), "f"(hi));
  }
  asm("mov.b64 %0, {%1, %1};" : "=l"(aa) : "f"(at));
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int r = 0; r < 16; ++r) asm volatile("fma.rn.f32x2 %0, %1, %0, %2;" : "+l"(x[r]) : "l"(aa), "l"(bb));
  }
  float s = 0;
#pragma unroll
  for (int r = 0; r < 16; ++r) {
    float lo, hi;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(x[r]));
    s += lo + hi;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* out; cudaMalloc(&out, 1 << 26);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int blocksPerSM : {2, 4, 8}) {
    int threads = 256, blocks = sms * blocksPerSM, iters = 8192;
    ffma_kernel<<<blocks, threads>>>(out, 16, 1.0000001f, 1e-9f);
    cudaEventRecord(e0);
    ffma_kernel<<<blocks, threads>>>(out, iters, 1.0000001f, 1e-9f);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 16 * iters * (double)blocks * threads;
    printf("FFMA   blocks/SM=%d: %.2f TFLOP/s (%.3f ms)\n", blocksPerSM, flops / ms / 1e9, ms);
  }
  for (int blocksPerSM : {2, 4, 8}) {
    int threads = 256, blocks = sms * blocksPerSM, iters = 8192;
    ffma2_kernel<<<blocks, threads>>>(out, 16, 1.0000001f, 1e-9f);
    cudaEventRecord(e0);
    ffma2_kernel<<<blocks, threads>>>(out, iters, 1.0000001f, 1e-9f);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 4.0 * 16 * iters * (double)blocks * threads;
    printf("FFMA2  blocks/SM=%d: %.2f TFLOP/s (%.3f ms)\n", blocksPerSM, flops / ms / 1e9, ms);
  }
  for (int blocksPerSM : {2, 4, 8}) {
    int threads = 256, blocks = sms * blocksPerSM, iters = 8192;
    ffma2_reg_kernel<<<blocks, threads>>>(out, 16, 1.0000001f, 1e-9f);
    cudaEventRecord(e0);
    ffma2_reg_kernel<<<blocks, threads>>>(out, iters, 1.0000001f, 1e-9f);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 4.0 * 16 * iters * (double)blocks * threads;
    printf("FFMA2r blocks/SM=%d: %.2f TFLOP/s (%.3f ms)\n", blocksPerSM, flops / ms / 1e9, ms);
  }
  printf("SMs=%d err=%s\n", sms, cudaGetErrorString(cudaGetLastError()));
}
