// LDS.128 / LDS.64 wavefront counts for the K3 lane->address patterns (run under ncu:
// l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum / smsp__inst_executed_op_shared_ld.sum).
#include <cstdio>
template <int MODE>
__global__ void k(float* out, int iters) {
  // MODE 0: lane&7 (8 distinct 16B words x4), 1: lane>>3 (4 distinct x8), 2: lane (32 distinct),
  // 3: broadcast, 4: 4 distinct same-bank; MODE 10+: the same as float2 (LDS.64)
  __shared__ float4 s[512];
  for (int i = threadIdx.x; i < 512; i += blockDim.x) s[i] = make_float4(i, i + 1, i + 2, i + 3);
  __syncthreads();
  const int lane = threadIdx.x & 31;
  int a;
  const int M = MODE % 10;
  if (M == 0) a = lane & 7;             // 8 distinct contiguous, x4
  else if (M == 1) a = lane >> 3;       // 4 distinct contiguous, x8
  else if (M == 2) a = lane;            // 32 distinct
  else if (M == 3) a = 0;               // broadcast
  else if (M == 4) a = (lane >> 3) * 32;  // 4 distinct, stride 512 B (same banks)
  else a = (lane & 7) + 8 * (lane >> 3);   // = lane
  float acc = 0;
  for (int it = 0; it < iters; ++it) {
    if (MODE < 10) {
      float4 v = s[a + (it & 1) * 64];
      acc += v.x + v.y + v.z + v.w;
    } else {
      float2 v = reinterpret_cast<float2*>(s)[a + (it & 1) * 64];
      acc += v.x + v.y;
    }
    asm volatile("" ::: "memory");
  }
  out[threadIdx.x + blockIdx.x * blockDim.x] = acc;
}
int main() {
  float* o;
  cudaMalloc(&o, 1 << 20);
  k<0><<<1, 32>>>(o, 1000);
  k<1><<<1, 32>>>(o, 1000);
  k<2><<<1, 32>>>(o, 1000);
  k<3><<<1, 32>>>(o, 1000);
  k<4><<<1, 32>>>(o, 1000);
  k<10><<<1, 32>>>(o, 1000);
  k<11><<<1, 32>>>(o, 1000);
  k<12><<<1, 32>>>(o, 1000);
  k<13><<<1, 32>>>(o, 1000);
  cudaDeviceSynchronize();
  printf("ok\n");
}
