// Probe: 2-D tiled TMA copies of {4 floats, R rows} boxes at 8-byte (not 16-byte) aligned
// start coordinates, plus a bulk copy on a second mbarrier.  Prints what arrived.
#include <cstdio>
#include <vector>
#include "../../paper_1901_06919_b200/csrc/tma.cuh"
using namespace fdl;
__global__ void probe(const __grid_constant__ CUtensorMap map, int c0, int rows, float* out, int boxes, int box) {
  extern __shared__ __align__(128) unsigned char sm[];
  unsigned long long* bar = reinterpret_cast<unsigned long long*>(sm);
  float* dst = reinterpret_cast<float*>(sm + 128);
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    mbar_expect_tx(bar, boxes * box * 16);
    for (int b = 0; b < boxes; ++b) tma_load_2d(dst + b * box * 4, &map, c0, b * box, bar);
  }
  mbar_wait(bar, 0);
  for (int e = threadIdx.x; e < boxes * box * 4; e += blockDim.x) out[e] = dst[e];
}
int main() {
  const int plane = 1000, planes = 867;  // floats per plane = 2 * plane
  std::vector<float> h((size_t)planes * plane * 2);
  for (size_t e = 0; e < h.size(); ++e) h[e] = (float)(e % 100003);
  float *d, *o;
  cudaMalloc(&d, h.size() * 4);
  cudaMemcpy(d, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
  const int nbox = 4, box = 224;
  cudaMalloc(&o, nbox * box * 16);
  EncodeTiledFn enc = encode_tiled_fn();
  CUtensorMap m;
  const cuuint64_t gdim[2] = {(cuuint64_t)plane * 2, (cuuint64_t)planes};
  const cuuint64_t gstride[1] = {(cuuint64_t)plane * 8};
  const cuuint32_t bx[2] = {4, (cuuint32_t)box};
  const cuuint32_t es[2] = {1, 1};
  CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, d, gdim, gstride, bx, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode %d\n", (int)r);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 128 + nbox * box * 16);
  for (int c0 : {0, 4, 2, 6, 1998}) {
    probe<<<1, 64, 128 + nbox * box * 16>>>(m, c0, planes, o, nbox, box);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<float> g(nbox * box * 4);
    cudaMemcpy(g.data(), o, g.size() * 4, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int row = 0; row < planes; ++row)
      for (int k = 0; k < 4; ++k) {
        const float want = (c0 + k < 2 * plane) ? h[(size_t)row * plane * 2 + c0 + k] : 0.f;
        if (g[row * 4 + k] != want) ++bad;
      }
    printf("c0=%d: %s, mismatches %d, tail row value %g\n", c0, cudaGetErrorString(e), bad, g[(nbox * box - 1) * 4]);
    if (e != cudaSuccess) break;
  }
  return 0;
}
