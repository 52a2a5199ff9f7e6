// K6: device-side pieces of the GPU-resident pipelines and the render service
// (SURVEY.md §8(f) row 2).
//
//   fdl_view_sqerr    per-(view, channel) sum of squared differences between
//                     rendered views (f32) and the input views (f32 or f64):
//                     the numerators of psnr / mse_per_channel
//                     (pipeline.py:30-51) without reading either image set
//                     back; fp64 accumulation in a fixed order, so the report
//                     does not depend on scheduling.
//   fdl_images_to_u8  the service's 8-bit quantisation
//                     (serve.py:127: (clip(img, 0, 1) * 255).round().astype(uint8),
//                     numpy's round-half-even, evaluated in float64) so a
//                     response leaves the device as 1 byte per sample.
//   fdl_dequantise_views  the loader's decode (io.py:54-59: arr.astype(float64) / 255.0
//                     or / 65535.0) on the device, so 8- / 16-bit views cross PCIe as
//                     1 / 2 bytes per sample instead of 4; float32(float64(v) / max),
//                     bit for bit what the host decode followed by the float32 upload gives.
#include "common.cuh"

namespace fdl {

namespace {

constexpr int SQ_THREADS = 256;
constexpr int SQ_SPLIT = 64;  // CTAs per view: fixed partition of the view's pixels

template <typename REF, int C>
__global__ void __launch_bounds__(SQ_THREADS) sqerr_partial_kernel(const float* __restrict__ img,
                                                                   const REF* __restrict__ ref, long long pixels,
                                                                   double* __restrict__ partial) {
  const int v = blockIdx.y, part = blockIdx.x;
  const long long per = (pixels + SQ_SPLIT - 1) / SQ_SPLIT;
  const long long p0 = (long long)part * per, p1 = min(pixels, p0 + per);
  const float* a = img + (size_t)v * pixels * C;
  const REF* b = ref + (size_t)v * pixels * C;
  double acc[C];
#pragma unroll
  for (int c = 0; c < C; ++c) acc[c] = 0.0;
  for (long long px = p0 + threadIdx.x; px < p1; px += SQ_THREADS) {
#pragma unroll
    for (int c = 0; c < C; ++c) {
      const double d = (double)a[px * C + c] - (double)b[px * C + c];
      acc[c] = fma(d, d, acc[c]);
    }
  }
  __shared__ double red[SQ_THREADS / 32][C];
#pragma unroll
  for (int c = 0; c < C; ++c) {
    double s = acc[c];
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5][c] = s;
  }
  __syncthreads();
  if (threadIdx.x < C) {
    double tot = 0.0;
    for (int w = 0; w < SQ_THREADS / 32; ++w) tot += red[w][threadIdx.x];
    partial[((size_t)v * SQ_SPLIT + part) * C + threadIdx.x] = tot;
  }
}

__global__ void sqerr_final_kernel(const double* __restrict__ partial, int V, int C, double* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;  // (v, c)
  if (i >= V * C) return;
  const int v = i / C, c = i % C;
  double tot = 0.0;
  for (int part = 0; part < SQ_SPLIT; ++part) tot += partial[((size_t)v * SQ_SPLIT + part) * C + c];
  out[i] = tot;
}

template <typename REF>
int launch_sqerr(const float* img, const REF* ref, int V, long long pixels, int C, double* partial, double* out,
                 cudaStream_t st) {
  dim3 grid(SQ_SPLIT, V);
  switch (C) {
    case 1: sqerr_partial_kernel<REF, 1><<<grid, SQ_THREADS, 0, st>>>(img, ref, pixels, partial); break;
    case 2: sqerr_partial_kernel<REF, 2><<<grid, SQ_THREADS, 0, st>>>(img, ref, pixels, partial); break;
    case 3: sqerr_partial_kernel<REF, 3><<<grid, SQ_THREADS, 0, st>>>(img, ref, pixels, partial); break;
    case 4: sqerr_partial_kernel<REF, 4><<<grid, SQ_THREADS, 0, st>>>(img, ref, pixels, partial); break;
    default: return fail(FDL_ERR_UNSUPPORTED, "images support 1..4 channels");
  }
  FDL_LAUNCH_CHECK("sqerr_partial_kernel");
  sqerr_final_kernel<<<(V * C + 127) / 128, 128, 0, st>>>(partial, V, C, out);
  FDL_LAUNCH_CHECK("sqerr_final_kernel");
  return FDL_OK;
}

__global__ void images_to_u8_kernel(const float* __restrict__ img, size_t count, unsigned char* __restrict__ out) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (size_t)gridDim.x * blockDim.x) {
    double x = (double)img[i];
    x = x < 0.0 ? 0.0 : (x > 1.0 ? 1.0 : x);  // np.clip (NaN propagates to 0 below, as astype(uint8) of NaN is undefined)
    const double r = rint(__dmul_rn(x, 255.0));  // np.round: half to even
    out[i] = (unsigned char)(r == r ? (int)r : 0);
  }
}

// 8-bit: the 256 possible results are formed once per CTA (correctly rounded fp64
// division, then RN to float32) and looked up; 16 samples per thread through 16-byte loads
__global__ void __launch_bounds__(256) dequant8_kernel(const uint8_t* __restrict__ q, size_t count,
                                                       float* __restrict__ out) {
  __shared__ float lut[256];
  lut[threadIdx.x] = __double2float_rn(__ddiv_rn((double)threadIdx.x, 255.0));
  __syncthreads();
  const bool aligned = reinterpret_cast<uintptr_t>(q) % 16 == 0 && reinterpret_cast<uintptr_t>(out) % 16 == 0;
  const size_t vec = aligned ? count / 16 : 0;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x; e < vec; e += stride) {
    const uint4 w = __ldg(reinterpret_cast<const uint4*>(q) + e);
    const unsigned ws[4] = {w.x, w.y, w.z, w.w};
    float4* o = reinterpret_cast<float4*>(out) + 4 * e;
#pragma unroll
    for (int k = 0; k < 4; ++k)
      o[k] = make_float4(lut[ws[k] & 255u], lut[(ws[k] >> 8) & 255u], lut[(ws[k] >> 16) & 255u], lut[ws[k] >> 24]);
  }
  for (size_t e = vec * 16 + (size_t)blockIdx.x * blockDim.x + threadIdx.x; e < count; e += stride) out[e] = lut[q[e]];
}

__global__ void __launch_bounds__(256) dequant16_kernel(const uint16_t* __restrict__ q, size_t count,
                                                        float* __restrict__ out) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x; e < count; e += stride)
    out[e] = __double2float_rn(__ddiv_rn((double)q[e], 65535.0));
}

}  // namespace
}  // namespace fdl

extern "C" {

size_t fdl_view_sqerr_workspace(int32_t V, int32_t C) {
  if (V < 0 || C < 1) return 0;
  return sizeof(double) * (size_t)(V > 0 ? V : 1) * fdl::SQ_SPLIT * C;
}

int fdl_view_sqerr(const float* images_dev, const void* ref_dev, int32_t ref_is_f64, int32_t V, int32_t H, int32_t W,
                   int32_t C, double* sqerr_dev, void* workspace_dev, size_t workspace_bytes, void* stream) {
  using namespace fdl;
  if (V < 0 || H < 1 || W < 1 || C < 1 || C > 4) return fail(FDL_ERR_INVALID, "fdl_view_sqerr: invalid shape");
  if (V == 0) return FDL_OK;
  if (!images_dev || !ref_dev || !sqerr_dev) return fail(FDL_ERR_INVALID, "fdl_view_sqerr: null buffer");
  if (!workspace_dev || workspace_bytes < fdl_view_sqerr_workspace(V, C))
    return fail(FDL_ERR_INVALID, "workspace too small for fdl_view_sqerr");
  double* partial = reinterpret_cast<double*>(workspace_dev);
  const long long pixels = (long long)H * W;
  cudaStream_t st = as_stream(stream);
  if (ref_is_f64)
    return launch_sqerr(images_dev, reinterpret_cast<const double*>(ref_dev), V, pixels, C, partial, sqerr_dev, st);
  return launch_sqerr(images_dev, reinterpret_cast<const float*>(ref_dev), V, pixels, C, partial, sqerr_dev, st);
}

int fdl_images_to_u8(const float* images_dev, int64_t count, uint8_t* out_dev, void* stream) {
  using namespace fdl;
  if (count < 0) return fail(FDL_ERR_INVALID, "fdl_images_to_u8: negative count");
  if (count == 0) return FDL_OK;
  if (!images_dev || !out_dev) return fail(FDL_ERR_INVALID, "fdl_images_to_u8: null buffer");
  const size_t blocks = ((size_t)count + 255) / 256;
  const int grid = (int)(blocks < 148 * 16 ? blocks : 148 * 16);
  images_to_u8_kernel<<<grid, 256, 0, as_stream(stream)>>>(images_dev, (size_t)count, out_dev);
  FDL_LAUNCH_CHECK("images_to_u8_kernel");
  return FDL_OK;
}

int fdl_dequantise_views(const void* q_dev, int32_t bits, int64_t count, float* out_dev, void* stream) {
  using namespace fdl;
  if (bits != 8 && bits != 16) return fail(FDL_ERR_INVALID, "fdl_dequantise_views: bits must be 8 or 16");
  if (count < 0) return fail(FDL_ERR_INVALID, "fdl_dequantise_views: negative count");
  if (count == 0) return FDL_OK;
  if (!q_dev || !out_dev) return fail(FDL_ERR_INVALID, "fdl_dequantise_views: null buffer");
  const size_t per = bits == 8 ? 256 * 16 : 256;
  const size_t blocks = ((size_t)count + per - 1) / per;
  const int grid = (int)(blocks < 148 * 16 ? blocks : 148 * 16);
  cudaStream_t st = as_stream(stream);
  if (bits == 8)
    dequant8_kernel<<<grid, 256, 0, st>>>(reinterpret_cast<const uint8_t*>(q_dev), (size_t)count, out_dev);
  else
    dequant16_kernel<<<grid, 256, 0, st>>>(reinterpret_cast<const uint16_t*>(q_dev), (size_t)count, out_dev);
  FDL_LAUNCH_CHECK("dequant_kernel");
  return FDL_OK;
}

}  // extern "C"
