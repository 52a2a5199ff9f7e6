// K0: zero-pad + batched R2C + per-view sum |b|^2  (construct.py:250-266).
// K4: Hermitian projection of self-conjugate columns + C2R + crop + sRGB
//     (spectra.py:202-208, render.py:210-225).
//
// Both are HBM-bound streaming kernels around cuFFT.  Plans are cached per
// host thread (cuFFT plans are not safe to share between concurrent callers)
// and never allocate: their work area comes from the caller's workspace.
#include <cufft.h>

#include <map>
#include <tuple>

#include "common.cuh"

namespace fdl {

// k0_fft.cu: the shared-memory FFT engine path
bool fft_engine_applies(int Hp, int Wp, int C);
bool fft_cufft_forced();
// k4_mr.cu: mixed-radix K4 (1920 x 1080 grids)
bool mr_engine_applies(int Hp, int Wp, int C);
size_t mr_engine_inv_ws(int V, int C, int Ho, int Wp);
int mr_engine_inv(const float2* spectra, int V, int C, int Hp, int Wp, int pad, int Ho, int Wo, int srgb, float* images,
                  void* ws, cudaStream_t st);
size_t engine_fwd_ws(int m, int H, int W, int C, int pad);
int engine_fwd(const float* views, int m, int H, int W, int C, int pad, float2* spectra, double* view_sumsq,
               void* ws, cudaStream_t st, int srgb);
size_t engine_inv_ws(int V, int C, int Hp, int Wp);
int engine_inv(const float2* spectra, int V, int C, int Hp, int Wp, int pad, int Ho, int Wo, int srgb, float* images,
               void* ws, cudaStream_t st);

namespace {

struct PlanKey {
  int h, w, batch, type;
  bool operator<(const PlanKey& o) const {
    return std::tie(h, w, batch, type) < std::tie(o.h, o.w, o.batch, o.type);
  }
};

struct Plan {
  cufftHandle handle = 0;
  size_t work = 0;
};

thread_local std::map<PlanKey, Plan> t_plans;

// type 0: R2C (real input H x W -> H x (W/2+1)), 1: C2R
int get_plan(int h, int w, int batch, int type, Plan** out) {
  PlanKey key{h, w, batch, type};
  auto it = t_plans.find(key);
  if (it != t_plans.end()) {
    *out = &it->second;
    return FDL_OK;
  }
  Plan p;
  if (cufftCreate(&p.handle) != CUFFT_SUCCESS) return fail(FDL_ERR_CUDA, "cufftCreate failed");
  cufftSetAutoAllocation(p.handle, 0);
  int n[2] = {h, w};
  int whp = w / 2 + 1;
  cufftResult r;
  if (type == 0) {
    int inembed[2] = {h, w}, onembed[2] = {h, whp};
    r = cufftMakePlanMany(p.handle, 2, n, inembed, 1, h * w, onembed, 1, h * whp, CUFFT_R2C, batch, &p.work);
  } else {
    int inembed[2] = {h, whp}, onembed[2] = {h, w};
    r = cufftMakePlanMany(p.handle, 2, n, inembed, 1, h * whp, onembed, 1, h * w, CUFFT_C2R, batch, &p.work);
  }
  if (r != CUFFT_SUCCESS) {
    cufftDestroy(p.handle);
    return fail(FDL_ERR_CUDA, "cufftMakePlanMany failed (" + std::to_string((int)r) + ")");
  }
  auto res = t_plans.emplace(key, p);
  *out = &res.first->second;
  return FDL_OK;
}

inline size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

// views (m,H,W,C) -> padded planar (m,C,Hp,Wp).  One thread per (view, padded
// row, 4 consecutive padded columns): reads the 4*C interleaved input floats,
// writes one float4 per channel plane (Wp % 4 == 0) or 4 scalars.
template <int C>
__global__ void pack_pad_kernel(const float* __restrict__ views, int m, int H, int W, int pad,
                                float* __restrict__ out, int srgb) {
  const int Hp = H + 2 * pad, Wp = W + 2 * pad;
  const int W4 = (Wp + 3) / 4;
  const size_t total = (size_t)m * Hp * W4;
  const bool vec = (Wp % 4) == 0;
  for (size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (size_t)gridDim.x * blockDim.x) {
    const int x4 = (int)(idx % W4);
    const size_t r = idx / W4;
    const int y = (int)(r % Hp);
    const int j = (int)(r / Hp);
    const int ys = y - pad;
    float v[4][C];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int xs = x4 * 4 + e - pad;
      const bool in = ys >= 0 && ys < H && xs >= 0 && xs < W;
      const float* src = views + (((size_t)j * H + (in ? ys : 0)) * W + (in ? xs : 0)) * C;
#pragma unroll
      for (int c = 0; c < C; ++c) {
        float x = in ? __ldg(src + c) : 0.f;
        // sRGB -> linear light (render.py:39-42), fused into the load
        if (srgb) x = x <= 0.04045f ? x / 12.92f : powf((fmaxf(x, 0.04045f) + 0.055f) / 1.055f, 2.4f);
        v[e][c] = x;
      }
    }
#pragma unroll
    for (int c = 0; c < C; ++c) {
      float* dst = out + (((size_t)j * C + c) * Hp + y) * Wp + x4 * 4;
      if (vec) {
        *reinterpret_cast<float4*>(dst) = make_float4(v[0][c], v[1][c], v[2][c], v[3][c]);
      } else {
#pragma unroll
        for (int e = 0; e < 4; ++e)
          if (x4 * 4 + e < Wp) dst[e] = v[e][c];
      }
    }
  }
}

template <int C>
void launch_pack(const float* views, int m, int H, int W, int pad, float* out, int grid, int srgb, cudaStream_t st) {
  pack_pad_kernel<C><<<grid, 256, 0, st>>>(views, m, H, W, pad, out, srgb);
}

// sum over (C, Hp, Whp) of |b|^2 per view in float64, deterministic: SPLIT
// blocks per view write partials, a second kernel adds them in a fixed order.
constexpr int SUMSQ_SPLIT = 16;
__global__ void view_sumsq_partial_kernel(const float2* __restrict__ spec, size_t per_view,
                                          double* __restrict__ partial) {
  const int view = blockIdx.x / SUMSQ_SPLIT, part = blockIdx.x % SUMSQ_SPLIT;
  const size_t chunk = (per_view + SUMSQ_SPLIT - 1) / SUMSQ_SPLIT;
  const size_t b0 = (size_t)part * chunk, b1 = min(per_view, b0 + chunk);
  const float2* p = spec + (size_t)view * per_view;
  double acc = 0.0;
  for (size_t i = b0 + threadIdx.x; i < b1; i += blockDim.x) {
    const float2 b = p[i];
    acc += (double)b.x * b.x + (double)b.y * b.y;
  }
  __shared__ double red[32];
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x < 32) {
    double v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (threadIdx.x == 0) partial[blockIdx.x] = v;
  }
}

__global__ void view_sumsq_final_kernel(const double* __restrict__ partial, int m, double* __restrict__ out) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= m) return;
  double s = 0.0;
  for (int k = 0; k < SUMSQ_SPLIT; ++k) s += partial[(size_t)j * SUMSQ_SPLIT + k];
  out[j] = s;
}

__global__ void gather_rows_kernel(const float2* __restrict__ src, int planes, int Hp, int Whp,
                                   const int* __restrict__ rows, int nrows, float2* __restrict__ dst) {
  const size_t total = (size_t)planes * nrows * Whp;
  for (size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (size_t)gridDim.x * blockDim.x) {
    int kx = (int)(idx % Whp);
    size_t r = idx / Whp;
    int i = (int)(r % nrows);
    size_t pl = r / nrows;
    dst[idx] = src[(pl * Hp + rows[i]) * Whp + kx];
  }
}

// Project the kx = 0 (and even-W Nyquist) columns onto their Hermitian part,
// v <- (v + conj(v[flip_y])) / 2: exactly the input numpy's irfft2 inverts
// (its c2r pass drops the imaginary part of those columns after the y pass).
__global__ void hermitize_cols_kernel(float2* __restrict__ spec, int planes, int Hp, int Wp) {
  const int Whp = Wp / 2 + 1;
  const int ncols = (Wp % 2 == 0) ? 2 : 1;
  const int half = Hp / 2 + 1;  // rows 0..Hp/2 pair with Hp-row
  const size_t total = (size_t)planes * ncols * half;
  for (size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (size_t)gridDim.x * blockDim.x) {
    int ky = (int)(idx % half);
    size_t r = idx / half;
    int ci = (int)(r % ncols);
    size_t pl = r / ncols;
    int kx = ci == 0 ? 0 : Wp / 2;
    int my = (Hp - ky) % Hp;
    float2* base = spec + pl * (size_t)Hp * Whp;
    float2 a = base[(size_t)ky * Whp + kx];
    float2 b = base[(size_t)my * Whp + kx];
    float2 na = make_float2(0.5f * (a.x + b.x), 0.5f * (a.y - b.y));
    float2 nb = make_float2(na.x, -na.y);
    base[(size_t)ky * Whp + kx] = na;
    if (my != ky) base[(size_t)my * Whp + kx] = nb;
  }
}

__device__ inline float srgb_enc(float x) {
  // render.py:45-48 (negative inputs clamp to 0)
  x = fmaxf(x, 0.f);
  return x <= 0.0031308f ? x * 12.92f : 1.055f * powf(x, 1.0f / 2.4f) - 0.055f;
}

// (V, C, Hp, Wp) real planes scaled by 1/(Hp Wp) -> (V, Ho, Wo, C) cropped.
// One thread per output pixel: C coalesced plane reads, C contiguous writes.
template <int C>
__global__ void crop_kernel(const float* __restrict__ planes, int V, int Hp, int Wp, int pad, int Ho, int Wo,
                            int srgb, float scale, float* __restrict__ out) {
  const size_t total = (size_t)V * Ho * Wo;
  for (size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (size_t)gridDim.x * blockDim.x) {
    const int x = (int)(idx % Wo);
    const size_t r = idx / Wo;
    const int y = (int)(r % Ho);
    const int v = (int)(r / Ho);
    const float* src = planes + ((size_t)v * C * Hp + (y + pad)) * Wp + (x + pad);
#pragma unroll
    for (int c = 0; c < C; ++c) {
      float val = __ldg(src + (size_t)c * Hp * Wp) * scale;
      if (srgb) val = srgb_enc(val);
      out[idx * C + c] = val;
    }
  }
}

inline int grid_for(size_t total, int threads) {
  size_t b = (total + threads - 1) / threads;
  int sms = 148;
  size_t cap = (size_t)sms * 16;
  return (int)(b < cap ? (b > 0 ? b : 1) : cap);
}

// default_lambda (construct.py:214-216) from the per-view sums, added in view
// order by one thread: the same double operations, in the same order, as the
// host formula (construct.lambda_from_sumsq), so the value is bit-identical.
__global__ void default_lambda_kernel(const double* __restrict__ sums, int m, long long Q, double* __restrict__ lam) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double tot = 0.0;
  for (int j = 0; j < m; ++j) tot = __dadd_rn(tot, sums[j]);
  lam[0] = __ddiv_rn(__dmul_rn(1e-4, __ddiv_rn(tot, (double)Q)), (double)m);
}

}  // namespace

int default_lambda(const double* sums, int m, long long Q, double* lam, cudaStream_t st) {
  default_lambda_kernel<<<1, 32, 0, st>>>(sums, m, Q, lam);
  FDL_LAUNCH_CHECK("default_lambda_kernel");
  return FDL_OK;
}

int views_to_spectra_ws(int m, int H, int W, int C, int pad, size_t* bytes) {
  const int Hp = H + 2 * pad, Wp = W + 2 * pad;
  if (fft_engine_applies(Hp, Wp, C)) {
    *bytes = engine_fwd_ws(m, H, W, C, pad);
    return FDL_OK;
  }
  Plan* plan;
  int rc = get_plan(Hp, Wp, m * C, 0, &plan);
  if (rc) return rc;
  *bytes = align256((size_t)m * C * Hp * Wp * sizeof(float)) + align256(plan->work) +
           align256(sizeof(double) * (size_t)m * SUMSQ_SPLIT);
  return FDL_OK;
}

int views_to_spectra(const float* views, int m, int H, int W, int C, int pad, fdl_c64* spectra,
                     double* view_sumsq, void* ws, size_t ws_bytes, cudaStream_t st, int srgb) {
  const int Hp = H + 2 * pad, Wp = W + 2 * pad, Whp = Wp / 2 + 1;
  size_t need;
  int rc = views_to_spectra_ws(m, H, W, C, pad, &need);
  if (rc) return rc;
  if (ws_bytes < need || (need && !ws)) return fail(FDL_ERR_INVALID, "workspace too small for fdl_views_to_spectra");
  if (fft_engine_applies(Hp, Wp, C))
    return engine_fwd(views, m, H, W, C, pad, reinterpret_cast<float2*>(spectra), view_sumsq, ws, st, srgb);
  Plan* plan;
  get_plan(Hp, Wp, m * C, 0, &plan);
  float* padded = reinterpret_cast<float*>(ws);
  void* fft_work = reinterpret_cast<char*>(ws) + align256((size_t)m * C * Hp * Wp * sizeof(float));
  const int g = grid_for((size_t)m * Hp * ((Wp + 3) / 4), 256);
  switch (C) {
    case 1: launch_pack<1>(views, m, H, W, pad, padded, g, srgb, st); break;
    case 2: launch_pack<2>(views, m, H, W, pad, padded, g, srgb, st); break;
    case 3: launch_pack<3>(views, m, H, W, pad, padded, g, srgb, st); break;
    case 4: launch_pack<4>(views, m, H, W, pad, padded, g, srgb, st); break;
    default: return fail(FDL_ERR_UNSUPPORTED, "views support 1..4 channels");
  }
  FDL_LAUNCH_CHECK("pack_pad_kernel");
  if (cufftSetStream(plan->handle, st) != CUFFT_SUCCESS) return fail(FDL_ERR_CUDA, "cufftSetStream");
  if (cufftSetWorkArea(plan->handle, fft_work) != CUFFT_SUCCESS) return fail(FDL_ERR_CUDA, "cufftSetWorkArea");
  if (cufftExecR2C(plan->handle, padded, reinterpret_cast<cufftComplex*>(spectra)) != CUFFT_SUCCESS)
    return fail(FDL_ERR_CUDA, "cufftExecR2C failed");
  if (view_sumsq) {
    double* partial = reinterpret_cast<double*>(reinterpret_cast<char*>(fft_work) + align256(plan->work));
    view_sumsq_partial_kernel<<<m * SUMSQ_SPLIT, 512, 0, st>>>(reinterpret_cast<const float2*>(spectra),
                                                              (size_t)C * Hp * Whp, partial);
    FDL_LAUNCH_CHECK("view_sumsq_partial_kernel");
    view_sumsq_final_kernel<<<(m + 127) / 128, 128, 0, st>>>(partial, m, view_sumsq);
    FDL_LAUNCH_CHECK("view_sumsq_final_kernel");
  }
  return FDL_OK;
}

int gather_rows(const fdl_c64* src, int m, int C, int Hp, int Whp, const int* rows_dev, int nrows, fdl_c64* dst,
                cudaStream_t st) {
  size_t total = (size_t)m * C * nrows * Whp;
  if (total == 0) return FDL_OK;
  gather_rows_kernel<<<grid_for(total, 256), 256, 0, st>>>(reinterpret_cast<const float2*>(src), m * C, Hp, Whp,
                                                           rows_dev, nrows, reinterpret_cast<float2*>(dst));
  FDL_LAUNCH_CHECK("gather_rows_kernel");
  return FDL_OK;
}

int spectra_to_images_ws(int V, int C, int Hp, int Wp, size_t* bytes) {
  if (fft_engine_applies(Hp, Wp, C)) {
    *bytes = engine_inv_ws(V, C, Hp, Wp);
    return FDL_OK;
  }
  if (mr_engine_applies(Hp, Wp, C) && !fft_cufft_forced()) {
    *bytes = mr_engine_inv_ws(V, C, Hp, Wp);  // (the crop is not known here: Ho <= Hp)
    return FDL_OK;
  }
  Plan* plan;
  int rc = get_plan(Hp, Wp, V * C, 1, &plan);
  if (rc) return rc;
  *bytes = align256((size_t)V * C * Hp * Wp * sizeof(float)) + align256(plan->work);
  return FDL_OK;
}

int spectra_to_images(fdl_c64* spectra, int V, int C, int Hp, int Wp, int pad, int Ho, int Wo, int srgb,
                      float* images, void* ws, size_t ws_bytes, cudaStream_t st) {
  size_t need;
  int rc = spectra_to_images_ws(V, C, Hp, Wp, &need);
  if (rc) return rc;
  if (ws_bytes < need || !ws) return fail(FDL_ERR_INVALID, "workspace too small for fdl_spectra_to_images");
  if (pad < 0 || Ho + pad > Hp || Wo + pad > Wp) return fail(FDL_ERR_INVALID, "crop window outside the grid");
  if (fft_engine_applies(Hp, Wp, C))
    return engine_inv(reinterpret_cast<const float2*>(spectra), V, C, Hp, Wp, pad, Ho, Wo, srgb, images, ws, st);
  if (mr_engine_applies(Hp, Wp, C) && !fft_cufft_forced())
    return mr_engine_inv(reinterpret_cast<const float2*>(spectra), V, C, Hp, Wp, pad, Ho, Wo, srgb, images, ws, st);
  Plan* plan;
  get_plan(Hp, Wp, V * C, 1, &plan);
  float* planes = reinterpret_cast<float*>(ws);
  void* fft_work = reinterpret_cast<char*>(ws) + align256((size_t)V * C * Hp * Wp * sizeof(float));
  size_t hn = (size_t)V * C * ((Wp % 2 == 0) ? 2 : 1) * (Hp / 2 + 1);
  hermitize_cols_kernel<<<grid_for(hn, 256), 256, 0, st>>>(reinterpret_cast<float2*>(spectra), V * C, Hp, Wp);
  FDL_LAUNCH_CHECK("hermitize_cols_kernel");
  if (cufftSetStream(plan->handle, st) != CUFFT_SUCCESS) return fail(FDL_ERR_CUDA, "cufftSetStream");
  if (cufftSetWorkArea(plan->handle, fft_work) != CUFFT_SUCCESS) return fail(FDL_ERR_CUDA, "cufftSetWorkArea");
  if (cufftExecC2R(plan->handle, reinterpret_cast<cufftComplex*>(spectra), planes) != CUFFT_SUCCESS)
    return fail(FDL_ERR_CUDA, "cufftExecC2R failed");
  size_t total = (size_t)V * Ho * Wo;
  float scale = (float)(1.0 / ((double)Hp * (double)Wp));
  const int g = grid_for(total, 256);
  switch (C) {
    case 1: crop_kernel<1><<<g, 256, 0, st>>>(planes, V, Hp, Wp, pad, Ho, Wo, srgb, scale, images); break;
    case 2: crop_kernel<2><<<g, 256, 0, st>>>(planes, V, Hp, Wp, pad, Ho, Wo, srgb, scale, images); break;
    case 3: crop_kernel<3><<<g, 256, 0, st>>>(planes, V, Hp, Wp, pad, Ho, Wo, srgb, scale, images); break;
    case 4: crop_kernel<4><<<g, 256, 0, st>>>(planes, V, Hp, Wp, pad, Ho, Wo, srgb, scale, images); break;
    default: return fail(FDL_ERR_UNSUPPORTED, "images support 1..4 channels");
  }
  FDL_LAUNCH_CHECK("crop_kernel");
  return FDL_OK;
}

}  // namespace fdl
