// K4 on the mixed-radix shared-memory FFT (fft_mr.cuh) for grids whose sides are
// in the plan list below (config 5: 1920 x 1080, either orientation):
//   cols pass : inverse column FFTs of a tile of CB adjacent columns of one plane,
//               only the cropped rows stored -> T2 (V, C, Ho, Whp) c64
//   rows pass : Hermitian completion of two rows (imaginary parts of the kx = 0 and
//               Nyquist columns dropped, as numpy's irfft does, spectra.py:202-208),
//               one complex inverse FFT, 1/(Hp Wp), crop, sRGB (render.py:210-225)
//               -> images (V, Ho, Wo, C) f32, channel-interleaved stores
// Two HBM passes in place of cuFFT's six kernels plus a crop kernel.
// Persistent CTAs, two per SM; the next tile's lines are prefetched into L2.
#include <algorithm>

#include "common.cuh"
#include "fft_mr.cuh"

namespace fdl {

namespace {

__device__ inline float srgb_enc_mr(float x) {
  x = fmaxf(x, 0.f);
  return x <= 0.0031308f ? x * 12.92f : 1.055f * powf(x, 1.0f / 2.4f) - 0.055f;
}

// ---------------------------------------------------------------- columns
// COL_THREADS is a multiple of every column-tile width, so a thread keeps one
// column of the tile and walks its rows with a fixed pointer step.
constexpr int COL_THREADS = 240;
constexpr int ROW_THREADS = 256;

template <class PL, int CB>
struct ColCfg {
  static constexpr int SMEM = 8 * (PL::TW + PL::N * CB);  // twiddle tables + [n][b] tile
};

template <class PL, int CB>
__global__ void __launch_bounds__(COL_THREADS, 2) mr_inv_cols_kernel(const float2* __restrict__ spec, int planes, int Whp,
                                                                     int pad, int Ho, float2* __restrict__ t2) {
  constexpr int N = PL::N, RSTEP = COL_THREADS / CB;
  static_assert(COL_THREADS % CB == 0, "one column per thread");
  extern __shared__ __align__(16) float2 smem_mr[];
  float2* tw = smem_mr;
  float2* buf = smem_mr + PL::TW;
  mr::build_roots<PL, true>(tw);
  const int cblocks = (Whp + CB - 1) / CB;
  const int items = planes * cblocks;
  const int b = threadIdx.x % CB, r0 = threadIdx.x / CB;
  for (int item = blockIdx.x; item < items; item += gridDim.x) {
    const int pl = item / cblocks, kx0 = (item - pl * cblocks) * CB;
    const bool colok = kx0 + b < Whp;
    __syncthreads();  // tables built (first tile) / the previous tile's stores have read the buffer
    {
      // the whole tile by asynchronous 8-byte copies: every row of this thread's
      // column is in flight at once (no registers held), zero-filled past the grid
      const float2* src = spec + ((size_t)pl * N + r0) * Whp + kx0 + (colok ? b : 0);
      float2* dstp = buf + r0 * CB + b;
      const size_t gstep = (size_t)RSTEP * Whp;
#pragma unroll 6
      for (int row = r0; row < N; row += RSTEP, src += gstep, dstp += RSTEP * CB) cpa8(dstp, src, colok);
      cpa_commit();
      cpa_wait_all();
    }
    __syncthreads();
    mr::transform<PL, mr::COLS, CB, true>(buf, tw);
    __syncthreads();
    if (colok) {
      float2* dst = t2 + ((size_t)pl * Ho + r0) * Whp + kx0 + b;
      const size_t gstep = (size_t)RSTEP * Whp;
#pragma unroll 4
      for (int y = r0; y < Ho; y += RSTEP, dst += gstep) *dst = buf[PL::where(y + pad) * CB + b];
    }
  }
}

// ---------------------------------------------------------------- rows
// A tile is RB transforms; transform tr -> (view, row pair, channel), channel
// fastest, and RB is a multiple of C, so a tile holds whole pixels and the
// image stores are contiguous.
template <class PL, int RB>
struct RowCfg {
  static constexpr int SMEM = 8 * (PL::TW + RB * PL::NP);
};

template <class PL, int RB, int C>
__global__ void __launch_bounds__(ROW_THREADS, 2) mr_inv_rows_kernel(const float2* __restrict__ t2, int V, int Ho,
                                                                     int Wo, int pad, int srgb, float scale,
                                                                     float* __restrict__ out) {
  constexpr int N = PL::N, Whp = N / 2 + 1, NP = PL::NP, GROUPS = RB / C;
  static_assert(RB % C == 0, "whole pixels per tile");
  extern __shared__ __align__(16) float2 smem_mr[];
  float2* tw = smem_mr;
  float2* buf = smem_mr + PL::TW;
  mr::build_roots<PL, true>(tw);
  const int HP2 = (Ho + 1) / 2;
  const int ngroups = V * HP2;  // (view, row pair)
  const int items = (ngroups + GROUPS - 1) / GROUPS;
  for (int item = blockIdx.x; item < items; item += gridDim.x) {
    __syncthreads();
    // Hermitian completion: Z[k] = X[k] + i Y[k], Z[N-k] = conj X[k] + i conj Y[k].
    // Per sweep of k the loads of all RB vectors are issued before any is used.
    {
      const float2* rowp[RB];
      bool ok1[RB];
#pragma unroll
      for (int bb = 0; bb < RB; ++bb) {
        const int grp = item * GROUPS + bb / C, c = bb % C;
        const bool ok = grp < ngroups;
        const int v = ok ? grp / HP2 : 0, y0 = ok ? 2 * (grp - v * HP2) : 0;
        rowp[bb] = ok ? t2 + (((size_t)v * C + c) * Ho + y0) * Whp : nullptr;
        ok1[bb] = ok && y0 + 1 < Ho;
      }
      for (int k = threadIdx.x; k < Whp; k += ROW_THREADS) {
        float2 X[RB], Y[RB];
#pragma unroll
        for (int bb = 0; bb < RB; ++bb) {
          X[bb] = rowp[bb] ? __ldg(rowp[bb] + k) : make_float2(0.f, 0.f);
          Y[bb] = ok1[bb] ? __ldg(rowp[bb] + Whp + k) : make_float2(0.f, 0.f);
        }
        const bool self = k == 0 || 2 * k == N;  // self-conjugate columns: real parts only
        const int pk = PL::phys(k), pm = PL::phys(N - k);
#pragma unroll
        for (int bb = 0; bb < RB; ++bb) {
          if (self) {
            X[bb].y = 0.f;
            Y[bb].y = 0.f;
          }
          float2* vb = buf + bb * NP;
          vb[pk] = make_float2(X[bb].x - Y[bb].y, X[bb].y + Y[bb].x);
          if (!self) vb[pm] = make_float2(X[bb].x + Y[bb].y, Y[bb].x - X[bb].y);
        }
      }
    }
    __syncthreads();
    {  // next tile's input rows into L2
#pragma unroll 1
      for (int bb = 0; bb < RB; ++bb) {
        const int grp = (item + gridDim.x) * GROUPS + bb / C, c = bb % C;
        if (grp >= ngroups) break;
        const int v = grp / HP2, y0 = 2 * (grp - v * HP2);
        const float2* i0 = t2 + (((size_t)v * C + c) * Ho + y0) * Whp;
        for (int e = threadIdx.x * 16; e < 2 * Whp; e += 16 * ROW_THREADS) prefetch_l2(i0 + e);
      }
    }
    mr::transform<PL, mr::ROWS, RB, true>(buf, tw);
    __syncthreads();
    // pixel (g, x, c) of the tile: lanes run over (x, c), c fastest -> contiguous stores
    const int per_group = Wo * C;
#pragma unroll 1
    for (int g = 0; g < GROUPS; ++g) {
      const int grp = item * GROUPS + g;
      if (grp >= ngroups) break;
      const int v = grp / HP2, y0 = 2 * (grp - v * HP2);
      const bool has1 = y0 + 1 < Ho;
      float* o0 = out + ((size_t)v * Ho + y0) * per_group;
      const float2* gb = buf + g * C * NP;
      for (int e = threadIdx.x; e < per_group; e += ROW_THREADS) {
        const int x = e / C, c = e - x * C;
        const float2 z = gb[c * NP + PL::phys_where(x + pad)];
        float a0 = z.x * scale, a1 = z.y * scale;
        if (srgb) {
          a0 = srgb_enc_mr(a0);
          a1 = srgb_enc_mr(a1);
        }
        o0[e] = a0;
        if (has1) o0[per_group + e] = a1;
      }
    }
  }
}

int sm_count_mr() {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms > 0 ? sms : 148;
}

// sides with a plan (keep with_mr_plan and mr_side in sync)
using P1080 = mr::Plan<1080, 8, 9, 15>;
using P1920 = mr::Plan<1920, 16, 8, 15>;

template <class F>
int with_mr_plan(int N, F&& f) {
  switch (N) {
    case 1080: return f(P1080());
    case 1920: return f(P1920());
    default: return fail(FDL_ERR_UNSUPPORTED, "mixed-radix FFT: unsupported side");
  }
}

bool mr_side(int N) { return N == 1080 || N == 1920; }

// columns per tile: two CTAs per SM (N = 1080: 12 columns, 112 KB per CTA)
template <class PL>
constexpr int col_tile() { return PL::N <= 1100 ? 12 : 6; }

template <class PL, int RB, int C>
int launch_rows(const float2* t2, int V, int Ho, int Wo, int pad, int srgb, float scale, float* images,
                cudaStream_t st) {
  auto k = mr_inv_rows_kernel<PL, RB, C>;
  FDL_CUDA_CHECK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, RowCfg<PL, RB>::SMEM));
  const int items = (V * ((Ho + 1) / 2) + RB / C - 1) / (RB / C);
  const int grid = std::max(1, std::min(2 * sm_count_mr(), items));
  k<<<grid, ROW_THREADS, RowCfg<PL, RB>::SMEM, st>>>(t2, V, Ho, Wo, pad, srgb, scale, images);
  FDL_LAUNCH_CHECK("mr_inv_rows_kernel");
  return FDL_OK;
}

}  // namespace

bool mr_engine_applies(int Hp, int Wp, int C) { return C >= 1 && C <= 4 && mr_side(Hp) && mr_side(Wp); }

size_t mr_engine_inv_ws(int V, int C, int Ho, int Wp) {
  return (sizeof(float2) * (size_t)V * C * Ho * (Wp / 2 + 1) + 255) & ~(size_t)255;
}

int mr_engine_inv(const float2* spectra, int V, int C, int Hp, int Wp, int pad, int Ho, int Wo, int srgb, float* images,
                  void* ws, cudaStream_t st) {
  const int Whp = Wp / 2 + 1;
  float2* t2 = reinterpret_cast<float2*>(ws);
  const float scale = (float)(1.0 / ((double)Hp * (double)Wp));
  int rc = with_mr_plan(Hp, [&](auto pl) {
    using PL = decltype(pl);
    constexpr int COL_TILE = col_tile<PL>();
    auto k = mr_inv_cols_kernel<PL, COL_TILE>;
    constexpr int smem = ColCfg<PL, COL_TILE>::SMEM;
    static_assert(2 * smem <= 227 * 1024, "two CTAs per SM");
    FDL_CUDA_CHECK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    const int items = V * C * ((Whp + COL_TILE - 1) / COL_TILE);
    const int grid = std::max(1, std::min(2 * sm_count_mr(), items));
    k<<<grid, COL_THREADS, smem, st>>>(spectra, V * C, Whp, pad, Ho, t2);
    FDL_LAUNCH_CHECK("mr_inv_cols_kernel");
    return FDL_OK;
  });
  if (rc) return rc;
  return with_mr_plan(Wp, [&](auto pl) {
    using PL = decltype(pl);
    switch (C) {
      case 1: return launch_rows<PL, 6, 1>(t2, V, Ho, Wo, pad, srgb, scale, images, st);
      case 2: return launch_rows<PL, 6, 2>(t2, V, Ho, Wo, pad, srgb, scale, images, st);
      case 3: return launch_rows<PL, 6, 3>(t2, V, Ho, Wo, pad, srgb, scale, images, st);
      default: return launch_rows<PL, 4, 4>(t2, V, Ho, Wo, pad, srgb, scale, images, st);
    }
  });
}

}  // namespace fdl
