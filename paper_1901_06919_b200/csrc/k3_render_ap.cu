// K3 aperture tile (render.py:190-207 with lfmodel.py:101-122 lookups) for
// batches whose aperture tables are all real (C5: one disk table, 4096 views).
//
//   out[v, c, ky, kx] = sum_k L[k, c, ky, kx] * py_vk[ky] * px_vk[kx] * psi(t_vk wx, t_vk wy)
//
// The factor pre-pass (k3_render.cu: render_factors_kernel) leaves, per (view,
// layer), one 16-byte entry {re, im, frac, idx} per column and per row: the
// axis phase and that axis' half of the bilinear lookup (absolute entry index
// into the difference-form quad table `dquad`).  This kernel is the hot loop.
//
// CTA = NG groups of 256 threads over one tile of 32 columns x 8 rows of bins;
// group g accumulates views v0 + g VB .. + VB - 1 of the tile (one bin per
// thread, VB x C packed complex accumulators), so the NG groups read the same
// layer values (the second read hits L1).  The factors of KL layers arrive per
// stage as two TMA boxes ({32 columns, KL layers, NG VB views} of the (V, n,
// Whp) column-factor tensor, {8 rows, KL, NG VB} of the row-factor tensor) on a
// two-stage mbarrier ring: one elected thread issues them, out-of-grid columns,
// rows, layers and views are zero-filled by the TMA unit (weight 0), and no
// thread spends instructions on staging.  Per (view, bin, layer):
//   2 LDS.128 (factors)  1 VIADDMNMX + 1 LDG.128 (quad, L1-resident)
//   (A, B) = (a, b) + fy (c, d)                FFMA2
//   s = A + fx B                               FFMA
//   w = s * (py * px)                          FMUL2 + FFMA2 + FMUL2
//   acc_c += w * L_c, c < C                    2 FFMA2 per channel
// (the swapped / negated pair and the broadcast scalar are SASS operand
// modifiers of FFMA2, not instructions).
#include <cuda.h>

#include <algorithm>
#include <mutex>
#include <string>

#include "common.cuh"
#include "k3_render.cuh"
#include "tma.cuh"

namespace fdl {

namespace {

constexpr int TXA = 32, TYA = 8;  // bin tile
constexpr int KLA = 4;            // layers per TMA stage

// layer values stream through once per CTA: keep them out of L1, which the quad-table gathers need
__device__ __forceinline__ float2 ld_stream2(const float2* p) {
  float2 v;
  asm volatile("ld.global.nc.L1::no_allocate.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "l"(p));
  return v;
}

// (re, im) pair of a float4's first / second half as one packed operand
__device__ __forceinline__ u64 lo2(const float4& f) { return pack2(f.x, f.y); }
__device__ __forceinline__ u64 hi2(const float4& f) { return pack2(f.z, f.w); }
__device__ __forceinline__ u64 mul2s(u64 a, float s) {
  u64 r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(pack2(s, s)));
  return r;
}
// acc + i * a * s = acc + (-a.im, a.re) * s
__device__ __forceinline__ u64 fma2_i(u64 acc, u64 a, float s) {
  const float2 f = as_f2(a);
  u64 r = acc;
  ffma2(r, pack2(f.y, f.x), pack2(-s, s));
  return r;
}

template <int C, int VB, int NG>
struct ApCfg {
  static constexpr int NV = VB * NG;                          // views per CTA
  static constexpr int FX_STAGE = NV * KLA * TXA;             // float4 entries
  static constexpr int FY_STAGE = NV * KLA * TYA;
  static constexpr int STAGE_BYTES = 16 * (FX_STAGE + FY_STAGE);
  static constexpr int SMEM = 2 * STAGE_BYTES;
  static constexpr int THREADS = 256 * NG;
};

template <int C, int VB, int NG>
__global__ void __launch_bounds__(256 * NG, NG == 1 ? 2 : 1)
    render_ap_tma(RenderParams p, const __grid_constant__ CUtensorMap mapx, const __grid_constant__ CUtensorMap mapy) {
  using Cfg = ApCfg<C, VB, NG>;
  extern __shared__ __align__(128) float4 stage0[];  // TMA destinations: 128-byte aligned
  __shared__ __align__(8) unsigned long long full[2];
  const int tid = threadIdx.x;
  const int tx = tid & 31, ty = (tid >> 5) & 7, g = tid >> 8;
  const int kx0 = blockIdx.y * TXA, ky0 = blockIdx.z * TYA;
  const int kx = kx0 + tx, ky = ky0 + ty;
  const int v0 = blockIdx.x * Cfg::NV;
  const long long Q = (long long)p.Hp * p.Whp;
  const bool inside = kx < p.Whp && ky < p.Hp;
  const long long q = inside ? (long long)ky * p.Whp + kx : 0;
  const int nstages = (p.n + KLA - 1) / KLA;

  auto issue = [&](int s) {  // one thread: both boxes of stage s into buffer s & 1
    float4* dst = stage0 + (size_t)(s & 1) * (Cfg::FX_STAGE + Cfg::FY_STAGE);
    mbar_expect_tx(&full[s & 1], Cfg::STAGE_BYTES);
    tma_load_3d(dst, &mapx, kx0 * 4, s * KLA, v0, &full[s & 1]);
    tma_load_3d(dst + Cfg::FX_STAGE, &mapy, ky0 * 4, s * KLA, v0, &full[s & 1]);
  };
  if (tid == 0) {
    mbar_init(&full[0], 1);
    mbar_init(&full[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (tid == 0) {
    issue(0);
    if (nstages > 1) issue(1);
  }

  u64 acc[VB][C];
#pragma unroll
  for (int b = 0; b < VB; ++b)
#pragma unroll
    for (int c = 0; c < C; ++c) acc[b][c] = 0ull;

  const float4* __restrict__ DQ = p.dquad;
  const int zero = p.dq_zero;
  const float2* lp = p.layers + q;        // walks one layer (C planes) per step
  const long long lstep = (long long)C * Q;
  float2 Lnext[C];
#pragma unroll
  for (int c = 0; c < C; ++c) Lnext[c] = inside ? __ldg(lp + c * Q) : make_float2(0.f, 0.f);

  for (int s = 0; s < nstages; ++s) {
    const float4* FX = stage0 + (size_t)(s & 1) * (Cfg::FX_STAGE + Cfg::FY_STAGE) + (g * VB) * KLA * TXA + tx;
    const float4* FY = stage0 + (size_t)(s & 1) * (Cfg::FX_STAGE + Cfg::FY_STAGE) + Cfg::FX_STAGE +
                       (g * VB) * KLA * TYA + ty;
    mbar_wait(&full[s & 1], (s >> 1) & 1);
    const int kcount = min(KLA, p.n - s * KLA);
#pragma unroll
    for (int kl = 0; kl < KLA; ++kl) {
      if (kl < kcount) {
        float2 L[C];
#pragma unroll
        for (int c = 0; c < C; ++c) L[c] = Lnext[c];
        lp += lstep;
        if (s * KLA + kl + 1 < p.n) {
#pragma unroll
          for (int c = 0; c < C; ++c) Lnext[c] = inside ? __ldg(lp + c * Q) : make_float2(0.f, 0.f);
        }
#pragma unroll
        for (int b = 0; b < VB; ++b) {
          const float4 x = FX[(b * KLA + kl) * TXA];
          const float4 y = FY[(b * KLA + kl) * TYA];
          const int qi = min(__float_as_int(x.w) + __float_as_int(y.w), zero);
          const float4 T = __ldg(DQ + qi);
          u64 ab = lo2(T);
          ffma2(ab, hi2(T), pack2(y.z, y.z));          // (a, b) + fy (c, d)
          const float2 AB = as_f2(ab);
          const float sc = fmaf(x.z, AB.y, AB.x);      // psi
          u64 w = fma2_i(mul2s(lo2(y), x.x), lo2(y), x.y);  // py * px
          w = mul2s(w, sc);
#pragma unroll
          for (int c = 0; c < C; ++c) {
            ffma2(acc[b][c], w, pack2(L[c].x, L[c].x));
            acc[b][c] = fma2_i(acc[b][c], w, L[c].y);
          }
        }
      }
    }
    __syncthreads();  // every thread is done with buffer s & 1
    if (tid == 0 && s + 2 < nstages) issue(s + 2);
  }
  if (!inside) return;
#pragma unroll
  for (int b = 0; b < VB; ++b) {
    const int v = v0 + g * VB + b;
    if (v >= p.V) break;
#pragma unroll
    for (int c = 0; c < C; ++c) p.out[((size_t)v * C + c) * Q + q] = as_f2(acc[b][c]);
  }
}

// ---------------------------------------------------------------------------
// Affine variant (shifts affine in the layer index: factored u_v d_k with d an
// arithmetic progression -- config 5 and every `render` call).  The tile above
// is bound by the L1/shared data pipe (12 wavefronts per (view, bin, layer)
// warp-instruction group: 16-byte column and row factors + the 16-byte quad).
// Here the phase is generated instead of loaded:
//   x_vk(bin) = x_v0(bin) + k delta_v(bin)            [radians, one fp32 FFMA, no running sum]
//   w = (cos, sin)(x)                                 2 MUFU on the idle XU pipe (sin/cos.approx.ftz)
// so the factor entries shrink to the 8-byte lookup halves {frac, idx}: 2 + 1
// shared wavefronts instead of 4 + 2.  x_v0 and delta_v come from fp64
// (pu_v0 wx + pv_v0 wy, alpha_v wx + beta_v wy, wrapped to [-1/2, 1/2] turns, times
// 2 pi) once per thread and view; |x_vk| <= (2 n - 1) pi, where the MUFU's own range
// reduction is good to ~1.5e-5 rad (142 dB against the oracle at 1920 x 1080).
// The self-conjugate Nyquist column / row, whose phases are cosines
// (construct.py:68-80), are recomputed by render_ap_nyquist_fix.
// ---------------------------------------------------------------------------
constexpr int KLB = 8;  // layers per TMA stage of the 8-byte lookup entries

// row pitch of the 8-byte lookup tensors: even, so that rows are 16-byte aligned (TMA strides)
__host__ __device__ inline int even_pitch(int len) { return (len + 1) & ~1; }

// {frac, idx} halves of the bilinear lookups (lfmodel.py:101-122), fp64 index math:
// LX (V, n, Whp): idx = table base + column, LY (V, n, Hp): idx = row * cols;
// out-of-range -> the zero entry, pinhole views -> the (1, 0, 0, 0) entry.
// Also the out-of-range counts (lfmodel.py:118-121), as render_factors_kernel.
__global__ void render_lookup_kernel(RenderParams p, float2* __restrict__ LX, float2* __restrict__ LY) {
  const int vk = blockIdx.x;  // v * n + k
  const int v = vk / p.n;
  const int ai = p.view_ap[v];
  const double t = (ai >= 0) ? p.t[vk] : 0.0;
  float2* X = LX + (size_t)vk * even_pitch(p.Whp);
  float2* Y = LY + (size_t)vk * even_pitch(p.Hp);
  int bad_x = 0, bad_y = 0;
  for (int kx = threadIdx.x; kx < p.Whp; kx += blockDim.x) {
    float fr = 0.f;
    int idx = p.dq_one;
    if (ai >= 0) {
      const DevAperture& ap = p.aps[ai];
      int i0;
      double f;
      const bool ok = axis_lookup(t * omega_x_label(kx, p.Wp), ap.xi0_x, ap.step_x, ap.cols, i0, f);
      idx = ok ? p.ap_qbase[ai] + i0 : p.dq_zero;
      fr = (float)f;
      bad_x += ok ? 0 : 1;
    }
    X[kx] = make_float2(fr, __int_as_float(idx));
  }
  for (int ky = threadIdx.x; ky < p.Hp; ky += blockDim.x) {
    float fr = 0.f;
    int idx = 0;
    if (ai >= 0) {
      const DevAperture& ap = p.aps[ai];
      int i0;
      double f;
      const bool ok = axis_lookup(t * omega_y_label(ky, p.Hp), ap.xi0_y, ap.step_y, ap.rows, i0, f);
      idx = ok ? i0 * ap.cols : p.dq_zero;
      fr = (float)f;
      bad_y += ok ? 0 : 1;
    }
    Y[ky] = make_float2(fr, __int_as_float(idx));
  }
  if (ai >= 0 && p.oob) {
    __shared__ int sx, sy;
    if (threadIdx.x == 0) {
      sx = 0;
      sy = 0;
    }
    __syncthreads();
    atomicAdd(&sx, bad_x);
    atomicAdd(&sy, bad_y);
    __syncthreads();
    if (threadIdx.x == 0) {
      const long long n_oob = (long long)sy * p.Whp + (long long)(p.Hp - sy) * sx;
      if (n_oob) atomicAdd(reinterpret_cast<unsigned long long*>(p.oob + v), (unsigned long long)n_oob);
    }
  }
}

template <int C, int VB>
struct AffCfg {
  static constexpr int LX_STAGE = VB * KLB * TXA;  // float2 entries
  static constexpr int LY_STAGE = VB * KLB * TYA;
  static constexpr int STAGE_BYTES = 8 * (LX_STAGE + LY_STAGE);
  static constexpr int SMEM = 2 * STAGE_BYTES;
};

#ifndef FDL_AP_MINB
#define FDL_AP_MINB 2
#endif
#ifndef FDL_AP_VB3
#define FDL_AP_VB3 8
#endif
template <int C, int VB>
__global__ void __launch_bounds__(256, FDL_AP_MINB)
    render_ap_aff(RenderParams p, const __grid_constant__ CUtensorMap mapx, const __grid_constant__ CUtensorMap mapy) {
  using Cfg = AffCfg<C, VB>;
  extern __shared__ __align__(128) float2 stage8[];  // TMA destinations
  __shared__ __align__(8) unsigned long long full[2];
  const int tid = threadIdx.x;
  const int tx = tid & 31, ty = tid >> 5;
  const int kx0 = blockIdx.y * TXA, ky0 = blockIdx.z * TYA;
  const int kx = kx0 + tx, ky = ky0 + ty;
  const int v0 = blockIdx.x * VB;
  const long long Q = (long long)p.Hp * p.Whp;
  const bool inside = kx < p.Whp && ky < p.Hp;
  const long long q = inside ? (long long)ky * p.Whp + kx : 0;
  const int nstages = (p.n + KLB - 1) / KLB;

  auto issue = [&](int s) {
    float2* dst = stage8 + (size_t)(s & 1) * (Cfg::LX_STAGE + Cfg::LY_STAGE);
    mbar_expect_tx(&full[s & 1], Cfg::STAGE_BYTES);
    tma_load_3d(dst, &mapx, kx0 * 2, s * KLB, v0, &full[s & 1]);
    tma_load_3d(dst + Cfg::LX_STAGE, &mapy, ky0 * 2, s * KLB, v0, &full[s & 1]);
  };
  if (tid == 0) {
    mbar_init(&full[0], 1);
    mbar_init(&full[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (tid == 0) {
    issue(0);
    if (nstages > 1) issue(1);
  }

  // per view: phase of layer 0 and per-layer increment at this bin, in turns
  float th[VB], dl[VB];
  {
    const double ox = omega_x_label(min(kx, p.Whp - 1), p.Wp), oy = omega_y_label(min(ky, p.Hp - 1), p.Hp);
#pragma unroll
    for (int b = 0; b < VB; ++b) {
      const int v = min(v0 + b, p.V - 1);
      double t0 = p.pu[(size_t)v * p.n] * ox + p.pv[(size_t)v * p.n] * oy;
      double d0 = p.h_alpha[v] * ox + p.h_beta[v] * oy;
      t0 -= rint(t0);
      d0 -= rint(d0);
      // radians: x_k = th + k dl, |x_k| <= (2 n - 1) pi; one FFMA per (view, layer), no running sum
      dl[b] = (float)(6.283185307179586476925 * d0);
      th[b] = (float)(6.283185307179586476925 * t0);
    }
  }

  u64 acc[VB][C];
#pragma unroll
  for (int b = 0; b < VB; ++b)
#pragma unroll
    for (int c = 0; c < C; ++c) acc[b][c] = 0ull;

  const float4* __restrict__ DQ = p.dquad;
  const int zero = p.dq_zero;
  const float2* lp = p.layers + q;
  const long long lstep = (long long)C * Q;
  float2 Lnext[C];
#pragma unroll
  for (int c = 0; c < C; ++c) Lnext[c] = inside ? ld_stream2(lp + c * Q) : make_float2(0.f, 0.f);

  for (int s = 0; s < nstages; ++s) {
    const float2* LXs = stage8 + (size_t)(s & 1) * (Cfg::LX_STAGE + Cfg::LY_STAGE) + tx;
    const float2* LYs = stage8 + (size_t)(s & 1) * (Cfg::LX_STAGE + Cfg::LY_STAGE) + Cfg::LX_STAGE + ty;
    mbar_wait(&full[s & 1], (s >> 1) & 1);
    const int kcount = min(KLB, p.n - s * KLB);
#pragma unroll 2
    for (int kl = 0; kl < KLB; ++kl) {
      if (kl >= kcount) break;
      float2 L[C];
#pragma unroll
      for (int c = 0; c < C; ++c) L[c] = Lnext[c];
      lp += lstep;
      if (s * KLB + kl + 1 < p.n) {
#pragma unroll
        for (int c = 0; c < C; ++c) Lnext[c] = inside ? ld_stream2(lp + c * Q) : make_float2(0.f, 0.f);
      }
      const float kf = (float)(s * KLB + kl);
#pragma unroll
      for (int b = 0; b < VB; ++b) {
        const float2 x = LXs[(b * KLB + kl) * TXA];
        const float2 y = LYs[(b * KLB + kl) * TYA];
        const int qi = min(__float_as_int(x.y) + __float_as_int(y.y), zero);
        const float4 T = __ldg(DQ + qi);
        u64 ab = lo2(T);
        ffma2(ab, hi2(T), pack2(y.x, y.x));        // (a, b) + fy (c, d)
        const float2 AB = as_f2(ab);
        const float sc = fmaf(x.x, AB.y, AB.x);    // psi
        // MUFU range-reduces the argument itself (x / 2 pi in fp32: <= 1.5e-5 rad at |x| = 200)
        const float xk = fmaf(kf, dl[b], th[b]);
        float sn, cs;
        asm("sin.approx.ftz.f32 %0, %1;" : "=f"(sn) : "f"(xk));
        asm("cos.approx.ftz.f32 %0, %1;" : "=f"(cs) : "f"(xk));
        const u64 w = mul2s(pack2(cs, sn), sc);
#pragma unroll
        for (int c = 0; c < C; ++c) {
          ffma2(acc[b][c], w, pack2(L[c].x, L[c].x));
          acc[b][c] = fma2_i(acc[b][c], w, L[c].y);
        }
      }
    }
    __syncthreads();
    if (tid == 0 && s + 2 < nstages) issue(s + 2);
  }
  if (!inside) return;
#pragma unroll
  for (int b = 0; b < VB; ++b) {
    const int v = v0 + b;
    if (v >= p.V) break;
#pragma unroll
    for (int c = 0; c < C; ++c) p.out[((size_t)v * C + c) * Q + q] = as_f2(acc[b][c]);
  }
}

// Direct sums on the self-conjugate Nyquist column / row of an aperture batch
// (cosine phases, construct.py:68-80): one thread per (line bin, view), fp64
// phases by axis_phase, the tile's own lookup halves and quad table.
template <int C>
__global__ void render_ap_nyquist_fix(RenderParams p, const float2* __restrict__ LX, const float2* __restrict__ LY) {
  const int ncol = (p.Wp % 2 == 0) ? p.Hp : 0;   // kx = Wp/2, every row
  const int nrow = (p.Hp % 2 == 0) ? p.Whp : 0;  // ky = Hp/2, every column
  const int nl = ncol + nrow;
  const long long total = (long long)nl * p.V;
  const long long Q = (long long)p.Hp * p.Whp;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total; e += (long long)gridDim.x * blockDim.x) {
    const int v = (int)(e / nl), l = (int)(e - (long long)v * nl);
    const int kx = l < ncol ? p.Wp / 2 : l - ncol;
    const int ky = l < ncol ? l : p.Hp / 2;
    if (l >= ncol && (p.Wp % 2 == 0) && kx == p.Wp / 2) continue;  // the corner belongs to the column pass
    const bool nx = (p.Wp % 2 == 0) && kx == p.Wp / 2, ny = (p.Hp % 2 == 0) && ky == p.Hp / 2;
    const double ox = omega_x_label(kx, p.Wp), oy = omega_y_label(ky, p.Hp);
    float2 acc[C];
#pragma unroll
    for (int c = 0; c < C; ++c) acc[c] = make_float2(0.f, 0.f);
    const long long q = (long long)ky * p.Whp + kx;
    for (int k = 0; k < p.n; ++k) {
      const size_t vk = (size_t)v * p.n + k;
      const cd w64 = cmul(axis_phase(p.pu[vk], ox, nx), axis_phase(p.pv[vk], oy, ny));
      const float2 x = LX[vk * even_pitch(p.Whp) + kx], y = LY[vk * even_pitch(p.Hp) + ky];
      const float4 T = __ldg(p.dquad + min(__float_as_int(x.y) + __float_as_int(y.y), p.dq_zero));
      const float A = fmaf(y.x, T.z, T.x), B = fmaf(y.x, T.w, T.y);
      const float sc = fmaf(x.x, B, A);
      const float wr = (float)w64.re * sc, wi = (float)w64.im * sc;
#pragma unroll
      for (int c = 0; c < C; ++c) {
        const float2 Lv = __ldg(p.layers + ((size_t)k * C + c) * Q + q);
        acc[c].x = fmaf(wr, Lv.x, fmaf(-wi, Lv.y, acc[c].x));
        acc[c].y = fmaf(wr, Lv.y, fmaf(wi, Lv.x, acc[c].y));
      }
    }
#pragma unroll
    for (int c = 0; c < C; ++c) p.out[((size_t)v * C + c) * Q + q] = acc[c];
  }
}

// (V, n, len) tensor of `words`-float entries (4: {re, im, frac, idx}; 2: {frac, idx})
// as a 3-D fp32 tensor map with boxes of {tile entries, layers, nv views}
int factor_map(CUtensorMap* map, const void* base, int words, int len, int pitch, int n, int V, int tile, int layers,
               int nv) {
  EncodeTiledFn enc = encode_tiled_fn();
  if (!enc) return fail(FDL_ERR_CUDA, "cuTensorMapEncodeTiled is not available from this driver");
  const cuuint64_t gdim[3] = {(cuuint64_t)len * words, (cuuint64_t)n, (cuuint64_t)V};
  const cuuint64_t gstride[2] = {(cuuint64_t)pitch * words * 4, (cuuint64_t)n * pitch * words * 4};
  const cuuint32_t box[3] = {(cuuint32_t)tile * words, (cuuint32_t)layers, (cuuint32_t)nv};
  const cuuint32_t estr[3] = {1, 1, 1};
  const CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<void*>(base), gdim, gstride, box,
                         estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(FDL_ERR_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
  return FDL_OK;
}

template <int C, int VB, int NG>
int launch_cfg(const RenderParams& p, cudaStream_t st) {
  using Cfg = ApCfg<C, VB, NG>;
  CUtensorMap mx, my;
  if (int rc = factor_map(&mx, p.px, 4, p.Whp, p.Whp, p.n, p.V, TXA, KLA, Cfg::NV)) return rc;
  if (int rc = factor_map(&my, p.py, 4, p.Hp, p.Hp, p.n, p.V, TYA, KLA, Cfg::NV)) return rc;
  auto k = render_ap_tma<C, VB, NG>;
  FDL_CUDA_CHECK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM));
  dim3 grid((unsigned)((p.V + Cfg::NV - 1) / Cfg::NV), (unsigned)((p.Whp + TXA - 1) / TXA),
            (unsigned)((p.Hp + TYA - 1) / TYA));
  ktimer_mark(1, 0, st);
  k<<<grid, Cfg::THREADS, Cfg::SMEM, st>>>(p, mx, my);
  ktimer_mark(1, 1, st);
  FDL_LAUNCH_CHECK("render_ap_tma");
  return FDL_OK;
}

// affine batches: lookup pre-pass, generated-phase tile, Nyquist-line fix-up
template <int C, int VB>
int launch_aff(const RenderParams& p, cudaStream_t st) {
  using Cfg = AffCfg<C, VB>;
  float2* LX = reinterpret_cast<float2*>(p.px);  // the factor buffers hold the 8-byte entries
  float2* LY = reinterpret_cast<float2*>(p.py);
  render_lookup_kernel<<<p.V * p.n, 256, 0, st>>>(p, LX, LY);
  FDL_LAUNCH_CHECK("render_lookup_kernel");
  CUtensorMap mx, my;
  if (int rc = factor_map(&mx, LX, 2, p.Whp, even_pitch(p.Whp), p.n, p.V, TXA, KLB, VB)) return rc;
  if (int rc = factor_map(&my, LY, 2, p.Hp, even_pitch(p.Hp), p.n, p.V, TYA, KLB, VB)) return rc;
  auto k = render_ap_aff<C, VB>;
  FDL_CUDA_CHECK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM));
  dim3 grid((unsigned)((p.V + VB - 1) / VB), (unsigned)((p.Whp + TXA - 1) / TXA), (unsigned)((p.Hp + TYA - 1) / TYA));
  ktimer_mark(1, 0, st);
  k<<<grid, 256, Cfg::SMEM, st>>>(p, mx, my);
  ktimer_mark(1, 1, st);
  FDL_LAUNCH_CHECK("render_ap_aff");
  if ((p.Wp % 2 == 0) || (p.Hp % 2 == 0)) {
    const long long total = (long long)p.V * (p.Hp + p.Whp);
    const int blocks = (int)std::min<long long>((total + 127) / 128, 148LL * 16);
    render_ap_nyquist_fix<C><<<std::max(blocks, 1), 128, 0, st>>>(p, LX, LY);
    FDL_LAUNCH_CHECK("render_ap_nyquist_fix");
  }
  return FDL_OK;
}

template <int C> struct ApVB;
template <> struct ApVB<1> { static constexpr int vb = 12; };
template <> struct ApVB<2> { static constexpr int vb = 8; };
template <> struct ApVB<3> { static constexpr int vb = 8; };
template <> struct ApVB<4> { static constexpr int vb = 6; };

}  // namespace

// Real-table aperture batches (p.fast_ap).
int render_ap_launch(const RenderParams& p, cudaStream_t st) {
  if (!p.fast_ap || !p.view_ap) return fail(FDL_ERR_INVALID, "render_ap_launch: not a real-table aperture batch");
  // one view group per CTA: two groups sharing the layer reads through L1 measured
  // slower on C5 (33.0 vs 29.1 ms per 256 views: one 512-thread CTA per SM)
  if (p.horner) {
    switch (p.C) {
      case 1: return launch_aff<1, ApVB<1>::vb>(p, st);
      case 2: return launch_aff<2, ApVB<2>::vb>(p, st);
      case 3: return launch_aff<3, FDL_AP_VB3>(p, st);
      case 4: return launch_aff<4, ApVB<4>::vb>(p, st);
      default: return fail(FDL_ERR_UNSUPPORTED, "render supports 1..4 channels");
    }
  }
  switch (p.C) {
    case 1: return launch_cfg<1, ApVB<1>::vb, 1>(p, st);
    case 2: return launch_cfg<2, ApVB<2>::vb, 1>(p, st);
    case 3: return launch_cfg<3, ApVB<3>::vb, 1>(p, st);
    case 4: return launch_cfg<4, ApVB<4>::vb, 1>(p, st);
    default: return fail(FDL_ERR_UNSUPPORTED, "render supports 1..4 channels");
  }
}

}  // namespace fdl
