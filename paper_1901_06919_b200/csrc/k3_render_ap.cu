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

#include <mutex>
#include <string>

#include "common.cuh"
#include "k3_render.cuh"

namespace fdl {

namespace {

constexpr int TXA = 32, TYA = 8;  // bin tile
constexpr int KLA = 4;            // layers per TMA stage

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  unsigned ok;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  } while (!ok);
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int c0, int c1, int c2,
                                            unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
      ::"r"(smem_u32(dst)), "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
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

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_tiled_fn() {
  static std::once_flag once;
  static EncodeTiledFn fn = nullptr;
  std::call_once(once, [] {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult qres;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &qres) == cudaSuccess &&
        qres == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(ptr);
  });
  return fn;
}

// (V, n, len) tensor of 16-byte factor entries as a 3-D fp32 tensor map with
// boxes of {tile entries, KLA layers, nv views}
int factor_map(CUtensorMap* map, const AxisFactor* base, int len, int n, int V, int tile, int nv) {
  EncodeTiledFn enc = encode_tiled_fn();
  if (!enc) return fail(FDL_ERR_CUDA, "cuTensorMapEncodeTiled is not available from this driver");
  const cuuint64_t gdim[3] = {(cuuint64_t)len * 4, (cuuint64_t)n, (cuuint64_t)V};
  const cuuint64_t gstride[2] = {(cuuint64_t)len * 16, (cuuint64_t)n * len * 16};
  const cuuint32_t box[3] = {(cuuint32_t)tile * 4, (cuuint32_t)KLA, (cuuint32_t)nv};
  const cuuint32_t estr[3] = {1, 1, 1};
  const CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<AxisFactor*>(base), gdim, gstride, box,
                         estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(FDL_ERR_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
  return FDL_OK;
}

template <int C, int VB, int NG>
int launch_cfg(const RenderParams& p, cudaStream_t st) {
  using Cfg = ApCfg<C, VB, NG>;
  CUtensorMap mx, my;
  if (int rc = factor_map(&mx, p.px, p.Whp, p.n, p.V, TXA, Cfg::NV)) return rc;
  if (int rc = factor_map(&my, p.py, p.Hp, p.n, p.V, TYA, Cfg::NV)) return rc;
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
  switch (p.C) {
    case 1: return launch_cfg<1, ApVB<1>::vb, 1>(p, st);
    case 2: return launch_cfg<2, ApVB<2>::vb, 1>(p, st);
    case 3: return launch_cfg<3, ApVB<3>::vb, 1>(p, st);
    case 4: return launch_cfg<4, ApVB<4>::vb, 1>(p, st);
    default: return fail(FDL_ERR_UNSUPPORTED, "render supports 1..4 channels");
  }
}

}  // namespace fdl
