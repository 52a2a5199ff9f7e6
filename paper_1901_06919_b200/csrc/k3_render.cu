// K3: batched render spectra (render.py:190-207, 238-245; lfmodel.py:101-122).
//
//   out[v, c, ky, kx] = sum_k L[k, c, ky, kx] * py_vk[ky] * px_vk[kx] * psi_v(t_vk wx, t_vk wy)
//
// The per-axis factors (phase exp(2 pi i P w) with cosine Nyquist lines, and
// the separable bilinear aperture indices/fractions) depend on one axis only,
// so a pre-pass evaluates them once per (view, layer, row|column) in float64
// and stores them as float32 (`AxisFactor`); the hot kernel then does, per
// (view, bin, layer), one complex product of the two axis phases, an optional
// 2x2 bilinear gather from the float32 table and the complex MAC over
// channels, all in float32 (>= 83 dB).
#include <cstdlib>

#include "common.cuh"
#include "k3_render.cuh"

namespace fdl {

namespace {

__global__ void render_factors_kernel(RenderParams p) {
  const int vk = blockIdx.x;  // v * n + k
  const int v = vk / p.n;
  const double P_u = p.pu[vk], P_v = p.pv[vk];
  const int ai = p.view_ap ? p.view_ap[v] : -1;
  const double t = (ai >= 0) ? p.t[vk] : 0.0;
  const bool even_w = (p.Wp % 2) == 0, even_h = (p.Hp % 2) == 0;
  AxisFactor* PX = p.px + (size_t)vk * p.Whp;
  AxisFactor* PY = p.py + (size_t)vk * p.Hp;
  // pinhole batches: view pairs interleaved, float2 phases: px2[(v/2, k, kx)][v&1]
  const bool pin = p.view_ap == nullptr;
  float2* PX2 = reinterpret_cast<float2*>(p.px) + (((size_t)(v >> 1) * p.n + (vk - v * p.n)) * p.Whp) * 2 + (v & 1);
  float2* PY2 = reinterpret_cast<float2*>(p.py) + (((size_t)(v >> 1) * p.n + (vk - v * p.n)) * p.Hp) * 2 + (v & 1);
  int bad_x = 0, bad_y = 0;
  for (int kx = threadIdx.x; kx < p.Whp; kx += blockDim.x) {
    const double ox = omega_x_label(kx, p.Wp);
    cd ph = axis_phase(P_u, ox, even_w && kx == p.Wp / 2);
    AxisFactor f;
    f.re = (float)ph.re;
    f.im = (float)ph.im;
    f.frac = 0.f;
    f.idx = 0;
    if (ai >= 0) {
      const DevAperture& ap = p.aps[ai];
      int i0;
      double fr;
      bool ok = axis_lookup(t * ox, ap.xi0_x, ap.step_x, ap.cols, i0, fr);
      f.idx = ok ? i0 : ap.rows * ap.cols;  // quad-table column; out of range -> the zero entry
      f.frac = (float)fr;
      bad_x += ok ? 0 : 1;
    }
    if (pin)
      PX2[2 * (size_t)kx] = make_float2(f.re, f.im);
    else
      PX[kx] = f;
  }
  for (int ky = threadIdx.x; ky < p.Hp; ky += blockDim.x) {
    const double oy = omega_y_label(ky, p.Hp);
    cd ph = axis_phase(P_v, oy, even_h && ky == p.Hp / 2);
    AxisFactor f;
    f.re = (float)ph.re;
    f.im = (float)ph.im;
    f.frac = 0.f;
    f.idx = 0;
    if (ai >= 0) {
      const DevAperture& ap = p.aps[ai];
      int i0;
      double fr;
      bool ok = axis_lookup(t * oy, ap.xi0_y, ap.step_y, ap.rows, i0, fr);
      f.idx = ok ? i0 * ap.cols : ap.rows * ap.cols;  // quad-table row offset
      f.frac = (float)fr;
      bad_y += ok ? 0 : 1;
    }
    if (pin)
      PY2[2 * (size_t)ky] = make_float2(f.re, f.im);
    else
      PY[ky] = f;
  }
  if (ai >= 0 && p.oob) {
    // lfmodel.py:118-121: n_oob = bad_rows * cols + ok_rows * bad_cols
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
      long long n_oob = (long long)sy * p.Whp + (long long)(p.Hp - sy) * sx;
      if (n_oob) atomicAdd(reinterpret_cast<unsigned long long*>(p.oob + v), (unsigned long long)n_oob);
    }
  }
}

// Tile kernel: CTA = 32 columns x 8 rows of bins for VB views; per layer k the
// (view, column) and (view, row) axis factors are staged in shared memory
// (double-buffered, one barrier per layer), each thread owns one bin and
// accumulates VB x C complex outputs in registers, and the layer values it
// needs for layer k+1 are prefetched while layer k is consumed.
constexpr int TX = 32, TY = 8;

__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gsrc, bool valid) {
  const unsigned dst = (unsigned)__cvta_generic_to_shared(smem_dst);
  const int src_size = valid ? 16 : 0;  // 0: zero-fill (weight 0)
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(gsrc), "r"(src_size));
}
__device__ __forceinline__ float2 ld_stream(const float2* p) {
  float2 v;
  asm volatile("ld.global.nc.L1::no_allocate.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "l"(p));
  return v;
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

constexpr int NSTAGE = 3;  // factor ring: layer k in use, k+1 and k+2 in flight

template <int C, int VB, bool AP, bool UNI>
__global__ void __launch_bounds__(TX * TY, (VB <= 8 && C <= 3) ? 3 : 2) render_tile_kernel(RenderParams p) {
  __shared__ __align__(16) AxisFactor FX[NSTAGE][VB][TX];
  __shared__ __align__(16) AxisFactor FY[NSTAGE][VB][TY];
  const int tx = threadIdx.x, ty = threadIdx.y, tid = ty * TX + tx;
  const int kx = blockIdx.y * TX + tx, ky = blockIdx.z * TY + ty;
  const int v0 = blockIdx.x * VB;
  const int nv = min(VB, p.V - v0);
  const long long Q = (long long)p.Hp * p.Whp;
  const bool inside = kx < p.Whp && ky < p.Hp;
  const long long q = inside ? (long long)ky * p.Whp + kx : 0;

  // asynchronous staging of layer k's VB*TX column + VB*TY row factors; entries
  // outside the grid / past the last view are zero-filled (weight 0), so the
  // compute loop runs branch-free for every thread and view slot
  auto stage = [&](int k) {
    const int buf = k % NSTAGE;
    for (int e = tid; e < VB * (TX + TY); e += TX * TY) {
      if (e < VB * TX) {
        const int b = e / TX, c = e % TX;
        const int col = blockIdx.y * TX + c;
        const bool ok = b < nv && col < p.Whp;
        cp_async16(&FX[buf][b][c], p.px + (ok ? ((size_t)(v0 + b) * p.n + k) * p.Whp + col : 0), ok);
      } else {
        const int e2 = e - VB * TX;
        const int b = e2 / TY, r = e2 % TY;
        const int row = blockIdx.z * TY + r;
        const bool ok = b < nv && row < p.Hp;
        cp_async16(&FY[buf][b][r], p.py + (ok ? ((size_t)(v0 + b) * p.n + k) * p.Hp + row : 0), ok);
      }
    }
    cp_async_commit();
  };

  __shared__ int TIDX[VB];
  __shared__ RenderTable TB[VB];
  if (tid < VB) {
    const int ai = (AP && tid < nv && p.view_ap) ? p.view_ap[v0 + tid] : -1;
    TIDX[tid] = ai;
    if (ai >= 0) TB[tid] = p.tables[ai];
  }
  RenderTable tb0{};
  if (UNI) tb0 = p.tables[p.uniform_ap];
  // (made visible by the first __syncthreads of the layer loop)

  u64 acc[VB][C];  // packed (re, im)
#pragma unroll
  for (int b = 0; b < VB; ++b)
#pragma unroll
    for (int c = 0; c < C; ++c) acc[b][c] = 0ull;

  float2 Lnext[C];
#pragma unroll
  for (int c = 0; c < C; ++c) Lnext[c] = inside ? ld_stream(p.layers + (size_t)c * Q + q) : make_float2(0.f, 0.f);
  stage(0);
  if (p.n > 1) stage(1);
  for (int k = 0; k < p.n; ++k) {
    const int buf = k % NSTAGE;
    cp_async_wait<0>();  // layers k and k+1 staged (k+1 was issued one layer ago)
    __syncthreads();     // ... and visible; everyone is done with layer k-1's buffer
    if (k + 2 < p.n) stage(k + 2);
    float2 L[C];
#pragma unroll
    for (int c = 0; c < C; ++c) L[c] = Lnext[c];
    if (k + 1 < p.n) {
#pragma unroll
      for (int c = 0; c < C; ++c)
        Lnext[c] = inside ? ld_stream(p.layers + ((size_t)(k + 1) * C + c) * Q + q) : make_float2(0.f, 0.f);
    }
    const AxisFactor* fxp = &FX[buf][0][tx];
    const AxisFactor* fyp = &FY[buf][0][ty];
#pragma unroll
    for (int b = 0; b < VB; ++b) {
      const AxisFactor fx = fxp[b * TX];
      const AxisFactor fy = fyp[b * TY];
      float wr = fy.re * fx.re - fy.im * fx.im;
      float wi = fy.re * fx.im + fy.im * fx.re;
      const int ai = UNI ? p.uniform_ap : (AP ? TIDX[b] : -1);
      if (AP && ai >= 0) {
        // one 16-byte quad-table load; out-of-range rows/columns hit the zero entry.
        // separable passes of lfmodel.py:115-116: rows (fy) first, then columns (fx)
        const RenderTable& tb = UNI ? tb0 : TB[b];
        const int qi = min(fy.idx + fx.idx, tb.zero);
        const float4 tr = __ldg(tb.re + qi);
        const float top = fmaf(fy.frac, tr.z - tr.x, tr.x);
        const float bot = fmaf(fy.frac, tr.w - tr.y, tr.y);
        const float sr = fmaf(fx.frac, bot - top, top);
        if (!UNI && tb.im) {
          const float4 ti = __ldg(tb.im + qi);
          const float tt = fmaf(fy.frac, ti.z - ti.x, ti.x);
          const float bb = fmaf(fy.frac, ti.w - ti.y, ti.y);
          const float si = fmaf(fx.frac, bb - tt, tt);
          const float nr = wr * sr - wi * si;
          wi = wr * si + wi * sr;
          wr = nr;
        } else {
          wr *= sr;
          wi *= sr;
        }
      }
#pragma unroll
      for (int c = 0; c < C; ++c) {
        cmac2(acc[b][c], wr, wi, L[c]);
      }
    }
    __syncthreads();  // buffer k % NSTAGE is refilled by stage(k + 3)
  }
  if (!inside) return;
#pragma unroll
  for (int b = 0; b < VB; ++b) {
    if (b >= nv) break;
#pragma unroll
    for (int c = 0; c < C; ++c) p.out[((size_t)(v0 + b) * C + c) * Q + q] = as_f2(acc[b][c]);
  }
}

// Pinhole tile kernel (no aperture in the batch): factors are view-pair
// interleaved float2 phases, so one 16-byte shared load serves two views and
// each layer's staging is one 16-byte cp.async per thread.
template <int C, int VB>
__global__ void __launch_bounds__(TX * TY, (VB <= 8 && C <= 3) ? 3 : 2) render_pin_kernel(RenderParams p) {
  constexpr int NP = VB / 2;
  __shared__ __align__(16) float4 FX2[NSTAGE][NP][TX];
  __shared__ __align__(16) float4 FY2[NSTAGE][NP][TY];
  const int tx = threadIdx.x, ty = threadIdx.y, tid = ty * TX + tx;
  const int kx = blockIdx.y * TX + tx, ky = blockIdx.z * TY + ty;
  const int v0 = blockIdx.x * VB;
  const int npairs = min(NP, (p.V - v0 + 1) / 2);
  const long long Q = (long long)p.Hp * p.Whp;
  const bool inside = kx < p.Whp && ky < p.Hp;
  const long long q = inside ? (long long)ky * p.Whp + kx : 0;
  const float4* PXG = reinterpret_cast<const float4*>(p.px);
  const float4* PYG = reinterpret_cast<const float4*>(p.py);
  const int pr0 = v0 / 2;

  // staging of one layer: NP*TX column pairs (one 16-byte cp.async per thread)
  // + NP*TY row pairs (threads < NP*TY); zero-filled outside the grid
  static_assert(NP * TX <= TX * TY, "at most one column-factor copy per thread");
  const int spr = tid / TX, sc = tid % TX;
  const int scol = blockIdx.y * TX + sc;
  const bool sxact = tid < NP * TX;
  const bool sxok = sxact && spr < npairs && scol < p.Whp;
  const float4* sx = PXG + (sxok ? (size_t)(pr0 + spr) * p.n * p.Whp + scol : 0);
  const int ypr = tid / TY, yr = tid % TY;
  const int srow = blockIdx.z * TY + yr;
  const bool syact = tid < NP * TY;
  const bool syok = syact && ypr < npairs && srow < p.Hp;
  const float4* sy = PYG + (syok ? (size_t)(pr0 + ypr) * p.n * p.Hp + srow : 0);
  auto stage = [&](int k) {
    const int buf = k % NSTAGE;
    if (sxact) cp_async16(&FX2[buf][spr][sc], sxok ? sx + (size_t)k * p.Whp : PXG, sxok);
    if (syact) cp_async16(&FY2[buf][ypr][yr], syok ? sy + (size_t)k * p.Hp : PYG, syok);
    cp_async_commit();
  };

  u64 acc[VB][C];  // packed (re, im): each complex MAC is two FFMA2
#pragma unroll
  for (int b = 0; b < VB; ++b)
#pragma unroll
    for (int c = 0; c < C; ++c) acc[b][c] = 0ull;
  float2 Lnext[C];
#pragma unroll
  for (int c = 0; c < C; ++c) Lnext[c] = inside ? ld_stream(p.layers + (size_t)c * Q + q) : make_float2(0.f, 0.f);
  stage(0);
  if (p.n > 1) stage(1);
  const float2* lp = p.layers + q;  // + (k * C + c) * Q
  for (int k = 0; k < p.n; ++k) {
    const int buf = k % NSTAGE;
    if (k + 1 < p.n) cp_async_wait<1>(); else cp_async_wait<0>();
    __syncthreads();  // layer k's factors visible; everyone is done with layer k-1's buffer
    if (k + 2 < p.n) stage(k + 2);  // refills the buffer of layer k-1
    float2 L[C];
#pragma unroll
    for (int c = 0; c < C; ++c) L[c] = Lnext[c];
    if (k + 1 < p.n) {
#pragma unroll
      for (int c = 0; c < C; ++c)
        Lnext[c] = inside ? ld_stream(lp + ((size_t)(k + 1) * C + c) * Q) : make_float2(0.f, 0.f);
    }
    const float4* fxp = &FX2[buf][0][tx];
    const float4* fyp = &FY2[buf][0][ty];
#pragma unroll
    for (int pr = 0; pr < NP; ++pr) {
      const float4 fx = fxp[pr * TX];
      const float4 fy = fyp[pr * TY];
      const float w0r = fy.x * fx.x - fy.y * fx.y, w0i = fy.x * fx.y + fy.y * fx.x;
      const float w1r = fy.z * fx.z - fy.w * fx.w, w1i = fy.z * fx.w + fy.w * fx.z;
#pragma unroll
      for (int c = 0; c < C; ++c) {
        cmac2(acc[2 * pr][c], w0r, w0i, L[c]);
        cmac2(acc[2 * pr + 1][c], w1r, w1i, L[c]);
      }
    }
  }
  if (!inside) return;
  const int nv = min(VB, p.V - v0);
#pragma unroll
  for (int b = 0; b < VB; ++b) {
    if (b >= nv) break;
#pragma unroll
    for (int c = 0; c < C; ++c) p.out[((size_t)(v0 + b) * C + c) * Q + q] = as_f2(acc[b][c]);
  }
}

template <int C, int VB>
void launch_ap(const RenderParams& p, dim3 grid, dim3 block, cudaStream_t st) {
  if (p.uniform_ap >= 0)  // every view on one real table
    render_tile_kernel<C, VB, true, true><<<grid, block, 0, st>>>(p);
  else  // mixed batch: per-view tables (real or complex)
    render_tile_kernel<C, VB, true, false><<<grid, block, 0, st>>>(p);
}

// views per thread of the render tiles: 16 for pinhole batches (register
// accumulators amortise the layer loads), 8 for aperture batches (occupancy
// hides the table-load latency: 4.5k vs 3.8k C5 views/s).  FDL_RENDER_VB overrides.
int render_vb_env(bool aperture) {
  const char* e = getenv("FDL_RENDER_VB");
  if (e) return atoi(e);
  return aperture ? 8 : 16;
}

template <int C>
int launch_sum(const RenderParams& p, cudaStream_t st) {
  constexpr int VB = C <= 3 ? 16 : 8;
  dim3 block(TX, TY);
  // view blocks vary fastest: the CTAs that share a layer tile run together and
  // re-read it from L2 instead of HBM (C4/C5 layers are GBs)
  dim3 grid((unsigned)((p.V + VB - 1) / VB), (unsigned)((p.Whp + TX - 1) / TX), (unsigned)((p.Hp + TY - 1) / TY));
  if (p.view_ap && VB == 16 && render_vb_env(true) == 8) {
    dim3 g8((unsigned)((p.V + 7) / 8), grid.y, grid.z);
    launch_ap<C, 8>(p, g8, block, st);
  } else if (p.view_ap) {
    launch_ap<C, VB>(p, grid, block, st);
  } else if (VB == 16 && render_vb_env(false) == 8) {
    dim3 g8((unsigned)((p.V + 7) / 8), grid.y, grid.z);
    render_pin_kernel<C, 8><<<g8, block, 0, st>>>(p);
  } else
    render_pin_kernel<C, VB><<<grid, block, 0, st>>>(p);
  FDL_LAUNCH_CHECK("render_tile_kernel");
  return FDL_OK;
}

}  // namespace

int render_launch(const RenderParams& p, cudaStream_t st) {
  if (p.V == 0) return FDL_OK;
  render_factors_kernel<<<p.V * p.n, 256, 0, st>>>(p);
  FDL_LAUNCH_CHECK("render_factors_kernel");
  switch (p.C) {
    case 1: return launch_sum<1>(p, st);
    case 2: return launch_sum<2>(p, st);
    case 3: return launch_sum<3>(p, st);
    case 4: return launch_sum<4>(p, st);
    default: return fail(FDL_ERR_UNSUPPORTED, "render supports 1..4 channels");
  }
}

}  // namespace fdl
