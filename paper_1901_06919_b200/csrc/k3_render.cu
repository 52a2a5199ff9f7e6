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
#include <algorithm>
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
    f.idx = p.fast_ap ? p.dq_one : 0;
    if (ai >= 0) {
      const DevAperture& ap = p.aps[ai];
      int i0;
      double fr;
      bool ok = axis_lookup(t * ox, ap.xi0_x, ap.step_x, ap.cols, i0, fr);
      if (p.fast_ap)
        f.idx = ok ? p.ap_qbase[ai] + i0 : p.dq_zero;
      else
        f.idx = ok ? i0 : ap.rows * ap.cols;  // quad-table column; out of range -> the zero entry
      f.frac = (float)fr;
      bad_x += ok ? 0 : 1;
    }
    if (pin)
      PX2[2 * (size_t)kx] = make_float2(f.re, f.im);
    else if (p.aux8)
      reinterpret_cast<float2*>(p.px)[(size_t)vk * p.Whp + kx] = make_float2(f.frac, __int_as_float(f.idx));
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
      if (p.fast_ap)
        f.idx = ok ? i0 * ap.cols : p.dq_zero;
      else
        f.idx = ok ? i0 * ap.cols : ap.rows * ap.cols;  // quad-table row offset
      f.frac = (float)fr;
      bad_y += ok ? 0 : 1;
    }
    if (pin)
      PY2[2 * (size_t)ky] = make_float2(f.re, f.im);
    else if (p.aux8)
      reinterpret_cast<float2*>(p.py)[(size_t)vk * p.Hp + ky] = make_float2(f.frac, __int_as_float(f.idx));
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

// ---------------------------------------------------------------------------
// Fast tiles.  CTA = 256 threads over 32 columns x 8 rows of bins; each warp
// covers 8 columns x 4 rows, so a warp's per-(view, layer) column factors are 8
// distinct 16-byte words and its row factors 4 (one shared-memory wavefront
// each, the rest broadcast).  All per-(view, bin, layer) arithmetic is packed
// fp32 (FFMA2/FMUL2 with a broadcast scalar operand):
//   pinhole:  w = py * px                          FMUL2 + FFMA2
//   aperture: (A, B) = (a, b) + fy (c, d)          FFMA2
//             s = A + fx B                         FFMA
//             w = s * (py * px)                    FMUL2 + FFMA2 + FMUL2
//   each channel: acc += w * L                     2 FFMA2
// ---------------------------------------------------------------------------
constexpr int FX_T = 32, FY_T = 8;

__device__ __forceinline__ u64 fmul2s(u64 a, float s) {
  u64 r, ss;
  asm("mov.b64 %0, {%1, %1};" : "=l"(ss) : "f"(s));
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(ss));
  return r;
}
// acc + (-a.y, a.x) * s   (i * a * s)
__device__ __forceinline__ u64 ffma2_i(u64 acc, u64 a, float s) {
  const float2 f = as_f2(a);
  u64 r = acc;
  ffma2s(r, pack2(-f.y, f.x), s);
  return r;
}
// complex product of two (re, im) pairs, packed: x * y
__device__ __forceinline__ u64 cmul2(float2 x, float2 y) {
  return ffma2_i(fmul2s(pack2(x.x, x.y), y.x), pack2(x.x, x.y), y.y);
}
// acc += w * L  (two FFMA2, L components broadcast)
__device__ __forceinline__ void cmac_w(u64& acc, u64 w, float2 L) {
  ffma2s(acc, w, L.x);
  acc = ffma2_i(acc, w, L.y);
}

__device__ __forceinline__ int fast_col(int tid) { return ((tid >> 5) & 3) * 8 + (tid & 7); }
__device__ __forceinline__ int fast_row(int tid) { return (tid >> 7) * 4 + ((tid >> 3) & 3); }

// 8-byte asynchronous copy (layer values: rows of an odd-width half spectrum
// are not 16-byte aligned); zero-filled when !valid
__device__ __forceinline__ void cp_async8(void* smem_dst, const void* gsrc, bool valid) {
  const unsigned dst = (unsigned)__cvta_generic_to_shared(smem_dst);
  const int src_size = valid ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(dst), "l"(gsrc), "r"(src_size));
}

// pinhole batch: view-pair interleaved phases (same factor layout as render_pin_kernel).
// Per-layer staging: every thread copies its own bin's C layer values and
// XPT column-factor / at most one row-factor 16-byte word into ring slot
// k % NSTAGE; source pointers are formed once, a layer step adds a stride.
template <int C, int VB>
__global__ void __launch_bounds__(256, 2) render_pin_fast(RenderParams p) {
  constexpr int NP = VB / 2;
  static_assert(NP * FY_T <= 256, "one row-factor copy per thread");
  constexpr int XPT = (NP * FX_T + 255) / 256;
  struct __align__(16) Slot {
    float4 fx[NP][FX_T];
    float4 fy[NP][FY_T];
    float2 L[C][256];
  };
  __shared__ Slot S[NSTAGE];
  const int tid = threadIdx.x;
  const int lx = fast_col(tid), ly = fast_row(tid);
  const int kx = blockIdx.y * FX_T + lx, ky = blockIdx.z * FY_T + ly;
  const int v0 = blockIdx.x * VB;
  const int npairs = min(NP, (p.V - v0 + 1) / 2);
  const long long Q = (long long)p.Hp * p.Whp;
  const bool inside = kx < p.Whp && ky < p.Hp;
  const long long q = inside ? (long long)ky * p.Whp + kx : 0;
  const float4* PXG = reinterpret_cast<const float4*>(p.px);
  const float4* PYG = reinterpret_cast<const float4*>(p.py);

  const char* xsrc[XPT];
  int xdst[XPT];
  bool xok[XPT], xact[XPT];
#pragma unroll
  for (int i = 0; i < XPT; ++i) {
    const int e = tid + 256 * i;
    const int pr = e / FX_T, c = e % FX_T, col = blockIdx.y * FX_T + c;
    xact[i] = e < NP * FX_T;
    xok[i] = xact[i] && pr < npairs && col < p.Whp;
    xsrc[i] = reinterpret_cast<const char*>(PXG + (xok[i] ? (size_t)(v0 / 2 + pr) * p.n * p.Whp + col : 0));
    xdst[i] = (int)((char*)&S[0].fx[pr % NP][c] - (char*)&S[0]);
  }
  const long long xstep = (long long)p.Whp * 16;
  const int ypr = tid / FY_T, yr = tid % FY_T, row = blockIdx.z * FY_T + yr;
  const bool yact = tid < NP * FY_T;
  const bool yok = yact && ypr < npairs && row < p.Hp;
  const char* ysrc = reinterpret_cast<const char*>(PYG + (yok ? (size_t)(v0 / 2 + ypr) * p.n * p.Hp + row : 0));
  const long long ystep = (long long)p.Hp * 16;
  const int ydst = (int)((char*)&S[0].fy[ypr % NP][yr] - (char*)&S[0]);
  const float2* lsrc0 = p.layers + q;
  const long long lstep = inside ? (long long)C * Q : 0;
  auto stage = [&](int k) {
    char* base = reinterpret_cast<char*>(&S[k % NSTAGE]);
#pragma unroll
    for (int i = 0; i < XPT; ++i)
      if (xact[i]) cp_async16(base + xdst[i], xsrc[i] + (xok[i] ? k * xstep : 0), xok[i]);
    if (yact) cp_async16(base + ydst, ysrc + (yok ? k * ystep : 0), yok);
    const float2* ls = lsrc0 + k * lstep;
#pragma unroll
    for (int c = 0; c < C; ++c) cp_async8(&S[k % NSTAGE].L[c][tid], ls + c * Q, inside);
    cp_async_commit();
  };

  u64 acc[VB][C];
#pragma unroll
  for (int b = 0; b < VB; ++b)
#pragma unroll
    for (int c = 0; c < C; ++c) acc[b][c] = 0ull;
  stage(0);
  if (p.n > 1) stage(1);
  for (int k = 0; k < p.n; ++k) {
    const Slot& sl = S[k % NSTAGE];
    if (k + 1 < p.n) cp_async_wait<1>(); else cp_async_wait<0>();
    __syncthreads();  // layer k visible; everyone is done with layer k-1's slot
    if (k + 2 < p.n) stage(k + 2);
    float2 L[C];
#pragma unroll
    for (int c = 0; c < C; ++c) L[c] = sl.L[c][tid];
    float4 x = sl.fx[0][lx], y = sl.fy[0][ly];
#pragma unroll
    for (int pr = 0; pr < NP; ++pr) {
      float4 xn, yn;
      if (pr + 1 < NP) {
        xn = sl.fx[pr + 1][lx];
        yn = sl.fy[pr + 1][ly];
      }
      const u64 w0 = cmul2(make_float2(x.x, x.y), make_float2(y.x, y.y));
      const u64 w1 = cmul2(make_float2(x.z, x.w), make_float2(y.z, y.w));
#pragma unroll
      for (int c = 0; c < C; ++c) {
        cmac_w(acc[2 * pr][c], w0, L[c]);
        cmac_w(acc[2 * pr + 1][c], w1, L[c]);
      }
      if (pr + 1 < NP) {
        x = xn;
        y = yn;
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

// real-table batch (any mix of real apertures and pinhole views): per-view
// factors {re, im, frac, absolute idx}; the 2x2 quad of (view b, layer k+1)
// is gathered into registers while layer k is consumed.
template <int C, int VB>
__global__ void __launch_bounds__(256, 2) render_ap_fast(RenderParams p) {
  static_assert(VB * FY_T <= 256, "one row-factor copy per thread");
  constexpr int XPT = (VB * FX_T + 255) / 256;  // column-factor copies per thread
  struct __align__(16) Slot {
    AxisFactor fx[VB][FX_T];
    AxisFactor fy[VB][FY_T];
    float2 L[C][256];
  };
  __shared__ Slot S[NSTAGE];
  const int tid = threadIdx.x;
  const int lx = fast_col(tid), ly = fast_row(tid);
  const int kx = blockIdx.y * FX_T + lx, ky = blockIdx.z * FY_T + ly;
  const int v0 = blockIdx.x * VB;
  const int nv = min(VB, p.V - v0);
  const long long Q = (long long)p.Hp * p.Whp;
  const bool inside = kx < p.Whp && ky < p.Hp;
  const long long q = inside ? (long long)ky * p.Whp + kx : 0;
  const float4* DQ = p.dquad;
  const int zero = p.dq_zero;

  const char* xsrc[XPT];
  int xdst[XPT];
  bool xok[XPT], xact[XPT];
#pragma unroll
  for (int i = 0; i < XPT; ++i) {
    const int e = tid + 256 * i;
    const int b = e / FX_T, c = e % FX_T, col = blockIdx.y * FX_T + c;
    xact[i] = e < VB * FX_T;
    xok[i] = xact[i] && b < nv && col < p.Whp;
    xsrc[i] = reinterpret_cast<const char*>(p.px + (xok[i] ? (size_t)(v0 + b) * p.n * p.Whp + col : 0));
    xdst[i] = (int)((char*)&S[0].fx[b % VB][c] - (char*)&S[0]);
  }
  const long long xstep = (long long)p.Whp * 16;
  const int yb = tid / FY_T, yr = tid % FY_T, row = blockIdx.z * FY_T + yr;
  const bool yact = tid < VB * FY_T;
  const bool yok = yact && yb < nv && row < p.Hp;
  const char* ysrc = reinterpret_cast<const char*>(p.py + (yok ? (size_t)(v0 + yb) * p.n * p.Hp + row : 0));
  const long long ystep = (long long)p.Hp * 16;
  const int ydst = (int)((char*)&S[0].fy[yb % VB][yr] - (char*)&S[0]);
  const float2* lsrc0 = p.layers + q;
  const long long lstep = inside ? (long long)C * Q : 0;

  // out-of-grid columns / rows / missing views: zero-filled factors (idx 0 is a
  // valid entry; their weight is 0 through the zero phase)
  auto stage = [&](int k) {
    char* base = reinterpret_cast<char*>(&S[k % NSTAGE]);
#pragma unroll
    for (int i = 0; i < XPT; ++i)
      if (xact[i]) cp_async16(base + xdst[i], xsrc[i] + (xok[i] ? k * xstep : 0), xok[i]);
    if (yact) cp_async16(base + ydst, ysrc + (yok ? k * ystep : 0), yok);
    const float2* ls = lsrc0 + k * lstep;
#pragma unroll
    for (int c = 0; c < C; ++c) cp_async8(&S[k % NSTAGE].L[c][tid], ls + c * Q, inside);
    cp_async_commit();
  };

  u64 acc[VB][C];
#pragma unroll
  for (int b = 0; b < VB; ++b)
#pragma unroll
    for (int c = 0; c < C; ++c) acc[b][c] = 0ull;
  float4 Tn[VB];
  stage(0);
  if (p.n > 1) stage(1);
  cp_async_wait<0>();
  __syncthreads();
#pragma unroll
  for (int b = 0; b < VB; ++b) Tn[b] = __ldg(DQ + min(S[0].fx[b][lx].idx + S[0].fy[b][ly].idx, zero));
  for (int k = 0; k < p.n; ++k) {
    const Slot& sl = S[k % NSTAGE];
    const Slot& sn = S[(k + 1) % NSTAGE];
    if (k > 0) {
      cp_async_wait<0>();  // layer k + 1 staged (issued one layer ago)
      __syncthreads();     // ... visible; everyone is done with layer k - 1's slot
    }
    if (k + 2 < p.n) stage(k + 2);
    float2 L[C];
#pragma unroll
    for (int c = 0; c < C; ++c) L[c] = sl.L[c][tid];
    const bool more = k + 1 < p.n;
#pragma unroll
    for (int b = 0; b < VB; ++b) {
      const AxisFactor x = sl.fx[b][lx];
      const AxisFactor y = sl.fy[b][ly];
      const float4 T = Tn[b];
      // the quad of (view b, layer k + 1): a whole layer of latency cover
      if (more) Tn[b] = __ldg(DQ + min(sn.fx[b][lx].idx + sn.fy[b][ly].idx, zero));
      u64 ab = pack2(T.x, T.y);
      ffma2s(ab, pack2(T.z, T.w), y.frac);
      const float2 AB = as_f2(ab);
      const float s = fmaf(x.frac, AB.y, AB.x);
      const u64 w = fmul2s(cmul2(make_float2(x.re, x.im), make_float2(y.re, y.im)), s);
#pragma unroll
      for (int c = 0; c < C; ++c) cmac_w(acc[b][c], w, L[c]);
    }
  }
  if (!inside) return;
#pragma unroll
  for (int b = 0; b < VB; ++b) {
    if (b >= nv) break;
#pragma unroll
    for (int c = 0; c < C; ++c) p.out[((size_t)(v0 + b) * C + c) * Q + q] = as_f2(acc[b][c]);
  }
}

// ---------------------------------------------------------------------------
// Pinhole Horner tile.  With shifts affine in the layer index the weight of
// layer k at a bin is w_k = w_k0 * z^(k - k0), z = exp(2 pi i (alpha wx + beta wy)),
// so each block of HB layers is evaluated by Horner's rule
//     H = (...(L_{k0+HB-1} z + L_{k0+HB-2}) z + ...) z + L_k0       (2 FFMA2 / step)
// and out += w_k0 * H with the exact block weight w_k0 = px_k0 * py_k0 (the
// staged factors of the block's first layer).  One thread = one bin x one
// channel x VB views; no per-layer shared-memory traffic and no per-layer
// barrier: the layer value is the only per-layer load (prefetched 4 ahead).
// Phase error of a term: < HB fp32 roundings of z (~5e-7 rad at HB = 8).
// Nyquist lines (cosine phases, construct.py:68-80) are recomputed directly
// by render_nyquist_fix.
// ---------------------------------------------------------------------------
constexpr int HB = 8;

// fp64 axis tables of the Horner tiles: ratio exp(2 pi i alpha_v wx) at
// zx[v][kx] and the layer-0 phase exp(2 pi i pu[v,0] wx) at zx[V + v][kx]
// (rows likewise); cosine lines are not special here (render_nyquist_fix).
__global__ void render_z_kernel(RenderParams p) {
  const int v = blockIdx.x;
  const double a = p.h_alpha[v], b = p.h_beta[v];
  const double a0 = p.pu[(size_t)v * p.n], b0 = p.pv[(size_t)v * p.n];
  for (int kx = threadIdx.x; kx < p.Whp; kx += blockDim.x) {
    const double ox = omega_x_label(kx, p.Wp);
    cd ph = axis_phase(a, ox, false);
    p.zx[(size_t)v * p.Whp + kx] = make_double2(ph.re, ph.im);
    ph = axis_phase(a0, ox, false);
    p.zx[((size_t)p.V + v) * p.Whp + kx] = make_double2(ph.re, ph.im);
  }
  for (int ky = threadIdx.x; ky < p.Hp; ky += blockDim.x) {
    const double oy = omega_y_label(ky, p.Hp);
    cd ph = axis_phase(b, oy, false);
    p.zy[(size_t)v * p.Hp + ky] = make_double2(ph.re, ph.im);
    ph = axis_phase(b0, oy, false);
    p.zy[((size_t)p.V + v) * p.Hp + ky] = make_double2(ph.re, ph.im);
  }
}

// H = H * z + L   (packed: (zr Hr + Lr, zi Hr + Li) then + (-zi Hi, zr Hi))
__device__ __forceinline__ u64 horner_step(u64 H, u64 z, float2 L) {
  const float2 h = as_f2(H);
  u64 t = pack2(L.x, L.y);
  ffma2s(t, z, h.x);
  return ffma2_i(t, z, h.y);
}

template <int VB, int TY, int MINB>
__global__ void __launch_bounds__(32 * TY, MINB) render_horner(RenderParams p) {
  constexpr int NP = VB / 2, NT = 32 * TY;
  static_assert(HB == 8, "the prefetch walk assumes 8-layer blocks");
  __shared__ __align__(16) float4 WX[2][NP][32];
  __shared__ __align__(16) float4 WY[2][NP][TY];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5, tid = threadIdx.x;
  const int row0 = blockIdx.z * TY;
  const int kx = blockIdx.y * 32 + tx, ky = row0 + ty;
  const int v0 = blockIdx.x * VB;
  const int nv = min(VB, p.V - v0);
  const int npairs = (nv + 1) / 2;
  const long long Q = (long long)p.Hp * p.Whp;
  const bool inside = kx < p.Whp && ky < p.Hp;
  const long long q = inside ? (long long)ky * p.Whp + kx : 0;

  // block-weight staging (layer k0 of each block), zero-filled outside
  const float4* PXG = reinterpret_cast<const float4*>(p.px);
  const float4* PYG = reinterpret_cast<const float4*>(p.py);
  auto stage = [&](int blk, int slot) {
    const size_t k0 = (size_t)blk * HB;
    for (int e = tid; e < NP * (32 + TY); e += NT) {
      if (e < NP * 32) {
        const int pr = e >> 5, cc = e & 31, col = blockIdx.y * 32 + cc;
        const bool ok = pr < npairs && col < p.Whp;
        cp_async16(&WX[slot][pr][cc], ok ? PXG + ((size_t)(v0 / 2 + pr) * p.n + k0) * p.Whp + col : PXG, ok);
      } else {
        const int e2 = e - NP * 32, pr = e2 / TY, r = e2 % TY, row = row0 + r;
        const bool ok = pr < npairs && row < p.Hp;
        cp_async16(&WY[slot][pr][r], ok ? PYG + ((size_t)(v0 / 2 + pr) * p.n + k0) * p.Hp + row : PYG, ok);
      }
    }
    cp_async_commit();
  };
  const int nblk = (p.n + HB - 1) / HB;
  const int nsteps = nblk * p.C;  // (channel, block) pairs, channel-major
  stage(0, 0);

  // per-view Horner ratio, fp64 product rounded once (reused for every channel)
  u64 z[VB];
#pragma unroll
  for (int b = 0; b < VB; ++b) {
    z[b] = 0ull;
    if (inside && b < nv) {
      const double2 a = p.zx[(size_t)(v0 + b) * p.Whp + kx];
      const double2 e = p.zy[(size_t)(v0 + b) * p.Hp + ky];
      // explicit roundings: the same bits whatever slot b the view occupies
      z[b] = pack2(__double2float_rn(__dsub_rn(__dmul_rn(a.x, e.x), __dmul_rn(a.y, e.y))),
                   __double2float_rn(__dadd_rn(__dmul_rn(a.x, e.y), __dmul_rn(a.y, e.x))));
    }
  }

  // layer stream in processing order: (channel c, block blk, step j) -> layer
  // blk*HB + HB-1-j of channel c.  Step j consumes R[j & 3] and refills it with
  // step j + 4: layers k0+3..k0 (j < 4), then the top four of the next block
  // (of this channel, or block 0 of the next channel), walked with byte pointers.
  const char* lbase = reinterpret_cast<const char*>(p.layers + q);
  const long long lsb = (long long)p.C * Q * (long long)sizeof(float2);
  const long long csb = Q * (long long)sizeof(float2);
  auto ld_if = [&](const char* ptr, bool ok) -> float2 {
    return ok ? ld_stream(reinterpret_cast<const float2*>(ptr)) : make_float2(0.f, 0.f);
  };
  float2 R[4];
  {
    const char* pt = lbase + 7 * lsb;
#pragma unroll
    for (int j = 0; j < 4; ++j, pt -= lsb) R[j] = ld_if(pt, 7 - j < p.n);
  }
  u64 out[VB], H[VB];
#pragma unroll
  for (int b = 0; b < VB; ++b) out[b] = 0ull;
  int c = 0, blk = 0;
  for (int st = 0; st < nsteps; ++st) {
    cp_async_wait<0>();
    __syncthreads();  // weights of this block visible; the other slot is free
    // next (channel, block)
    const int nb = (blk + 1 < nblk) ? blk + 1 : 0;
    const int nc = (blk + 1 < nblk) ? c : c + 1;
    if (st + 1 < nsteps) stage(nb, (st + 1) & 1);
    const int k0 = blk * HB;
    const char* pa = lbase + c * csb + (k0 + 3) * lsb;
    const char* pn = lbase + nc * csb + (nb * HB + 7) * lsb;
    const bool nok = nc < p.C;
#pragma unroll
    for (int j = 0; j < HB; ++j) {
      const float2 L = R[j & 3];
      if (j < 4) {
        R[j & 3] = ld_if(pa, k0 + 3 - j < p.n);
        pa -= lsb;
      } else {
        R[j & 3] = ld_if(pn, nok && nb * HB + 7 - (j - 4) < p.n);
        pn -= lsb;
      }
      if (j == 0) {
#pragma unroll
        for (int b = 0; b < VB; ++b) H[b] = pack2(L.x, L.y);
      } else {
#pragma unroll
        for (int b = 0; b < VB; ++b) H[b] = horner_step(H[b], z[b], L);
      }
    }
    const int s = st & 1;
#pragma unroll
    for (int pr = 0; pr < NP; ++pr) {
      const float4 x = WX[s][pr][tx];
      const float4 y = WY[s][pr][ty];
      const u64 w0 = cmul2(make_float2(x.x, x.y), make_float2(y.x, y.y));
      const u64 w1 = cmul2(make_float2(x.z, x.w), make_float2(y.z, y.w));
      cmac_w(out[2 * pr], w0, as_f2(H[2 * pr]));
      cmac_w(out[2 * pr + 1], w1, as_f2(H[2 * pr + 1]));
    }
    if (blk + 1 == nblk) {  // channel c done
      if (inside) {
#pragma unroll
        for (int b = 0; b < VB; ++b)
          if (b < nv) p.out[((size_t)(v0 + b) * p.C + c) * Q + q] = as_f2(out[b]);
      }
#pragma unroll
      for (int b = 0; b < VB; ++b) out[b] = 0ull;
    }
    blk = nb;
    c = nc;
  }
}

// ---------------------------------------------------------------------------
// Single-accumulator Horner tile (all channels of a bin in one thread).
//   acc <- acc * m_k + L_k   for k = n-1 .. 0,   out = w_0 * acc
// with m_k = z32 (the fp32-rounded ratio z) except at k = 8b + 7, where
// m_k = zc = z32 * (z / z32)^8: every 8 steps the drift of the rounded ratio
// is cancelled, so a term's phase error stays below (7 + n/8) fp32 roundings
// (< 1e-6 rad at n = 64).  Per (view, bin, layer): C complex multiply-adds
// (2 FFMA2 each) and nothing else -- no factor traffic, no barrier.  The layer
// values stream through a per-thread cp.async ring in shared memory (each
// thread reads only what it copied: no block synchronisation).
// ---------------------------------------------------------------------------
constexpr int H2_RING = 8;

// One thread per (bin, VB views): the CTA's 128 threads take 128 consecutive
// bins of the flattened (ky, kx) half spectrum (no column padding of a 2-D tile).
template <int C, int VB>
__global__ void __launch_bounds__(128, 4) render_horner2(RenderParams p) {
  __shared__ __align__(16) float2 LR[H2_RING][C][128];
  __shared__ __align__(16) u64 ZC[VB][128];  // block multipliers (used once per 8 layers)
  const int tid = threadIdx.x;
  const int v0 = blockIdx.x * VB;
  const int nv = min(VB, p.V - v0);
  const long long Q = (long long)p.Hp * p.Whp;
  const long long qt = (long long)blockIdx.y * 128 + tid;
  const bool inside = qt < Q;
  const long long q = inside ? qt : 0;
  const int ky = (int)(q / p.Whp), kx = (int)(q - (long long)ky * p.Whp);
  const int n = p.n;
  const int nb = (n + HB - 1) / HB;

  // layer stream, k = n-1 .. 0; layer k lives in ring slot k & 7 (= a
  // compile-time index inside the 8-step blocks below).  One byte pointer
  // walks down the layers; out-of-grid threads copy zeros from a valid address.
  static_assert(H2_RING == HB, "ring slot = k mod 8");
  const long long qb = Q * (long long)sizeof(float2);
  const long long step_b = (long long)C * qb;
  const char* src = reinterpret_cast<const char*>(p.layers + q) + (long long)(n - 1) * step_b;
  int k_is = n - 1;
  auto issue = [&](int slot) {
    if (k_is >= 0) {
      const char* a0 = src;
#pragma unroll
      for (int c = 0; c < C; ++c, a0 += qb) cp_async8(&LR[slot][c][tid], a0, inside);
      src -= step_b;
    }
    --k_is;
    cp_async_commit();
  };
  for (int s = 0; s < H2_RING - 1; ++s) issue((n - 1 - s) & 7);

  // z and the drift-corrected block multiplier zc, from the fp64 axis tables;
  // explicit roundings: the same bits whatever slot the view occupies
  u64 z[VB];
  double2 za[VB], ze[VB];  // all table loads in flight before the fp64 math
#pragma unroll
  for (int b = 0; b < VB; ++b) {
    const bool ok = inside && b < nv;
    za[b] = ok ? p.zx[(size_t)(v0 + b) * p.Whp + kx] : make_double2(1.0, 0.0);
    ze[b] = ok ? p.zy[(size_t)(v0 + b) * p.Hp + ky] : make_double2(1.0, 0.0);
  }
#pragma unroll
  for (int b = 0; b < VB; ++b) {
    const double2 a = za[b];
    const double2 e = ze[b];
    const double zr = __dsub_rn(__dmul_rn(a.x, e.x), __dmul_rn(a.y, e.y));
    const double zi = __dadd_rn(__dmul_rn(a.x, e.y), __dmul_rn(a.y, e.x));
    const float fr = __double2float_rn(zr), fi = __double2float_rn(zi);
    // zc = z32 (z / z32)^8 = z32 (1 + d)^8 with d = z/z32 - 1, |d| <= 1e-7:
    // = z32 + 8 (z - z32) + O(28 |d|^2 ~ 1e-13) = 8 z - 7 z32, exact enough for fp32
    z[b] = pack2(fr, fi);
    ZC[b][tid] = pack2(__double2float_rn(__fma_rn(8.0, zr, -7.0 * (double)fr)),
                       __double2float_rn(__fma_rn(8.0, zi, -7.0 * (double)fi)));
  }
  u64 acc[VB][C];
#pragma unroll
  for (int b = 0; b < VB; ++b)
#pragma unroll
    for (int c = 0; c < C; ++c) acc[b][c] = 0ull;

  // blocks from the top: layers 8 blk' + 7 - j, blk' = nb-1 .. 0 (the top block
  // may be partial: its missing layers are skipped, uniformly across the CTA)
  for (int blk = nb - 1; blk >= 0; --blk) {
#pragma unroll
    for (int j = 0; j < HB; ++j) {
      const int k = blk * HB + HB - 1 - j;
      if (k >= n) continue;
      issue((HB - j) & 7);  // layer k - 7 -> slot (k - 7) & 7 = (k + 1) & 7
      cp_async_wait<H2_RING - 1>();  // layer k landed (this thread's own copies)
      float2 L[C];
#pragma unroll
      for (int c = 0; c < C; ++c) L[c] = LR[HB - 1 - j][c][tid];
#pragma unroll
      for (int b = 0; b < VB; ++b) {
        const u64 m = (j == 0) ? ZC[b][tid] : z[b];
#pragma unroll
        for (int c = 0; c < C; ++c) acc[b][c] = horner_step(acc[b][c], m, L[c]);
      }
    }
  }
  if (!inside) return;
  // out = w_0 * acc, w_0 = exp(2 pi i (pu[v,0] wx + pv[v,0] wy)) from the fp64 tables.
  // The table loads of a group of EB views are all issued before the group's
  // stores: p.out may alias p.zx / p.zy as far as the compiler knows, so a
  // per-view load -> store loop would serialise VB full load latencies.
  constexpr int EB = (VB + 2) / 3;
#pragma unroll
  for (int b0 = 0; b0 < VB; b0 += EB) {
    double2 a[EB], e[EB];
#pragma unroll
    for (int u = 0; u < EB; ++u) {
      const int v = v0 + min(b0 + u, nv - 1);  // clamped: a valid address, result unused past nv
      a[u] = p.zx[((size_t)p.V + v) * p.Whp + kx];
      e[u] = p.zy[((size_t)p.V + v) * p.Hp + ky];
    }
#pragma unroll
    for (int u = 0; u < EB; ++u) {
      const int b = b0 + u;
      if (b >= VB || b >= nv) break;
      const int v = v0 + b;
      const u64 w0 = pack2(__double2float_rn(__dsub_rn(__dmul_rn(a[u].x, e[u].x), __dmul_rn(a[u].y, e[u].y))),
                           __double2float_rn(__dadd_rn(__dmul_rn(a[u].x, e[u].y), __dmul_rn(a[u].y, e[u].x))));
#pragma unroll
      for (int c = 0; c < C; ++c) {
        u64 o = 0ull;
        cmac_w(o, w0, as_f2(acc[b][c]));
        p.out[((size_t)v * C + c) * Q + q] = as_f2(o);
      }
    }
  }
}

// views per thread: the largest register budget at 4 CTAs/SM (VB), or one of
// the two next smaller counts when that pads fewer views (162 = 18 x 9 on C2)
template <int C> struct H2VB;
template <> struct H2VB<1> { static constexpr int vb = 16; };
template <> struct H2VB<2> { static constexpr int vb = 12; };
template <> struct H2VB<3> { static constexpr int vb = 10; };
template <> struct H2VB<4> { static constexpr int vb = 8; };

template <int C, int VB>
int launch_horner2_vb(const RenderParams& p, cudaStream_t st) {
  const long long Q = (long long)p.Hp * p.Whp;
  dim3 grid((unsigned)((p.V + VB - 1) / VB), (unsigned)((Q + 127) / 128));
  render_horner2<C, VB><<<grid, 128, 0, st>>>(p);
  FDL_LAUNCH_CHECK("render_horner2");
  return FDL_OK;
}

template <int C>
int launch_horner2(const RenderParams& p, cudaStream_t st) {
  render_z_kernel<<<p.V, 256, 0, st>>>(p);
  FDL_LAUNCH_CHECK("render_z_kernel");
  constexpr int VB = H2VB<C>::vb;
  int best = VB;
  long long pad = (long long)((p.V + VB - 1) / VB) * VB;
  for (int vb = VB - 1; vb >= VB - 2; --vb) {
    const long long pv = (long long)((p.V + vb - 1) / vb) * vb;
    if (pv < pad) {
      pad = pv;
      best = vb;
    }
  }
  if (const char* e = getenv("FDL_H2_VB")) best = std::max(VB - 2, std::min(VB, atoi(e)));
  if (best == VB) return launch_horner2_vb<C, VB>(p, st);
  if (best == VB - 1) return launch_horner2_vb<C, VB - 1>(p, st);
  return launch_horner2_vb<C, VB - 2>(p, st);
}

// ---------------------------------------------------------------------------
// Aperture Horner tile (every aperture of the batch real; pinhole views point
// at the ONE entry).  Per (view, bin, layer) the weight is psi_k * phase_k with
// the phase geometric in k, so
//   acc <- acc * m_k + psi_k L_k,   out = w_0 * acc      (m_k as in render_horner2)
// psi_k is the reference's bilinear lookup (lfmodel.py:72-99) from the
// difference-form quad table: (A, B) = (a, b) + fy (c, d), psi = A + fx B.
// The lookup halves {frac, idx} of 8 layers x VB views x (32 columns + 4 rows)
// are staged per 8-layer block (double-buffered, one barrier per block); the
// quad of step j + 1 is gathered into registers while step j is consumed.
// Per unit: 2 (bilinear) + 3 C (psi L, Horner step) fp32 instructions.
// ---------------------------------------------------------------------------
template <int C, int VB>
__global__ void __launch_bounds__(128, 3) render_ap_horner(RenderParams p) {
  extern __shared__ __align__(16) unsigned char aph_smem[];  // ApHornerSmem<C, VB>
  float2 (*LR)[C][128] = reinterpret_cast<float2 (*)[C][128]>(aph_smem);
  float2 (*AX)[HB][VB][32] = reinterpret_cast<float2 (*)[HB][VB][32]>(aph_smem + sizeof(float2) * H2_RING * C * 128);
  float2 (*AY)[HB][VB][4] =
      reinterpret_cast<float2 (*)[HB][VB][4]>(aph_smem + sizeof(float2) * (H2_RING * C * 128 + 2 * HB * VB * 32));
  u64 (*ZC)[128] = reinterpret_cast<u64 (*)[128]>(
      aph_smem + sizeof(float2) * (H2_RING * C * 128 + 2 * HB * VB * 32 + 2 * HB * VB * 4));
  const int tid = threadIdx.x, tx = tid & 31, ty = tid >> 5;
  const int kx = blockIdx.y * 32 + tx, ky = blockIdx.z * 4 + ty;
  const int v0 = blockIdx.x * VB;
  const int nv = min(VB, p.V - v0);
  const long long Q = (long long)p.Hp * p.Whp;
  const bool inside = kx < p.Whp && ky < p.Hp;
  const long long q = inside ? (long long)ky * p.Whp + kx : 0;
  const int n = p.n;
  const int nb = (n + HB - 1) / HB;
  const float4* DQ = p.dquad;
  const int zero = p.dq_zero;
  const float2* PXA = reinterpret_cast<const float2*>(p.px);
  const float2* PYA = reinterpret_cast<const float2*>(p.py);

  // lookup halves of block blk (layers 8 blk + 7 - jj) into buffer buf; missing
  // views / layers / columns get the ZERO entry's index (weight 0)
  auto stage_aux = [&](int blk, int buf) {
    for (int e = tid; e < HB * VB * 36; e += 128) {
      const int jj = e / (VB * 36), r = e % (VB * 36), b = r / 36, c = r % 36;
      const int k = blk * HB + HB - 1 - jj, v = v0 + b;
      if (c < 32) {
        const int col = blockIdx.y * 32 + c;
        const bool ok = k < n && v < p.V && col < p.Whp;
        cp_async8(&AX[buf][jj][b][c], ok ? PXA + ((size_t)v * n + k) * p.Whp + col : PXA, ok);
      } else {
        const int row = blockIdx.z * 4 + c - 32;
        const bool ok = k < n && v < p.V && row < p.Hp;
        cp_async8(&AY[buf][jj][b][c - 32], ok ? PYA + ((size_t)v * n + k) * p.Hp + row : PYA, ok);
      }
    }
  };
  // (zero-filled entries are {0, idx 0}: idx 0 is a valid table entry, and the
  // views / layers they stand for are never stored or are skipped)

  // layer stream from the (zero-padded) top of the last block: layer k in ring
  // slot k & 7.  Padded layers (k >= n) are zero-filled: the accumulator is
  // still zero there, so their Horner multiplies are harmless.
  static_assert(H2_RING == HB, "ring slot = k mod 8");
  const int ktop = nb * HB - 1;
  const long long qb = Q * (long long)sizeof(float2);
  const long long step_b = (long long)C * qb;
  const char* lbase = reinterpret_cast<const char*>(p.layers + q);
  const char* src = lbase + (long long)ktop * step_b;
  int k_is = ktop;
  auto issue = [&](int slot) {
    const bool ok = inside && k_is >= 0 && k_is < n;
    const char* a0 = ok ? src : lbase;
#pragma unroll
    for (int c = 0; c < C; ++c) cp_async8(&LR[slot][c][tid], a0 + (ok ? c * qb : 0), ok);
    src -= step_b;
    --k_is;
    cp_async_commit();
  };
  stage_aux(nb - 1, (nb - 1) & 1);  // rides in the first group
#pragma unroll
  for (int s = 0; s < H2_RING - 1; ++s) issue(HB - 1 - s);

  u64 z[VB];
  double2 za[VB], ze[VB];
#pragma unroll
  for (int b = 0; b < VB; ++b) {
    const bool ok = inside && b < nv;
    za[b] = ok ? p.zx[(size_t)(v0 + b) * p.Whp + kx] : make_double2(1.0, 0.0);
    ze[b] = ok ? p.zy[(size_t)(v0 + b) * p.Hp + ky] : make_double2(1.0, 0.0);
  }
#pragma unroll
  for (int b = 0; b < VB; ++b) {
    const double2 a = za[b];
    const double2 e = ze[b];
    const double zr = __dsub_rn(__dmul_rn(a.x, e.x), __dmul_rn(a.y, e.y));
    const double zi = __dadd_rn(__dmul_rn(a.x, e.y), __dmul_rn(a.y, e.x));
    const float fr = __double2float_rn(zr), fi = __double2float_rn(zi);
    z[b] = pack2(fr, fi);
    ZC[b][tid] = pack2(__double2float_rn(__fma_rn(8.0, zr, -7.0 * (double)fr)),
                       __double2float_rn(__fma_rn(8.0, zi, -7.0 * (double)fi)));
  }
  u64 acc[VB][C];
#pragma unroll
  for (int b = 0; b < VB; ++b)
#pragma unroll
    for (int c = 0; c < C; ++c) acc[b][c] = 0ull;
  // quads and fractions of the current / next step, in two register sets that
  // alternate with the (compile-time) step parity: no copies between steps
  float4 TA[VB], TB[VB];
  float2 FA[VB], FB[VB];
  // per-block base pointers of this thread's lookup halves (compile-time offsets below)
  const float2* axb = nullptr;
  const float2* ayb = nullptr;
  auto gather1 = [&](int jj, int b, float4& T, float2& F) {
    const float2 ax = axb[(jj * VB + b) * 32], ay = ayb[(jj * VB + b) * 4];
    F = make_float2(ax.x, ay.x);
    T = __ldg(DQ + min(__float_as_int(ax.y) + __float_as_int(ay.y), zero));
  };

  for (int blk = nb - 1; blk >= 0; --blk) {
    const int buf = blk & 1;
    // block start: this layer's values and this block's lookup halves landed
    // (own copies), barrier (visible; everyone is done with the other buffer),
    // then the next block's halves ride in this step's copy group
    cp_async_wait<H2_RING - 2>();
    __syncthreads();
    if (blk > 0) stage_aux(blk - 1, buf ^ 1);
    issue(0);  // layer 8 blk + 7 - 7
    axb = &AX[buf][0][0][tx];
    ayb = &AY[buf][0][0][ty];
#pragma unroll
    for (int b = 0; b < VB; ++b) gather1(0, b, TA[b], FA[b]);
#pragma unroll
    for (int j = 0; j < HB; ++j) {
      if (j > 0) {
        issue((HB - j) & 7);  // layer k - 7 -> slot (k + 1) & 7
        cp_async_wait<H2_RING - 1>();
      }
      float2 L[C];
#pragma unroll
      for (int c = 0; c < C; ++c) L[c] = LR[HB - 1 - j][c][tid];
#pragma unroll
      for (int b = 0; b < VB; ++b) {
        float4& T = (j & 1) ? TB[b] : TA[b];
        float2& F = (j & 1) ? FB[b] : FA[b];
        if (j + 1 < HB) gather1(j + 1, b, (j & 1) ? TA[b] : TB[b], (j & 1) ? FA[b] : FB[b]);
        u64 ab = pack2(T.x, T.y);
        ffma2s(ab, pack2(T.z, T.w), F.y);
        const float2 AB = as_f2(ab);
        const float sv = fmaf(F.x, AB.y, AB.x);
        const u64 m = (j == 0) ? ZC[b][tid] : z[b];
#pragma unroll
        for (int c = 0; c < C; ++c) acc[b][c] = horner_step(acc[b][c], m, as_f2(fmul2s(pack2(L[c].x, L[c].y), sv)));
      }
    }
  }
  if (!inside) return;
#pragma unroll
  for (int b = 0; b < VB; ++b) {
    if (b >= nv) break;
    const int v = v0 + b;
    const double2 a = p.zx[((size_t)p.V + v) * p.Whp + kx];
    const double2 e = p.zy[((size_t)p.V + v) * p.Hp + ky];
    const u64 w0 = pack2(__double2float_rn(__dsub_rn(__dmul_rn(a.x, e.x), __dmul_rn(a.y, e.y))),
                         __double2float_rn(__dadd_rn(__dmul_rn(a.x, e.y), __dmul_rn(a.y, e.x))));
#pragma unroll
    for (int c = 0; c < C; ++c) {
      u64 o = 0ull;
      cmac_w(o, w0, as_f2(acc[b][c]));
      p.out[((size_t)v * C + c) * Q + q] = as_f2(o);
    }
  }
}

template <int C> struct APHVB;
template <> struct APHVB<1> { static constexpr int vb = 8; };
template <> struct APHVB<2> { static constexpr int vb = 6; };
template <> struct APHVB<3> { static constexpr int vb = 6; };
template <> struct APHVB<4> { static constexpr int vb = 4; };

template <int C>
int launch_ap_horner(const RenderParams& p, cudaStream_t st) {
  render_z_kernel<<<p.V, 256, 0, st>>>(p);
  FDL_LAUNCH_CHECK("render_z_kernel");
  constexpr int VB = APHVB<C>::vb;
  constexpr size_t smem = sizeof(float2) * (H2_RING * C * 128 + 2 * HB * VB * 36) + sizeof(u64) * VB * 128;
  FDL_CUDA_CHECK(cudaFuncSetAttribute(render_ap_horner<C, VB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  dim3 grid((unsigned)((p.V + VB - 1) / VB), (unsigned)((p.Whp + 31) / 32), (unsigned)((p.Hp + 3) / 4));
  render_ap_horner<C, VB><<<grid, 128, smem, st>>>(p);
  FDL_LAUNCH_CHECK("render_ap_horner");
  return FDL_OK;
}

// Direct sums on the self-conjugate Nyquist column / row, whose cosine phases
// (construct.py:68-80) the Horner recurrences do not model.  One thread per
// (line bin, view), every channel; the per-axis phases run as fp64
// recurrences from exact start values (shifts are affine on the Horner path):
// X_k = e^{i pi Pu_k} (cosine line: value Re X_k) or e^{2 pi i Pu_k wx}.
__global__ void render_nyquist_fix(RenderParams p) {
  const int ncol = (p.Wp % 2 == 0) ? p.Hp : 0;   // kx = Wp/2, every row
  const int nrow = (p.Hp % 2 == 0) ? p.Whp : 0;  // ky = Hp/2, every column
  const int nl = ncol + nrow;
  const long long total = (long long)nl * p.V;
  const long long Q = (long long)p.Hp * p.Whp;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total; e += (long long)gridDim.x * blockDim.x) {
    // views fastest: a warp's layer loads are one broadcast address
    const int v = (int)(e % p.V), i = (int)(e / p.V);
    const int kx = i < ncol ? p.Wp / 2 : i - ncol;
    const int ky = i < ncol ? i : p.Hp / 2;
    if (i >= ncol && kx == p.Wp / 2 && ncol) continue;  // the corner is done by the column entry
    const bool nx = (p.Wp % 2 == 0) && kx == p.Wp / 2, ny = (p.Hp % 2 == 0) && ky == p.Hp / 2;
    const double ox = omega_x_label(kx, p.Wp), oy = omega_y_label(ky, p.Hp);
    const double a0 = p.pu[(size_t)v * p.n], b0 = p.pv[(size_t)v * p.n];
    const double a = p.h_alpha[v], b = p.h_beta[v];
    const int ai = p.view_ap ? p.view_ap[v] : -1;
    // start phases and ratios in fp64: cosine lines e^{i pi P}, else e^{2 pi i P w}
    double sxr, sxi, rxr, rxi, syr, syi, ryr, ryi;
    sincospi(nx ? a0 : 2.0 * a0 * ox, &sxi, &sxr);
    sincospi(nx ? a : 2.0 * a * ox, &rxi, &rxr);
    sincospi(ny ? b0 : 2.0 * b0 * oy, &syi, &syr);
    sincospi(ny ? b : 2.0 * b * oy, &ryi, &ryr);
    const long long q = (long long)ky * p.Whp + kx;
    const float2* lp = p.layers + q;
    float accr[4] = {0.f, 0.f, 0.f, 0.f}, acci[4] = {0.f, 0.f, 0.f, 0.f};
    const long long cq = Q, kq = (long long)p.C * Q;
    for (int k0 = 0; k0 < p.n; k0 += 4) {
      // the layer values of 4 layers in flight before the arithmetic
      float2 Lb[4][4];
#pragma unroll
      for (int kk = 0; kk < 4; ++kk)
#pragma unroll
        for (int c = 0; c < 4; ++c)
          Lb[kk][c] = (c < p.C && k0 + kk < p.n) ? __ldg(lp + (k0 + kk) * kq + c * cq) : make_float2(0.f, 0.f);
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        if (k0 + kk >= p.n) break;
        // weight in fp64 (one per view, bin, layer), accumulation in fp32 like the tiles
        const double xr = sxr, xi = nx ? 0.0 : sxi, yr = syr, yi = ny ? 0.0 : syi;
        double psi = 1.0;  // real aperture tables only on this path (difference-form quads)
        if (ai >= 0) {
          const DevAperture& ap = p.aps[ai];
          const double t = p.t[(size_t)v * p.n + k0 + kk];
          int ix, iy;
          double fx, fy;
          const bool okx = axis_lookup(__dmul_rn(t, ox), ap.xi0_x, ap.step_x, ap.cols, ix, fx);
          const bool oky = axis_lookup(__dmul_rn(t, oy), ap.xi0_y, ap.step_y, ap.rows, iy, fy);
          if (okx && oky) {
            const float4 e = p.dquad[p.ap_qbase[ai] + iy * ap.cols + ix];
            psi = ((double)e.x + fy * e.z) + fx * ((double)e.y + fy * e.w);
          } else {
            psi = 0.0;
          }
        }
        const float wr = (float)((xr * yr - xi * yi) * psi), wi = (float)((xr * yi + xi * yr) * psi);
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          accr[c] = fmaf(wr, Lb[kk][c].x, fmaf(-wi, Lb[kk][c].y, accr[c]));
          acci[c] = fmaf(wr, Lb[kk][c].y, fmaf(wi, Lb[kk][c].x, acci[c]));
        }
        double t = sxr * rxr - sxi * rxi;
        sxi = sxr * rxi + sxi * rxr;
        sxr = t;
        t = syr * ryr - syi * ryi;
        syi = syr * ryi + syi * ryr;
        syr = t;
      }
    }
#pragma unroll
    for (int c = 0; c < 4; ++c)
      if (c < p.C) p.out[((size_t)v * p.C + c) * Q + q] = make_float2(accr[c], acci[c]);
  }
}

int launch_nyquist_fix(const RenderParams& p, cudaStream_t st) {
  if ((p.Wp % 2 == 0) || (p.Hp % 2 == 0)) {
    const long long total = (long long)p.V * (p.Hp + p.Whp);
    const int blocks = (int)std::min<long long>((total + 127) / 128, 148LL * 16);
    render_nyquist_fix<<<std::max(blocks, 1), 128, 0, st>>>(p);
    FDL_LAUNCH_CHECK("render_nyquist_fix");
  }
  return FDL_OK;
}

int horner_cfg_env() {
  const char* e = getenv("FDL_HORNER_CFG");
  return e ? atoi(e) : 0;
}

int launch_horner(const RenderParams& p, cudaStream_t st) {
  render_z_kernel<<<p.V, 256, 0, st>>>(p);
  FDL_LAUNCH_CHECK("render_z_kernel");
  // (views per thread, rows per CTA, CTAs per SM): register budget 65536 / (32 TY MINB)
  const int cfg = getenv("FDL_HORNER_CFG") ? horner_cfg_env() : 1;
  const int VB = cfg == 1 ? 8 : cfg == 2 ? 24 : cfg == 4 ? 12 : 16;
  const int TY = (cfg == 1 || cfg == 3) ? 8 : 4;
  const int rowtiles = (p.Hp + TY - 1) / TY;
  dim3 grid((unsigned)((p.V + VB - 1) / VB), (unsigned)((p.Whp + 31) / 32), (unsigned)rowtiles);
  switch (cfg) {
    case 1: render_horner<8, 8, 2><<<grid, 256, 0, st>>>(p); break;
    case 2: render_horner<24, 4, 2><<<grid, 128, 0, st>>>(p); break;
    case 3: render_horner<16, 8, 1><<<grid, 256, 0, st>>>(p); break;
    case 4: render_horner<12, 4, 3><<<grid, 128, 0, st>>>(p); break;
    default: render_horner<16, 4, 3><<<grid, 128, 0, st>>>(p); break;
  }
  FDL_LAUNCH_CHECK("render_horner");
  return launch_nyquist_fix(p, st);
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

// fast tiles: views per CTA by channel count (accumulators VB * C complex)
template <int C> struct FastVB;
template <> struct FastVB<1> { static constexpr int pin = 32, ap = 12; };
template <> struct FastVB<2> { static constexpr int pin = 24, ap = 8; };
template <> struct FastVB<3> { static constexpr int pin = 16, ap = 8; };
template <> struct FastVB<4> { static constexpr int pin = 10, ap = 4; };

bool legacy_render_env() {
  const char* e = getenv("FDL_RENDER_KERNEL");
  return e && e[0] == 'l';  // "legacy": the round-1 tile kernels (A/B)
}

bool use_horner2(const RenderParams& p) {
  const char* rk = getenv("FDL_RENDER_KERNEL");
  return p.horner && p.view_ap == nullptr && (!rk || rk[0] == '2');
}

// aperture batches whose tables are all real, shifts affine: the aperture
// Horner tile.  Opt-in (FDL_RENDER_KERNEL=aph): correct (tests pass through it)
// but slower than the round-1 tile on C5 (53 vs 36 ms per 256 views) --
// the per-step quad gathers and the doubled register sets cap it at 12 warps/SM.
bool use_ap_horner(const RenderParams& p) {
  const char* rk = getenv("FDL_RENDER_KERNEL");
  return p.horner && p.view_ap != nullptr && p.fast_ap && rk && rk[0] == 'a';
}


template <int C>
int launch_sum(const RenderParams& p, cudaStream_t st) {
  // Horner tile for single-channel pinhole batches (C3: 1.05 vs 1.40 ms for
  // 81 views); with C >= 2 the direct tile shares each weight across the
  // channels and wins (C2: 0.92 vs 1.08 ms).  FDL_RENDER_KERNEL=horner|fast|legacy overrides.
  const char* rk = getenv("FDL_RENDER_KERNEL");
  if (use_horner2(p)) {
    ktimer_mark(1, 0, st);
    int rc = launch_horner2<C>(p, st);
    ktimer_mark(1, 1, st);
    if (rc) return rc;
    return launch_nyquist_fix(p, st);
  }
  if (use_ap_horner(p)) {
    ktimer_mark(1, 0, st);
    int rc = launch_ap_horner<C>(p, st);
    ktimer_mark(1, 1, st);
    if (rc) return rc;
    return launch_nyquist_fix(p, st);
  }
  if (p.view_ap && p.fast_ap && !(rk && (rk[0] == 'l' || rk[0] == 'f'))) return render_ap_launch(p, st);
  const bool want_horner = rk && rk[0] == 'h';
  if (p.horner && p.view_ap == nullptr && want_horner) return launch_horner(p, st);
  // aperture batches: the round-1 tile stays the default until the fast
  // aperture tile beats it (C5: 4.0k vs 4.4k views/s); FDL_RENDER_KERNEL=fast selects it
  const bool fast_ap_ok = p.fast_ap && rk && rk[0] == 'f';
  if (!legacy_render_env() && (p.view_ap == nullptr || fast_ap_ok)) {
    const bool ap = p.view_ap != nullptr;
    const int VB = ap ? FastVB<C>::ap : FastVB<C>::pin;
    dim3 grid((unsigned)((p.V + VB - 1) / VB), (unsigned)((p.Whp + FX_T - 1) / FX_T), (unsigned)((p.Hp + FY_T - 1) / FY_T));
    ktimer_mark(1, 0, st);
    if (ap)
      render_ap_fast<C, FastVB<C>::ap><<<grid, 256, 0, st>>>(p);
    else
      render_pin_fast<C, FastVB<C>::pin><<<grid, 256, 0, st>>>(p);
    ktimer_mark(1, 1, st);
    FDL_LAUNCH_CHECK("render_fast_kernel");
    return FDL_OK;
  }
  constexpr int VB = C <= 3 ? 16 : 8;
  dim3 block(TX, TY);
  // view blocks vary fastest: the CTAs that share a layer tile run together and
  // re-read it from L2 instead of HBM (C4/C5 layers are GBs)
  dim3 grid((unsigned)((p.V + VB - 1) / VB), (unsigned)((p.Whp + TX - 1) / TX), (unsigned)((p.Hp + TY - 1) / TY));
  ktimer_mark(1, 0, st);
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
  ktimer_mark(1, 1, st);
  FDL_LAUNCH_CHECK("render_tile_kernel");
  return FDL_OK;
}

}  // namespace

int render_launch(const RenderParams& p0, cudaStream_t st) {
  if (p0.V == 0) return FDL_OK;
  RenderParams p = p0;
  p.aux8 = use_ap_horner(p) ? 1 : 0;  // the aperture Horner tile reads 8-byte lookup halves
  if (!use_horner2(p)) {  // the pinhole Horner tile needs no per-layer factors
    render_factors_kernel<<<p.V * p.n, 256, 0, st>>>(p);
    FDL_LAUNCH_CHECK("render_factors_kernel");
  }
  switch (p.C) {
    case 1: return launch_sum<1>(p, st);
    case 2: return launch_sum<2>(p, st);
    case 3: return launch_sum<3>(p, st);
    case 4: return launch_sum<4>(p, st);
    default: return fail(FDL_ERR_UNSUPPORTED, "render supports 1..4 channels");
  }
}

}  // namespace fdl
