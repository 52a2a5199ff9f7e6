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

template <int C, int VB>
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
    const int ai = (tid < nv && p.view_ap) ? p.view_ap[v0 + tid] : -1;
    TIDX[tid] = ai;
    if (ai >= 0) TB[tid] = p.tables[ai];
  }
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
      const int ai = TIDX[b];
      if (ai >= 0) {
        // one 16-byte quad-table load; out-of-range rows/columns hit the zero entry.
        // separable passes of lfmodel.py:115-116: rows (fy) first, then columns (fx)
        const RenderTable& tb = TB[b];
        const int qi = min(fy.idx + fx.idx, tb.zero);
        const float4 tr = __ldg(tb.re + qi);
        const float top = fmaf(fy.frac, tr.z - tr.x, tr.x);
        const float bot = fmaf(fy.frac, tr.w - tr.y, tr.y);
        const float sr = fmaf(fx.frac, bot - top, top);
        if (tb.im) {
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
  if (best == VB) return launch_horner2_vb<C, VB>(p, st);
  if (best == VB - 1) return launch_horner2_vb<C, VB - 1>(p, st);
  return launch_horner2_vb<C, VB - 2>(p, st);
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

// views per CTA of the direct pinhole tile by channel count (accumulators VB * C complex)
template <int C> struct PinVB;
template <> struct PinVB<1> { static constexpr int vb = 32; };
template <> struct PinVB<2> { static constexpr int vb = 24; };
template <> struct PinVB<3> { static constexpr int vb = 16; };
template <> struct PinVB<4> { static constexpr int vb = 10; };

// One tile per batch kind:
//   pinhole, shifts affine in the layer index  -> Horner tile + Nyquist-line fix-up
//   pinhole, any shifts (relaxed calibrations) -> direct pinhole tile
//   apertures, every table real                -> TMA-staged aperture tile (k3_render_ap.cu)
//   apertures, some table complex              -> generic tile (per-view tables)
template <int C>
int launch_sum(const RenderParams& p, cudaStream_t st) {
  if (p.view_ap == nullptr && p.horner) {
    ktimer_mark(1, 0, st);
    int rc = launch_horner2<C>(p, st);
    ktimer_mark(1, 1, st);
    if (rc) return rc;
    return launch_nyquist_fix(p, st);
  }
  if (p.view_ap == nullptr) {
    constexpr int VB = PinVB<C>::vb;
    dim3 grid((unsigned)((p.V + VB - 1) / VB), (unsigned)((p.Whp + FX_T - 1) / FX_T), (unsigned)((p.Hp + FY_T - 1) / FY_T));
    ktimer_mark(1, 0, st);
    render_pin_fast<C, VB><<<grid, 256, 0, st>>>(p);
    ktimer_mark(1, 1, st);
    FDL_LAUNCH_CHECK("render_pin_fast");
    return FDL_OK;
  }
  if (p.fast_ap) return render_ap_launch(p, st);
  constexpr int VB = 8;
  dim3 block(TX, TY);
  // view blocks vary fastest: the CTAs that share a layer tile run together
  dim3 grid((unsigned)((p.V + VB - 1) / VB), (unsigned)((p.Whp + TX - 1) / TX), (unsigned)((p.Hp + TY - 1) / TY));
  ktimer_mark(1, 0, st);
  render_tile_kernel<C, VB><<<grid, block, 0, st>>>(p);
  ktimer_mark(1, 1, st);
  FDL_LAUNCH_CHECK("render_tile_kernel");
  return FDL_OK;
}

}  // namespace

int render_factors_kernel_launch(const RenderParams& p, cudaStream_t st) {
  render_factors_kernel<<<p.V * p.n, 256, 0, st>>>(p);
  FDL_LAUNCH_CHECK("render_factors_kernel");
  return FDL_OK;
}

int render_launch(const RenderParams& p0, cudaStream_t st) {
  if (p0.V == 0) return FDL_OK;
  const RenderParams& p = p0;
  // per-layer factor tables: every tile but the pinhole Horner tile and the affine
  // aperture tile (k3_render_ap.cu, which runs its own 8-byte lookup pre-pass)
  const bool own_prepass = p.horner && (p.view_ap == nullptr || p.fast_ap);
  if (!own_prepass) {
    if (int rc = render_factors_kernel_launch(p, st)) return rc;
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
