// K0 / K4 on the shared-memory FFT engine (fft_engine.cuh) for grids whose
// sides cuFFT only reaches through its large-prime path.
//
// K0 (forward, construct.py:250-266): views (m,H,W,C) f32
//   rows pass : pack + zero-pad + real row FFTs, two real rows per complex
//               transform, unpacked to half spectra -> T1 (m,C,H,Whp) c64
//               (the Hp-H all-zero padded rows are never transformed)
//   cols pass : column FFTs over Hp (zero rows supplied on load) -> spectra
//               (m,C,Hp,Whp) + fp64 per-tile sum |b|^2 partials
// K4 (inverse, spectra.py:202-208 + render.py:210-225): spectra (V,C,Hp,Whp)
//   cols pass : inverse column FFTs, only the cropped rows stored -> T2
//   rows pass : Hermitian row completion (imaginary parts of the kx = 0 and
//               Nyquist columns dropped, as numpy's irfft does), two real rows
//               per complex inverse FFT, 1/(Hp Wp), crop, sRGB -> images
//               (V,Ho,Wo,C) f32
// Persistent CTAs loop over tiles; twiddle tables are built once per CTA.
#include <algorithm>
#include <map>
#include <tuple>
#include <cstdlib>
#include <type_traits>

#include "common.cuh"
#include "fft_engine.cuh"

namespace fdl {

namespace {

using fft::Geo;

// sRGB-encoded value -> linear light (render.py:39-42; fused into the K0 load)
__device__ inline float srgb_dec_f(float x) {
  return x <= 0.04045f ? x / 12.92f : powf((fmaxf(x, 0.04045f) + 0.055f) / 1.055f, 2.4f);
}

__device__ inline float srgb_enc_f(float x) {
  x = fmaxf(x, 0.f);
  return x <= 0.0031308f ? x * 12.92f : 1.055f * powf(x, 1.0f / 2.4f) - 0.055f;
}

struct SmemPtrs {
  float2 *tw1, *tw2, *data;
};
__device__ inline SmemPtrs carve(const Geo& g) {
  extern __shared__ __align__(16) float2 smem_f2[];
  SmemPtrs p;
  p.tw1 = smem_f2;
  p.tw2 = p.tw1 + g.tw1_len();
  p.data = p.tw2 + g.N;
  return p;
}

// Loads are issued in batches of U per thread before any shared-memory store,
// so each thread keeps U global loads in flight instead of one.
constexpr int U = 4;

// ---------------------------------------------------------------- K0 rows
// tile = (view j, RB image rows); real row q = c*RB + r; transform b = q % B
// carries row q (< B) in its real part and row q (>= B) in its imaginary part.
// Threads own columns n (load) / frequencies k (unpack) so the index math is
// done once per column; per-row offsets come from a small table.
constexpr int MAXQ = 640;  // >= 2B for every rows plan (B <= rows_threads)
constexpr int UB = 4;      // transforms per load batch (2*UB loads in flight)

template <int M, int C>
__global__ void __launch_bounds__(fft::rows_threads(M), fft::rows_blocks(M)) fwd_rows_kernel(const float* __restrict__ views, int m, int H,
                                                                       int W, int pad, Geo g, int RB,
                                                                       float2* __restrict__ t1, int srgb) {
  SmemPtrs s = carve(g);
  fft::build_tables(g, s.tw1, s.tw2);
  __shared__ int qsrc[MAXQ], qdst[MAXQ];
  const int N = g.N, B = g.B, Whp = N / 2 + 1;
  const int rblocks = (H + RB - 1) / RB;
  const int tiles = m * rblocks;
  for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
    const int j = tile / rblocks, y0 = (tile % rblocks) * RB;
    __syncthreads();  // previous tile's readers are done with data and tables
    for (int q = threadIdx.x; q < 2 * B; q += blockDim.x) {
      const int c = q / RB, r = q - c * RB;
      const bool ok = y0 + r < H;
      qsrc[q] = ok ? r * W * C + c : -1;                   // within the tile's first image row
      qdst[q] = ok ? (c * H + y0 + r) * Whp : -1;           // within view j of T1
    }
    __syncthreads();
    const float* vrow = views + ((size_t)j * H + y0) * W * C;
    for (int n = threadIdx.x; n < N; n += blockDim.x) {
      const int x = n - pad;
      float2* dst = s.data + fft::slot_in<M>(g, n);
      if (x < 0 || x >= W) {
        for (int b = 0; b < B; ++b) dst[b] = make_float2(0.f, 0.f);
        continue;
      }
      const float* px = vrow + x * C;
      for (int b0 = 0; b0 < B; b0 += UB) {
        float re[UB], im[UB];
#pragma unroll
        for (int u = 0; u < UB; ++u) {
          const int b = b0 + u;
          const int o1 = b < B ? qsrc[b] : -1, o2 = b < B ? qsrc[b + B] : -1;
          re[u] = o1 >= 0 ? __ldg(px + o1) : 0.f;
          im[u] = o2 >= 0 ? __ldg(px + o2) : 0.f;
        }
        if (srgb) {
#pragma unroll
          for (int u = 0; u < UB; ++u) {
            re[u] = srgb_dec_f(re[u]);
            im[u] = srgb_dec_f(im[u]);
          }
        }
#pragma unroll
        for (int u = 0; u < UB; ++u)
          if (b0 + u < B) dst[b0 + u] = make_float2(re[u], im[u]);
      }
    }
    __syncthreads();
    fft::stage1<M, false>(g, s.data, s.tw1, s.tw2);
    fft::stage2<M, false>(g, s.data);
    __syncthreads();
    // unpack: Z = X + iY  ->  X[k] = (Z[k] + conj Z[N-k]) / 2,  Y[k] = (Z[k] - conj Z[N-k]) / 2i
    float2* vout = t1 + (size_t)j * C * H * Whp;
    for (int k = threadIdx.x; k < Whp; k += blockDim.x) {
      const float2* zk = s.data + fft::slot_out(g, k);
      const float2* zm = s.data + fft::slot_out(g, k == 0 ? 0 : N - k);
      for (int b = 0; b < B; ++b) {
        const float2 z = zk[b], zc = zm[b];
        const int d1 = qdst[b], d2 = qdst[b + B];
        if (d1 >= 0) vout[d1 + k] = make_float2(0.5f * (z.x + zc.x), 0.5f * (z.y - zc.y));
        if (d2 >= 0) vout[d2 + k] = make_float2(0.5f * (z.y + zc.y), 0.5f * (zc.x - z.x));
      }
    }
  }
}

// ---------------------------------------------------------------- K0 cols
// B is a power of two (1 << lb): b = idx & (B-1), row = idx >> lb.
template <int M>
__global__ void __launch_bounds__(fft::cols_threads(M), fft::cols_blocks(M)) fwd_cols_kernel(const float2* __restrict__ t1, int planes,
                                                                       int H, int pad, int Whp, Geo g, int lb,
                                                                       float2* __restrict__ spec,
                                                                       double* __restrict__ partial) {
  SmemPtrs s = carve(g);
  fft::build_tables(g, s.tw1, s.tw2);
  const int N = g.N, B = g.B;
  const int cblocks = (Whp + B - 1) / B;
  const int tiles = planes * cblocks;
  const int nzero = (N - H) * B;
  __shared__ double red[32];
  for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
    const int pl = tile / cblocks, k0 = (tile % cblocks) * B;
    // thread = (column b, rows y0 + t*R): pointer and slot walks, no per-element index math
    const int b = threadIdx.x & (B - 1), R = blockDim.x >> lb, ys = threadIdx.x >> lb;
    const bool colok = k0 + b < Whp;
    const float2* src = t1 + ((size_t)pl * H + ys) * Whp + k0 + b;
    const size_t step = (size_t)R * Whp;
    __syncthreads();
    for (int y = ys; y < H; y += U * R, src += U * step) {
      float2 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u)
        v[u] = (colok && y + u * R < H) ? __ldg(src + u * step) : make_float2(0.f, 0.f);
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (y + u * R < H) s.data[fft::slot_in<M>(g, y + u * R + pad) + b] = v[u];
    }
    for (int i = threadIdx.x; i < nzero; i += blockDim.x) {
      const int e = i >> lb;
      s.data[fft::slot_in<M>(g, e < pad ? e : H + e) + (i & (B - 1))] = make_float2(0.f, 0.f);
    }
    __syncthreads();
    fft::stage1<M, false>(g, s.data, s.tw1, s.tw2);
    fft::stage2<M, false>(g, s.data);
    __syncthreads();
    double acc = 0.0;
    if (colok) {
      float2* dst = spec + ((size_t)pl * N + ys) * Whp + k0 + b;
      int k2 = g.divP.div(ys), k1 = ys - k2 * g.P;  // k = ys + t*R = k1 + P*k2
      for (int k = ys; k < N; k += R, dst += step) {
        const float2 v = s.data[k1 * g.SR + k2 * g.SC + b];
        *dst = v;
        acc = fma((double)v.x, (double)v.x, acc);
        acc = fma((double)v.y, (double)v.y, acc);
        k1 += R;
        while (k1 >= g.P) {
          k1 -= g.P;
          ++k2;
        }
      }
    }
    if (partial) {
      for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
      __syncthreads();
      if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
        partial[tile] = t;
      }
    }
  }
}

// ---------------------------------------------------------------- pipelined column passes
// Same transforms as fwd_cols_kernel / inv_cols_kernel, but the column tile is
// brought in by cp.async into the second of two tile buffers while the current
// tile is transformed, so the global-load latency hides under stage 1 instead
// of stalling the CTA between its barriers (ncu: long_scoreboard was the top
// stall of both column kernels).  Zero rows / out-of-range columns use the
// zero-fill form of the copy.  One thread = (column b, rows ys + t*R), as in
// the unpipelined kernels; the sum |b|^2 partials keep the same fixed order.
template <int M>
__device__ __forceinline__ void cols_issue(const Geo& g, int lb, float2* buf, const float2* __restrict__ src_plane,
                                           int Whp, int k0, int row_lo, int row_hi, int row_off) {
  const int B = g.B, b = threadIdx.x & (B - 1), R = blockDim.x >> lb, ys = threadIdx.x >> lb;
  const bool colok = k0 + b < Whp;
  // slot n of the transform holds source row n - row_off when row_lo <= n < row_hi
  for (int n = ys; n < g.N; n += R) {
    const bool ok = colok && n >= row_lo && n < row_hi;
    const float2* src = ok ? src_plane + (size_t)(n - row_off) * Whp + k0 + b : src_plane;
    cpa8(buf + fft::slot_in<M>(g, n) + b, src, ok);
  }
  cpa_commit();
}

template <int M>
__global__ void __launch_bounds__(fft::cols_threads(M), fft::cols_blocks(M)) fwd_cols_pipe_kernel(
    const float2* __restrict__ t1, int planes, int H, int pad, int Whp, Geo g, int lb, float2* __restrict__ spec,
    double* __restrict__ partial) {
  SmemPtrs s = carve(g);
  fft::build_tables(g, s.tw1, s.tw2);
  const int N = g.N, B = g.B, slots = g.slots();
  const int cblocks = (Whp + B - 1) / B;
  const int tiles = planes * cblocks;
  __shared__ double red[32];
  auto issue = [&](int tile, float2* buf) {
    const int pl = tile / cblocks, k0 = (tile % cblocks) * B;
    cols_issue<M>(g, lb, buf, t1 + (size_t)pl * H * Whp, Whp, k0, pad, pad + H, pad);
  };
  if ((int)blockIdx.x < tiles) issue(blockIdx.x, s.data);
  int it = 0;
  for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x, ++it) {
    float2* cur = s.data + (it & 1) * slots;
    const int pl = tile / cblocks, k0 = (tile % cblocks) * B;
    const int b = threadIdx.x & (B - 1), R = blockDim.x >> lb, ys = threadIdx.x >> lb;
    const bool colok = k0 + b < Whp;
    __syncthreads();  // the other buffer's previous tile is fully stored
    if (tile + (int)gridDim.x < tiles) {
      issue(tile + gridDim.x, s.data + ((it + 1) & 1) * slots);
      cpa_wait_1();
    } else {
      cpa_wait_all();
    }
    __syncthreads();
    fft::stage1<M, false>(g, cur, s.tw1, s.tw2);
    fft::stage2<M, false>(g, cur);
    __syncthreads();
    double acc = 0.0;
    if (colok) {
      float2* dst = spec + ((size_t)pl * N + ys) * Whp + k0 + b;
      const size_t step = (size_t)R * Whp;
      int k2 = g.divP.div(ys), k1 = ys - k2 * g.P;
      for (int k = ys; k < N; k += R, dst += step) {
        const float2 v = cur[k1 * g.SR + k2 * g.SC + b];
        *dst = v;
        acc = fma((double)v.x, (double)v.x, acc);
        acc = fma((double)v.y, (double)v.y, acc);
        k1 += R;
        while (k1 >= g.P) {
          k1 -= g.P;
          ++k2;
        }
      }
    }
    if (partial) {
      for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
      __syncthreads();
      if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
        partial[tile] = t;
      }
    }
  }
}

template <int M>
__global__ void __launch_bounds__(fft::cols_threads(M), fft::cols_blocks(M)) inv_cols_pipe_kernel(
    const float2* __restrict__ spec, int planes, int Whp, int pad, int Ho, Geo g, int lb, float2* __restrict__ t2) {
  SmemPtrs s = carve(g);
  fft::build_tables(g, s.tw1, s.tw2);
  const int N = g.N, B = g.B, slots = g.slots();
  const int cblocks = (Whp + B - 1) / B;
  const int tiles = planes * cblocks;
  auto issue = [&](int tile, float2* buf) {
    const int pl = tile / cblocks, k0 = (tile % cblocks) * B;
    cols_issue<M>(g, lb, buf, spec + (size_t)pl * N * Whp, Whp, k0, 0, N, 0);
  };
  if ((int)blockIdx.x < tiles) issue(blockIdx.x, s.data);
  int it = 0;
  for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x, ++it) {
    float2* cur = s.data + (it & 1) * slots;
    const int pl = tile / cblocks, k0 = (tile % cblocks) * B;
    const int b = threadIdx.x & (B - 1), R = blockDim.x >> lb, ys = threadIdx.x >> lb;
    const bool colok = k0 + b < Whp;
    __syncthreads();
    if (tile + (int)gridDim.x < tiles) {
      issue(tile + gridDim.x, s.data + ((it + 1) & 1) * slots);
      cpa_wait_1();
    } else {
      cpa_wait_all();
    }
    __syncthreads();
    fft::stage1<M, true>(g, cur, s.tw1, s.tw2);
    fft::stage2<M, true>(g, cur);
    __syncthreads();
    if (colok) {
      const size_t step = (size_t)R * Whp;
      float2* dst = t2 + ((size_t)pl * Ho + ys) * Whp + k0 + b;
      int k2 = g.divP.div(ys + pad), k1 = ys + pad - k2 * g.P;
      for (int y = ys; y < Ho; y += R, dst += step) {
        *dst = cur[k1 * g.SR + k2 * g.SC + b];
        k1 += R;
        while (k1 >= g.P) {
          k1 -= g.P;
          ++k2;
        }
      }
    }
  }
}

inline bool cols_pipe_enabled() {
  const char* e = getenv("FDL_FFT_PIPE");
  return e && e[0] == '1';  // opt-in: measured slower (C2b, C4: the second buffer costs a resident CTA)
}

// per view: sum of its C * cblocks tile partials, fixed order
__global__ void sumsq_tiles_kernel(const double* __restrict__ partial, int m, int per_view,
                                   double* __restrict__ out) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= m) return;
  double s = 0.0;
  for (int i = 0; i < per_view; ++i) s += partial[(size_t)j * per_view + i];
  out[j] = s;
}

// ---------------------------------------------------------------- K4 cols
template <int M>
__global__ void __launch_bounds__(fft::cols_threads(M), fft::cols_blocks(M)) inv_cols_kernel(const float2* __restrict__ spec, int planes,
                                                                       int Whp, int pad, int Ho, Geo g, int lb,
                                                                       float2* __restrict__ t2) {
  SmemPtrs s = carve(g);
  fft::build_tables(g, s.tw1, s.tw2);
  const int N = g.N, B = g.B;
  const int cblocks = (Whp + B - 1) / B;
  const int tiles = planes * cblocks;
  for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
    const int pl = tile / cblocks, k0 = (tile % cblocks) * B;
    const int b = threadIdx.x & (B - 1), R = blockDim.x >> lb, ys = threadIdx.x >> lb;
    const bool colok = k0 + b < Whp;
    const float2* src = spec + ((size_t)pl * N + ys) * Whp + k0 + b;
    const size_t step = (size_t)R * Whp;
    __syncthreads();
    for (int n = ys; n < N; n += U * R, src += U * step) {
      float2 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u)
        v[u] = (colok && n + u * R < N) ? __ldg(src + u * step) : make_float2(0.f, 0.f);
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (n + u * R < N) s.data[fft::slot_in<M>(g, n + u * R) + b] = v[u];
    }
    __syncthreads();
    fft::stage1<M, true>(g, s.data, s.tw1, s.tw2);
    fft::stage2<M, true>(g, s.data);
    __syncthreads();
    if (colok) {
      float2* dst = t2 + ((size_t)pl * Ho + ys) * Whp + k0 + b;
      int k2 = g.divP.div(ys + pad), k1 = ys + pad - k2 * g.P;  // output row y = ys + t*R, index y + pad
      for (int y = ys; y < Ho; y += R, dst += step) {
        *dst = s.data[k1 * g.SR + k2 * g.SC + b];
        k1 += R;
        while (k1 >= g.P) {
          k1 -= g.P;
          ++k2;
        }
      }
    }
  }
}

// ---------------------------------------------------------------- K4 rows
template <int M, int C>
__global__ void __launch_bounds__(fft::rows_threads(M), fft::rows_blocks(M)) inv_rows_kernel(const float2* __restrict__ t2, int V, int Ho,
                                                                       int Wo, int pad, Geo g, int RB, int srgb,
                                                                       float scale, float* __restrict__ out) {
  SmemPtrs s = carve(g);
  fft::build_tables(g, s.tw1, s.tw2);
  __shared__ int qsrc[MAXQ];
  const int N = g.N, B = g.B, Whp = N / 2 + 1;
  const bool even = (N & 1) == 0;
  const int rblocks = (Ho + RB - 1) / RB;
  const int tiles = V * rblocks;
  for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
    const int v = tile / rblocks, y0 = (tile % rblocks) * RB;
    __syncthreads();
    for (int q = threadIdx.x; q < 2 * B; q += blockDim.x) {
      const int c = q / RB, r = q - c * RB;
      qsrc[q] = y0 + r < Ho ? (c * Ho + y0 + r) * Whp : -1;
    }
    __syncthreads();
    const float2* vin = t2 + (size_t)v * C * Ho * Whp;
    for (int k = threadIdx.x; k < Whp; k += blockDim.x) {
      float2* d1 = s.data + fft::slot_in<M>(g, k);
      float2* d2 = s.data + fft::slot_in<M>(g, k == 0 ? 0 : N - k);
      const bool self = k == 0 || (even && 2 * k == N);  // self-conjugate: keep the real part only
      for (int b0 = 0; b0 < B; b0 += UB) {
        float2 X[UB], Y[UB];
#pragma unroll
        for (int u = 0; u < UB; ++u) {
          const int b = b0 + u;
          const int o1 = b < B ? qsrc[b] : -1, o2 = b < B ? qsrc[b + B] : -1;
          X[u] = o1 >= 0 ? __ldg(vin + o1 + k) : make_float2(0.f, 0.f);
          Y[u] = o2 >= 0 ? __ldg(vin + o2 + k) : make_float2(0.f, 0.f);
        }
#pragma unroll
        for (int u = 0; u < UB; ++u) {
          const int b = b0 + u;
          if (b < B) {
            float2 x = X[u], y = Y[u];
            if (self) x.y = y.y = 0.f;
            d1[b] = make_float2(x.x - y.y, x.y + y.x);
            if (!self) d2[b] = make_float2(x.x + y.y, y.x - x.y);
          }
        }
      }
    }
    __syncthreads();
    fft::stage1<M, true>(g, s.data, s.tw1, s.tw2);
    fft::stage2<M, true>(g, s.data);
    __syncthreads();
    const int rows = min(RB, Ho - y0);
    for (int x = threadIdx.x; x < Wo; x += blockDim.x) {
      const float2* zx = s.data + fft::slot_out(g, x + pad);
      float* o = out + (((size_t)v * Ho + y0) * Wo + x) * C;
      for (int r = 0; r < rows; ++r) {
#pragma unroll
        for (int c = 0; c < C; ++c) {
          const int q = c * RB + r;
          const int hi = q >= B;
          const float2 z = zx[q - hi * B];
          float val = (hi ? z.y : z.x) * scale;
          if (srgb) val = srgb_enc_f(val);
          o[(size_t)r * Wo * C + c] = val;
        }
      }
    }
  }
}

// ---------------------------------------------------------------- planning
// Tiles are sized for several resident CTAs per SM (one CTA's loads overlap
// another's transforms): at most target_threads() per CTA and kSmemTarget of
// shared memory.  FDL_FFT_THREADS / FDL_FFT_SMEM_KB override (tuning).
inline size_t smem_target() {
  const char* e = getenv("FDL_FFT_SMEM_KB");
  return (e ? (size_t)atoi(e) : 100) * 1024;
}
inline int target_threads(int M, bool rows) {
  const int cap = rows ? fft::rows_threads(M) : fft::cols_threads(M);
  const char* e = getenv("FDL_FFT_THREADS");
  return e ? std::min(atoi(e), cap) : cap;
}

inline size_t al256(size_t x) { return (x + 255) & ~(size_t)255; }

// conflict-minimising strides, cached per (N, B, kind); kept only if the
// tile still fits the shared-memory budget
inline void tuned(Geo& g, bool rows) {
  static thread_local std::map<std::tuple<int, int, bool>, std::pair<int, int>> cache;
  const auto key = std::make_tuple(g.N, g.B, rows);
  auto it = cache.find(key);
  if (it == cache.end()) {
    Geo t = g;
    fft::tune_strides(t, rows, ((fft::threads_for(t) + 31) / 32) * 32);
    if (fft::smem_bytes(t) > fft::smem_bytes(g) + 4096) t = g;
    it = cache.emplace(key, std::make_pair(t.SC, t.SR)).first;
  }
  g.SC = it->second.first;
  g.SR = it->second.second;
}

// rows pass: B = RB*C/2 complex transforms, RB*C even
bool plan_rows(int N, int C, Geo* g, int* RB) {
  int best = 0;
  const Geo g1 = fft::make_geo(N, 1);
  const int cap = target_threads(g1.M, true);
  for (int rb = 1; rb <= 256; ++rb) {
    if ((rb * C) % 2) continue;
    const Geo t = fft::make_geo(N, rb * C / 2);
    if (fft::threads_for(t) > cap || fft::smem_bytes(t) > smem_target()) break;
    best = rb;
  }
  if (!best) {  // the smallest legal tile, if it fits at all
    const int rb = (C % 2) ? 2 : 1;
    const Geo t = fft::make_geo(N, rb * C / 2);
    if (fft::threads_for(t) > fft::rows_threads(t.M) || fft::smem_bytes(t) > 220 * 1024) return false;
    best = rb;
  }
  *RB = best;
  *g = fft::make_geo(N, best * C / 2);
  tuned(*g, true);
  return true;
}

// cols pass: B a power of two (index math by shifts)
bool plan_cols(int N, Geo* g) {
  const Geo g1 = fft::make_geo(N, 1);
  const int cap = target_threads(g1.M, false);
  for (int B = 32; B >= 1; B >>= 1) {
    const Geo t = fft::make_geo(N, B);
    if (fft::threads_for(t) <= cap && fft::smem_bytes(t) <= smem_target()) {
      *g = t;
      tuned(*g, false);
      return true;
    }
  }
  for (int B = 8; B >= 1; B >>= 1) {
    const Geo t = fft::make_geo(N, B);
    if (fft::threads_for(t) <= fft::cols_threads(t.M) && fft::smem_bytes(t) <= 220 * 1024) {
      *g = t;
      return true;
    }
  }
  return false;
}

inline int round_threads(const Geo& g) { return ((fft::threads_for(g) + 31) / 32) * 32; }

template <typename K>
int persistent_grid(K kernel, int threads, size_t smem, int tiles) {
  static thread_local int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  int per_sm = 0;
  cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, smem);
  if (per_sm < 1) per_sm = 1;
  return std::max(1, std::min(tiles, sms * per_sm));
}

template <int M>
int launch_fwd_rows_m(int C, const float* views, int m, int H, int W, int pad, const Geo& g, int RB, float2* t1,
                      int srgb, cudaStream_t st) {
  if (2 * g.B > MAXQ) return fail(FDL_ERR_UNSUPPORTED, "FFT engine: rows tile too large");
  const int threads = round_threads(g);
  const size_t smem = fft::smem_bytes(g);
  const int tiles = m * ((H + RB - 1) / RB);
#define FDL_ROWS(CC)                                                                               \
  case CC: {                                                                                       \
    auto k = fwd_rows_kernel<M, CC>;                                                               \
    k<<<persistent_grid(k, threads, smem, tiles), threads, smem, st>>>(views, m, H, W, pad, g, RB, t1, srgb); \
    break;                                                                                         \
  }
  switch (C) {
    FDL_ROWS(1)
    FDL_ROWS(2)
    FDL_ROWS(3)
    FDL_ROWS(4)
    default: return fail(FDL_ERR_UNSUPPORTED, "views support 1..4 channels");
  }
#undef FDL_ROWS
  FDL_LAUNCH_CHECK("fwd_rows_kernel");
  return FDL_OK;
}

template <int M>
int launch_inv_rows_m(int C, const float2* t2, int V, int Ho, int Wo, int pad, const Geo& g, int RB, int srgb,
                      float scale, float* out, cudaStream_t st) {
  if (2 * g.B > MAXQ) return fail(FDL_ERR_UNSUPPORTED, "FFT engine: rows tile too large");
  const int threads = round_threads(g);
  const size_t smem = fft::smem_bytes(g);
  const int tiles = V * ((Ho + RB - 1) / RB);
#define FDL_ROWS(CC)                                                                                            \
  case CC: {                                                                                                    \
    auto k = inv_rows_kernel<M, CC>;                                                                            \
    k<<<persistent_grid(k, threads, smem, tiles), threads, smem, st>>>(t2, V, Ho, Wo, pad, g, RB, srgb, scale, \
                                                                       out);                                    \
    break;                                                                                                      \
  }
  switch (C) {
    FDL_ROWS(1)
    FDL_ROWS(2)
    FDL_ROWS(3)
    FDL_ROWS(4)
    default: return fail(FDL_ERR_UNSUPPORTED, "images support 1..4 channels");
  }
#undef FDL_ROWS
  FDL_LAUNCH_CHECK("inv_rows_kernel");
  return FDL_OK;
}

inline int log2i(int b) {
  int l = 0;
  while ((1 << l) < b) ++l;
  return l;
}

template <int M>
int launch_fwd_cols_m(const float2* t1, int planes, int H, int pad, int Whp, const Geo& g, float2* spec,
                      double* partial, cudaStream_t st) {
  const int threads = round_threads(g);
  const size_t smem = fft::smem_bytes(g);
  const int tiles = planes * ((Whp + g.B - 1) / g.B);
  const size_t smem2 = smem + sizeof(float2) * (size_t)g.slots();  // second tile buffer
  if (cols_pipe_enabled() && smem2 <= 227 * 1024) {
    auto k = fwd_cols_pipe_kernel<M>;
    k<<<persistent_grid(k, threads, smem2, tiles), threads, smem2, st>>>(t1, planes, H, pad, Whp, g, log2i(g.B),
                                                                         spec, partial);
    FDL_LAUNCH_CHECK("fwd_cols_pipe_kernel");
    return FDL_OK;
  }
  auto k = fwd_cols_kernel<M>;
  k<<<persistent_grid(k, threads, smem, tiles), threads, smem, st>>>(t1, planes, H, pad, Whp, g, log2i(g.B), spec,
                                                                     partial);
  FDL_LAUNCH_CHECK("fwd_cols_kernel");
  return FDL_OK;
}

template <int M>
int launch_inv_cols_m(const float2* spec, int planes, int Whp, int pad, int Ho, const Geo& g, float2* t2,
                      cudaStream_t st) {
  const int threads = round_threads(g);
  const size_t smem = fft::smem_bytes(g);
  const int tiles = planes * ((Whp + g.B - 1) / g.B);
  const size_t smem2 = smem + sizeof(float2) * (size_t)g.slots();
  if (cols_pipe_enabled() && smem2 <= 227 * 1024) {
    auto k = inv_cols_pipe_kernel<M>;
    k<<<persistent_grid(k, threads, smem2, tiles), threads, smem2, st>>>(spec, planes, Whp, pad, Ho, g, log2i(g.B),
                                                                         t2);
    FDL_LAUNCH_CHECK("inv_cols_pipe_kernel");
    return FDL_OK;
  }
  auto k = inv_cols_kernel<M>;
  k<<<persistent_grid(k, threads, smem, tiles), threads, smem, st>>>(spec, planes, Whp, pad, Ho, g, log2i(g.B), t2);
  FDL_LAUNCH_CHECK("inv_cols_kernel");
  return FDL_OK;
}

}  // namespace

// ------------------------------------------------------------------ entry points used by k0_spectra.cu
bool fft_engine_applies(int Hp, int Wp, int C) {
  const char* env = getenv("FDL_FFT");
  if (env && env[0] == 'c') return false;  // FDL_FFT=cufft
  int P, M;
  if (!fft::split(Hp, &P, &M) || !fft::split(Wp, &P, &M)) return false;
  if (!(fft::wanted(Hp) || fft::wanted(Wp)) && !(env && env[0] == 'e')) return false;  // FDL_FFT=engine forces
  Geo g;
  int rb;
  return C >= 1 && C <= 4 && plan_rows(Wp, C, &g, &rb) && plan_cols(Hp, &g);
}

size_t engine_fwd_ws(int m, int H, int W, int C, int pad) {
  const int Hp = H + 2 * pad, Wp = W + 2 * pad, Whp = Wp / 2 + 1;
  Geo gc;
  plan_cols(Hp, &gc);
  const int cblocks = (Whp + gc.B - 1) / gc.B;
  return al256(sizeof(float2) * (size_t)m * C * H * Whp) + al256(sizeof(double) * (size_t)m * C * cblocks);
}

int engine_fwd(const float* views, int m, int H, int W, int C, int pad, float2* spectra, double* view_sumsq,
               void* ws, cudaStream_t st, int srgb) {
  const int Hp = H + 2 * pad, Wp = W + 2 * pad, Whp = Wp / 2 + 1;
  Geo gr, gc;
  int RB;
  if (!plan_rows(Wp, C, &gr, &RB) || !plan_cols(Hp, &gc)) return fail(FDL_ERR_UNSUPPORTED, "FFT engine plan");
  float2* t1 = reinterpret_cast<float2*>(ws);
  double* partial = reinterpret_cast<double*>(reinterpret_cast<char*>(ws) + al256(sizeof(float2) * (size_t)m * C * H * Whp));
  int rc;
  {
    auto call = [&](auto mm) { return launch_fwd_rows_m<decltype(mm)::value>(C, views, m, H, W, pad, gr, RB, t1, srgb, st); };
    switch (gr.M) {
      case 1: rc = call(std::integral_constant<int, 1>()); break;
      case 2: rc = call(std::integral_constant<int, 2>()); break;
      case 4: rc = call(std::integral_constant<int, 4>()); break;
      case 8: rc = call(std::integral_constant<int, 8>()); break;
      case 16: rc = call(std::integral_constant<int, 16>()); break;
      case 32: rc = call(std::integral_constant<int, 32>()); break;
      default: return fail(FDL_ERR_UNSUPPORTED, "FFT engine: power-of-two factor > 32");
    }
  }
  if (rc) return rc;
  {
    auto call = [&](auto mm) {
      return launch_fwd_cols_m<decltype(mm)::value>(t1, m * C, H, pad, Whp, gc, spectra,
                                                    view_sumsq ? partial : nullptr, st);
    };
    switch (gc.M) {
      case 1: rc = call(std::integral_constant<int, 1>()); break;
      case 2: rc = call(std::integral_constant<int, 2>()); break;
      case 4: rc = call(std::integral_constant<int, 4>()); break;
      case 8: rc = call(std::integral_constant<int, 8>()); break;
      case 16: rc = call(std::integral_constant<int, 16>()); break;
      case 32: rc = call(std::integral_constant<int, 32>()); break;
      default: return fail(FDL_ERR_UNSUPPORTED, "FFT engine: power-of-two factor > 32");
    }
  }
  if (rc) return rc;
  if (view_sumsq) {
    const int per_view = C * ((Whp + gc.B - 1) / gc.B);
    sumsq_tiles_kernel<<<(m + 127) / 128, 128, 0, st>>>(partial, m, per_view, view_sumsq);
    FDL_LAUNCH_CHECK("sumsq_tiles_kernel");
  }
  return FDL_OK;
}

size_t engine_inv_ws(int V, int C, int Hp, int Wp) {
  return al256(sizeof(float2) * (size_t)V * C * Hp * (Wp / 2 + 1));
}

int engine_inv(const float2* spectra, int V, int C, int Hp, int Wp, int pad, int Ho, int Wo, int srgb, float* images,
               void* ws, cudaStream_t st) {
  const int Whp = Wp / 2 + 1;
  Geo gr, gc;
  int RB;
  if (!plan_rows(Wp, C, &gr, &RB) || !plan_cols(Hp, &gc)) return fail(FDL_ERR_UNSUPPORTED, "FFT engine plan");
  float2* t2 = reinterpret_cast<float2*>(ws);
  const float scale = (float)(1.0 / ((double)Hp * (double)Wp));
  int rc;
  {
    auto call = [&](auto mm) {
      return launch_inv_cols_m<decltype(mm)::value>(spectra, V * C, Whp, pad, Ho, gc, t2, st);
    };
    switch (gc.M) {
      case 1: rc = call(std::integral_constant<int, 1>()); break;
      case 2: rc = call(std::integral_constant<int, 2>()); break;
      case 4: rc = call(std::integral_constant<int, 4>()); break;
      case 8: rc = call(std::integral_constant<int, 8>()); break;
      case 16: rc = call(std::integral_constant<int, 16>()); break;
      case 32: rc = call(std::integral_constant<int, 32>()); break;
      default: return fail(FDL_ERR_UNSUPPORTED, "FFT engine: power-of-two factor > 32");
    }
  }
  if (rc) return rc;
  {
    auto call = [&](auto mm) {
      return launch_inv_rows_m<decltype(mm)::value>(C, t2, V, Ho, Wo, pad, gr, RB, srgb, scale, images, st);
    };
    switch (gr.M) {
      case 1: rc = call(std::integral_constant<int, 1>()); break;
      case 2: rc = call(std::integral_constant<int, 2>()); break;
      case 4: rc = call(std::integral_constant<int, 4>()); break;
      case 8: rc = call(std::integral_constant<int, 8>()); break;
      case 16: rc = call(std::integral_constant<int, 16>()); break;
      case 32: rc = call(std::integral_constant<int, 32>()); break;
      default: return fail(FDL_ERR_UNSUPPORTED, "FFT engine: power-of-two factor > 32");
    }
  }
  return rc;
}

}  // namespace fdl
