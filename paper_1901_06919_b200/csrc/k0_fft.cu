// K0 / K4 on the warp-per-transform FFT engine (fft2.cuh) for grids whose
// sides are 67 * 2^a or 131 * 2^a (the reference's padded C1 / C2 / C2b / C4
// grids: 134, 536, 1048, 2144), which cuFFT only reaches through its slow
// large-prime path.
//
// K0 (forward, construct.py:250-266): views (m,H,W,C) f32
//   rows pass : pack + zero-pad two real image rows (y, y+1) of one channel
//               as one complex transform, unpacked to the two half spectra
//               -> T1 (m,C,H,Whp) c64 (the all-zero padded rows are never
//               transformed)
//   cols pass : column FFTs over Hp (zero rows supplied on load) -> spectra
//               (m,C,Hp,Whp) + one fp64 sum |b|^2 per (plane, column),
//               reduced per view in a fixed order (lambda does not depend on
//               batching or scheduling)
// K4 (inverse, spectra.py:202-208 + render.py:210-225): spectra (V,C,Hp,Whp)
//   cols pass : inverse column FFTs, only the cropped rows stored -> T2
//   rows pass : Hermitian completion of two rows (the imaginary parts of the
//               kx = 0 and Nyquist columns dropped, as numpy's irfft does),
//               one complex inverse FFT, 1/(Hp Wp), crop, sRGB -> images
//               (V,Ho,Wo,C) f32
// Persistent CTAs, one per SM; warps take work items independently.
#include <algorithm>
#include <cmath>
#include <mutex>
#include <type_traits>
#include <vector>

#include "common.cuh"
#include "fft2.cuh"

namespace fdl {

namespace {

// sRGB-encoded value -> linear light (render.py:39-42; fused into the K0 load)
__device__ inline float srgb_dec_f(float x) {
  return x <= 0.04045f ? x / 12.92f : powf((fmaxf(x, 0.04045f) + 0.055f) / 1.055f, 2.4f);
}

__device__ inline float srgb_enc_f(float x) {
  x = fmaxf(x, 0.f);
  return x <= 0.0031308f ? x * 12.92f : 1.055f * powf(x, 1.0f / 2.4f) - 0.055f;
}

template <class PL>
struct Smem {
  float2 *tw2, *buf;
};
template <class PL>
__device__ inline Smem<PL> carve_and_build() {
  extern __shared__ __align__(16) float2 smem_f2[];
  Smem<PL> s;
  s.tw2 = smem_f2;
  s.buf = s.tw2 + PL::N + ((threadIdx.x >> 5) / PL::TEAM_WARPS) * PL::SLOTS;
  fft2::build_tables<PL>(s.tw2);
  __syncthreads();  // the only block barrier
  return s;
}


// ---------------------------------------------------------------- K0 rows
// transform tr -> (view j, row pair yp, channel c), channels fastest so the
// warps of a CTA read the same interleaved image rows at about the same time.
template <class PL>
__global__ void __launch_bounds__(PL::THREADS, 1) fwd_rows_kernel(const float* __restrict__ views, int m, int H, int W,
                                                                   int C, int pad, float2* __restrict__ t1, int srgb,
                                                                   int gcs) {
  constexpr int N = PL::N, M = PL::M, T = PL::T, P = PL::P, Whp = N / 2 + 1;
  const Smem<PL> s = carve_and_build<PL>();
  const int lane = threadIdx.x % PL::TL;  // lane within the team
  const int HP2 = (H + 1) / 2;
  const int ntr = m * HP2 * C;
  const int items = (ntr + T - 1) / T;
  // team index, made visibly warp-uniform (lets stage 1 use the uniform datapath)
  const int gw = __shfl_sync(0xffffffffu, blockIdx.x * PL::TEAMS + (threadIdx.x >> 5) / PL::TEAM_WARPS, 0);
  const int tw = gridDim.x * PL::TEAMS;
  // load mapping: lane = (t, n2, g) as in stage 1; rows n1 = g, g + LV, ...
  const int lg = lane >> 5, lt = (lane & 31) / M, ln2 = lane % M;  // warp lg loads rows n1 = lg (mod LV)
  // The teams of a CTA take consecutive transforms (= the channels of the same
  // image rows) and start every round together: their loads of the shared
  // interleaved sectors then reach L2 within microseconds of each other (at
  // TB/s an L2 line lives ~40 us; unsynchronised teams re-read the views 2.3x).
  for (int base = blockIdx.x * PL::TEAMS; base < items; base += tw) {
    __syncthreads();
    const int item = base + (gw - blockIdx.x * PL::TEAMS);
    if (item >= items) continue;
    {
      const int tr = item * T + lt;
      const bool ok = tr < ntr;
      const int c = tr % C, rest = tr / C;
      const int yp = rest % HP2, j = rest / HP2;
      const int y0 = 2 * yp;
      const bool has1 = y0 + 1 < H;
      const float* r0 = views + (((size_t)j * H + y0) * W) * C + c;
      const float* r1 = r0 + (size_t)W * C;
      // elements n1 = lg + LV i: x = x0 + i LV M; every load in flight at once
      const int x0 = lg * M + ln2 - pad;
      float2* dst = s.buf + lt * M + ln2 + lg * PL::RS;
      constexpr int NI = (P + PL::LV - 1) / PL::LV;
      float re[NI], im[NI];
#pragma unroll
      for (int i = 0; i < NI; ++i) {
        const int x = x0 + i * PL::LV * M;
        const bool in = ok && lg + i * PL::LV < P && (unsigned)x < (unsigned)W;
        re[i] = in ? __ldg(r0 + x * C) : 0.f;
        im[i] = (in && has1) ? __ldg(r1 + x * C) : 0.f;
      }
#pragma unroll
      for (int i = 0; i < NI; ++i) {
        if (lg + i * PL::LV < P) {
          float a = re[i], b = im[i];
          if (srgb) {
            a = srgb_dec_f(a);
            b = srgb_dec_f(b);
          }
          dst[i * PL::LV * PL::RS] = make_float2(a, b);
        }
      }
    }
    fft2::team_sync<PL>();
    fft2::transform<PL, false>(s.buf, s.tw2, lane);
    // unpack: Z = X + iY  ->  X[k] = (Z[k] + conj Z[N-k]) / 2,  Y[k] = (Z[k] - conj Z[N-k]) / 2i
#pragma unroll 1
    for (int t = 0; t < T; ++t) {
      const int tr = item * T + t;
      if (tr >= ntr) break;
      const int c = tr % C, rest = tr / C;
      const int yp = rest % HP2, j = rest / HP2;
      const int y0 = 2 * yp;
      const bool has1 = y0 + 1 < H;
      // T1 is blocked for the column pass: [plane][column block of 2^gcs][row][2^gcs columns],
      // so a column tile is ONE contiguous run of H * 2^gcs values (the scattered side of the
      // transpose is this pass's stores, which nothing waits for, not the column pass's loads)
      const int cblk = (Whp + (1 << gcs) - 1) >> gcs;
      float2* o0 = t1 + ((size_t)(j * C + c) * cblk * H + y0) * (size_t)(1 << gcs);
      const size_t bstep = (size_t)H << gcs;  // next column block, same row
      const int gmask = (1 << gcs) - 1;
      const float2* b = s.buf + t * M;
      // k = k1 + P k2 and N - k = m1 + P m2, stepped incrementally (TL < P)
      int k1 = lane % P, k2 = lane / P;
      int mk0 = lane == 0 ? 0 : N - lane;
      int m1 = mk0 % P, m2 = mk0 / P;
#pragma unroll 2
      for (int k = lane; k < Whp; k += PL::TL) {
        const float2 z = b[k1 * PL::RS + k2], zc = b[m1 * PL::RS + m2];
        float2* o = o0 + (size_t)(k >> gcs) * bstep + (k & gmask);
        o[0] = make_float2(0.5f * (z.x + zc.x), 0.5f * (z.y - zc.y));
        if (has1) o[1 << gcs] = make_float2(0.5f * (z.y + zc.y), 0.5f * (zc.x - z.x));
        k1 += PL::TL;
        if (k1 >= P) {
          k1 -= P;
          ++k2;
        }
        if (k == 0) {  // lane 0: N - 0 wrapped to 0; next is N - TL
          m1 = (N - PL::TL) % P;
          m2 = (N - PL::TL) / P;
        } else {
          m1 -= PL::TL;
          if (m1 < 0) {
            m1 += P;
            --m2;
          }
        }
      }
    }
    fft2::team_sync<PL>();  // the buffer is reused by the next item's loads
  }
}

// ---------------------------------------------------------------- column passes
// A group of QT teams takes GC adjacent columns of one plane: the group loads
// the GC-column tile row by row (lane = (row, column), column fastest) into
// the teams' buffers, each team transforms its T columns, and the group
// stores the outputs row by row again.  Column c of the group belongs to team
// c / T, transform c % T.
template <class PL>
__device__ __forceinline__ float2* col_slot(float2* buf0, int c, int n_slot_in) {
  return buf0 + (c / PL::T) * PL::SLOTS + (c % PL::T) * PL::M + n_slot_in;
}

// item = (plane, block of GC adjacent columns); output rows all N, sum |b|^2
// per (plane, column) into partial[plane * Whp + kx].
template <class PL>
__global__ void __launch_bounds__(PL::THREADS, 1) fwd_cols_kernel(const float2* __restrict__ t1, int planes, int H,
                                                                   int pad, int Whp, float2* __restrict__ spec,
                                                                   double* __restrict__ partial) {
  constexpr int N = PL::N, GC = PL::GC, GL = PL::GL, RG = GL / GC;  // RG rows per group-wide step
  const Smem<PL> s = carve_and_build<PL>();
  __shared__ double red[16][PL::GC];
  const int lane = threadIdx.x % PL::TL;                     // lane within the team
  const int gl = threadIdx.x % GL;                           // lane within the group
  const int group = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5) / (PL::TEAM_WARPS * PL::QT), 0);
  float2* gbuf = s.buf - ((threadIdx.x / PL::TL) % PL::QT) * PL::SLOTS;  // the group's first team buffer
  const int cblocks = (Whp + GC - 1) / GC;
  const int items = planes * cblocks;
  const int gid = blockIdx.x * PL::GROUPS + group, gstride = gridDim.x * PL::GROUPS;
  const int gc = gl % GC, gr = gl / GC;  // this lane's column and first row
  for (int item = gid; item < items; item += gstride) {
    const int pl = item / cblocks, kx0 = (item - pl * cblocks) * GC;
    const int kx = kx0 + gc;
    const bool colok = kx < Whp;
    {
      // blocked T1 (see fwd_rows_kernel): the tile is contiguous, row stride GC
      const float2* src = t1 + (size_t)item * H * GC + gc;
      constexpr int NI = (N + RG - 1) / RG;
      float2 v[NI];
#pragma unroll
      for (int i = 0; i < NI; ++i) {
        const int row = gr + i * RG - pad;
        v[i] = (colok && (unsigned)row < (unsigned)H && gr + i * RG < N) ? __ldg(src + row * GC)
                                                                          : make_float2(0.f, 0.f);
      }
#pragma unroll
      for (int i = 0; i < NI; ++i) {
        const int n = gr + i * RG;
        if (n < N) *col_slot<PL>(gbuf, gc, PL::slot_in(n, 0)) = v[i];
      }
    }
    fft2::group_sync<PL>();
    {  // the next item's tile into L2 while this one transforms
      const int nx = item + gstride;
      if (nx < items) {
        const float2* src = t1 + (size_t)nx * H * GC;  // contiguous: one prefetch per 128 bytes
        for (int e = gl * 16; e < H * GC; e += 16 * GL) prefetch_l2(src + e);
      }
    }
    fft2::transform<PL, false>(s.buf, s.tw2, lane);
    fft2::group_sync<PL>();
    double acc = 0.0;
    const int pl2 = item / cblocks, kxb = (item - pl2 * cblocks) * GC + gc;
    if (kxb < Whp) {
      float2* dst = spec + (size_t)pl2 * N * Whp + kxb + (size_t)gr * Whp;
      const float2* b = col_slot<PL>(gbuf, gc, 0);
      int k1 = gr % PL::P, k2 = gr / PL::P;  // k = gr + i RG = k1 + P k2
      static_assert(RG <= PL::P, "one wrap per step");
#pragma unroll 4
      for (int k = gr; k < N; k += RG, dst += (size_t)RG * Whp) {
        const float2 v = b[k1 * PL::RS + k2];
        *dst = v;
        acc += (double)fmaf(v.x, v.x, v.y * v.y);
        k1 += RG;
        if (k1 >= PL::P) {
          k1 -= PL::P;
          ++k2;
        }
      }
    }
    if (partial) {
      // lanes of one column (gl % GC == gc): warp reduce, then warps in order
#pragma unroll
      for (int o = GC; o < 32; o <<= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      if ((threadIdx.x & 31) < GC) red[threadIdx.x >> 5][gc] = acc;
      fft2::group_sync<PL>();
      if (gl < GC && kxb < Whp) {
        double tot = 0.0;
        const int w0 = group * PL::TEAM_WARPS * PL::QT;
        for (int w = 0; w < PL::TEAM_WARPS * PL::QT; ++w) tot += red[w0 + w][gc];
        partial[(size_t)pl2 * Whp + kxb] = tot;
      }
    }
    fft2::group_sync<PL>();  // buffers and red[] are reused by the next item
  }
}

// per view: the sum of its C * Whp column partials, fixed order
__global__ void sumsq_cols_kernel(const double* __restrict__ partial, int m, int per_view, double* __restrict__ out) {
  const int j = blockIdx.x;
  __shared__ double red[32];
  double acc = 0.0;
  // fixed partition: thread i sums elements i, i + blockDim, ... in order
  for (int i = threadIdx.x; i < per_view; i += blockDim.x) acc += partial[(size_t)j * per_view + i];
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double tot = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) tot += red[w];
    out[j] = tot;
  }
}

// ---------------------------------------------------------------- K4 cols
template <class PL>
__global__ void __launch_bounds__(PL::THREADS, 1) inv_cols_kernel(const float2* __restrict__ spec, int planes, int Whp,
                                                                   int pad, int Ho, float2* __restrict__ t2) {
  constexpr int N = PL::N, GC = PL::GC, GL = PL::GL, RG = GL / GC;
  const Smem<PL> s = carve_and_build<PL>();
  const int lane = threadIdx.x % PL::TL;
  const int gl = threadIdx.x % GL;
  const int group = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5) / (PL::TEAM_WARPS * PL::QT), 0);
  float2* gbuf = s.buf - ((threadIdx.x / PL::TL) % PL::QT) * PL::SLOTS;
  const int cblocks = (Whp + GC - 1) / GC;
  const int items = planes * cblocks;
  const int gid = blockIdx.x * PL::GROUPS + group, gstride = gridDim.x * PL::GROUPS;
  const int gc = gl % GC, gr = gl / GC;
  for (int item = gid; item < items; item += gstride) {
    const int pl = item / cblocks, kx0 = (item - pl * cblocks) * GC;
    const int kx = kx0 + gc;
    const bool colok = kx < Whp;
    {
      const float2* src = spec + (size_t)pl * N * Whp + kx;
      constexpr int NI = (N + RG - 1) / RG;
      float2 v[NI];
#pragma unroll
      for (int i = 0; i < NI; ++i) {
        const int row = gr + i * RG;
        v[i] = (colok && row < N) ? __ldg(src + row * Whp) : make_float2(0.f, 0.f);
      }
#pragma unroll
      for (int i = 0; i < NI; ++i) {
        const int n = gr + i * RG;
        if (n < N) *col_slot<PL>(gbuf, gc, PL::slot_in(n, 0)) = v[i];
      }
    }
    fft2::group_sync<PL>();
    {  // the next item's tile into L2 while this one transforms
      const int nx = item + gstride;
      if (nx < items) {
        const int npl = nx / cblocks, nkx = (nx - npl * cblocks) * GC + gc;
        const float2* src = spec + (size_t)npl * N * Whp + min(nkx, Whp - 1);
        for (int row = gr; row < N; row += 4 * RG) prefetch_l2(src + row * Whp);
      }
    }
    fft2::transform<PL, true>(s.buf, s.tw2, lane);
    fft2::group_sync<PL>();
    const int pl2 = item / cblocks, kxb = (item - pl2 * cblocks) * GC + gc;
    if (kxb < Whp) {
      float2* dst = t2 + (size_t)pl2 * Ho * Whp + kxb + (size_t)gr * Whp;
      const float2* b = col_slot<PL>(gbuf, gc, 0);
      int k = gr + pad, k1 = k % PL::P, k2 = k / PL::P;  // output row y = index y + pad
      static_assert(RG <= PL::P, "one wrap per step");
#pragma unroll 2
      for (int y = gr; y < Ho; y += RG, dst += (size_t)RG * Whp) {
        *dst = b[k1 * PL::RS + k2];
        k1 += RG;
        if (k1 >= PL::P) {
          k1 -= PL::P;
          ++k2;
        }
      }
    }
    fft2::group_sync<PL>();
  }
}

// ---------------------------------------------------------------- K4 rows
template <class PL>
__global__ void __launch_bounds__(PL::THREADS, 1) inv_rows_kernel(const float2* __restrict__ t2, int V, int C, int Ho,
                                                                   int Wo, int pad, int srgb, float scale,
                                                                   float* __restrict__ out) {
  constexpr int N = PL::N, M = PL::M, T = PL::T, Whp = N / 2 + 1;
  const Smem<PL> s = carve_and_build<PL>();
  const int lane = threadIdx.x % PL::TL;  // lane within the team
  const int HP2 = (Ho + 1) / 2;
  const int ntr = V * HP2 * C;
  const int items = (ntr + T - 1) / T;
  // team index, made visibly warp-uniform (lets stage 1 use the uniform datapath)
  const int gw = __shfl_sync(0xffffffffu, blockIdx.x * PL::TEAMS + (threadIdx.x >> 5) / PL::TEAM_WARPS, 0);
  const int tw = gridDim.x * PL::TEAMS;
  // every load of a transform's two input rows in flight at once (<= 18 x 2 float2 per lane)
  constexpr int ULR = (Whp + PL::TL - 1) / PL::TL < 18 ? (Whp + PL::TL - 1) / PL::TL : 18;
  // rounds start together (see fwd_rows_kernel): the teams' channel-interleaved
  // stores to the same sectors then merge in L2
  for (int base = blockIdx.x * PL::TEAMS; base < items; base += tw) {
    __syncthreads();
    const int item = base + (gw - blockIdx.x * PL::TEAMS);
    if (item >= items) continue;
    // Hermitian completion: Z[k] = X[k] + i Y[k], Z[N-k] = conj X[k] + i conj Y[k]
#pragma unroll 1
    for (int t = 0; t < T; ++t) {
      const int tr = item * T + t;
      const bool ok = tr < ntr;
      const int c = tr % C, rest = tr / C;
      const int yp = rest % HP2, v = rest / HP2;
      const int y0 = 2 * yp;
      const bool has1 = y0 + 1 < Ho;
      const float2* i0 = t2 + (((size_t)v * C + c) * Ho + y0) * Whp;
      const float2* i1 = i0 + Whp;
      float2* b = s.buf + t * M;
#pragma unroll 1
      for (int k0 = lane; k0 < Whp; k0 += PL::TL * ULR) {
        float2 X[ULR], Y[ULR];
#pragma unroll
        for (int u = 0; u < ULR; ++u) {
          const int k = k0 + PL::TL * u;
          X[u] = (ok && k < Whp) ? __ldg(i0 + k) : make_float2(0.f, 0.f);
          Y[u] = (ok && has1 && k < Whp) ? __ldg(i1 + k) : make_float2(0.f, 0.f);
        }
#pragma unroll
        for (int u = 0; u < ULR; ++u) {
          const int k = k0 + PL::TL * u;
          if (k >= Whp) break;
          const bool self = k == 0 || 2 * k == N;  // self-conjugate: keep the real parts only
          if (self) {
            X[u].y = 0.f;
            Y[u].y = 0.f;
          }
          b[PL::slot_in(k, 0)] = make_float2(X[u].x - Y[u].y, X[u].y + Y[u].x);
          if (!self) b[PL::slot_in(N - k, 0)] = make_float2(X[u].x + Y[u].y, Y[u].x - X[u].y);
        }
      }
    }
    fft2::team_sync<PL>();
    {  // the next item's input rows into L2 while this one transforms
      for (int t = 0; t < T; ++t) {
        const int tr = (item + tw) * T + t;
        if (tr >= ntr) break;
        const int c = tr % C, rest = tr / C;
        const int yp = rest % HP2, v = rest / HP2;
        const float2* i0 = t2 + (((size_t)v * C + c) * Ho + 2 * yp) * Whp;
        for (int e = lane * 16; e < 2 * Whp; e += 16 * PL::TL) prefetch_l2(i0 + e);
      }
    }
    fft2::transform<PL, true>(s.buf, s.tw2, lane);
#pragma unroll 1
    for (int t = 0; t < T; ++t) {
      const int tr = item * T + t;
      if (tr >= ntr) break;
      const int c = tr % C, rest = tr / C;
      const int yp = rest % HP2, v = rest / HP2;
      const int y0 = 2 * yp;
      const bool has1 = y0 + 1 < Ho;
      float* o0 = out + (((size_t)v * Ho + y0) * Wo) * C + c;
      const float2* b = s.buf + t * M;
      // sample n = x + pad sits at slot (n % P) RS + n / P: stepped incrementally (TL < 2 P)
      static_assert(PL::TL < 2 * PL::P, "at most two wraps per step");
      int n1 = (lane + pad) % PL::P, n2 = (lane + pad) / PL::P;
      const size_t ostep = (size_t)PL::TL * C;
      float* p0 = o0 + (size_t)lane * C;
#pragma unroll 4
      for (int x = lane; x < Wo; x += PL::TL, p0 += ostep) {
        const float2 z = b[n1 * PL::RS + n2];
        float a0 = z.x * scale, a1 = z.y * scale;
        if (srgb) {
          a0 = srgb_enc_f(a0);
          a1 = srgb_enc_f(a1);
        }
        p0[0] = a0;
        if (has1) p0[(size_t)Wo * C] = a1;
        n1 += PL::TL;
        if (n1 >= PL::P) {
          n1 -= PL::P;
          ++n2;
        }
        if (PL::TL > PL::P && n1 >= PL::P) {
          n1 -= PL::P;
          ++n2;
        }
      }
    }
    fft2::team_sync<PL>();
  }
}

inline size_t al256(size_t x) { return (x + 255) & ~(size_t)255; }

int sm_count() {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms > 0 ? sms : 148;
}

template <class PL, class KFN>
int prepare(KFN k) {
  // the attribute is per device: set it on every call (cheap) so a thread
  // that switches devices never launches without it
  FDL_CUDA_CHECK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, PL::SMEM));
  return FDL_OK;
}

template <class PL>
int grid_for_groups(int items) {
  return std::max(1, std::min(sm_count(), (items + PL::GROUPS - 1) / PL::GROUPS));
}

template <class PL>
int grid_for_items(int items) {
  const int per = PL::TEAMS;
  return std::max(1, std::min(sm_count(), (items + per - 1) / per));
}

// ---------------------------------------------------------------- plans
// dispatch a side N = P * 2^a to a compile-time plan
template <class F>
int with_plan(int N, F&& f) {
  switch (N) {
    case 67 * 2: return f(fft2::Plan<67, 2>());
    case 67 * 4: return f(fft2::Plan<67, 4>());
    case 67 * 8: return f(fft2::Plan<67, 8>());
    case 67 * 32: return f(fft2::Plan<67, 32>());
    case 131 * 4: return f(fft2::Plan<131, 4>());
    case 131 * 8: return f(fft2::Plan<131, 8>());
    default: return fail(FDL_ERR_UNSUPPORTED, "FFT engine: unsupported side");
  }
}

bool side_supported(int N) {  // keep in sync with with_plan
  switch (N) {
    case 67 * 2: case 67 * 4: case 67 * 8: case 67 * 32:
    case 131 * 4: case 131 * 8:
      return true;
    default:
      return false;
  }
}

thread_local int t_force_cufft = 0;

template <int P, int LV, int KP, int K>
void fill_tw1(std::vector<float2>& out) {
  constexpr int H = (P - 1) / 2;
  out.assign((size_t)H * LV * KP, make_float2(0.f, 0.f));
  for (int j = 1; j <= H; ++j)
    for (int g = 0; g < LV; ++g)
      for (int i = 0; i < K; ++i) {
        const int k = g * K + i + 1;
        if (k > H) continue;
        const double a = 2.0 * M_PI * (double)((j * k) % P) / (double)P;
        out[((size_t)(j - 1) * LV + g) * KP + i] = make_float2((float)std::cos(a), (float)std::sin(a));
      }
}

}  // namespace

namespace fft2 {
int fft2_upload_constants() {
  static std::mutex mu;
  static bool done[64] = {};
  int dev = 0;
  FDL_CUDA_CHECK(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(mu);
  if (dev < 64 && done[dev]) return FDL_OK;
  std::vector<float2> t;
  using P67 = Plan<67, 32>;
  using P131 = Plan<131, 8>;
  fill_tw1<67, P67::LV, P67::KP, P67::K>(t);
  FDL_CUDA_CHECK(cudaMemcpyToSymbol(c_tw1_67, t.data(), t.size() * sizeof(float2)));
  fill_tw1<131, P131::LV, P131::KP, P131::K>(t);
  FDL_CUDA_CHECK(cudaMemcpyToSymbol(c_tw1_131, t.data(), t.size() * sizeof(float2)));
  if (dev < 64) done[dev] = true;
  return FDL_OK;
}
}  // namespace fft2

extern "C" int fdl_fft_force_cufft(int32_t force_cufft) {
  t_force_cufft = force_cufft ? 1 : 0;
  return FDL_OK;
}

// ------------------------------------------------------------------ entry points used by k0_spectra.cu
bool fft_cufft_forced() { return t_force_cufft != 0; }

bool fft_engine_applies(int Hp, int Wp, int C) {
  return !t_force_cufft && C >= 1 && C <= 4 && side_supported(Hp) && side_supported(Wp);
}

// column-group width of the column plan of side Hp (the block width of T1)
int col_group(int Hp) {
  int gc = 8;
  with_plan(Hp, [&](auto pl) {
    gc = decltype(pl)::GC;
    return FDL_OK;
  });
  return gc;
}

size_t t1_elems(int m, int H, int W, int C, int pad) {
  const int Hp = H + 2 * pad, Wp = W + 2 * pad, Whp = Wp / 2 + 1, gc = col_group(Hp);
  return (size_t)m * C * ((Whp + gc - 1) / gc) * H * gc;
}

size_t engine_fwd_ws(int m, int H, int W, int C, int pad) {
  const int Wp = W + 2 * pad, Whp = Wp / 2 + 1;
  return al256(sizeof(float2) * t1_elems(m, H, W, C, pad)) + al256(sizeof(double) * (size_t)m * C * Whp);
}

int engine_fwd(const float* views, int m, int H, int W, int C, int pad, float2* spectra, double* view_sumsq,
               void* ws, cudaStream_t st, int srgb) {
  if (int e = fft2::fft2_upload_constants()) return e;
  const int Hp = H + 2 * pad, Wp = W + 2 * pad, Whp = Wp / 2 + 1;
  float2* t1 = reinterpret_cast<float2*>(ws);
  double* partial =
      reinterpret_cast<double*>(reinterpret_cast<char*>(ws) + al256(sizeof(float2) * t1_elems(m, H, W, C, pad)));
  const int gc = col_group(Hp);
  int gcs = 0;
  while ((1 << gcs) < gc) ++gcs;
  int rc = with_plan(Wp, [&](auto pl) {
    using PL = decltype(pl);
    auto k = fwd_rows_kernel<PL>;
    int r = prepare<PL>(k);
    if (r) return r;
    const int items = (m * ((H + 1) / 2) * C + PL::T - 1) / PL::T;
    k<<<grid_for_items<PL>(items), PL::THREADS, PL::SMEM, st>>>(views, m, H, W, C, pad, t1, srgb, gcs);
    FDL_LAUNCH_CHECK("fwd_rows_kernel");
    return FDL_OK;
  });
  if (rc) return rc;
  rc = with_plan(Hp, [&](auto pl) {
    using PL = decltype(pl);
    auto k = fwd_cols_kernel<PL>;
    int r = prepare<PL>(k);
    if (r) return r;
    const int items = m * C * ((Whp + PL::GC - 1) / PL::GC);
    k<<<grid_for_groups<PL>(items), PL::THREADS, PL::SMEM, st>>>(t1, m * C, H, pad, Whp, spectra,
                                                               view_sumsq ? partial : nullptr);
    FDL_LAUNCH_CHECK("fwd_cols_kernel");
    return FDL_OK;
  });
  if (rc) return rc;
  if (view_sumsq) {
    sumsq_cols_kernel<<<m, 256, 0, st>>>(partial, m, C * Whp, view_sumsq);
    FDL_LAUNCH_CHECK("sumsq_cols_kernel");
  }
  return FDL_OK;
}

size_t engine_inv_ws(int V, int C, int Hp, int Wp) {
  return al256(sizeof(float2) * (size_t)V * C * Hp * (Wp / 2 + 1));
}

int engine_inv(const float2* spectra, int V, int C, int Hp, int Wp, int pad, int Ho, int Wo, int srgb, float* images,
               void* ws, cudaStream_t st) {
  if (int e = fft2::fft2_upload_constants()) return e;
  const int Whp = Wp / 2 + 1;
  float2* t2 = reinterpret_cast<float2*>(ws);
  const float scale = (float)(1.0 / ((double)Hp * (double)Wp));
  int rc = with_plan(Hp, [&](auto pl) {
    using PL = decltype(pl);
    auto k = inv_cols_kernel<PL>;
    int r = prepare<PL>(k);
    if (r) return r;
    const int items = V * C * ((Whp + PL::GC - 1) / PL::GC);
    k<<<grid_for_groups<PL>(items), PL::THREADS, PL::SMEM, st>>>(spectra, V * C, Whp, pad, Ho, t2);
    FDL_LAUNCH_CHECK("inv_cols_kernel");
    return FDL_OK;
  });
  if (rc) return rc;
  return with_plan(Wp, [&](auto pl) {
    using PL = decltype(pl);
    auto k = inv_rows_kernel<PL>;
    int r = prepare<PL>(k);
    if (r) return r;
    const int items = (V * ((Ho + 1) / 2) * C + PL::T - 1) / PL::T;
    k<<<grid_for_items<PL>(items), PL::THREADS, PL::SMEM, st>>>(t2, V, C, Ho, Wo, pad, srgb, scale, images);
    FDL_LAUNCH_CHECK("inv_rows_kernel");
    return FDL_OK;
  });
}

}  // namespace fdl
