// Shared-memory FFT engine for lengths N = P * M (P odd, M = 2^a <= 32) that
// cuFFT handles through its slow large-prime path (C2's 536 = 8 * 67,
// C2b's 1048 = 8 * 131, C4's 2144 = 32 * 67).
//
// One CTA transforms a batch of B length-N complex vectors held in shared
// memory, slot(r, c, b) = r * SR + c * SC + b, by one Cooley-Tukey split
// N = P x M:
//   natural index  n = M * n1 + n2   lives in slot(n1, n2, b)
//   frequency      k = k1 + P * k2   ends up in slot(k1, k2, b)
// stage 1: for every (n2, b), a length-P DFT over n1, computed directly with
//          the symmetric pairing x_j +- x_{P-j} (P^2/4 real multiply-adds per
//          pair of outputs instead of P^2 complex ones), then the inter-stage
//          twiddle W_N^{n2 k1};
// stage 2: for every (k1, b), a radix-2 length-M DFT in registers.
// Twiddles are fp32 roundings of fp64 sincospi values (tables in shared
// memory, built by the CTA).  Forward = exp(-2 pi i nk/N) (numpy's sign),
// inverse = exp(+...) without the 1/N (callers scale).
#pragma once
#include <cuda_runtime.h>

namespace fdl {
namespace fft {

constexpr int KOUT = 12;        // output pairs per stage-1 work item
// CTA size cap per power-of-two factor: stage 2 keeps 2M floats live per
// thread, so larger M needs more registers per thread (no spills at these caps)
__host__ __device__ constexpr int max_threads(int M) { return M >= 16 ? 384 : 320; }

// n / d for 0 <= n < 2^31 by multiply-high (round-up method): 3 instructions
// instead of the ~20 of a runtime 32-bit division.
struct FastDiv {
  unsigned d, mul, shr;
  __host__ static FastDiv make(unsigned d) {
    FastDiv f{d, 0u, 0u};
    while ((1ull << f.shr) < d) ++f.shr;
    f.mul = (unsigned)(((1ull << 32) * ((1ull << f.shr) - d)) / d + 1);
    if (d == 1) f.mul = 0;
    return f;
  }
  __device__ __forceinline__ int div(int n) const {
    return (int)((__umulhi((unsigned)n, mul) + (unsigned)n) >> shr);
  }
};

struct Geo {
  int N, P, M, h, G;  // h = (P-1)/2 output pairs, G = ceil(h / KOUT) groups
  int B, SC, SR;      // batch and slot strides (complex units)
  FastDiv divP;
  __host__ __device__ int slots() const { return P * SR; }
  __host__ __device__ int tw1_len() const { return h * G * KOUT; }  // float2 entries
};

__host__ inline bool split(int N, int* P, int* M) {
  int m = 1;
  while (N % (2 * m) == 0) m *= 2;
  *P = N / m;
  *M = m;
  return m <= 32 && *P >= 3 && *P <= 255 && (*P & 1);
}

// Engine applies when N splits and the odd part has a prime factor >= 11
// (cuFFT's radix-2/3/5/7 kernels are fast; its large-prime path is not).
__host__ inline bool wanted(int N) {
  int P, M;
  if (!split(N, &P, &M)) return false;
  int p = P;
  for (int f : {3, 5, 7})
    while (p % f == 0) p /= f;
  return p >= 11;
}

__host__ inline Geo make_geo(int N, int B) {
  Geo g;
  g.N = N;
  split(N, &g.P, &g.M);
  g.h = (g.P - 1) / 2;
  g.G = (g.h + KOUT - 1) / KOUT;
  g.divP = FastDiv::make(g.P);
  g.B = B;
  g.SC = B + 1;
  g.SR = g.M * g.SC;
  if ((g.SR & 1) == 0) g.SR += 1;  // odd row stride: conflict-free walks over k1
  return g;
}

__host__ inline int threads_for(const Geo& g) { return g.B * g.M * g.G; }
__host__ inline size_t smem_bytes(const Geo& g) {
  return sizeof(float2) * ((size_t)g.slots() + g.tw1_len() + g.N);
}

// cos/sin(2 pi e / 32)
__device__ __constant__ static float kCos32[32] = {
    1.000000000e+00f,  9.807852804e-01f,  9.238795325e-01f,  8.314696123e-01f,  7.071067812e-01f,
    5.555702330e-01f,  3.826834324e-01f,  1.950903220e-01f,  0.0f,              -1.950903220e-01f,
    -3.826834324e-01f, -5.555702330e-01f, -7.071067812e-01f, -8.314696123e-01f, -9.238795325e-01f,
    -9.807852804e-01f, -1.000000000e+00f, -9.807852804e-01f, -9.238795325e-01f, -8.314696123e-01f,
    -7.071067812e-01f, -5.555702330e-01f, -3.826834324e-01f, -1.950903220e-01f, 0.0f,
    1.950903220e-01f,  3.826834324e-01f,  5.555702330e-01f,  7.071067812e-01f,  8.314696123e-01f,
    9.238795325e-01f,  9.807852804e-01f};

// Build the twiddle tables in shared memory (all threads).
//   tw1[(j-1) * G*KOUT + kk] = (cos, sin)(2 pi j (kk+1) / P), 0 beyond h
//   tw2[e] = (cos, sin)(2 pi e / N)
__device__ inline void build_tables(const Geo& g, float2* tw1, float2* tw2) {
  const int gk = g.G * KOUT;
  for (int i = threadIdx.x; i < g.h * gk; i += blockDim.x) {
    const int j = i / gk + 1, k = i % gk + 1;
    float2 w = make_float2(0.f, 0.f);
    if (k <= g.h) {
      double s, c;
      sincospi(2.0 * (double)((j * k) % g.P) / (double)g.P, &s, &c);
      w = make_float2((float)c, (float)s);
    }
    tw1[i] = w;
  }
  for (int e = threadIdx.x; e < g.N; e += blockDim.x) {
    double s, c;
    sincospi(2.0 * (double)e / (double)g.N, &s, &c);
    tw2[e] = make_float2((float)c, (float)s);
  }
}

// Stage 1 (all threads of the CTA; blockDim.x >= B*M*G).  Contains the two
// barriers that separate reading the inputs from overwriting them in place.
template <int M, bool INV>
__device__ inline void stage1(const Geo& g, float2* data, const float2* tw1, const float2* tw2) {
  const int item = threadIdx.x;
  const bool active = item < g.B * M * g.G;
  const int b = item % g.B;
  const int n2 = (item / g.B) % M;
  const int grp = item / (g.B * M);
  float2 A[KOUT], D[KOUT];
  float2 x0 = make_float2(0.f, 0.f), ssum = make_float2(0.f, 0.f);
  if (active) {
    const float2* x = data + n2 * g.SC + b;
    x0 = x[0];
#pragma unroll
    for (int t = 0; t < KOUT; ++t) {
      A[t] = x0;
      D[t] = make_float2(0.f, 0.f);
    }
    const float4* tw = reinterpret_cast<const float4*>(tw1 + grp * KOUT);
    const int twstride = g.G * KOUT / 2;  // float4 per j
    const float2* xa = x + g.SR;
    const float2* xc = x + (g.P - 1) * g.SR;
#pragma unroll 1
    for (int j = 1; j <= g.h; ++j) {
      const float2 a = *xa, c = *xc;
      xa += g.SR;
      xc -= g.SR;
      const float2 s = make_float2(a.x + c.x, a.y + c.y);
      const float2 d = make_float2(a.x - c.x, a.y - c.y);
      ssum.x += s.x;
      ssum.y += s.y;
#pragma unroll
      for (int t = 0; t < KOUT / 2; ++t) {
        const float4 w = tw[t];  // (cos, sin) of outputs 2t, 2t+1
        A[2 * t].x = fmaf(s.x, w.x, A[2 * t].x);
        A[2 * t].y = fmaf(s.y, w.x, A[2 * t].y);
        D[2 * t].x = fmaf(d.x, w.y, D[2 * t].x);
        D[2 * t].y = fmaf(d.y, w.y, D[2 * t].y);
        A[2 * t + 1].x = fmaf(s.x, w.z, A[2 * t + 1].x);
        A[2 * t + 1].y = fmaf(s.y, w.z, A[2 * t + 1].y);
        D[2 * t + 1].x = fmaf(d.x, w.w, D[2 * t + 1].x);
        D[2 * t + 1].y = fmaf(d.y, w.w, D[2 * t + 1].y);
      }
      tw += twstride;
    }
  }
  __syncthreads();
  if (active) {
    float2* y = data + n2 * g.SC + b;
    // twiddled store of output k1: W_N^{sign n2 k1}
    auto put = [&](int k1, float2 v) {
      const float2 w = tw2[n2 * k1];
      const float ws = INV ? w.y : -w.y;
      y[k1 * g.SR] = make_float2(v.x * w.x - v.y * ws, v.x * ws + v.y * w.x);
    };
    if (grp == 0) y[0] = make_float2(x0.x + ssum.x, x0.y + ssum.y);  // k1 = 0: W = 1
#pragma unroll
    for (int t = 0; t < KOUT; ++t) {
      const int k = grp * KOUT + 1 + t;
      if (k <= g.h) {
        // X_k = A -+ i D, X_{P-k} = A +- i D   (forward: upper signs)
        const float2 iD = make_float2(-D[t].y, D[t].x);
        const float2 lo = INV ? make_float2(A[t].x + iD.x, A[t].y + iD.y) : make_float2(A[t].x - iD.x, A[t].y - iD.y);
        const float2 hi = INV ? make_float2(A[t].x - iD.x, A[t].y - iD.y) : make_float2(A[t].x + iD.x, A[t].y + iD.y);
        put(k, lo);
        put(g.P - k, hi);
      }
    }
  }
  __syncthreads();
}

template <int M>
__host__ __device__ constexpr int bitrev(int k) {
  int r = 0;
#pragma unroll
  for (int s = 1; s < M; s <<= 1) {
    r = (r << 1) | (k & 1);
    k >>= 1;
  }
  return r;
}

// One radix-2 DIF level of span SPAN on a register array, then the next.
template <int M, int SPAN, bool INV>
__device__ __forceinline__ void dif_level(float2 (&v)[M]) {
  if constexpr (SPAN >= 1) {
#pragma unroll
    for (int st = 0; st < M; st += 2 * SPAN) {
#pragma unroll
      for (int t = 0; t < SPAN; ++t) {
        const float2 a = v[st + t], c = v[st + t + SPAN];
        v[st + t] = make_float2(a.x + c.x, a.y + c.y);
        const float2 dd = make_float2(a.x - c.x, a.y - c.y);
        const int e = t * (32 / (2 * SPAN));
        if (e == 0) {
          v[st + t + SPAN] = dd;
        } else {
          const float wc = kCos32[e];
          const float ws = INV ? kCos32[(e + 24) & 31] : -kCos32[(e + 24) & 31];  // sin = cos(x - pi/2)
          v[st + t + SPAN] = make_float2(dd.x * wc - dd.y * ws, dd.x * ws + dd.y * wc);
        }
      }
    }
    dif_level<M, SPAN / 2, INV>(v);
  }
}

// Stage 2: every thread takes (k1, b) items; in place, no barrier needed
// inside (each item owns its M slots).  Caller syncs afterwards.
template <int M, bool INV>
__device__ inline void stage2(const Geo& g, float2* data) {
  if (M == 1) return;
  const int items = g.P * g.B;
  for (int it = threadIdx.x; it < items; it += blockDim.x) {
    const int b = it % g.B, k1 = it / g.B;
    float2* p = data + k1 * g.SR + b;
    float2 v[M];
#pragma unroll
    for (int i = 0; i < M; ++i) v[i] = p[i * g.SC];
    dif_level<M, M / 2, INV>(v);  // radix-2 decimation in frequency, bit-reversed output
#pragma unroll
    for (int i = 0; i < M; ++i) p[bitrev<M>(i) * g.SC] = v[i];  // v[i] = X[bitrev(i)]
  }
}

// slot of natural index n / of frequency k
template <int M>
__device__ __forceinline__ int slot_in(const Geo& g, int n) { return (n / M) * g.SR + (n % M) * g.SC; }
__device__ __forceinline__ int slot_out(const Geo& g, int k) {
  const int k2 = g.divP.div(k);
  return (k - k2 * g.P) * g.SR + k2 * g.SC;
}

}  // namespace fft
}  // namespace fdl
