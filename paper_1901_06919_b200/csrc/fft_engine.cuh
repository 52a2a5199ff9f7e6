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

#include "common.cuh"

namespace fdl {
namespace fft {

constexpr int KOUT = 12;        // output pairs per stage-1 work item
// CTA size cap per power-of-two factor: stage 2 keeps 2M floats live per
// thread, so larger M needs more registers per thread (no spills at these caps)
// Rows kernels: 288 threads, 2 CTAs/SM; cols kernels: 192 threads, 3 CTAs/SM
// (register caps 113 / 113); M >= 16: one 384-thread CTA per SM.
__host__ __device__ constexpr int max_threads(int M) { return M >= 16 ? 384 : 320; }
__host__ __device__ constexpr int rows_threads(int M) { return M >= 16 ? 384 : 288; }
__host__ __device__ constexpr int rows_blocks(int M) { return M >= 16 ? 1 : 2; }
__host__ __device__ constexpr int cols_threads(int M) { return M >= 16 ? 384 : 192; }
__host__ __device__ constexpr int cols_blocks(int M) { return M >= 16 ? 1 : 3; }

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

// Shared-memory wavefronts of one warp's 8-byte accesses (bank = word % 32;
// a bank serves one distinct word per wavefront).
__host__ inline int warp_wavefronts(const int* slots) {
  int best = 0;
  for (int bank = 0; bank < 32; ++bank) {
    int words[64], nw = 0;
    for (int l = 0; l < 32; ++l)
      for (int h = 0; h < 2; ++h) {
        const int w = 2 * slots[l] + h;
        if (w % 32 != bank) continue;
        bool seen = false;
        for (int i = 0; i < nw; ++i) seen |= words[i] == w;
        if (!seen) words[nw++] = w;
      }
    best = nw > best ? nw : best;
  }
  return best;
}

// Pick the slot strides (SC, SR) that minimise bank conflicts over the
// kernels' access patterns (lane -> slot maps of the loads, both stages and
// the stores; rows = the row kernels' column-owning threads, else the column
// kernels' (b, row) threads).
__host__ inline void tune_strides(Geo& g, bool rows, int threads) {
  const int B = g.B, M = g.M, P = g.P;
  const int warps = (threads + 31) / 32;
  long best_cost = -1;
  int bsc = g.SC, bsr = g.SR;
  for (int sc = B; sc <= B + 8; ++sc) {
    for (int sr = M * sc; sr <= M * sc + 15; ++sr) {
      if (M == 1 && sr != sc * M && sr > sc + 15) break;
      auto sin = [&](int n) { return (n / M) * sr + (n % M) * sc; };
      auto sout = [&](int k) { return (k % P) * sr + (k / P) * sc; };
      long cost = 0;
      int sl[32];
      for (int w = 0; w < warps; ++w) {
        for (int l = 0; l < 32; ++l) {  // stage 1 reads (and per-j strides)
          const int t = 32 * w + l;
          sl[l] = (t / B % M) * sc + t % B + 3 * sr;
        }
        cost += 2 * warp_wavefronts(sl);
        for (int l = 0; l < 32; ++l) {  // stage 1 writes
          const int t = 32 * w + l;
          sl[l] = (t / (B * M) * KOUT + 1) * sr + (t / B % M) * sc + t % B;
        }
        cost += warp_wavefronts(sl);
        for (int l = 0; l < 32; ++l) {  // stage 2
          const int t = 32 * w + l;
          sl[l] = (t / B % P) * sr + 1 * sc + t % B;
        }
        cost += warp_wavefronts(sl);
        if (rows) {
          for (int l = 0; l < 32; ++l) sl[l] = sin((32 * w + l) % g.N);  // loads: thread owns n
          cost += warp_wavefronts(sl);
          for (int l = 0; l < 32; ++l) sl[l] = sout((32 * w + l) % g.N);  // unpack / output: owns k
          cost += warp_wavefronts(sl);
        } else {
          for (int l = 0; l < 32; ++l) {
            const int t = 32 * w + l;
            sl[l] = sin((t / B + 5) % g.N) + t % B;
          }
          cost += warp_wavefronts(sl);
          for (int l = 0; l < 32; ++l) {
            const int t = 32 * w + l;
            sl[l] = sout((t / B) % g.N) + t % B;
          }
          cost += warp_wavefronts(sl);
        }
      }
      if (best_cost < 0 || cost < best_cost) {
        best_cost = cost;
        bsc = sc;
        bsr = sr;
      }
    }
  }
  g.SC = bsc;
  g.SR = bsr;
}
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
  // packed (re, im) pairs: one FFMA2 per complex-by-real multiply-add
  u64 A[KOUT], D[KOUT];
  u64 x0 = 0ull, ssum = 0ull;
  if (active) {
    const float2* x = data + n2 * g.SC + b;
    x0 = as_u64(x[0]);
#pragma unroll
    for (int t = 0; t < KOUT; ++t) {
      A[t] = x0;
      D[t] = 0ull;
    }
    const float4* tw = reinterpret_cast<const float4*>(tw1 + grp * KOUT);
    const int twstride = g.G * KOUT / 2;  // float4 per j
    const float2* xa = x + g.SR;
    const float2* xc = x + (g.P - 1) * g.SR;
#pragma unroll 1
    for (int j = 1; j <= g.h; ++j) {
      const u64 a = as_u64(*xa), c = as_u64(*xc);
      xa += g.SR;
      xc -= g.SR;
      const u64 sv = add2(a, c), dv = sub2(a, c);
      ssum = add2(ssum, sv);
#pragma unroll
      for (int t = 0; t < KOUT / 2; ++t) {
        const float4 w = tw[t];  // (cos, sin) of outputs 2t, 2t+1
        ffma2s(A[2 * t], sv, w.x);
        ffma2s(D[2 * t], dv, w.y);
        ffma2s(A[2 * t + 1], sv, w.z);
        ffma2s(D[2 * t + 1], dv, w.w);
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
    if (grp == 0) y[0] = as_f2(add2(x0, ssum));  // k1 = 0: W = 1
#pragma unroll
    for (int t = 0; t < KOUT; ++t) {
      const int k = grp * KOUT + 1 + t;
      if (k <= g.h) {
        // X_k = A -+ i D, X_{P-k} = A +- i D   (forward: upper signs)
        const float2 At = as_f2(A[t]), Dt = as_f2(D[t]);
        const float2 iD = make_float2(-Dt.y, Dt.x);
        const float2 lo = INV ? make_float2(At.x + iD.x, At.y + iD.y) : make_float2(At.x - iD.x, At.y - iD.y);
        const float2 hi = INV ? make_float2(At.x - iD.x, At.y - iD.y) : make_float2(At.x + iD.x, At.y + iD.y);
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
  const int kstep = blockDim.x / g.B;  // threads beyond kstep*B idle here
  const int b = threadIdx.x % g.B;
  for (int k1 = threadIdx.x / g.B; k1 < g.P && threadIdx.x < kstep * g.B; k1 += kstep) {
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
