// Mixed-radix shared-memory FFT for lengths N = R0 * R1 * R2 with small
// radices (products of 2, 3, 4, 5): the 1920 x 1080 grid of config 5
// (1920 = 16 * 8 * 15, 1080 = 8 * 9 * 15), which cuFFT runs as three
// HBM round trips per axis (K4 at 0.10 of the HBM roofline in round 1).
//
// A CTA holds a tile of vectors in shared memory and transforms them in place
// by three decimation-in-frequency passes; pass p takes radix-R_p butterflies
// over elements M_p = L_p / R_p apart inside blocks of length L_p (L_0 = N,
// L_{p+1} = M_p), multiplies output k1 of the butterfly at offset n2 by
// W_{L_p}^{n2 k1} (per-pass tables laid out so a warp's reads are consecutive),
// and leaves frequency k at the mixed-radix digit-reversed position
//   pos(k) = (k % R0) M0 + ((k / R0) % R1) M1 + k / (R0 R1),
// which the caller's store loop reads (no reordering pass).  Butterflies are
// computed in registers by a compile-time Cooley-Tukey split of the radix
// (Dft<R>), all twiddles inside a butterfly are compile-time constants.
//
// Two tile layouts (element n of vector b):
//   COLS  [n][b]   b fastest: the tile is B adjacent columns of a plane, every
//                  shared access of a half-warp covers one 128-byte row;
//   ROWS  [b][n]   n fastest, one pad element per top-level block when M0 is
//                  even (so the digit-reversed output reads of consecutive k hit
//                  distinct banks) and one per vector.
#pragma once
#include <cuda_runtime.h>

#include "common.cuh"

namespace fdl {
namespace mr {

// ---------------------------------------------------------------- compile-time roots of unity
__host__ __device__ constexpr double c_sin_series(double x) {  // |x| <= pi
  double term = x, sum = x;
  for (int i = 1; i < 20; ++i) {
    term *= -x * x / ((2.0 * i) * (2.0 * i + 1.0));
    sum += term;
  }
  return sum;
}
__host__ __device__ constexpr double c_cos_series(double x) {
  double term = 1.0, sum = 1.0;
  for (int i = 1; i < 20; ++i) {
    term *= -x * x / ((2.0 * i - 1.0) * (2.0 * i));
    sum += term;
  }
  return sum;
}
__host__ __device__ constexpr double c_angle(int e, int R) {  // 2 pi e / R folded into (-pi, pi]
  e %= R;
  if (e < 0) e += R;
  const double f = (2 * e > R) ? (double)(e - R) / (double)R : (double)e / (double)R;
  return 6.283185307179586476925286766559 * f;
}
__host__ __device__ constexpr float c_cos(int e, int R) { return (float)c_cos_series(c_angle(e, R)); }
__host__ __device__ constexpr float c_sin(int e, int R) { return (float)c_sin_series(c_angle(e, R)); }

// Complex values are packed (re, im) pairs in one 64-bit register (common.cuh: u64) and
// every add / subtract / multiply is one packed fp32 instruction (FADD2 / FMUL2 / FFMA2):
// half the issue slots of scalar code.  The swapped / negated forms of an operand are
// SASS operand modifiers, not instructions.
using cx = u64;
__device__ __forceinline__ cx cadd(cx a, cx b) { return add2(a, b); }
__device__ __forceinline__ cx csub(cx a, cx b) { return sub2(a, b); }
__device__ __forceinline__ cx bcast(float s) { return pack2(s, s); }
__device__ __forceinline__ cx mul2(cx a, cx b) {
  cx r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
// i * a = (-a.im, a.re); -i * a = (a.im, -a.re)
__device__ __forceinline__ cx times_i(cx a) {
  const float2 f = as_f2(a);
  return pack2(-f.y, f.x);
}
__device__ __forceinline__ cx times_mi(cx a) {
  const float2 f = as_f2(a);
  return pack2(f.y, -f.x);
}
// a * (c + i s)
__device__ __forceinline__ cx cmul_cs(cx a, float c, float s) {
  cx r = mul2(a, bcast(c));
  ffma2(r, times_i(a), bcast(s));
  return r;
}
__device__ __forceinline__ cx cmulf(cx a, float2 w) { return cmul_cs(a, w.x, w.y); }
// acc + a * s (s real)
__device__ __forceinline__ cx fma_s(cx acc, cx a, float s) {
  cx r = acc;
  ffma2(r, a, bcast(s));
  return r;
}
// x * (-i) forward / x * (+i) inverse
template <bool INV>
__device__ __forceinline__ cx rot(cx a) { return INV ? times_i(a) : times_mi(a); }

// x * W_R^e, W_R = exp(-+ 2 pi i / R) (forward: minus), e and R compile-time
template <int E, int R, bool INV>
__device__ __forceinline__ cx mul_root(cx a) {
  constexpr int e = ((E % R) + R) % R;
  if constexpr (e == 0) return a;
  else if constexpr (2 * e == R) {
    const float2 f = as_f2(a);
    return pack2(-f.x, -f.y);
  } else if constexpr (4 * e == R) return rot<INV>(a);
  else if constexpr (4 * e == 3 * R) return rot<!INV>(a);
  else {
    constexpr float c = c_cos(e, R), s = INV ? c_sin(e, R) : -c_sin(e, R);
    return cmul_cs(a, c, s);
  }
}

// ---------------------------------------------------------------- in-register DFTs (natural in, natural out)
template <int R, bool INV>
struct Dft;

template <bool INV>
struct Dft<2, INV> {
  __device__ static __forceinline__ void run(cx (&v)[2]) {
    const cx a = v[0], b = v[1];
    v[0] = cadd(a, b);
    v[1] = csub(a, b);
  }
};

template <bool INV>
struct Dft<3, INV> {
  __device__ static __forceinline__ void run(cx (&v)[3]) {
    const cx t1 = cadd(v[1], v[2]);
    const cx t2 = fma_s(v[0], t1, -0.5f);
    constexpr float s = 0.86602540378443864676f;
    const cx r = rot<INV>(mul2(csub(v[1], v[2]), bcast(s)));  // -+ i s (b - c)
    v[0] = cadd(v[0], t1);
    v[1] = cadd(t2, r);
    v[2] = csub(t2, r);
  }
};

template <bool INV>
struct Dft<4, INV> {
  __device__ static __forceinline__ void run(cx (&v)[4]) {
    const cx a = cadd(v[0], v[2]), b = csub(v[0], v[2]);
    const cx c = cadd(v[1], v[3]), d = rot<INV>(csub(v[1], v[3]));
    v[0] = cadd(a, c);
    v[2] = csub(a, c);
    v[1] = cadd(b, d);
    v[3] = csub(b, d);
  }
};

template <bool INV>
struct Dft<5, INV> {
  __device__ static __forceinline__ void run(cx (&v)[5]) {
    constexpr float c1 = 0.30901699437494742410f, c2 = -0.80901699437494742410f;
    constexpr float s1 = 0.95105651629515357212f, s2 = 0.58778525229247312917f;
    const cx t1 = cadd(v[1], v[4]), t2 = cadd(v[2], v[3]);
    const cx t3 = csub(v[1], v[4]), t4 = csub(v[2], v[3]);
    const cx a1 = fma_s(fma_s(v[0], t1, c1), t2, c2);
    const cx a2 = fma_s(fma_s(v[0], t1, c2), t2, c1);
    const cx b1 = rot<INV>(fma_s(mul2(t3, bcast(s1)), t4, s2));   // -+ i (s1 t3 + s2 t4)
    const cx b2 = rot<INV>(fma_s(mul2(t3, bcast(s2)), t4, -s1));  // -+ i (s2 t3 - s1 t4)
    v[0] = cadd(cadd(v[0], t1), t2);
    v[1] = cadd(a1, b1);
    v[4] = csub(a1, b1);
    v[2] = cadd(a2, b2);
    v[3] = csub(a2, b2);
  }
};

template <int R>
__host__ __device__ constexpr int first_factor() {
  return (R % 4 == 0) ? 4 : (R % 3 == 0) ? 3 : (R % 5 == 0) ? 5 : 2;
}

// composite radix R = A * B: A-point DFTs over n1 (stride B), constant twiddles, B-point DFTs over n2
template <int R, bool INV>
struct Dft {
  static constexpr int A = first_factor<R>(), B = R / A;
  static_assert(A * B == R && B > 1, "radix must factor into 2, 3, 4, 5");

  template <int N2, int K1>
  __device__ static __forceinline__ void twiddle_col(cx (&s)[A]) {
    if constexpr (K1 < A) {
      s[K1] = mul_root<N2 * K1, R, INV>(s[K1]);
      twiddle_col<N2, K1 + 1>(s);
    }
  }
  template <int N2>
  __device__ static __forceinline__ void first(const cx (&v)[R], cx (&t)[B][A]) {
    if constexpr (N2 < B) {
      cx s[A];
#pragma unroll
      for (int n1 = 0; n1 < A; ++n1) s[n1] = v[n1 * B + N2];
      Dft<A, INV>::run(s);
      twiddle_col<N2, 1>(s);
#pragma unroll
      for (int k1 = 0; k1 < A; ++k1) t[N2][k1] = s[k1];
      first<N2 + 1>(v, t);
    }
  }
  __device__ static __forceinline__ void run(cx (&v)[R]) {
    cx t[B][A];
    first<0>(v, t);
#pragma unroll
    for (int k1 = 0; k1 < A; ++k1) {
      cx s[B];
#pragma unroll
      for (int n2 = 0; n2 < B; ++n2) s[n2] = t[n2][k1];
      Dft<B, INV>::run(s);
#pragma unroll
      for (int k2 = 0; k2 < B; ++k2) v[k1 + A * k2] = s[k2];
    }
  }
};

// ---------------------------------------------------------------- plans
enum Layout { COLS = 0, ROWS = 1 };

template <int N_, int R0_, int R1_, int R2_>
struct Plan {
  static constexpr int N = N_, R0 = R0_, R1 = R1_, R2 = R2_;
  static_assert(R0 * R1 * R2 == N, "radices must multiply to N");
  static constexpr int M0 = N / R0, M1 = M0 / R1;  // butterfly strides of passes 0 and 1 (pass 2: 1)
  static constexpr int PAD = (M0 % 2 == 0) ? 1 : 0;  // ROWS layout: pad element per top-level block
  static constexpr int NP = R0 * (M0 + PAD) + 1;     // ROWS layout: vector pitch (odd)
  // per-pass twiddle tables, output-major so that lanes over n2 read consecutive words:
  //   pass 0: T0[(k1 - 1) M0 + n2] = W_N^(n2 k1), pass 1: T1[(k1 - 1) M1 + n2] = W_M0^(n2 k1)
  static constexpr int TW0 = (R0 - 1) * M0, TW1 = (R1 - 1) * M1, TW = TW0 + TW1;
  // logical position -> physical offset inside a ROWS vector
  __host__ __device__ static constexpr int phys(int pos) { return pos + (pos / M0) * PAD; }
  // where frequency (or, inverse, sample) k ends up
  __host__ __device__ static constexpr int where(int k) { return (k % R0) * M0 + ((k / R0) % R1) * M1 + k / (R0 * R1); }
  // phys(where(k)) without the division by M0: the top-level block of where(k) is k % R0
  __host__ __device__ static constexpr int phys_where(int k) {
    return (k % R0) * (M0 + PAD) + ((k / R0) % R1) * M1 + k / (R0 * R1);
  }
};

// the CTA's twiddle tables (every thread; caller syncs)
template <class PL, bool INV>
__device__ inline void build_roots(float2* tw) {
  for (int e = threadIdx.x; e < PL::TW; e += blockDim.x) {
    int num;  // exponent over N
    if (e < PL::TW0) {
      const int k1 = e / PL::M0 + 1, n2 = e % PL::M0;
      num = n2 * k1;
    } else {
      const int f = e - PL::TW0;
      const int k1 = f / PL::M1 + 1, n2 = f % PL::M1;
      num = PL::R0 * n2 * k1;
    }
    double s, c;
    sincospi(2.0 * (double)num / (double)PL::N, &s, &c);
    tw[e] = make_float2((float)c, INV ? (float)s : (float)-s);
  }
}

// One pass (PASS = 0, 1, 2) over a tile of B vectors.  Thread -> butterfly
// mapping follows the layout so that a warp's shared accesses are contiguous;
// all index arithmetic is by compile-time constants.
template <class PL, int LAYOUT, int B, int PASS, bool INV>
__device__ __forceinline__ void pass(float2* buf, const float2* tw) {
  constexpr int N = PL::N;
  constexpr int R = PASS == 0 ? PL::R0 : PASS == 1 ? PL::R1 : PL::R2;
  constexpr int L = PASS == 0 ? N : PASS == 1 ? PL::M0 : PL::M1;
  constexpr int M = L / R, PERVEC = N / R, ITEMS = B * PERVEC;
  const float2* twp = tw + (PASS == 1 ? PL::TW0 : 0);
  const int T = blockDim.x;
  int b = 0, j = threadIdx.x;  // ROWS: item = b PERVEC + j, stepped without divisions
  if (LAYOUT == ROWS) {
    while (j >= PERVEC) {
      j -= PERVEC;
      ++b;
    }
  }
  for (int item = threadIdx.x; item < ITEMS; item += T) {
    if (LAYOUT == COLS) {
      b = item % B;
      j = item / B;
    }
    const int n2 = j % M, blk = j / M;
    float2* p;
    int stride;
    if (LAYOUT == COLS) {
      p = buf + (blk * L + n2) * B + b;
      stride = M * B;
    } else {
      // physical = logical + (top-level block) * PAD; the block is n1 itself in pass 0
      const int k0 = PASS == 0 ? 0 : PASS == 1 ? blk : blk / PL::R1;
      p = buf + b * PL::NP + blk * L + n2 + k0 * PL::PAD;
      stride = PASS == 0 ? M + PL::PAD : M;
    }
    cx v[R];
#pragma unroll
    for (int n1 = 0; n1 < R; ++n1) v[n1] = as_u64(p[n1 * stride]);
    Dft<R, INV>::run(v);
    if (M > 1) {
#pragma unroll
      for (int k1 = 1; k1 < R; ++k1) v[k1] = cmulf(v[k1], twp[(k1 - 1) * M + n2]);
    }
#pragma unroll
    for (int k1 = 0; k1 < R; ++k1) p[k1 * stride] = as_f2(v[k1]);
    if (LAYOUT == ROWS) {
      j += T;
      while (j >= PERVEC) {
        j -= PERVEC;
        ++b;
      }
    }
  }
}

// The whole transform of a tile (block-wide; barriers between the passes, none at the ends).
template <class PL, int LAYOUT, int B, bool INV>
__device__ __forceinline__ void transform(float2* buf, const float2* tw) {
  pass<PL, LAYOUT, B, 0, INV>(buf, tw);
  __syncthreads();
  pass<PL, LAYOUT, B, 1, INV>(buf, tw);
  __syncthreads();
  pass<PL, LAYOUT, B, 2, INV>(buf, tw);
}

}  // namespace mr
}  // namespace fdl
