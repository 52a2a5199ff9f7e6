// Team-per-transform FFT engine for lengths N = P * M (P = 67 or 131, the odd
// prime factor the reference's pad gives C1/C2/C2b/C4 grids: 134, 536, 1048,
// 2144; M = 2^a <= 32).  cuFFT reaches these sides only through its
// large-prime path (867 x 2144^2 rfft2: 66.7 ms on a B200, 0.48 TB/s).
//
// A team of LV warps owns T = 32 / M transforms (32 length-P vectors) in a
// private shared-memory buffer; the CTA shares only the inter-stage twiddle
// table, so there is no block barrier after the table build: teams load,
// transform and store independently (named barriers) and the SM interleaves
// their phases.  Buffer layout (complex slots): row r (0..P-1) of RS = 33
// slots, element (r, t, c) at r*RS + t*M + c.  Natural index n = M*n1 + n2
// lives in (n1, t, n2); frequency k = k1 + P*k2 ends up in (k1, t, k2).
//
// stage 1: lane v = (t, n2) of warp g computes output pairs g*K+1 .. (g+1)*K
//          of the length-P DFT over n1 of vector v directly, with the
//          symmetric pairing s_j = x_j + x_{P-j}, d_j = x_j - x_{P-j}
//          (X_k = x_0 + sum_j s_j cos -+ i sum_j d_j sin): the K <= 17 output
//          pairs accumulate in registers as packed fp32 pairs (one FFMA2 per
//          complex-by-real multiply-add).  The twiddle rows are indexed by the
//          warp-uniform (j, g), so they come from constant memory through the
//          uniform datapath (LDCU -> FFMA2 with a uniform scalar operand) and
//          only the inputs move through shared memory.  Then the inter-stage
//          twiddle W_N^{n2 k1} (shared table of N entries).
// stage 2: lanes take items (t, k1): a radix-2 DIF length-M DFT in registers.
// Twiddles are fp32 roundings of fp64 values.  Forward = exp(-2 pi i nk/N)
// (numpy's sign); inverse = exp(+...), unscaled.
#pragma once
#include <cuda_runtime.h>

#include "common.cuh"

namespace fdl {
namespace fft2 {

constexpr int SMEM_CAP = 227 * 1024 - 1024;  // opt-in shared memory per CTA minus the runtime's reserve

// DFT-P twiddle rows of stage 1 (fft2_upload_constants fills them):
//   c_tw1_P[((j-1)*LV + g)*KP + i] = (cos, sin)(2 pi j k / P), k = g*K + i + 1 (0 beyond H)
__constant__ float2 c_tw1_67[33 * 2 * 18];
__constant__ float2 c_tw1_131[65 * 4 * 18];

template <int P_, int M_>
struct Plan {
  static constexpr int P = P_, M = M_, N = P * M;
  static constexpr int H = (P - 1) / 2;                  // output pairs of the length-P DFT
  static constexpr int LV = H > 34 ? 4 : 2;              // warps per team = output groups (K <= 17)
  static constexpr int K = (H + LV - 1) / LV;            // output pairs per lane
  static constexpr int KP = (K + 1) & ~1;                // table row pitch
  static constexpr int TEAM_WARPS = LV;
  static constexpr int TL = 32 * TEAM_WARPS;             // lanes per team
  static constexpr int T = 32 / M;                       // transforms per team (32 vectors)
  static constexpr int RS = 33;                          // row stride (complex): 2 (mod 32) words
  static constexpr int SLOTS = P * RS;                   // complex slots per team buffer
  static constexpr int TW1 = H * LV * KP;                // float2 entries of the stage-1 table
  static constexpr int TABLE_BYTES = 8 * N;              // shared: the inter-stage twiddles
  static constexpr int TEAM_BYTES = 8 * SLOTS;
  static constexpr int TEAMS_FIT = (SMEM_CAP - TABLE_BYTES) / TEAM_BYTES;
  static constexpr int TEAMS_MAX = 16 / TEAM_WARPS;      // <= 16 warps (128 registers per thread)
  static constexpr int TEAMS = TEAMS_FIT < TEAMS_MAX ? TEAMS_FIT : TEAMS_MAX;
  static constexpr int WARPS = TEAMS * TEAM_WARPS;
  static constexpr int THREADS = WARPS * 32;
  static constexpr int SMEM = TABLE_BYTES + TEAMS * TEAM_BYTES;
  // column passes: a group of QT teams moves GC adjacent columns together, so
  // every row segment a warp loads or stores is GC * 8 contiguous bytes
#ifndef FDL_FFT_GC
#define FDL_FFT_GC 8
#endif
  static constexpr int GC0 = T >= FDL_FFT_GC ? T : FDL_FFT_GC;  // columns per group: 64-byte row segments
  static constexpr int GC = GC0 / T <= TEAMS ? GC0 : T * TEAMS; // (at most the CTA's teams)
  static constexpr int QT = GC / T;                      // teams per group
  static constexpr int GROUPS = TEAMS / QT;
  static constexpr int GL = QT * TL;                     // lanes per group
  static_assert(M <= 32 && 32 % M == 0, "unsupported split");
  static_assert(P == 67 || P == 131, "stage-1 constant table");
  static_assert(TW1 <= (P == 67 ? 33 * 2 * 18 : 65 * 4 * 18), "table size");
  static_assert(TEAMS % QT == 0, "teams per group");
  static_assert(TEAMS >= 2 && TEAMS + (QT > 1 ? GROUPS : 0) <= 15, "team count (named barrier ids)");
  __host__ __device__ static constexpr int slot_in(int n, int t) { return (n / M) * RS + t * M + (n % M); }
  __host__ __device__ static constexpr int slot_out(int k, int t) { return (k % P) * RS + t * M + k / P; }
};

// Barrier of one team (named barrier 1 + team; id 0 is __syncthreads).
template <class PL>
__device__ __forceinline__ void team_sync() {
  const int team = (threadIdx.x >> 5) / PL::TEAM_WARPS;
  asm volatile("bar.sync %0, %1;" ::"r"(1 + team), "r"(PL::TL) : "memory");
}

// Barrier of one column group (ids after the team barriers).
template <class PL>
__device__ __forceinline__ void group_sync() {
  if constexpr (PL::QT == 1) {
    team_sync<PL>();
  } else {
    const int group = (threadIdx.x >> 5) / (PL::TEAM_WARPS * PL::QT);
    asm volatile("bar.sync %0, %1;" ::"r"(1 + PL::TEAMS + group), "r"(PL::GL) : "memory");
  }
}

// Build the CTA's inter-stage twiddle table (all threads; one barrier by the caller).
//   tw2[e] = (cos, sin)(2 pi e / N)
template <class PL>
__device__ inline void build_tables(float2* tw2) {
  for (int e = threadIdx.x; e < PL::N; e += blockDim.x) {
    double s, c;
    sincospi(2.0 * (double)e / (double)PL::N, &s, &c);
    tw2[e] = make_float2((float)c, (float)s);
  }
}

// Stage 1 body for output group g.
template <class PL, bool INV, int g>
__device__ __forceinline__ void stage1_g(float2* buf, const float2* tw2, int tl) {
  constexpr int K = PL::K, KP = PL::KP, RS = PL::RS, P = PL::P;
  const int v = tl & 31;  // vector (t, n2)
  const int n2 = v % PL::M;
  float2* x = buf + v;
  u64 A[K], D[K];
  const u64 x0 = as_u64(x[0]);
  u64 ssum = 0ull;
#pragma unroll
  for (int i = 0; i < K; ++i) {
    A[i] = x0;
    D[i] = 0ull;
  }
  const float2* xa = x + RS;
  const float2* xc = x + (P - 1) * RS;
  // H = 33 = 3 * 11 at P = 67: unrolled by 3 (measured 2-4 % over unroll 1; 11 is no better).
  // P = 131 (H = 65) stays rolled: unroll 5 measured 3 % slower, 11 (remainder loop) 40 % slower.
  constexpr int JU = PL::H % 3 == 0 ? 3 : 1;
#pragma unroll JU
  for (int j = 1; j <= PL::H; ++j) {
    const u64 a = as_u64(*xa), c = as_u64(*xc);
    xa += RS;
    xc -= RS;
    const u64 sv = add2(a, c), dv = sub2(a, c);
    ssum = add2(ssum, sv);
    const int row = ((j - 1) * PL::LV + g) * KP;  // warp-uniform
#pragma unroll
    for (int i = 0; i < K; ++i) {
      float2 w;  // (cos, sin) of output g*K + i + 1 (the constant arrays indexed directly: LDCU)
      if constexpr (P == 67) w = c_tw1_67[row + i];
      else w = c_tw1_131[row + i];
      ffma2s(A[i], sv, w.x);
      ffma2s(D[i], dv, w.y);
    }
  }
  team_sync<PL>();  // every warp is done reading the inputs
  // twiddled store of output k1: W_N^{-+ n2 k1}
  auto put = [&](int k1, float2 val) {
    const float2 w = tw2[n2 * k1];
    const float ws = INV ? w.y : -w.y;
    x[k1 * RS] = make_float2(val.x * w.x - val.y * ws, val.x * ws + val.y * w.x);
  };
  if (g == 0) x[0] = as_f2(add2(x0, ssum));  // k1 = 0: W = 1
#pragma unroll
  for (int i = 0; i < K; ++i) {
    const int k = g * K + i + 1;
    if (k <= PL::H) {
      // X_k = A -+ i D, X_{P-k} = A +- i D   (forward: upper signs)
      const float2 At = as_f2(A[i]), Dt = as_f2(D[i]);
      const float2 lo = INV ? make_float2(At.x - Dt.y, At.y + Dt.x) : make_float2(At.x + Dt.y, At.y - Dt.x);
      const float2 hi = INV ? make_float2(At.x + Dt.y, At.y - Dt.x) : make_float2(At.x - Dt.y, At.y + Dt.x);
      put(k, lo);
      put(P - k, hi);
    }
  }
  team_sync<PL>();
}

// Stage 1 (whole team, in place on the team's buffer); tl = lane within the team.
// The output group g (= warp of the team) is a compile-time constant inside
// stage1_g, so the twiddle rows are warp-uniform constant loads (LDCU).
template <class PL, bool INV>
__device__ __forceinline__ void stage1(float2* buf, const float2* tw2, int tl) {
  const int g = tl >> 5;
  if constexpr (PL::LV == 2) {
    if (g == 0) stage1_g<PL, INV, 0>(buf, tw2, tl);
    else stage1_g<PL, INV, 1>(buf, tw2, tl);
  } else {
    if (g == 0) stage1_g<PL, INV, 0>(buf, tw2, tl);
    else if (g == 1) stage1_g<PL, INV, 1>(buf, tw2, tl);
    else if (g == 2) stage1_g<PL, INV, 2>(buf, tw2, tl);
    else stage1_g<PL, INV, 3>(buf, tw2, tl);
  }
}

// cos(2 pi e / 32) (e compile-time after unrolling: folds to an immediate)
__host__ __device__ constexpr float cos32(int e) {
  constexpr float c[9] = {1.0f, 0.98078528040323043f, 0.92387953251128674f, 0.83146961230254524f,
                          0.70710678118654752f, 0.55557023301960222f, 0.38268343236508977f,
                          0.19509032201612827f, 0.0f};
  e &= 31;
  const int q = e >> 3, r = e & 7;
  return q == 0 ? c[r] : q == 1 ? -c[8 - r] : q == 2 ? -c[r] : c[8 - r];
}

template <int M, int SPAN, bool INV>
__device__ __forceinline__ void dif_level(u64 (&v)[M]) {
  if constexpr (SPAN >= 1) {
#pragma unroll
    for (int st = 0; st < M; st += 2 * SPAN) {
#pragma unroll
      for (int t = 0; t < SPAN; ++t) {
        const u64 a = v[st + t], c = v[st + t + SPAN];
        v[st + t] = add2(a, c);
        const u64 dd = sub2(a, c);
        const int e = t * (32 / (2 * SPAN));  // twiddle W_32^e (compile-time after unrolling)
        if (e == 0) {
          v[st + t + SPAN] = dd;
        } else if (e == 8) {  // -+ i
          const float2 d = as_f2(dd);
          v[st + t + SPAN] = as_u64(INV ? make_float2(-d.y, d.x) : make_float2(d.y, -d.x));
        } else {
          const float wc = cos32(e);
          const float wsn = cos32(e + 24);  // sin(x) = cos(x - pi/2)
          const float ws = INV ? wsn : -wsn;
          const float2 d = as_f2(dd);
          v[st + t + SPAN] = as_u64(make_float2(d.x * wc - d.y * ws, d.x * ws + d.y * wc));
        }
      }
    }
    dif_level<M, SPAN / 2, INV>(v);
  }
}

template <int M>
__host__ __device__ constexpr int bitrev(int k) {
  int r = 0;
  for (int s = 1; s < M; s <<= 1) {
    r = (r << 1) | (k & 1);
    k >>= 1;
  }
  return r;
}

// Stage 2 (whole team): items (t, k1), k1 fastest, each a length-M DFT over n2.
template <class PL, bool INV>
__device__ __forceinline__ void stage2(float2* buf, int tl) {
  constexpr int M = PL::M;
  if constexpr (M > 1) {
    constexpr int ITEMS = PL::P * PL::T;
#pragma unroll 1
    for (int it = tl; it < ITEMS; it += PL::TL) {
      const int t = it / PL::P, k1 = it - t * PL::P;
      float2* p = buf + k1 * PL::RS + t * M;
      u64 v[M];
#pragma unroll
      for (int i = 0; i < M; ++i) v[i] = as_u64(p[i]);
      dif_level<M, M / 2, INV>(v);
#pragma unroll
      for (int i = 0; i < M; ++i) p[bitrev<M>(i)] = as_f2(v[i]);  // v[i] = X[bitrev(i)]
    }
  }
  team_sync<PL>();
}

template <class PL, bool INV>
__device__ __forceinline__ void transform(float2* buf, const float2* tw2, int tl) {
  stage1<PL, INV>(buf, tw2, tl);
  stage2<PL, INV>(buf, tl);
}

}  // namespace fft2
}  // namespace fdl
