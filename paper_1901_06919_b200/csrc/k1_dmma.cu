// K1 fast path: one warp per frequency bin, everything on the FP64 tensor
// cores (DMMA m8n8k4, measured 36.9 TF/s on B200 vs 34.2 TF/s for DFMA) with
// the normal matrix resident in registers.
//
// Per bin (k1_solve.cuh explains the real re-writes):
//   1. rows of the real design matrix M (and of B) are generated per lane
//      directly in DMMA fragment layout, 4 rows per k-step;
//        RHS_I += M_I^T B           (NB DMMAs / k-step)
//        G_IJ  += M_I^T M_J, J <= I (NB(NB+1)/2 DMMAs / k-step)
//   2. G += lam diag(reg') (reg' = reg of the layer pair; padding -> identity);
//   3. blocked right-looking Cholesky, block 8, all blocks in registers as
//      accumulator fragments: per step K the 8x8 diagonal block is factored
//      and inverted by 8 lanes (W = L_KK^-1), the panel is L_IK = G_IK W^T
//      (DMMA), the trailing update G_IJ -= L_IK L_JK^T (DMMA) and the forward
//      substitution y_K = W r_K, r_I -= L_IK y_K (DMMA) run interleaved;
//   4. backward substitution x_K = W^T (y_K - sum_{I>K} L_IK^T x_I) (DMMA);
//   5. x mapped back to complex layer coefficients, written as complex64.
// Staging: the bin's spectra words and phase-table column arrive by TMA (a tile per
// warp pair, a bulk copy per warp) where the plane stride allows, else by cp.async.
//
// DMMA fragment layouts (m8n8k4, row.col, f64; lane l, q = l>>2, t = l&3):
//   A (8x4): A[q][t]   B (4x8): B[t][q]   C (8x8): C[q][2t], C[q][2t+1]
// (checked on the device by fdl_selftest).
#include <algorithm>

#include "k1_solve.cuh"
#include "tma.cuh"

namespace fdl {

namespace {

constexpr unsigned FULL = 0xffffffffu;
constexpr int WARPS = 8;  // bins (consecutive kx of one row) per CTA
// Row stride (doubles) of the per-warp 8x8 scratch blocks (S, T, W) and of X:
// 12 makes the DMMA-fragment-layout reads/writes ([q][t], [t][q], [q][2t])
// conflict-free (8 would put rows q and q+2 on the same banks).
constexpr int LD = 8;
#ifndef FDL_K1_KUNROLL
#define FDL_K1_KUNROLL 2
#endif
constexpr int kKUnroll = FDL_K1_KUNROLL;  // k-step loop unroll (A/B builds)
#ifndef FDL_K1_TH
#define FDL_K1_TH 1  // Toeplitz-Hankel Gram from spare RHS columns (0: Gram by DMMA, A/B)
#endif
#ifndef FDL_K1_TMA
#define FDL_K1_TMA 1  // stage spectra / phase tables through the TMA unit where the layout allows
#endif
#ifndef FDL_K1_W12
#define FDL_K1_W12 1  // 12-warp CTAs for 7-8 block mirror-pair systems (K1Cfg)
#endif
#ifndef FDL_K1_TH_PAIR_MINNB
#define FDL_K1_TH_PAIR_MINNB 4
#endif
#ifndef FDL_K1_PAIR3
#define FDL_K1_PAIR3 4  // PAIR kernels with NB <= this get 3 CTAs/SM (80 registers: measured 2 % faster on C2)
#endif

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c[0]), "+d"(c[1])
      : "d"(a), "d"(b));
}

// accumulator fragment -> A-fragment pair (C[q][t], C[q][4+t]) of the same block
__device__ __forceinline__ void c_to_a(const double (&c)[2], double& a0, double& a1, int lane) {
  const int q = lane >> 2, t = lane & 3;
  const int s0 = (q << 2) + (t >> 1), s1 = s0 + 2;
  const double x0 = __shfl_sync(FULL, c[0], s0), x1 = __shfl_sync(FULL, c[1], s0);
  const double y0 = __shfl_sync(FULL, c[0], s1), y1 = __shfl_sync(FULL, c[1], s1);
  a0 = (t & 1) ? x1 : x0;
  a1 = (t & 1) ? y1 : y0;
}

// accumulator fragment -> A-fragment pair of the TRANSPOSED block (C[t][q], C[4+t][q])
__device__ __forceinline__ void c_to_at(const double (&c)[2], double& a0, double& a1, int lane) {
  const int q = lane >> 2, t = lane & 3;
  const int s0 = (t << 2) + (q >> 1), s1 = s0 + 16;
  const double x0 = __shfl_sync(FULL, c[0], s0), x1 = __shfl_sync(FULL, c[1], s0);
  const double y0 = __shfl_sync(FULL, c[0], s1), y1 = __shfl_sync(FULL, c[1], s1);
  a0 = (q & 1) ? x1 : x0;
  a1 = (q & 1) ? y1 : y0;
}

// 1/sqrt(x) in full double precision: MUFU approximation + two Newton steps
// (CUDA's rsqrt(double) is a ~30-instruction library routine).
__device__ __forceinline__ double rsqrt_fast(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double hx = 0.5 * x;
  y = y * fma(-hx * y, y, 1.5);
  y = y * fma(-hx * y, y, 1.5);
  return y;
}

// accumulator fragment -> row-major 8x8 block (row stride LD): one 16-byte
// store per lane, conflict-free (a quarter warp covers all 32 banks)
__device__ __forceinline__ void store_c(double* S, const double (&c)[2], int lane) {
  const int q = lane >> 2, t = lane & 3;
  *reinterpret_cast<double2*>(S + q * LD + 2 * t) = make_double2(c[0], c[1]);
}
// Diagonal-block scratch: row stride LDD = 9 doubles, so the 8 rows' column c
// fall on distinct banks (the factorisation's lane = row accesses); the
// second block's scratch starts an odd number of doubles later, so the two
// 8-lane groups of a paired step never share a bank either.
constexpr int LDD = 9;
constexpr int DSZ = 8 * LDD;  // D1 - D0 = 144 words = 16 (mod 32): the complementary banks
__device__ __forceinline__ void store_cd(double* D, const double (&c)[2], int lane) {
  const int q = lane >> 2, t = lane & 3;
  D[q * LDD + 2 * t] = c[0];
  D[q * LDD + 2 * t + 1] = c[1];
}

struct FastParams {
  const int* u_idx;     // (m) index of u_j among the distinct u values
  const int* v_idx;     // (m)
  const double* u_val;  // (nu)
  const double* v_val;  // (nv)
  int nu, nv;
  int H8;               // columns per cos/sin half, multiple of 8 (mode 1)
  int hw;               // phase-table width: h + (n odd)
  int hwp;              // shared-memory row pitch of the tables (double2): = 2 mod 8, so the
                        // 4 views x 2 layers of a quarter-warp hit distinct banks
  const double2* px_all;  // (Whp, nu, hwp) exp(2 pi i fl(u d_p) wx), cosine on the Nyquist column
  const double2* py_all;  // (nrows, nv, hwp); the shared-memory pitch, so staging is a flat copy
  // TMA staging (mode 1, 16-byte plane stride): warps 2w and 2w + 1 solve the bins
  // (kx, kx + 1) of one 16-byte word per plane; one tensor copy per `bs_box` planes
  // lands the pair's spectra as a shared [plane][2] float2 tile, and each bin's
  // phase-table column is one bulk copy
  int tma, bs_box, bs_nbox;
};

__host__ __device__ constexpr int blk(int I, int J) { return I * (I + 1) / 2 + J; }
// per-warp Toeplitz scratch X (t[] and E of the spare-column Gram): none for the
// split systems whose Gram the k-steps form by DMMA
template <int NB, int PAIR>
__host__ __device__ constexpr int xwords() { return (FDL_K1_TH && (!PAIR || NB > FDL_K1_TH_PAIR_MINNB)) ? NB * 8 * LD : 0; }
// mode 1 block groups: 0 = cos half (+ the middle column of odd n), 1 = sin half.
// With mirror pairs (PAIR) blocks of different groups are exactly zero.
__host__ __device__ constexpr int grp(int I, int NBc) { return (I >= NBc && I < 2 * NBc) ? 1 : 0; }

// mode 2: per-(view, layer) half of the aperture lookup, shared by a CTA's row of bins
struct YEntry {
  double t, fy;
  int iyoff, ai;
};

// Per-axis phase tables of mode 1, once per column / row of the slab (the
// reference's `_phase_tables`, construct.py:68-80, restricted to the distinct
// u and v values and the first half of the layers).
__global__ void k1_axis_tables_kernel(SolveParams p, FastParams f) {
  const long long nx = (long long)p.Whp * f.nu * f.hwp;
  const long long ny = (long long)p.nrows * f.nv * f.hwp;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < nx + ny;
       e += (long long)gridDim.x * blockDim.x) {
    if (e < nx) {
      const int pp = (int)(e % f.hwp);
      const long long r = e / f.hwp;
      const int iu = (int)(r % f.nu), kx = (int)(r / f.nu);
      cd ph{0.0, 0.0};  // pitch padding stays zero
      if (pp < f.hw) ph = axis_phase(f.u_val[iu] * p.d[pp], omega_x_label(kx, p.Wp), (p.Wp % 2 == 0) && kx == p.Wp / 2);
      const_cast<double2*>(f.px_all)[e] = make_double2(ph.re, ph.im);
    } else {
      const long long e2 = e - nx;
      const int pp = (int)(e2 % f.hwp);
      const long long r = e2 / f.hwp;
      const int iv = (int)(r % f.nv), i = (int)(r / f.nv);
      const int ky = p.rows[i];
      cd ph{0.0, 0.0};
      if (pp < f.hw) ph = axis_phase(f.v_val[iv] * p.d[pp], omega_y_label(ky, p.Hp), (p.Hp % 2 == 0) && ky == p.Hp / 2);
      const_cast<double2*>(f.py_all)[e2] = make_double2(ph.re, ph.im);
    }
  }
}

// Warps (= bins in flight) per CTA and CTAs per SM.  Mode 2 systems of >= 5
// blocks (C3: 48 layers, real A) hold the full Gram in registers; at 8 warps x
// 2 CTAs (128 registers) they spilled 272 B per thread and the spills doubled
// the kernel's DRAM writes, so they run FDL_K1_REALA_WARPS warps x 2 CTAs.
#ifndef FDL_K1_REALA_WARPS
#define FDL_K1_REALA_WARPS 6
#endif
#ifndef FDL_K1_PAIR_WARPS
#define FDL_K1_PAIR_WARPS 8  // split (mirror-pair) systems of 3..FDL_K1_PAIR3 blocks (C2)
#endif
#ifndef FDL_K1_PAIR_MINB
#define FDL_K1_PAIR_MINB 3
#endif
// W12: 12-warp CTAs for the mirror-pair systems of 7-8 blocks (C4) when their shared memory fits (TMA
// staging, phase tables of the non-negative u only, Toeplitz scratch aliased onto the table column):
// three warps per scheduler instead of two at 168 registers (tools/k1_occ_probe.py: -10 %; 10 warps lose)
template <int NB, int MODE, int PAIR, int W12 = 0>
struct K1Cfg {
  static constexpr bool pair_small = PAIR && NB > 2 && NB <= FDL_K1_PAIR3;
  static constexpr int warps =
      W12 ? 12 : ((MODE == MODE_REALA && NB >= 5 && NB <= 6) ? FDL_K1_REALA_WARPS : (pair_small ? FDL_K1_PAIR_WARPS : WARPS));
  static constexpr int minb = NB <= 2 ? 3 : (pair_small ? FDL_K1_PAIR_MINB : (NB <= 6 ? 2 : 1));
};

template <int NB, int MODE, int ODD, int PAIR, int W12 = 0>
__global__ void __launch_bounds__(K1Cfg<NB, MODE, PAIR, W12>::warps * 32, K1Cfg<NB, MODE, PAIR, W12>::minb) k1_fast_kernel(SolveParams p, FastParams f, const __grid_constant__ CUtensorMap smap) {
  constexpr int WARPS = K1Cfg<NB, MODE, PAIR, W12>::warps;  // shadows the file-wide default
  constexpr int NBc = (NB - ODD) / 2;  // blocks of the cos half (= of the sin half), mode 1
  // blocks I, J interact (PAIR: only within a group)
  auto linked = [](int I, int J) { return !PAIR || grp(I, NBc) == grp(J, NBc); };
  constexpr int NBLK = NB * (NB + 1) / 2;
  constexpr int NP = NB * 8;
  extern __shared__ __align__(128) double smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, q = lane >> 2, t = lane & 3;
  const int i = blockIdx.y;
  const bool tma = MODE == MODE_SYMREAL && f.tma;
  const int bss = tma ? 2 : 1;  // BS entries per (view, channel)
  const int ky = p.rows[i];
  const double oy = omega_y_label(ky, p.Hp);
  const bool nyq_y = (p.Hp % 2 == 0) && ky == p.Hp / 2;

  // shared layout: [PY: nv*hwp complex | ROW4 | RG] then per warp
  // [PX: nu*hwp complex | D 2*73 | S 64 | Wst (NB-1)*64 | X NP*8 | BS].  Lifetimes let
  // buffers double up: the W = L^-1 of the last diagonal block lives in S, and
  // the Toeplitz build keeps t[] in X's upper half and E in its lower half.
  // TMA mode: per warp [PX (= X after the k-steps) | D | S | Wst], then the mbarriers
  // (2 per warp) and one 128-byte aligned [plane][2] spectra tile per warp PAIR.
  double* PY = smem;
  const int py_words = (MODE == MODE_SYMREAL) ? 2 * (f.nv + 1) * f.hwp : 0;  // + one all-zero row (padding rows)
  const int px_words = (MODE == MODE_SYMREAL) ? 2 * f.nu * f.hwp : 0;
  // mode 1 equation rows: one per view, or one per mirror pair (p.mrow)
  const int mrow = (MODE == MODE_SYMREAL) ? p.mrow : p.m;
  const int m4 = (mrow + 3) & ~3;
  const int ro_words = (MODE == MODE_SYMREAL) ? 2 * m4 : 3 * p.m * p.n;  // mode 2: YEntry per (view, layer)
  // mode 1: per row (u-table offset, v-table offset, BS offset of j, of j' or -1)
  int4* ROW4 = reinterpret_cast<int4*>(PY + py_words);
  YEntry* YT = reinterpret_cast<YEntry*>(PY + py_words);
  // staged spectra, one float2 per (view, channel); keeps 16-B alignment (TMA mode: own region below)
  const int bs_words = tma ? 0 : ((p.m * p.C + 1) & ~1);
  constexpr int XW = xwords<NB, PAIR>();  // Toeplitz scratch (none when the Gram is formed by DMMA)
  // TMA mode: the Toeplitz scratch X lives in the table column's region (the next column is
  // fetched after the Toeplitz build instead of right after the k-steps)
  const int pxr_words = tma ? (px_words > XW ? px_words : XW) : px_words;
  const int xw_alloc = tma ? 0 : XW;
  const int per_warp = pxr_words + 2 * DSZ + 8 * LD + (NB - 1) * 8 * LD + xw_alloc + bs_words;
  // per column of the real system: (d^4 of its layer(s)) for the lam reg' diagonal
  const int rg_off = py_words + ((ro_words + 1) & ~1);  // 16-byte aligned
  double2* RG = reinterpret_cast<double2*>(smem + rg_off);
  double* base = smem + rg_off + 2 * NP + warp * per_warp;
  double* PX = base;
  double* D0 = PX + pxr_words;  // diagonal-block scratch (LDD layout) of block Ka ...
  double* D1 = D0 + DSZ;       // ... and of Kb
  double* S = D1 + DSZ;
  double* Wst = S + 8 * LD;
  double* X = tma ? PX : Wst + (NB - 1) * 8 * LD;
  // W = L_KK^-1 of diagonal block K
  auto Wblk = [&](int K) { return K == NB - 1 ? S : Wst + K * 8 * LD; };
  float2* BS = reinterpret_cast<float2*>(Wst + (NB - 1) * 8 * LD + xw_alloc);
  // TMA mode: [2 mbarriers per warp | 128-byte aligned [plane][2] tile per warp pair] behind the
  // per-warp regions; bar_px: this warp's phase-table column, bar_bs: the pair's spectra tile
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(smem + rg_off + 2 * NP + WARPS * per_warp);
  unsigned long long* bar_px = bars + 2 * warp;
  unsigned long long* bar_bs = bars + 2 * (warp & ~1) + 1;
  const bool lead = !(warp & 1);  // issues the pair's tensor copies
  const unsigned bs_bytes = tma ? (unsigned)f.bs_nbox * f.bs_box * 16u : 0u;
  if (tma) {
    const unsigned off = (unsigned)(rg_off + 2 * NP + WARPS * per_warp + 2 * WARPS) * 8u;
    BS = reinterpret_cast<float2*>(reinterpret_cast<char*>(smem) + ((off + 127u) & ~127u) + (warp >> 1) * bs_bytes);
    if (lane == 0) {
      mbar_init(bar_px, 1);
      if (lead) mbar_init(bar_bs, 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
  }

  if (MODE == MODE_SYMREAL) {
    const double2* src = f.py_all + (size_t)i * f.nv * f.hwp;
    for (int e = threadIdx.x; e < f.nv * f.hwp; e += blockDim.x) reinterpret_cast<double2*>(PY)[e] = src[e];
    // rows past mrow (the last k-step's padding) read an all-zero y table row: A = 0, so they add
    // nothing to the Gram matrix or the right-hand sides and need no special k-step
    for (int e = threadIdx.x; e < f.hwp; e += blockDim.x)
      reinterpret_cast<double2*>(PY)[f.nv * f.hwp + e] = make_double2(0.0, 0.0);
    for (int e = threadIdx.x; e < m4; e += blockDim.x) {
      int4 ro = make_int4(0, f.nv * f.hwp, 0, -1);
      if (e < mrow) {
        const int2 jj = PAIR ? p.row_pairs[e] : make_int2(e, -1);
        ro = make_int4(f.u_idx[jj.x] * f.hwp, f.v_idx[jj.x] * f.hwp, jj.x * p.C * bss, jj.y >= 0 ? jj.y * p.C * bss : -1);
      }
      ROW4[e] = ro;
    }
  } else {
    // mode 2: the y half of every bilinear lookup depends only on (view, layer, row):
    // t_jk = scale_j (s_j - d_k), (iy, fy) of t_jk wy -- shared by the CTA's bins
    for (int e = threadIdx.x; e < p.m * p.n; e += blockDim.x) {
      const int j = e / p.n, k = e - j * p.n;
      const int ai = p.view_ap ? p.view_ap[j] : -1;
      YEntry ye;
      ye.ai = ai;
      ye.t = 0.0;
      ye.fy = 0.0;
      ye.iyoff = 0;
      if (ai >= 0) {
        const DevAperture& ap = p.aps[ai];
        ye.t = __dmul_rn(p.scale[j], __dsub_rn(p.s[j], p.d[k]));
        int iy;
        double fy;
        const bool ok = axis_lookup(__dmul_rn(ye.t, oy), ap.xi0_y, ap.step_y, ap.rows, iy, fy);
        ye.fy = fy;
        ye.iyoff = ok ? iy * ap.cols : ap.rows * ap.cols;  // the quad table's zero entry
      }
      YT[e] = ye;
    }
  }
  for (int col = threadIdx.x; col < NP; col += blockDim.x) {
    // (d4_p, d4_{n-1-p}) for a symmetric pair, (d4_k, -1) for one layer, (-1, -1) for padding
    double2 ab = make_double2(-1.0, -1.0);
    if (MODE == MODE_SYMREAL) {
      const int I = col >> 3;
      const bool cpart = I < NBc, spart = I >= NBc && I < 2 * NBc;
      const int pp = cpart ? col : (spart ? col - NBc * 8 : p.h);
      if ((cpart || spart) && pp < p.h) ab = make_double2(p.d4[pp], p.d4[p.n - 1 - pp]);
      else if (!cpart && !spart && ODD && col == 2 * NBc * 8) ab = make_double2(p.d4[p.h], -1.0);
    } else if (col < p.n) {
      ab = make_double2(p.d4[col], -1.0);
    }
    RG[col] = ab;
  }
  __syncthreads();
  // no block barriers below: each warp solves p.reps bins of this row,
  // columns (blockIdx.x * reps + rep) * WARPS + warp
  // mode 2 with one shared aperture: its lookup constants live in registers
  const bool uap = MODE == MODE_REALA && p.uniform_ap >= 0;
  const double2* uq = nullptr;
  double u_xi0 = 0.0, u_inv = 0.0;
  int u_cols = 0, u_zero = 0;
  if (uap) {
    const DevAperture& a0 = p.aps[p.uniform_ap];
    uq = a0.quad;
    u_xi0 = a0.xi0_x;
    u_inv = a0.inv_step_x;
    u_cols = a0.cols;
    u_zero = a0.rows * a0.cols;
  }
  // The bin's m x C spectra values (one 8-byte word per view plane) and, in
  // mode 1, its column of phase tables are copied asynchronously: the copy for
  // bin rep + 1 is issued as soon as bin rep's k-steps have read the buffers,
  // so it lands under bin rep's factorisation.
  auto stage_bin = [&](int kxs) {
    const size_t plane_ = sp_plane(p);
    const float2* src = p.spectra + sp_boff(p, i, kxs);
    for (int e = lane; e < p.m * p.C; e += 32) cpa8(&BS[e], src + (size_t)e * plane_, true);
    if (MODE == MODE_SYMREAL) {
      const double2* srcx = f.px_all + (size_t)kxs * f.nu * f.hwp;
      for (int e = lane; e < f.nu * f.hwp; e += 32) cpa16(reinterpret_cast<double2*>(PX) + e, srcx + e, true);
    }
    cpa_commit();
  };
  // TMA mode: a tensor copy must start on a 16-byte boundary, so the pairs are
  // aligned on the flat bin index: rows at an odd offset shift their bins left by
  // one (the first pair starts at kx = -1).  A warp whose bin lies outside the row
  // while its partner's does not only takes part in the hand-over.
  const int odd0 = tma ? (int)(sp_boff(p, i, 0) & 1) : 0;
  auto kx_of = [&](int rep) { return (int)(blockIdx.x * p.reps + rep) * WARPS + warp - odd0; };
  unsigned px_phase = 0, bs_phase = 0;
  auto stage_px = [&](int kxs) {
    if (lane == 0) {
      const unsigned bytes = (unsigned)(f.nu * f.hwp) * 16u;
      mbar_expect_tx(bar_px, bytes);
      bulk_load(PX, f.px_all + (size_t)kxs * f.nu * f.hwp, bytes, bar_px);
    }
  };
  auto stage_pair = [&](int kxp) {  // lead warp: the tile of bins (kxp, kxp + 1)
    if (lane == 0) {
      mbar_expect_tx(bar_bs, bs_bytes);
      const int c0 = (int)(2 * (long long)sp_boff(p, i, 0)) + 2 * kxp;
      for (int b = 0; b < f.bs_nbox; ++b) tma_load_2d(BS + 2 * b * f.bs_box, &smap, c0, b * f.bs_box, bar_bs);
    }
  };
  // after a bin's k-steps: the pair hands the tile back (named barrier 1 + pair: the
  // partner arrives, the lead waits and re-issues), each warp re-stages its own column
  auto stage_next = [&](int rep) {
    const int kxn = kx_of(rep + 1), kxpn = kxn - (warp & 1);
    if (rep + 1 >= p.reps || kxpn >= p.Whp) return;  // pair-uniform
    if (lead) {
      asm volatile("bar.sync %0, 64;" ::"r"(1 + (warp >> 1)) : "memory");
      stage_pair(kxpn);
    } else {
      asm volatile("bar.arrive %0, 64;" ::"r"(1 + (warp >> 1)) : "memory");
    }
  };
  // this warp's next table column (after the Toeplitz build when that used the column's region)
  auto stage_px_next = [&](int rep) {
    const int kxn = kx_of(rep + 1);
    if (rep + 1 < p.reps && kxn - (warp & 1) < p.Whp && kxn >= 0 && kxn < p.Whp) stage_px(kxn);
  };
  {
    const int kx0 = kx_of(0);
    if (tma) {
      if (kx0 - (warp & 1) < p.Whp) {
        if (lead) stage_pair(kx0);
        if (kx0 >= 0 && kx0 < p.Whp) stage_px(kx0);
      }
    } else if (kx0 < p.Whp) {
      stage_bin(kx0);
    }
  }
  for (int rep = 0; rep < p.reps; ++rep) {
  const int kx = kx_of(rep);
  if (kx - (tma ? (warp & 1) : 0) >= p.Whp) break;  // warp-uniform (TMA: pair-uniform)
  if (tma && (kx < 0 || kx >= p.Whp)) {             // only the partner's bin exists
    bs_phase ^= 1u;
    stage_next(rep);
    stage_px_next(rep);
    continue;
  }
  const int kx_next = kx_of(rep + 1);
  const bool has_next = rep + 1 < p.reps && kx_next < p.Whp;
  const double ox = omega_x_label(kx, p.Wp);
  const bool nyq_x = (p.Wp % 2 == 0) && kx == p.Wp / 2;
  if (tma) {
    mbar_wait(bar_px, px_phase);
    px_phase ^= 1u;
    mbar_wait(bar_bs, bs_phase);
    bs_phase ^= 1u;
  } else {
    cpa_wait_all();
  }
  __syncwarp();  // this bin's staged values visible to the whole warp

  double g[NBLK][2];
  double r[NB][2];
#pragma unroll
  for (int b = 0; b < NBLK; ++b) g[b][0] = g[b][1] = 0.0;
#pragma unroll
  for (int b = 0; b < NB; ++b) r[b][0] = r[b][1] = 0.0;

  const size_t plane = sp_plane(p);
  const size_t boff = sp_boff(p, i, kx);      // spectra / layers
  const size_t soff = (size_t)i * p.Whp + kx;  // status (slab-indexed)
  const int h = p.h;
  // Toeplitz-Hankel Gram (mode 1, uniform d, off the Nyquist lines, <= 3 channels):
  // G' follows from t[r] = sum_j conj(A_j0) A_jr, which the RHS DMMAs produce for
  // free in the two spare right-hand-side columns (6: Re A_j0, 7: Im A_j0).
  // (split systems of <= 2 blocks each -- C2's 15 + 15 -- form the Gram by DMMA instead:
  //  3 + 3 blocks per k-step are cheaper than the spare-column bookkeeping; measured)
  const bool th = FDL_K1_TH && (!PAIR || NB > FDL_K1_TH_PAIR_MINNB) && (MODE == MODE_SYMREAL) && p.uniform_d &&
                  !nyq_x && !nyq_y && p.C <= 3;

  // ---------------------------------------------------------------- 1. Gram + RHS
  // mode 1 design matrix (unscaled): M = [Re A_p | -Im A_p | Re A_mid]; the
  // unknowns are x_p = (v+_p + i v-_p)/2, x_{n-1-p} = (v+_p - i v-_p)/2 (powers of
  // two only, so no rounding beyond A's own).
  const bool bcol = q < 2 * p.C;
  const int bc = bcol ? (q >> 1) : 0;
  const int bcs = bc * bss + (tma ? (warp & 1) : 0);  // BS index of this lane's channel (TMA: this bin of the pair)
  const float* BSq = reinterpret_cast<const float*>(BS) + (q & 1);
  const float bmask = bcol ? 1.f : 0.f;
  const double2* PX2 = reinterpret_cast<const double2*>(PX);
  const double2* PY2 = reinterpret_cast<const double2*>(PY);

  // spare-column weights of a paired row: column 6 (Re A_j0) counts twice in the cos group and
  // not at all in the sin group, column 7 (Im A_j0) the other way round
  const double sp_c = (q == 6) ? 2.0 : 0.0, sp_s = (q == 6) ? 0.0 : 2.0;
  // one k-step: 4 rows (views) r0..r0+3, lane row j = r0 + t
  auto kstep = [&](int r0, bool tail) {
    const int j = r0 + t;
    const bool valid = !tail || j < mrow;
    double mf[NB];
#pragma unroll
    for (int I = 0; I < NB; ++I) mf[I] = 0.0;
    double bf = 0.0;   // B fragment (RHS columns); PAIR: of the cos group (b_j + b_j')
    double bfm = 0.0;  // PAIR: B fragment of the sin group (b_j - b_j')
    bool paired = false;
    if (MODE == MODE_SYMREAL) {
      const int4 ro = ROW4[j];
      // this lane's RHS column is the real (q even) or imaginary (q odd) part of channel bc:
      // one 4-byte read, masked by a per-lane 1.0f / 0.0f (columns past 2 C carry no data)
      const double v1 = (double)(BSq[2 * (ro.z + bcs)] * bmask);
      if (PAIR) {
        paired = ro.w >= 0;
        const float f2 = BSq[2 * ((paired ? ro.w : ro.z) + bcs)];
        const double v2 = (double)((paired ? f2 : 0.f) * bmask);
        bf = v1 + v2;
        bfm = v1 - v2;
      } else {
        bf = v1;
      }
      const double2* pxr = PX2 + ro.x;
      const double2* pyr = PY2 + ro.y;
      if (th && q >= 6) {
        const double2 x0 = pxr[0], y0 = pyr[0];
        const double re = fma(x0.x, y0.x, -x0.y * y0.y), im = fma(x0.x, y0.y, x0.y * y0.x);
        if (PAIR) {
          // the partner's A_j'0 = conj(A_j0): column 6 (Re) sums, column 7 (Im) cancels; the
          // weights of a paired row are per-lane constants (sp_c, sp_s), exact powers of two
          const double val = (q == 6) ? re : im;
          bf = val * (paired ? sp_c : 1.0);
          bfm = val * (paired ? sp_s : 1.0);
        } else {
          bf = (q == 6) ? re : im;
        }
      }
#pragma unroll
      for (int I = 0; I < NBc; ++I) {
        const int pp = I * 8 + q;
        // even n: table entries past h are zero-filled (k1_table_pitch), no bound check needed
        if (!ODD || pp < h) {
          const double2 x = pxr[pp], y = pyr[pp];
          mf[I] = fma(x.x, y.x, -x.y * y.y);
          mf[I + NBc] = -fma(x.x, y.y, x.y * y.x);
        }
      }
      if (ODD && q == 0) {
        const double2 x = pxr[h], y = pyr[h];
        mf[NB - 1] = fma(x.x, y.x, -x.y * y.y);
      }
      if (tail && !valid) {
#pragma unroll
        for (int I = 0; I < NB; ++I) mf[I] = 0.0;
        bf = bfm = 0.0;
      }
    } else {  // MODE_REALA: A_jk = psi_j(t_jk wx, t_jk wy) (all shifts are zero)
      const float2 bcur = BS[(valid ? j : 0) * p.C + bc];
      bf = (bcol && valid) ? ((q & 1) ? (double)bcur.y : (double)bcur.x) : 0.0;
      if (uq) {
        // shared real aperture (warp-uniform): every lane evaluates its entry unconditionally on a
        // clamped table address and masks the result, so the NB lookups of a k-step carry no control
        // dependence and their loads / fp64 chains overlap
#pragma unroll
        for (int I = 0; I < NB; ++I) {
          const int k = I * 8 + q;
          const bool on = valid && k < p.n;
          // x half of the bilinear lookup + one quad read
          const YEntry ye = YT[on ? j * p.n + k : 0];
          const double pos = (__dmul_rn(ye.t, ox) - u_xi0) * u_inv;
          const bool okx = (pos >= 0.0) && (pos <= (double)(u_cols - 1));
          const int ix = okx ? min((int)pos, u_cols - 2) : 0;
          const double fx = pos - (double)ix;
          const int qi = okx ? min(ye.iyoff + ix, u_zero) : u_zero;
          const double2 top = uq[2 * qi], bot = uq[2 * qi + 1];
          // bilinear weights as two lerps along y and one along x (6 fp64 operations instead of 10;
          // within an ulp of the product form)
          const double left = fma(ye.fy, bot.x - top.x, top.x), right = fma(ye.fy, bot.y - top.y, top.y);
          const double val = fma(fx, right - left, left);
          mf[I] = on ? val : 0.0;
        }
      } else {
#pragma unroll
      for (int I = 0; I < NB; ++I) {
        const int k = I * 8 + q;
        if (valid && k < p.n) {
          const YEntry ye = YT[j * p.n + k];
          if (ye.ai < 0) {
            mf[I] = 1.0;
          } else {
            const DevAperture& ap = p.aps[ye.ai];
            if (ap.quad) {
              // x half of the bilinear lookup (lfmodel.py:72-99) + one 32-byte quad-table read
              const double pos = (__dmul_rn(ye.t, ox) - ap.xi0_x) * ap.inv_step_x;
              const bool okx = (pos >= 0.0) && (pos <= (double)(ap.cols - 1));
              // inside the table pos >= 0, so truncation is floor; the clip to cols-2
              // only bites at pos == cols-1 (then fx = 1) -- no fp64 min/max needed
              const int ix = okx ? min((int)pos, ap.cols - 2) : 0;
              const double fx = pos - (double)ix;
              const int zero = ap.rows * ap.cols;
              const int qi = okx ? min(ye.iyoff + ix, zero) : zero;
              const double2 top = ap.quad[2 * qi], bot = ap.quad[2 * qi + 1];
              const double gy = 1.0 - ye.fy, gx = 1.0 - fx;
              mf[I] = (top.x * gy) * gx + (top.y * gy) * fx + (bot.x * ye.fy) * gx + (bot.y * ye.fy) * fx;
            } else {
              mf[I] = aperture_eval(ap, __dmul_rn(ye.t, ox), __dmul_rn(ye.t, oy)).re;
            }
          }
        }
      }
      }
    }
#pragma unroll
    for (int I = 0; I < NB; ++I) dmma(r[I], mf[I], (PAIR && grp(I, NBc)) ? bfm : bf);
    if (!th) {
      // PAIR: a pair row stands for two views with equal c c^T and s s^T terms
      const double w = paired ? 2.0 : 1.0;
#pragma unroll
      for (int I = 0; I < NB; ++I)
#pragma unroll
        for (int J = 0; J <= I; ++J)
          if (linked(I, J)) dmma(g[blk(I, J)], mf[I], PAIR ? w * mf[J] : mf[J]);
    }
  };
  const int mfull = mrow & ~3;
  // (the 80-register split kernels of 3-4 blocks, C2, run faster without unrolling: 0.90 -> 0.86 ms)
  constexpr int KU = K1Cfg<NB, MODE, PAIR, W12>::pair_small ? 1 : kKUnroll;
  if (MODE == MODE_SYMREAL) {
#pragma unroll KU
    for (int r0 = 0; r0 < m4; r0 += 4) kstep(r0, false);
  } else {
#pragma unroll KU
    for (int r0 = 0; r0 < mfull; r0 += 4) kstep(r0, false);
    if (mfull < mrow) kstep(mfull, true);
  }
  __syncwarp();  // every lane is done with BS / PX of this bin
  if (tma) {
    stage_next(rep);
    if (!(MODE == MODE_SYMREAL && th && XW > 0)) stage_px_next(rep);
  } else if (has_next) {
    stage_bin(kx_next);
  }

  if (MODE == MODE_SYMREAL && th) {
    // RHS columns 6/7 = M^T [Re A_0, Im A_0]  ->  t[r], r = 0..n-1  ->  G fragments
#pragma unroll
    for (int I = 0; I < NB; ++I) {
      X[(I * 8 + q) * LD + 2 * t] = r[I][0];
      X[(I * 8 + q) * LD + 2 * t + 1] = r[I][1];
    }
    __syncwarp();
    double* TT = X + NP * LD / 2;  // t[0..n-1] (complex) in X's upper half, E below it
    const int H8 = NBc * 8;
    double tre[2] = {0.0, 0.0}, tim[2] = {0.0, 0.0};
#pragma unroll
    for (int it = 0; it < 2; ++it) {
      const int rr = lane + 32 * it;
      if (rr >= p.n) continue;
      double re, im;
      if (ODD && rr == h) {
        re = X[(2 * H8) * LD + 6];
        im = -X[(2 * H8) * LD + 7];
      } else if (rr < h) {
        re = X[rr * LD + 6] - X[(H8 + rr) * LD + 7];
        im = -X[(H8 + rr) * LD + 6] - X[rr * LD + 7];
      } else {
        const int pq = p.n - 1 - rr;
        re = X[pq * LD + 6] + X[(H8 + pq) * LD + 7];
        im = X[(H8 + pq) * LD + 6] - X[pq * LD + 7];
      }
      tre[it] = re;
      tim[it] = im;
    }
    __syncwarp();  // every lane is done reading the RHS columns out of X
#pragma unroll
    for (int it = 0; it < 2; ++it) {
      const int rr = lane + 32 * it;
      if (rr >= p.n) continue;
      TT[2 * rr] = tre[it];
      TT[2 * rr + 1] = tim[it];
    }
    __syncwarp();
    // extended table E[k + n - 1] = t[k] for k in [-(n-1), n-1] (t[-k] = conj t[k]), in X
    const int nm1 = p.n - 1;
    double2* E = reinterpret_cast<double2*>(X);
    for (int k = lane; k < 2 * p.n - 1; k += 32) {
      const int kk = k - nm1;
      const int ak = kk < 0 ? -kk : kk;
      E[k] = make_double2(TT[2 * ak], kk < 0 ? -TT[2 * ak + 1] : TT[2 * ak + 1]);
    }
    __syncwarp();
#pragma unroll
    for (int I = 0; I < NB; ++I)
#pragma unroll
      for (int J = 0; J <= I; ++J)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          if (!linked(I, J)) continue;
          // quadrant (cos / sin / middle) of block row I and block column J is compile-time
          const bool rc = I < NBc, rs = I >= NBc && I < 2 * NBc;
          const bool cc_ = J < NBc, cs = J >= NBc && J < 2 * NBc;
          const int a = rc ? I * 8 + q : (rs ? (I - NBc) * 8 + q : h);
          const int b = cc_ ? J * 8 + 2 * t + e : (cs ? (J - NBc) * 8 + 2 * t + e : h);
          const bool va = (rc || rs) ? a < h : q == 0;
          const bool vb = (cc_ || cs) ? b < h : (2 * t + e) == 0;
          double v = 0.0;
          if (!(va && vb)) {
          } else if (rc && cc_) v = 0.5 * (E[a - b + nm1].x + E[a + b].x);
          else if (rs && cs) v = 0.5 * (E[a - b + nm1].x - E[a + b].x);
          else if (rs && cc_) v = -0.5 * (E[a + b].y + E[a - b + nm1].y);
          else if (rc && cs) v = -0.5 * (E[a + b].y + E[b - a + nm1].y);
          else if (!rc && !rs && cc_) v = E[b - h + nm1].x;
          else if (!rc && !rs && cs) v = -E[b - h + nm1].y;
          else if (rc && !cc_ && !cs) v = E[a - h + nm1].x;
          else if (rs && !cc_ && !cs) v = -E[a - h + nm1].y;
          else v = E[nm1].x;
          g[blk(I, J)][e] = v;
        }
    __syncwarp();
    if (tma) stage_px_next(rep);  // X (= the table column's region in TMA mode) is free again
  }

  // ---------------------------------------------------------------- 2. + lam reg'
  {
    // reference rounding: ((wx^2 + wy^2)^2 * d^4 + eps), G += lam * reg (construct.py:283,194)
    const double lam = solve_lam(p);
    const double osq = __dadd_rn(__dmul_rn(ox, ox), __dmul_rn(oy, oy));
    const double w4 = __dmul_rn(osq, osq);
    // lane (q, t) holds diagonal entry (q, q) of each diagonal block iff q >> 1 == t
    const bool dlane = (q >> 1) == t;
    const int e = q & 1;
#pragma unroll
    for (int I = 0; I < NB; ++I) {
      if (dlane) {
        const double2 ab = RG[I * 8 + q];
        double add = 1.0;  // padding column: identity
        if (ab.x >= 0.0) {
          const double r1 = __dadd_rn(__dmul_rn(w4, ab.x), p.eps);
          if (ab.y >= 0.0) {
            // pair (p, n-1-p): lam (reg_p + reg_{n-1-p}) / 4 on the unscaled basis
            const double r2 = __dadd_rn(__dmul_rn(w4, ab.y), p.eps);
            add = __dmul_rn(lam, 0.25 * __dadd_rn(r1, r2));
          } else {
            add = __dmul_rn(lam, r1);
          }
          if (!(lam > 0.0)) add = 0.0;
        }
        if (e) g[blk(I, I)][1] = __dadd_rn(g[blk(I, I)][1], add);
        else g[blk(I, I)][0] = __dadd_rn(g[blk(I, I)][0], add);
      }
    }
  }

  // screen inputs of the reference's residual test (abi.cu: k1_screen_kernel):
  // ||rhs||_F^2 over the 2C right-hand sides and the largest diagonal entry of G
  if (p.audit) {
    double rs = 0.0, dm = 0.0;
    const bool dl = (q >> 1) == t;
#pragma unroll
    for (int I = 0; I < NB; ++I) {
      if (2 * t < 2 * p.C) rs = fma(r[I][0], r[I][0], rs);
      if (2 * t + 1 < 2 * p.C) rs = fma(r[I][1], r[I][1], rs);
      if (dl && RG[I * 8 + q].x >= 0.0) dm = fmax(dm, (q & 1) ? g[blk(I, I)][1] : g[blk(I, I)][0]);
    }
    float rsf = (float)rs, dmf = (float)dm;  // a screen with a 10x margin: fp32 reductions
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      rsf += __shfl_xor_sync(FULL, rsf, o);
      dmf = fmaxf(dmf, __shfl_xor_sync(FULL, dmf, o));
    }
    if (lane == 0) p.audit[soff] = make_float2(rsf, dmf);
  }

  // ---------------------------------------------------------------- 3. Cholesky + forward
  // Steps of one diagonal block, or (PAIR) of two -- cos block s and sin block
  // NBc + s, factored side by side by lanes 0..7 and 8..15 -- then the middle
  // block of odd n.
  bool ok = true;
  constexpr int NSTEP = PAIR ? NBc + ODD : NB;
#pragma unroll
  for (int st = 0; st < NSTEP; ++st) {
    const int Ka = PAIR ? (st < NBc ? st : NB - 1) : st;
    const int Kb = PAIR && st < NBc ? NBc + st : -1;
    // (a) factor the diagonal block(s) with 8 lanes each (lane = row) and invert;
    //     column values are broadcast by shuffles, pivots by rsqrt.
    store_cd(D0, g[blk(Ka, Ka)], lane);
    if (Kb >= 0) store_cd(D1, g[blk(Kb, Kb)], lane);
    __syncwarp();
    bool lok = true;
    if (lane < 16) {
      const int hi = lane >> 3, row = lane & 7;
      const bool own = hi == 0 || Kb >= 0;  // lanes 8..15 of a one-block step repeat lanes 0..7
      double* Sx = (hi && Kb >= 0) ? D1 : D0;
      double a[8], dinv[8];
#pragma unroll
      for (int c = 0; c < 8; ++c) a[c] = Sx[row * LDD + c];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const double akk = __shfl_sync(0xffffu, a[k], (lane & 8) | k);
        const bool good = (akk > 0.0) && isfinite(akk);
        lok = lok && good;
        const double inv = rsqrt_fast(good ? akk : 1.0);
        dinv[k] = inv;
        a[k] = (row == k) ? (good ? akk : 1.0) * inv : a[k] * inv;  // rows < k: unused upper part
#pragma unroll
        for (int c = k + 1; c < 8; ++c) a[c] = fma(-a[k], __shfl_sync(0xffffu, a[k], (lane & 8) | c), a[c]);  // upper: harmless
      }
      __syncwarp(0xffffu);
      if (own) {
#pragma unroll
        for (int c = 0; c < 8; ++c) Sx[row * LDD + c] = a[c];  // upper triangle ignored below
      }
      __syncwarp(0xffffu);
      // column `row` of W = L^-1: w_rr = (delta_rc - sum_{k<rr} L_rk w_k) / L_rr  (zero above c)
      const int c = row;
      double w[8];
#pragma unroll
      for (int rr = 0; rr < 8; ++rr) {
        double acc = (rr == c) ? 1.0 : 0.0;
#pragma unroll
        for (int k = 0; k < rr; ++k) acc = fma(-Sx[rr * LDD + k], w[k], acc);
        w[rr] = acc * dinv[rr];
      }
      if (own) {
        double* Wd = Wblk(hi ? Kb : Ka);
#pragma unroll
        for (int rr = 0; rr < 8; ++rr) Wd[rr * LD + c] = w[rr];
      }
    }
    ok = ok && __all_sync(FULL, lok);
    __syncwarp();
#pragma unroll
    for (int side = 0; side < 2; ++side) {
      const int K = side ? Kb : Ka;
      if (K < 0) continue;
      const double* Wk = Wblk(K);
      // A-fragment of W (= B-fragment of W^T): W[q][t], W[q][4+t]
      const double wa0 = Wk[q * LD + t], wa1 = Wk[q * LD + 4 + t];

      // (b) panel L_IK = G_IK W^T, kept in place (accumulator layout) and as A-fragments
      double lf[NB][2];
#pragma unroll
      for (int I = K + 1; I < NB; ++I) {
        if (!linked(I, K)) continue;
        double a0, a1;
        c_to_a(g[blk(I, K)], a0, a1, lane);
        double d[2] = {0.0, 0.0};
        dmma(d, a0, wa0);
        dmma(d, a1, wa1);
        g[blk(I, K)][0] = d[0];
        g[blk(I, K)][1] = d[1];
        c_to_a(d, lf[I][0], lf[I][1], lane);
      }
      // (c) trailing update
#pragma unroll
      for (int I = K + 1; I < NB; ++I)
#pragma unroll
        for (int J = K + 1; J <= I; ++J) {
          if (!linked(I, K) || !linked(J, K)) continue;
          dmma(g[blk(I, J)], -lf[I][0], lf[J][0]);
          dmma(g[blk(I, J)], -lf[I][1], lf[J][1]);
        }
      // (d) forward substitution: y_K = W r_K; r_I -= L_IK y_K
      //     (accumulator -> B fragment by shuffles: C[t][q], C[4+t][q])
      {
        double b0, b1;
        c_to_at(r[K], b0, b1, lane);
        double y[2] = {0.0, 0.0};
        dmma(y, wa0, b0);
        dmma(y, wa1, b1);
        r[K][0] = y[0];
        r[K][1] = y[1];
        c_to_at(y, b0, b1, lane);
#pragma unroll
        for (int I = K + 1; I < NB; ++I) {
          if (!linked(I, K)) continue;
          dmma(r[I], -lf[I][0], b0);
          dmma(r[I], -lf[I][1], b1);
        }
      }
    }
  }

  // ---------------------------------------------------------------- 4. backward
  bool finite = true;  // of the solution columns this lane holds
  double xa[NB][2];    // solved blocks, accumulator layout (the sin half waits for its cos partner)
  double xb[NB][2];    // solved blocks as B fragments (x[t][q], x[4+t][q])
#pragma unroll
  for (int K = NB - 1; K >= 0; --K) {
    double z[2] = {r[K][0], r[K][1]};
#pragma unroll
    for (int I = K + 1; I < NB; ++I) {
      if (!linked(I, K)) continue;
      double a0, a1;
      c_to_at(g[blk(I, K)], a0, a1, lane);  // L_IK^T
      dmma(z, -a0, xb[I][0]);
      dmma(z, -a1, xb[I][1]);
    }
    double b0, b1;
    c_to_at(z, b0, b1, lane);
    const double* Wk = Wblk(K);
    const double at0 = Wk[t * LD + q], at1 = Wk[(4 + t) * LD + q];  // W^T A-fragment
    double x[2] = {0.0, 0.0};
    dmma(x, at0, b0);
    dmma(x, at1, b1);
    finite = finite && (2 * t >= 2 * p.C || isfinite(x[0])) && (2 * t + 1 >= 2 * p.C || isfinite(x[1]));
    xa[K][0] = x[0];
    xa[K][1] = x[1];
    c_to_at(x, xb[K][0], xb[K][1], lane);
    // layer coefficients straight from this lane's solution entries (row K*8+q,
    // channel t): the sin block of a (cos, sin) pair is solved first
    if (t < p.C) {
      const size_t cb = (size_t)t * plane + boff;
      const size_t kst = (size_t)p.C * plane;
      if (MODE == MODE_SYMREAL) {
        const int pp = K * 8 + q;
        if (K < NBc && pp < h) {
          // v+ = aa + i bb, v- = cc + i dd;  x_p = (v+ + i v-)/2, x_{n-1-p} = (v+ - i v-)/2
          const double aa = x[0], bb = x[1], cc = xa[K + NBc][0], dd = xa[K + NBc][1];
          p.layers[(size_t)pp * kst + cb] = make_float2((float)(0.5 * (aa - dd)), (float)(0.5 * (bb + cc)));
          p.layers[(size_t)(p.n - 1 - pp) * kst + cb] = make_float2((float)(0.5 * (aa + dd)), (float)(0.5 * (bb - cc)));
        } else if (ODD && K == NB - 1 && q == 0) {
          p.layers[(size_t)h * kst + cb] = make_float2((float)x[0], (float)x[1]);
        }
      } else if (K * 8 + q < p.n) {
        p.layers[(size_t)(K * 8 + q) * kst + cb] = make_float2((float)x[0], (float)x[1]);
      }
    }
  }

  // ---------------------------------------------------------------- 5. output
  ok = __all_sync(FULL, finite) && ok;
  if (p.status && lane == 0) p.status[soff] = ok ? FDL_BIN_OK : FDL_BIN_BREAKDOWN;
  if (!ok) {  // breakdown (rare): the bin's layers become NaN (overwriting what backward stored)
    const float nanf_ = __int_as_float(0x7fc00000);
    for (int e = lane; e < p.n * p.C; e += 32) p.layers[(size_t)e * plane + boff] = make_float2(nanf_, nanf_);
  }
  }  // bins of this warp
}

// W12: returns FDL_OK with *launched = false when the 12-warp configuration does not apply
template <int NB, int MODE, int ODD, int PAIR, int W12>
int launch_fast_cfg(const SolveParams& p, const FastParams& f_in, cudaStream_t st, bool* launched) {
  constexpr int WARPS = K1Cfg<NB, MODE, PAIR, W12>::warps;
  constexpr int XW = xwords<NB, PAIR>();
  *launched = false;
  FastParams f = f_in;
  f.tma = 0;
  const int py_words = (MODE == MODE_SYMREAL) ? 2 * (f.nv + 1) * f.hwp : 0;  // + one all-zero row (padding rows)
  const int px_words = (MODE == MODE_SYMREAL) ? 2 * f.nu * f.hwp : 0;
  const int ro_words = (MODE == MODE_SYMREAL) ? 2 * ((p.mrow + 3) & ~3) : 3 * p.m * p.n;
  const size_t fixed_words = (size_t)py_words + ro_words + 1 + 2 * NB * 8;
  const size_t scratch_words = 2 * DSZ + 8 * LD + (NB - 1) * 8 * LD;
  size_t smem = sizeof(double) * (fixed_words + (size_t)WARPS * (px_words + scratch_words + XW + (((size_t)p.m * p.C + 1) & ~(size_t)1)));
  // TMA staging of the spectra (FastParams::tma): needs 16-byte plane strides, bins in
  // pairs, and room for the [plane][2] tiles
  CUtensorMap smap{};
  const size_t plane = (size_t)(p.plane_rows ? p.plane_rows : p.nrows) * p.Whp;
  if (MODE == MODE_SYMREAL && FDL_K1_TMA && WARPS % 2 == 0 && plane % 2 == 0 && plane * 2 < (1ull << 31) &&
      reinterpret_cast<uintptr_t>(p.spectra) % 16 == 0 && reinterpret_cast<uintptr_t>(f.px_all) % 16 == 0) {
    const int planes = p.m * p.C;
    // boxes of <= 256 planes, a multiple of 8 (128-byte shared-memory destinations); fewest padded planes
    int nbox = 0, box = 0;
    for (int nb = (planes + 255) / 256; nb <= (planes + 255) / 256 + 4; ++nb) {
      const int bx = (((planes + nb - 1) / nb) + 7) & ~7;
      if (bx <= 256 && (!nbox || nb * bx < nbox * box)) nbox = nb, box = bx;
    }
    // (the Toeplitz scratch shares the table column's region in this mode)
    const size_t warp_words = (size_t)(px_words > XW ? px_words : XW) + scratch_words + 2;
    const size_t tma_smem = ((sizeof(double) * (fixed_words + (size_t)WARPS * warp_words) + 127) & ~(size_t)127) +
                            (size_t)(WARPS / 2) * nbox * box * 16;
    EncodeTiledFn enc = encode_tiled_fn();
    if (enc && nbox && tma_smem <= 224 * 1024) {
      const cuuint64_t gdim[2] = {(cuuint64_t)plane * 2, (cuuint64_t)planes};
      const cuuint64_t gstride[1] = {(cuuint64_t)plane * 8};
      const cuuint32_t bx[2] = {4, (cuuint32_t)box};
      const cuuint32_t estr[2] = {1, 1};
      const CUresult r = enc(&smap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float2*>(p.spectra), gdim, gstride,
                             bx, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r == CUDA_SUCCESS) {
        f.tma = 1;
        f.bs_box = box;
        f.bs_nbox = nbox;
        smem = tma_smem;
      }
    }
  }
  if (W12 && !f.tma) return FDL_OK;  // the 12-warp CTA only fits with the TMA layout: caller falls back
  if (smem > 224 * 1024) return fail(FDL_ERR_UNSUPPORTED, "K1 fast path: phase tables exceed shared memory");
  auto kern = k1_fast_kernel<NB, MODE, ODD, PAIR, W12>;
  FDL_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  if (p.reps < 1) return fail(FDL_ERR_INVALID, "K1 fast path: reps < 1");
  // (TMA pairs: rows at an odd flat offset are shifted left by one bin)
  dim3 grid((unsigned)((p.Whp + f.tma + WARPS * p.reps - 1) / (WARPS * p.reps)), (unsigned)p.nrows);
  ktimer_mark(0, 0, st);
  kern<<<grid, WARPS * 32, smem, st>>>(p, f, smap);
  ktimer_mark(0, 1, st);
  FDL_LAUNCH_CHECK("k1_fast_kernel");
  *launched = true;
  return FDL_OK;
}

template <int NB, int MODE, int ODD, int PAIR>
int launch_fast(const SolveParams& p, const FastParams& f, cudaStream_t st) {
  bool launched = false;
  if constexpr (MODE == MODE_SYMREAL && PAIR && NB >= 7 && FDL_K1_W12) {
    const int rc = launch_fast_cfg<NB, MODE, ODD, PAIR, 1>(p, f, st, &launched);
    if (rc != FDL_OK || launched) return rc;
  }
  return launch_fast_cfg<NB, MODE, ODD, PAIR, 0>(p, f, st, &launched);
}

template <int MODE, int ODD, int PAIR>
int dispatch_nb(int NB, const SolveParams& p, const FastParams& f, cudaStream_t st) {
  switch (NB) {
    case 1: return launch_fast<1, MODE, ODD, PAIR>(p, f, st);
    case 2: return launch_fast<2, MODE, ODD, PAIR>(p, f, st);
    case 3: return launch_fast<3, MODE, ODD, PAIR>(p, f, st);
    case 4: return launch_fast<4, MODE, ODD, PAIR>(p, f, st);
    case 5: return launch_fast<5, MODE, ODD, PAIR>(p, f, st);
    case 6: return launch_fast<6, MODE, ODD, PAIR>(p, f, st);
    case 7: return launch_fast<7, MODE, ODD, PAIR>(p, f, st);
    case 8: return launch_fast<8, MODE, ODD, PAIR>(p, f, st);
    default: return fail(FDL_ERR_UNSUPPORTED, "NB");
  }
}

// ---------------------------------------------------------------- self test
__global__ void selftest_dmma_kernel(const double* A, const double* B, double* C) {
  // C (8x8) = A (8x8) B (8x8) through two k4 steps, all layouts as documented
  const int lane = threadIdx.x, q = lane >> 2, t = lane & 3;
  double c[2] = {0.0, 0.0};
  dmma(c, A[q * 8 + t], B[t * 8 + q]);
  dmma(c, A[q * 8 + 4 + t], B[(4 + t) * 8 + q]);
  C[q * 8 + 2 * t] = c[0];
  C[q * 8 + 2 * t + 1] = c[1];
  // and the shuffle converters: C-frag -> A-frag / transposed A-frag
  double a0, a1, b0, b1;
  c_to_a(c, a0, a1, lane);
  c_to_at(c, b0, b1, lane);
  C[64 + q * 8 + t] = a0;
  C[64 + q * 8 + 4 + t] = a1;
  C[128 + q * 8 + t] = b0;      // = C[t][q]
  C[128 + q * 8 + 4 + t] = b1;  // = C[4+t][q]
}

}  // namespace

int selftest_dmma(cudaStream_t st, double* max_err) {
  double hA[64], hB[64], ref[64], out[192];
  for (int e = 0; e < 64; ++e) {
    hA[e] = 0.25 * (e % 7) - 0.5 + 0.01 * e;
    hB[e] = 0.125 * (e % 5) + 0.003 * e - 0.2;
  }
  for (int r = 0; r < 8; ++r)
    for (int c = 0; c < 8; ++c) {
      double s = 0;
      for (int k = 0; k < 8; ++k) s += hA[r * 8 + k] * hB[k * 8 + c];
      ref[r * 8 + c] = s;
    }
  double* d;
  FDL_CUDA_CHECK(cudaMalloc(&d, sizeof(double) * (64 + 64 + 192)));
  FDL_CUDA_CHECK(cudaMemcpyAsync(d, hA, sizeof(hA), cudaMemcpyHostToDevice, st));
  FDL_CUDA_CHECK(cudaMemcpyAsync(d + 64, hB, sizeof(hB), cudaMemcpyHostToDevice, st));
  selftest_dmma_kernel<<<1, 32, 0, st>>>(d, d + 64, d + 128);
  FDL_CUDA_CHECK(cudaMemcpyAsync(out, d + 128, sizeof(out), cudaMemcpyDeviceToHost, st));
  FDL_CUDA_CHECK(cudaStreamSynchronize(st));
  cudaFree(d);
  double err = 0;
  for (int r = 0; r < 8; ++r)
    for (int c = 0; c < 8; ++c) {
      err = fmax(err, fabs(out[r * 8 + c] - ref[r * 8 + c]));
      err = fmax(err, fabs(out[64 + r * 8 + c] - ref[r * 8 + c]));
      err = fmax(err, fabs(out[128 + r * 8 + c] - ref[c * 8 + r]));
    }
  *max_err = err;
  return FDL_OK;
}

int k1_fast_launch(const SolveParams& p, cudaStream_t st, bool* handled) {
  *handled = false;
  if (p.mode == MODE_COMPLEX) return FDL_OK;
  if (p.C * 2 > 8) return FDL_OK;
  int NB;
  FastParams f{};
  if (p.mode == MODE_SYMREAL) {
    const int h = p.n / 2;
    f.H8 = ((h + 7) / 8) * 8;
    NB = 2 * f.H8 / 8 + (p.n & 1);
    f.hw = h + (p.n & 1);
    if (f.hw == 0) return FDL_OK;
    f.hwp = k1_table_pitch(p.n);
    // distinct u / v values (uploaded with the parameter block by the caller)
    if (!p.fast_u_idx || !p.fast_tables) return FDL_OK;
    f.u_idx = p.fast_u_idx;
    f.v_idx = p.fast_v_idx;
    f.u_val = p.fast_u_val;
    f.v_val = p.fast_v_val;
    f.nu = p.fast_nu;
    f.nv = p.fast_nv;
  } else {
    NB = (p.n + 7) / 8;
  }
  if (NB < 1 || NB > 8) return FDL_OK;
  *handled = true;
  if (p.mode == MODE_SYMREAL) {
    f.px_all = reinterpret_cast<const double2*>(p.fast_tables);
    f.py_all = f.px_all + (size_t)p.Whp * f.nu * f.hwp;
    const long long tot = ((long long)p.Whp * f.nu + (long long)p.nrows * f.nv) * f.hwp;
    int blocks = (int)std::min<long long>((tot + 255) / 256, 148LL * 8);
    k1_axis_tables_kernel<<<blocks, 256, 0, st>>>(p, f);
    FDL_LAUNCH_CHECK("k1_axis_tables_kernel");
    if (p.row_pairs)
      return (p.n & 1) ? dispatch_nb<MODE_SYMREAL, 1, 1>(NB, p, f, st) : dispatch_nb<MODE_SYMREAL, 0, 1>(NB, p, f, st);
    return (p.n & 1) ? dispatch_nb<MODE_SYMREAL, 1, 0>(NB, p, f, st) : dispatch_nb<MODE_SYMREAL, 0, 0>(NB, p, f, st);
  }
  return dispatch_nb<MODE_REALA, 0, 0>(NB, p, f, st);
}

}  // namespace fdl
