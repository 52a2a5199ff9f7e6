// K1 shared definitions: the per-bin real ridge system.
//
// Every stored frequency bin q = (ky, kx) carries the complex Tikhonov problem
// of construct.py:183-211:
//     x = argmin ||A x - b||^2 + lam * sum_k reg_k |x_k|^2,
//     A_jk = px_jk * py_jk * psi_j(t_jk wx, t_jk wy),  reg_k = (wx^2+wy^2)^2 d_k^4 + eps.
// The kernels solve it as a REAL ridge regression  min ||M y - B||^2 + lam sum reg'_p y_p^2
// built on the fly from the bin's frequency, in one of three exact re-writes:
//
//  SYMREAL (mode 1): pinhole factored views and d symmetric about 0
//      (d_k = -d_{n-1-k}).  Then A_{j,n-1-k} = conj(A_jk), the Gram matrix is
//      centro-Hermitian (J G J = conj G) and the unitary change of basis
//      e+_p = (e_p + e_{n-1-p})/sqrt2, e-_p = i (e_p - e_{n-1-p})/sqrt2 makes
//      M = A U real: M[:, p] = sqrt2 Re A_p, M[:, h+p] = -sqrt2 Im A_p (p < h = n/2),
//      M[:, 2h] = Re A_mid for odd n.  Re b and Im b are independent right-hand
//      sides (R = 2C); N = n.  reg'_p = reg'_{h+p} = reg_p.
//      Mirror pairs: if every view j has a partner j' with (u, v)_j' = -(u, v)_j
//      (or sits at the origin), then A_j'k = conj(A_jk), so Re A_j' = Re A_j and
//      Im A_j' = -Im A_j.  Summing the pair's normal-equation contributions,
//          G = sum_j M_j^T M_j = [[2 sum' c c^T, 0], [0, 2 sum' s s^T]] (+ origin rows),
//          M^T b = [sum' c (b_j + b_j'); -sum' s (b_j - b_j')],
//      (sum' over one view per pair), the cos and sin halves decouple exactly:
//      two independent systems of half the size, each built from half the rows.
//  REALA   (mode 2): every P = 0 (all views at u = v = 0, the focal-stack
//      input, construct.py:170-179) and real aperture tables -> A is real:
//      M = A, R = 2C, N = n.
//  COMPLEX (mode 3): anything else, through the real embedding
//      M = [[Re A, -Im A], [Im A, Re A]] (2m x 2n), B = [Re b; Im b], R = C, N = 2n.
//
// All three are orthogonal re-writes of the same least-squares problem, so
// the solution is the reference's up to rounding.
#pragma once
#include "common.cuh"

namespace fdl {

enum SolveMode { MODE_SYMREAL = 1, MODE_REALA = 2, MODE_COMPLEX = 3 };

struct SolveParams {
  int m, n, C, Hp, Wp, Whp, nrows;
  int mode, N, R, rowsM, h;  // real system: N unknowns, R right-hand sides, rowsM equations
  const int* rows;           // (nrows) ky of each slab row
  const double* pu;          // (m, n)
  const double* pv;          // (m, n)
  const double* d4;          // (n) d^4
  const int* view_ap;        // (m) or nullptr
  const double* s;           // (m)
  const double* scale;       // (m)
  const DevAperture* aps;
  const double* d;           // (n)
  double lam, eps;
  const double* lam_dev;     // device lambda (overrides lam) or nullptr
  const float2* spectra;     // (m, C, nrows, Whp)
  float2* layers;            // (n, C, nrows, Whp)
  signed char* status;       // (nrows, Whp) or nullptr
  float2* audit;             // (nrows, Whp) per-bin (||rhs||_F^2, max diag G) for the residual screen, or nullptr
  int uniform_d;             // d_k = d_0 + k delta (Toeplitz Gram available)
  int uniform_ap;            // >= 0: every view uses aperture uniform_ap (mode 2 hoists its fields)
  int reps;                  // K1 fast path: bins per warp (CTAs cover reps * 8 columns)
  int plane_rows;            // 0: slab buffers (row i); > 0: full-grid buffers of plane_rows rows (row rows[i])
  double delta;
  // factored shifts: distinct u / v values (per-axis phase tables of the fast path)
  const int* fast_u_idx;
  const int* fast_v_idx;
  const double* fast_u_val;
  const double* fast_v_val;
  int fast_nu, fast_nv;
  double* fast_tables;       // workspace for the per-axis phase tables (fast path)
  // SYMREAL with a mirror-symmetric view set (every view j has a partner j'
  // with (u, v)_j' = -(u, v)_j, or sits at u = v = 0): the fast path sums the
  // pair's equations (see the header) and solves the cos and sin halves as two
  // independent systems.  row_pairs[r] = (j, j' or -1), r < mrow.
  const int2* row_pairs;     // nullptr: no pairing (mrow = m)
  int mrow;
};

// lambda of this solve: the device scalar when the caller computed it there
__device__ __forceinline__ double solve_lam(const SolveParams& p) { return p.lam_dev ? __ldg(p.lam_dev) : p.lam; }

// Row pitch (double2 entries) of the mode-1 per-axis phase tables: covers the n/2 (+1 for odd n)
// entries AND every column of the 8-wide blocks (zero-filled, so the k-steps read them
// unconditionally), and is 2 (mod 8) so that 4 views x 2 layers of a quarter-warp hit distinct banks.
__host__ __device__ inline int k1_table_pitch(int n) {
  const int hw = n / 2 + (n & 1), h8 = ((n / 2 + 7) / 8) * 8;
  const int w = hw > h8 ? hw : h8;
  return w + ((2 - w % 8) + 8) % 8;
}

// spectra / layers addressing: slab buffers or full-grid buffers (plane_rows)
__device__ __forceinline__ size_t sp_plane(const SolveParams& p) {
  return (size_t)(p.plane_rows ? p.plane_rows : p.nrows) * p.Whp;
}
__device__ __forceinline__ size_t sp_boff(const SolveParams& p, int i, int kx) {
  return (size_t)(p.plane_rows ? p.rows[i] : i) * p.Whp + kx;
}

// A_jk (construct.py:168-180 with build_system_row's Nyquist handling, construct.py:83-109)
__device__ inline cd system_entry(const SolveParams& p, int j, int k, int kx, int ky, double ox, double oy,
                                  bool nyq_x, bool nyq_y) {
  const double Pu = p.pu[(size_t)j * p.n + k];
  const double Pv = p.pv[(size_t)j * p.n + k];
  cd a = cmul_rn(axis_phase(Pu, ox, nyq_x), axis_phase(Pv, oy, nyq_y));
  if (p.view_ap) {
    int ai = p.view_ap[j];
    if (ai >= 0) {
      const double t = __dmul_rn(p.scale[j], __dsub_rn(p.s[j], p.d[k]));
      cd psi = aperture_eval(p.aps[ai], __dmul_rn(t, ox), __dmul_rn(t, oy));
      // numpy complex * complex(psi): for a real table psi.im = 0
      a = psi.im == 0.0 ? cd{__dmul_rn(a.re, psi.re), __dmul_rn(a.im, psi.re)} : cmul_rn(a, psi);
    }
  }
  return a;
}

// reg'_col of the real system (see header)
__device__ inline double real_reg(const SolveParams& p, int col, double w4) {
  int k;
  if (p.mode == MODE_SYMREAL) {
    k = col < p.h ? col : (col < 2 * p.h ? col - p.h : p.n / 2);
  } else if (p.mode == MODE_REALA) {
    k = col;
  } else {
    k = col < p.n ? col : col - p.n;
  }
  return w4 * p.d4[k] + p.eps;
}

}  // namespace fdl
