// Calibration batch kernels (calibrate.py:139-229): the closed-form layer
// solve of a batch of frequency bins at given shift matrices, the regularised
// objective and its analytic gradient with respect to Pu and Pv.
//
//  * calib_solve_kernel (one CTA per bin): A_jk = px_jk py_jk from the
//    reference's `_phase_tables` rounding (construct.py:68-80, via axis_phase),
//    G = A^H A + lam Gamma^T Gamma and rhs = A^H b in shared memory
//    (calibrate.py:157-163), complex Cholesky + two triangular solves -> x.
//    G is Hermitian positive definite whenever the reference's LU succeeds
//    with lam > 0 (Gamma^T Gamma is); a non-positive pivot flags the bin
//    (status 2) and leaves G and rhs for the minimum-norm fallback, the
//    reference's `lstsq(G, rhs)` (calibrate.py:164-169).
//  * calib_terms_kernel (persistent CTAs): r = A x - b, the per-bin objective
//    sum |r|^2 + lam |Gamma x|^2 (calibrate.py:172-178) and, optionally, the
//    gradient partials Im(conj(A_jk) w r_j conj(x_k)) with w = omega_x / omega_y
//    (calibrate.py:219-229) accumulated per CTA in shared memory;
//  * calib_reduce_kernel: CTA partials and per-bin objective terms summed in a
//    fixed order (the result does not depend on scheduling).
#include <algorithm>
#include <cmath>

#include "common.cuh"

namespace fdl {

namespace {

constexpr int CT = 128;  // threads per CTA

struct CalibParams {
  int m, n, B, H, W, Wh;
  const int* bins;       // (B) q = ky * Wh + kx
  const double* pu;      // (m, n)
  const double* pv;      // (m, n)
  const double2* spec;   // (H * Wh, m)
  const double* gram;    // (n, n) Gamma^T Gamma
  const double* gamma;   // (n, n)
  double lam;
  double2* x;            // (B, n)
  signed char* status;   // (B)
  double2* gfall;        // (B, n, n) G of flagged bins
  double2* rfall;        // (B, n) rhs of flagged bins
  double* obj_bins;      // (B) per-bin objective terms
  double* gpart;         // (nCTA, 2, m, n) gradient partials, or nullptr
};

__device__ inline double2 cjmul(double2 a, double2 b) {  // conj(a) * b, numpy rounding
  return make_double2(__dadd_rn(__dmul_rn(a.x, b.x), __dmul_rn(a.y, b.y)),
                      __dsub_rn(__dmul_rn(a.x, b.y), __dmul_rn(a.y, b.x)));
}

__device__ inline void bin_freq(const CalibParams& p, int bin, int& q, double& ox, double& oy, bool& nx, bool& ny) {
  q = p.bins[bin];
  const int ky = q / p.Wh, kx = q - ky * p.Wh;
  ox = omega_x_label(kx, p.W);
  oy = omega_y_label(ky, p.H);
  nx = (p.W % 2 == 0) && kx == p.W / 2;
  ny = (p.H % 2 == 0) && ky == p.H / 2;
}

// A (m x n, row-major) of one bin into shared memory (calibrate.py:139-141)
__device__ inline void build_A(const CalibParams& p, double2* A, double ox, double oy, bool nx, bool ny) {
  for (int e = threadIdx.x; e < p.m * p.n; e += blockDim.x) {
    const cd a = cmul_rn(axis_phase(p.pu[e], ox, nx), axis_phase(p.pv[e], oy, ny));
    A[e] = make_double2(a.re, a.im);
  }
}

__device__ inline double block_sum(double v, double* red) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double t = 0.0;
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
  return t;
}

__global__ void __launch_bounds__(CT) calib_solve_kernel(CalibParams p) {
  extern __shared__ double2 sh[];
  const int m = p.m, n = p.n, bin = blockIdx.x;
  double2* A = sh;              // m x n
  double2* G = A + m * n;       // n x n (lower triangle used)
  double2* rhs = G + n * n;     // n
  double2* bv = rhs + n;        // m
  __shared__ int fail_flag;
  int q;
  double ox, oy;
  bool nx, ny;
  bin_freq(p, bin, q, ox, oy, nx, ny);
  if (threadIdx.x == 0) fail_flag = 0;
  for (int j = threadIdx.x; j < m; j += blockDim.x) bv[j] = p.spec[(size_t)q * m + j];
  build_A(p, A, ox, oy, nx, ny);
  __syncthreads();
  // G_kl = sum_j conj(A_jk) A_jl + lam gram_kl (l <= k), rhs_k = sum_j conj(A_jk) b_j
  auto form = [&]() {
    for (int e = threadIdx.x; e < n * n + n; e += blockDim.x) {
      if (e < n * n) {
        const int k = e / n, l = e - k * n;
        if (l > k) continue;
        double2 acc = make_double2(0.0, 0.0);
        for (int j = 0; j < m; ++j) {
          const double2 t = cjmul(A[j * n + k], A[j * n + l]);
          acc.x += t.x;
          acc.y += t.y;
        }
        if (p.lam > 0.0) acc.x += p.lam * p.gram[e];
        G[e] = acc;
      } else {
        const int k = e - n * n;
        double2 acc = make_double2(0.0, 0.0);
        for (int j = 0; j < m; ++j) {
          const double2 t = cjmul(A[j * n + k], bv[j]);
          acc.x += t.x;
          acc.y += t.y;
        }
        rhs[k] = acc;
      }
    }
  };
  form();
  __syncthreads();
  // right-looking complex Cholesky G = L L^H in place (lower triangle)
  for (int k = 0; k < n; ++k) {
    const double d = G[k * n + k].x;
    if (!(d > 0.0) || !isfinite(d)) {
      if (threadIdx.x == 0) fail_flag = 1;
      break;  // uniform: every thread read the same d
    }
    const double ld = sqrt(d), inv = 1.0 / ld;
    __syncthreads();  // everyone has read d before column k changes
    for (int i = k + threadIdx.x; i < n; i += blockDim.x) {
      if (i == k) G[k * n + k] = make_double2(ld, 0.0);
      else G[i * n + k] = make_double2(G[i * n + k].x * inv, G[i * n + k].y * inv);
    }
    __syncthreads();
    const int rem = n - k - 1;
    for (int e = threadIdx.x; e < rem * rem; e += blockDim.x) {
      const int i = k + 1 + e / rem, jj = k + 1 + e % rem;
      if (jj > i) continue;
      const double2 li = G[i * n + k], lj = G[jj * n + k];
      // G_ij -= L_ik conj(L_jk)
      G[i * n + jj].x -= li.x * lj.x + li.y * lj.y;
      G[i * n + jj].y -= li.y * lj.x - li.x * lj.y;
    }
    __syncthreads();
  }
  __syncthreads();
  if (fail_flag) {
    // leave G and rhs for the minimum-norm fallback (G rebuilt: the factorisation overwrote it)
    __syncthreads();
    form();
    __syncthreads();
    for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
      const int k = e / n, l = e - k * n;
      p.gfall[(size_t)bin * n * n + e] = l <= k ? G[e] : make_double2(G[l * n + k].x, -G[l * n + k].y);
    }
    for (int k = threadIdx.x; k < n; k += blockDim.x) p.rfall[(size_t)bin * n + k] = rhs[k];
    if (threadIdx.x == 0) p.status[bin] = 2;
    return;
  }
  // L y = rhs, L^H x = y (one warp; n <= 64 so two lanes' worth of rows per pass)
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    for (int k = 0; k < n; ++k) {
      double2 s = make_double2(0.0, 0.0);
      for (int l = lane; l < k; l += 32) {
        const double2 a = G[k * n + l], y = rhs[l];
        s.x += a.x * y.x - a.y * y.y;
        s.y += a.x * y.y + a.y * y.x;
      }
      for (int o = 16; o > 0; o >>= 1) {
        s.x += __shfl_xor_sync(0xffffffffu, s.x, o);
        s.y += __shfl_xor_sync(0xffffffffu, s.y, o);
      }
      if (lane == 0) {
        const double l = G[k * n + k].x;
        rhs[k] = make_double2((rhs[k].x - s.x) / l, (rhs[k].y - s.y) / l);
      }
      __syncwarp();
    }
    for (int k = n - 1; k >= 0; --k) {
      double2 s = make_double2(0.0, 0.0);
      for (int i = k + 1 + lane; i < n; i += 32) {  // sum_i conj(L_ik) x_i
        const double2 a = G[i * n + k], y = rhs[i];
        s.x += a.x * y.x + a.y * y.y;
        s.y += a.x * y.y - a.y * y.x;
      }
      for (int o = 16; o > 0; o >>= 1) {
        s.x += __shfl_xor_sync(0xffffffffu, s.x, o);
        s.y += __shfl_xor_sync(0xffffffffu, s.y, o);
      }
      if (lane == 0) {
        const double l = G[k * n + k].x;
        rhs[k] = make_double2((rhs[k].x - s.x) / l, (rhs[k].y - s.y) / l);
      }
      __syncwarp();
    }
    for (int k = lane; k < n; k += 32) p.x[(size_t)bin * n + k] = rhs[k];
    if (lane == 0) p.status[bin] = 0;
  }
}

__global__ void __launch_bounds__(CT) calib_terms_kernel(CalibParams p) {
  extern __shared__ double2 sh[];
  const int m = p.m, n = p.n;
  double2* A = sh;             // m x n
  double2* xs = A + m * n;     // n
  double2* r = xs + n;         // m
  double* gu = reinterpret_cast<double*>(r + m);  // m x n
  double* gv = gu + m * n;                        // m x n
  __shared__ double red[CT / 32];
  const bool grad = p.gpart != nullptr;
  if (grad)
    for (int e = threadIdx.x; e < 2 * m * n; e += blockDim.x) gu[e] = 0.0;
  for (int bin = blockIdx.x; bin < p.B; bin += gridDim.x) {
    int q;
    double ox, oy;
    bool nx, ny;
    bin_freq(p, bin, q, ox, oy, nx, ny);
    __syncthreads();  // previous bin's readers are done
    for (int k = threadIdx.x; k < n; k += blockDim.x) xs[k] = p.x[(size_t)bin * n + k];
    build_A(p, A, ox, oy, nx, ny);
    __syncthreads();
    // r = A x - b (calibrate.py:173)
    double part = 0.0;
    for (int j = threadIdx.x; j < m; j += blockDim.x) {
      double2 s = make_double2(0.0, 0.0);
      for (int k = 0; k < n; ++k) {
        const double2 a = A[j * n + k], xv = xs[k];
        s.x += a.x * xv.x - a.y * xv.y;
        s.y += a.x * xv.y + a.y * xv.x;
      }
      const double2 b = p.spec[(size_t)q * m + j];
      s.x -= b.x;
      s.y -= b.y;
      r[j] = s;
      part += s.x * s.x + s.y * s.y;
    }
    // lam |Gamma x|^2 (calibrate.py:175-177)
    if (p.lam > 0.0) {
      for (int k = threadIdx.x; k < n; k += blockDim.x) {
        double2 s = make_double2(0.0, 0.0);
        for (int l = 0; l < n; ++l) {
          const double g = p.gamma[k * n + l];
          s.x += g * xs[l].x;
          s.y += g * xs[l].y;
        }
        part += p.lam * (s.x * s.x + s.y * s.y);
      }
    }
    const double tot = block_sum(part, red);
    if (threadIdx.x == 0) p.obj_bins[bin] = tot;
    if (grad) {
      __syncthreads();  // r complete
      for (int e = threadIdx.x; e < m * n; e += blockDim.x) {
        const int j = e / n, k = e - j * n;
        // Im(conj(A_jk) r_j conj(x_k))
        const double2 a = A[e], rj = r[j], xk = xs[k];
        const double2 t = make_double2(a.x * rj.x + a.y * rj.y, a.x * rj.y - a.y * rj.x);  // conj(a) r
        const double im = t.y * xk.x - t.x * xk.y;                                           // Im(t conj(x))
        gu[e] += ox * im;
        gv[e] += oy * im;
      }
    }
  }
  if (grad) {
    __syncthreads();
    for (int e = threadIdx.x; e < 2 * m * n; e += blockDim.x) p.gpart[(size_t)blockIdx.x * 2 * m * n + e] = gu[e];
  }
}

// block 0: obj = sum of the per-bin objective terms (strided partial sums and a
// shared-memory tree, a fixed order); blocks >= 1: grad[e] = 4 pi sum_cta partial[cta][e]
__global__ void calib_reduce_kernel(const double* obj_bins, int B, const double* gpart, int nparts, int len,
                                    double* obj, double* grad) {
  if (blockIdx.x == 0) {
    __shared__ double t[256];
    double s = 0.0;
    for (int b = threadIdx.x; b < B; b += blockDim.x) s += obj_bins[b];
    t[threadIdx.x] = s;
    __syncthreads();
    for (int w = blockDim.x / 2; w > 0; w >>= 1) {
      if ((int)threadIdx.x < w) t[threadIdx.x] += t[threadIdx.x + w];
      __syncthreads();
    }
    if (threadIdx.x == 0) *obj = t[0];
    return;
  }
  const int e = (blockIdx.x - 1) * blockDim.x + threadIdx.x;
  if (e < len && gpart) {
    double s = 0.0;
    for (int c = 0; c < nparts; ++c) s += gpart[(size_t)c * len + e];
    grad[e] = 4.0 * M_PI * s;
  }
}

}  // namespace

size_t calib_solve_smem(int m, int n) { return sizeof(double2) * ((size_t)m * n + (size_t)n * n + n + m); }
size_t calib_terms_smem(int m, int n) { return sizeof(double2) * ((size_t)m * n + n + m) + 2 * sizeof(double) * m * n; }
int calib_terms_ctas(int B) { return std::max(1, std::min(B, 2 * 148)); }

int calib_launch(int m, int n, int B, int H, int W, const int* bins, const double* pu, const double* pv,
                 const double2* spec, const double* gram, const double* gamma, double lam, double2* x,
                 signed char* status, double2* gfall, double2* rfall, double* obj_bins, double* gpart,
                 double* obj, double* grad, bool solve, bool terms, cudaStream_t st) {
  CalibParams p{m, n, B, H, W, W / 2 + 1, bins, pu, pv, spec, gram, gamma, lam, x, status, gfall, rfall, obj_bins, gpart};
  if (B == 0) return FDL_OK;
  if (solve) {
    const size_t smem = calib_solve_smem(m, n);
    if (smem > 200 * 1024) return fail(FDL_ERR_UNSUPPORTED, "calibration: m * n too large for one CTA");
    FDL_CUDA_CHECK(cudaFuncSetAttribute(calib_solve_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    calib_solve_kernel<<<B, CT, smem, st>>>(p);
    FDL_LAUNCH_CHECK("calib_solve_kernel");
  }
  if (terms) {
    const size_t smem = calib_terms_smem(m, n);
    if (smem > 200 * 1024) return fail(FDL_ERR_UNSUPPORTED, "calibration: m * n too large for one CTA");
    FDL_CUDA_CHECK(cudaFuncSetAttribute(calib_terms_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const int ctas = calib_terms_ctas(B);
    calib_terms_kernel<<<ctas, CT, smem, st>>>(p);
    FDL_LAUNCH_CHECK("calib_terms_kernel");
    const int len = 2 * m * n;
    calib_reduce_kernel<<<1 + (gpart ? (len + 255) / 256 : 0), 256, 0, st>>>(obj_bins, B, gpart, ctas, len, obj, grad);
    FDL_LAUNCH_CHECK("calib_reduce_kernel");
  }
  return FDL_OK;
}

}  // namespace fdl
