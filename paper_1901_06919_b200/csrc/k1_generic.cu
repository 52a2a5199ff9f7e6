// K1 generic path: one warp per frequency bin, the real ridge system in shared
// memory, right-looking Cholesky.  Any N <= 128 and any mode; it is the
// correctness baseline and the path for shapes the register-resident DMMA
// kernel (k1_dmma.cu) does not cover.
#include "k1_solve.cuh"

namespace fdl {

namespace {

// Row `r` of the real system (M row of N entries, B row of R entries).
__device__ void build_row(const SolveParams& p, int r, int i, int kx, int ky, double* Mrow, double* Brow) {
  const double ox = omega_x_label(kx, p.Wp);
  const double oy = omega_y_label(ky, p.Hp);
  const bool nyq_x = (p.Wp % 2 == 0) && kx == p.Wp / 2;
  const bool nyq_y = (p.Hp % 2 == 0) && ky == p.Hp / 2;
  const size_t plane = sp_plane(p);
  const size_t boff = sp_boff(p, i, kx);
  if (p.mode == MODE_SYMREAL) {
    const int j = r;
    for (int q = 0; q < p.h; ++q) {
      cd a = system_entry(p, j, q, kx, ky, ox, oy, nyq_x, nyq_y);
      Mrow[q] = M_SQRT2 * a.re;
      Mrow[p.h + q] = -M_SQRT2 * a.im;
    }
    if (p.n & 1) Mrow[2 * p.h] = system_entry(p, j, p.h, kx, ky, ox, oy, nyq_x, nyq_y).re;
    for (int c = 0; c < p.C; ++c) {
      float2 b = p.spectra[((size_t)j * p.C + c) * plane + boff];
      Brow[2 * c] = b.x;
      Brow[2 * c + 1] = b.y;
    }
  } else if (p.mode == MODE_REALA) {
    const int j = r;
    for (int k = 0; k < p.n; ++k) Mrow[k] = system_entry(p, j, k, kx, ky, ox, oy, nyq_x, nyq_y).re;
    for (int c = 0; c < p.C; ++c) {
      float2 b = p.spectra[((size_t)j * p.C + c) * plane + boff];
      Brow[2 * c] = b.x;
      Brow[2 * c + 1] = b.y;
    }
  } else {
    const bool lower = r >= p.m;
    const int j = lower ? r - p.m : r;
    for (int k = 0; k < p.n; ++k) {
      cd a = system_entry(p, j, k, kx, ky, ox, oy, nyq_x, nyq_y);
      if (!lower) {
        Mrow[k] = a.re;
        Mrow[p.n + k] = -a.im;
      } else {
        Mrow[k] = a.im;
        Mrow[p.n + k] = a.re;
      }
    }
    for (int c = 0; c < p.C; ++c) {
      float2 b = p.spectra[((size_t)j * p.C + c) * plane + boff];
      Brow[c] = lower ? b.y : b.x;
    }
  }
}

__global__ void k1_generic_kernel(SolveParams p) {
  extern __shared__ double smem[];
  const int warps = blockDim.x >> 5, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long nbins = (long long)p.nrows * p.Whp;
  const long long bin = (long long)blockIdx.x * warps + warp;
  if (bin >= nbins) return;  // warp-uniform; no block-level barriers below
  const int N = p.N, R = p.R, ld = N + 1;
  const size_t per_warp = (size_t)N * ld + (size_t)N * R + 32 * (size_t)N + 32 * (size_t)R;
  double* G = smem + warp * per_warp;
  double* Rh = G + (size_t)N * ld;
  double* Ms = Rh + (size_t)N * R;
  double* Bs = Ms + 32 * (size_t)N;
  const int i = (int)(bin / p.Whp), kx = (int)(bin % p.Whp);
  const int ky = p.rows[i];

  for (int e = lane; e < N * ld; e += 32) G[e] = 0.0;
  for (int e = lane; e < N * R; e += 32) Rh[e] = 0.0;
  __syncwarp();

  const int npairs = N * (N + 1) / 2;
  for (int r0 = 0; r0 < p.rowsM; r0 += 32) {
    const int cnt = min(32, p.rowsM - r0);
    if (lane < cnt) build_row(p, r0 + lane, i, kx, ky, Ms + lane * N, Bs + lane * R);
    __syncwarp();
    for (int e = lane; e < npairs; e += 32) {
      // e -> (a, b) with a >= b, row-major lower triangle
      int a = (int)((sqrt(8.0 * e + 1.0) - 1.0) * 0.5);
      while ((a + 1) * (a + 2) / 2 <= e) ++a;
      while (a * (a + 1) / 2 > e) --a;
      int b = e - a * (a + 1) / 2;
      double acc = 0.0;
      for (int rr = 0; rr < cnt; ++rr) acc = fma(Ms[rr * N + a], Ms[rr * N + b], acc);
      G[a * ld + b] += acc;
    }
    for (int e = lane; e < N * R; e += 32) {
      int a = e / R, c = e % R;
      double acc = 0.0;
      for (int rr = 0; rr < cnt; ++rr) acc = fma(Ms[rr * N + a], Bs[rr * R + c], acc);
      Rh[a * R + c] += acc;
    }
    __syncwarp();
  }

  // + lam * reg'
  const double ox = omega_x_label(kx, p.Wp), oy = omega_y_label(ky, p.Hp);
  const double w2 = ox * ox + oy * oy, w4 = w2 * w2;
  const double lam = solve_lam(p);
  if (lam > 0.0)
    for (int a = lane; a < N; a += 32) G[a * ld + a] += lam * real_reg(p, a, w4);
  __syncwarp();

  if (p.audit) {  // screen inputs of the residual test: ||rhs||_F^2 and max diag(G)
    double rs = 0.0, dm = 0.0;
    for (int e = lane; e < N * R; e += 32) rs = fma(Rh[e], Rh[e], rs);
    for (int a = lane; a < N; a += 32) dm = fmax(dm, G[a * ld + a]);
    for (int o = 16; o > 0; o >>= 1) {
      rs += __shfl_xor_sync(0xffffffffu, rs, o);
      dm = fmax(dm, __shfl_xor_sync(0xffffffffu, dm, o));
    }
    if (lane == 0) p.audit[bin] = make_float2((float)rs, (float)dm);
  }

  // right-looking Cholesky, lower triangle in place
  bool ok = true;
  for (int k = 0; k < N; ++k) {
    double piv = G[k * ld + k];
    if (!(piv > 0.0) || !isfinite(piv)) {
      ok = false;
      break;
    }
    double lkk = sqrt(piv), inv = 1.0 / lkk;
    __syncwarp();
    for (int a = k + 1 + lane; a < N; a += 32) G[a * ld + k] *= inv;
    if (lane == 0) G[k * ld + k] = lkk;
    __syncwarp();
    const int t = N - k - 1, tp = t * (t + 1) / 2;
    for (int e = lane; e < tp; e += 32) {
      int a = (int)((sqrt(8.0 * e + 1.0) - 1.0) * 0.5);
      while ((a + 1) * (a + 2) / 2 <= e) ++a;
      while (a * (a + 1) / 2 > e) --a;
      int b = e - a * (a + 1) / 2;
      a += k + 1;
      b += k + 1;
      G[a * ld + b] = fma(-G[a * ld + k], G[b * ld + k], G[a * ld + b]);
    }
    __syncwarp();
  }

  const size_t plane = sp_plane(p);
  const size_t boff = sp_boff(p, i, kx);
  if (!ok) {
    if (p.status && lane == 0) p.status[bin] = FDL_BIN_BREAKDOWN;
    const float nanf_ = __int_as_float(0x7fc00000);
    for (int e = lane; e < p.n * p.C; e += 32) p.layers[(size_t)e * plane + boff] = make_float2(nanf_, nanf_);
    return;
  }
  // forward / backward substitution, one lane per right-hand side
  if (lane < R) {
    const int c = lane;
    for (int a = 0; a < N; ++a) {
      double v = Rh[a * R + c];
      for (int k = 0; k < a; ++k) v = fma(-G[a * ld + k], Rh[k * R + c], v);
      Rh[a * R + c] = v / G[a * ld + a];
    }
    for (int a = N - 1; a >= 0; --a) {
      double v = Rh[a * R + c];
      for (int k = a + 1; k < N; ++k) v = fma(-G[k * ld + a], Rh[k * R + c], v);
      Rh[a * R + c] = v / G[a * ld + a];
    }
  }
  __syncwarp();
  bool finite = true;
  for (int e = lane; e < N * R; e += 32) finite &= isfinite(Rh[e]);
  finite = __all_sync(0xffffffffu, finite);
  if (p.status && lane == 0) p.status[bin] = finite ? FDL_BIN_OK : FDL_BIN_BREAKDOWN;

  // back to complex layer coefficients x_k (channel c)
  for (int e = lane; e < p.n * p.C; e += 32) {
    const int k = e / p.C, c = e % p.C;
    double xr, xi;
    if (p.mode == MODE_SYMREAL) {
      const int h = p.h;
      if ((p.n & 1) && k == h) {
        xr = Rh[(2 * h) * R + 2 * c];
        xi = Rh[(2 * h) * R + 2 * c + 1];
      } else {
        const bool hi = k >= h;
        const int q = hi ? p.n - 1 - k : k;
        // y+ = (a + i b), y- = (cc + i dd);  x_q = (y+ + i y-)/sqrt2, x_{n-1-q} = (y+ - i y-)/sqrt2
        const double a = Rh[q * R + 2 * c], b = Rh[q * R + 2 * c + 1];
        const double cc = Rh[(h + q) * R + 2 * c], dd = Rh[(h + q) * R + 2 * c + 1];
        if (!hi) {
          xr = (a - dd) * M_SQRT1_2;
          xi = (b + cc) * M_SQRT1_2;
        } else {
          xr = (a + dd) * M_SQRT1_2;
          xi = (b - cc) * M_SQRT1_2;
        }
      }
    } else if (p.mode == MODE_REALA) {
      xr = Rh[k * R + 2 * c];
      xi = Rh[k * R + 2 * c + 1];
    } else {
      xr = Rh[k * R + c];
      xi = Rh[(p.n + k) * R + c];
    }
    p.layers[((size_t)k * p.C + c) * plane + boff] = make_float2((float)xr, (float)xi);
  }
}

}  // namespace

size_t k1_generic_smem_per_warp(int N, int R) {
  return sizeof(double) * ((size_t)N * (N + 1) + (size_t)N * R + 32 * (size_t)N + 32 * (size_t)R);
}

int k1_generic_launch(const SolveParams& p, cudaStream_t st) {
  const size_t per_warp = k1_generic_smem_per_warp(p.N, p.R);
  int warps = (int)((200u * 1024u) / per_warp);
  if (warps > 8) warps = 8;
  if (warps < 1) return fail(FDL_ERR_UNSUPPORTED, "system too large for the generic K1 kernel");
  const size_t smem = per_warp * warps;
  FDL_CUDA_CHECK(cudaFuncSetAttribute(k1_generic_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const long long nbins = (long long)p.nrows * p.Whp;
  const long long blocks = (nbins + warps - 1) / warps;
  if (blocks == 0) return FDL_OK;
  ktimer_mark(0, 0, st);
  k1_generic_kernel<<<(unsigned)blocks, warps * 32, smem, st>>>(p);
  ktimer_mark(0, 1, st);
  FDL_LAUNCH_CHECK("k1_generic_kernel");
  return FDL_OK;
}

}  // namespace fdl
