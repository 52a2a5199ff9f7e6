// Shared helpers for the FDL B200 kernels (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <string>

#include "fdl_b200.h"

namespace fdl {

// ---------------------------------------------------------------------------
// thread-local error reporting for the C ABI
// ---------------------------------------------------------------------------
void set_error(const std::string& msg);
int fail(int code, const std::string& msg);
int cuda_fail(cudaError_t e, const char* where);

#define FDL_CUDA_CHECK(expr)                                  \
  do {                                                        \
    cudaError_t _e = (expr);                                  \
    if (_e != cudaSuccess) return ::fdl::cuda_fail(_e, #expr); \
  } while (0)

#define FDL_LAUNCH_CHECK(name)                                   \
  do {                                                           \
    cudaError_t _e = cudaGetLastError();                         \
    if (_e != cudaSuccess) return ::fdl::cuda_fail(_e, name);    \
  } while (0)

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// ---------------------------------------------------------------------------
// small numeric helpers
// ---------------------------------------------------------------------------
struct cd {  // complex double
  double re, im;
};
__host__ __device__ inline cd cmul(cd a, cd b) { return {a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re}; }

// omega labels, bit-identical to the reference grid (spectra.py:55-66):
// omega_x = arange(W//2+1) / W with the even-W Nyquist column labelled -0.5;
// omega_y = numpy.fft.fftfreq(H) = k_signed * (1.0 / H)  (numpy multiplies by
// the reciprocal).
__host__ __device__ inline double omega_x_label(int kx, int Wp) {
  if ((Wp & 1) == 0 && kx == Wp / 2) return -0.5;
  return (double)kx / (double)Wp;
}
__host__ __device__ inline double omega_y_label(int ky, int Hp) {
  int half = (Hp - 1) / 2 + 1;
  int ks = ky < half ? ky : ky - Hp;
  return (double)ks * (1.0 / (double)Hp);
}

// Aperture table on the device (fdl_aperture with device pointers).
struct DevAperture {
  int rows, cols;
  const double* re;
  const double* im;  // nullptr for a real table
  double xi0_x, step_x, xi0_y, step_y;
  // fast path (real tables, construction K1 mode 2): "quad" table, entry (iy, ix)
  // = {(T[iy][ix], T[iy][ix+1]), (T[iy+1][ix], T[iy+1][ix+1])}, entry rows*cols = 0
  const double2* quad;
  double inv_step_x;
};

// Bilinear axis lookup of ApertureSpec._axis_lookup (lfmodel.py:72-79):
// pos = (q - xi0) / step; valid = 0 <= pos <= n-1; i0 = clip(floor(pos), 0, n-2);
// frac = clip(pos - i0, 0, 1).
__host__ __device__ inline bool axis_lookup(double q, double xi0, double step, int n, int& i0, double& fr) {
  double pos = (q - xi0) / step;
  bool ok = (pos >= 0.0) && (pos <= (double)(n - 1));
  double fl = floor(pos);
  // clip in double first: pos may be huge or NaN for out-of-range queries
  if (!(fl >= 0.0)) fl = 0.0;
  if (fl > (double)(n - 2)) fl = (double)(n - 2);
  i0 = (int)fl;
  fr = pos - (double)i0;
  if (!(fr >= 0.0)) fr = 0.0;
  if (fr > 1.0) fr = 1.0;
  return ok;
}

// psi_hat(qx, qy) by ApertureSpec.evaluate (lfmodel.py:81-99); 0 outside the table.
__device__ inline cd aperture_eval(const DevAperture& ap, double qx, double qy) {
  int ix, iy;
  double fx, fy;
  bool okx = axis_lookup(qx, ap.xi0_x, ap.step_x, ap.cols, ix, fx);
  bool oky = axis_lookup(qy, ap.xi0_y, ap.step_y, ap.rows, iy, fy);
  if (!(okx && oky)) return {0.0, 0.0};
  const size_t r0 = (size_t)iy * ap.cols, r1 = r0 + ap.cols;
  // lfmodel.py:89-94 evaluation order: ((t*(1-fy))*(1-fx)) + ... left to right
  const double gy = __dsub_rn(1.0, fy), gx = __dsub_rn(1.0, fx);
  cd out;
  out.re = __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(__dmul_rn(ap.re[r0 + ix], gy), gx),
                                         __dmul_rn(__dmul_rn(ap.re[r0 + ix + 1], gy), fx)),
                               __dmul_rn(__dmul_rn(ap.re[r1 + ix], fy), gx)),
                     __dmul_rn(__dmul_rn(ap.re[r1 + ix + 1], fy), fx));
  if (ap.im) {
    out.im = __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(__dmul_rn(ap.im[r0 + ix], gy), gx),
                                           __dmul_rn(__dmul_rn(ap.im[r0 + ix + 1], gy), fx)),
                                 __dmul_rn(__dmul_rn(ap.im[r1 + ix], fy), gx)),
                       __dmul_rn(__dmul_rn(ap.im[r1 + ix + 1], fy), fx));
  } else {
    out.im = 0.0;
  }
  return out;
}

// exp(+2 pi i P omega) with the symmetric cosine on a self-conjugate Nyquist
// line (construct.py:68-80), evaluated with the reference's own rounding:
// numpy forms the argument as fl(fl(2 pi P) omega) (`2j * np.pi * P * omega`)
// and takes libm cos/sin of it; the Nyquist value is cos(fl(pi P)).  The
// low-frequency bins are conditioned up to ~1e13 at small image sizes, so a
// 1-ulp change of A moves their solution by ~1e-3: keep A within an ulp of
// the reference (explicit _rn intrinsics, no FMA contraction).
__device__ inline cd axis_phase(double P, double omega, bool nyq) {
  if (nyq) return {cos(__dmul_rn(M_PI, P)), 0.0};
  const double arg = __dmul_rn(__dmul_rn(2.0 * M_PI, P), omega);
  double s, c;
  sincos(arg, &s, &c);
  return {c, s};
}

// complex product without FMA contraction (numpy's (ac - bd) + i(ad + bc))
__device__ inline cd cmul_rn(cd a, cd b) {
  return {__dsub_rn(__dmul_rn(a.re, b.re), __dmul_rn(a.im, b.im)),
          __dadd_rn(__dmul_rn(a.re, b.im), __dmul_rn(a.im, b.re))};
}

// Packed fp32 pairs (sm_100 FFMA2 / FADD2): (re, im) in one 64-bit register pair.
typedef unsigned long long u64;
__device__ __forceinline__ u64 as_u64(float2 v) { return *reinterpret_cast<const u64*>(&v); }
__device__ __forceinline__ float2 as_f2(u64 v) { return *reinterpret_cast<const float2*>(&v); }
__device__ __forceinline__ u64 add2(u64 a, u64 b) {
  u64 r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ u64 sub2(u64 a, u64 b) {
  u64 r;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
// acc += v * (w, w)
__device__ __forceinline__ void ffma2s(u64& acc, u64 v, float w) {
  u64 ww;
  asm("mov.b64 %0, {%1, %1};" : "=l"(ww) : "f"(w));
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc) : "l"(v), "l"(ww));
}

__device__ __forceinline__ u64 pack2(float a, float b) {
  u64 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ void ffma2(u64& acc, u64 a, u64 b) {
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc) : "l"(a), "l"(b));
}
// acc += w * z  (complex w, z): two FFMA2; the swapped / partially negated
// operands are free operand modifiers (.LO_HI, .NP) in SASS
__device__ __forceinline__ void cmac2(u64& acc, float wr, float wi, float2 z) {
  ffma2(acc, pack2(z.x, z.y), pack2(wr, wr));
  ffma2(acc, pack2(z.y, z.x), pack2(-wi, wi));
}

// asynchronous global -> shared copies (sm_80+ cp.async), zero-filled when !valid
__device__ __forceinline__ void cpa4(void* smem_dst, const void* gsrc, bool valid) {
  const unsigned dst = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(dst), "l"(gsrc), "r"(valid ? 4 : 0));
}
__device__ __forceinline__ void cpa8(void* smem_dst, const void* gsrc, bool valid) {
  const unsigned dst = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(dst), "l"(gsrc), "r"(valid ? 8 : 0));
}
__device__ __forceinline__ void cpa16(void* smem_dst, const void* gsrc, bool valid) {
  const unsigned dst = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(gsrc), "r"(valid ? 16 : 0));
}
// bring a line into L2 ahead of a later load (no registers held)
__device__ __forceinline__ void prefetch_l2(const void* p) { asm volatile("prefetch.global.L2 [%0];" ::"l"(p)); }
__device__ __forceinline__ void cpa_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cpa_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::); }
__device__ __forceinline__ void cpa_wait_1() { asm volatile("cp.async.wait_group 1;\n" ::); }

// kernel-launch timer (abi.cu: fdl_kernel_timer); phase 0 before, 1 after a launch
void ktimer_mark(int which, int phase, cudaStream_t st);

}  // namespace fdl
