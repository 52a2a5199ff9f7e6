#pragma once
#include "common.cuh"

namespace fdl {

// one axis factor of one (view, layer): phase and bilinear lookup (idx < 0: out of range)
struct __align__(16) AxisFactor {
  float re, im, frac;
  int idx;
};

// Aperture table for the render hot loop: "quad" layout, entry (iy, ix) holds
// (T[iy][ix], T[iy][ix+1], T[iy+1][ix], T[iy+1][ix+1]) so one 16-byte load
// feeds a bilinear lookup; entry `zero` (= rows * cols) is all zeros and is
// where out-of-range lookups point (lfmodel.py:118-121 sets them to 0).
struct RenderTable {
  int rows, cols, zero;
  const float4* re;
  const float4* im;  // nullptr for a real table
};

struct RenderParams {
  int uniform_ap;         // >= 0: every view of the batch uses this real table (fast path)
  int n, C, Hp, Wp, Whp, V;
  const double* pu;        // (V, n)
  const double* pv;        // (V, n)
  const double* t;         // (V, n)
  const int* view_ap;      // (V) or nullptr
  const DevAperture* aps;  // float64 tables (index math)
  const RenderTable* tables;  // float32 copies (hot loop)
  const float2* layers;    // (n, C, Hp, Whp)
  float2* out;             // (V, C, Hp, Whp)
  long long* oob;          // (V) or nullptr
  AxisFactor* px;          // (V, n, Whp)
  AxisFactor* py;          // (V, n, Hp)
  // real-table fast path (every aperture of the batch real; pinhole views allowed):
  // difference-form quads (a, b, c, d) = (T00, T01-T00, T10-T00, T11-T10-T01+T00)
  // so psi = (a + fy c) + fx (b + fy d); tables concatenated, then the ONE entry
  // (1,0,0,0) that non-aperture views point at and the ZERO entry that
  // out-of-range lookups point at.  Factor idx fields are absolute entry indices
  // (x: table base + column, y: row * cols; either axis out of range: dq_zero).
  int fast_ap;
  const float4* dquad;
  const int* ap_qbase;     // (n_apertures) first entry of each table in dquad
  int dq_one, dq_zero;
  // pinhole Horner path (every view's shifts affine in the layer index:
  // pu[v, k] = pu[v, 0] + k * alpha_v, pv likewise): per-bin ratio of
  // consecutive layer phases z = exp(2 pi i (alpha wx + beta wy)), fp64 tables
  int horner;
  const double* h_alpha;   // (V)
  const double* h_beta;    // (V)
  double2* zx;             // (V, Whp)
  double2* zy;             // (V, Hp)
};

int render_launch(const RenderParams& p, cudaStream_t st);
// real-table aperture batches: the TMA-staged tile (k3_render_ap.cu)
int render_ap_launch(const RenderParams& p, cudaStream_t st);
// the 16-byte per-(view, layer) axis factor pre-pass (k3_render.cu)
int render_factors_kernel_launch(const RenderParams& p, cudaStream_t st);

}  // namespace fdl
