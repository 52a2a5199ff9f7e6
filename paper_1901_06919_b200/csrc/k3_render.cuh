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
  int uniform_ap;          // >= 0: every view of the batch uses this real table (fast path)
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
};

int render_launch(const RenderParams& p, cudaStream_t st);

}  // namespace fdl
