#pragma once
#include "common.cuh"

namespace fdl {

// one axis factor of one (view, layer): phase and bilinear lookup (idx < 0: out of range)
struct __align__(16) AxisFactor {
  float re, im, frac;
  int idx;
};

struct RenderTable {
  int rows, cols;
  const float* re;
  const float* im;  // nullptr for a real table
};

struct RenderParams {
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
