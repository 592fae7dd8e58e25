// NURBS building blocks on the device, shared by K4 (observers) and K6 (the
// operator assembly): find_span and the first-derivative Cox-de Boor table
// ("The NURBS Book" A2.1/A2.3, as KnotVector::find_span / basis_ders,
// proj/src/splines.cpp:27-109) and the 3x3 determinant (Mat3::det). Include
// only from translation units compiled with -fmad=false (_build.NO_FMAD): every
// product and sum is then rounded separately in the reference's order.
#pragma once

#include "k4_eval.cuh"

namespace tgb {

__device__ inline bool find_span(const double* U, int p, int n, double u, int& span) {
  const double lo = U[p], hi = U[n];
  const double tol = 1e-12 * (hi - lo);
  if (u < lo - tol || u > hi + tol) return false;
  u = fmin(fmax(u, lo), hi);
  if (u >= hi) {
    span = n - 1;
    return true;
  }
  if (u <= lo) {
    span = p;
    return true;
  }
  int a = p, b = n, mid = (a + b) / 2;
  while (u < U[mid] || u >= U[mid + 1]) {
    if (u < U[mid]) b = mid;
    else a = mid;
    mid = (a + b) / 2;
  }
  span = mid;
  return true;
}

// values out[0..p] and first derivatives out[p+1..2p+1]
__device__ inline void basis_ders1(const double* U, int p, double u, int span, double* out) {
  constexpr int M = kNurbsMaxP + 1;
  const int w = p + 1;
  double tri[M * M], lft[M], rgt[M], coef[2 * M];
  for (int e = 0; e < 2 * w; ++e) out[e] = 0.0;
  tri[0] = 1.0;
  for (int j = 1; j <= p; ++j) {
    lft[j] = u - U[span + 1 - j];
    rgt[j] = U[span + j] - u;
    double carry = 0.0;
    for (int r = 0; r < j; ++r) {
      tri[j * w + r] = rgt[r + 1] + lft[j - r];
      const double q = tri[r * w + j - 1] / tri[j * w + r];
      tri[r * w + j] = carry + rgt[r + 1] * q;
      carry = lft[j - r] * q;
    }
    tri[j * w + j] = carry;
  }
  for (int j = 0; j <= p; ++j) out[j] = tri[j * w + p];
  if (p == 0) return;
  for (int r = 0; r <= p; ++r) {
    int cur = 0, nxt = 1;
    coef[0] = 1.0;
    const int k = 1;
    double d = 0.0;
    const int rk = r - k, pk = p - k;
    if (r >= k) {
      coef[nxt * w] = coef[cur * w] / tri[(pk + 1) * w + rk];
      d = coef[nxt * w] * tri[rk * w + pk];
    }
    const int j1 = rk >= -1 ? 1 : -rk;
    const int j2 = (r - 1 <= pk) ? k - 1 : p - r;
    for (int j = j1; j <= j2; ++j) {
      coef[nxt * w + j] = (coef[cur * w + j] - coef[cur * w + j - 1]) / tri[(pk + 1) * w + rk + j];
      d += coef[nxt * w + j] * tri[(rk + j) * w + pk];
    }
    if (r <= pk) {
      coef[nxt * w + k] = -coef[cur * w + k - 1] / tri[(pk + 1) * w + r];
      d += coef[nxt * w + k] * tri[r * w + pk];
    }
    out[w + r] = d;
  }
  const double f = p;
  for (int j = 0; j <= p; ++j) out[w + j] *= f;
}

__device__ inline double det3(const double* a) {
  return a[0] * (a[4] * a[8] - a[5] * a[7]) - a[1] * (a[3] * a[8] - a[5] * a[6]) +
         a[2] * (a[3] * a[7] - a[4] * a[6]);
}

}  // namespace tgb
