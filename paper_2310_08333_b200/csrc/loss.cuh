// Loss value / derivatives / conjugate of problems.py:35-111, bit-compatible
// with the NumPy expressions the reference evaluates (shared by vec.cu and
// rowpass.cu).
#pragma once
#include <math.h>
#include "common.cuh"

namespace nys {

__device__ __forceinline__ double expit_d(double x) { return 1.0 / (1.0 + exp(-x)); }

// numpy npy_logaddexp(0, w)
__device__ __forceinline__ double logaddexp0(double w) {
  if (w == 0.0) return 0.6931471805599453;  // log(2)
  const double tmp = -w;
  if (tmp > 0.0) return log1p(exp(-tmp));
  if (tmp <= 0.0) return w + log1p(exp(tmp));
  return tmp;  // NaN
}

__device__ __forceinline__ double loss_val(int loss, double w) {
  if (loss == NYS_LOSS_SQUARE) return 0.5 * (w * w);
  if (loss == NYS_LOSS_LOGISTIC) return logaddexp0(w);
  return fabs(w) <= 1.0 ? w * w : 2.0 * fabs(w) - 1.0;
}
__device__ __forceinline__ double loss_d1(int loss, double w) {
  if (loss == NYS_LOSS_SQUARE) return w;
  if (loss == NYS_LOSS_LOGISTIC) return expit_d(w);
  return fabs(w) <= 1.0 ? 2.0 * w : (w > 0.0 ? 2.0 : (w < 0.0 ? -2.0 : 0.0));
}
__device__ __forceinline__ double loss_d2(int loss, double w) {
  if (loss == NYS_LOSS_SQUARE) return 1.0;
  if (loss == NYS_LOSS_LOGISTIC) return expit_d(w) * expit_d(-w);
  return fabs(w) <= 1.0 ? 2.0 : 0.0;
}
// conjugate; returns +inf outside the domain (problems.py:60, 65-73, 107-109)
__device__ __forceinline__ double loss_conj(int loss, double y) {
  if (loss == NYS_LOSS_SQUARE) return 0.5 * (y * y);
  if (loss == NYS_LOSS_LOGISTIC) {
    if (y == 0.0 || y == 1.0) return 0.0;
    if (!(y >= 0.0 && y <= 1.0)) return INFINITY;
    const double yc = fmin(fmax(y, 1e-12), 1.0 - 1e-12);
    return yc * log(yc) + (1.0 - yc) * log1p(-yc);
  }
  return fabs(y) <= 2.0 ? 0.25 * (y * y) : INFINITY;
}

}  // namespace nys
