// SBX spread factor and Deb's bounded polynomial mutation in FP64 (oracle order,
// oracle/manyobj_ref/variation.py:37-68), shared by the fused engine kernel (k_vary.cu) and the
// op-level sbx_pair / polynomial_mutation entry points (k_ops.cu).
// Reference ops: variation.sbx_pair, polynomial_mutation.
#pragma once

namespace mo {

__device__ __forceinline__ double sbx_beta(double u, double eta) {
  double e = 1.0 / (eta + 1.0);
  return u <= 0.5 ? pow(2.0 * u, e) : pow(1.0 / (2.0 * (1.0 - u)), e);
}

// x + delta(u) * span on [lo, hi]; delta(0.5) = 0; with lo = 0, hi = 1 every operation is the
// engine's (x - 0) / 1 = x exactly.
__device__ __forceinline__ double pm_apply(double x, double u, double eta, double lo = 0.0, double hi = 1.0) {
  const double span = hi - lo;
  double d1 = (x - lo) / span, d2 = (hi - x) / span;
  double mp = 1.0 / (eta + 1.0);
  double dq;
  if (u < 0.5) {
    double v = 2.0 * u + (1.0 - 2.0 * u) * pow(1.0 - d1, eta + 1.0);
    dq = pow(v, mp) - 1.0;
  } else {
    double v = 2.0 * (1.0 - u) + 2.0 * (u - 0.5) * pow(1.0 - d2, eta + 1.0);
    dq = 1.0 - pow(v, mp);
  }
  return x + dq * span;
}

__device__ __forceinline__ double clamp_to(double v, double lo, double hi) { return v < lo ? lo : (v > hi ? hi : v); }
__device__ __forceinline__ double clamp01(double v) { return clamp_to(v, 0.0, 1.0); }

}  // namespace mo
