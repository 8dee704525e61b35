// DTLZ1-7 objective evaluation of one individual (device).
//
// SPEC.md:520-528 (DTLZ2/3/5/7) + the standard DTLZ1/4/6.
// Inputs are FP32, arithmetic is FP64 with the oracle's operation order
// (oracle/manyobj_ref/problems.py), the result is rounded once to FP32, so
// GPU and CPU objectives agree to within one FP32 rounding.  The whole
// library is compiled with -fmad=false, so no mul+add is contracted.
#pragma once
#include <math.h>
#include <stdint.h>

namespace mo {

// One term of the g sum (distance variable t = v - (m-1)), FP64.
__device__ __forceinline__ double dtlz_g_term(int problem, float xv) {
  const double PI = 3.141592653589793;
  if (problem == 1 || problem == 3) {
    const double t = (double)xv - 0.5;
    return t * t - cos(20.0 * PI * t);
  }
  if (problem == 2 || problem == 4 || problem == 5) {
    const double t = (double)xv - 0.5;
    return t * t;
  }
  if (problem == 6) return pow((double)xv, 0.1);
  return (double)xv;  // DTLZ7
}

// g from the summed terms.
__device__ __forceinline__ double dtlz_g_finish(int problem, double s, int k) {
  if (problem == 1 || problem == 3) return 100.0 * ((double)k + s);
  if (problem == 7) return 1.0 + (9.0 / (double)k) * s;
  return s;
}

// Partial sum of lane l (of G_LANES) of the g terms: terms l, l + 8, ... left to right.
constexpr int G_LANES = 8;
__device__ __forceinline__ double dtlz_g_partial(int problem, const float* __restrict__ x, int d, int m, int l) {
  double s = 0.0;
  for (int v = m - 1 + l; v < d; v += G_LANES) s = s + dtlz_g_term(problem, x[v]);
  return s;
}

// The whole g sum in the pinned order (8 strided partials, then ((p0+p4)+(p2+p6)) + ((p1+p5)+(p3+p7)),
// = the xor butterfly of an 8-lane group), sequentially.
__device__ inline double dtlz_g(int problem, const float* __restrict__ x, int d, int m) {
  double p[G_LANES];
  for (int l = 0; l < G_LANES; ++l) p[l] = dtlz_g_partial(problem, x, d, m, l);
  const double a0 = p[0] + p[4], a1 = p[1] + p[5], a2 = p[2] + p[6], a3 = p[3] + p[7];
  return dtlz_g_finish(problem, (a0 + a2) + (a1 + a3), d - m + 1);
}

// x: FP32 row (d entries, stride 1); f: FP32 output (m entries).  Returns
// true iff every x lies in [0,1] (DomainError otherwise).
__device__ inline bool dtlz_eval_row(int problem, const float* __restrict__ x, int d, int m,
                                     float* __restrict__ f) {
  const double PI = 3.141592653589793;
  bool ok = true;
  for (int v = 0; v < d; ++v) {
    float xv = x[v];
    ok = ok && (xv >= 0.0f) && (xv <= 1.0f);
  }
  // g over the distance variables x[m-1 .. d-1] (pinned grouped order, dtlz_g)
  const double g = dtlz_g(problem, x, d, m);

  if (problem == 1) {
    for (int j = 0; j < m; ++j) {
      double val = 0.5 * (1.0 + g);
      for (int i = 0; i < m - 1 - j; ++i) val = val * (double)x[i];
      if (j > 0) val = val * (1.0 - (double)x[m - 1 - j]);
      f[j] = (float)val;
    }
  } else if (problem == 7) {
    double h = 0.0;
    for (int j = 0; j < m - 1; ++j) {
      double fj = (double)x[j];
      f[j] = x[j];
      h = h + fj / (1.0 + g) * (1.0 + sin(3.0 * PI * fj));
    }
    f[m - 1] = (float)((1.0 + g) * ((double)m - h));
  } else {
    // spherical family: theta_i (i < m-1)
    const double hp = PI / 2.0;
    for (int j = 0; j < m; ++j) {
      double val = 1.0 + g;
      for (int i = 0; i < m - 1 - j; ++i) {
        double th;
        double xi = (double)x[i];
        if (problem == 4) xi = pow(xi, 100.0);
        if ((problem == 5 || problem == 6) && i > 0)
          th = PI / (4.0 * (1.0 + g)) * (1.0 + 2.0 * g * xi);
        else
          th = xi * hp;
        val = val * cos(th);
      }
      if (j > 0) {
        int i = m - 1 - j;
        double th;
        double xi = (double)x[i];
        if (problem == 4) xi = pow(xi, 100.0);
        if ((problem == 5 || problem == 6) && i > 0)
          th = PI / (4.0 * (1.0 + g)) * (1.0 + 2.0 * g * xi);
        else
          th = xi * hp;
        val = val * sin(th);
      }
      f[j] = (float)val;
    }
  }
  return ok;
}

// Objective j of one individual given its g -- the same operation order as
// dtlz_eval_row (so the two agree bit for bit); used by the fused variation
// kernel, which sums g with 8 lanes per child and then evaluates one (child,
// objective) per thread.
__device__ inline float dtlz_eval_obj(int problem, const float* __restrict__ x, int m, int j, double g) {
  const double PI = 3.141592653589793;
  if (problem == 1) {
    double val = 0.5 * (1.0 + g);
    for (int i = 0; i < m - 1 - j; ++i) val = val * (double)x[i];
    if (j > 0) val = val * (1.0 - (double)x[m - 1 - j]);
    return (float)val;
  }
  if (problem == 7) {
    if (j < m - 1) return x[j];
    double h = 0.0;
    for (int q = 0; q < m - 1; ++q) {
      double fj = (double)x[q];
      h = h + fj / (1.0 + g) * (1.0 + sin(3.0 * PI * fj));
    }
    return (float)((1.0 + g) * ((double)m - h));
  }
  const double hp = PI / 2.0;
  double val = 1.0 + g;
  for (int i = 0; i <= m - 1 - j && i < m - 1; ++i) {
    double xi = (double)x[i];
    if (problem == 4) xi = pow(xi, 100.0);
    const double th = ((problem == 5 || problem == 6) && i > 0) ? PI / (4.0 * (1.0 + g)) * (1.0 + 2.0 * g * xi)
                                                                 : xi * hp;
    if (i < m - 1 - j)
      val = val * cos(th);
    else if (j > 0)
      val = val * sin(th);
  }
  return (float)val;
}

// Factor pair of variable t < m-1 for the prefix form below: cf multiplies the running prefix,
// sf closes objective m-1-t (DTLZ1: x_t and 1 - x_t; DTLZ2-6: cos and sin of the same angle).
__device__ inline void dtlz_factors(int problem, const float* __restrict__ x, int t, double g, double& cf,
                                    double& sf) {
  const double PI = 3.141592653589793;
  if (problem == 1) {
    cf = (double)x[t];
    sf = 1.0 - (double)x[t];
    return;
  }
  double xi = (double)x[t];
  if (problem == 4) xi = pow(xi, 100.0);
  const double th = ((problem == 5 || problem == 6) && t > 0) ? PI / (4.0 * (1.0 + g)) * (1.0 + 2.0 * g * xi)
                                                               : xi * (PI / 2.0);
  cf = cos(th);
  sf = sin(th);
}

// All m objectives of one row in O(m) (wide m): every product of dtlz_eval_obj is a left fold over the
// same leading factors, so after t factors the running prefix is objective (m-1-t)'s partial product and
// out(j, f_j) receives bit-identical values (same factors, same order, same sin / cos calls).
template <class Out>
__device__ inline void dtlz_eval_prefix(int problem, const float* __restrict__ x, int m, double g, Out out) {
  const double PI = 3.141592653589793;
  if (problem == 7) {
    for (int j = 0; j < m; ++j) out(j, dtlz_eval_obj(problem, x, m, j, g));
    return;
  }
  if (problem == 1) {
    double P = 0.5 * (1.0 + g);
    for (int t = 0; t < m - 1; ++t) {
      out(m - 1 - t, (float)(P * (1.0 - (double)x[t])));
      P = P * (double)x[t];
    }
    out(0, (float)P);
    return;
  }
  const double hp = PI / 2.0;
  double P = 1.0 + g;
  for (int t = 0; t < m - 1; ++t) {
    double xi = (double)x[t];
    if (problem == 4) xi = pow(xi, 100.0);
    const double th = ((problem == 5 || problem == 6) && t > 0) ? PI / (4.0 * (1.0 + g)) * (1.0 + 2.0 * g * xi)
                                                                 : xi * hp;
    out(m - 1 - t, (float)(P * sin(th)));
    P = P * cos(th);
  }
  out(0, (float)P);
}

}  // namespace mo
