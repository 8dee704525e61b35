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

// x: FP32 row (d entries, stride 1); f: FP32 output (m entries).  Returns
// true iff every x lies in [0,1] (DomainError otherwise).
__device__ inline bool dtlz_eval_row(int problem, const float* __restrict__ x, int d, int m,
                                     float* __restrict__ f) {
  const double PI = 3.141592653589793;
  const int k = d - m + 1;
  bool ok = true;
  for (int v = 0; v < d; ++v) {
    float xv = x[v];
    ok = ok && (xv >= 0.0f) && (xv <= 1.0f);
  }
  // g over the distance variables x[m-1 .. d-1], summed left to right
  double g = 0.0;
  if (problem == 1 || problem == 3) {
    const double c20 = 20.0 * PI;
    double s = 0.0;
    for (int v = m - 1; v < d; ++v) {
      double t = (double)x[v] - 0.5;
      s = s + (t * t - cos(c20 * t));
    }
    g = 100.0 * ((double)k + s);
  } else if (problem == 2 || problem == 4 || problem == 5) {
    double s = 0.0;
    for (int v = m - 1; v < d; ++v) {
      double t = (double)x[v] - 0.5;
      s = s + t * t;
    }
    g = s;
  } else if (problem == 6) {
    double s = 0.0;
    for (int v = m - 1; v < d; ++v) s = s + pow((double)x[v], 0.1);
    g = s;
  } else {  // DTLZ7
    double s = 0.0;
    for (int v = m - 1; v < d; ++v) s = s + (double)x[v];
    g = 1.0 + (9.0 / (double)k) * s;
  }

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

// Objective j of one individual -- the same operation order as dtlz_eval_row
// (so the two agree bit for bit); used by the fused variation kernel, which
// evaluates one (child, objective) per thread.
__device__ inline float dtlz_eval_obj(int problem, const float* __restrict__ x, int d, int m, int j) {
  const double PI = 3.141592653589793;
  const int k = d - m + 1;
  double g = 0.0;
  if (problem == 1 || problem == 3) {
    const double c20 = 20.0 * PI;
    double s = 0.0;
    for (int v = m - 1; v < d; ++v) {
      double t = (double)x[v] - 0.5;
      s = s + (t * t - cos(c20 * t));
    }
    g = 100.0 * ((double)k + s);
  } else if (problem == 2 || problem == 4 || problem == 5) {
    double s = 0.0;
    for (int v = m - 1; v < d; ++v) {
      double t = (double)x[v] - 0.5;
      s = s + t * t;
    }
    g = s;
  } else if (problem == 6) {
    double s = 0.0;
    for (int v = m - 1; v < d; ++v) s = s + pow((double)x[v], 0.1);
    g = s;
  } else {
    double s = 0.0;
    for (int v = m - 1; v < d; ++v) s = s + (double)x[v];
    g = 1.0 + (9.0 / (double)k) * s;
  }
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

}  // namespace mo
