// Host-side NF4 level table, decision thresholds and the kernels' bucket
// table.  Independent of the CPU oracle: Phi^-1 here is Acklam's rational
// approximation refined by Halley steps on std::erfc (the oracle uses
// scipy.special.ndtri); both must round to the same fp32 bits, which the
// tests check.
//
// PAPER.md:201 names NF4 (4-bit NormalFloat, cited from QLoRA); the explicit
// quantile recipe is SPEC.md:55-63.
#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>
#include <mutex>

#include "nqkv_internal.h"

namespace nqkv {
namespace {

// Acklam (2003) initial guess, |rel err| < 1.2e-9, then two Halley steps.
double inv_normal_cdf(double p) {
  static const double a[] = {-3.969683028665376e+01, 2.209460984245205e+02,
                             -2.759285104469687e+02, 1.383577518672690e+02,
                             -3.066479806614716e+01, 2.506628277459239e+00};
  static const double b[] = {-5.447609879822406e+01, 1.615858368580409e+02,
                             -1.556989798598866e+02, 6.680131188771972e+01,
                             -1.328068155288572e+01};
  static const double c[] = {-7.784894002430293e-03, -3.223964580411365e-01,
                             -2.400758277161838e+00, -2.549732539343734e+00,
                             4.374664141464968e+00, 2.938163982698783e+00};
  static const double d[] = {7.784695709041462e-03, 3.224671290700398e-01,
                             2.445134137142996e+00, 3.754408661907416e+00};
  if (p == 0.5) return 0.0;
  const double plow = 0.02425, phigh = 1 - plow;
  double x;
  if (p < plow) {
    double q = std::sqrt(-2 * std::log(p));
    x = (((((c[0] * q + c[1]) * q + c[2]) * q + c[3]) * q + c[4]) * q + c[5]) /
        ((((d[0] * q + d[1]) * q + d[2]) * q + d[3]) * q + 1);
  } else if (p <= phigh) {
    double q = p - 0.5, r = q * q;
    x = (((((a[0] * r + a[1]) * r + a[2]) * r + a[3]) * r + a[4]) * r + a[5]) * q /
        (((((b[0] * r + b[1]) * r + b[2]) * r + b[3]) * r + b[4]) * r + 1);
  } else {
    double q = std::sqrt(-2 * std::log(1 - p));
    x = -(((((c[0] * q + c[1]) * q + c[2]) * q + c[3]) * q + c[4]) * q + c[5]) /
        ((((d[0] * q + d[1]) * q + d[2]) * q + d[3]) * q + 1);
  }
  const double sqrt2pi = 2.50662827463100050242;
  for (int it = 0; it < 2; ++it) {
    double e = 0.5 * std::erfc(-x / std::sqrt(2.0)) - p;   // Phi(x) - p
    double u = e * sqrt2pi * std::exp(0.5 * x * x);
    x = x - u / (1 + 0.5 * x * u);
  }
  return x;
}

float round_down_f32(double v) {
  float f = static_cast<float>(v);
  if (static_cast<double>(f) > v) f = std::nextafter(f, -std::numeric_limits<float>::infinity());
  return f;
}

struct Tables {
  float levels[16];
  float thresholds[15];
  BucketEntry buckets[kNumBuckets];
  int status = -7;
};

Tables g_tables;
std::once_flag g_once;

void build() {
  Tables& t = g_tables;
  // delta = 1 - 1/2 (1/(2*16) + 1/(2*15))
  const double delta = 1.0 - 0.5 * (1.0 / 32.0 + 1.0 / 30.0);
  double v[16];
  int k = 0;
  for (int i = 0; i < 7; ++i) v[k++] = -inv_normal_cdf(delta + i * (0.5 - delta) / 7.0);
  v[k++] = 0.0;
  for (int i = 1; i <= 8; ++i) v[k++] = inv_normal_cdf(0.5 + i * (delta - 0.5) / 8.0);
  const double norm = inv_normal_cdf(delta);
  for (int i = 0; i < 16; ++i) v[i] /= norm;
  // ascending order: negatives were produced from -1 upward already
  for (int i = 0; i < 16; ++i) t.levels[i] = static_cast<float>(v[i]);
  bool ok = t.levels[0] == -1.0f && t.levels[15] == 1.0f && t.levels[7] == 0.0f;
  for (int i = 0; i < 15; ++i) ok = ok && t.levels[i] < t.levels[i + 1];
  // thresholds: exact double midpoint of adjacent fp32 levels, rounded down
  for (int i = 0; i < 15; ++i) {
    double mid = (static_cast<double>(t.levels[i]) + static_cast<double>(t.levels[i + 1])) * 0.5;
    t.thresholds[i] = round_down_f32(mid);
  }
  // Kernel bucket table: idx = RN(16 n + 16) in [0, 32]; bucket idx covers
  // [(idx-16.5)/16, (idx-15.5)/16].  Each bucket must hold at most one
  // threshold and no threshold may sit on a bucket edge; then
  // code(n) = lo[idx] + (n > thr[idx]) exactly.
  for (int idx = 0; idx < kNumBuckets; ++idx) {
    const double a = (idx - 16.5) / 16.0, b = (idx - 15.5) / 16.0;
    int lo = 0, inside = 0;
    float thr = std::numeric_limits<float>::infinity();
    for (int i = 0; i < 15; ++i) {
      const double ti = t.thresholds[i];
      if (ti < a) ++lo;
      if (ti >= a && ti <= b) { ++inside; thr = t.thresholds[i]; }
      if (ti == a || ti == b) ok = false;
    }
    if (inside > 1) ok = false;
    t.buckets[idx].thr = thr;
    t.buckets[idx].lo = static_cast<uint32_t>(lo);
  }
  t.status = ok ? 0 : -7;
}

}  // namespace

const float* level_table() { std::call_once(g_once, build); return g_tables.levels; }
const float* threshold_table() { std::call_once(g_once, build); return g_tables.thresholds; }
const BucketEntry* bucket_table() { std::call_once(g_once, build); return g_tables.buckets; }
int tables_status() { std::call_once(g_once, build); return g_tables.status; }

}  // namespace nqkv
