// Device-side data structures and bit-exact arithmetic helpers for b200md.
//
// Bit-exactness contract: the partner search and the site-site cutoff test
// must reproduce the reference's double arithmetic bit for bit
// (include/tmd/potentials.hpp:176-181 minimum_image, include/tmd/geom.hpp:29-33
// dot/norm2, geom.hpp:62-66 rotate).  The reference binary has no FMA, so these
// paths use explicit __dmul_rn/__dadd_rn/__dsub_rn (never contracted) in the
// reference's evaluation order.  Force arithmetic is free to contract (the
// parity bar there is 1e-10 relative).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace b2md {

constexpr int kMaxSpecies = 8;
constexpr int kMaxSitesDev = 16;  // == B2MD_MAX_SITES
constexpr int kMaxLjTerms = 1024;
constexpr int kMaxQqTerms = 1024;
constexpr int kNumRowScalars = 7;  // u_lj, u_elec_real, u_rf, s1, s2, virial, com_pairs
constexpr int kNumSums = 8;        // the 7 above + u_recip

struct DevLjTerm {
  int a, b;
  double c12, c6;
};
struct DevQTerm {
  int a, b;
  double qq;
};
struct DevPairInfo {
  int lj_begin, lj_count, qq_begin, qq_count;
  double rmax2;
};
struct DevSpecies {
  int n_sites;
  int rotational_dof;
  int centred;  // single site at the COM: offsets are exactly zero (potentials.cpp:110-111)
  int pad_;
  double inv_mass_half_dt;  // unused placeholder (kept for alignment)
  double total_mass;
  double inertia[3];
  double body[kMaxSitesDev][3];
};
struct DevTables {
  int ns;
  int pad_;
  DevSpecies species[kMaxSpecies];
  DevPairInfo pair[kMaxSpecies * kMaxSpecies];
  DevLjTerm lj[kMaxLjTerms];
  DevQTerm qq[kMaxQqTerms];
};

struct DevKVec {
  double kx, ky, kz, coeff;
  int nx, ny, nz, pad_;
};

// Minimum-image thresholds on the high 32 bits of |d| (see min_image below).
struct MinImage {
  double L;
  double negL;
  int hi_lo;   // hi32(L/2)
  int hi_hi;   // hi_lo + 1
  int hi_max;  // hi32(1.5 L) - 1
  int pad_;
};

// ---------------------------------------------------------------- arithmetic
__device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }

// (x*x + y*y) + z*z without contraction (geom.hpp:29,33)
__device__ __forceinline__ double norm2_exact(double x, double y, double z) {
  return add(add(mul(x, x), mul(y, y)), mul(z, z));
}

// d - L*nearbyint(d/L) (potentials.hpp:177), exactly.
// Fast path: with |d| < L/2 (strictly, by a 2^-20 relative margin) the
// quotient rounds to 0; with L/2 < |d| < 1.5L (same margin) it rounds to +-1
// and the result is d -+ L, a single correctly rounded add — the same bits as
// the reference's d - L*1.0.  Anything within the margins (probability
// ~1e-6 per axis) or beyond 1.5L, and NaN/Inf, takes the exact IEEE
// divide + round-half-even path.  The compares run on the integer pipe.
static __device__ __noinline__ double min_image_exact_slow(double d, double L) {
  const double n = rint(__ddiv_rn(d, L));
  return sub(d, mul(L, n));
}

__device__ __forceinline__ double min_image(double d, const MinImage& m) {
  const int hi = __double2hiint(d);
  const int ahi = hi & 0x7fffffff;
  const bool amb = (ahi >= m.hi_lo && ahi <= m.hi_hi) || ahi >= m.hi_max;
  if (__builtin_expect(amb, 0)) return min_image_exact_slow(d, m.L);
  const double s = (ahi > m.hi_hi) ? (hi < 0 ? m.L : m.negL) : 0.0;
  return add(d, s);
}

// rotate(q, v) = v + 2w t + 2 u x t, t = u x v (geom.hpp:62-66), no FMA
struct D3 {
  double x, y, z;
};
__device__ __forceinline__ D3 cross_exact(D3 a, D3 b) {
  return {sub(mul(a.y, b.z), mul(a.z, b.y)), sub(mul(a.z, b.x), mul(a.x, b.z)),
          sub(mul(a.x, b.y), mul(a.y, b.x))};
}
__device__ __forceinline__ D3 rotate_exact(double qw, double qx, double qy, double qz, D3 v) {
  const D3 u{qx, qy, qz};
  const D3 t = cross_exact(u, v);
  const double w2 = mul(2.0, qw);
  const D3 c = cross_exact(u, t);
  return {add(add(v.x, mul(t.x, w2)), mul(c.x, 2.0)), add(add(v.y, mul(t.y, w2)), mul(c.y, 2.0)),
          add(add(v.z, mul(t.z, w2)), mul(c.z, 2.0))};
}
// rotate_inv (geom.hpp:69-73): conjugate quaternion
__device__ __forceinline__ D3 rotate_inv_exact(double qw, double qx, double qy, double qz, D3 v) {
  return rotate_exact(qw, -qx, -qy, -qz, v);
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

}  // namespace b2md
