// Radial distribution histograms: tmd::RdfHistogram::accumulate
// (src/structure.cpp:38-76) on the device.
//
// Every LJ / dummy site of every molecule is a sampling site; the reference
// counts, for every intermolecular site pair (a in molecule mi < mj owning b)
// with d2 = norm2(minimum_image(x_a - x_b)) < r_max^2, bin = int(sqrt(d2) /
// bin_width) (< bins) of the unordered site-type pair.  Counts are integers,
// so the device reproduces them exactly: lab-frame site positions pos +
// rotate(q, body) with the reference's operation order, the exact minimum
// image, IEEE sqrt and division, truncation.  Per-CTA uint32 histograms in
// shared memory are merged into the uint64 totals with integer atomics (exact
// and order-independent).
#pragma once

#include "kernels.cuh"

namespace b2md {

constexpr int kRdfSharedCounters = 12 * 1024;  // uint32 counters that fit 48 KB

struct RdfArgs {
  SysDev s;
  const double *px, *py, *pz;              // external-order state
  const double *qw, *qx, *qy, *qz;
  const int* site_mol;                     // S: molecule of eligible site q
  const int* site_k;                       // S: site index within its species
  const int* site_type;                    // S: RDF site type
  int S;                                   // eligible sites per replica
  int n_types, bins, n_pairs;
  double rmax2, bin_width;
  double inv_bw;                           // RN(1 / bin_width): fast-path bin only
  double4* sites;                          // R * S: lab position (w: type bits)
  uint4* fix;                              // R * S: (round(frac(x/L) 2^32), .., .., type)
  double L;
  // fp32 certified fast path (k_rdf_pairs): L / 2^32, squared-radius and bin margins
  float scale, rmax2_lo, rmax2_hi, inv_bw_f, bin_abs;
  unsigned long long* counts;              // R * n_pairs * bins
};

// structure.cpp:45-58: site_pos = pos[m] + rotate(orient[m], body_pos)
static __global__ void k_rdf_stage(RdfArgs a) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= a.S * a.s.R) return;
  const int r = e / a.S, q = e - r * a.S;
  const int m = a.site_mol[q];
  const size_t g = size_t(r) * a.s.n + m;
  const DevSpecies& sp = a.s.tab->species[a.s.species_of[m]];
  const int k = a.site_k[q];
  const D3 o = rotate_exact(a.qw[g], a.qx[g], a.qy[g], a.qz[g], {sp.body[k][0], sp.body[k][1], sp.body[k][2]});
  const double x = add(a.px[g], o.x), y = add(a.py[g], o.y), z = add(a.pz[g], o.z);
  a.sites[e] = make_double4(x, y, z, __hiloint2double(0, a.site_type[q]));
  // fixed point on the periodic circle: the wrapping int32 difference of two
  // coordinates is their minimum image (in units of L / 2^32, error <= 1)
  auto fx = [&](double v) {
    double f = v / a.L;
    f -= floor(f);
    return uint32_t(static_cast<unsigned long long>(__double2ll_rn(f * 4294967296.0)));
  };
  a.fix[e] = make_uint4(fx(x), fx(y), fx(z), uint32_t(a.site_type[q]));
}

// bin = (int)(sqrt(d2) / bin_width) exactly as the reference rounds it
// (structure.cpp:67).  d2 * rsqrt(d2) * RN(1/w) is within a few ulps of the
// reference's RN(RN(sqrt(d2)) / w); whenever it lies further than 1e-12 t
// from an integer both truncate to the same bin.  The rest (and d2 = 0) take
// the reference's IEEE sqrt and division.
__device__ __forceinline__ int rdf_bin(double d2, double bin_width, double inv_bw) {
  if (d2 > 0.0) {
    const double t = d2 * rsqrt(d2) * inv_bw;
    const double f = floor(t);
    const double m = 1e-12 * t;
    if (t - f > m && f + 1.0 - t > m) return int(f);
  }
  return int(__ddiv_rn(__dsqrt_rn(d2), bin_width));
}

// The reference's decision for one site pair (structure.cpp:62-67), exactly;
// returns the bin or -1 (outside r_max or beyond the last bin).
static __device__ __noinline__ int rdf_exact(double4 pa, double4 pb, const RdfArgs& a) {
  const MinImage mi = a.s.mi;
  const double dx = min_image(sub(pa.x, pb.x), mi);
  const double dy = min_image(sub(pa.y, pb.y), mi);
  const double dz = min_image(sub(pa.z, pb.z), mi);
  const double d2 = norm2_exact(dx, dy, dz);
  if (d2 >= a.rmax2) return -1;
  const int bin = rdf_bin(d2, a.bin_width, a.inv_bw);
  return bin < a.bins ? bin : -1;
}

// Tile of T x T sites (A block y, B block x), y <= x: thread t owns site
// b = x T + t and visits the tile's a sites from shared memory; pairs with
// mol_a < mol_b are the reference's (mi < mj) pairs.
// Certified fp32 fast path: the fixed-point minimum image d (error <= sqrt(3)
// units of L/2^32) in fp32 gives d2 within 5.4e-7 relative (9 roundings of
// 2^-24) + the quantisation, and t = sqrt(d2)/w within 4.5e-7 relative; the
// margins below are 2e-6 on d2 and 1e-6 on t (+ 4 units of quantisation).
// Only pairs whose r_max test or bin is not settled by them replay the
// reference's fp64 arithmetic (rdf_exact).
// SHARED: a per-CTA uint32 histogram merged with integer atomics; else global
// uint64 atomics.
constexpr int kRdfMaxTypes = 16;  // pair-offset table; more types: computed inline

template <int T, bool SHARED>
__global__ void __launch_bounds__(T) k_rdf_pairs(RdfArgs a) {
  extern __shared__ unsigned rdf_hist[];
  __shared__ uint4 fa_s[T];
  __shared__ int ma_s[T];
  __shared__ int pair_off[kRdfMaxTypes * kRdfMaxTypes];  // [ta][tb] -> pair(min, max) * bins
  const int bx = blockIdx.x, by = blockIdx.y, r = blockIdx.z;
  if (by > bx) return;
  const int tid = threadIdx.x;
  const int nc = a.n_pairs * a.bins;
  unsigned long long* gcounts = a.counts + size_t(r) * nc;
  if (SHARED)
    for (int k = tid; k < nc; k += T) rdf_hist[k] = 0u;
  const double4* sites = a.sites + size_t(r) * a.S;
  const uint4* fix = a.fix + size_t(r) * a.S;
  const int a0 = by * T;
  const int ia = a0 + tid;
  fa_s[tid] = ia < a.S ? fix[ia] : make_uint4(0u, 0u, 0u, 0u);
  ma_s[tid] = ia < a.S ? a.site_mol[ia] : INT_MAX;
  const bool table = a.n_types <= kRdfMaxTypes;
  if (table)
    for (int k = tid; k < a.n_types * a.n_types; k += T) {
      const int x = k / a.n_types, y = k - x * a.n_types;
      const int t1 = min(x, y), t2 = max(x, y);
      pair_off[x * kRdfMaxTypes + y] = (t1 * a.n_types - t1 * (t1 + 1) / 2 + t2) * a.bins;  // structure.hpp:51-54
    }
  __syncthreads();
  const int ib = bx * T + tid;
  if (ib < a.S) {
    const uint4 fb = fix[ib];
    const int mb = a.site_mol[ib];
    const int tb = int(fb.w);
    const float sc = a.scale, lo = a.rmax2_lo, hi = a.rmax2_hi, ibw = a.inv_bw_f, babs = a.bin_abs;
    const int na = min(T, a.S - a0);
    for (int k = 0; k < na; ++k) {
      if (ma_s[k] >= mb) continue;  // intermolecular, each pair once
      const uint4 fa = fa_s[k];
      const float dx = float(int(fa.x - fb.x)) * sc;
      const float dy = float(int(fa.y - fb.y)) * sc;
      const float dz = float(int(fa.z - fb.z)) * sc;
      const float d2 = dx * dx + dy * dy + dz * dz;
      if (d2 >= hi) continue;  // outside r_max for certain
      int bin = -2;
      if (d2 < lo) {
        const float t = __fsqrt_rn(d2) * ibw;
        const float f = floorf(t);
        const float m = 1e-6f * t + babs;
        if (t - f > m && f + 1.0f - t > m) bin = int(f) < a.bins ? int(f) : -1;
      }
      if (bin == -2) bin = rdf_exact(sites[a0 + k], sites[ib], a);
      if (bin < 0) continue;
      const int ta = int(fa.w);
      int idx;
      if (table) {
        idx = pair_off[ta * kRdfMaxTypes + tb] + bin;
      } else {
        const int t1 = min(ta, tb), t2 = max(ta, tb);
        idx = (t1 * a.n_types - t1 * (t1 + 1) / 2 + t2) * a.bins + bin;  // structure.hpp:51-54
      }
      if (SHARED)
        atomicAdd(&rdf_hist[idx], 1u);
      else
        atomicAdd(&gcounts[idx], 1ull);
    }
  }
  if (SHARED) {
    __syncthreads();
    for (int k = tid; k < nc; k += T)
      if (rdf_hist[k]) atomicAdd(&gcounts[k], static_cast<unsigned long long>(rdf_hist[k]));
  }
}

}  // namespace b2md
