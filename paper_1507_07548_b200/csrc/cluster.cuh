// Cluster walk of the single-site path: evaluate_range_single_site
// (src/potentials.cpp:148-181) without a partner bit matrix.
//
// The reference visits every pair i < j, takes R = minimum_image(x_i - x_j),
// r2 = norm2(R) and keeps the pair iff r2 < rc2: the partner test IS the
// cutoff test on the force's own r2.  So the force kernel can decide pairs
// itself, on the reference's bits (min_image_wrapped + norm2_exact, exact for
// every pair within rc < L/2), for every candidate a conservative spatial cull
// leaves -- the pair set is identical by construction.
//
// Slots are in spatial order (resort: columns of cross-section ~(8/rho)^(1/3),
// x inside), so kCS consecutive slots form a compact cluster.  Per step:
//   k_cluster_arcs  bounding arcs of every cluster (and of every kSC-cluster
//                   super-cluster) on the periodic fixed-point circle;
//   k_cluster_list  per i-cluster, the clusters whose arcs come within rc
//                   (one warp per i-cluster: super-clusters first, then their
//                   clusters; ballot-compacted, ascending);
//   k_force_cluster one warp per row i: the row's point-vs-arc filter over
//                   its cluster's list, then 4 clusters x 8 members = 32
//                   candidates per warp step under a conservative fixed-point
//                   bound; the maybes are ballot-compacted into a per-warp
//                   ring queue and decided + evaluated 32 at a time on the
//                   reference's fp64 bits with every lane busy.
// Summation order is fixed (list, survivor and lane order), so results are
// deterministic; culls only ever keep extra candidates.
#pragma once

#include "kernels.cuh"

namespace b2md {

#ifndef B2MD_CLUSTER_MINB
#define B2MD_CLUSTER_MINB 4
#endif
constexpr int kCS = 8;          // molecules (consecutive slots) per cluster
constexpr int kSC = 32;         // clusters per super-cluster (list kernel's first cull)
constexpr int kRing = 128;      // per-warp queue (< 64 carried + 64 new)
constexpr float kArcMargin = 2048.0f;  // fixed-point units: float rounding + coordinate rounding

struct ClusterArgs {
  int n, nc, nsup;              // molecules, clusters, super-clusters per replica
  const uint4* fixpos;          // R * n slots: round(x 2^32 / L), w = in-box flag
  uint4* arcs;                  // R * nc: arc centres (fixed point)
  float4* half;                 // R * nc: arc half extents (fixed-point units)
  uint4* sup_arcs;              // R * nsup
  float4* sup_half;             // R * nsup
  int* list;                    // R * nc * nc: candidate clusters of each i-cluster
  int* count;                   // R * nc
  float lim;                    // (rc 2^32 / L)^2 (1 + 1e-5): cull radius^2
  float lim_pair;               // (rc 2^32 / L + 4)^2 (1 + 1e-5): stage-1 pair bound
};

// Lower bound of the circle distance between two arcs (centres x, y, half
// extents summing to hs) on one axis, in fixed-point units.  The wrapping
// int32 difference is the minimum image; the circle distance obeys the
// triangle inequality, so every member pair is at least this far apart.
// float arithmetic: |error| < 1200 units, covered by kArcMargin (which also
// covers the rounding of the coordinates), so the bound stays conservative.
__device__ __forceinline__ float arc_gap(uint32_t x, uint32_t y, float hs) {
  return fmaxf(float(static_cast<unsigned>(abs(int(x - y)))) - hs, 0.0f);
}

__device__ __forceinline__ bool arcs_near(uint4 ca, float4 ha, uint4 cb, float4 hb, float lim) {
  const float gx = arc_gap(ca.x, cb.x, ha.x + hb.x + kArcMargin);
  const float gy = arc_gap(ca.y, cb.y, ha.y + hb.y + kArcMargin);
  const float gz = arc_gap(ca.z, cb.z, ha.z + hb.z + kArcMargin);
  return gx * gx + gy * gy + gz * gz <= lim;
}

// Arc of points given by their wrapping offsets from an anchor (min, max).
__device__ __forceinline__ uint32_t arc_centre(uint32_t anchor, int mn, int mx) {
  return anchor + uint32_t(int((static_cast<long long>(mn) + mx) >> 1));
}
__device__ __forceinline__ float arc_half(int mn, int mx) {
  return float((static_cast<long long>(mx) - mn + 1) >> 1) + 1.0f;
}

// One warp per (replica, super-cluster); lane L owns cluster 32 s + L (its
// kCS slots): the cluster's arc from offsets to its first member, the
// super-cluster's from offsets to the warp's first slot.  A member outside
// [0, L) (fixed point saturated) makes its arcs whole-circle: never culled.
static __global__ void __launch_bounds__(256) k_cluster_arcs(ClusterArgs a, int R) {
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (w >= R * a.nsup) return;  // warp-uniform
  const int r = w / a.nsup, sc = w - r * a.nsup;
  const uint4* f = a.fixpos + size_t(r) * a.n;
  const int cl = sc * kSC + lane;
  const int k0 = cl * kCS, k1 = min(a.n, k0 + kCS);
  const uint4 wa = f[sc * kSC * kCS];  // warp anchor (exists: sc < nsup)
  uint4 u0 = wa;
  bool in = true;
  int mnx = 0, mxx = 0, mny = 0, mxy = 0, mnz = 0, mxz = 0;          // cluster
  int smnx = INT_MAX, smxx = INT_MIN, smny = INT_MAX, smxy = INT_MIN, smnz = INT_MAX, smxz = INT_MIN;
  if (k0 < k1) {
    u0 = f[k0];
    for (int k = k0; k < k1; ++k) {
      const uint4 u = f[k];
      in = in && u.w != 0u;
      const int ox = int(u.x - u0.x), oy = int(u.y - u0.y), oz = int(u.z - u0.z);
      mnx = min(mnx, ox), mxx = max(mxx, ox);
      mny = min(mny, oy), mxy = max(mxy, oy);
      mnz = min(mnz, oz), mxz = max(mxz, oz);
      const int px = int(u.x - wa.x), py = int(u.y - wa.y), pz = int(u.z - wa.z);
      smnx = min(smnx, px), smxx = max(smxx, px);
      smny = min(smny, py), smxy = max(smxy, py);
      smnz = min(smnz, pz), smxz = max(smxz, pz);
    }
    const size_t g = size_t(r) * a.nc + cl;
    a.arcs[g] = make_uint4(arc_centre(u0.x, mnx, mxx), arc_centre(u0.y, mny, mxy),
                           arc_centre(u0.z, mnz, mxz), 0u);
    a.half[g] = in ? make_float4(arc_half(mnx, mxx), arc_half(mny, mxy), arc_half(mnz, mxz), 0.0f)
                   : make_float4(3e9f, 3e9f, 3e9f, 0.0f);
  }
  const unsigned all = 0xffffffffu;
  in = __all_sync(all, in);
  smnx = __reduce_min_sync(all, smnx), smxx = __reduce_max_sync(all, smxx);
  smny = __reduce_min_sync(all, smny), smxy = __reduce_max_sync(all, smxy);
  smnz = __reduce_min_sync(all, smnz), smxz = __reduce_max_sync(all, smxz);
  if (lane == 0) {
    a.sup_arcs[w] = make_uint4(arc_centre(wa.x, smnx, smxx), arc_centre(wa.y, smny, smxy),
                               arc_centre(wa.z, smnz, smxz), 0u);
    a.sup_half[w] = in ? make_float4(arc_half(smnx, smxx), arc_half(smny, smxy),
                                     arc_half(smnz, smxz), 0.0f)
                       : make_float4(3e9f, 3e9f, 3e9f, 0.0f);
  }
}

// One warp per (replica, i-cluster): the clusters (itself included) whose
// arcs come within rc, ascending -- super-clusters first, then the clusters
// of each surviving super-cluster.
static __global__ void __launch_bounds__(256) k_cluster_list(ClusterArgs a, int R) {
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (w >= R * a.nc) return;  // warp-uniform
  const int r = w / a.nc;
  const uint4* __restrict__ arcs = a.arcs + size_t(r) * a.nc;
  const float4* __restrict__ half = a.half + size_t(r) * a.nc;
  const uint4* __restrict__ sarcs = a.sup_arcs + size_t(r) * a.nsup;
  const float4* __restrict__ shalf = a.sup_half + size_t(r) * a.nsup;
  const uint4 ci = a.arcs[w];
  const float4 hi = a.half[w];
  int* __restrict__ out = a.list + size_t(w) * a.nc;
  const unsigned lt = (1u << lane) - 1u;
  int cnt = 0;
  for (int s0 = 0; s0 < a.nsup; s0 += 32) {
    bool near = false;
    if (s0 + lane < a.nsup) near = arcs_near(ci, hi, sarcs[s0 + lane], shalf[s0 + lane], a.lim);
    unsigned sv = __ballot_sync(0xffffffffu, near);
    while (sv) {
      const int sc = s0 + __ffs(sv) - 1;
      sv &= sv - 1u;
      const int j = sc * kSC + lane;
      const bool keep = j < a.nc && arcs_near(ci, hi, arcs[j], half[j], a.lim);
      const unsigned b = __ballot_sync(0xffffffffu, keep);
      if (keep) out[cnt + __popc(b & lt)] = j;
      cnt += __popc(b);
    }
  }
  if (lane == 0) a.count[w] = cnt;
}

// One warp per row (slot) i.  WRAPPED: positions in [0, L) and rc < L/2
// (min_image_wrapped); else the exact minimum image (same bits).
// Stage 1 (every candidate, 32 per warp step): the wrapping int32 difference
// of the fixed-point positions is the minimum image to 1 unit; its fp32 norm
// is compared with (rc + 4 units)^2 (1 + 1e-5) -- a conservative "may be
// within rc" (the rounding of the coordinates, the float conversions and
// sums are all inside the margins).  Maybes (the hits, plus a ~1e-5 shell)
// are ballot-compacted into the warp's ring queue of slots.
// Stage 2 (32 queued maybes at a time, every lane busy): the reference's
// R = minimum_image(x_i - x_j), r2 = norm2(R) on its own bits, the pair kept
// iff r2 < rc2 (potentials.cpp:159-161), and its terms (162-178).
template <bool MULTI_SPECIES, bool WRAPPED, bool VDERIV>
__global__ void __launch_bounds__(kForceWarps * 32, B2MD_CLUSTER_MINB) k_force_cluster(ForceArgs a, ClusterArgs ca) {
  __shared__ int qj[kForceWarps][kRing];      // queued candidate slots (ring)
  __shared__ int sv_list[kForceWarps][32];    // surviving clusters of a list batch
  const SysDev& s = a.s;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int r = blockIdx.y;
  const size_t roff = size_t(r) * s.n;
  const double4* __restrict__ p4 = a.st.pos4 + roff;
  const uint4* __restrict__ fx4 = ca.fixpos + roff;
  const uint4* __restrict__ arcs = ca.arcs + size_t(r) * ca.nc;
  const float4* __restrict__ half = ca.half + size_t(r) * ca.nc;
  const MinImage mi = s.mi;
  const float thr = a.thr;
  auto mimg = [&](double d) {
    return WRAPPED ? min_image_wrapped(d, mi.negL, thr) : min_image(d, mi);
  };
  const double rc2 = a.rc2;
  const float lim_pair = ca.lim_pair;
  const unsigned lt = (1u << lane) - 1u;
  int* __restrict__ wj = qj[warp];
  int* __restrict__ wsv = sv_list[warp];
  double A12 = 0, A6 = 0;  // sum over this warp's pairs (i < j side)
  int cnt = 0;
  const int wpb = blockDim.x >> 5;
  for (int i = blockIdx.x * wpb + warp; i < s.n; i += gridDim.x * wpb) {
    const double4 pi = p4[i];
    const uint4 fi = fx4[i];
    const int si = MULTI_SPECIES ? s.sp_slot[roff + i] : 0;
    const int ic = i / kCS;
    const int* __restrict__ list = ca.list + (size_t(r) * ca.nc + ic) * ca.nc;
    const int nl = ca.count[size_t(r) * ca.nc + ic];
    double fx = 0, fy = 0, fz = 0;
    // stage 2 for candidate slot j (position pj) on this lane
    auto terms = [&](int j, const double4& pj, bool on) {
      const double dx = mimg(sub(pi.x, pj.x));
      const double dy = mimg(sub(pi.y, pj.y));
      const double dz = mimg(sub(pi.z, pj.z));
      const double r2 = norm2_exact(dx, dy, dz);
      if (!(on && r2 < rc2)) return;  // potentials.cpp:161
      double c12 = a.c12, c6 = a.c6;
      if constexpr (MULTI_SPECIES) {
        const int sj = s.sp_slot[roff + j];
        const DevPairInfo& pinfo = s.tab->pair[(i < j) ? si * s.ns + sj : sj * s.ns + si];
        c12 = pinfo.lj_count ? s.tab->lj[pinfo.lj_begin].c12 : 0.0;
        c6 = pinfo.lj_count ? s.tab->lj[pinfo.lj_begin].c6 : 0.0;
      }
      const double inv_r2 = rcp_nr(r2);
      const double ir6 = inv_r2 * inv_r2 * inv_r2;
      const double a12 = c12 * ir6 * ir6;
      const double a6 = c6 * ir6;
      const double du_r = -12.0 * a12 + 6.0 * a6;
      const double fs = -du_r * inv_r2;
      const double gx = fs * dx, gy = fs * dy, gz = fs * dz;
      fx += gx;
      fy += gy;
      fz += gz;
      // the pair's scalars (i < j side) are linear in a12, a6 -- u = a12 - a6,
      // s1 = du_r, s2 = 156 a12 - 42 a6, and dot(R, f) = fs r2 = -du_r --
      // so their sums are taken from sum a12, sum a6 in the epilogue
      const double w = i < j ? 1.0 : 0.0;
      A12 = fma(w, a12, A12);
      A6 = fma(w, a6, A6);
      cnt += i < j;
    };
    // queued slot q on this lane (on: the lane holds an entry)
    auto eval = [&](int q, bool on) {
      const int j = on ? wj[q] : i;
      terms(j, p4[j], on);
    };
    // two full batches, both gathers in flight
    auto eval2 = [&](int qa, int qb) {
      const int ja = wj[qa], jb = wj[qb];
      const double4 pa = p4[ja], pb = p4[jb];
      terms(ja, pa, true);
      terms(jb, pb, true);
    };
    int head = 0, tail = 0;  // warp-uniform ring counters, tail - head < kRing
    for (int l0 = 0; l0 < nl; l0 += 32) {
      // the row's own cull: this point against each listed cluster's arc;
      // survivors compacted (ascending) into the warp's cluster list
      bool keep = false;
      int jc = 0;
      if (l0 + lane < nl) {
        jc = list[l0 + lane];
        keep = arcs_near(fi, make_float4(0.0f, 0.0f, 0.0f, 0.0f), arcs[jc], half[jc], ca.lim);
      }
      const unsigned sv = __ballot_sync(0xffffffffu, keep);
      if (keep) wsv[__popc(sv & lt)] = jc;
      __syncwarp();
      const int nsv = __popc(sv);
      // stage 1, 8 surviving clusters per step (two loads in flight):
      // lane = (cluster lane >> 3, member lane & 7) of each half
      for (int g0 = 0; g0 < nsv; g0 += 8) {
        const int ta = g0 + (lane >> 3), tb = ta + 4;
        const int ja = wsv[ta & 31] * kCS + (lane & 7);
        const int jb = wsv[tb & 31] * kCS + (lane & 7);
        const bool va = ta < nsv && ja < s.n && ja != i;
        const bool vb = tb < nsv && jb < s.n && jb != i;
        const uint4 fa = fx4[va ? ja : i];
        const uint4 fb = fx4[vb ? jb : i];
        // (a saturated fixed point -- position outside [0, L) -- always passes)
        auto maybe = [&](uint4 fj) {
          const float ex = float(int(fi.x - fj.x));
          const float ey = float(int(fi.y - fj.y));
          const float ez = float(int(fi.z - fj.z));
          return !(fi.w & fj.w) || ex * ex + ey * ey + ez * ez <= lim_pair;
        };
        const bool ma = va && maybe(fa), mbb = vb && maybe(fb);
        const unsigned ba = __ballot_sync(0xffffffffu, ma);
        const unsigned bb = __ballot_sync(0xffffffffu, mbb);
        if (ma) wj[(tail + __popc(ba & lt)) & (kRing - 1)] = ja;
        tail += __popc(ba);
        if (mbb) wj[(tail + __popc(bb & lt)) & (kRing - 1)] = jb;
        tail += __popc(bb);
        if (tail - head >= 64) {
          __syncwarp();
          eval2((head + lane) & (kRing - 1), (head + 32 + lane) & (kRing - 1));
          head += 64;
          __syncwarp();
        }
      }
      __syncwarp();  // wsv is rewritten by the next batch
    }
    __syncwarp();
    if (tail - head >= 32) {
      eval((head + lane) & (kRing - 1), true);
      head += 32;
    }
    eval((head + lane) & (kRing - 1), lane < tail - head);
    __syncwarp();
    fx = warp_sum(fx);
    fy = warp_sum(fy);
    fz = warp_sum(fz);
    if (lane == 0) {
      const size_t e = roff + ext_of(pi);
      a.st.fx[e] = fx;
      a.st.fy[e] = fy;
      a.st.fz[e] = fz;
      if (a.kick_dt > 0.0) fused_kick(a, e);
    }
  }
  A12 = warp_sum(A12);
  A6 = warp_sum(A6);
  const double s1 = -12.0 * A12 + 6.0 * A6;  // sum du_r
  double v[kNumRowScalars] = {A12 - A6, 0.0, 0.0, VDERIV ? s1 : 0.0,
                              VDERIV ? 156.0 * A12 - 42.0 * A6 : 0.0, -s1, warp_sum(double(cnt))};
  finalize_scalars<kNumRowScalars>(v, a.cta_part, a.ticket, a.sums, r, 0);
}

}  // namespace b2md
