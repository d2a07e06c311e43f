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
//   k_force_cpair   one warp per half cluster against whole j-clusters (below).
// Summation order is fixed (cluster and lane order), so results are
// deterministic; culls only ever keep extra candidates.
#pragma once

#include "kernels.cuh"

namespace b2md {

constexpr int kCS = 8;          // molecules (consecutive slots) per cluster
constexpr int kSC = 32;         // clusters per super-cluster (the first cull)
constexpr int kRing = 128;      // per-warp queue (< 64 carried + 64 new)
constexpr float kArcMargin = 2048.0f;  // fixed-point units: float rounding + coordinate rounding

struct ClusterArgs {
  int n, nc, nsup;              // molecules, clusters, super-clusters per replica
  const uint4* fixpos;          // R * n slots: round(x 2^32 / L), w = in-box flag
  uint4* arcs;                  // R * nc: arc centres (fixed point)
  float4* half;                 // R * nc: arc half extents (fixed-point units)
  uint4* sup_arcs;              // R * nsup
  float4* sup_half;             // R * nsup
  float lim;                    // (rc 2^32 / L)^2 (1 + 1e-5): cull radius^2
  int grp_begin, grp_end;       // this rank's i-groups (row shard; all of them on one rank)
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

// One CTA per (replica, super-cluster), one thread per slot: a cluster is 8
// consecutive lanes (offsets to its first member, min/max by a 3-level xor
// shuffle), the super-cluster the whole CTA (offsets to its first slot,
// warp REDUX then shared memory).  A member outside [0, L) (fixed point
// saturated) makes its arcs whole-circle: never culled.
// The arcs of one super-cluster's clusters and of the super-cluster itself
// from the fixed-point position u of slot sc * 256 + threadIdx.x (valid: the
// slot exists).  Called by all 256 threads of the CTA.
__device__ __forceinline__ void cluster_arcs_block(const ClusterArgs& a, int r, int sc, uint4 u,
                                                   bool valid) {
  static_assert(kSC * kCS == 256 && kCS == 8, "one CTA of 256 slots per super-cluster");
  __shared__ int red[8][6];
  __shared__ int sin_[8];
  __shared__ uint4 anchor;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) anchor = u;  // slot sc * 256 always exists
  __syncthreads();
  const uint4 wa = anchor;           // super-cluster anchor
  if (!valid) u = wa;
  const unsigned full = 0xffffffffu;
  const int src = lane & ~(kCS - 1);
  const uint4 u0 = make_uint4(__shfl_sync(full, u.x, src), __shfl_sync(full, u.y, src),
                              __shfl_sync(full, u.z, src), 0u);
  // invalid slots repeat the cluster anchor (offset 0, in-box as the anchor)
  int mnx = valid ? int(u.x - u0.x) : 0, mny = valid ? int(u.y - u0.y) : 0;
  int mnz = valid ? int(u.z - u0.z) : 0;
  int mxx = mnx, mxy = mny, mxz = mnz;
  int in = valid ? int(u.w != 0u) : 1;
#pragma unroll
  for (int o = 1; o < kCS; o <<= 1) {
    mnx = min(mnx, __shfl_xor_sync(full, mnx, o)), mxx = max(mxx, __shfl_xor_sync(full, mxx, o));
    mny = min(mny, __shfl_xor_sync(full, mny, o)), mxy = max(mxy, __shfl_xor_sync(full, mxy, o));
    mnz = min(mnz, __shfl_xor_sync(full, mnz, o)), mxz = max(mxz, __shfl_xor_sync(full, mxz, o));
    in &= __shfl_xor_sync(full, in, o);
  }
  const int cl = (sc * kSC * kCS + threadIdx.x) / kCS;
  if ((lane & (kCS - 1)) == 0 && cl < a.nc) {
    const size_t g = size_t(r) * a.nc + cl;
    a.arcs[g] = make_uint4(arc_centre(u0.x, mnx, mxx), arc_centre(u0.y, mny, mxy),
                           arc_centre(u0.z, mnz, mxz), 0u);
    a.half[g] = in ? make_float4(arc_half(mnx, mxx), arc_half(mny, mxy), arc_half(mnz, mxz), 0.0f)
                   : make_float4(3e9f, 3e9f, 3e9f, 0.0f);
  }
  // super-cluster: offsets to wa over the valid slots
  const int px = valid ? int(u.x - wa.x) : 0, py = valid ? int(u.y - wa.y) : 0;
  const int pz = valid ? int(u.z - wa.z) : 0;
  const int v[6] = {__reduce_min_sync(full, px), __reduce_max_sync(full, px),
                    __reduce_min_sync(full, py), __reduce_max_sync(full, py),
                    __reduce_min_sync(full, pz), __reduce_max_sync(full, pz)};
  const int win = __all_sync(full, in != 0);
  if (lane == 0) {
#pragma unroll
    for (int q = 0; q < 6; ++q) red[warp][q] = v[q];
    sin_[warp] = win;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int m[6] = {red[0][0], red[0][1], red[0][2], red[0][3], red[0][4], red[0][5]};
    int all_in = sin_[0];
    for (int w = 1; w < 8; ++w) {
      m[0] = min(m[0], red[w][0]), m[1] = max(m[1], red[w][1]);
      m[2] = min(m[2], red[w][2]), m[3] = max(m[3], red[w][3]);
      m[4] = min(m[4], red[w][4]), m[5] = max(m[5], red[w][5]);
      all_in &= sin_[w];
    }
    const size_t g = size_t(r) * a.nsup + sc;
    a.sup_arcs[g] = make_uint4(arc_centre(wa.x, m[0], m[1]), arc_centre(wa.y, m[2], m[3]),
                               arc_centre(wa.z, m[4], m[5]), 0u);
    a.sup_half[g] = all_in ? make_float4(arc_half(m[0], m[1]), arc_half(m[2], m[3]),
                                         arc_half(m[4], m[5]), 0.0f)
                           : make_float4(3e9f, 3e9f, 3e9f, 0.0f);
  }
}

// One CTA per (replica, super-cluster), one thread per slot: arcs from the
// staged fixed-point positions (after a re-sort or a state upload).
static __global__ void __launch_bounds__(kSC * kCS) k_cluster_arcs(ClusterArgs a, int R) {
  const int r = blockIdx.x / a.nsup, sc = blockIdx.x - r * a.nsup;
  const int k = sc * kSC * kCS + threadIdx.x;  // slot
  const bool valid = k < a.n;
  const uint4 u = a.fixpos[size_t(r) * a.n + (valid ? k : sc * kSC * kCS)];
  cluster_arcs_block(a, r, sc, u, valid);
}

// The step's first half (k_kick_drift, or the end-of-step kick fused with
// the next drift, k_kick_kick_drift) over slot-ordered threads, with the
// cluster arcs of the new positions in the same launch: one CTA per
// (replica, super-cluster), thread = slot, molecule perm[slot].  A frozen
// state (failed step) only re-derives the arcs.
template <bool KICK_FIRST>
static __global__ void __launch_bounds__(kSC * kCS) k_step_drift_arcs(StepArgs sa, ClusterArgs a) {
  const int r = blockIdx.x / a.nsup, sc = blockIdx.x - r * a.nsup;
  const int k = sc * kSC * kCS + threadIdx.x;  // slot
  const bool valid = k < a.n;
  const size_t p = size_t(r) * a.n + (valid ? k : sc * kSC * kCS);
  uint4 u = a.fixpos[p];  // kept when frozen or failing
  if (valid) {
    const int gid = r * a.n + sa.s.perm[p];
    bool frozen = false, ok = true;
    if constexpr (KICK_FIRST) {
      ok = kick_one(sa, gid, &frozen);
      if (!ok) atomicMin(sa.error_mol, gid);
      if (ok && !frozen) u = kick_drift_one(sa, gid);
    } else {
      const uint4 f = kick_drift_one(sa, gid, &frozen);
      if (!frozen) u = f;
    }
  }
  cluster_arcs_block(a, r, sc, u, valid);
}

// ---------------------------------------------------------------------------
// Cluster-pair walk: one warp per i-group (kGR = 4 consecutive slots, half a
// cluster); lane = (j-member jl = lane >> 2, row il = lane & 3), so one warp
// step takes a whole j-cluster against the group, each j position loaded once
// for its 4 rows.  The group's own arc (from its 4 fixed-point points) is
// culled against the super-cluster arcs, then against the clusters of each
// surviving super-cluster -- no list buffer, no list kernel.  Every lane of a
// step computes its pair's R = minimum_image(x_i - x_j), r2 = norm2(R) on the
// reference's bits (potentials.cpp:156-161); a step with no r2 < rc2 in the
// warp ends there, otherwise all lanes run the LJ terms (162-178) with the
// out-of-range lanes zeroed (ir6 = 0 => no force, no energy).  A lane's row
// is fixed, so its force accumulates in registers; the 8 lanes of a row are
// summed by a fixed xor tree at the end (no atomics, deterministic).
// Each pair is visited from both rows with bit-identical r2, so the LJ sums
// are taken over all visits and halved (u, s1, s2, virial); the pair count is
// taken on the i < j side (exact on every row shard).
constexpr int kGR = 4;       // rows per i-group
constexpr int kGWarps = 4;   // warps (i-groups) per CTA
// 7 CTAs (28 warps) per SM: cfg3's 4096 groups still fit one wave, and the
// 72 registers this allows beat 64 at 8 CTAs/SM (10.7k vs 9.5k steps/s; 6
// CTAs / 80 registers: 10.5k)
constexpr int kGMinBlocks = 7;
constexpr int kGList = 256;  // per-warp chunk of surviving clusters (+1: odd-tail pad)
constexpr int kGDepth = 4;   // staged cluster pairs in flight per warp (power of 2)

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void cp_async16(unsigned smem, const void* gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(smem), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// The cluster walk of one i-group (one warp; rows g0 + (lane & 3), this
// lane's row i with position pi / fixed point fi, valid iv): the group's arc
// against the super-cluster and cluster arcs, surviving clusters staged in
// pairs, and for every pair step with some r2 < rc2 in the warp
//   pair(ja, ina, ra, ax, ay, az, jb, inb, rb, bx, by, bz)
// with each lane's partner slot j, in-cutoff flag, r2 and R = min_image(x_i -
// x_j) on the reference's bits (potentials.cpp:156-161).
template <bool WRAPPED, class Pair>
__device__ __forceinline__ void cpair_walk(const ClusterArgs& ca, const double4* __restrict__ p4,
                                           int r, int n, int i, bool iv, const double4& pi,
                                           uint4 fi, double rc2, const MinImage mi, float thr,
                                           int* __restrict__ wl, double4 (*stage)[2][kCS],
                                           Pair&& pair) {
  const int lane = threadIdx.x & 31, jl = lane >> 2;
  const unsigned full = 0xffffffffu, lt = (1u << lane) - 1u;
  const uint4* __restrict__ arcs = ca.arcs + size_t(r) * ca.nc;
  const float4* __restrict__ half = ca.half + size_t(r) * ca.nc;
  const uint4* __restrict__ sarcs = ca.sup_arcs + size_t(r) * ca.nsup;
  const float4* __restrict__ shalf = ca.sup_half + size_t(r) * ca.nsup;
  const float lim = ca.lim;
  auto mimg = [&](double d) {
    return WRAPPED ? min_image_wrapped(d, mi.negL, thr) : min_image(d, mi);
  };
  // the group's arc (offsets from lane 0's point; lanes repeat the 4 rows)
  uint4 gc;
  float4 gh;
  {
    const uint4 f0 = make_uint4(__shfl_sync(full, fi.x, 0), __shfl_sync(full, fi.y, 0),
                                __shfl_sync(full, fi.z, 0), 0u);
    const int ox = int(fi.x - f0.x), oy = int(fi.y - f0.y), oz = int(fi.z - f0.z);
    const int mnx = __reduce_min_sync(full, ox), mxx = __reduce_max_sync(full, ox);
    const int mny = __reduce_min_sync(full, oy), mxy = __reduce_max_sync(full, oy);
    const int mnz = __reduce_min_sync(full, oz), mxz = __reduce_max_sync(full, oz);
    const bool in = __all_sync(full, fi.w != 0u);
    gc = make_uint4(arc_centre(f0.x, mnx, mxx), arc_centre(f0.y, mny, mxy),
                    arc_centre(f0.z, mnz, mxz), 0u);
    gh = in ? make_float4(arc_half(mnx, mxx), arc_half(mny, mxy), arc_half(mnz, mxz), 0.0f)
            : make_float4(3e9f, 3e9f, 3e9f, 0.0f);
  }
  // one lane's pair: distance on the reference's bits
  auto dist = [&](const double4& pj, double& dx, double& dy, double& dz) {
    dx = mimg(sub(pi.x, pj.x));
    dy = mimg(sub(pi.y, pj.y));
    dz = mimg(sub(pi.z, pj.z));
    return norm2_exact(dx, dy, dz);
  };
  // staging ring: slot k holds a cluster pair as 512 contiguous bytes;
  // lane L copies bytes [16 L, 16 L + 16) (lanes 0-15 the first cluster's
  // 8 double4, lanes 16-31 the second's)
  const unsigned ring = smem_u32(&stage[0][0][0]) + 16u * lane;
  const char* __restrict__ src0 = reinterpret_cast<const char*>(p4) + 16 * (lane & 15);
  const int half_sel = lane >> 4;
  const int ilim = iv ? n : 0;  // j < ilim: a real partner slot of a real row
  // surviving clusters, in chunks of <= kGList: super-cluster batch sb
  // (ballot sv), then each super-cluster's clusters (ballot, compacted)
  int sb = 0;
  unsigned sv = 0u;
  for (;;) {
    int nl = 0;
    for (;;) {
      if (sv == 0u) {
        if (sb >= ca.nsup) break;
        const bool near = sb + lane < ca.nsup && arcs_near(gc, gh, sarcs[sb + lane], shalf[sb + lane], lim);
        sv = __ballot_sync(full, near);
        sb += 32;
        continue;
      }
      if (nl > kGList - 32) break;
      const int sc = sb - 32 + __ffs(sv) - 1;
      sv &= sv - 1u;
      const int jc = sc * kSC + lane;
      const bool keep = jc < ca.nc && arcs_near(gc, gh, arcs[jc], half[jc], lim);
      const unsigned cv = __ballot_sync(full, keep);
      if (keep) wl[nl + __popc(cv & lt)] = jc;
      nl += __popc(cv);
    }
    if (nl == 0) break;
    // odd tail: a cluster past the end (all j >= n; staged from pos4's
    // zeroed padding or the next replica, so every lane's r2 is finite)
    if (lane == 0) wl[nl] = ca.nc;
    __syncwarp();
    const int nsteps = (nl + 1) >> 1;
    int next = 0;        // next pair to stage
    unsigned wslot = 0;  // its ring slot (bytes)
    auto issue = [&]() {
      const int e = 2 * next + half_sel;
      if (next < nsteps) cp_async16(ring + wslot, src0 + size_t(wl[e]) * (kCS * 32));
      cp_async_commit();
      ++next;
      wslot = (wslot + 512u) & (512u * kGDepth - 1u);
    };
#pragma unroll
    for (int k = 0; k < kGDepth - 1; ++k) issue();
    const double4* rs = &stage[0][0][jl];
    for (int st = 0; st < nsteps; ++st) {
      issue();
      cp_async_wait<kGDepth - 1>();
      __syncwarp();
      const int slot = st & (kGDepth - 1);
      const int ja = wl[2 * st] * kCS + jl, jb = wl[2 * st + 1] * kCS + jl;
      const bool va = ja < ilim && ja != i;
      const bool vb = jb < ilim && jb != i;
      double ax, ay, az, bx, by, bz;
      const double ra = dist(rs[slot * 2 * kCS], ax, ay, az);
      const double rb = dist(rs[slot * 2 * kCS + kCS], bx, by, bz);
      __syncwarp();  // the slot's reads are consumed before it is refilled
      const bool ina = va && ra < rc2, inb = vb && rb < rc2;  // potentials.cpp:161
      if (__ballot_sync(full, ina || inb) == 0u) continue;
      pair(ja, ina, ra, ax, ay, az, jb, inb, rb, bx, by, bz);
    }
    cp_async_wait<0>();
    __syncwarp();  // wl and the ring are rewritten by the next chunk
  }
}

template <bool MULTI_SPECIES, bool WRAPPED, bool VDERIV>
__global__ void __launch_bounds__(kGWarps * 32, kGMinBlocks) k_force_cpair(ForceArgs a, ClusterArgs ca) {
  __shared__ int clist[kGWarps][kGList + 1];
  __shared__ __align__(128) double4 stage[kGWarps][kGDepth][2][kCS];
  const SysDev& s = a.s;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int r = blockIdx.y;
  const size_t roff = size_t(r) * s.n;
  const double4* __restrict__ p4 = a.st.pos4 + roff;
  const uint4* __restrict__ fx4 = ca.fixpos + roff;
  const unsigned full = 0xffffffffu;
  const int n = s.n;
  const int g0 = (blockIdx.x * kGWarps + warp) * kGR;  // the group's first slot
  // sums over all visits: single species B12 = sum ir6^2, B6 = sum ir6
  // (a12 = c12 B12, a6 = c6 B6); mixtures sum a12, a6 directly
  double B12 = 0, B6 = 0;
  int cnt = 0;
  const int grp = blockIdx.x * kGWarps + warp;
  if (g0 < n && (grp < ca.grp_begin || grp >= ca.grp_end)) {
    // another rank's rows (row shard): zero forces into the all-reduce
    if (lane < kGR && g0 + lane < n) {
      const size_t e = roff + ext_of(p4[g0 + lane]);
      a.st.fx[e] = 0.0;
      a.st.fy[e] = 0.0;
      a.st.fz[e] = 0.0;
    }
  } else if (g0 < n) {  // warp-uniform
    const int i = g0 + (lane & (kGR - 1));
    const bool iv = i < n;
    const int ic = iv ? i : g0;  // clamped row
    const double4 pi = p4[ic];
    const int si = MULTI_SPECIES ? s.sp_slot[roff + ic] : 0;
    double fx = 0, fy = 0, fz = 0;
    auto terms = [&](int j, bool in, double r2, double dx, double dy, double dz) {
      const double inv_r2 = rcp_nr(in ? r2 : 1.0);
      const double t6 = inv_r2 * inv_r2 * inv_r2;
      const double ir6 = in ? t6 : 0.0;
      double fs;
      if constexpr (MULTI_SPECIES) {
        // lanes past the last slot (partial / odd-tail pad cluster) have no
        // species: their ir6 is 0, any valid species index keeps c12, c6 finite
        const int sj = in ? s.sp_slot[roff + j] : si;
        const DevPairInfo& pinfo = s.tab->pair[(i < j) ? si * s.ns + sj : sj * s.ns + si];
        const double c12 = pinfo.lj_count ? s.tab->lj[pinfo.lj_begin].c12 : 0.0;
        const double c6 = pinfo.lj_count ? s.tab->lj[pinfo.lj_begin].c6 : 0.0;
        const double a12 = c12 * ir6 * ir6, a6 = c6 * ir6;
        fs = (12.0 * a12 - 6.0 * a6) * inv_r2;  // -du_r / r2
        B12 += a12;
        B6 += a6;
      } else {
        fs = fma(ir6, a.c12x12, -a.c6x6) * ir6 * inv_r2;
        B12 = fma(ir6, ir6, B12);
        B6 += ir6;
      }
      if (in) {  // (predicated: an excluded pair's R may be NaN -- a NaN position
                 // fails the reference's r2 < rc2 test and touches nobody)
        fx = fma(fs, dx, fx);
        fy = fma(fs, dy, fy);
        fz = fma(fs, dz, fz);
      }
      cnt += in && i < j;  // exact per shard: the pair's i < j side
    };
    cpair_walk<WRAPPED>(ca, p4, r, n, i, iv, pi, fx4[ic], a.rc2, s.mi, a.thr, clist[warp],
                        stage[warp],
                        [&](int ja, bool ina, double ra, double ax, double ay, double az, int jb,
                            bool inb, double rb, double bx, double by, double bz) {
                          terms(ja, ina, ra, ax, ay, az);
                          terms(jb, inb, rb, bx, by, bz);
                        });
    // a row's 8 lanes (il fixed, jl = lane >> 2): fixed xor tree
#pragma unroll
    for (int o = 4; o < 32; o <<= 1) {
      fx += __shfl_xor_sync(full, fx, o);
      fy += __shfl_xor_sync(full, fy, o);
      fz += __shfl_xor_sync(full, fz, o);
    }
    if (lane < kGR && iv) {
      const size_t e = roff + ext_of(pi);
      a.st.fx[e] = fx;
      a.st.fy[e] = fy;
      a.st.fz[e] = fz;
      if (a.kick_dt > 0.0) fused_kick(a, e);
    }
  }
  // every pair was visited twice (bit-identical terms): halve the sums
  double A12 = 0.5 * warp_sum(B12), A6 = 0.5 * warp_sum(B6);
  if constexpr (!MULTI_SPECIES) {
    A12 *= a.c12;
    A6 *= a.c6;
  }
  const double s1 = -12.0 * A12 + 6.0 * A6;  // sum du_r
  double v[kNumRowScalars] = {A12 - A6, 0.0, 0.0, VDERIV ? s1 : 0.0,
                              VDERIV ? 156.0 * A12 - 42.0 * A6 : 0.0, -s1,
                              warp_sum(double(cnt))};
  finalize_scalars<kNumRowScalars>(v, a.cta_part, a.ticket, a.sums, r, 0);
}

// heat_flux (greenkubo.cpp:182-266) of a single-species, centred, LJ-only
// system on the cluster walk (no partner search): the same row split as
// k_heat_flux -- row i adds 0.5 (f_i . v_i) R_i over its partners (f_i the
// pair's force on i, R_i = min_image(com_i - com_j)), 0.5 sum_p u_p v_i and,
// where `kinetic` is set, (e_kin_i - h) v_i.  In-range lanes only carry
// terms (ir6 = 0 elsewhere); per-row lane sums by a fixed xor tree.
template <bool WRAPPED>
__global__ void __launch_bounds__(kGWarps * 32, kGMinBlocks) k_heat_flux_cpair(FluxArgs fa, ClusterArgs ca) {
  __shared__ int clist[kGWarps][kGList + 1];
  __shared__ __align__(128) double4 stage[kGWarps][kGDepth][2][kCS];
  const ForceArgs& a = fa.f;
  const SysDev& s = a.s;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int r = blockIdx.y;
  const size_t roff = size_t(r) * s.n;
  const double4* __restrict__ p4 = a.st.pos4 + roff;
  const uint4* __restrict__ fx4 = ca.fixpos + roff;
  const unsigned full = 0xffffffffu;
  const int n = s.n;
  const int grp = blockIdx.x * kGWarps + warp;
  const int g0 = grp * kGR;  // the group's first slot
  double jx = 0, jy = 0, jz = 0;
  if (g0 < n && grp >= ca.grp_begin && grp < ca.grp_end) {  // warp-uniform
    const int i = g0 + (lane & (kGR - 1));
    const bool iv = i < n;
    const int ic = iv ? i : g0;  // clamped row
    const double4 pi = p4[ic];
    const size_t ge = roff + ext_of(pi);
    const double vix = a.st.vx[ge], viy = a.st.vy[ge], viz = a.st.vz[ge];
    double tx = 0, ty = 0, tz = 0, up = 0;  // sum_p 0.5 (f.v_i) R_p, sum_p u_p
    auto term = [&](bool in, double r2, double dx, double dy, double dz) {
      const double inv_r2 = rcp_nr(in ? r2 : 1.0);
      const double t6 = inv_r2 * inv_r2 * inv_r2;
      const double ir6 = in ? t6 : 0.0;
      const double a12 = a.c12 * ir6 * ir6, a6 = a.c6 * ir6;
      const double fs = (12.0 * a12 - 6.0 * a6) * inv_r2;  // -du_r / r2
      if (in) {  // (an excluded pair's R may be NaN: see k_force_cpair)
        const double sp = 0.5 * fs * (dx * vix + dy * viy + dz * viz);
        tx += sp * dx;
        ty += sp * dy;
        tz += sp * dz;
      }
      up += a12 - a6;
    };
    cpair_walk<WRAPPED>(ca, p4, r, n, i, iv, pi, fx4[ic], a.rc2, s.mi, a.thr, clist[warp],
                        stage[warp],
                        [&](int, bool ina, double ra, double ax, double ay, double az, int,
                            bool inb, double rb, double bx, double by, double bz) {
                          term(ina, ra, ax, ay, az);
                          term(inb, rb, bx, by, bz);
                        });
#pragma unroll
    for (int o = 4; o < 32; o <<= 1) {
      tx += __shfl_xor_sync(full, tx, o);
      ty += __shfl_xor_sync(full, ty, o);
      tz += __shfl_xor_sync(full, tz, o);
      up += __shfl_xor_sync(full, up, o);
    }
    if (lane < kGR && iv) {
      double e = 0.5 * up;
      if (fa.kinetic) {
        const DevSpecies& sp = s.tab->species[0];
        const double wbx = a.st.wx[ge], wby = a.st.wy[ge], wbz = a.st.wz[ge];
        const double ek = 0.5 * sp.total_mass * (vix * vix + viy * viy + viz * viz) +
                          0.5 * (sp.inertia[0] * wbx * wbx + sp.inertia[1] * wby * wby +
                                 sp.inertia[2] * wbz * wbz);
        e += ek - fa.enthalpy[0];
      }
      jx = tx + e * vix;
      jy = ty + e * viy;
      jz = tz + e * viz;
    }
  }
  double v[3] = {warp_sum(jx), warp_sum(jy), warp_sum(jz)};
  finalize_scalars<3>(v, a.cta_part, a.ticket, fa.out, r, 0);
}

}  // namespace b2md
