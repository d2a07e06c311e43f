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

// ---------------------------------------------------------------------------
// Once-per-pair cluster walk (Newton's third law), the north star's race-free
// scheme: every molecule pair is evaluated ONCE, its force applied to both
// partners, and the partner-side contributions go to a per-pair contribution
// buffer that is reduced in a fixed order -- the GPU form of the reference's
// per-worker buffers summed in worker order (src/potentials.cpp:166-170,
// src/parallel.cpp:84-95).  No atomics on floating-point data: results are
// bit-identical run to run.
//
// * k_cpair_build -- one warp per cluster c, one cull (c's arc against
//   super-cluster and cluster arcs) for both of c's roles.  Cluster pair
//   {ci, jc} belongs to ci iff ci == jc (pairs j > i inside the cluster) or
//   (ci < jc) == (ci + jc even) -- the checker rule, so every cluster owns
//   about half of its neighbours wherever it sits in the spatial order.
//   As owner, c's owned list goes to global memory, cut into work units of
//   <= kUnit j-clusters (a contiguous unit range).  As receiver, c's owners
//   (found in increasing index) get a contiguous record range: owner x's
//   j-side record for c goes to slot in_base[c] + rank(x), published in a
//   dense [owner][receiver] slot map.
// * k_force_cpair_n3 -- persistent warps take work units from a counter
//   (which warp runs a unit does not change its result).  lane = (j-member
//   jl = lane >> 2, il = lane & 3) owns rows ia = 8 ci + il and ib = ia + 4;
//   one warp step takes a whole j-cluster (64 pairs).  A unit's i-side force
//   is one record; the j-side force of each step (the 8 rows summed through
//   shared memory in a fixed order) is one 192-byte record per owned cluster
//   pair at the pair's triangular index.  Small dynamically assigned units
//   keep a cluster with a large neighbourhood (one straddling two columns)
//   from setting the kernel's length.
// * k_cpair_jsum -- one warp per cluster: its unit records in unit order,
//   then its receiver records in owner order -- two contiguous ranges, a
//   fixed order -- force = i-side - j-side, the fused end-of-step kick.
// Each pair's r2 and cutoff decision are the reference's bits (as in
// k_force_cpair); energy, virial, s1, s2 and the pair count are taken once
// per pair (no halving).
constexpr int kUnit = 16;  // j-clusters per work unit

struct PairBuf {
  double* rec;      // R * nc (nc + 1) / 2 j-side records of 8 x 3 doubles (i-side sign),
                    // receiver-major: cluster c's records are slots in_base[c] + rank(owner)
  double* irec;     // R * max_units i-side records (8 x 3 doubles)
  int* olist;       // R * nc * nc: owned listed j-clusters of each cluster
  int* ilist;       // R * nc * nc: owners of each cluster (increasing), build scratch
  int* inslot;      // R * nc * nc: [owner][receiver] -> record slot
  int* ocnt;        // R * nc
  int* ustart;      // R * nc: first unit of each cluster (its units are contiguous)
  int* umap;        // R * max_units: unit -> cluster
  int* in_base;     // R * nc: first record slot of each receiver
  int* in_cnt;      // R * nc: owners of each receiver
  int* units;       // R: units of this evaluation (reset by the walk's last CTA)
  int* in_total;    // R: record slots of this evaluation (reset by the walk's last CTA)
  int* next_unit;   // R: work counter (reset by the walk's last CTA)
  unsigned* ticket; // R: the walk's last-CTA ticket
  int max_units;
  int cbeg, cend;   // this rank's owner clusters (row shard)
};

// triangular index of the unordered cluster pair {a, b}, a <= b (32-bit: the
// record array is capped at 8 GB, i.e. < 2^26 pairs)
__device__ __forceinline__ int tri_index(int a, int b, int nc) {
  return a * nc - ((a * (a - 1)) >> 1) + (b - a);
}

__device__ __forceinline__ bool owns_pair(int ci, int jc) {
  return ci == jc || ((ci < jc) == (((ci ^ jc) & 1) == 0));
}

constexpr int kBuildWarps = 4;

// 32-byte load through L2 (data another SM wrote during this launch)
__device__ __forceinline__ double4 ldcg4(const double4* p) {
  const double2* q = reinterpret_cast<const double2*>(p);
  const double2 a = __ldcg(q), b = __ldcg(q + 1);
  return make_double4(a.x, a.y, b.x, b.y);
}

static __global__ void __launch_bounds__(kBuildWarps * 32)
    k_cpair_build(ForceArgs a, ClusterArgs ca, PairBuf pb) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int r = blockIdx.y;
  const int nc = ca.nc, n = a.s.n;
  const unsigned full = 0xffffffffu, lt = (1u << lane) - 1u;
  const int c = blockIdx.x * kBuildWarps + warp;
  if (c >= nc) return;
  const bool mine = c >= pb.cbeg && c < pb.cend;  // this rank owns c's pairs
  const uint4* __restrict__ arcs = ca.arcs + size_t(r) * nc;
  const float4* __restrict__ half = ca.half + size_t(r) * nc;
  const uint4* __restrict__ sarcs = ca.sup_arcs + size_t(r) * ca.nsup;
  const float4* __restrict__ shalf = ca.sup_half + size_t(r) * ca.nsup;
  const uint4 gc = arcs[c];
  const float4 gh = half[c];
  int* __restrict__ out = pb.olist + (size_t(r) * nc + c) * nc;
  int* __restrict__ inl = pb.ilist + (size_t(r) * nc + c) * nc;
  int nl = 0, ni = 0;
  for (int sb = 0; sb < ca.nsup; sb += 32) {
    const int sc0 = sb + lane;
    unsigned sv =
        __ballot_sync(full, sc0 < ca.nsup && arcs_near(gc, gh, sarcs[sc0], shalf[sc0], ca.lim));
    // 4 surviving super-clusters per round (their arc loads in flight together),
    // in increasing index: owners are found in increasing order
    while (sv) {
      int scs[4];
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        scs[b] = sv ? sb + __ffs(sv) - 1 : -1;
        sv &= sv ? sv - 1u : 0u;
      }
      bool near[4];
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const int jc = scs[b] * kSC + lane;
        near[b] = scs[b] >= 0 && jc < nc && arcs_near(gc, gh, arcs[jc], half[jc], ca.lim);
      }
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const int jc = scs[b] * kSC + lane;
        const bool own = near[b] && owns_pair(c, jc);
        const bool inc = near[b] && (jc == c || !own);
        // owned pairs only on the rank that owns c; owners: those on their rank
        const bool o = own && mine;
        const bool x = inc && jc >= pb.cbeg && jc < pb.cend;
        const unsigned ov = __ballot_sync(full, o), xv = __ballot_sync(full, x);
        if (o) out[nl + __popc(ov & lt)] = jc;
        if (x) inl[ni + __popc(xv & lt)] = jc;
        nl += __popc(ov);
        ni += __popc(xv);
      }
    }
  }
  if (!mine && lane < kCS && c * kCS + lane < n) {
    // another rank's rows (row shard): written 0 here, overwritten by
    // k_cpair_jsum when this rank has records for them
    const size_t roff = size_t(r) * n;
    const size_t e = roff + ext_of(a.st.pos4[roff + c * kCS + lane]);
    a.st.fx[e] = 0.0;
    a.st.fy[e] = 0.0;
    a.st.fz[e] = 0.0;
  }
  const int nu = (nl + kUnit - 1) / kUnit;
  int ubase = 0, ibase = 0;
  if (lane == 0) {
    if (nu) ubase = atomicAdd(&pb.units[r], nu);
    if (ni) ibase = atomicAdd(&pb.in_total[r], ni);
    pb.ocnt[size_t(r) * nc + c] = nl;
    pb.ustart[size_t(r) * nc + c] = ubase;
    pb.in_cnt[size_t(r) * nc + c] = ni;
    pb.in_base[size_t(r) * nc + c] = ibase;
  }
  ubase = __shfl_sync(full, ubase, 0);
  ibase = __shfl_sync(full, ibase, 0);
  for (int k = lane; k < nu; k += 32) pb.umap[size_t(r) * pb.max_units + ubase + k] = c;
  __syncwarp();
  for (int t = lane; t < ni; t += 32)
    pb.inslot[(size_t(r) * nc + inl[t]) * nc + c] = ibase + t;
}

// L2 cache-policy hints for the contribution records: stored evict_last
// (read back by k_cpair_jsum right after the walk), loaded evict_first
__device__ __forceinline__ uint64_t l2_policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t l2_policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void st_hint(double* a, double v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(a), "d"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ double4 ld4_hint(const double4* a, uint64_t pol) {
  double4 v;
  const double2* q = reinterpret_cast<const double2*>(a);
  asm volatile("ld.global.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;"
               : "=d"(v.x), "=d"(v.y) : "l"(q), "l"(pol));
  asm volatile("ld.global.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;"
               : "=d"(v.z), "=d"(v.w) : "l"(q + 1), "l"(pol));
  return v;
}

// 28 resident warps per SM (72 registers)
constexpr int kNWarpsPerSM = 28;
constexpr int kJStride = 20;    // doubles per jl row of the j-side transpose (bank-conflict free)

template <int NW, bool MULTI_SPECIES, bool WRAPPED, bool VDERIV>
__global__ void __launch_bounds__(NW * 32, kNWarpsPerSM / NW)
    k_force_cpair_n3(ForceArgs a, ClusterArgs ca, PairBuf pb) {
  __shared__ int wl_s[NW][kUnit + 2];
  __shared__ int wr_s[NW][kUnit + 2];
  __shared__ __align__(128) double4 stage[NW][kGDepth][2][kCS];
  __shared__ __align__(16) double jt[NW][kCS * kJStride];  // j-side transpose
  const SysDev& s = a.s;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int jl = lane >> 2, il = lane & 3;
  const int r = blockIdx.y;
  const size_t roff = size_t(r) * s.n;
  const double4* __restrict__ p4 = a.st.pos4 + roff;
  const unsigned full = 0xffffffffu;
  const int n = s.n, nc = ca.nc;
  const int* __restrict__ ustart = pb.ustart + size_t(r) * nc;
  const int* __restrict__ umap = pb.umap + size_t(r) * pb.max_units;
  const int* __restrict__ ocnt = pb.ocnt + size_t(r) * nc;
  double* __restrict__ rec = pb.rec + size_t(r) * (size_t(nc) * (nc + 1) / 2) * (kCS * 3);
  double* __restrict__ irec = pb.irec + size_t(r) * pb.max_units * (kCS * 3);
  const int total = pb.units[r];
  const uint64_t pol = l2_policy_evict_last();
  int* wl = wl_s[warp];
  int* wr = wr_s[warp];
  double* jtw = jt[warp];
  const unsigned ring = smem_u32(&stage[warp][0][0][0]) + 16u * lane;
  const char* __restrict__ src0 = reinterpret_cast<const char*>(p4) + 16 * (lane & 15);
  const int half_sel = lane >> 4;
  const MinImage mi = s.mi;
  const float thr = a.thr;
  const double rc2 = a.rc2;
  auto mimg = [&](double d) {
    return WRAPPED ? min_image_wrapped(d, mi.negL, thr) : min_image(d, mi);
  };
  auto dist = [&](const double4& pi, const double4& pj, double& dx, double& dy, double& dz) {
    dx = mimg(sub(pi.x, pj.x));
    dy = mimg(sub(pi.y, pj.y));
    dz = mimg(sub(pi.z, pj.z));
    return norm2_exact(dx, dy, dz);
  };
  double B12 = 0, B6 = 0;
  int cnt = 0;
  // LJ force scalar -du_r / r2 of one pair (0 when out of range; the
  // in-range flag also keeps a NaN position's R out of every sum)
  auto lj = [&](bool in, double r2, int si, int sj) {
    const double inv_r2 = rcp_nr(in ? r2 : 1.0);
    const double t6 = inv_r2 * inv_r2 * inv_r2;
    const double ir6 = in ? t6 : 0.0;
    double fs;
    if constexpr (MULTI_SPECIES) {
      // Lorentz-Berthelot terms are symmetric in the species pair
      const DevPairInfo& pinfo = s.tab->pair[si * s.ns + sj];
      const double c12 = pinfo.lj_count ? s.tab->lj[pinfo.lj_begin].c12 : 0.0;
      const double c6 = pinfo.lj_count ? s.tab->lj[pinfo.lj_begin].c6 : 0.0;
      const double a12 = c12 * ir6 * ir6, a6 = c6 * ir6;
      fs = (12.0 * a12 - 6.0 * a6) * inv_r2;
      B12 += a12;
      B6 += a6;
    } else {
      fs = fma(ir6, a.c12x12, -a.c6x6) * ir6 * inv_r2;
      B12 = fma(ir6, ir6, B12);
      B6 += ir6;
    }
    return fs;
  };
  for (;;) {
    int u = 0;
    if (lane == 0) u = atomicAdd(&pb.next_unit[r], 1);
    u = __shfl_sync(full, u, 0);
    if (u >= total) break;  // warp-uniform
    const int ci = umap[u];
    const int k0 = (u - ustart[ci]) * kUnit;
    const int len = min(kUnit, ocnt[ci] - k0);
    if (lane < len) {
      const int jc = pb.olist[(size_t(r) * nc + ci) * nc + k0 + lane];
      wl[lane] = jc;
      wr[lane] = pb.inslot[(size_t(r) * nc + ci) * nc + jc] * (kCS * 3);  // in jc's range
    }
    if (lane == 0 && (len & 1)) {  // odd tail: a pad cluster past the end (no valid j)
      wl[len] = nc;
      wr[len] = -1;
    }
    const int ia = ci * kCS + il, ib = ia + 4;
    const bool iva = ia < n, ivb = ib < n;
    const double4 pa = p4[iva ? ia : ci * kCS], pbp = p4[ivb ? ib : ci * kCS];
    const int sia = MULTI_SPECIES ? s.sp_slot[roff + (iva ? ia : ci * kCS)] : 0;
    const int sib = MULTI_SPECIES ? s.sp_slot[roff + (ivb ? ib : ci * kCS)] : 0;
    double fax = 0, fay = 0, faz = 0, fbx = 0, fby = 0, fbz = 0;
    __syncwarp();
    const int nsteps = (len + 1) >> 1;
    int next = 0;
    unsigned wslot = 0;
    auto issue = [&]() {
      const int e = 2 * next + half_sel;
      if (next < nsteps) cp_async16(ring + wslot, src0 + size_t(wl[e]) * (kCS * 32));
      cp_async_commit();
      ++next;
      wslot = (wslot + 512u) & (512u * kGDepth - 1u);
    };
#pragma unroll
    for (int k = 0; k < kGDepth - 1; ++k) issue();
    for (int st = 0; st < nsteps; ++st) {
      issue();
      cp_async_wait<kGDepth - 1>();
      __syncwarp();
      const int slot = st & (kGDepth - 1);
#pragma unroll 1
      for (int h = 0; h < 2; ++h) {
        const int jc = wl[2 * st + h];
        const int ro = wr[2 * st + h];
        const int j = jc * kCS + jl;
        const double4 pj = stage[warp][slot][h][jl];
        const bool vj = j < n;
        const bool self = jc == ci;
        const bool va = iva && vj && (!self || j > ia);
        const bool vb = ivb && vj && (!self || j > ib);
        double dxa, dya, dza, dxb, dyb, dzb;
        const double r2a = dist(pa, pj, dxa, dya, dza);
        const double r2b = dist(pbp, pj, dxb, dyb, dzb);
        const bool ina = va && r2a < rc2, inb = vb && r2b < rc2;  // potentials.cpp:161
        double* rj = rec + ro + jl * 3 + il;
        if (__ballot_sync(full, ina || inb) == 0u) {
          if (ro >= 0 && il < 3) st_hint(rj, 0.0, pol);  // listed: the record is read
          continue;
        }
        const int sj = MULTI_SPECIES ? (vj ? s.sp_slot[roff + j] : sia) : 0;
        const double fsa = lj(ina, r2a, sia, sj);
        const double fsb = lj(inb, r2b, sib, sj);
        double gx = 0, gy = 0, gz = 0;
        if (ina) {
          gx = fsa * dxa, gy = fsa * dya, gz = fsa * dza;
          fax += gx, fay += gy, faz += gz;
        }
        if (inb) {
          const double hx = fsb * dxb, hy = fsb * dyb, hz = fsb * dzb;
          fbx += hx, fby += hy, fbz += hz;
          gx += hx, gy += hy, gz += hz;
        }
        cnt += int(ina) + int(inb);
        // j-side: the 4 il lanes of member jl summed through shared memory
        // (lane (jl, c) adds component c of rows il = 0..3 in order)
        double* t = jtw + jl * kJStride + il * 4;
        *reinterpret_cast<double2*>(t) = make_double2(gx, gy);
        t[2] = gz;
        __syncwarp();
        if (il < 3) {
          const double* v = jtw + jl * kJStride + il;
          st_hint(rj, ((v[0] + v[4]) + v[8]) + v[12], pol);
        }
        __syncwarp();  // jt is rewritten by the next step
      }
      __syncwarp();  // the slot's reads are consumed before it is refilled
    }
    cp_async_wait<0>();
    // rows ia / ib: their 8 jl lanes by a fixed xor tree
#pragma unroll
    for (int o = 4; o < 32; o <<= 1) {
      fax += __shfl_xor_sync(full, fax, o);
      fay += __shfl_xor_sync(full, fay, o);
      faz += __shfl_xor_sync(full, faz, o);
      fbx += __shfl_xor_sync(full, fbx, o);
      fby += __shfl_xor_sync(full, fby, o);
      fbz += __shfl_xor_sync(full, fbz, o);
    }
    if (lane < 4) {  // the unit's i-side record: member m, component c at 3 m + c
      double* q = irec + size_t(u) * (kCS * 3);
      q[3 * il] = fax, q[3 * il + 1] = fay, q[3 * il + 2] = faz;
      q[3 * (il + 4)] = fbx, q[3 * (il + 4) + 1] = fby, q[3 * (il + 4) + 2] = fbz;
    }
    __syncwarp();  // wl / wr / the ring are rewritten by the next unit
  }
  // once per pair: no halving
  double A12 = warp_sum(B12), A6 = warp_sum(B6);
  if constexpr (!MULTI_SPECIES) {
    A12 *= a.c12;
    A6 *= a.c6;
  }
  const double s1 = -12.0 * A12 + 6.0 * A6;  // sum du_r
  double v[kNumRowScalars] = {A12 - A6, 0.0, 0.0, VDERIV ? s1 : 0.0,
                              VDERIV ? 156.0 * A12 - 42.0 * A6 : 0.0, -s1,
                              warp_sum(double(cnt))};
  finalize_scalars<kNumRowScalars>(v, a.cta_part, a.ticket, a.sums, r, 0);
  // the last CTA re-arms the unit counters for the next evaluation
  __shared__ bool lastcta;
  __syncthreads();
  if (threadIdx.x == 0) lastcta = atomicAdd(&pb.ticket[r], 1u) == gridDim.x - 1;
  __syncthreads();
  if (lastcta && threadIdx.x == 0) {
    pb.units[r] = 0;
    pb.in_total[r] = 0;
    pb.next_unit[r] = 0;
    pb.ticket[r] = 0u;
  }
}

// The fixed-order reduction of the contribution buffers: one warp per
// cluster c.  Its records are two contiguous ranges -- its unit records
// (i-side, unit order) and its receiver records (j-side, increasing owner)
// -- read 5 at a time as double4 (lane = (record q = lane / 6, quarter p =
// lane % 6)), each lane summing its quarter over records q, q + 5, ... (8
// loads in flight); the 5 partial sums are added in q order.  Force =
// i-side - j-side, then the fused end-of-step kick.
constexpr int kJsumWarps = 4;

static __global__ void __launch_bounds__(kJsumWarps * 32) k_cpair_jsum(ForceArgs a, ClusterArgs ca,
                                                                        PairBuf pb) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int r = blockIdx.y;
  const int n = a.s.n, nc = ca.nc;
  const int c = blockIdx.x * kJsumWarps + warp;
  if (c >= nc) return;
  const unsigned full = 0xffffffffu;
  const size_t roff = size_t(r) * n;
  const int q = lane / 6, p = lane - 6 * (lane / 6);  // record in a group of 5, quarter
  const int u0 = pb.ustart[size_t(r) * nc + c];
  const int nu = (pb.ocnt[size_t(r) * nc + c] + kUnit - 1) / kUnit;
  const int i0 = pb.in_base[size_t(r) * nc + c];
  const int ni = pb.in_cnt[size_t(r) * nc + c];
  const int slot = c * kCS + (lane & 7);
  const int ext = slot < n ? ext_of(a.st.pos4[roff + slot]) : 0;
  const uint64_t pol = l2_policy_evict_first();
  auto sum_range = [&](const double4* __restrict__ base, int cnt) {
    double4 acc = make_double4(0.0, 0.0, 0.0, 0.0);
    if (q < 5) {
      int e = q;
      for (; e + 35 < cnt; e += 40) {
        double4 v[8];
#pragma unroll
        for (int b = 0; b < 8; ++b) v[b] = ld4_hint(base + size_t(e + 5 * b) * 6 + p, pol);
#pragma unroll
        for (int b = 0; b < 8; ++b) acc.x += v[b].x, acc.y += v[b].y, acc.z += v[b].z, acc.w += v[b].w;
      }
      for (; e < cnt; e += 5) {
        const double4 v = ld4_hint(base + size_t(e) * 6 + p, pol);
        acc.x += v.x, acc.y += v.y, acc.z += v.z, acc.w += v.w;
      }
    }
    return acc;
  };
  double4 ai = sum_range(reinterpret_cast<const double4*>(pb.irec + size_t(r) * pb.max_units * (kCS * 3)) +
                             size_t(u0) * 6, nu);
  double4 aj = sum_range(reinterpret_cast<const double4*>(
                             pb.rec + size_t(r) * (size_t(nc) * (nc + 1) / 2) * (kCS * 3)) +
                             size_t(i0) * 6, ni);
#pragma unroll
  for (int g = 1; g < 5; ++g) {
    const int src = g * 6 + p;
    const double xi = __shfl_sync(full, ai.x, src), yi = __shfl_sync(full, ai.y, src);
    const double zi = __shfl_sync(full, ai.z, src), wi = __shfl_sync(full, ai.w, src);
    const double xj = __shfl_sync(full, aj.x, src), yj = __shfl_sync(full, aj.y, src);
    const double zj = __shfl_sync(full, aj.z, src), wj = __shfl_sync(full, aj.w, src);
    if (q == 0) {
      ai.x += xi, ai.y += yi, ai.z += zi, ai.w += wi;
      aj.x += xj, aj.y += yj, aj.z += zj, aj.w += wj;
    }
  }
  // lane p < 6 holds doubles 4p .. 4p + 3 of the 24 (member d / 3, component d % 3)
  const double v[4] = {ai.x - aj.x, ai.y - aj.y, ai.z - aj.z, ai.w - aj.w};
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    const int d = 4 * p + t, m = d / 3, cc = d - 3 * (d / 3);
    const int e = __shfl_sync(full, ext, m);
    if (q == 0 && c * kCS + m < n) {
      double* f = cc == 0 ? a.st.fx : (cc == 1 ? a.st.fy : a.st.fz);
      f[roff + e] = v[t];
    }
  }
  __syncwarp();
  if (lane < kCS && slot < n && a.kick_dt > 0.0) fused_kick(a, roff + ext);
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
