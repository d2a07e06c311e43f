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

#include <cub/block/block_scan.cuh>

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
  // once-per-pair list (k_force_nl): build positions and control words; the
  // drift keeps the largest displacement^2 since the build (null: no list)
  const uint4* fixref;
  int* nl_ctl;
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
  if (a.nl_ctl) {
    // the largest displacement^2 since the list build (fixed-point circle
    // distance; float bits compare as integers, a NaN or out-of-box position
    // above +inf): one atomicMax per CTA
    __shared__ unsigned dmax[kSC * kCS / 32];
    unsigned db = 0u;
    if (valid) {
      const uint4 f0 = a.fixref[p];
      const float dx = float(int(u.x - f0.x)), dy = float(int(u.y - f0.y)),
                  dz = float(int(u.z - f0.z));
      db = u.w ? __float_as_uint(dx * dx + dy * dy + dz * dz) : 0x7fc00000u;
    }
    db = __reduce_max_sync(0xffffffffu, db);
    if ((threadIdx.x & 31) == 0) dmax[threadIdx.x >> 5] = db;
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned m = 0u;
      for (int w = 0; w < kSC * kCS / 32; ++w) m = max(m, dmax[w]);
      atomicMax(reinterpret_cast<unsigned*>(a.nl_ctl) + size_t(r) * 8 + 6, m);  // kNLD2
    }
  }
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
template <int OFF>
__device__ __forceinline__ void sts_f64(unsigned addr, double v) {
  asm volatile("st.shared.f64 [%0+%2], %1;" ::"r"(addr), "d"(v), "n"(OFF) : "memory");
}
template <int OFF>
__device__ __forceinline__ double lds_f64(unsigned addr) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1+%2];" : "=d"(v) : "r"(addr), "n"(OFF) : "memory");
  return v;
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// Bulk (TMA) copies global -> shared completing on an mbarrier (tx bytes)
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned phase) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

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

// The both-rows walk of one i-group grp (one warp): forces of its 4 rows
// written (with the fused end-of-step kick when a.kick_dt > 0), the LJ sums
// of every visit into B12 / B6 (each pair is visited from both rows: the
// caller halves them) and the pair count on the i < j side into cnt.
// Another rank's groups (row shard) write zero forces into the all-reduce.
template <bool MULTI_SPECIES, bool WRAPPED>
__device__ __forceinline__ void cpair_group_forces(const ForceArgs& a, const ClusterArgs& ca, int r,
                                                   int grp, int* __restrict__ clist,
                                                   double4 (*stage)[2][kCS], double& B12,
                                                   double& B6, int& cnt) {
  const SysDev& s = a.s;
  const int lane = threadIdx.x & 31;
  const size_t roff = size_t(r) * s.n;
  const double4* __restrict__ p4 = a.st.pos4 + roff;
  const uint4* __restrict__ fx4 = ca.fixpos + roff;
  const unsigned full = 0xffffffffu;
  const int n = s.n;
  const int g0 = grp * kGR;  // the group's first slot
  if (g0 >= n) return;       // warp-uniform
  if (grp < ca.grp_begin || grp >= ca.grp_end) {
    // another rank's rows (row shard): zero forces into the all-reduce
    if (lane < kGR && g0 + lane < n) {
      const size_t e = roff + ext_of(p4[g0 + lane]);
      a.st.fx[e] = 0.0;
      a.st.fy[e] = 0.0;
      a.st.fz[e] = 0.0;
    }
    return;
  }
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
  cpair_walk<WRAPPED>(ca, p4, r, n, i, iv, pi, fx4[ic], a.rc2, s.mi, a.thr, clist, stage,
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

template <bool MULTI_SPECIES, bool WRAPPED, bool VDERIV>
__global__ void __launch_bounds__(kGWarps * 32, kGMinBlocks) k_force_cpair(ForceArgs a, ClusterArgs ca) {
  __shared__ int clist[kGWarps][kGList + 1];
  __shared__ __align__(128) double4 stage[kGWarps][kGDepth][2][kCS];
  const int warp = threadIdx.x >> 5;
  const int r = blockIdx.y;
  // sums over all visits: single species B12 = sum ir6^2, B6 = sum ir6
  // (a12 = c12 B12, a6 = c6 B6); mixtures sum a12, a6 directly
  double B12 = 0, B6 = 0;
  int cnt = 0;
  cpair_group_forces<MULTI_SPECIES, WRAPPED>(a, ca, r, blockIdx.x * kGWarps + warp, clist[warp],
                                             stage[warp], B12, B6, cnt);
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
// Once-per-pair cluster-pair list (Newton's third law): the north star's
// race-free scheme.  Every molecule pair is evaluated ONCE, its force applied
// to both partners; the partner-side contributions go to a per-pair
// contribution buffer that is summed in a fixed order -- the GPU form of the
// reference's +-f per pair (src/potentials.cpp:166-170) and its per-worker
// buffers summed in worker order (src/parallel.cpp:84-95).  No atomics on
// floating-point data: results are bit-identical run to run.
//
// * The list (built after every re-sort / staging and every nl_interval
//   steps): every cluster pair whose bounding arcs were within rc + skin,
//   each owned by one of its clusters -- ci == cj (pairs j > i inside the
//   cluster) or (ci < cj) == (ci + cj even), the checker rule, so every
//   cluster owns about half of its neighbours wherever it sits in the spatial
//   order.  An owner's entries {cj | shift codes, ci, record slot, build gap}
//   are contiguous (increasing cj), padded to a multiple of kB with entries
//   that never pass the cull, so a batch of kB entries has one owner; a
//   receiver's incoming records are contiguous (receiver-major slots, owner
//   order).  Built by k_nl_count, k_nl_scan, k_nl_fill, k_nl_zfill (no
//   atomics: the layout is a pure function of the arcs).
// * Periodic images per entry: where neither cluster's arc (widened by the
//   skin) can reach the box boundary on an axis, every member pair's raw
//   difference d = x_i - x_j lies in one interval for the list's lifetime;
//   when that interval is inside (-L/2, L/2), (L/2, 3L/2) or (-3L/2, -L/2)
//   with a 1e-5 margin, the reference's nearbyint(d / L) is 0, 1 or -1 for
//   every pair and its d - L nearbyint(d / L) is d, d - L or d + L: one
//   correctly rounded add per axis, the reference's bits
//   (potentials.hpp:176-181).  An entry with an axis that cannot be decided
//   (code 3) takes min_image_wrapped per pair.
// * Exactness of the pair set: the drift keeps D^2, the largest squared
//   displacement of any molecule since the build (fixed-point circle
//   distance).  A pair within rc now was within rc + 2 D at the build, so an
//   entry whose build gap is >= rc + 2 D is skipped this step (the skin costs
//   list length, not pair work), and while D <= skin / 2 every pair within rc
//   is listed.  Beyond that the list is stale and never used -- k_force_nl
//   runs the exact per-step cull walk (both rows, cpair_group_forces) until
//   the next build.
// * k_force_nl: batches of kB entries (one owner ci) dealt round-robin to
//   the warps; a batch's surviving entries and the owner's 8 positions are
//   staged into shared memory by bulk (TMA) copies on the warp's mbarrier,
//   one batch ahead of the compute (double buffer).  lane = (j-member jl =
//   lane >> 2, il = lane & 3) owns rows ia = 8 ci + il and ib = ia + 4; a
//   warp step takes a whole j-cluster (64 pairs).  Each pair's r2 and cutoff
//   decision are the reference's bits (potentials.cpp:156-161).  An entry
//   with a pair in cutoff writes its 256-byte j-side record -- lane (jl, c)
//   component c of member jl's sum over the 4 row lanes (fixed order, through
//   shared memory), lane (jl, 3) the evaluation's epoch stamp -- and a batch
//   its i-side record in the same layout.
// * k_nl_reduce: one warp per cluster: its batches' i-side records, then its
//   stamped incoming records -- force = i-side - j-side, a fixed order -- and
//   the fused end-of-step kick.
constexpr int kNLBuildWarps = 4;  // warps (clusters) per CTA of the build / reduce kernels
constexpr int kNLParts = 4;       // build warps per cluster (contiguous super-cluster ranges)
constexpr int kNLWarps = 4;       // warps per CTA of k_force_nl
#ifndef B2MD_NL_MINBLOCKS
#define B2MD_NL_MINBLOCKS 5
#endif
constexpr int kNLMinBlocks = B2MD_NL_MINBLOCKS;  // 20 warps per SM (<= 96 registers)
#ifndef B2MD_NL_BATCH
#define B2MD_NL_BATCH 16
#endif
constexpr int kB = B2MD_NL_BATCH;  // entries per batch (one owner)
#ifndef B2MD_NL_TMA
#define B2MD_NL_TMA 0             // stage by bulk (TMA) copies instead of per-lane cp.async
#endif
constexpr int kRecD = kCS * 4;    // doubles per i-side record: 8 members x (x, y, z, epoch stamp)
constexpr int kRecP = kCS * 3;    // doubles per j-side record: 8 members x (x, y, z); stamp apart
constexpr int kNLCtl = 8;         // control words per replica
constexpr int kJcBits = 24;       // entry.x = cj | shift codes << 24 (2 bits per axis)
constexpr int kJcMask = (1 << kJcBits) - 1;
// ctl words: entries (padded), incoming slots, epoch, ticket, overflow, D^2 bits
enum { kNLEntries = 0, kNLIncoming = 1, kNLEpoch = 2, kNLTicket = 3, kNLOverflow = 5, kNLD2 = 6 };

struct NListArgs {
  int* ocnt;       // R * nc: owned entries of each cluster, padded to kB (0 for another rank's)
  int* ocp;        // R * nc * kNLParts: owned entries found by each build part (unpadded)
  int* icp;        // R * nc * kNLParts: incoming slots found by each build part
  int* icnt;       // R * nc: incoming slots (owners x of {x, c}, c itself included)
  int* ebase;      // R * (nc + 1): first entry of each cluster (per-replica numbering)
  int* ibase;      // R * (nc + 1): first incoming slot
  int4* ent;       // R * max_ent: {cj | codes << 24, ci, record slot, build gap^2 bits}
  int* in_src;     // R * max_ent: owner of each incoming slot (build scratch)
  int* smap;       // R * nc * nc: [owner][receiver] -> incoming slot (build scratch; null when
                   // too large: k_nl_inrec's binary searches instead)
  double* rec;     // R * max_ent * kRecP: j-side sums g = sum_i f_ij (force on j: -g),
                   // receiver-major (cluster c's incoming slots ibase[c] .. ibase[c + 1])
  int* rstamp;     // R * max_ent: epoch of the evaluation that wrote each j-side record
  double* irec;    // R * (max_ent / kB) * kRecD: i-side force of each batch
  uint4* fixref;   // R * n: fixed-point positions at the build (slot order)
  int* ctl;        // R * kNLCtl
  float lim_build;  // ((rc + skin) 2^32 / L)^2 (1 + 1e-5)
  float skin_half;  // skin / 2 in fixed-point units (+ margin): the displacement bound
  float rc_fix;     // rc 2^32 / L
  unsigned d2_stale;  // bits of ((skin / 2) 2^32 / L)^2 (1 - 1e-4): D^2 above is stale
  int max_ent;
  int cbeg, cend;  // this rank's owner clusters
};

// The list cannot be used this evaluation (overflow at the build, or a
// molecule moved more than skin / 2 since): read by k_force_nl and k_nl_reduce
__device__ __forceinline__ bool nl_stale(const NListArgs& nl, const int* ctl) {
  return ctl[kNLOverflow] != 0 || unsigned(ctl[kNLD2]) > nl.d2_stale;
}

// c's neighbour clusters within the cull radius^2 lim (fixed-point units)
// among super-clusters [sb0, sb1), in increasing order: for every batch of 32
// candidates (one surviving
// super-cluster) visit(jc, near) runs on all lanes (warp-uniform call).  Up
// to 4 surviving super-clusters have their arc loads in flight together.
template <class Visit>
__device__ __forceinline__ void nl_scan(const ClusterArgs& ca, int r, uint4 gc, float4 gh, float lim,
                                        int sb0, int sb1, Visit&& visit) {
  const int lane = threadIdx.x & 31;
  const unsigned full = 0xffffffffu;
  const uint4* __restrict__ arcs = ca.arcs + size_t(r) * ca.nc;
  const float4* __restrict__ half = ca.half + size_t(r) * ca.nc;
  const uint4* __restrict__ sarcs = ca.sup_arcs + size_t(r) * ca.nsup;
  const float4* __restrict__ shalf = ca.sup_half + size_t(r) * ca.nsup;
  for (int sb = sb0; sb < sb1; sb += 32) {
    unsigned sv = __ballot_sync(
        full, sb + lane < sb1 && arcs_near(gc, gh, sarcs[sb + lane], shalf[sb + lane], lim));
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
        near[b] = scs[b] >= 0 && jc < ca.nc && arcs_near(gc, gh, arcs[jc], half[jc], lim);
      }
#pragma unroll
      for (int b = 0; b < 4; ++b)
        if (scs[b] >= 0) visit(scs[b] * kSC + lane, near[b]);
    }
  }
}

__device__ __forceinline__ bool owns_pair(int ci, int jc) {
  return ci == jc || ((ci < jc) == (((ci ^ jc) & 1) == 0));
}

// Squared gap between two arcs (fixed-point units, a lower bound: arcs_near's margins)
__device__ __forceinline__ float arcs_gap2(uint4 ca, float4 ha, uint4 cb, float4 hb) {
  const float gx = arc_gap(ca.x, cb.x, ha.x + hb.x + kArcMargin);
  const float gy = arc_gap(ca.y, cb.y, ha.y + hb.y + kArcMargin);
  const float gz = arc_gap(ca.z, cb.z, ha.z + hb.z + kArcMargin);
  return gx * gx + gy * gy + gz * gz;
}

// Shift code of one axis for the member pairs of arcs (ca, ha) x (cb, hb)
// over the list's lifetime (every member within w = skin / 2 + margin of its
// build position): 0: d, 1: d - L, 2: d + L for every pair; 3: per pair.
// Fixed-point units (L = 2^32); double arithmetic on integers < 2^34 is exact.
__device__ __forceinline__ int shift_code(uint32_t ca, float ha, uint32_t cb, float hb, float w) {
  const double H = 4294967296.0, half = 2147483648.0, tol = 2147483648.0 * 1e-5 + 4096.0;
  const double a0 = double(ca) - (double(ha) + w), a1 = double(ca) + (double(ha) + w);
  const double b0 = double(cb) - (double(hb) + w), b1 = double(cb) + (double(hb) + w);
  if (a0 < 0.0 || a1 >= H || b0 < 0.0 || b1 >= H) return 3;  // an arc may cross the boundary
  const double lo = a0 - b1, hi = a1 - b0;                    // every raw difference d
  if (lo > -half + tol && hi < half - tol) return 0;
  if (lo > half + tol && hi < 3.0 * half - tol) return 1;
  if (lo > -3.0 * half + tol && hi < -half - tol) return 2;
  return 3;
}

// pass 1: owned entries and incoming slots of every cluster, kNLParts warps
// per cluster (part p: super-clusters [p nsup / P, (p+1) nsup / P))
static __global__ void __launch_bounds__(kNLBuildWarps * 32)
    k_nl_count(ClusterArgs ca, NListArgs nl) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int r = blockIdx.y, nc = ca.nc;
  const int w = blockIdx.x * kNLBuildWarps + warp, c = w / kNLParts, part = w - c * kNLParts;
  if (c >= nc) return;
  const unsigned full = 0xffffffffu;
  const uint4 gc = ca.arcs[size_t(r) * nc + c];
  const float4 gh = ca.half[size_t(r) * nc + c];
  const int sb0 = part * ca.nsup / kNLParts, sb1 = (part + 1) * ca.nsup / kNLParts;
  int no = 0, ni = 0;
  nl_scan(ca, r, gc, gh, nl.lim_build, sb0, sb1, [&](int jc, bool near) {
    const bool own = near && owns_pair(c, jc);
    no += __popc(__ballot_sync(full, own));
    ni += __popc(__ballot_sync(full, near && (jc == c || !own)));
  });
  if (lane == 0) {
    const bool mine = c >= nl.cbeg && c < nl.cend;
    nl.ocp[size_t(r) * nc * kNLParts + w] = mine ? no : 0;
    nl.icp[size_t(r) * nc * kNLParts + w] = ni;
  }
}

// pass 2: exclusive scans of entries and incoming slots (one CTA per
// replica); totals, overflow check and a fresh displacement bound into ctl
// (an overflowing list is never used: the exact per-step walk runs instead)
constexpr int kNLScanThreads = 1024;
static __global__ void __launch_bounds__(kNLScanThreads) k_nl_scan(NListArgs nl, int nc) {
  using Scan = cub::BlockScan<int, kNLScanThreads>;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ int carry[2];
  const int r = blockIdx.x;
  int* eb = nl.ebase + size_t(r) * (nc + 1);
  int* ib = nl.ibase + size_t(r) * (nc + 1);
  if (threadIdx.x < 2) carry[threadIdx.x] = 0;
  __syncthreads();
  for (int b = 0; b < nc; b += kNLScanThreads) {
    const int c = b + threadIdx.x;
    int ov = 0, iv = 0;
    if (c < nc) {
#pragma unroll
      for (int q = 0; q < kNLParts; ++q) {
        ov += nl.ocp[(size_t(r) * nc + c) * kNLParts + q];
        iv += nl.icp[(size_t(r) * nc + c) * kNLParts + q];
      }
      ov = (ov + kB - 1) / kB * kB;  // padded to whole batches
      nl.ocnt[size_t(r) * nc + c] = ov;
      nl.icnt[size_t(r) * nc + c] = iv;
    }
    int x0, x1, t0, t1;
    Scan(tmp).ExclusiveSum(ov, x0, t0);
    __syncthreads();
    Scan(tmp).ExclusiveSum(iv, x1, t1);
    if (c < nc) {
      eb[c] = carry[0] + x0;
      ib[c] = carry[1] + x1;
    }
    __syncthreads();
    if (threadIdx.x == 0) carry[0] += t0, carry[1] += t1;
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    eb[nc] = carry[0];
    ib[nc] = carry[1];
    int* ctl = nl.ctl + size_t(r) * kNLCtl;
    ctl[kNLEntries] = carry[0];
    ctl[kNLIncoming] = carry[1];
    ctl[kNLTicket] = 0;
    ctl[kNLOverflow] = (carry[0] > nl.max_ent || carry[1] > nl.max_ent) ? 1 : 0;
    ctl[kNLD2] = 0;
  }
}

// pass 3: entries (owned, increasing cj, shift codes, build gap; padding
// entries that never pass the cull), incoming owners (increasing) and the
// build positions of the displacement bound
static __global__ void __launch_bounds__(kNLBuildWarps * 32)
    k_nl_fill(ClusterArgs ca, NListArgs nl) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int r = blockIdx.y, nc = ca.nc, n = ca.n;
  const int w = blockIdx.x * kNLBuildWarps + warp, c = w / kNLParts, part = w - c * kNLParts;
  if (c >= nc) return;
  if (part == 0 && lane < kCS && c * kCS + lane < n)
    nl.fixref[size_t(r) * n + c * kCS + lane] = ca.fixpos[size_t(r) * n + c * kCS + lane];
  if (nl.ctl[size_t(r) * kNLCtl + kNLOverflow]) return;  // never read
  const unsigned full = 0xffffffffu, lt = (1u << lane) - 1u;
  const uint4 gc = ca.arcs[size_t(r) * nc + c];
  const float4 gh = ca.half[size_t(r) * nc + c];
  const bool mine = c >= nl.cbeg && c < nl.cend;
  // this part's offsets: the earlier parts' counts
  int eb = nl.ebase[size_t(r) * (nc + 1) + c], ib = nl.ibase[size_t(r) * (nc + 1) + c];
  const int ee = nl.ebase[size_t(r) * (nc + 1) + c + 1];
  for (int q = 0; q < part; ++q) {
    eb += nl.ocp[(size_t(r) * nc + c) * kNLParts + q];
    ib += nl.icp[(size_t(r) * nc + c) * kNLParts + q];
  }
  const int sb0 = part * ca.nsup / kNLParts, sb1 = (part + 1) * ca.nsup / kNLParts;
  int4* __restrict__ ent = nl.ent + size_t(r) * nl.max_ent;
  int* __restrict__ src = nl.in_src + size_t(r) * nl.max_ent;
  const uint4* __restrict__ arcs = ca.arcs + size_t(r) * nc;
  const float4* __restrict__ half = ca.half + size_t(r) * nc;
  int no = 0, ni = 0;
  nl_scan(ca, r, gc, gh, nl.lim_build, sb0, sb1, [&](int jc, bool near) {
    const bool own = near && owns_pair(c, jc);
    const bool inc = near && (jc == c || !own);
    const unsigned ov = __ballot_sync(full, own && mine), iv = __ballot_sync(full, inc);
    if (own && mine) {
      const uint4 cj = arcs[jc];
      const float4 hj = half[jc];
      const int code = shift_code(gc.x, gh.x, cj.x, hj.x, nl.skin_half) |
                       shift_code(gc.y, gh.y, cj.y, hj.y, nl.skin_half) << 2 |
                       shift_code(gc.z, gh.z, cj.z, hj.z, nl.skin_half) << 4;
      const float g2 = jc == c ? 0.0f : arcs_gap2(gc, gh, cj, hj);
      ent[eb + no + __popc(ov & lt)] = make_int4(jc | code << kJcBits, c, 0, __float_as_int(g2));
    }
    if (inc) {
      src[ib + ni + __popc(iv & lt)] = jc;
      if (nl.smap) nl.smap[(size_t(r) * nc + jc) * nc + c] = ib + ni + __popc(iv & lt);
    }
    no += __popc(ov);
    ni += __popc(iv);
  });
  if (part == kNLParts - 1)
    for (int e = eb + no + lane; e < ee; e += 32)  // padding: above every c, never culled in
      ent[e] = make_int4(kJcMask, c, 0, 0x7f800000);
}

// pass 4: the record slot of every entry: receiver c's incoming slot t of
// owner x, found in x's (sorted) entries by binary search (owners on another
// rank have no entries here: the slot is never written)
static __global__ void __launch_bounds__(kNLBuildWarps * 32) k_nl_inrec(NListArgs nl, int nc) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int r = blockIdx.y;
  const int c = blockIdx.x * kNLBuildWarps + warp;
  if (c >= nc || nl.ctl[size_t(r) * kNLCtl + kNLOverflow]) return;
  const int* eb = nl.ebase + size_t(r) * (nc + 1);
  int4* ent = nl.ent + size_t(r) * nl.max_ent;
  const int i0 = nl.ibase[size_t(r) * (nc + 1) + c], i1 = nl.ibase[size_t(r) * (nc + 1) + c + 1];
  for (int t = i0 + lane; t < i1; t += 32) {
    const int x = nl.in_src[size_t(r) * nl.max_ent + t];
    int lo = eb[x], hi = eb[x + 1];
    while (lo < hi) {  // first entry >= c
      const int mid = (lo + hi) >> 1;
      if ((ent[mid].x & kJcMask) < c) lo = mid + 1; else hi = mid;
    }
    if (lo < eb[x + 1] && (ent[lo].x & kJcMask) == c) ent[lo].z = t;
  }
}

// pass 4 with the dense [owner][receiver] slot map: every entry's record
// slot in one gather (one warp per owner)
static __global__ void __launch_bounds__(kNLBuildWarps * 32) k_nl_zfill(NListArgs nl, int nc) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int r = blockIdx.y;
  const int x = blockIdx.x * kNLBuildWarps + warp;
  if (x >= nc || nl.ctl[size_t(r) * kNLCtl + kNLOverflow]) return;
  const int* eb = nl.ebase + size_t(r) * (nc + 1);
  int4* ent = nl.ent + size_t(r) * nl.max_ent;
  const int* sm = nl.smap + (size_t(r) * nc + x) * nc;
  for (int e = eb[x] + lane; e < eb[x + 1]; e += 32) {
    const int jc = ent[e].x & kJcMask;
    if (jc != kJcMask) ent[e].z = sm[jc];
  }
}

// pass 5: every entry's build gap tightened from the arcs' bound to the
// smallest member-pair distance at the build.  One warp per batch (one owner:
// its 8 members in registers), two lanes per entry (4 j-members each against
// the 8 i-members).  Integer arithmetic on the wrapping fixed-point
// differences (the minimum image), truncated to 16 bits per axis: each
// component is off by < 1 unit of 2^16, the distance by < sqrt(3) units; 2
// units are taken off (the rest covers the coordinates' own rounding) and
// 1e-6 relative for the float conversion, square root and square -- a lower
// bound, so `gap >= rc + 2 D` still proves that no member pair is within rc.
// Entries whose members are all beyond rc + skin get a gap the per-step cull
// never passes while the list is valid.  A member outside [0, L) keeps the
// arcs' bound (0: whole-circle arcs).
static __global__ void __launch_bounds__(kNLBuildWarps * 32) k_nl_gaps(ClusterArgs ca, NListArgs nl) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int r = blockIdx.y, n = ca.n;
  const int* ctl = nl.ctl + size_t(r) * kNLCtl;
  if (ctl[kNLOverflow]) return;
  const int nbt = ctl[kNLEntries] / kB;
  int4* __restrict__ ent = nl.ent + size_t(r) * nl.max_ent;
  const uint4* __restrict__ fix = ca.fixpos + size_t(r) * n;
  constexpr int kLPE = 32 / kB;       // lanes per entry
  constexpr int kJPL = kCS / kLPE;    // j-members per lane
  static_assert(kB * kLPE == 32 && kJPL * kLPE == kCS, "whole entries per warp, whole members per lane");
  for (int bt = blockIdx.x * kNLBuildWarps + warp; bt < nbt; bt += gridDim.x * kNLBuildWarps) {
    const int e = bt * kB + lane / kLPE;
    const int4 en = ent[e];
    const int ci = en.y;
    // padding entries never pass the cull and a cluster's own entry has gap 0
    const bool live = (en.x & kJcMask) != kJcMask && (en.x & kJcMask) != ci;
    const int jc = live ? (en.x & kJcMask) : ci;
    bool inbox = true;
    int ix[kCS], iy[kCS], iz[kCS];
    bool iv[kCS];
#pragma unroll
    for (int m = 0; m < kCS; ++m) {
      iv[m] = ci * kCS + m < n;
      const uint4 u = fix[iv[m] ? ci * kCS + m : ci * kCS];
      ix[m] = int(u.x), iy[m] = int(u.y), iz[m] = int(u.z);
      inbox = inbox && u.w != 0u;
    }
    unsigned best = 0xffffffffu;
#pragma unroll
    for (int k = 0; k < kJPL; ++k) {
      const int j = jc * kCS + (lane % kLPE) * kJPL + k;
      const bool vj = j < n;
      const uint4 u = fix[vj ? j : jc * kCS];
      inbox = inbox && u.w != 0u;
#pragma unroll
      for (int m = 0; m < kCS; ++m) {
        const int dx = (ix[m] - int(u.x)) >> 16, dy = (iy[m] - int(u.y)) >> 16,
                  dz = (iz[m] - int(u.z)) >> 16;
        const unsigned d2 = unsigned(dx * dx) + unsigned(dy * dy) + unsigned(dz * dz);
        if (vj && iv[m]) best = min(best, d2);
      }
    }
#pragma unroll
    for (int o = 1; o < kLPE; o <<= 1) {
      best = min(best, __shfl_xor_sync(0xffffffffu, best, o));
      inbox = __shfl_xor_sync(0xffffffffu, int(inbox), o) != 0 && inbox;
    }
    if (lane % kLPE == 0 && inbox && live) {
      const float g = fmaxf(sqrtf(float(best)) - 2.0f, 0.0f) * (65536.0f * (1.0f - 1e-6f));
      const float g2 = fmaxf(g * g, __int_as_float(en.w));
      ent[e].w = __float_as_int(g2);
    }
  }
}

__device__ __forceinline__ double stamp_of(int epoch) { return __longlong_as_double((long long)epoch); }

template <bool MULTI_SPECIES, bool WRAPPED, bool VDERIV>
__global__ void __launch_bounds__(kNLWarps * 32, kNLMinBlocks)
    k_force_nl(ForceArgs a, ClusterArgs ca, NListArgs nl) {
  const SysDev& s = a.s;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int jl = lane >> 2, il = lane & 3;
  const int r = blockIdx.y;
  const size_t roff = size_t(r) * s.n;
  const unsigned full = 0xffffffffu;
  const int n = s.n;
  int* ctl = nl.ctl + size_t(r) * kNLCtl;
  double B12 = 0, B6 = 0;  // once per pair (no halving)
  int cnt = 0;
  const int epoch = ctl[kNLEpoch];
  // shared memory: the exact walk's per-warp lists and staging ring, or the
  // list walk's staged batches (2 buffers x (kB j-clusters + the owner) per warp)
  constexpr int kSlots = kB + 1;
  __shared__ __align__(128) unsigned char smem[kNLWarps * 2 * kSlots * kCS * sizeof(double4)];
  static_assert(sizeof(smem) >= (kNLWarps * (kGList + 1) * sizeof(int) + 127) / 128 * 128 +
                                    kNLWarps * kGDepth * 2 * kCS * sizeof(double4),
                "exact walk scratch");
  if (nl_stale(nl, ctl)) {
    // stale list: the exact per-step cull walk (both rows) for every group
    auto clist = reinterpret_cast<int (*)[kGList + 1]>(smem);
    constexpr size_t off = (kNLWarps * (kGList + 1) * sizeof(int) + 127) / 128 * 128;
    auto stage = reinterpret_cast<double4 (*)[kGDepth][2][kCS]>(smem + off);
    double b12 = 0, b6 = 0;
    ForceArgs af = a;
    af.kick_dt = 0.0;  // k_nl_reduce kicks
    for (int grp = blockIdx.x * kNLWarps + warp; grp * kGR < n; grp += gridDim.x * kNLWarps)
      cpair_group_forces<MULTI_SPECIES, WRAPPED>(af, ca, r, grp, clist[warp], stage[warp], b12, b6,
                                                 cnt);
    B12 = 0.5 * b12;  // both visits
    B6 = 0.5 * b6;
  } else {
    const int E = ctl[kNLEntries];  // a multiple of kB
    const int nbt = E / kB;
    const int nw = gridDim.x * kNLWarps;
    const int gw = blockIdx.x * kNLWarps + warp;
    const int4* __restrict__ ent = nl.ent + size_t(r) * nl.max_ent;
    double* __restrict__ rec = nl.rec + size_t(r) * nl.max_ent * kRecP + 3 * jl + (il < 3 ? il : 2);
    int* __restrict__ rstamp = nl.rstamp + size_t(r) * nl.max_ent;
    const double4* __restrict__ p4 = a.st.pos4 + roff;
    const double L = s.mi.L;
    const double stamp = stamp_of(epoch);
    // this evaluation's cull: build gap^2 < (rc + 2 D)^2 (fixed-point units)
    const float dd = nl.rc_fix + 2.0f * sqrtf(__uint_as_float(unsigned(ctl[kNLD2])));
    const float lim_now = dd * dd * (1.0f + 1e-5f);
    // LJ force scalar -du_r / r2 of one pair (0 when out of range; the
    // in-range flag also keeps a NaN position's R out of every sum)
    auto lj = [&](bool in, double r2, int si, int sj) {
      const double inv_r2 = rcp_nr(r2);
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
    // per-warp scratch: the staged batches' surviving entries {cj | codes,
    // record slot}, their j-clusters and the owner's cluster (256 contiguous
    // bytes of pos4 each, bulk copies completing on the buffer's mbarrier),
    // and two buffers of the j-side transpose (lane (jl, il) -> lane (jl, c))
    __shared__ int2 elist[kNLWarps][2][kB];
    __shared__ double jt[kNLWarps][2][4 * kCS * 3];
    __shared__ __align__(8) uint64_t mbar[kNLWarps][2];
    double4 (*jst)[kSlots][kCS] = reinterpret_cast<double4 (*)[kSlots][kCS]>(smem) + warp * 2;
    if (lane < 2) mbar_init(&mbar[warp][lane], 1);
    __syncwarp();
    unsigned phase = 0u;  // bit p: parity of buffer p's next completion
    const int cw = il < 3 ? il : 2;  // component read by this lane in the transpose
    // the entry loop's per-lane addresses, kept in registers (opaque to the
    // compiler, which otherwise re-derives them from the kernel arguments in
    // every entry): the transpose's write / read slots (buffer 0; buffer 1 is
    // jt_flip bytes on) and this lane's word of record 0
    unsigned jt_wr = smem_u32(&jt[warp][0][il * 24 + jl * 3]);
    unsigned jt_rd = smem_u32(&jt[warp][0][jl * 3 + cw]);
    unsigned jt_par = 0u;
    constexpr unsigned jt_flip = 4 * kCS * 3 * sizeof(double);
    unsigned jt_wr0 = smem_u32(&jt[warp][0][0]);
    asm volatile("" : "+r"(jt_wr), "+r"(jt_rd), "+r"(jt_wr0));
    asm volatile("" : "+l"(rec), "+l"(rstamp));
    // only the partial last cluster has members that do not exist
    const int last_c = (n & (kCS - 1)) ? n / kCS : -1;
    // batch bt's cull, compaction and copies into buffer p (the surviving
    // j-clusters and the owner's cluster); returns the number of survivors
    // (0: no copies, no mbarrier phase)
    auto stage_batch = [&](int p, const int4& en) {
      const bool near = lane < kB && __int_as_float(en.w) < lim_now;
      const unsigned act = __ballot_sync(full, near);
      const int na = __popc(act);
      const int owner = __shfl_sync(full, en.y, 0);
      if (na == 0) return 0;
#if B2MD_NL_TMA
      fence_proxy_async();  // earlier reads of this buffer precede the copies
      if (lane == 0)
        mbar_arrive_expect_tx(&mbar[warp][p], unsigned(na + 1) * kCS * sizeof(double4));
      __syncwarp();
      if (near) {
        const int t = __popc(act & ((1u << lane) - 1u));
        elist[warp][p][t] = make_int2(en.x, en.z);
        bulk_g2s(jst[p][t], p4 + (en.x & kJcMask) * kCS, kCS * sizeof(double4), &mbar[warp][p]);
      }
      if (lane == 31) bulk_g2s(jst[p][kB], p4 + owner * kCS, kCS * sizeof(double4), &mbar[warp][p]);
#else
      // 16-byte cp.async per lane: chunk q of the (na + 1) x 256 contiguous bytes
      // (survivors in order, then the owner), one commit group per batch
      if (near) {
        const int t = __popc(act & ((1u << lane) - 1u));
        elist[warp][p][t] = make_int2(en.x, en.z);
      }
      __syncwarp();
      // lane = (half h = lane >> 4, 16-byte chunk k = lane & 15): survivor t's 256 bytes
      // by the 16 lanes of half t & 1, the owner's by half na & 1
      const unsigned dst = smem_u32(jst[p]) + 16 * (lane & 15);
      const char* src = reinterpret_cast<const char*>(p4) + 16 * (lane & 15);
      for (int t = lane >> 4; t <= na; t += 2) {
        const int jc = t < na ? (elist[warp][p][t].x & kJcMask) : owner;
        cp_async16(dst + (t < na ? t : kB) * 256, src + size_t(jc) * (kCS * sizeof(double4)));
      }
      cp_async_commit();
#endif
      return na;
    };
    auto load_batch = [&](int bt) {
      return (bt < nbt && lane < kB) ? ent[bt * kB + lane] : make_int4(0, 0, 0, 0x7f800000);
    };
    int4 en = load_batch(gw);
    int ci = en.y;  // (lane 0's owner: broadcast below)
    int na = gw < nbt ? stage_batch(0, en) : 0;
    ci = __shfl_sync(full, ci, 0);
    en = load_batch(gw + nw);
    int p = 0;
    for (int bt = gw; bt < nbt; bt += nw, p ^= 1) {
      // stage the next batch into the other buffer, load the one after
      const int ci_next = __shfl_sync(full, en.y, 0);
      const int na_next = bt + nw < nbt ? stage_batch(p ^ 1, en) : 0;
      en = load_batch(bt + 2 * nw);
      if (na) {
#if B2MD_NL_TMA
        mbar_wait(&mbar[warp][p], (phase >> p) & 1u);
        phase ^= 1u << p;
#else
        if (na_next) cp_async_wait<1>(); else cp_async_wait<0>();
#endif
        __syncwarp();  // elist, staged data
        const int ia = ci * kCS + il, ib = ia + 4;
        const bool iva = ia < n, ivb = ib < n;
        const double4 qa = jst[p][kB][il], qb = jst[p][kB][il + 4];
        const double pax = qa.x, pay = qa.y, paz = qa.z, pbx = qb.x, pby = qb.y, pbz = qb.z;
        int sia = 0, sib = 0;
        if constexpr (MULTI_SPECIES) {
          sia = s.sp_slot[roff + (iva ? ia : ci * kCS)];
          sib = s.sp_slot[roff + (ivb ? ib : ci * kCS)];
        }
        double fax = 0, fay = 0, faz = 0, fbx = 0, fby = 0, fbz = 0;
        bool dirty = false;
        for (int t = 0; t < na; ++t) {  // warp-uniform
          const int2 cur = elist[warp][p][t];
          const double4 pj = jst[p][t][jl];
          const int jc = cur.x & kJcMask, code = cur.x >> kJcBits;
          const int j = jc * kCS + jl;
          bool va = true, vb = true;
          if (jc == ci || jc == last_c || ci == last_c) {  // warp-uniform, rare
            const bool vj = j < n, self = jc == ci;
            va = iva && vj && (!self || j > ia);
            vb = ivb && vj && (!self || j > ib);
          }
          double dxa = sub(pax, pj.x), dya = sub(pay, pj.y), dza = sub(paz, pj.z);
          double dxb = sub(pbx, pj.x), dyb = sub(pby, pj.y), dzb = sub(pbz, pj.z);
          if constexpr (WRAPPED) {
            if (code) {  // warp-uniform; per axis: 3 the per-pair image, 1 / 2 one add of -+L
              const float thr = a.thr;
              const double negL = s.mi.negL;
              auto image = [&](int c, double& da, double& db) {
                if (c == 3) {
                  da = min_image_wrapped(da, negL, thr), db = min_image_wrapped(db, negL, thr);
                } else if (c) {
                  const double sh = c == 1 ? negL : L;
                  da = add(da, sh), db = add(db, sh);
                }
              };
              image(code & 3, dxa, dxb);
              image((code >> 2) & 3, dya, dyb);
              image(code >> 4, dza, dzb);
            }
          } else {
            const MinImage mi = s.mi;
            dxa = min_image(dxa, mi), dya = min_image(dya, mi), dza = min_image(dza, mi);
            dxb = min_image(dxb, mi), dyb = min_image(dyb, mi), dzb = min_image(dzb, mi);
          }
          const double r2a = norm2_exact(dxa, dya, dza), r2b = norm2_exact(dxb, dyb, dzb);
          const bool ina = va && r2a < a.rc2, inb = vb && r2b < a.rc2;  // potentials.cpp:161
          if (__ballot_sync(full, ina || inb) == 0u) continue;  // no record: its stamp stays old
          const int sj = MULTI_SPECIES ? (j < n ? s.sp_slot[roff + j] : sia) : 0;
          // both rows' terms in one block (two independent dependency chains)
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
          dirty = true;
          cnt += int(ina) + int(inb);
          // j-side: member jl's 4 row lanes summed in row order through
          // shared memory (lane (jl, c) adds component c), stamped record
          sts_f64<0>(jt_wr + jt_par, gx);
          sts_f64<8>(jt_wr + jt_par, gy);
          sts_f64<16>(jt_wr + jt_par, gz);
          __syncwarp();
          const unsigned jr = jt_rd + jt_par;
          jt_par ^= jt_flip;
          const double res = ((lds_f64<0>(jr) + lds_f64<192>(jr)) + lds_f64<384>(jr)) + lds_f64<576>(jr);
          if (il < 3)
            asm volatile("st.global.f64 [%0], %1;" ::"l"(rec + size_t(cur.y) * kRecP), "d"(res) : "memory");
          if (lane == 0)
            asm volatile("st.global.u32 [%0], %1;" ::"l"(rstamp + cur.y), "r"(epoch) : "memory");
        }
        if (dirty) {
          // the batch's i-side record: rows ia / ib summed over their 8 jl lanes
          // in jl order through the (idle) transpose buffers, laid out
          // [component][lane]; lane (member m, component c) adds and stores
          // one word, lanes 24..31 the members' stamps
          static_assert(2 * 4 * kCS * 3 >= 6 * 32, "transpose buffers hold 6 words per lane");
          __syncwarp();  // the last entry's transpose reads are complete
          sts_f64<0>(jt_wr0 + 8 * lane, fax);
          sts_f64<256>(jt_wr0 + 8 * lane, fay);
          sts_f64<512>(jt_wr0 + 8 * lane, faz);
          sts_f64<768>(jt_wr0 + 8 * lane, fbx);
          sts_f64<1024>(jt_wr0 + 8 * lane, fby);
          sts_f64<1280>(jt_wr0 + 8 * lane, fbz);
          __syncwarp();
          double* q = nl.irec + (size_t(r) * (nl.max_ent / kB) + bt) * kRecD;
          if (lane < 24) {
            const int m = lane / 3, c = lane - 3 * m;
            const unsigned src = jt_wr0 + 256 * ((m >> 2) * 3 + c) + 8 * (m & 3);
            double sum = lds_f64<0>(src);
            sum += lds_f64<32>(src);
            sum += lds_f64<64>(src);
            sum += lds_f64<96>(src);
            sum += lds_f64<128>(src);
            sum += lds_f64<160>(src);
            sum += lds_f64<192>(src);
            sum += lds_f64<224>(src);
            q[4 * m + c] = sum;
          } else {
            q[4 * (lane - 24) + 3] = stamp;
          }
        }
      }
      __syncwarp();  // this buffer's reads are done before it is restaged
      ci = ci_next;
      na = na_next;
    }
  }
  double A12 = warp_sum(B12), A6 = warp_sum(B6);
  if constexpr (!MULTI_SPECIES) {
    A12 *= a.c12;
    A6 *= a.c6;
  }
  const double s1 = -12.0 * A12 + 6.0 * A6;  // sum du_r
  double v[kNumRowScalars] = {A12 - A6, 0.0, 0.0, VDERIV ? s1 : 0.0,
                              VDERIV ? 156.0 * A12 - 42.0 * A6 : 0.0, -s1,
                              warp_sum(double(cnt))};
  // the last CTA (the scalars' ticket) advances the epoch: k_nl_reduce reads
  // the stamps of this one
  if (finalize_scalars<kNumRowScalars>(v, a.cta_part, a.ticket, a.sums, r, 0) && threadIdx.x == 0)
    ctl[kNLEpoch] = epoch + 1;
}

// The fixed-order reduction of the contribution records: one warp per
// cluster c, lane = (record offset q = lane >> 3, member m = lane & 7).  Group
// q = 0 first adds c's batches' i-side records; then c's incoming records --
// a contiguous, receiver-major range in owner order -- are subtracted, record
// t by group t % 4 (32 records' loads in flight per round); the 4 groups are
// combined by a fixed xor tree.  Only records stamped by this evaluation
// count (an entry without a pair in cutoff writes nothing).  Then the fused
// end-of-step kick.  On a stale list the forces were written by the exact
// walk: only the kick.
static __global__ void __launch_bounds__(kNLBuildWarps * 32)
    k_nl_reduce(ForceArgs a, ClusterArgs ca, NListArgs nl) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int q = lane >> 3, m = lane & 7;
  const int r = blockIdx.y;
  const int n = a.s.n, nc = ca.nc;
  const int c = blockIdx.x * kNLBuildWarps + warp;
  if (c >= nc) return;
  const unsigned full = 0xffffffffu;
  const size_t roff = size_t(r) * n;
  const int slot = c * kCS + m;
  const int* ctl = nl.ctl + size_t(r) * kNLCtl;
  // the end-of-step kick's inputs (engine.cpp:131-142, kick_one) are fetched by
  // the 8 member lanes before the record loop, so their (dependent, scattered)
  // round trips overlap the records'
  const bool kicker = q == 0 && slot < n && a.kick_dt > 0.0;
  size_t ke = 0;
  bool kpoint = false, kfrozen = false;
  double kv[3] = {0, 0, 0}, kp[3] = {0, 0, 0}, kw[3] = {0, 0, 0}, kqw = 0, kmass = 1.0;
  if (kicker) {
    ke = roff + ext_of(a.st.pos4[roff + slot]);
    const DevSpecies& sp = a.s.tab->species[a.s.ns == 1 ? 0 : a.s.species_of[ke - roff]];
    kpoint = sp.rotational_dof == 0;
    kmass = sp.total_mass;
    kfrozen = *a.error_mol != 0x7fffffff;
    kv[0] = a.st.vx[ke], kv[1] = a.st.vy[ke], kv[2] = a.st.vz[ke];
    kp[0] = a.st.px[ke], kp[1] = a.st.py[ke], kp[2] = a.st.pz[ke];
    kw[0] = a.st.wx[ke], kw[1] = a.st.wy[ke], kw[2] = a.st.wz[ke];
    kqw = a.st.qw[ke];
  }
  double fx = 0.0, fy = 0.0, fz = 0.0;
  const bool listed = !nl_stale(nl, ctl);
  if (listed) {
    const long long epoch = ctl[kNLEpoch] - 1;  // advanced by the force kernel's last CTA
    const int* eb = nl.ebase + size_t(r) * (nc + 1);
    const double* __restrict__ irec = nl.irec + size_t(r) * (nl.max_ent / kB) * kRecD + 4 * m;
    const double* __restrict__ rec = nl.rec + size_t(r) * nl.max_ent * kRecP + 3 * m;
    const int* __restrict__ rstamp = nl.rstamp + size_t(r) * nl.max_ent;
    // the stamps of the first span are requested before the i-side records
    // are waited for (independent round trips)
    constexpr int kSpan = 256;
    const int i0 = nl.ibase[size_t(r) * (nc + 1) + c], i1 = nl.ibase[size_t(r) * (nc + 1) + c + 1];
    int st[kSpan / 32];
#pragma unroll
    for (int j = 0; j < kSpan / 32; ++j) {
      const int t = i0 + 32 * j + lane;
      st[j] = t < i1 ? rstamp[t] : -1;
    }
    {  // the batches' i-side records: batch b by group (b - first) % 4, 8 in flight
      const int b0 = eb[c] / kB, b1 = eb[c + 1] / kB;
      for (int bb = b0; bb < b1; bb += 8) {
        double4 u[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int b = bb + 4 * h + q;
          u[h] = b < b1 ? *reinterpret_cast<const double4*>(irec + size_t(b) * kRecD)
                        : make_double4(0.0, 0.0, 0.0, __longlong_as_double(-1ll));
        }
#pragma unroll
        for (int h = 0; h < 2; ++h)
          if (__double_as_longlong(u[h].w) == epoch) fx += u[h].x, fy += u[h].y, fz += u[h].z;
      }
    }
    // the stamps of up to 256 slots at once (one round trip) compacted into
    // the warp's list of stamped slots (slot order), then only the stamped
    // payloads: the k-th listed slot by group k % 4, 16 payloads in flight
    __shared__ int slist[kNLBuildWarps][kSpan];
    int* sl = slist[warp];
    for (int s0 = i0; s0 < i1; s0 += kSpan) {
      if (s0 != i0) {
#pragma unroll
        for (int j = 0; j < kSpan / 32; ++j) {
          const int t = s0 + 32 * j + lane;
          st[j] = t < i1 ? rstamp[t] : -1;
        }
      }
      int cnt = 0;
#pragma unroll
      for (int j = 0; j < kSpan / 32; ++j) {
        const bool okl = st[j] == int(epoch);
        const unsigned ok = __ballot_sync(full, okl);
        if (okl) sl[cnt + __popc(ok & ((1u << lane) - 1u))] = s0 + 32 * j + lane;
        cnt += __popc(ok);
      }
      __syncwarp();
      for (int k0 = 0; k0 < cnt; k0 += 32) {
        double px[8], py[8], pz[8];
#pragma unroll
        for (int h = 0; h < 8; ++h) {
          const int k = k0 + 4 * h + q;
          px[h] = py[h] = pz[h] = 0.0;
          if (k < cnt) {
            const double* pr = rec + size_t(sl[k]) * kRecP;
            px[h] = __ldg(pr), py[h] = __ldg(pr + 1), pz[h] = __ldg(pr + 2);
          }
        }
#pragma unroll
        for (int h = 0; h < 8; ++h) fx -= px[h], fy -= py[h], fz -= pz[h];
      }
      __syncwarp();  // the list is rewritten by the next span
    }
#pragma unroll
    for (int o = 8; o < 32; o <<= 1) {
      fx += __shfl_xor_sync(full, fx, o);
      fy += __shfl_xor_sync(full, fy, o);
      fz += __shfl_xor_sync(full, fz, o);
    }
    if (q == 0 && slot < n) {
      const size_t e = roff + ext_of(a.st.pos4[roff + slot]);
      a.st.fx[e] = fx;
      a.st.fy[e] = fy;
      a.st.fz[e] = fz;
    }
  }
  __syncwarp();
  if (kicker && !kfrozen) {
    if (!kpoint) {  // rigid rotor terms: the general kick
      fused_kick(a, ke);
    } else {
      if (!listed) fx = a.st.fx[ke], fy = a.st.fy[ke], fz = a.st.fz[ke];  // the exact walk's rows
      const double cm = __ddiv_rn(mul(0.5, a.kick_dt), kmass);
      const double vx = add(kv[0], mul(fx, cm)), vy = add(kv[1], mul(fy, cm)),
                   vz = add(kv[2], mul(fz, cm));
      a.st.vx[ke] = vx;
      a.st.vy[ke] = vy;
      a.st.vz[ke] = vz;
      const bool ok = isfinite(kp[0]) && isfinite(kp[1]) && isfinite(kp[2]) && isfinite(vx) &&
                      isfinite(vy) && isfinite(vz) && isfinite(kw[0]) && isfinite(kw[1]) &&
                      isfinite(kw[2]) && isfinite(kqw);
      if (!ok) atomicMin(a.error_mol, int(ke));
    }
  }
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
