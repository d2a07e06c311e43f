// b200md device kernels (sm_100a, fp64 CUDA cores).
//
// Per evaluation (ForceField::evaluate, src/parallel.cpp:79-122):
//   k_offsets       site offsets rotate(q, body)            potentials.cpp:106-116
//   k_search        COM minimum-image partner search        potentials.cpp:156-158, 209-213
//                   -> symmetric bit matrix (warp ballots)
//   k_force_single  single-site LJ                          potentials.cpp:148-181
//   k_force_multi   multi-site LJ + charge terms + torques  potentials.cpp:218-283
//   k_ewald_*       reciprocal space                        ewald.cpp:107-180
//   (scalars: per-CTA partials, last-CTA fixed-order total; parallel.cpp:93-95)
// Per step (Engine::step, src/engine.cpp:102-143):
//   k_kick_drift    half kick, drift, NO_SQUISH rotation, wrap, offsets
//   k_kick          half kick + check_finite
//
// Race-free by construction, no floating-point atomics: every molecule's
// force/torque is owned by one warp that walks its row of the symmetric pair
// bit matrix (both i<j and j<i partners, pair terms always evaluated in the
// reference's canonical i<j orientation and negated for the partner) and
// reduces with a fixed xor-shuffle tree.  Scalars are taken from the i<j side
// only and reduced rows -> replica in a fixed order, so repeated runs are
// bit-identical (the reference's fixed-W determinism, parallel.hpp:1-5).
#pragma once

#include "device.cuh"

namespace b2md {

struct StateDev {
  double *px, *py, *pz;
  double *qw, *qx, *qy, *qz;
  double *vx, *vy, *vz;
  double *wx, *wy, *wz;
  double *fx, *fy, *fz;
  double *tx, *ty, *tz;
  double4* off;   // site offsets (x, y, z, -), R * total_sites
  double4* pos4;  // positions (x, y, z, -), R * n: one 32-byte gather per partner
};

struct SysDev {
  int n;            // molecules per replica
  int R;            // replicas
  int total_sites;  // per replica
  int n_pad;        // bit matrix rows per replica
  int words;        // bit matrix words per row
  int ns;
  MinImage mi;
  const int* species_of;  // n
  const int* site_begin;  // n + 1
  const DevTables* tab;
  // spatial order (b2md_ctx::resort): the search, the bit matrix, pos4,
  // fixpos and the site offsets are indexed by slot k; state arrays by the
  // external molecule index perm[k].  All R * n, replica-major.
  const int* perm;     // external index of slot k
  const int* slot_of;  // slot of external molecule i
  const int* sp_slot;  // species of slot k
  const int* sb_slot;  // first site of slot k in slot-ordered site numbering
};

// pos4.w carries the slot's external index (integer bits; never used as a
// double), so a partner gather yields it with the position.
__device__ __forceinline__ double4 pack_pos(double x, double y, double z, int ext) {
  return make_double4(x, y, z, __hiloint2double(0, ext));
}
__device__ __forceinline__ int ext_of(const double4& p) { return __double2loint(p.w); }

// slot-ordered offset index of external molecule m's site `site` (external
// site numbering site_begin[m] + k)
__device__ __forceinline__ int site_slot(const SysDev& s, int r, int m, int site) {
  const size_t ro = size_t(r) * s.n;
  return s.sb_slot[ro + s.slot_of[ro + m]] + (site - s.site_begin[m]);
}

// ------------------------------------------------------------ site offsets
// build_scene (potentials.cpp:106-116): off = rotate(orient, body_pos); a single
// centred site has offset exactly 0.
static __global__ void k_offsets(SysDev s, StateDev st) {
  const int gid = blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= s.n * s.R) return;
  const int r = gid / s.n, i = gid - r * s.n;
  const DevSpecies& sp = s.tab->species[s.ns == 1 ? 0 : s.species_of[i]];
  const int base = r * s.total_sites + s.sb_slot[size_t(r) * s.n + s.slot_of[gid]];
  if (sp.centred) {
    st.off[base] = make_double4(0.0, 0.0, 0.0, 0.0);
    return;
  }
  const double qw = st.qw[gid], qx = st.qx[gid], qy = st.qy[gid], qz = st.qz[gid];
  for (int k = 0; k < sp.n_sites; ++k) {
    const D3 o = rotate_exact(qw, qx, qy, qz, {sp.body[k][0], sp.body[k][1], sp.body[k][2]});
    st.off[base + k] = make_double4(o.x, o.y, o.z, 0.0);
  }
}

// ----------------------------------------------------------- partner search
struct SearchArgs {
  SysDev s;
  const double4* pos4;  // slot-ordered positions (exact fallback)
  uint32_t* mask;               // R * n_pad * words
  const uint32_t* super_tiles;  // (SI << 16) | SJ, this rank's list
  const uint4* fixpos;          // R * n: (round(x 2^32/L), .., .., in-box flag)
  double rc2;                   // single-species COM radius^2
  // certified fixed-point prefilter (single species, rmax < L/2 (1-1e-6))
  int fix_ok;
  double fix_scale;  // 2^32 / L
  uint32_t fix_lo, fix_width;  // 15-bit test (units (L/32768)^2)
  uint32_t fix_lo32, fix_w32;  // 32-bit refinement (units L^2/2^32)
  // tile culling (fixed-point path): skip a 32x32 tile when the bounding arcs
  // of its two molecule blocks are further apart than rmax
  int cull;
  double cull_r2;  // (rmax 2^32 / L)^2 (1 + 1e-6), fixed-point units squared
};

// Branch-free minimum image for |d| < L (both positions wrapped to [0, L)),
// used by the force kernels on pairs the search already accepted.
// shift <=> hi32(|d|) > hi32(L/2), compared on the integer pattern viewed as a
// float (monotone for these magnitudes).  Outside the hi-word bucket of L/2
// the decision equals nearbyint(d/L) != 0 exactly, and d - L*n is formed by
// one correctly rounded DFMA with n = +-1 (exact product) — the reference's
// bits.  Accepted pairs have every component below rmax < L/2 (1-2^-16), so
// they never reach the bucket.
__device__ __forceinline__ double min_image_wrapped(double d, double negL, float thr) {
  const int hi = __double2hiint(d);
  const bool shift = fabsf(__int_as_float(hi)) > thr;
  int sgn_one;  // (hi & 0x80000000) | 0x3ff00000: +-1.0 high word, one LOP3
  asm("lop3.b32 %0, %1, 0x80000000, %2, 0xEA;" : "=r"(sgn_one) : "r"(hi), "r"(0x3ff00000));
  const int nh = shift ? sgn_one : 0;
  return __fma_rn(__hiloint2double(nh, 0), negL, d);
}

// ---- certified fixed-point prefilter
// Positions in [0, L) are mapped to u = round(x 2^32 / L) (uint32).  The
// wrapping difference u_i - u_j read as int32 IS the minimum image (mod 2^32
// == mod L); its top 15 bits d = (u_i - u_j) >> 17 (arithmetic) are squared
// with full-rate 32-bit IMADs: r2_fix = dx^2 + dy^2 + dz^2 approximates
// r^2 (32768/L)^2 with |error| <= sum (2|d| + 1) (floor of each component),
// bounded on the host by K from rmax; the reference's own fp64 rounding of r^2
// is < 1e-3 units.  With t = r2_fix - (floor(rmax^2 (65536/L)^2) - K):
//   t <  0           => the reference passes,
//   t >= W = 2K + 2  => the reference fails,
// and the candidates with 0 <= t < W (~2e-4 of all) are re-decided with the
// exact fp64 test.  Near |dx| = L/2 the integer wrap may pick the other image,
// but then |d| ~ 2^14 for either image and, because rmax < L/2 (1 - 1e-3),
// the pair fails both ways.  The pass bits are the reference's bits.
//
// Each lane accumulates its own pass bits over the 32 i rows (the L word of
// its j); the U words (row i over 32 j) are one warp bit-transpose per tile.

// 32x32 bit transpose across a warp: lane k holds row k on entry and column k
// on exit (block-recursive swap of off-diagonal halves, 5 shuffle stages).
__device__ __forceinline__ uint32_t warp_transpose32(uint32_t x, int lane) {
  uint32_t m = 0x0000ffffu;
#pragma unroll
  for (int j = 16; j != 0; j >>= 1, m ^= (m << j)) {
    const uint32_t y = __shfl_xor_sync(0xffffffffu, x, j);
    x = (lane & j) ? ((x & ~m) | ((y & ~m) >> j)) : ((x & m) | ((y & m) << j));
  }
  return x;
}

// t = r2_fix - lo (signed; 15-bit components: r2_fix <= 3 * 2^28 < 2^31, no overflow)
__device__ __forceinline__ int fix_t(uint4 pi, uint32_t xj, uint32_t yj, uint32_t zj, int neglo) {
  const int dx = int(pi.x - xj) >> 17, dy = int(pi.y - yj) >> 17, dz = int(pi.z - zj) >> 17;
  return dx * dx + dy * dy + dz * dz + neglo;
}

// 32 i-rows (local tile row at `ib`) x JB column tiles c0.. : U words (row
// ib+ii, columns c0..) to wu, L words to wl.
// Exact decision of one band candidate: the 32-bit fixed-point distance
// (sum hi32(d^2), |error| <= 6 units of L^2/2^32) settles all but ~1e-7 of
// them; the rest take the reference's fp64 test.
struct FixRefine {
  uint32_t lo32, w32;  // pass if r2_32 < lo32, fail if r2_32 >= lo32 + w32
  double rc2;
};

__device__ __forceinline__ bool refine_pair(uint4 pi, uint4 pj, int ig, int jg,
                                         const double4* __restrict__ gp, const FixRefine& f,
                                         const MinImage& mi) {
  const int dx = int(pi.x - pj.x), dy = int(pi.y - pj.y), dz = int(pi.z - pj.z);
  const uint32_t r2 =
      uint32_t(__mulhi(dx, dx)) + uint32_t(__mulhi(dy, dy)) + uint32_t(__mulhi(dz, dz));
  if (r2 < f.lo32) return true;
  if (r2 - f.lo32 >= f.w32) return false;
  const double4 a = gp[ig], b = gp[jg];
  const double ex = min_image(sub(a.x, b.x), mi);
  const double ey = min_image(sub(a.y, b.y), mi);
  const double ez = min_image(sub(a.z, b.z), mi);
  return norm2_exact(ex, ey, ez) < f.rc2;
}

// 32 i-rows (local tile row at `ib`) x JB column tiles c0.. : U words (row
// ib+ii, columns c0..) to wu, L words to wl.
// Column tiles c0 and (JB == 2) c1, not necessarily adjacent.
template <int JB, bool DIAG, bool PARTIAL_I>
__device__ __forceinline__ void search_tile_fix(
    const uint4* __restrict__ siu, const uint4* __restrict__ sju, const double4* __restrict__ gp,
    int ig0, int jg0, int ib, int c0, int c1, int I, int lane, int ST, int ilim, int jlim,
    int neglo, int width, const FixRefine& f, const MinImage& mi, uint32_t* wu, uint32_t* wl) {
  uint32_t xj[JB], yj[JB], zj[JB], lw[JB], bw[JB];
  int nl[JB];
  auto col = [&](int b) { return b == 0 ? c0 : c1; };
#pragma unroll
  for (int b = 0; b < JB; ++b) {
    const int jl = col(b) * 32 + lane;
    const uint4 pj = sju[jl];
    xj[b] = pj.x;
    yj[b] = pj.y;
    zj[b] = pj.z;
    nl[b] = jl < jlim ? neglo : (1 << 30);  // invalid j: t > W always
    lw[b] = 0u;
    bw[b] = 0u;
  }
  // rows are visited from ii = 31 down to 0 and bits are shifted in at the
  // bottom, so bit ii ends up at position ii: lw = [t < 0] (pass), bw =
  // [t < W] (pass or band).  Diagonal / partial-tile masks are applied after.
#pragma unroll 8
  for (int k = 0; k < 32; ++k) {
    const uint4 pi = siu[ib + 31 - k];  // (x, y, z, -)
#pragma unroll
    for (int b = 0; b < JB; ++b) {
      const int t = fix_t(pi, xj[b], yj[b], zj[b], nl[b]);
      lw[b] = lw[b] + lw[b] + (uint32_t(t) >> 31);
      bw[b] = bw[b] + bw[b] + (uint32_t(t - width) >> 31);
    }
  }
  uint32_t valid = 0xffffffffu;
  if (PARTIAL_I) valid = ilim <= 0 ? 0u : (ilim >= 32 ? 0xffffffffu : ((1u << ilim) - 1u));
#pragma unroll
  for (int b = 0; b < JB; ++b) {
    uint32_t m = valid;
    if (DIAG && b == 0) m &= (1u << lane) - 1u;  // j = lane > i = ii only
    lw[b] &= m;
    // rare: band members are decided exactly, lane by lane (no collectives)
    uint32_t band = bw[b] & ~lw[b] & m;
    if (band) {
      const int jl = col(b) * 32 + lane;
      const uint4 pj = sju[jl];
      while (band) {
        const int ii = __ffs(band) - 1;
        band &= band - 1u;
        if (refine_pair(siu[ib + ii], pj, ig0 + ib + ii, jg0 + jl, gp, f, mi))
          lw[b] |= 1u << ii;
      }
    }
  }
#pragma unroll
  for (int b = 0; b < JB; ++b) {
    wl[(col(b) * 32 + lane) * ST + I] = lw[b];
    wu[(ib + lane) * ST + col(b)] = warp_transpose32(lw[b], lane);
  }
}

// Bounding arc of 32 fixed-point coordinates on the periodic axis (2^32 =
// L): anchored at lane 0, the wrapping int32 offsets of all lanes lie in
// [mn, mx], so every point is within h of the centre c.  Valid for any
// spread (a block spanning the box gets an arc of ~the whole circle).
__device__ __forceinline__ void bounding_arc(uint32_t u, uint32_t& c, uint32_t& h) {
  const uint32_t anchor = __shfl_sync(0xffffffffu, u, 0);
  const int off = int(u - anchor);
  const int mn = __reduce_min_sync(0xffffffffu, off);
  const int mx = __reduce_max_sync(0xffffffffu, off);
  c = anchor + uint32_t(int((static_cast<long long>(mn) + mx) >> 1));
  h = uint32_t((static_cast<long long>(mx) - mn + 1) >> 1) + 1u;
}

// Conservative "no pair of these two blocks is within rmax": per axis the
// circular gap between the arcs, less 2 units for the rounding of u.
__device__ __forceinline__ bool tiles_apart(uint4 ca, uint4 ha, uint4 cb, uint4 hb, double lim) {
  auto gap = [](uint32_t x, uint32_t y, uint32_t hx, uint32_t hy) {
    const long long d = llabs(static_cast<long long>(int(x - y)));
    const long long g = d - static_cast<long long>(hx) - static_cast<long long>(hy) - 2;
    return g > 0 ? double(g) : 0.0;
  };
  const double gx = gap(ca.x, cb.x, ha.x, hb.x);
  const double gy = gap(ca.y, cb.y, ha.y, hb.y);
  const double gz = gap(ca.z, cb.z, ha.z, hb.z);
  return gx * gx + gy * gy + gz * gz > lim;
}

// One CTA = one super-tile (SI, SJ), SI <= SJ, of ST x ST 32-molecule tiles;
// warp w owns tile row I = SI*ST + w.  Lane <-> j (register), i broadcast from
// shared memory.  The warp ballot of a fixed i over 32 j is the U word (row
// i, column tile J); the warp transpose of a tile's 32 U words gives the L
// words (row j, column tile I).  Words are staged in shared memory and stored
// as whole 32-byte sectors of the row-major bit matrix M[r][row][word].
// Certified fixed-point path for single-species, in-box tiles; the exact
// generic fp64 path (any position, mixtures, rmax >= L/2) otherwise.
template <int ST, bool MULTI, int RS = 1>
__global__ void __launch_bounds__(ST * 32 * RS, (ST * RS >= 8 ? 4 : 8)) k_search(SearchArgs a) {
  // RS > 1 (generic path only): RS warps share each tile row, 32 / RS rows
  // each -- small systems have few tiles, and a lone warp per tile is
  // latency-bound on the exact fp64 chain
  constexpr int T = ST * 32;
  __shared__ uint4 ui[T], uj[T];
  __shared__ int ispec[MULTI ? T : 1], jspec[MULTI ? T : 1];
  __shared__ double rmax2_s[MULTI ? kMaxSpecies * kMaxSpecies : 1];
  __shared__ __align__(16) uint32_t wu[T * ST];
  __shared__ __align__(16) uint32_t wl[T * ST];
  __shared__ uint4 arc_c[2 * ST], arc_h[2 * ST];  // i tiles [0, ST), j tiles [ST, 2 ST)

  const SysDev& s = a.s;
  const int r = blockIdx.y;
  const uint32_t code = a.super_tiles[blockIdx.x];
  const int SI = int(code >> 16), SJ = int(code & 0xffffu);
  const bool diag = SI == SJ;
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int n = s.n;
  const int ibase = SI * T, jbase = SJ * T;
  const size_t roff = size_t(r) * n;
  const double4* __restrict__ gp = a.pos4 + roff;

  bool inbox = true;
  if (tid < T) {
    const int i = ibase + tid, j = jbase + tid;
    // fixed-point positions + in-box flag, written by the integrator
    // (k_kick_drift) or k_fix_positions
    const uint4 fi = i < n ? a.fixpos[roff + i] : make_uint4(0u, 0u, 0u, 1u);
    const uint4 fj = j < n ? a.fixpos[roff + j] : make_uint4(0u, 0u, 0u, 1u);
    ui[tid] = fi;
    uj[tid] = fj;
    inbox = fi.w != 0u && fj.w != 0u;
    if constexpr (MULTI) {
      ispec[tid] = i < n ? s.sp_slot[roff + i] : 0;
      jspec[tid] = j < n ? s.sp_slot[roff + j] : 0;
      for (int k = tid; k < s.ns * s.ns; k += T) rmax2_s[k] = s.tab->pair[k].rmax2;
    }
    if (diag || !a.fix_ok || MULTI) {  // only partially written there: merge needs zeros
#pragma unroll
      for (int c = 0; c < ST; ++c) {
        wu[tid * ST + c] = 0u;
        wl[tid * ST + c] = 0u;
      }
    }
  }
  const bool boxed = __syncthreads_and(inbox);

  const int I = warp % ST;  // local tile row
  const int part = warp / ST;
  const int ib = I * 32;
  const int ilim = n - (ibase + ib);
  if (RS == 1 && boxed && a.fix_ok && !MULTI) {
    const int jlim = n - jbase;
    const int neglo = -int(a.fix_lo);
    const int wd = int(a.fix_width);
    FixRefine refine;
    refine.lo32 = a.fix_lo32;
    refine.w32 = a.fix_w32;
    refine.rc2 = a.rc2;
    // tiles kept after culling: bit c = column tile c of this warp's tile row
    uint32_t keep = (1u << ST) - 1u;
    if (a.cull) {
      {
        const uint4 p = ui[ib + lane];
        uint4 c, h;
        bounding_arc(p.x, c.x, h.x);
        bounding_arc(p.y, c.y, h.y);
        bounding_arc(p.z, c.z, h.z);
        const uint4 q = uj[ib + lane];
        uint4 cj, hj;
        bounding_arc(q.x, cj.x, hj.x);
        bounding_arc(q.y, cj.y, hj.y);
        bounding_arc(q.z, cj.z, hj.z);
        if (lane == 0) {
          arc_c[I] = c;
          arc_h[I] = h;
          arc_c[ST + I] = cj;
          arc_h[ST + I] = hj;
        }
      }
      __syncthreads();
      uint32_t k = 0;
      for (int c = 0; c < ST; ++c) {
        if (!tiles_apart(arc_c[I], arc_h[I], arc_c[ST + c], arc_h[ST + c], a.cull_r2)) {
          k |= 1u << c;
        } else {  // no pairs: zero words (the non-diagonal path does not pre-zero)
          wu[(ib + lane) * ST + c] = 0u;
          wl[(c * 32 + lane) * ST + I] = 0u;
        }
      }
      keep = __shfl_sync(0xffffffffu, k, 0);
    }
    if (!diag && n - ibase >= T) {
      // hot path (all ST tile rows full): each tile row's kept column tiles
      // are paired into jobs and the CTA's jobs are dealt to the warps
      // round-robin, so culling leaves no warp idle at the final barrier.
      // A tile's words have fixed places in wu / wl: any warp may do it.
      __shared__ int njob_s[ST];
      __shared__ uint32_t jobs[ST * ((ST + 1) / 2)];
      const int nj = (__popc(keep) + 1) >> 1;
      if (lane == 0) njob_s[I] = nj;
      __syncthreads();
      int base = 0, total = 0;
      for (int w = 0; w < ST; ++w) {
        base += w < I ? njob_s[w] : 0;
        total += njob_s[w];
      }
      if (lane == 0) {
        uint32_t k = keep;
        for (int q = 0; q < nj; ++q) {
          const uint32_t c0 = __ffs(k) - 1;
          k &= k - 1u;
          const uint32_t c1 = k ? uint32_t(__ffs(k) - 1) : 0xffu;
          if (k) k &= k - 1u;
          jobs[base + q] = (uint32_t(I) << 16) | (c0 << 8) | c1;
        }
      }
      __syncthreads();
#pragma unroll 1
      for (int q = warp; q < total; q += ST) {
        const uint32_t jb = jobs[q];
        const int Iq = int(jb >> 16), c0 = int((jb >> 8) & 0xffu), c1 = int(jb & 0xffu);
        if (ST >= 2 && c1 != 0xff)
          search_tile_fix<(ST >= 2 ? 2 : 1), false, false>(ui, uj, gp, ibase, jbase,
                                                           Iq * 32, c0, c1, Iq, lane, ST, 32,
                                                           jlim, neglo, wd, refine, s.mi, wu, wl);
        else
          search_tile_fix<1, false, false>(ui, uj, gp, ibase, jbase, Iq * 32, c0, c0,
                                           Iq, lane, ST, 32, jlim, neglo, wd, refine, s.mi, wu,
                                           wl);
      }
    } else if (diag && ilim >= 32) {
      search_tile_fix<1, true, false>(ui, uj, gp, ibase, jbase, ib, I, I, I, lane,
                                      ST, ilim, jlim, neglo, wd, refine, s.mi, wu, wl);
      for (int c = I + 1; c < ST; ++c)
        if (keep >> c & 1u)
          search_tile_fix<1, false, false>(ui, uj, gp, ibase, jbase, ib, c, c, I,
                                           lane, ST, ilim, jlim, neglo, wd, refine, s.mi, wu, wl);
    } else {  // last, partial tile row (arcs include the padding: conservative)
      for (int c = diag ? I : 0; c < ST; ++c) {
        if (diag && c == I)
          search_tile_fix<1, true, true>(ui, uj, gp, ibase, jbase, ib, c, c, I,
                                         lane, ST, ilim, jlim, neglo, wd, refine, s.mi, wu, wl);
        else if (keep >> c & 1u)
          search_tile_fix<1, false, true>(ui, uj, gp, ibase, jbase, ib, c, c, I,
                                          lane, ST, ilim, jlim, neglo, wd, refine, s.mi, wu, wl);
      }
    }
  } else {
    // generic path: exact minimum image for any input, partial tiles, mixtures
    const MinImage mi = s.mi;
    for (int c = diag ? I : 0; c < ST; ++c) {
      const int jl = c * 32 + lane;
      const bool jvalid = jbase + jl < n;
      const int jg = jvalid ? jbase + jl : 0;
      const double4 pj = gp[jg];
      const double xj = pj.x, yj = pj.y, zj = pj.z;
      const int sj = MULTI ? jspec[jl] : 0;
      const bool diag_tile = diag && c == I;
      for (int ii = part * (32 / RS); ii < (part + 1) * (32 / RS); ++ii) {
        const int il = ib + ii;
        const int ig = ii < ilim ? ibase + il : 0;
        const double4 pi = gp[ig];
        const double dx = min_image(sub(pi.x, xj), mi);
        const double dy = min_image(sub(pi.y, yj), mi);
        const double dz = min_image(sub(pi.z, zj), mi);
        const double r2 = norm2_exact(dx, dy, dz);
        double lim;
        if constexpr (MULTI)
          lim = rmax2_s[ispec[il] * s.ns + sj];
        else
          lim = a.rc2;
        bool pass = r2 < lim && jvalid && ii < ilim;
        if (diag_tile) pass = pass && lane > ii;
        const uint32_t b = __ballot_sync(0xffffffffu, pass);
        if (lane == 0) wu[(ib + ii) * ST + c] = b;
      }
      if constexpr (RS == 1) {
        __syncwarp();
        wl[(c * 32 + lane) * ST + I] = warp_transpose32(wu[(ib + lane) * ST + c], lane);
      }
    }
    if constexpr (RS > 1) {  // the tile's rows come from RS warps
      __syncthreads();
      if (part == 0)
        for (int c = diag ? I : 0; c < ST; ++c)
          wl[(c * 32 + lane) * ST + I] = warp_transpose32(wu[(ib + lane) * ST + c], lane);
    }
  }
  __syncthreads();
  if (tid >= T) return;

  // store: rows of tile-row block SI get columns SJ*ST.. (wu); rows of block SJ
  // get columns SI*ST.. (wl).  Diagonal super-tiles merge both.
  uint32_t* M = a.mask + size_t(r) * s.n_pad * s.words;
  const int row = tid;
  if (diag) {
    uint32_t* dst = M + size_t(ibase + row) * s.words + SI * ST;
#pragma unroll
    for (int c = 0; c < ST; ++c) dst[c] = wu[row * ST + c] | wl[row * ST + c];
  } else {
    uint32_t* du = M + size_t(ibase + row) * s.words + SJ * ST;
    uint32_t* dl = M + size_t(jbase + row) * s.words + SI * ST;
    if constexpr (ST % 4 == 0) {
#pragma unroll
      for (int c = 0; c < ST; c += 4) {
        *reinterpret_cast<uint4*>(du + c) = *reinterpret_cast<const uint4*>(&wu[row * ST + c]);
        *reinterpret_cast<uint4*>(dl + c) = *reinterpret_cast<const uint4*>(&wl[row * ST + c]);
      }
    } else {
#pragma unroll
      for (int c = 0; c < ST; ++c) {
        du[c] = wu[row * ST + c];
        dl[c] = wl[row * ST + c];
      }
    }
  }
}

// ------------------------------------------------- partner enumeration
// Walks the set bits of one bit-matrix row (the molecule's partners j, both
// j<i and j>i) in chunks of 32 words: each lane loads one word, a ballot
// skips empty chunks, a warp bit-transpose + prefix sum of popcounts
// compacts the chunk's partners into a shared-memory queue (ballot /
// prefix-sum compaction), full batches of 32 partners are evaluated
// lane-parallel by `body(j)` (no collectives inside) and the partial batch is
// carried to the next chunk.  Partner order, hence the accumulation order, is
// a fixed function of the bit matrix: results are reproducible.
constexpr int kChunkWords = 32;
constexpr int kForceWarps = 8;  // warps per CTA of the partner walks
constexpr double kErfcxMax = 6.0;
constexpr int kErfcxDeg = 18;

__device__ __forceinline__ int warp_incl_scan(int v, int lane) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += t;
  }
  return v;
}

// Queue capacity per warp: a carried partial batch (< 32) + one chunk (<= 1024).
constexpr int kQueue = kChunkWords * 32 + 32;

// Row split (part, nparts > 1): the nparts warps of a row all expand it and
// warp `part` evaluates the batches with index = part mod nparts, so short
// rows of small systems still occupy the GPU; each batch is evaluated by
// exactly one warp.
template <bool DUAL = true, typename Body>
__device__ __forceinline__ void for_each_partner(const uint32_t* __restrict__ row, int words,
                                                 int lane, int* __restrict__ q, Body&& body,
                                                 int part = 0, int nparts = 1) {
  int fill = 0;  // warp-uniform queue length carried between chunks
  int bk = 0;    // batches of this row so far (row split)
  const int nchunks = (words + kChunkWords - 1) / kChunkWords;
  for (int g0 = 0; g0 < nchunks; g0 += 64) {
    // Occupancy pass over (up to) 64 chunks: the words are loaded with eight
    // loads in flight and OR-reduced per chunk, so empty chunks (most of a
    // short-cutoff row) cost no dependent memory round trip in the walk.
    const int gn = min(64, nchunks - g0);
    uint64_t cm = 0;
#pragma unroll 8
    for (int k = 0; k < gn; ++k) {
      const int w = (g0 + k) * kChunkWords + lane;
      const uint32_t m = w < words ? __ldg(row + w) : 0u;
      if (__reduce_or_sync(0xffffffffu, m)) cm |= 1ull << k;
    }
    // nonempty chunks; the next one's word is loaded (L1) before the
    // current one is expanded
    uint32_t next = 0;
    if (cm) {
      const int w = (g0 + __ffsll(static_cast<long long>(cm)) - 1) * kChunkWords + lane;
      next = w < words ? __ldg(row + w) : 0u;
    }
    while (cm) {
      const int c = __ffsll(static_cast<long long>(cm)) - 1;
      cm &= cm - 1;
      const int w0 = (g0 + c) * kChunkWords;
      const uint32_t m = next;
      if (cm) {
        const int w = (g0 + __ffsll(static_cast<long long>(cm)) - 1) * kChunkWords + lane;
        next = w < words ? __ldg(row + w) : 0u;
      }
      const int c0 = __popc(m);
      const int total = int(__reduce_add_sync(0xffffffffu, unsigned(c0)));
      const int mx = int(__reduce_max_sync(0xffffffffu, unsigned(c0)));
      if (mx * 32 > 2 * total + 128) {
        // bits concentrated in a few words (clustered partner runs): a 32x32
        // bit transpose gives lane b bit b of every word, i.e. partners
        // j = (w0 + k) * 32 + b, which spreads each run across lanes
        uint32_t t = warp_transpose32(m, lane);
        const int cc = __popc(t);
        int off = fill + warp_incl_scan(cc, lane) - cc;
        while (t) {
          const int k = __ffs(t) - 1;
          t &= t - 1u;
          q[off++] = (w0 + k) * 32 + lane;
        }
      } else {
        // balanced chunk: lane k expands word k (ascending j, gather-friendly)
        uint32_t t = m;
        int off = fill + warp_incl_scan(c0, lane) - c0;
        while (t) {
          q[off++] = (w0 + lane) * 32 + __ffs(t) - 1;
          t &= t - 1u;
        }
      }
      fill += total;
      __syncwarp();
      int e = 0;
      if (nparts > 1) {
        for (; e + 32 <= fill; e += 32, ++bk)
          if (bk % nparts == part) body(q[e + lane]);
      } else {
        if (DUAL)
          for (; e + 64 <= fill; e += 64) {  // two full batches: both gathers in flight
            const int j0 = q[e + lane], j1 = q[e + 32 + lane];
            body(j0);
            body(j1);
          }
        else
          for (; e + 64 <= fill; e += 32) body(q[e + lane]);
        if (e + 32 <= fill) {
          body(q[e + lane]);
          e += 32;
        }
      }
      const int rem = fill - e;  // carry the partial batch
      const int v = lane < rem ? q[e + lane] : 0;
      __syncwarp();
      if (lane < rem) q[lane] = v;
      __syncwarp();
      fill = rem;
    }
  }
  if (lane < fill && bk % nparts == part) body(q[lane]);
}

// Row-split epilogue: the parts of row group `rl` are summed in part order
// (deterministic) by part 0; returns true on the lane that owns the totals.
template <int NV>
__device__ __forceinline__ bool combine_parts(double (&v)[NV], double (*slab)[NV], int warp,
                                              int lane, int S) {
  if (lane == 0)
    for (int k = 0; k < NV; ++k) slab[warp][k] = v[k];
  __syncthreads();
  const bool owner = warp % S == 0 && lane == 0;
  if (owner)
    for (int k = 0; k < NV; ++k) {
      double t = slab[warp][k];
      for (int p = 1; p < S; ++p) t += slab[warp + p][k];
      v[k] = t;
    }
  __syncthreads();  // the slab is rewritten by the next row group
  return owner;
}

__device__ __forceinline__ double rcp_nr(double x);
// erfcx(x) for 0 <= x < kErfcxMax: the degree-kErfcxDeg interpolant in
// u = 2 (t - t_lo) / (1 - t_lo) - 1, t = 1 / (1 + x/2), by Horner's rule on its
// monomial coefficients c (from the Chebyshev series, on the host);
// u_scale = 2 / (1 - t_lo), the reciprocal by rcp_nr (no IEEE-division slow paths)
__device__ __forceinline__ double erfcx_cheb(double x, const double* c, double t_lo, double u_scale) {
  const double t = rcp_nr(fma(0.5, x, 1.0));
  const double u = fma(t - t_lo, u_scale, -1.0);
  double p = c[kErfcxDeg];
#pragma unroll
  for (int j = kErfcxDeg - 1; j >= 0; --j) p = fma(p, u, c[j]);
  return p;
}

// 1/x to ~1 ulp without the IEEE-division slow path: hardware reciprocal
// seed (relative error e ~ 2^-20) + one third-order step r (1 + e + e^2),
// error e^3 ~ 2^-60 -- three dependent DFMAs instead of the four of two
// Newton steps (force arithmetic; tolerance 1e-10).
__device__ __forceinline__ double rcp_nr(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  const double e = fma(-x, r, 1.0);
  return fma(r, fma(e, e, e), r);
}

// 1/sqrt(x) to ~1 ulp: hardware seed (relative error ~2^-20) + one third-order
// step y (1 + e/2 + 3 e^2/8), e = 1 - x y^2 (charge terms: r = x y, 1/r^2 = y^2).
__device__ __forceinline__ double rsqrt_nr(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double e = fma(-x, y * y, 1.0);
  return fma(y, e * fma(0.375, e, 0.5), y);
}

// Per-CTA scalar partials -> one fixed-order total per replica, done by the
// last CTA to finish (integer ticket; no floating-point atomics).
// Returns true on the last CTA (all its threads), false elsewhere.
template <int NS>
__device__ bool finalize_scalars(const double* v /* NS values, valid on lane 0 of each warp */,
                                 double* cta_part, unsigned* ticket, double* sums, int r,
                                 int sum_offset) {
  __shared__ double red[kForceWarps][NS];
  __shared__ bool last;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nw = blockDim.x >> 5;
  const int nblk = gridDim.x;
  if (lane == 0)
    for (int k = 0; k < NS; ++k) red[warp][k] = v[k];
  __syncthreads();
  if (threadIdx.x < NS) {
    double t = 0.0;
    for (int w = 0; w < nw; ++w) t += red[w][threadIdx.x];
    cta_part[(size_t(r) * NS + threadIdx.x) * nblk + blockIdx.x] = t;
    // release: the writers' stores precede the ticket (only they fence: a
    // fence also waits for the thread's other outstanding stores -- the
    // walks' record / force stores -- which the kernel boundary orders)
    __threadfence();
  }
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(&ticket[r], 1u) == unsigned(nblk - 1);
  __syncthreads();
  if (!last) return false;
  __threadfence();
  // fixed-order totals: every thread sums its strided slice of all NS
  // columns at once (__ldcg: L2, not a possibly stale L1; all loads in
  // flight together), then one fixed shuffle tree and warp-order sum
  double t[NS];
#pragma unroll
  for (int k = 0; k < NS; ++k) t[k] = 0.0;
  const double* base = cta_part + size_t(r) * NS * nblk;
#pragma unroll 2
  for (int b = threadIdx.x; b < nblk; b += blockDim.x) {
#pragma unroll
    for (int k = 0; k < NS; ++k) t[k] += __ldcg(base + size_t(k) * nblk + b);
  }
#pragma unroll
  for (int k = 0; k < NS; ++k) t[k] = warp_sum(t[k]);
  __syncthreads();  // red is reused
  if (lane == 0)
#pragma unroll
    for (int k = 0; k < NS; ++k) red[warp][k] = t[k];
  __syncthreads();
  if (threadIdx.x < NS) {
    double tt = 0.0;
    for (int w = 0; w < nw; ++w) tt += red[w][threadIdx.x];
    sums[size_t(r) * kNumSums + sum_offset + threadIdx.x] = tt;
  }
  if (threadIdx.x == 0) ticket[r] = 0u;  // re-armed for the next launch / graph replay
  return true;
}

// ------------------------------------------------------- single-site forces
// evaluate_range_single_site (potentials.cpp:148-181).  One warp per molecule
// row (grid-stride over rows), partners from the bit matrix.  With
// R = min_image(com_i - com_j) the reference's canonical vector is +-R with
// identical magnitude bits (IEEE subtraction and round-half-even are
// sign-symmetric), so the force on row i is always fs * R.  Energy, virial
// and s1/s2 are taken on the i < j side only.
struct ForceArgs {
  SysDev s;
  StateDev st;
  const uint32_t* mask;
  double* cta_part;  // R * kNumRowScalars * gridDim.x
  unsigned* ticket;  // R
  double* sums;      // R * kNumSums
  double c12, c6;    // single-species LJ term (PairTable lj[0])
  double c12x12, c6x6;  // 12 c12, 6 c6 (kernel constants, not registers)
  double rc2;
  double alpha, two_alpha_over_sqrt_pi;
  double rf_r3inv, rf_shift;
  // erfcx(x) = erfc(x) exp(x^2) on [0, kErfcxMax] as a polynomial (monomial form) in
  // t = 1 / (1 + x/2) (host-interpolated, ~1e-14 relative): the Ewald
  // real-space term then shares exp(-x^2) with its force factor
  double erfcx_c[19];
  double erfcx_tlo, erfcx_uscale;  // t_lo = 1 / (1 + kErfcxMax / 2), 2 / (1 - t_lo)
  int vderiv;
  float thr;  // hi32(L/2) as float (min_image_wrapped)
  // fused end-of-step half kick (kick_one) in the row epilogue: dt > 0 when
  // the forces are complete after this kernel (no Ewald term, no all-reduce)
  double kick_dt;
  double rmax2;  // single-species COM radius^2 (rc + 2 reach)^2 (potentials.cpp:211-212)
  int* error_mol;
  int split;  // warps per row (row-split kernels)
};

struct StepArgs;
__device__ __forceinline__ void fused_kick(const ForceArgs& a, size_t gid);


template <bool MULTI_SPECIES, bool WRAPPED, bool SPLIT>
__global__ void __launch_bounds__(kForceWarps * 32) k_force_single(ForceArgs a) {
  __shared__ int plist[kForceWarps][kQueue];
  const SysDev& s = a.s;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int r = blockIdx.y;
  const size_t roff = size_t(r) * s.n;
  const double4* __restrict__ p4 = a.st.pos4 + roff;
  const MinImage mi = s.mi;
  const float thr = a.thr;
  auto mimg = [&](double d) {
    return WRAPPED ? min_image_wrapped(d, mi.negL, thr) : min_image(d, mi);
  };
  double u = 0, vir = 0, s1 = 0, s2 = 0, cnt = 0;
  const int wpb = blockDim.x >> 5;  // warps per CTA (<= kForceWarps; fewer for small systems)
  // row groups: S warps per row when SPLIT (S divides the CTA's warps)
  const int S = SPLIT ? a.split : 1;
  const int rpc = wpb / S, rl = warp / S, part = warp % S;
  __shared__ double slab[SPLIT ? kForceWarps : 1][3];
  for (int base = blockIdx.x * rpc;; base += gridDim.x * rpc) {
    if (SPLIT ? base >= s.n : base + rl >= s.n) break;  // CTA-uniform when SPLIT
    const int i_ = base + rl;
    const bool has = i_ < s.n;
    const int i = has ? i_ : 0;
    const double4 pi = p4[i];  // i, j: slots (single-site terms are symmetric)
    const int si = MULTI_SPECIES ? s.sp_slot[roff + i] : 0;
    double fx = 0, fy = 0, fz = 0;
    const uint32_t* row = a.mask + (size_t(r) * s.n_pad + i) * s.words;
    if (has)
    for_each_partner(row, s.words, lane, plist[warp], [&](int j) {
      const double4 pj = p4[j];
      const double dx = mimg(sub(pi.x, pj.x));
      const double dy = mimg(sub(pi.y, pj.y));
      const double dz = mimg(sub(pi.z, pj.z));
      const double r2 = norm2_exact(dx, dy, dz);
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
      if (i < j) {
        u += a12 - a6;
        vir += dx * gx + dy * gy + dz * gz;
        s1 += du_r;
        s2 += 156.0 * a12 - 42.0 * a6;
        cnt += 1.0;
      }
    }, part, S);
    fx = warp_sum(fx);
    fy = warp_sum(fy);
    fz = warp_sum(fz);
    bool own = lane == 0 && has;
    if constexpr (SPLIT) {
      double vv[3] = {fx, fy, fz};
      own = combine_parts<3>(vv, slab, warp, lane, S) && has;
      fx = vv[0];
      fy = vv[1];
      fz = vv[2];
    }
    if (own) {
      const size_t e = roff + ext_of(pi);
      a.st.fx[e] = fx;
      a.st.fy[e] = fy;
      a.st.fz[e] = fz;
      if (a.kick_dt > 0.0) fused_kick(a, e);
    }
  }
  double v[kNumRowScalars] = {warp_sum(u), 0.0, 0.0, a.vderiv ? warp_sum(s1) : 0.0,
                              a.vderiv ? warp_sum(s2) : 0.0, warp_sum(vir), warp_sum(cnt)};
  finalize_scalars<kNumRowScalars>(v, a.cta_part, a.ticket, a.sums, r, 0);
}

// -------------------------------------------------------- multi-site forces
// evaluate_pair_range general path (potentials.cpp:204-292): the COM pair
// passed the search; LJ terms (218-242) and charge terms (244-283).  With
// R = min_image(com_i - com_j) the site vector from row i's side is
//   i < j:  rv = (R + d_i,a) - d_j,b            (the reference's own bits)
//   i > j:  rv = (R - d_j,a) + d_i,b  = -rv_ref (bit-exact negation)
// so the site cutoff r2 < rc2 is decided on the reference's bits either way;
// force on i is fs*rv and torque d_i x (fs*rv).
// METHOD: 0 none, 1 reaction field, 2 ewald real space.
template <int METHOD, bool WRAPPED, bool SPLIT>
__global__ void __launch_bounds__(kForceWarps * 32) k_force_multi(ForceArgs a) {
  __shared__ int plist[kForceWarps][kQueue];
  const SysDev& s = a.s;
  const DevTables* __restrict__ tab = s.tab;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int r = blockIdx.y;
  const size_t roff = size_t(r) * s.n;
  const size_t soff = size_t(r) * s.total_sites;
  const double4* __restrict__ p4 = a.st.pos4 + roff;
  const double4* __restrict__ o4 = a.st.off + soff;
  const MinImage mi = s.mi;
  const float thr = a.thr;
  auto mimg = [&](double d) {
    return WRAPPED ? min_image_wrapped(d, mi.negL, thr) : min_image(d, mi);
  };
  const double rc2 = a.rc2;
  double ulj = 0, uel = 0, urf = 0, vir = 0, s1 = 0, s2 = 0, cnt = 0;
  const int wpb = blockDim.x >> 5;  // warps per CTA (<= kForceWarps; fewer for small systems)
  // row groups: S warps per row when SPLIT (S divides the CTA's warps)
  const int S = SPLIT ? a.split : 1;
  const int rpc = wpb / S, rl = warp / S, part = warp % S;
  __shared__ double slab[SPLIT ? kForceWarps : 1][6];
  for (int base = blockIdx.x * rpc;; base += gridDim.x * rpc) {
    if (SPLIT ? base >= s.n : base + rl >= s.n) break;  // CTA-uniform when SPLIT
    const int i_ = base + rl;
    const bool has = i_ < s.n;
    const int i = has ? i_ : 0;
    const double4 pi = p4[i];  // i, j: slots; the reference's order is that of ext_of
    const int ei = ext_of(pi);
    const int si = s.sp_slot[roff + i];
    const int bi = s.sb_slot[roff + i];
    double fx = 0, fy = 0, fz = 0, tx = 0, ty = 0, tz = 0;
    const uint32_t* row = a.mask + (size_t(r) * s.n_pad + i) * s.words;
    if (has)
    for_each_partner(row, s.words, lane, plist[warp], [&](int j) {
      const double4 pj = p4[j];
      const bool lo = ei < ext_of(pj);
      const double Rx = mimg(sub(pi.x, pj.x));
      const double Ry = mimg(sub(pi.y, pj.y));
      const double Rz = mimg(sub(pi.z, pj.z));
      const int sj = s.sp_slot[roff + j];
      const int bj = s.sb_slot[roff + j];
      const DevPairInfo pinfo = tab->pair[lo ? si * s.ns + sj : sj * s.ns + si];
      double R2 = 0.0, s1p = 0.0, s2p = 0.0;
      if (lo) {
        R2 = norm2_exact(Rx, Ry, Rz);
        cnt += 1.0;
      }
      auto site_term = [&](int ta, int tb, double& rx, double& ry, double& rz, double& dix,
                           double& diy, double& diz) -> double {
        const int ki = bi + (lo ? ta : tb), kj = bj + (lo ? tb : ta);
        const double4 di = o4[ki], dj = o4[kj];
        dix = di.x;
        diy = di.y;
        diz = di.z;
        const double djx = dj.x, djy = dj.y, djz = dj.z;
        if (lo) {
          rx = sub(add(Rx, dix), djx);
          ry = sub(add(Ry, diy), djy);
          rz = sub(add(Rz, diz), djz);
        } else {
          rx = add(sub(Rx, djx), dix);
          ry = add(sub(Ry, djy), diy);
          rz = add(sub(Rz, djz), diz);
        }
        return norm2_exact(rx, ry, rz);
      };
      for (int q = 0; q < pinfo.lj_count; ++q) {
        const DevLjTerm t = tab->lj[pinfo.lj_begin + q];
        double rx, ry, rz, dix, diy, diz;
        const double r2 = site_term(t.a, t.b, rx, ry, rz, dix, diy, diz);
        if (r2 >= rc2) continue;
        const double inv_r2 = rcp_nr(r2);
        const double ir6 = inv_r2 * inv_r2 * inv_r2;
        const double a12 = t.c12 * ir6 * ir6;
        const double a6 = t.c6 * ir6;
        const double du_r = -12.0 * a12 + 6.0 * a6;
        const double fs = -du_r * inv_r2;
        const double gx = fs * rx, gy = fs * ry, gz = fs * rz;
        fx += gx;
        fy += gy;
        fz += gz;
        tx += diy * gz - diz * gy;
        ty += diz * gx - dix * gz;
        tz += dix * gy - diy * gx;
        if (lo) {
          ulj += a12 - a6;
          vir += Rx * gx + Ry * gy + Rz * gz;
          if (a.vderiv) {
            const double d2u_r2 = 156.0 * a12 - 42.0 * a6;
            const double rvR = rx * Rx + ry * Ry + rz * Rz;
            const double arr = rvR * inv_r2;
            s1p += du_r * arr;
            s2p += d2u_r2 * arr * arr + du_r * inv_r2 * (R2 - rvR * arr);
          }
        }
      }
      if constexpr (METHOD != 0) {
        for (int q = 0; q < pinfo.qq_count; ++q) {
          const DevQTerm t = tab->qq[pinfo.qq_begin + q];
          double rx, ry, rz, dix, diy, diz;
          const double r2 = site_term(t.a, t.b, rx, ry, rz, dix, diy, diz);
          if (r2 >= rc2) continue;
          const double inv_rr = rsqrt_nr(r2);
          const double inv_r2 = inv_rr * inv_rr, rr = r2 * inv_rr;
          double uu, du_r, d2u_r2 = 0.0, rfu = 0.0;
          if constexpr (METHOD == 2) {
            // potentials.cpp:252-258: erfc(alpha r) qq / r and the force factor
            // qq 2 alpha/sqrt(pi) exp(-alpha^2 r^2), one exponential for both
            const double x = a.alpha * rr;
            const double ex = exp(-x * x);
            const double ec = x < kErfcxMax
                                  ? ex * erfcx_cheb(x, a.erfcx_c, a.erfcx_tlo, a.erfcx_uscale)
                                  : erfc(x);
            const double e = ec * t.qq * inv_rr;
            const double g = t.qq * a.two_alpha_over_sqrt_pi * ex;
            uu = e;
            du_r = -(e + g);
          } else {
            uu = t.qq * inv_rr;
            du_r = -uu;
            d2u_r2 = 2.0 * uu;
            const double rf = t.qq * a.rf_r3inv * r2;
            rfu = rf + t.qq * a.rf_shift;
            du_r += 2.0 * rf;
            d2u_r2 += 2.0 * rf;
          }
          const double fs = -du_r * inv_r2;
          const double gx = fs * rx, gy = fs * ry, gz = fs * rz;
          fx += gx;
          fy += gy;
          fz += gz;
          tx += diy * gz - diz * gy;
          ty += diz * gx - dix * gz;
          tz += dix * gy - diy * gx;
          if (lo) {
            uel += uu;
            urf += rfu;
            vir += Rx * gx + Ry * gy + Rz * gz;
            if (METHOD != 2 && a.vderiv) {
              const double rvR = rx * Rx + ry * Ry + rz * Rz;
              const double arr = rvR * inv_r2;
              s1p += du_r * arr;
              s2p += d2u_r2 * arr * arr + du_r * inv_r2 * (R2 - rvR * arr);
            }
          }
        }
      }
      s1 += s1p;
      s2 += s2p;
    }, part, S);
    fx = warp_sum(fx);
    fy = warp_sum(fy);
    fz = warp_sum(fz);
    tx = warp_sum(tx);
    ty = warp_sum(ty);
    tz = warp_sum(tz);
    bool own = lane == 0 && has;
    if constexpr (SPLIT) {
      double vv[6] = {fx, fy, fz, tx, ty, tz};
      own = combine_parts<6>(vv, slab, warp, lane, S) && has;
      fx = vv[0];
      fy = vv[1];
      fz = vv[2];
      tx = vv[3];
      ty = vv[4];
      tz = vv[5];
    }
    if (own) {
      const size_t e = roff + ext_of(pi);
      a.st.fx[e] = fx;
      a.st.fy[e] = fy;
      a.st.fz[e] = fz;
      a.st.tx[e] = tx;
      a.st.ty[e] = ty;
      a.st.tz[e] = tz;
      if (a.kick_dt > 0.0) fused_kick(a, e);
    }
  }
  double v[kNumRowScalars] = {warp_sum(ulj), warp_sum(uel), warp_sum(urf), warp_sum(s1),
                              warp_sum(s2),  warp_sum(vir), warp_sum(cnt)};
  finalize_scalars<kNumRowScalars>(v, a.cta_part, a.ticket, a.sums, r, 0);
}

// ------------------------------------------------------------- heat flux
// heat_flux (greenkubo.cpp:182-266), split by row instead of by pair: the
// reference adds, per i<j pair with any site term inside rc,
//   0.5 (f.v_i + g_ij.w_i + f.v_j - g_ji.w_j) R    and  u to pair_u[i], pair_u[j].
// From row i's side the pair's force and torque on i are (f_i, g_i) and the
// row's own vector R_i = min_image(com_i - com_j); from row j's side they are
// (-f, -g_ji) with R_j = -R, so the pair term is the sum over both rows of
//   0.5 (f_row.v_row + g_row.w_row) R_row
// (the decomposition of the reference's own check, test_greenkubo.cpp:244-266).
// Each row adds 0.5 (sum_p u_p) v_i + (e_kin_i - h_i) v_i; the kinetic part
// only where `kinetic` is set (rank 0 of a sharded run: pair parts are
// linear in the pairs, so shard partials sum to the whole).  Site terms use
// the same orientation rules as k_force_multi; charges are plain Coulomb
// (+ reaction field), never the Ewald real-space form (greenkubo.cpp:235-247).
// METHOD: 0 LJ only, 1 Coulomb + reaction field, 2 plain Coulomb.
struct FluxArgs {
  ForceArgs f;
  double enthalpy[kMaxSpecies];  // per species (by value: no upload)
  double* out;             // R * kNumSums (jq in the first 3)
  int kinetic;
};

// ONE_SPECIES: the pair's term list and site numbering are row-invariant
// (species 0 throughout; molecule j's sites start at j * n_sites).
template <int METHOD, bool OFFS, bool WRAPPED, bool ONE_SPECIES>
__global__ void __launch_bounds__(kForceWarps * 32, OFFS ? 2 : 4) k_heat_flux(FluxArgs fa) {
  __shared__ int plist[kForceWarps][kQueue];
  const ForceArgs& a = fa.f;
  const SysDev& s = a.s;
  const DevTables* __restrict__ tab = s.tab;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int r = blockIdx.y;
  const size_t roff = size_t(r) * s.n;
  const size_t soff = size_t(r) * s.total_sites;
  const double4* __restrict__ p4 = a.st.pos4 + roff;
  const double4* __restrict__ o4 = a.st.off + soff;
  const MinImage mi = s.mi;
  const float thr = a.thr;
  auto mimg = [&](double d) {
    return WRAPPED ? min_image_wrapped(d, mi.negL, thr) : min_image(d, mi);
  };
  const double rc2 = a.rc2;
  double jx = 0, jy = 0, jz = 0;  // this warp's rows (lane 0)
  const int wpb = blockDim.x >> 5;
  const int nsite0 = tab->species[0].n_sites;
  const DevPairInfo pinfo0 = tab->pair[0];
  for (int i = blockIdx.x * wpb + warp; i < s.n; i += gridDim.x * wpb) {
    const double4 pi = p4[i];  // i, j: slots; the reference's order is that of ext_of
    const int ei = ext_of(pi);
    const size_t ge = roff + ei;
    const int si = ONE_SPECIES ? 0 : s.sp_slot[roff + i];
    const int bi = ONE_SPECIES ? i * nsite0 : s.sb_slot[roff + i];
    const double vix = a.st.vx[ge], viy = a.st.vy[ge], viz = a.st.vz[ge];
    D3 wl{0.0, 0.0, 0.0};  // lab-frame angular velocity (only torques use it)
    if constexpr (OFFS)
      wl = rotate_exact(a.st.qw[ge], a.st.qx[ge], a.st.qy[ge], a.st.qz[ge],
                        {a.st.wx[ge], a.st.wy[ge], a.st.wz[ge]});
    double tx = 0, ty = 0, tz = 0, up = 0;  // sum_p 0.5 s_p R_p, sum_p u_p
    const uint32_t* row = a.mask + (size_t(r) * s.n_pad + i) * s.words;
    for_each_partner(row, s.words, lane, plist[warp], [&](int j) {
      const double4 pj = p4[j];
      const bool lo = ei < ext_of(pj);
      const double Rx = mimg(sub(pi.x, pj.x));
      const double Ry = mimg(sub(pi.y, pj.y));
      const double Rz = mimg(sub(pi.z, pj.z));
      int bj;
      DevPairInfo pinfo;
      if constexpr (ONE_SPECIES) {
        bj = j * nsite0;
        pinfo = pinfo0;
      } else {
        const int sj = s.sp_slot[roff + j];
        bj = s.sb_slot[roff + j];
        pinfo = tab->pair[lo ? si * s.ns + sj : sj * s.ns + si];
      }
      double u = 0, fx = 0, fy = 0, fz = 0, gx = 0, gy = 0, gz = 0;
      auto term = [&](double uu, double du_r, double inv_r2, double rx, double ry,
                      double rz, double dix, double diy, double diz) {
        u += uu;
        const double fs = -du_r * inv_r2;
        const double ex = fs * rx, ey = fs * ry, ez = fs * rz;
        fx += ex;
        fy += ey;
        fz += ez;
        if constexpr (OFFS) {  // centred sites: no torque
          gx += diy * ez - diz * ey;
          gy += diz * ex - dix * ez;
          gz += dix * ey - diy * ex;
        }
      };
      auto site = [&](int ta, int tb, double& rx, double& ry, double& rz, double& dix,
                      double& diy, double& diz) -> double {
        if constexpr (!OFFS) {
          dix = diy = diz = 0.0;
          rx = Rx;
          ry = Ry;
          rz = Rz;
        } else {
          const int ki = bi + (lo ? ta : tb), kj = bj + (lo ? tb : ta);
          const double4 di = o4[ki], dj = o4[kj];
          dix = di.x;
          diy = di.y;
          diz = di.z;
          if (lo) {
            rx = sub(add(Rx, dix), dj.x);
            ry = sub(add(Ry, diy), dj.y);
            rz = sub(add(Rz, diz), dj.z);
          } else {
            rx = add(sub(Rx, dj.x), dix);
            ry = add(sub(Ry, dj.y), diy);
            rz = add(sub(Rz, dj.z), diz);
          }
        }
        return norm2_exact(rx, ry, rz);
      };
      if constexpr (ONE_SPECIES && !OFFS && METHOD == 0) {
        // one centred site: at most one LJ term, its coefficients in a.c12 /
        // a.c6 (zero when the table has none)
        const double r2 = norm2_exact(Rx, Ry, Rz);
        if (r2 < rc2) {
          const double inv_r2 = rcp_nr(r2);
          const double ir6 = inv_r2 * inv_r2 * inv_r2;
          const double a12 = a.c12 * ir6 * ir6;
          const double a6 = a.c6 * ir6;
          term(a12 - a6, -12.0 * a12 + 6.0 * a6, inv_r2, Rx, Ry, Rz, 0.0, 0.0, 0.0);
        }
      } else {
        for (int q = 0; q < pinfo.lj_count; ++q) {
          const DevLjTerm t = tab->lj[pinfo.lj_begin + q];
          double rx, ry, rz, dix, diy, diz;
          const double r2 = site(t.a, t.b, rx, ry, rz, dix, diy, diz);
          if (r2 >= rc2) continue;
          const double inv_r2 = rcp_nr(r2);
          const double ir6 = inv_r2 * inv_r2 * inv_r2;
          const double a12 = t.c12 * ir6 * ir6;
          const double a6 = t.c6 * ir6;
          term(a12 - a6, -12.0 * a12 + 6.0 * a6, inv_r2, rx, ry, rz, dix, diy, diz);
        }
      }
      if constexpr (METHOD != 0) {
        for (int q = 0; q < pinfo.qq_count; ++q) {
          const DevQTerm t = tab->qq[pinfo.qq_begin + q];
          double rx, ry, rz, dix, diy, diz;
          const double r2 = site(t.a, t.b, rx, ry, rz, dix, diy, diz);
          if (r2 >= rc2) continue;
          const double inv_r2 = rcp_nr(r2);
          const double uc = t.qq / sqrt(r2);
          double uu = uc, du_r = -uc;
          if constexpr (METHOD == 1) {
            const double rf = t.qq * a.rf_r3inv * r2;
            uu += rf + t.qq * a.rf_shift;
            du_r += 2.0 * rf;
          }
          term(uu, du_r, inv_r2, rx, ry, rz, dix, diy, diz);
        }
      }
      const double sp = OFFS ? 0.5 * (fx * vix + fy * viy + fz * viz + gx * wl.x + gy * wl.y + gz * wl.z)
                             : 0.5 * (fx * vix + fy * viy + fz * viz);
      tx += sp * Rx;
      ty += sp * Ry;
      tz += sp * Rz;
      up += u;
    });
    tx = warp_sum(tx);
    ty = warp_sum(ty);
    tz = warp_sum(tz);
    up = warp_sum(up);
    if (lane == 0) {
      double e = 0.5 * up;
      if (fa.kinetic) {
        const DevSpecies& sp = tab->species[si];
        const double wbx = a.st.wx[ge], wby = a.st.wy[ge], wbz = a.st.wz[ge];
        const double ek = 0.5 * sp.total_mass * (vix * vix + viy * viy + viz * viz) +
                          0.5 * (sp.inertia[0] * wbx * wbx + sp.inertia[1] * wby * wby +
                                 sp.inertia[2] * wbz * wbz);
        e += ek - fa.enthalpy[si];
      }
      jx += tx + e * vix;
      jy += ty + e * viy;
      jz += tz + e * viz;
    }
  }
  double v[3] = {jx, jy, jz};
  finalize_scalars<3>(v, a.cta_part, a.ticket, fa.out, r, 0);
}

// ------------------------------------ single-species all-LJ rigid molecules
// The general path of potentials.cpp:204-242 specialised to one species whose
// site pairs are all LJ terms in the PairTable's (ia, ib) order
// (potentials.cpp:54-70) and no charges: 2CLJ (BASELINE cfg1, cfg4) and the
// 3-site rotors of the reference tests.  Term parameters and the row's site
// offsets sit in registers; each partner's site offsets are gathered once per
// pair (not once per term).  Same arithmetic and orientation rules as
// k_force_multi.
template <int NS, bool WRAPPED, bool SPLIT>
__global__ void __launch_bounds__(kForceWarps * 32, 2) k_force_rigid(ForceArgs a) {
  __shared__ int plist[kForceWarps][kQueue];
  const SysDev& s = a.s;
  const DevTables* __restrict__ tab = s.tab;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int r = blockIdx.y;
  const size_t roff = size_t(r) * s.n;
  const size_t soff = size_t(r) * s.total_sites;
  const double4* __restrict__ p4 = a.st.pos4 + roff;
  const double4* __restrict__ o4 = a.st.off + soff;
  const MinImage mi = s.mi;
  const float thr = a.thr;
  auto mimg = [&](double d) {
    return WRAPPED ? min_image_wrapped(d, mi.negL, thr) : min_image(d, mi);
  };
  double c12[NS][NS], c6[NS][NS];
#pragma unroll
  for (int ta = 0; ta < NS; ++ta)
#pragma unroll
    for (int tb = 0; tb < NS; ++tb) {
      c12[ta][tb] = tab->lj[ta * NS + tb].c12;
      c6[ta][tb] = tab->lj[ta * NS + tb].c6;
    }
  const double rc2 = a.rc2;
  double ulj = 0, vir = 0, s1 = 0, s2 = 0, cnt = 0;
  const int wpb = blockDim.x >> 5;  // warps per CTA (<= kForceWarps; fewer for small systems)
  // row groups: S warps per row when SPLIT (S divides the CTA's warps)
  const int S = SPLIT ? a.split : 1;
  const int rpc = wpb / S, rl = warp / S, part = warp % S;
  __shared__ double slab[SPLIT ? kForceWarps : 1][6];
  for (int base = blockIdx.x * rpc;; base += gridDim.x * rpc) {
    if (SPLIT ? base >= s.n : base + rl >= s.n) break;  // CTA-uniform when SPLIT
    const int i_ = base + rl;
    const bool has = i_ < s.n;
    const int i = has ? i_ : 0;
    const double4 pi = p4[i];  // i, j: slots; the reference's order is that of ext_of
    const int ei = ext_of(pi);
    const int bi = i * NS;  // single species: slot-ordered sites start at i * NS
    double4 di[NS];
#pragma unroll
    for (int k = 0; k < NS; ++k) di[k] = o4[bi + k];
    double fx = 0, fy = 0, fz = 0, tx = 0, ty = 0, tz = 0;
    const uint32_t* row = a.mask + (size_t(r) * s.n_pad + i) * s.words;
    if (has)
    for_each_partner<false>(row, s.words, lane, plist[warp], [&](int j) {
      const double4 pj = p4[j];
      const bool lo = ei < ext_of(pj);
      double4 dj[NS];
#pragma unroll
      for (int k = 0; k < NS; ++k) dj[k] = o4[j * NS + k];
      const double Rx = mimg(sub(pi.x, pj.x));
      const double Ry = mimg(sub(pi.y, pj.y));
      const double Rz = mimg(sub(pi.z, pj.z));
      const double R2 = lo ? norm2_exact(Rx, Ry, Rz) : 0.0;
      cnt += lo ? 1.0 : 0.0;
      double s1p = 0.0, s2p = 0.0;
#pragma unroll
      for (int ta = 0; ta < NS; ++ta)
#pragma unroll
        for (int tb = 0; tb < NS; ++tb) {
          // reference term (ta on the lower molecule, tb on the upper one)
          const double4 dI = lo ? di[ta] : di[tb];
          const double4 dJ = lo ? dj[tb] : dj[ta];
          double rx, ry, rz;
          if (lo) {
            rx = sub(add(Rx, dI.x), dJ.x);
            ry = sub(add(Ry, dI.y), dJ.y);
            rz = sub(add(Rz, dI.z), dJ.z);
          } else {
            rx = add(sub(Rx, dJ.x), dI.x);
            ry = add(sub(Ry, dJ.y), dI.y);
            rz = add(sub(Rz, dJ.z), dI.z);
          }
          const double r2 = norm2_exact(rx, ry, rz);
          // branch-free (the NS^2 terms are independent dependency chains the
          // compiler interleaves): out-of-range terms take r2 = 1 and ir6 = 0,
          // and their R (NaN for a NaN position) reaches no sum
          const bool in = r2 < rc2;
          const double inv_r2 = rcp_nr(in ? r2 : 1.0);
          const double t6 = inv_r2 * inv_r2 * inv_r2;
          const double ir6 = in ? t6 : 0.0;
          const double a12 = c12[ta][tb] * ir6 * ir6;
          const double a6 = c6[ta][tb] * ir6;
          const double du_r = -12.0 * a12 + 6.0 * a6;
          const double fs = -du_r * inv_r2;
          if (in) {
            const double gx = fs * rx, gy = fs * ry, gz = fs * rz;
            fx += gx;
            fy += gy;
            fz += gz;
            tx += dI.y * gz - dI.z * gy;
            ty += dI.z * gx - dI.x * gz;
            tz += dI.x * gy - dI.y * gx;
            if (lo) {
              ulj += a12 - a6;
              vir += Rx * gx + Ry * gy + Rz * gz;
              if (a.vderiv) {
                const double d2u_r2 = 156.0 * a12 - 42.0 * a6;
                const double rvR = rx * Rx + ry * Ry + rz * Rz;
                const double arr = rvR * inv_r2;
                s1p += du_r * arr;
                s2p += d2u_r2 * arr * arr + du_r * inv_r2 * (R2 - rvR * arr);
              }
            }
          }
        }
      s1 += s1p;
      s2 += s2p;
    }, part, S);
    fx = warp_sum(fx);
    fy = warp_sum(fy);
    fz = warp_sum(fz);
    tx = warp_sum(tx);
    ty = warp_sum(ty);
    tz = warp_sum(tz);
    bool own = lane == 0 && has;
    if constexpr (SPLIT) {
      double vv[6] = {fx, fy, fz, tx, ty, tz};
      own = combine_parts<6>(vv, slab, warp, lane, S) && has;
      fx = vv[0];
      fy = vv[1];
      fz = vv[2];
      tx = vv[3];
      ty = vv[4];
      tz = vv[5];
    }
    if (own) {
      const size_t e = roff + ext_of(pi);
      a.st.fx[e] = fx;
      a.st.fy[e] = fy;
      a.st.fz[e] = fz;
      a.st.tx[e] = tx;
      a.st.ty[e] = ty;
      a.st.tz[e] = tz;
      if (a.kick_dt > 0.0) fused_kick(a, e);
    }
  }
  double v[kNumRowScalars] = {warp_sum(ulj), 0.0, 0.0, warp_sum(s1),
                              warp_sum(s2),  warp_sum(vir), warp_sum(cnt)};
  finalize_scalars<kNumRowScalars>(v, a.cta_part, a.ticket, a.sums, r, 0);
}

// ------------------------- rigid molecules, once per pair (Newton's third law)
// evaluate_pair_range (potentials.cpp:204-242) for one species of NS LJ sites
// (2CLJ: BASELINE cfg1, cfg4), every molecule pair evaluated ONCE -- the
// reference's own scheme (F_i += f, F_j -= f) -- with the partner side
// accumulated without atomics:
// * one warp per 32 x 32 block pair (BI <= BJ) of slots; lane l owns
//   molecule BI*32 + l (position and site offsets in registers, force and
//   torque accumulated in registers); the J block's positions and offsets
//   are staged in shared memory;
// * step k pairs lane l with j = (l + k) & 31 (k = 0..31; 1..16 on the
//   diagonal block, k = 16 on lanes < 16 only), so in every step the 32
//   lanes touch 32 distinct partners: each lane adds the pair's partner-side
//   force and torque into the partner's shared-memory accumulator without
//   conflicts, in step order (deterministic);
// * each pair is computed in the reference's orientation (the lower
//   external index is i: R = min_image(com_i - com_j), site vectors
//   (R + d_a) - d_b, exactly as k_force_rigid), so COM and site cutoffs are
//   decided on the reference's bits; energy, virial, s1, s2 once per pair;
// * the block pair writes two records (32 molecules x force, torque): the
//   I side and the J side; k_rigid_reduce sums each block's records in a
//   fixed order (block-pair order) -- the per-pair contribution buffer and
//   segmented reduction of the north star, at block-pair granularity.
constexpr int kTileWarps = 4;
#ifndef B2MD_TILE_MINBLOCKS
#define B2MD_TILE_MINBLOCKS 5
#endif
constexpr int kTileMinBlocks = B2MD_TILE_MINBLOCKS;  // 20 warps per SM (<= 96 registers)
constexpr int kTileSplit = 2;      // work items per block pair (parts of its 32 steps)

struct TileArgs {
  double* rec;   // R * nbp * kTileSplit * 2 records of 32 x 6 doubles:
                 // [bp][part][side][lane][fx fy fz tx ty tz]
  int nb;        // 32-slot blocks per replica
  int nbp;       // block pairs per replica nb (nb + 1) / 2
  int bp_begin, bp_end;  // this rank's block pairs (row shard)
};

__device__ __forceinline__ void tile_of(int bp, int nb, int& bi, int& bj) {
  // bp = bi nb - bi (bi - 1) / 2 + (bj - bi): invert over the rows
  int lo = 0, hi = nb - 1;
  while (lo < hi) {  // largest bi with start(bi) <= bp
    const int mid = (lo + hi + 1) >> 1;
    const int st = mid * nb - ((mid * (mid - 1)) >> 1);
    if (st <= bp) lo = mid; else hi = mid - 1;
  }
  bi = lo;
  bj = bi + (bp - (bi * nb - ((bi * (bi - 1)) >> 1)));
}

template <int NS, bool WRAPPED>
__global__ void __launch_bounds__(kTileWarps * 32, kTileMinBlocks) k_force_rigid_tile(ForceArgs a, TileArgs ta_) {
  constexpr int kJW = 3 + 3 * NS;  // staged doubles per partner: com, site offsets
  __shared__ double jdat[kTileWarps][kJW][33];  // [field][j] (+1 pad: no bank conflicts)
  __shared__ int jext[kTileWarps][32];
  __shared__ double cpar[2][NS][NS];            // c12, c6
  const SysDev& s = a.s;
  const DevTables* __restrict__ tab = s.tab;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int r = blockIdx.y;
  const int n = s.n;
  const unsigned full = 0xffffffffu;
  const size_t roff = size_t(r) * n;
  const size_t soff = size_t(r) * s.total_sites;
  const double4* __restrict__ p4 = a.st.pos4 + roff;
  const double4* __restrict__ o4 = a.st.off + soff;
  if (threadIdx.x < NS * NS) {
    cpar[0][threadIdx.x / NS][threadIdx.x % NS] = tab->lj[threadIdx.x].c12;
    cpar[1][threadIdx.x / NS][threadIdx.x % NS] = tab->lj[threadIdx.x].c6;
  }
  __syncthreads();
  const MinImage mi = s.mi;
  const float thr = a.thr;
  auto mimg = [&](double d) {
    return WRAPPED ? min_image_wrapped(d, mi.negL, thr) : min_image(d, mi);
  };
  const double rc2 = a.rc2, rmax2 = a.rmax2;
  double ulj = 0, vir = 0, s1 = 0, s2 = 0, cnt = 0;
  double (*jd)[33] = jdat[warp];
  const int items = ta_.nbp * kTileSplit;
  // one work item (block pair, part of its steps) per warp: a fixed
  // assignment, so every scalar sum is taken in the same order every run
  for (int it = blockIdx.x * kTileWarps + warp; it < items; it += gridDim.x * kTileWarps) {
    const int bp = it / kTileSplit, part = it - bp * kTileSplit;
    int bi, bj;
    tile_of(bp, ta_.nb, bi, bj);
    const bool diag = bi == bj;
    // steps of this part: k0 .. k1 (the diagonal block pair has steps 1 .. 16,
    // step 16 on lanes < 16 only)
    const int span = diag ? 16 : 32;
    const int k0 = (diag ? 1 : 0) + part * span / kTileSplit;
    const int k1 = (diag ? 1 : 0) + (part + 1) * span / kTileSplit - 1;
    const int i = bi * 32 + lane;
    const bool iv = i < n;
    const int ic = iv ? i : bi * 32;
    const double4 pi = p4[ic];
    const int ei = ext_of(pi);
    double dix[NS], diy[NS], diz[NS];
#pragma unroll
    for (int k = 0; k < NS; ++k) {
      const double4 o = o4[ic * NS + k];
      dix[k] = o.x, diy[k] = o.y, diz[k] = o.z;
    }
    {
      const int j = bj * 32 + lane;
      const int jc = j < n ? j : bj * 32;
      const double4 pj = p4[jc];
      jd[0][lane] = pj.x, jd[1][lane] = pj.y, jd[2][lane] = pj.z;
      jext[warp][lane] = j < n ? ext_of(pj) : -1;
#pragma unroll
      for (int k = 0; k < NS; ++k) {
        const double4 o = o4[jc * NS + k];
        jd[3 + 3 * k][lane] = o.x, jd[4 + 3 * k][lane] = o.y, jd[5 + 3 * k][lane] = o.z;
      }
    }
    __syncwarp();
    double fx = 0, fy = 0, fz = 0, tx = 0, ty = 0, tz = 0;
    // the partner side travels with its partner: at step k lane l holds the
    // accumulators of partner (l + k) & 31 and passes them to lane l - 1
    double gfx = 0, gfy = 0, gfz = 0, gtx = 0, gty = 0, gtz = 0;
    const bool mine = bp >= ta_.bp_begin && bp < ta_.bp_end;
    const int src = (lane + 1) & 31;
    if (mine)
      for (int k = k0; k <= k1; ++k) {
        const int jl = (lane + k) & 31;
        const int ej = jext[warp][jl];
        const bool valid = iv && ej >= 0 && !(diag && k == 16 && lane >= 16);
        const bool lo = ei < ej;
        const double Rx = mimg(sub(pi.x, jd[0][jl]));
        const double Ry = mimg(sub(pi.y, jd[1][jl]));
        const double Rz = mimg(sub(pi.z, jd[2][jl]));
        const double R2 = norm2_exact(Rx, Ry, Rz);
        const bool pass = valid && R2 < rmax2;  // potentials.cpp:212
        if (__ballot_sync(full, pass)) {
          cnt += pass ? 1.0 : 0.0;
          double s1p = 0.0, s2p = 0.0;
#pragma unroll
          for (int ta = 0; ta < NS; ++ta)
#pragma unroll
            for (int tb = 0; tb < NS; ++tb) {
              // reference term: ta on the lower molecule, tb on the upper one
              const int ka = lo ? ta : tb, kb = lo ? tb : ta;  // this lane's site, partner's site
              const double ax = NS == 2 ? (ka ? dix[1] : dix[0]) : dix[ka];
              const double ay = NS == 2 ? (ka ? diy[1] : diy[0]) : diy[ka];
              const double az = NS == 2 ? (ka ? diz[1] : diz[0]) : diz[ka];
              const double bx = jd[3 + 3 * kb][jl], by = jd[4 + 3 * kb][jl], bz = jd[5 + 3 * kb][jl];
              double rx, ry, rz;
              if (lo) {
                rx = sub(add(Rx, ax), bx);
                ry = sub(add(Ry, ay), by);
                rz = sub(add(Rz, az), bz);
              } else {
                rx = add(sub(Rx, bx), ax);
                ry = add(sub(Ry, by), ay);
                rz = add(sub(Rz, bz), az);
              }
              const double r2 = norm2_exact(rx, ry, rz);
              const bool in = pass && r2 < rc2;
              const double inv_r2 = rcp_nr(in ? r2 : 1.0);
              const double t6 = inv_r2 * inv_r2 * inv_r2;
              const double ir6 = in ? t6 : 0.0;
              const double a12 = cpar[0][ta][tb] * ir6 * ir6;
              const double a6 = cpar[1][ta][tb] * ir6;
              const double du_r = -12.0 * a12 + 6.0 * a6;
              const double fs = -du_r * inv_r2;
              if (in) {  // an excluded pair's R may be NaN: it reaches no sum
                const double gx = fs * rx, gy = fs * ry, gz = fs * rz;
                fx += gx, fy += gy, fz += gz;
                tx += ay * gz - az * gy;
                ty += az * gx - ax * gz;
                tz += ax * gy - ay * gx;
                gfx -= gx, gfy -= gy, gfz -= gz;
                gtx -= by * gz - bz * gy;
                gty -= bz * gx - bx * gz;
                gtz -= bx * gy - by * gx;
                ulj += a12 - a6;
                vir += Rx * gx + Ry * gy + Rz * gz;
                if (a.vderiv) {
                  const double d2u_r2 = 156.0 * a12 - 42.0 * a6;
                  const double rvR = rx * Rx + ry * Ry + rz * Rz;
                  const double arr = rvR * inv_r2;
                  s1p += du_r * arr;
                  s2p += d2u_r2 * arr * arr + du_r * inv_r2 * (R2 - rvR * arr);
                }
              }
            }
          s1 += s1p;
          s2 += s2p;
        }
        gfx = __shfl_sync(full, gfx, src), gfy = __shfl_sync(full, gfy, src);
        gfz = __shfl_sync(full, gfz, src), gtx = __shfl_sync(full, gtx, src);
        gty = __shfl_sync(full, gty, src), gtz = __shfl_sync(full, gtz, src);
      }
    // records of the item: side 0 = the I block (lane l: molecule l), side 1
    // = the J block (lane l holds partner (l + k1 + 1) & 31 after the last pass)
    double* rec = ta_.rec + ((size_t(r) * ta_.nbp + bp) * kTileSplit + part) * 2 * 32 * 6;
    const int jp = (lane + k1 + 1) & 31;
    rec[lane * 6 + 0] = fx, rec[lane * 6 + 1] = fy, rec[lane * 6 + 2] = fz;
    rec[lane * 6 + 3] = tx, rec[lane * 6 + 4] = ty, rec[lane * 6 + 5] = tz;
    double* rj = rec + (32 + jp) * 6;
    rj[0] = gfx, rj[1] = gfy, rj[2] = gfz, rj[3] = gtx, rj[4] = gty, rj[5] = gtz;
    __syncwarp();  // jd / jext are restaged by the next item
  }
  double v[kNumRowScalars] = {warp_sum(ulj), 0.0, 0.0, warp_sum(s1),
                              warp_sum(s2),  warp_sum(vir), warp_sum(cnt)};
  finalize_scalars<kNumRowScalars>(v, a.cta_part, a.ticket, a.sums, r, 0);
}

// Block B's force and torque: the records of every item touching B in
// (block pair, part) order -- the I side of (B, x) for x >= B, the J side of
// (x, B) for x <= B, both for the diagonal block pair -- thread (m, c) sums
// component c of molecule m, 8 loads in flight.  Block pairs outside this
// rank's range contribute nothing (not read).
static __global__ void __launch_bounds__(192) k_rigid_reduce(ForceArgs a, TileArgs ta_) {
  const int b = blockIdx.x, r = blockIdx.y;
  const int n = a.s.n;
  const int t = threadIdx.x, m = t / 6, c = t - 6 * (t / 6);
  const int slot = b * 32 + m;
  const int nb = ta_.nb;
  const double* rec = ta_.rec + size_t(r) * ta_.nbp * kTileSplit * 2 * 32 * 6 + m * 6 + c;
  auto rec_of = [&](int x, int side, int part) -> long {  // record offset, or -1
    const int lo = min(b, x), hi = max(b, x);
    const int bp = lo * nb - ((lo * (lo - 1)) >> 1) + (hi - lo);
    if (bp < ta_.bp_begin || bp >= ta_.bp_end) return -1;
    return ((long(bp) * kTileSplit + part) * 2 + side) * 32 * 6;
  };
  const int total = (nb + 1) * kTileSplit;  // x = nb: the diagonal's J side
  double acc = 0.0;
  for (int u0 = 0; u0 < total; u0 += 8) {
    double v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int uu = u0 + u, x = uu / kTileSplit, part = uu - x * kTileSplit;
      long o = -1;
      if (x < nb) o = rec_of(x, b <= x ? 0 : 1, part);
      else if (x == nb) o = rec_of(b, 1, part);
      v[u] = o >= 0 ? rec[o] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) acc += v[u];
  }
  const size_t roff = size_t(r) * n;
  __shared__ int ext[32];
  if (t < 32) ext[t] = b * 32 + t < n ? ext_of(a.st.pos4[roff + b * 32 + t]) : 0;
  __syncthreads();
  if (slot < n) {
    double* f[6] = {a.st.fx, a.st.fy, a.st.fz, a.st.tx, a.st.ty, a.st.tz};
    f[c][roff + ext[m]] = acc;
  }
  __syncthreads();
  if (c == 0 && slot < n && a.kick_dt > 0.0) fused_kick(a, roff + ext[m]);
}

// ------------------------------------------------------------------- Ewald
// ewald.cpp:134-151: per charged site, per axis e^{i 2 pi n x / L}, n=0..kmax,
// by the same complex recurrence.  Layout [r][axis][n][site] (site fastest).
struct EwaldArgs {
  SysDev s;
  StateDev st;
  int nq;               // charged sites per replica
  int kmax;
  int nk;               // k-vectors in this rank's range
  int k_begin;
  const int* q_mol;     // nq
  const int* q_site;    // nq
  const double* q_val;  // nq
  const int* mol_qbegin;  // n + 1: charged entries of each molecule
  const DevKVec* kv;    // all k-vectors
  double2* tab;         // R * 3 * (kmax+1) * nq
  double2* S;           // R * nk_total
  double* uk;           // R * nk (per-CTA partials of U_recip)
  unsigned* ticket;     // R
  double* sums;         // R * kNumSums
  int nk_total;
  int kparts;           // warps per molecule in k_ewald_force (1, 2, 4, 8)
  double two_pi_over_L;
  // k_ewald_force's output: null: added to the (complete) real-space totals;
  // else written (=) to frec[6][R n] -- the kernel then runs beside the
  // real-space kernel and the end-of-step kick adds the two (StepArgs::frec)
  double* frec;
};

static __global__ void k_ewald_tables(EwaldArgs a) {
  const int gid = blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= a.nq * a.s.R) return;
  const int r = gid / a.nq, q = gid - r * a.nq;
  const int m = a.q_mol[q];
  const size_t roff = size_t(r) * a.s.n;
  const size_t soff = size_t(r) * a.s.total_sites + site_slot(a.s, r, m, a.q_site[q]);
  const double4 o = a.st.off[soff];
  const double p[3] = {a.st.px[roff + m] + o.x, a.st.py[roff + m] + o.y, a.st.pz[roff + m] + o.z};
  const int K = a.kmax + 1;
  double2* base = a.tab + size_t(r) * 3 * K * a.nq;
  for (int ax = 0; ax < 3; ++ax) {
    double sn, cs;
    sincos(a.two_pi_over_L * p[ax], &sn, &cs);
    double re = 1.0, im = 0.0;
    double2* t = base + size_t(ax) * K * a.nq + q;
    t[0] = make_double2(1.0, 0.0);
    for (int k = 1; k < K; ++k) {
      const double nre = re * cs - im * sn;
      const double nim = re * sn + im * cs;
      re = nre;
      im = nim;
      t[size_t(k) * a.nq] = make_double2(re, im);
    }
  }
}

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}

__device__ __forceinline__ double2 site_phase(const double2* base, int K, int nq, int q,
                                              const DevKVec& k) {
  double2 e = base[size_t(k.nx) * nq + q];
  double2 vy = base[size_t(K + abs(k.ny)) * nq + q];
  if (k.ny < 0) vy.y = -vy.y;
  e = cmul(e, vy);
  double2 vz = base[size_t(2 * K + abs(k.nz)) * nq + q];
  if (k.nz < 0) vz.y = -vz.y;
  return cmul(e, vz);
}

// ewald.cpp:163-169: one CTA per (k, replica), fixed-order block reduction;
// U_recip = sum_k 0.5 coeff |S|^2 finalized by the last CTA (sums[7]).
static __global__ void __launch_bounds__(256) k_ewald_sk(EwaldArgs a) {
  const int kk = a.k_begin + blockIdx.x;
  const int r = blockIdx.y;
  const DevKVec k = a.kv[kk];
  const int K = a.kmax + 1;
  const double2* base = a.tab + size_t(r) * 3 * K * a.nq;
  double sre = 0.0, sim = 0.0;
#pragma unroll 4
  for (int q = threadIdx.x; q < a.nq; q += blockDim.x) {
    const double2 e = site_phase(base, K, a.nq, q, k);
    sre += e.x * a.q_val[q];
    sim += e.y * a.q_val[q];
  }
  __shared__ double red[2][8];
  __shared__ double ukv;
  sre = warp_sum(sre);
  sim = warp_sum(sim);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) {
    red[0][w] = sre;
    red[1][w] = sim;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double tr = 0.0, ti = 0.0;
    for (int v = 0; v < int(blockDim.x >> 5); ++v) {
      tr += red[0][v];
      ti += red[1][v];
    }
    a.S[size_t(r) * a.nk_total + kk] = make_double2(tr, ti);
    ukv = 0.5 * k.coeff * (tr * tr + ti * ti);
  }
  __syncthreads();
  const double v[1] = {threadIdx.x == 0 ? ukv : 0.0};
  finalize_scalars<1>(v, a.uk, a.ticket, a.sums, r, kNumRowScalars);
}

// ewald.cpp:171-178: P = a.kparts warps per molecule with charges, warp part
// p takes the k-vectors p*32 + lane, +32P, ...; the parts' forces and
// torques (= off x F) are summed in part order (deterministic) and added to
// the (already written) real-space totals.  P > 1 puts short systems' few
// molecules on enough warps to hide the table gathers.
static __global__ void __launch_bounds__(256) k_ewald_force(EwaldArgs a) {
  __shared__ double slab[8][6];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int P = a.kparts;
  const int m = blockIdx.x * ((blockDim.x >> 5) / P) + warp / P, part = warp % P;
  const int r = blockIdx.y;
  const bool in = m < a.s.n;
  const int q0 = in ? a.mol_qbegin[m] : 0, q1 = in ? a.mol_qbegin[m + 1] : 0;
  const int K = a.kmax + 1;
  const double2* base = a.tab + size_t(r) * 3 * K * a.nq;
  const size_t soff = size_t(r) * a.s.total_sites;
  double fx = 0, fy = 0, fz = 0, tx = 0, ty = 0, tz = 0;
  for (int q = q0; q < q1; ++q) {
    const int site = site_slot(a.s, r, m, a.q_site[q]);
    const double4 o4 = a.st.off[soff + site];
    const double ox = o4.x, oy = o4.y, oz = o4.z;
    const double qv = a.q_val[q];
    double sfx = 0, sfy = 0, sfz = 0;
    for (int kk = a.k_begin + part * 32 + lane; kk < a.k_begin + a.nk; kk += 32 * P) {
      const DevKVec k = a.kv[kk];
      const double2 e = site_phase(base, K, a.nq, q, k);
      const double2 S = a.S[size_t(r) * a.nk_total + kk];
      const double im = e.y * S.x - e.x * S.y;
      const double c = qv * k.coeff * im;
      sfx += c * k.kx;
      sfy += c * k.ky;
      sfz += c * k.kz;
    }
    fx += sfx;
    fy += sfy;
    fz += sfz;
    tx += oy * sfz - oz * sfy;
    ty += oz * sfx - ox * sfz;
    tz += ox * sfy - oy * sfx;
  }
  double v[6] = {warp_sum(fx), warp_sum(fy), warp_sum(fz), warp_sum(tx), warp_sum(ty), warp_sum(tz)};
  bool own = lane == 0;
  if (P > 1) own = combine_parts<6>(v, slab, warp, lane, P);
  if (own && in) {
    const size_t roff = size_t(r) * a.s.n;
    if (a.frec) {  // every molecule (zeros without charges)
      const size_t nt = size_t(a.s.R) * a.s.n;
#pragma unroll
      for (int k = 0; k < 6; ++k) a.frec[k * nt + roff + m] = v[k];
    } else if (q0 != q1) {
      a.st.fx[roff + m] += v[0];
      a.st.fy[roff + m] += v[1];
      a.st.fz[roff + m] += v[2];
      a.st.tx[roff + m] += v[3];
      a.st.ty[roff + m] += v[4];
      a.st.tz[roff + m] += v[5];
    }
  }
}

// ------------------------------------------------- Ewald, tiled (default)
// S(k) and the reciprocal forces with the per-charge phase tables staged in
// shared memory instead of gathered per (k, charge) from L2 (which read the
// 3 x 16-byte table entries of every charge for every k-vector: ~100 MB per
// evaluation on cfg2).  Same arithmetic as k_ewald_sk / k_ewald_force
// (ewald.cpp:156-178); the summation orders are fixed (deterministic).
constexpr int kEwSkQ = 32;    // charges per CTA of k_ewald_sk_tiled (tables in shared memory)
constexpr int kEwFQ = 32;     // charges per CTA of k_ewald_force_tiled
constexpr int kEwFParts = 16; // k-ranges per CTA (one warp each) of k_ewald_force_tiled
constexpr int kEwMaxK = 12;   // kmax + 1 <= kEwMaxK for the tiled kernels (else the gather form)

struct EwaldTiled {
  double2* Sp;  // R * nchunks * nk: S(k) partials of each charge chunk
  double* fq;   // R * nq * 3: reciprocal force of every charge
  int nchunks;
};

// staged tables of charges [q0, q0 + cnt): t[(axis * K + n) * (Q + 1) + ql]
// (rows padded by one entry: different rows of one column fall in different banks)
template <int Q>
__device__ __forceinline__ void ewald_stage(const EwaldArgs& a, int r, int q0, int cnt,
                                            double2* __restrict__ t) {
  const int K = a.kmax + 1;
  const double2* base = a.tab + size_t(r) * 3 * K * a.nq;
  for (int e = threadIdx.x; e < 3 * K * Q; e += blockDim.x) {
    const int row = e / Q, ql = e - row * Q;
    t[row * (Q + 1) + ql] = ql < cnt ? base[size_t(row) * a.nq + q0 + ql] : make_double2(0.0, 0.0);
  }
}

template <int Q>
__device__ __forceinline__ double2 ewald_phase_s(const double2* __restrict__ t, int K, int ql,
                                                 const DevKVec& k) {
  double2 e = t[k.nx * (Q + 1) + ql];
  double2 vy = t[(K + abs(k.ny)) * (Q + 1) + ql];
  if (k.ny < 0) vy.y = -vy.y;
  e = cmul(e, vy);
  double2 vz = t[(2 * K + abs(k.nz)) * (Q + 1) + ql];
  if (k.nz < 0) vz.y = -vz.y;
  return cmul(e, vz);
}

// S(k) partials: one CTA per chunk of kEwSkQ charges, thread per k-vector
// (strided): every charge's tables are read once per evaluation
static __global__ void __launch_bounds__(256) k_ewald_sk_tiled(EwaldArgs a, EwaldTiled et) {
  __shared__ double2 t[3 * kEwMaxK * (kEwSkQ + 1)];
  const int chunk = blockIdx.x, r = blockIdx.y;
  const int q0 = chunk * kEwSkQ, cnt = min(kEwSkQ, a.nq - q0);
  const int K = a.kmax + 1;
  ewald_stage<kEwSkQ>(a, r, q0, cnt, t);
  __shared__ double qs[kEwSkQ];
  if (threadIdx.x < kEwSkQ) qs[threadIdx.x] = threadIdx.x < cnt ? a.q_val[q0 + threadIdx.x] : 0.0;
  __syncthreads();
  double2* Sp = et.Sp + (size_t(r) * et.nchunks + chunk) * a.nk;
  for (int kl = threadIdx.x; kl < a.nk; kl += blockDim.x) {
    const DevKVec k = a.kv[a.k_begin + kl];
    // four independent accumulators (charges ql = 4 i + c), summed in order
    double sre[4] = {0.0, 0.0, 0.0, 0.0}, sim[4] = {0.0, 0.0, 0.0, 0.0};
    for (int q4 = 0; q4 < kEwSkQ; q4 += 4) {
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const double2 e = ewald_phase_s<kEwSkQ>(t, K, q4 + c, k);  // (zero past cnt)
        sre[c] = fma(e.x, qs[q4 + c], sre[c]);
        sim[c] = fma(e.y, qs[q4 + c], sim[c]);
      }
    }
    Sp[kl] = make_double2((sre[0] + sre[1]) + (sre[2] + sre[3]), (sim[0] + sim[1]) + (sim[2] + sim[3]));
  }
}

// S(k) = the chunks' partials in chunk order (lanes q of a k split the chunks,
// fixed xor tree), U_recip = sum_k 0.5 coeff |S|^2 by per-CTA partials totalled
// in order by the last CTA (ewald.cpp:163-169)
constexpr int kEwSumK = 32;  // k-vectors per CTA of k_ewald_sk_sum (8 lanes each)
static __global__ void __launch_bounds__(kEwSumK * 8) k_ewald_sk_sum(EwaldArgs a, EwaldTiled et) {
  const int r = blockIdx.y;
  const int kl = blockIdx.x * kEwSumK + (threadIdx.x >> 3), sub8 = threadIdx.x & 7;
  const double2* P = et.Sp + size_t(r) * et.nchunks * a.nk;
  double sre = 0.0, sim = 0.0;
  if (kl < a.nk) {
#pragma unroll 4
    for (int c = sub8; c < et.nchunks; c += 8) {
      const double2 v = P[size_t(c) * a.nk + kl];
      sre += v.x;
      sim += v.y;
    }
  }
#pragma unroll
  for (int o = 1; o < 8; o <<= 1) {
    sre += __shfl_xor_sync(0xffffffffu, sre, o);
    sim += __shfl_xor_sync(0xffffffffu, sim, o);
  }
  double u = 0.0;
  if (kl < a.nk && sub8 == 0) {
    a.S[size_t(r) * a.nk_total + a.k_begin + kl] = make_double2(sre, sim);
    u = 0.5 * a.kv[a.k_begin + kl].coeff * (sre * sre + sim * sim);
  }
  const double v[1] = {warp_sum(u)};
  finalize_scalars<1>(v, a.uk, a.ticket, a.sums, r, kNumRowScalars);
}

// Reciprocal force of every charge: one CTA per kEwFQ charges (lane = charge),
// warp p takes the p-th of kEwFParts contiguous k-ranges; the parts are
// summed in part order through shared memory (ewald.cpp:171-178)
static __global__ void __launch_bounds__(kEwFQ * kEwFParts) k_ewald_force_tiled(EwaldArgs a, EwaldTiled et) {
  __shared__ double2 t[3 * kEwMaxK * (kEwFQ + 1)];
  __shared__ double part[kEwFParts][3][kEwFQ];
  const int r = blockIdx.y;
  const int q0 = blockIdx.x * kEwFQ, cnt = min(kEwFQ, a.nq - q0);
  const int K = a.kmax + 1;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  ewald_stage<kEwFQ>(a, r, q0, cnt, t);
  __syncthreads();
  const int per = (a.nk + kEwFParts - 1) / kEwFParts;
  const int k0 = warp * per, k1 = min(a.nk, k0 + per);
  const double2* S = a.S + size_t(r) * a.nk_total + a.k_begin;
  // two independent accumulator sets (even / odd k of the range), summed in order
  double fx[2] = {0.0, 0.0}, fy[2] = {0.0, 0.0}, fz[2] = {0.0, 0.0};
#pragma unroll 2
  for (int kl = k0; kl < k1; ++kl) {
    const DevKVec k = a.kv[a.k_begin + kl];  // (warp-uniform: broadcast loads)
    const double2 Sk = S[kl];
    const double2 e = ewald_phase_s<kEwFQ>(t, K, lane, k);
    const double im = e.y * Sk.x - e.x * Sk.y;
    const double c = k.coeff * im;
    const int h = (kl - k0) & 1;
    fx[h] = fma(c, k.kx, fx[h]);
    fy[h] = fma(c, k.ky, fy[h]);
    fz[h] = fma(c, k.kz, fz[h]);
  }
  part[warp][0][lane] = fx[0] + fx[1];
  part[warp][1][lane] = fy[0] + fy[1];
  part[warp][2][lane] = fz[0] + fz[1];
  __syncthreads();
  if (threadIdx.x < 3 * kEwFQ) {
    const int comp = threadIdx.x / kEwFQ, ql = threadIdx.x - comp * kEwFQ;
    if (ql < cnt) {
      double v = 0.0;
      for (int p = 0; p < kEwFParts; ++p) v += part[p][comp][ql];
      et.fq[(size_t(r) * a.nq + q0 + ql) * 3 + comp] = a.q_val[q0 + ql] * v;
    }
  }
}

// Per molecule: its charges' reciprocal forces (in charge order) and their
// torques off x F, added to the real-space totals
static __global__ void __launch_bounds__(256) k_ewald_apply(EwaldArgs a, EwaldTiled et) {
  const int m = blockIdx.x * blockDim.x + threadIdx.x, r = blockIdx.y;
  if (m >= a.s.n) return;
  const int q0 = a.mol_qbegin[m], q1 = a.mol_qbegin[m + 1];
  if (q0 == q1) return;
  const size_t soff = size_t(r) * a.s.total_sites;
  double fx = 0, fy = 0, fz = 0, tx = 0, ty = 0, tz = 0;
  for (int q = q0; q < q1; ++q) {
    const double* f = et.fq + (size_t(r) * a.nq + q) * 3;
    const double4 o = a.st.off[soff + site_slot(a.s, r, m, a.q_site[q])];
    fx += f[0], fy += f[1], fz += f[2];
    tx += o.y * f[2] - o.z * f[1];
    ty += o.z * f[0] - o.x * f[2];
    tz += o.x * f[1] - o.y * f[0];
  }
  const size_t e = size_t(r) * a.s.n + m;
  a.st.fx[e] += fx;
  a.st.fy[e] += fy;
  a.st.fz[e] += fz;
  a.st.tx[e] += tx;
  a.st.ty[e] += ty;
  a.st.tz[e] += tz;
}

// ------------------------------------------------------------- integrator
// engine.cpp:13-19
__device__ __forceinline__ void permute4(int axis, const double q[4], double o[4]) {
  if (axis == 1) {
    o[0] = -q[1]; o[1] = q[0]; o[2] = q[3]; o[3] = -q[2];
  } else if (axis == 2) {
    o[0] = -q[2]; o[1] = -q[3]; o[2] = q[0]; o[3] = q[1];
  } else {
    o[0] = -q[3]; o[1] = q[2]; o[2] = -q[1]; o[3] = q[0];
  }
}
__device__ __forceinline__ double dot4x(const double a[4], const double b[4]) {
  return add(add(add(mul(a[0], b[0]), mul(a[1], b[1])), mul(a[2], b[2])), mul(a[3], b[3]));
}

// free_rotate (engine.cpp:28-59), reference operation order, no FMA.
static __device__ void free_rotate_dev(double q[4], double L[3], const double I[3], double dt) {
  double p[4] = {0.0, 0.0, 0.0, 0.0};
  for (int k = 1; k <= 3; ++k) {
    const double pk = L[k - 1];
    if (pk == 0.0) continue;
    double pq[4];
    permute4(k, q, pq);
    const double tp = mul(2.0, pk);
    for (int c = 0; c < 4; ++c) p[c] = add(p[c], mul(tp, pq[c]));
  }
  const int axis_seq[5] = {3, 2, 1, 2, 3};
  const double hd = mul(0.5, dt);
  for (int stage = 0; stage < 5; ++stage) {
    const int k = axis_seq[stage];
    const double ik = I[k - 1];
    if (ik <= 0.0) continue;
    double pq[4], pp[4];
    permute4(k, q, pq);
    const double zeta = __ddiv_rn(dot4x(p, pq), mul(4.0, ik));
    const double h = stage == 2 ? dt : hd;
    double sn, cs;
    sincos(mul(h, zeta), &sn, &cs);
    permute4(k, p, pp);
    for (int c = 0; c < 4; ++c) {
      q[c] = add(mul(cs, q[c]), mul(sn, pq[c]));
      p[c] = add(mul(cs, p[c]), mul(sn, pp[c]));
    }
  }
  for (int k = 1; k <= 3; ++k) {
    double pq[4];
    permute4(k, q, pq);
    L[k - 1] = (I[k - 1] > 0.0) ? mul(0.5, dot4x(p, pq)) : 0.0;
  }
  const double nrm = __dsqrt_rn(add(add(add(mul(q[0], q[0]), mul(q[1], q[1])), mul(q[2], q[2])), mul(q[3], q[3])));
  for (int c = 0; c < 4; ++c) q[c] = __ddiv_rn(q[c], nrm);
}

struct StepArgs {
  SysDev s;
  StateDev st;
  double dt;
  int* error_mol;  // first non-finite molecule (global index), INT_MAX if none
  int write_offsets;
  uint4* fixpos;     // fixed-point positions for the search (may be null)
  double fix_scale;  // 2^32 / L
  // end-of-step kick after an Ewald evaluation whose reciprocal forces were
  // computed beside the real-space kernel: frec[6][R n] is added to the
  // forces / torques first (ewald.cpp:171-178's +=) and the totals stored
  const double* frec = nullptr;
};

__device__ __forceinline__ double wrap1(double x, double L) {
  // inside (0, L (1 - 2^-40)): x / L rounds below 1, floor is 0 and the
  // reference's x - L * 0 is x itself -- no division
  if (x > 0.0 && x < L * (1.0 - 9.094947017729282e-13)) return x;  // (-0.0 -> +0.0 below)
  return sub(x, mul(L, floor(__ddiv_rn(x, L))));  // model.cpp:282
}

// Fixed-point copy of the positions for the partner search's certified
// prefilter: (round(x 2^32/L), .., .., [x, y, z all in [0, L)]).
__device__ __forceinline__ uint4 fix_position(double x, double y, double z, double L, double scale) {
  const bool in = x >= 0.0 && x < L && y >= 0.0 && y < L && z >= 0.0 && z < L;
  return make_uint4(__double2uint_rn(x * scale), __double2uint_rn(y * scale),
                    __double2uint_rn(z * scale), in ? 1u : 0u);
}

// Positions as the search (fixed point) and the force kernels (packed) read
// them; the integrator writes both itself.
static __global__ void k_stage_positions(const double* px, const double* py, const double* pz, int count,
                                  int n, const int* slot_of, double L, double scale,
                                  uint4* fixpos, double4* pos4) {
  const int gid = blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= count) return;
  const int r = gid / n;
  const size_t k = size_t(r) * n + slot_of[gid];
  const double x = px[gid], y = py[gid], z = pz[gid];
  fixpos[k] = fix_position(x, y, z, L, scale);
  pos4[k] = pack_pos(x, y, z, gid - r * n);
}

// engine.cpp:107-127 (+ build_scene offsets for the new orientation)
// returns the new fixed-point position (zero without a.fixpos)
__device__ __forceinline__ uint4 kick_drift_one(const StepArgs& a, int gid, bool* frozen = nullptr) {
  const SysDev& s = a.s;
  const int r = gid / s.n, i = gid - r * s.n;
  // every input first (independent loads in flight together -- after an L2
  // flush each dependent round trip is a DRAM latency), then the error flag,
  // then the stores
  const int err = frozen ? *a.error_mol : 0x7fffffff;
  const DevSpecies& sp = s.tab->species[s.ns == 1 ? 0 : s.species_of[i]];
  const double vx0 = a.st.vx[gid], vy0 = a.st.vy[gid], vz0 = a.st.vz[gid];
  const double fx0 = a.st.fx[gid], fy0 = a.st.fy[gid], fz0 = a.st.fz[gid];
  const double px0 = a.st.px[gid], py0 = a.st.py[gid], pz0 = a.st.pz[gid];
  double q[4] = {a.st.qw[gid], a.st.qx[gid], a.st.qy[gid], a.st.qz[gid]};
  const double tx0 = a.st.tx[gid], ty0 = a.st.ty[gid], tz0 = a.st.tz[gid];
  const double w[3] = {a.st.wx[gid], a.st.wy[gid], a.st.wz[gid]};
  const size_t slot = size_t(r) * s.n + s.slot_of[gid];
  const double dt = a.dt, half = mul(0.5, dt);
  const double c = __ddiv_rn(half, sp.total_mass);
  const double vx = add(vx0, mul(fx0, c));
  const double vy = add(vy0, mul(fy0, c));
  const double vz = add(vz0, mul(fz0, c));
  double px = add(px0, mul(vx, dt));
  double py = add(py0, mul(vy, dt));
  double pz = add(pz0, mul(vz, dt));
  if (frozen) {
    *frozen = err != 0x7fffffff;  // state frozen after a failed step
    if (*frozen) return make_uint4(0u, 0u, 0u, 0u);
  }
  a.st.vx[gid] = vx;
  a.st.vy[gid] = vy;
  a.st.vz[gid] = vz;
  if (sp.rotational_dof > 0) {
    const D3 tb = rotate_inv_exact(q[0], q[1], q[2], q[3], {tx0, ty0, tz0});
    const double tbv[3] = {tb.x, tb.y, tb.z};
    double L[3];
    for (int k = 0; k < 3; ++k)
      L[k] = sp.inertia[k] > 0.0 ? add(mul(sp.inertia[k], w[k]), mul(half, tbv[k])) : 0.0;
    free_rotate_dev(q, L, sp.inertia, dt);
    double wn[3];
    for (int k = 0; k < 3; ++k) wn[k] = sp.inertia[k] > 0.0 ? __ddiv_rn(L[k], sp.inertia[k]) : 0.0;
    a.st.wx[gid] = wn[0];
    a.st.wy[gid] = wn[1];
    a.st.wz[gid] = wn[2];
    a.st.qw[gid] = q[0];
    a.st.qx[gid] = q[1];
    a.st.qy[gid] = q[2];
    a.st.qz[gid] = q[3];
  }
  px = wrap1(px, s.mi.L);
  py = wrap1(py, s.mi.L);
  pz = wrap1(pz, s.mi.L);
  a.st.px[gid] = px;
  a.st.py[gid] = py;
  a.st.pz[gid] = pz;
  a.st.pos4[slot] = pack_pos(px, py, pz, i);
  uint4 fix = make_uint4(0u, 0u, 0u, 0u);
  if (a.fixpos) {
    fix = fix_position(px, py, pz, s.mi.L, a.fix_scale);
    a.fixpos[slot] = fix;
  }
  if (a.write_offsets) {
    const int base = r * s.total_sites + s.sb_slot[slot];
    if (sp.centred) {
      a.st.off[base] = make_double4(0.0, 0.0, 0.0, 0.0);
    } else {
      for (int k = 0; k < sp.n_sites; ++k) {
        const D3 o = rotate_exact(q[0], q[1], q[2], q[3], {sp.body[k][0], sp.body[k][1], sp.body[k][2]});
        a.st.off[base + k] = make_double4(o.x, o.y, o.z, 0.0);
      }
    }
  }
  return fix;
}

// engine.cpp:131-142; returns check_finite (model.cpp:288-302)
__device__ __forceinline__ bool kick_one(const StepArgs& a, int gid, bool* frozen = nullptr) {
  const SysDev& s = a.s;
  const int i = gid % s.n;
  // inputs first, then the error flag, then the stores (kick_drift_one)
  const int err = frozen ? *a.error_mol : 0x7fffffff;
  const DevSpecies& sp = s.tab->species[s.ns == 1 ? 0 : s.species_of[i]];
  const double vx0 = a.st.vx[gid], vy0 = a.st.vy[gid], vz0 = a.st.vz[gid];
  double fx0 = a.st.fx[gid], fy0 = a.st.fy[gid], fz0 = a.st.fz[gid];
  const double px = a.st.px[gid], py = a.st.py[gid], pz = a.st.pz[gid];
  const double qw = a.st.qw[gid], qx = a.st.qx[gid], qy = a.st.qy[gid], qz = a.st.qz[gid];
  double tx = a.st.tx[gid], ty = a.st.ty[gid], tz = a.st.tz[gid];
  double w0 = a.st.wx[gid], w1 = a.st.wy[gid], w2 = a.st.wz[gid];
  if (a.frec) {
    const size_t nt = size_t(s.R) * s.n;
    fx0 = add(fx0, a.frec[gid]), fy0 = add(fy0, a.frec[nt + gid]), fz0 = add(fz0, a.frec[2 * nt + gid]);
    tx = add(tx, a.frec[3 * nt + gid]), ty = add(ty, a.frec[4 * nt + gid]), tz = add(tz, a.frec[5 * nt + gid]);
  }
  const double half = mul(0.5, a.dt);
  const double c = __ddiv_rn(half, sp.total_mass);
  const double vx = add(vx0, mul(fx0, c));
  const double vy = add(vy0, mul(fy0, c));
  const double vz = add(vz0, mul(fz0, c));
  if (frozen) {
    *frozen = err != 0x7fffffff;
    if (*frozen) return true;
  }
  a.st.vx[gid] = vx;
  a.st.vy[gid] = vy;
  a.st.vz[gid] = vz;
  if (a.frec) {  // the totals (Engine::state's forces, the next step's first kick)
    a.st.fx[gid] = fx0, a.st.fy[gid] = fy0, a.st.fz[gid] = fz0;
    a.st.tx[gid] = tx, a.st.ty[gid] = ty, a.st.tz[gid] = tz;
  }
  if (sp.rotational_dof > 0) {
    const D3 tb = rotate_inv_exact(qw, qx, qy, qz, {tx, ty, tz});
    if (sp.inertia[0] > 0.0) w0 = add(w0, __ddiv_rn(mul(half, tb.x), sp.inertia[0]));
    if (sp.inertia[1] > 0.0) w1 = add(w1, __ddiv_rn(mul(half, tb.y), sp.inertia[1]));
    if (sp.inertia[2] > 0.0) w2 = add(w2, __ddiv_rn(mul(half, tb.z), sp.inertia[2]));
    a.st.wx[gid] = w0;
    a.st.wy[gid] = w1;
    a.st.wz[gid] = w2;
  }
  return isfinite(px) && isfinite(py) && isfinite(pz) && isfinite(vx) && isfinite(vy) &&
         isfinite(vz) && isfinite(w0) && isfinite(w1) && isfinite(w2) && isfinite(qw);
}

// k_kick's work for one molecule inside a force kernel's row epilogue: its
// force and torque were just written by this thread (engine.cpp:131-142)
__device__ __forceinline__ void fused_kick(const ForceArgs& f, size_t gid) {
  if (*f.error_mol != 0x7fffffff) return;  // state frozen after a failed step
  StepArgs a;
  a.s = f.s;
  a.st = f.st;
  a.dt = f.kick_dt;
  a.error_mol = f.error_mol;
  a.write_offsets = 0;
  a.fixpos = nullptr;
  a.fix_scale = 0.0;
  if (!kick_one(a, int(gid))) atomicMin(f.error_mol, int(gid));
}

// first half of a step: half kick, drift, rotate, wrap, offsets
static __global__ void __launch_bounds__(256) k_kick_drift(StepArgs a) {
  const int gid = blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= a.s.n * a.s.R) return;
  bool frozen;  // state frozen after a failed step
  kick_drift_one(a, gid, &frozen);
}

// second half of a step: half kick + check_finite
static __global__ void __launch_bounds__(256) k_kick(StepArgs a) {
  const int gid = blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= a.s.n * a.s.R) return;
  bool frozen;
  if (!kick_one(a, gid, &frozen)) atomicMin(a.error_mol, gid);
}

// end of step k fused with the start of step k+1 (one launch in the step loop).
// A molecule that fails check_finite stops the run; the others may already
// have started step k+1, so the failing molecule index is recorded and the
// host reports the failure (the reference throws at the end of step k).
static __global__ void __launch_bounds__(256) k_kick_kick_drift(StepArgs a) {
  const int gid = blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= a.s.n * a.s.R) return;
  bool frozen;
  if (!kick_one(a, gid, &frozen)) {
    atomicMin(a.error_mol, gid);
    return;
  }
  if (!frozen) kick_drift_one(a, gid);
}

// wrap (model.cpp:279-286) for set_state
static __global__ void k_wrap(double* p, int count, double L) {
  const int gid = blockIdx.x * blockDim.x + threadIdx.x;
  if (gid < count) p[gid] = wrap1(p[gid], L);
}

// --------------------------------------------------- pair-list compaction
// Prefix-sum compaction of the upper triangle (j > i) of the bit matrix into
// an (i, j) list sorted by i then j: per-row popcounts, then a row scan.
// Pair export (b2md_pair_list): slot row k holds external molecule
// i = perm[k]; its partners l with perm[l] > i are the reference pairs (i, j).
// Rows are counted / filled by external index; the host orders each row's j.
static __global__ void k_pair_count(const uint32_t* mask, const int* perm, int n, int words,
                             int64_t* row_count) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  const uint32_t* row = mask + size_t(k) * words;
  const int i = perm[k];
  int64_t c = 0;
  for (int w = 0; w < words; ++w) {
    uint32_t m = row[w];
    while (m) {
      const int b = __ffs(m) - 1;
      m &= m - 1;
      c += perm[w * 32 + b] > i ? 1 : 0;
    }
  }
  row_count[i] = c;
}

static __global__ void k_pair_fill(const uint32_t* mask, const int* perm, int n, int words,
                            const int64_t* row_start, int32_t* pairs) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  const uint32_t* row = mask + size_t(k) * words;
  const int i = perm[k];
  int64_t o = row_start[i];
  for (int w = 0; w < words; ++w) {
    uint32_t m = row[w];
    while (m) {
      const int b = __ffs(m) - 1;
      m &= m - 1;
      const int j = perm[w * 32 + b];
      if (j > i) {
        pairs[2 * o] = i;
        pairs[2 * o + 1] = j;
        ++o;
      }
    }
  }
}

// ------------------------------------------------------------ thermostat
// kinetic_energy_trans / kinetic_energy_rot (model.cpp:304-319) per replica:
// one CTA per replica, thread-strided partial sums in a fixed order and a
// fixed tree (deterministic; the reference's serial order differs only in
// rounding).  out[r] = {ke_t, ke_r}.
constexpr int kKeThreads = 512;
static __global__ void __launch_bounds__(kKeThreads) k_kinetic(SysDev s, StateDev st, double2* out) {
  __shared__ double red_t[kKeThreads], red_r[kKeThreads];
  const int r = blockIdx.x, tid = threadIdx.x;
  double kt = 0.0, kr = 0.0;
  for (int i = tid; i < s.n; i += kKeThreads) {
    const size_t g = size_t(r) * s.n + i;
    const DevSpecies& sp = s.tab->species[s.ns == 1 ? 0 : s.species_of[i]];
    kt += 0.5 * sp.total_mass * norm2_exact(st.vx[g], st.vy[g], st.vz[g]);
    const double wx = st.wx[g], wy = st.wy[g], wz = st.wz[g];
    kr += 0.5 * (sp.inertia[0] * wx * wx + sp.inertia[1] * wy * wy + sp.inertia[2] * wz * wz);
  }
  red_t[tid] = kt;
  red_r[tid] = kr;
  __syncthreads();
  for (int w = kKeThreads / 2; w > 0; w >>= 1) {
    if (tid < w) {
      red_t[tid] += red_t[tid + w];
      red_r[tid] += red_r[tid + w];
    }
    __syncthreads();
  }
  if (tid == 0) out[r] = make_double2(red_t[0], red_r[0]);
}

// Engine::apply_thermostat (engine.cpp:145-160): isokinetic rescale of the
// translational and (dof_r > 0) rotational velocities to the target T.
// A zero kinetic energy is the reference's NumericalError: error code
// 1 (translational) / 2 (rotational) per replica in err[r], state unchanged.
struct ThermoArgs {
  SysDev s;
  StateDev st;
  const double2* ke;
  int* err;
  double temperature;
  int dof_t, dof_r;
};
static __global__ void k_thermostat(ThermoArgs a) {
  const int gid = blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= a.s.n * a.s.R) return;
  const int r = gid / a.s.n;
  const double2 ke = a.ke[r];
  if (ke.x <= 0.0) {
    if (gid == r * a.s.n) a.err[r] = 1;
    return;
  }
  if (a.dof_r > 0 && ke.y <= 0.0) {
    if (gid == r * a.s.n) a.err[r] = 2;
    return;
  }
  const double st_ = sqrt(0.5 * a.dof_t * a.temperature / ke.x);
  a.st.vx[gid] *= st_;
  a.st.vy[gid] *= st_;
  a.st.vz[gid] *= st_;
  if (a.dof_r > 0) {
    const double sr = sqrt(0.5 * a.dof_r * a.temperature / ke.y);
    a.st.wx[gid] *= sr;
    a.st.wy[gid] *= sr;
    a.st.wz[gid] *= sr;
  }
}

// ------------------------------------------------------- checkpoint state
// Engine::checkpoint_bytes' per-molecule record (engine.cpp:434-440):
// pos.xyz, orient.wxyz, vel.xyz, ang_vel.xyz as 13 f64, molecule-major.
static __global__ void k_pack_state(StateDev st, int n, int r, double* out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const size_t g = size_t(r) * n + i;
  double* o = out + size_t(i) * 13;
  o[0] = st.px[g];
  o[1] = st.py[g];
  o[2] = st.pz[g];
  o[3] = st.qw[g];
  o[4] = st.qx[g];
  o[5] = st.qy[g];
  o[6] = st.qz[g];
  o[7] = st.vx[g];
  o[8] = st.vy[g];
  o[9] = st.vz[g];
  o[10] = st.wx[g];
  o[11] = st.wy[g];
  o[12] = st.wz[g];
}

// Engine::restore_dynamic's state loop (engine.cpp:483-491)
static __global__ void k_unpack_state(StateDev st, int n, int r, const double* in) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const size_t g = size_t(r) * n + i;
  const double* o = in + size_t(i) * 13;
  st.px[g] = o[0];
  st.py[g] = o[1];
  st.pz[g] = o[2];
  st.qw[g] = o[3];
  st.qx[g] = o[4];
  st.qy[g] = o[5];
  st.qz[g] = o[6];
  st.vx[g] = o[7];
  st.vy[g] = o[8];
  st.vz[g] = o[9];
  st.wx[g] = o[10];
  st.wy[g] = o[11];
  st.wz[g] = o[12];
}

// ------------------------------------------------------ spatial ordering
// Sort keys for b2md_ctx::resort: molecules are binned into G x G columns
// along x (cross-section c x c, c^2 = 32 / (rho L): about one 32-slot block
// per column), columns in (z, y) order, molecules by x within a column.  A
// block is then a thin line, which is what the search's per-axis bounding-arc
// cull rejects best, and a row's partners fall in a few runs of consecutive
// words.  Key = (replica, column, x on 2^20 bins); values are global
// molecule indices; the stable radix sort makes the order a deterministic
// function of the positions.
// key = replica | column (cbits) | x (kSortXBits): as few radix digits as the grid needs
constexpr int kSortXBits = 14;
static __global__ void k_sort_keys(const double* px, const double* py, const double* pz, int count,
                            int n, double L, int G, int cbits, unsigned long long* keys, int* vals) {
  const int gid = blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= count) return;
  auto bin = [L](double x, int nb) {
    double f = x / L;
    f -= floor(f);  // wrapped
    const int c = int(f * nb);
    return unsigned(c < 0 ? 0 : (c >= nb ? nb - 1 : c));
  };
  const unsigned long long col = bin(pz[gid], G) * unsigned(G) + bin(py[gid], G);
  keys[gid] = (static_cast<unsigned long long>(gid / n) << (cbits + kSortXBits)) | (col << kSortXBits) |
              bin(px[gid], 1 << kSortXBits);
  vals[gid] = gid;
}

// sorted position p (= r n + k) -> perm, slot_of, species and site count
static __global__ void k_apply_order(const int* sorted_vals, int count, int n, const int* species_of,
                              const DevTables* tab, int* perm, int* slot_of, int* sp_slot,
                              int* nsites_slot) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= count) return;
  const int g = sorted_vals[p];
  const int r = g / n, i = g - r * n;
  perm[p] = i;
  slot_of[g] = p - r * n;
  const int sp = species_of[i];
  sp_slot[p] = sp;
  nsites_slot[p] = tab->species[sp].n_sites;
}

// global exclusive scan -> per-replica slot-ordered first site
static __global__ void k_site_starts(const int* scan, int count, int n, int total_sites, int* sb_slot) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= count) return;
  sb_slot[p] = scan[p] - (p / n) * total_sites;
}

// --------------------------------------------------------------- DFMA peak
static __global__ void k_dfma_peak(double* out, int iters, double a, double b) {
  double x0 = threadIdx.x * 1e-9, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5,
         x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
    x0 = fma(x0, a, b);
    x1 = fma(x1, a, b);
    x2 = fma(x2, a, b);
    x3 = fma(x3, a, b);
    x4 = fma(x4, a, b);
    x5 = fma(x5, a, b);
    x6 = fma(x6, a, b);
    x7 = fma(x7, a, b);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}

}  // namespace b2md
