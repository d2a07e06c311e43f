// b200md device kernels (sm_100a, fp64 CUDA cores).
//
// Per evaluation (ForceField::evaluate, src/parallel.cpp:79-122):
//   k_offsets       site offsets rotate(q, body)            potentials.cpp:106-116
//   k_search        COM minimum-image partner search        potentials.cpp:156-158, 209-213
//                   -> symmetric bit matrix (warp ballots)
//   k_force_single  single-site LJ                          potentials.cpp:148-181
//   k_force_multi   multi-site LJ + charge terms + torques  potentials.cpp:218-283
//   k_ewald_*       reciprocal space                        ewald.cpp:107-180
//   k_reduce_sums   fixed-order scalar reduction            parallel.cpp:93-95
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
  double *ox, *oy, *oz;  // site offsets, R * total_sites
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
};

// ------------------------------------------------------------ site offsets
// build_scene (potentials.cpp:106-116): off = rotate(orient, body_pos); a single
// centred site has offset exactly 0.
__global__ void k_offsets(SysDev s, StateDev st) {
  const int gid = blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= s.n * s.R) return;
  const int r = gid / s.n, i = gid - r * s.n;
  const DevSpecies& sp = s.tab->species[s.species_of[i]];
  const int base = r * s.total_sites + s.site_begin[i];
  if (sp.centred) {
    st.ox[base] = 0.0;
    st.oy[base] = 0.0;
    st.oz[base] = 0.0;
    return;
  }
  const double qw = st.qw[gid], qx = st.qx[gid], qy = st.qy[gid], qz = st.qz[gid];
  for (int k = 0; k < sp.n_sites; ++k) {
    const D3 o = rotate_exact(qw, qx, qy, qz, {sp.body[k][0], sp.body[k][1], sp.body[k][2]});
    st.ox[base + k] = o.x;
    st.oy[base + k] = o.y;
    st.oz[base + k] = o.z;
  }
}

// ----------------------------------------------------------- partner search
// One CTA = one super-tile (SI, SJ), SI <= SJ, of ST x ST 32-molecule tiles;
// warp w owns tile row I = SI*ST + w.  Lane <-> j (register), i broadcast from
// shared memory.  Each candidate runs the reference's exact COM test; the
// warp ballot of a fixed i over 32 j is the U word (row i, column tile J), and
// each lane's bits over the 32 i of tile I form the transposed L word (row j,
// column tile I).  Words are staged in shared memory and stored as whole
// 32-byte sectors of the row-major bit matrix M[r][row][word].
struct SearchArgs {
  SysDev s;
  const double *px, *py, *pz;
  uint32_t* mask;                // R * n_pad * words
  const uint32_t* super_tiles;   // (SI << 16) | SJ, this rank's list
  double rc2;                    // single-species COM radius^2
};

template <int ST, bool MULTI>
__global__ void __launch_bounds__(ST * 32) k_search(SearchArgs a) {
  constexpr int T = ST * 32;
  __shared__ double ix[T], iy[T], iz[T];
  __shared__ double jx[T], jy[T], jz[T];
  __shared__ int ispec[MULTI ? T : 1], jspec[MULTI ? T : 1];
  __shared__ double rmax2_s[MULTI ? kMaxSpecies * kMaxSpecies : 1];
  __shared__ uint32_t wu[T][ST + (ST == 1 ? 0 : 0)];
  __shared__ uint32_t wl[T][ST];

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

  {
    const int i = ibase + tid, j = jbase + tid;
    ix[tid] = i < n ? a.px[roff + i] : 0.0;
    iy[tid] = i < n ? a.py[roff + i] : 0.0;
    iz[tid] = i < n ? a.pz[roff + i] : 0.0;
    jx[tid] = j < n ? a.px[roff + j] : 0.0;
    jy[tid] = j < n ? a.py[roff + j] : 0.0;
    jz[tid] = j < n ? a.pz[roff + j] : 0.0;
    if constexpr (MULTI) {
      ispec[tid] = i < n ? s.species_of[i] : 0;
      jspec[tid] = j < n ? s.species_of[j] : 0;
      for (int k = tid; k < s.ns * s.ns; k += T) rmax2_s[k] = s.tab->pair[k].rmax2;
    }
#pragma unroll
    for (int c = 0; c < ST; ++c) {
      wu[tid][c] = 0u;
      wl[tid][c] = 0u;
    }
  }
  __syncthreads();

  const MinImage mi = s.mi;
  const int I = warp;  // local tile row
  const int ilim = n - (ibase + I * 32);  // rows of this tile that exist
  for (int c = diag ? I : 0; c < ST; ++c) {
    const int jl = c * 32 + lane;
    const int jg = jbase + jl;
    const double xj = jx[jl], yj = jy[jl], zj = jz[jl];
    const int sj = MULTI ? jspec[jl] : 0;
    const bool jvalid = jg < n;
    uint32_t lword = 0u, uword = 0u;
    const bool diag_tile = diag && c == I;
#pragma unroll 4
    for (int ii = 0; ii < 32; ++ii) {
      const int il = I * 32 + ii;
      const double dx = min_image(sub(ix[il], xj), mi);
      const double dy = min_image(sub(iy[il], yj), mi);
      const double dz = min_image(sub(iz[il], zj), mi);
      const double r2 = norm2_exact(dx, dy, dz);
      double lim;
      if constexpr (MULTI)
        lim = rmax2_s[ispec[il] * s.ns + sj];
      else
        lim = a.rc2;
      bool pass = r2 < lim && jvalid && ii < ilim;
      if (diag_tile) pass = pass && lane > ii;
      const uint32_t b = __ballot_sync(0xffffffffu, pass);
      if (lane == ii) uword = b;
      lword |= uint32_t(pass) << ii;
    }
    wu[I * 32 + lane][c] = uword;
    wl[c * 32 + lane][I] = lword;
  }
  __syncthreads();

  // store: rows of tile-row block SI get columns SJ*ST.. (wu); rows of block SJ
  // get columns SI*ST.. (wl).  Diagonal super-tiles merge both.
  uint32_t* M = a.mask + size_t(r) * s.n_pad * s.words;
  {
    const int row = tid;
    if (diag) {
      uint32_t* dst = M + size_t(ibase + row) * s.words + SI * ST;
#pragma unroll
      for (int c = 0; c < ST; ++c) dst[c] = wu[row][c] | wl[row][c];
    } else {
      uint32_t* du = M + size_t(ibase + row) * s.words + SJ * ST;
      uint32_t* dl = M + size_t(jbase + row) * s.words + SI * ST;
      if constexpr (ST % 4 == 0) {
#pragma unroll
        for (int c = 0; c < ST; c += 4) {
          *reinterpret_cast<uint4*>(du + c) = make_uint4(wu[row][c], wu[row][c + 1], wu[row][c + 2], wu[row][c + 3]);
          *reinterpret_cast<uint4*>(dl + c) = make_uint4(wl[row][c], wl[row][c + 1], wl[row][c + 2], wl[row][c + 3]);
        }
      } else {
#pragma unroll
        for (int c = 0; c < ST; ++c) {
          du[c] = wu[row][c];
          dl[c] = wl[row][c];
        }
      }
    }
  }
}

// ------------------------------------------------------- single-site forces
// evaluate_range_single_site (potentials.cpp:148-181).  One warp per molecule
// row; lanes stride over the row's bit words.  Pair (lo, hi) is always
// evaluated as R = min_image(com_lo - com_hi) and negated for the hi row.
struct ForceArgs {
  SysDev s;
  StateDev st;
  const uint32_t* mask;
  double* row_scal;  // R * kNumRowScalars * n_pad
  double c12, c6;    // single-species LJ term (PairTable lj[0])
  double rc2;
  double alpha, two_alpha_over_sqrt_pi;
  double rf_r3inv, rf_shift;
  int vderiv;
  int row_begin, row_end;  // rows processed (all rows normally)
};

template <bool MULTI_SPECIES>
__global__ void __launch_bounds__(256) k_force_single(ForceArgs a) {
  const SysDev& s = a.s;
  const int lane = threadIdx.x & 31;
  const int row_g = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int r = blockIdx.y;
  const int i = row_g;
  if (i >= s.n) return;
  const size_t roff = size_t(r) * s.n;
  const double xi = a.st.px[roff + i], yi = a.st.py[roff + i], zi = a.st.pz[roff + i];
  const uint32_t* row = a.mask + (size_t(r) * s.n_pad + i) * s.words;
  const MinImage mi = s.mi;
  double fx = 0, fy = 0, fz = 0, u = 0, vir = 0, s1 = 0, s2 = 0, cnt = 0;
  const int si = MULTI_SPECIES ? s.species_of[i] : 0;
  for (int w = lane; w < s.words; w += 32) {
    uint32_t m = row[w];
    while (m) {
      const int b = __ffs(m) - 1;
      m &= m - 1;
      const int j = w * 32 + b;
      const double xj = a.st.px[roff + j], yj = a.st.py[roff + j], zj = a.st.pz[roff + j];
      const bool lo = i < j;
      double dx, dy, dz;
      if (lo) {
        dx = min_image(sub(xi, xj), mi);
        dy = min_image(sub(yi, yj), mi);
        dz = min_image(sub(zi, zj), mi);
      } else {
        dx = min_image(sub(xj, xi), mi);
        dy = min_image(sub(yj, yi), mi);
        dz = min_image(sub(zj, zi), mi);
      }
      const double r2 = norm2_exact(dx, dy, dz);
      double c12 = a.c12, c6 = a.c6;
      if constexpr (MULTI_SPECIES) {
        const int sj = s.species_of[j];
        const DevPairInfo& pinfo = s.tab->pair[(lo ? si : sj) * s.ns + (lo ? sj : si)];
        c12 = pinfo.lj_count ? s.tab->lj[pinfo.lj_begin].c12 : 0.0;
        c6 = pinfo.lj_count ? s.tab->lj[pinfo.lj_begin].c6 : 0.0;
      }
      const double inv_r2 = 1.0 / r2;
      const double ir6 = inv_r2 * inv_r2 * inv_r2;
      const double a12 = c12 * ir6 * ir6;
      const double a6 = c6 * ir6;
      const double du_r = -12.0 * a12 + 6.0 * a6;
      const double fs = -du_r * inv_r2;
      const double gx = fs * dx, gy = fs * dy, gz = fs * dz;  // force on the lower molecule
      if (lo) {
        fx += gx;
        fy += gy;
        fz += gz;
        u += a12 - a6;
        vir += dx * gx + dy * gy + dz * gz;
        s1 += du_r;
        s2 += 156.0 * a12 - 42.0 * a6;
        cnt += 1.0;
      } else {
        fx -= gx;
        fy -= gy;
        fz -= gz;
      }
    }
  }
  fx = warp_sum(fx);
  fy = warp_sum(fy);
  fz = warp_sum(fz);
  u = warp_sum(u);
  vir = warp_sum(vir);
  s1 = warp_sum(s1);
  s2 = warp_sum(s2);
  cnt = warp_sum(cnt);
  if (lane == 0) {
    a.st.fx[roff + i] = fx;
    a.st.fy[roff + i] = fy;
    a.st.fz[roff + i] = fz;
    double* rs = a.row_scal + size_t(r) * kNumRowScalars * s.n_pad;
    rs[0 * s.n_pad + i] = u;
    rs[1 * s.n_pad + i] = 0.0;
    rs[2 * s.n_pad + i] = 0.0;
    rs[3 * s.n_pad + i] = a.vderiv ? s1 : 0.0;
    rs[4 * s.n_pad + i] = a.vderiv ? s2 : 0.0;
    rs[5 * s.n_pad + i] = vir;
    rs[6 * s.n_pad + i] = cnt;
  }
}

// -------------------------------------------------------- multi-site forces
// evaluate_pair_range general path (potentials.cpp:204-292): COM pair passed
// the search; LJ terms (218-242) and charge terms (244-283) with the site-site
// cutoff decided on canonically computed rv = (R + da) - db, bit-exact.
// METHOD: 0 none, 1 reaction field, 2 ewald real space.
template <int METHOD>
__global__ void __launch_bounds__(256) k_force_multi(ForceArgs a) {
  const SysDev& s = a.s;
  const DevTables* tab = s.tab;
  const int lane = threadIdx.x & 31;
  const int i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int r = blockIdx.y;
  if (i >= s.n) return;
  const size_t roff = size_t(r) * s.n;
  const size_t soff = size_t(r) * s.total_sites;
  const double xi = a.st.px[roff + i], yi = a.st.py[roff + i], zi = a.st.pz[roff + i];
  const int si = s.species_of[i];
  const int bi = s.site_begin[i];
  const uint32_t* row = a.mask + (size_t(r) * s.n_pad + i) * s.words;
  const MinImage mi = s.mi;
  const double rc2 = a.rc2;
  double fx = 0, fy = 0, fz = 0, tx = 0, ty = 0, tz = 0;
  double ulj = 0, uel = 0, urf = 0, vir = 0, s1 = 0, s2 = 0, cnt = 0;
  for (int w = lane; w < s.words; w += 32) {
    uint32_t m = row[w];
    while (m) {
      const int b = __ffs(m) - 1;
      m &= m - 1;
      const int j = w * 32 + b;
      const bool lo = i < j;
      const int l = lo ? i : j, h = lo ? j : i;
      const double xl = lo ? xi : a.st.px[roff + j], yl = lo ? yi : a.st.py[roff + j],
                   zl = lo ? zi : a.st.pz[roff + j];
      const double xh = lo ? a.st.px[roff + j] : xi, yh = lo ? a.st.py[roff + j] : yi,
                   zh = lo ? a.st.pz[roff + j] : zi;
      const double Rx = min_image(sub(xl, xh), mi);
      const double Ry = min_image(sub(yl, yh), mi);
      const double Rz = min_image(sub(zl, zh), mi);
      const double R2 = norm2_exact(Rx, Ry, Rz);
      const int sl = lo ? si : s.species_of[j];
      const int sh = lo ? s.species_of[j] : si;
      const int bl = lo ? bi : s.site_begin[j];
      const int bh = lo ? s.site_begin[j] : bi;
      const DevPairInfo pinfo = tab->pair[sl * s.ns + sh];
      double s1p = 0.0, s2p = 0.0;
      cnt += lo ? 1.0 : 0.0;
      // LJ terms
      for (int q = 0; q < pinfo.lj_count; ++q) {
        const DevLjTerm t = tab->lj[pinfo.lj_begin + q];
        const double dax = a.st.ox[soff + bl + t.a], day = a.st.oy[soff + bl + t.a],
                     daz = a.st.oz[soff + bl + t.a];
        const double dbx = a.st.ox[soff + bh + t.b], dby = a.st.oy[soff + bh + t.b],
                     dbz = a.st.oz[soff + bh + t.b];
        const double rx = sub(add(Rx, dax), dbx), ry = sub(add(Ry, day), dby),
                     rz = sub(add(Rz, daz), dbz);
        const double r2 = norm2_exact(rx, ry, rz);
        if (r2 >= rc2) continue;
        const double inv_r2 = 1.0 / r2;
        const double ir6 = inv_r2 * inv_r2 * inv_r2;
        const double a12 = t.c12 * ir6 * ir6;
        const double a6 = t.c6 * ir6;
        const double du_r = -12.0 * a12 + 6.0 * a6;
        const double fs = -du_r * inv_r2;
        const double gx = fs * rx, gy = fs * ry, gz = fs * rz;
        if (lo) {
          fx += gx;
          fy += gy;
          fz += gz;
          tx += day * gz - daz * gy;
          ty += daz * gx - dax * gz;
          tz += dax * gy - day * gx;
          ulj += a12 - a6;
          vir += Rx * gx + Ry * gy + Rz * gz;
          if (a.vderiv) {
            const double d2u_r2 = 156.0 * a12 - 42.0 * a6;
            const double rvR = rx * Rx + ry * Ry + rz * Rz;
            const double arr = rvR * inv_r2;
            s1p += du_r * arr;
            s2p += d2u_r2 * arr * arr + du_r * inv_r2 * (R2 - rvR * arr);
          }
        } else {
          fx -= gx;
          fy -= gy;
          fz -= gz;
          tx -= dby * gz - dbz * gy;
          ty -= dbz * gx - dbx * gz;
          tz -= dbx * gy - dby * gx;
        }
      }
      if constexpr (METHOD != 0) {
        for (int q = 0; q < pinfo.qq_count; ++q) {
          const DevQTerm t = tab->qq[pinfo.qq_begin + q];
          const double dax = a.st.ox[soff + bl + t.a], day = a.st.oy[soff + bl + t.a],
                       daz = a.st.oz[soff + bl + t.a];
          const double dbx = a.st.ox[soff + bh + t.b], dby = a.st.oy[soff + bh + t.b],
                       dbz = a.st.oz[soff + bh + t.b];
          const double rx = sub(add(Rx, dax), dbx), ry = sub(add(Ry, day), dby),
                       rz = sub(add(Rz, daz), dbz);
          const double r2 = norm2_exact(rx, ry, rz);
          if (r2 >= rc2) continue;
          const double inv_r2 = 1.0 / r2;
          const double rr = sqrt(r2);
          double uu, du_r, d2u_r2 = 0.0, rfu = 0.0;
          if constexpr (METHOD == 2) {
            const double e = erfc(a.alpha * rr) * t.qq / rr;
            const double g = t.qq * a.two_alpha_over_sqrt_pi * exp(-a.alpha * a.alpha * r2);
            uu = e;
            du_r = -(e + g);
          } else {
            uu = t.qq / rr;
            du_r = -uu;
            d2u_r2 = 2.0 * uu;
            const double rf = t.qq * a.rf_r3inv * r2;
            rfu = rf + t.qq * a.rf_shift;
            du_r += 2.0 * rf;
            d2u_r2 += 2.0 * rf;
          }
          const double fs = -du_r * inv_r2;
          const double gx = fs * rx, gy = fs * ry, gz = fs * rz;
          if (lo) {
            fx += gx;
            fy += gy;
            fz += gz;
            tx += day * gz - daz * gy;
            ty += daz * gx - dax * gz;
            tz += dax * gy - day * gx;
            uel += uu;
            urf += rfu;
            vir += Rx * gx + Ry * gy + Rz * gz;
            if (METHOD != 2 && a.vderiv) {
              const double rvR = rx * Rx + ry * Ry + rz * Rz;
              const double arr = rvR * inv_r2;
              s1p += du_r * arr;
              s2p += d2u_r2 * arr * arr + du_r * inv_r2 * (R2 - rvR * arr);
            }
          } else {
            fx -= gx;
            fy -= gy;
            fz -= gz;
            tx -= dby * gz - dbz * gy;
            ty -= dbz * gx - dbx * gz;
            tz -= dbx * gy - dby * gx;
          }
        }
      }
      s1 += s1p;
      s2 += s2p;
    }
  }
  fx = warp_sum(fx);
  fy = warp_sum(fy);
  fz = warp_sum(fz);
  tx = warp_sum(tx);
  ty = warp_sum(ty);
  tz = warp_sum(tz);
  ulj = warp_sum(ulj);
  uel = warp_sum(uel);
  urf = warp_sum(urf);
  vir = warp_sum(vir);
  s1 = warp_sum(s1);
  s2 = warp_sum(s2);
  cnt = warp_sum(cnt);
  if (lane == 0) {
    a.st.fx[roff + i] = fx;
    a.st.fy[roff + i] = fy;
    a.st.fz[roff + i] = fz;
    a.st.tx[roff + i] = tx;
    a.st.ty[roff + i] = ty;
    a.st.tz[roff + i] = tz;
    double* rs = a.row_scal + size_t(r) * kNumRowScalars * s.n_pad;
    rs[0 * s.n_pad + i] = ulj;
    rs[1 * s.n_pad + i] = uel;
    rs[2 * s.n_pad + i] = urf;
    rs[3 * s.n_pad + i] = s1;
    rs[4 * s.n_pad + i] = s2;
    rs[5 * s.n_pad + i] = vir;
    rs[6 * s.n_pad + i] = cnt;
  }
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
  double* uk;           // R * nk_total (0.5 coeff |S|^2)
  int nk_total;
  double two_pi_over_L;
};

__global__ void k_ewald_tables(EwaldArgs a) {
  const int gid = blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= a.nq * a.s.R) return;
  const int r = gid / a.nq, q = gid - r * a.nq;
  const int m = a.q_mol[q];
  const size_t roff = size_t(r) * a.s.n;
  const size_t soff = size_t(r) * a.s.total_sites + a.q_site[q];
  const double p[3] = {a.st.px[roff + m] + a.st.ox[soff], a.st.py[roff + m] + a.st.oy[soff],
                       a.st.pz[roff + m] + a.st.oz[soff]};
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

// ewald.cpp:163-169: one CTA per (k, replica), fixed-order block reduction.
__global__ void __launch_bounds__(256) k_ewald_sk(EwaldArgs a) {
  const int kk = a.k_begin + blockIdx.x;
  const int r = blockIdx.y;
  const DevKVec k = a.kv[kk];
  const int K = a.kmax + 1;
  const double2* base = a.tab + size_t(r) * 3 * K * a.nq;
  double sre = 0.0, sim = 0.0;
  for (int q = threadIdx.x; q < a.nq; q += blockDim.x) {
    const double2 e = site_phase(base, K, a.nq, q, k);
    sre += e.x * a.q_val[q];
    sim += e.y * a.q_val[q];
  }
  __shared__ double red[2][8];
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
    a.uk[size_t(r) * a.nk_total + kk] = 0.5 * k.coeff * (tr * tr + ti * ti);
  }
}

// ewald.cpp:171-178: one warp per molecule with charges; lanes over k; adds
// F and torque = off x F into the (already written) real-space totals.
__global__ void __launch_bounds__(256) k_ewald_force(EwaldArgs a) {
  const int m = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  const int r = blockIdx.y;
  if (m >= a.s.n) return;
  const int q0 = a.mol_qbegin[m], q1 = a.mol_qbegin[m + 1];
  if (q0 == q1) return;
  const int K = a.kmax + 1;
  const double2* base = a.tab + size_t(r) * 3 * K * a.nq;
  const size_t soff = size_t(r) * a.s.total_sites;
  double fx = 0, fy = 0, fz = 0, tx = 0, ty = 0, tz = 0;
  for (int q = q0; q < q1; ++q) {
    const int site = a.q_site[q];
    const double ox = a.st.ox[soff + site], oy = a.st.oy[soff + site], oz = a.st.oz[soff + site];
    const double qv = a.q_val[q];
    double sfx = 0, sfy = 0, sfz = 0;
    for (int kk = a.k_begin + lane; kk < a.k_begin + a.nk; kk += 32) {
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
  fx = warp_sum(fx);
  fy = warp_sum(fy);
  fz = warp_sum(fz);
  tx = warp_sum(tx);
  ty = warp_sum(ty);
  tz = warp_sum(tz);
  if (lane == 0) {
    const size_t roff = size_t(r) * a.s.n;
    a.st.fx[roff + m] += fx;
    a.st.fy[roff + m] += fy;
    a.st.fz[roff + m] += fz;
    a.st.tx[roff + m] += tx;
    a.st.ty[roff + m] += ty;
    a.st.tz[roff + m] += tz;
  }
}

// ------------------------------------------------------- scalar reduction
// One CTA per (scalar, replica): rows in fixed strided order, then a fixed
// tree; u_recip from the per-k energies.
__global__ void __launch_bounds__(256) k_reduce_sums(const double* row_scal, const double* uk,
                                                     int n, int n_pad, int nk_total, int k_begin,
                                                     int k_end, double* sums) {
  const int c = blockIdx.x;  // 0..kNumSums-1
  const int r = blockIdx.y;
  double acc = 0.0;
  if (c < kNumRowScalars) {
    const double* v = row_scal + (size_t(r) * kNumRowScalars + c) * n_pad;
    for (int i = threadIdx.x; i < n; i += blockDim.x) acc += v[i];
  } else if (uk) {
    const double* v = uk + size_t(r) * nk_total;
    for (int k = k_begin + threadIdx.x; k < k_end; k += blockDim.x) acc += v[k];
  }
  __shared__ double red[8];
  acc = warp_sum(acc);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < int(blockDim.x >> 5); ++w) t += red[w];
    sums[size_t(r) * kNumSums + c] = t;
  }
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
__device__ void free_rotate_dev(double q[4], double L[3], const double I[3], double dt) {
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
};

__device__ __forceinline__ double wrap1(double x, double L) {
  return sub(x, mul(L, floor(__ddiv_rn(x, L))));  // model.cpp:282
}

// engine.cpp:107-127 (+ build_scene offsets for the new orientation)
__global__ void __launch_bounds__(256) k_kick_drift(StepArgs a) {
  const int gid = blockIdx.x * blockDim.x + threadIdx.x;
  const SysDev& s = a.s;
  if (gid >= s.n * s.R) return;
  if (*a.error_mol != 0x7fffffff) return;  // state frozen after a failed step
  const int r = gid / s.n, i = gid - r * s.n;
  const DevSpecies& sp = s.tab->species[s.species_of[i]];
  const double dt = a.dt, half = mul(0.5, dt);
  const double c = __ddiv_rn(half, sp.total_mass);
  double vx = add(a.st.vx[gid], mul(a.st.fx[gid], c));
  double vy = add(a.st.vy[gid], mul(a.st.fy[gid], c));
  double vz = add(a.st.vz[gid], mul(a.st.fz[gid], c));
  a.st.vx[gid] = vx;
  a.st.vy[gid] = vy;
  a.st.vz[gid] = vz;
  double px = add(a.st.px[gid], mul(vx, dt));
  double py = add(a.st.py[gid], mul(vy, dt));
  double pz = add(a.st.pz[gid], mul(vz, dt));
  if (sp.rotational_dof > 0) {
    double q[4] = {a.st.qw[gid], a.st.qx[gid], a.st.qy[gid], a.st.qz[gid]};
    const D3 tb = rotate_inv_exact(q[0], q[1], q[2], q[3], {a.st.tx[gid], a.st.ty[gid], a.st.tz[gid]});
    const double tbv[3] = {tb.x, tb.y, tb.z};
    const double w[3] = {a.st.wx[gid], a.st.wy[gid], a.st.wz[gid]};
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
  if (a.write_offsets) {
    const int base = r * s.total_sites + s.site_begin[i];
    if (sp.centred) {
      a.st.ox[base] = 0.0;
      a.st.oy[base] = 0.0;
      a.st.oz[base] = 0.0;
    } else {
      const double qw = a.st.qw[gid], qx = a.st.qx[gid], qy = a.st.qy[gid], qz = a.st.qz[gid];
      for (int k = 0; k < sp.n_sites; ++k) {
        const D3 o = rotate_exact(qw, qx, qy, qz, {sp.body[k][0], sp.body[k][1], sp.body[k][2]});
        a.st.ox[base + k] = o.x;
        a.st.oy[base + k] = o.y;
        a.st.oz[base + k] = o.z;
      }
    }
  }
}

// engine.cpp:131-142
__global__ void __launch_bounds__(256) k_kick(StepArgs a) {
  const int gid = blockIdx.x * blockDim.x + threadIdx.x;
  const SysDev& s = a.s;
  if (gid >= s.n * s.R) return;
  if (*a.error_mol != 0x7fffffff) return;
  const int i = gid % s.n;
  const DevSpecies& sp = s.tab->species[s.species_of[i]];
  const double half = mul(0.5, a.dt);
  const double c = __ddiv_rn(half, sp.total_mass);
  const double vx = add(a.st.vx[gid], mul(a.st.fx[gid], c));
  const double vy = add(a.st.vy[gid], mul(a.st.fy[gid], c));
  const double vz = add(a.st.vz[gid], mul(a.st.fz[gid], c));
  a.st.vx[gid] = vx;
  a.st.vy[gid] = vy;
  a.st.vz[gid] = vz;
  double w0 = a.st.wx[gid], w1 = a.st.wy[gid], w2 = a.st.wz[gid];
  if (sp.rotational_dof > 0) {
    const D3 tb = rotate_inv_exact(a.st.qw[gid], a.st.qx[gid], a.st.qy[gid], a.st.qz[gid],
                                   {a.st.tx[gid], a.st.ty[gid], a.st.tz[gid]});
    if (sp.inertia[0] > 0.0) w0 = add(w0, __ddiv_rn(mul(half, tb.x), sp.inertia[0]));
    if (sp.inertia[1] > 0.0) w1 = add(w1, __ddiv_rn(mul(half, tb.y), sp.inertia[1]));
    if (sp.inertia[2] > 0.0) w2 = add(w2, __ddiv_rn(mul(half, tb.z), sp.inertia[2]));
    a.st.wx[gid] = w0;
    a.st.wy[gid] = w1;
    a.st.wz[gid] = w2;
  }
  // check_finite (model.cpp:288-302)
  const bool ok = isfinite(a.st.px[gid]) && isfinite(a.st.py[gid]) && isfinite(a.st.pz[gid]) &&
                  isfinite(vx) && isfinite(vy) && isfinite(vz) && isfinite(w0) && isfinite(w1) &&
                  isfinite(w2) && isfinite(a.st.qw[gid]);
  if (!ok) atomicMin(a.error_mol, gid);
}

// wrap (model.cpp:279-286) for set_state
__global__ void k_wrap(double* p, int count, double L) {
  const int gid = blockIdx.x * blockDim.x + threadIdx.x;
  if (gid < count) p[gid] = wrap1(p[gid], L);
}

// --------------------------------------------------- pair-list compaction
// Prefix-sum compaction of the upper triangle (j > i) of the bit matrix into
// an (i, j) list sorted by i then j: per-row popcounts, then a row scan.
__global__ void k_pair_count(const uint32_t* mask, int n, int n_pad, int words, int64_t* row_count) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t* row = mask + size_t(i) * words;
  int64_t c = 0;
  const int w0 = i >> 5;
  for (int w = w0; w < words; ++w) {
    uint32_t m = row[w];
    if (w == w0) m &= (i & 31) == 31 ? 0u : (0xffffffffu << ((i & 31) + 1));
    c += __popc(m);
  }
  row_count[i] = c;
}

__global__ void k_pair_fill(const uint32_t* mask, int n, int words, const int64_t* row_start,
                            int32_t* pairs) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t* row = mask + size_t(i) * words;
  int64_t o = row_start[i];
  const int w0 = i >> 5;
  for (int w = w0; w < words; ++w) {
    uint32_t m = row[w];
    if (w == w0) m &= (i & 31) == 31 ? 0u : (0xffffffffu << ((i & 31) + 1));
    while (m) {
      const int b = __ffs(m) - 1;
      m &= m - 1;
      pairs[2 * o] = i;
      pairs[2 * o + 1] = w * 32 + b;
      ++o;
    }
  }
}

// --------------------------------------------------------------- DFMA peak
__global__ void k_dfma_peak(double* out, int iters, double a, double b) {
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
