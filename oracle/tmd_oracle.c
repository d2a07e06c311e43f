/*
 * tmd_oracle.c — TEST INFRASTRUCTURE ONLY (see tmd_oracle.h).
 *
 * Plain-C restatement of the reference tmd force/energy path, serial.  Every
 * expression keeps the reference's evaluation order (C++ left-to-right
 * associativity of the Vec3 operators in include/tmd/geom.hpp), so with
 * -ffp-contract=off the results are bit-identical to the reference compiled
 * with its own Release flags (no FMA: no -march).
 */
#include "tmd_oracle.h"

#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static const double PI = 3.14159265358979323846;

static __thread char g_err[512];

static int fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof g_err, fmt, ap);
  va_end(ap);
  return code;
}

const char* oracle_last_error(void) { return g_err; }

/* ------------------------------------------------------------------ geom.hpp */

typedef struct { double x, y, z; } vec3;
typedef struct { double w, x, y, z; } quat;

static inline vec3 v3(double x, double y, double z) { vec3 r = {x, y, z}; return r; }
static inline vec3 vadd(vec3 a, vec3 b) { return v3(a.x + b.x, a.y + b.y, a.z + b.z); }
static inline vec3 vsub(vec3 a, vec3 b) { return v3(a.x - b.x, a.y - b.y, a.z - b.z); }
static inline vec3 vscale(double s, vec3 a) { return v3(a.x * s, a.y * s, a.z * s); }
/* geom.hpp:29 */
static inline double vdot(vec3 a, vec3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
/* geom.hpp:30-32 */
static inline vec3 vcross(vec3 a, vec3 b) {
  return v3(a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x);
}
static inline double vnorm2(vec3 a) { return vdot(a, a); }
static inline double vnorm(vec3 a) { return sqrt(vnorm2(a)); }
static inline double vget(vec3 a, int k) { return k == 0 ? a.x : (k == 1 ? a.y : a.z); }
static inline void vset(vec3* a, int k, double v) {
  if (k == 0) a->x = v; else if (k == 1) a->y = v; else a->z = v;
}

/* geom.hpp:62-66: v + 2 w t + 2 u x t, t = u x v */
static inline vec3 rotate(quat q, vec3 v) {
  const vec3 u = v3(q.x, q.y, q.z);
  const vec3 t = vcross(u, v);
  return vadd(vadd(v, vscale(2.0 * q.w, t)), vscale(2.0, vcross(u, t)));
}
/* geom.hpp:69-73 */
static inline vec3 rotate_inv(quat q, vec3 v) {
  const vec3 u = v3(-q.x, -q.y, -q.z);
  const vec3 t = vcross(u, v);
  return vadd(vadd(v, vscale(2.0 * q.w, t)), vscale(2.0, vcross(u, t)));
}

/* potentials.hpp:176-181 */
static inline vec3 minimum_image(vec3 d, double box) {
  d.x -= box * nearbyint(d.x / box);
  d.y -= box * nearbyint(d.y / box);
  d.z -= box * nearbyint(d.z / box);
  return d;
}

static inline vec3 load3(const double* a, long i) { return v3(a[3 * i], a[3 * i + 1], a[3 * i + 2]); }
static inline void store3(double* a, long i, vec3 v) {
  a[3 * i] = v.x; a[3 * i + 1] = v.y; a[3 * i + 2] = v.z;
}
static inline quat load4(const double* a, long i) {
  quat q = {a[4 * i], a[4 * i + 1], a[4 * i + 2], a[4 * i + 3]};
  return q;
}

/* ------------------------------------------------------- model.cpp:12-129 */

typedef struct { double a[3][3]; } mat3;

/* model.cpp:12-60 (Jacobi sweep, then stable ascending sort) */
static void jacobi_eigen3(const mat3* m, double vals[3], mat3* vecs) {
  mat3 a = *m;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) vecs->a[i][j] = (i == j) ? 1.0 : 0.0;
  for (int sweep = 0; sweep < 64; ++sweep) {
    double off = 0.0;
    for (int p = 0; p < 3; ++p)
      for (int q = p + 1; q < 3; ++q) off += a.a[p][q] * a.a[p][q];
    if (off < 1e-30) break;
    for (int p = 0; p < 3; ++p) {
      for (int q = p + 1; q < 3; ++q) {
        if (fabs(a.a[p][q]) < 1e-300) continue;
        const double theta = (a.a[q][q] - a.a[p][p]) / (2.0 * a.a[p][q]);
        const double t = (theta >= 0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
        const double c = 1.0 / sqrt(t * t + 1.0);
        const double s = t * c;
        for (int k = 0; k < 3; ++k) {
          const double akp = a.a[k][p], akq = a.a[k][q];
          a.a[k][p] = c * akp - s * akq;
          a.a[k][q] = s * akp + c * akq;
        }
        for (int k = 0; k < 3; ++k) {
          const double apk = a.a[p][k], aqk = a.a[q][k];
          a.a[p][k] = c * apk - s * aqk;
          a.a[q][k] = s * apk + c * aqk;
        }
        for (int k = 0; k < 3; ++k) {
          const double vkp = vecs->a[k][p], vkq = vecs->a[k][q];
          vecs->a[k][p] = c * vkp - s * vkq;
          vecs->a[k][q] = s * vkp + c * vkq;
        }
      }
    }
  }
  /* std::sort on 3 keys is an insertion sort: stable for equal keys */
  int order[3] = {0, 1, 2};
  for (int i = 1; i < 3; ++i) {
    const int v = order[i];
    int j = i;
    while (j > 0 && a.a[v][v] < a.a[order[j - 1]][order[j - 1]]) {
      order[j] = order[j - 1];
      --j;
    }
    order[j] = v;
  }
  mat3 sorted = *vecs;
  for (int j = 0; j < 3; ++j) {
    vals[j] = a.a[order[j]][order[j]];
    for (int i = 0; i < 3; ++i) sorted.a[i][j] = vecs->a[i][order[j]];
  }
  *vecs = sorted;
}

/* model.cpp:68-129 */
int oracle_build_species(const b2md_site* in, int n, b2md_species* sp) {
  if (!in || !sp) return fail(B2MD_INVALID_ARGUMENT, "build_species: null pointer");
  if (n <= 0) return fail(B2MD_MODEL_ERROR, "species: no sites");
  if (n > B2MD_MAX_SITES) return fail(B2MD_MODEL_ERROR, "species: too many sites");
  b2md_site sites[B2MD_MAX_SITES];
  memcpy(sites, in, sizeof(b2md_site) * n);
  double mass = 0.0;
  vec3 com = v3(0, 0, 0);
  for (int k = 0; k < n; ++k) {
    const b2md_site* s = &sites[k];
    if (s->kind == B2MD_SITE_DUMMY && (s->sigma != 0.0 || s->epsilon != 0.0))
      return fail(B2MD_MODEL_ERROR, "species: dummy site with nonzero sigma or epsilon");
    if (s->kind == B2MD_SITE_LJ && s->sigma <= 0.0)
      return fail(B2MD_MODEL_ERROR, "species: LJ site with sigma <= 0");
    if (s->kind == B2MD_SITE_LJ && s->epsilon < 0.0)
      return fail(B2MD_MODEL_ERROR, "species: LJ site with epsilon < 0");
    if (s->mass < 0.0) return fail(B2MD_MODEL_ERROR, "species: negative site mass");
    mass += s->mass;
    com = vadd(com, vscale(s->mass, v3(s->body_pos[0], s->body_pos[1], s->body_pos[2])));
  }
  if (mass <= 0.0) return fail(B2MD_MODEL_ERROR, "species: non-positive total mass");
  com = vscale(1.0 / mass, com);
  for (int k = 0; k < n; ++k) {
    sites[k].body_pos[0] -= com.x;
    sites[k].body_pos[1] -= com.y;
    sites[k].body_pos[2] -= com.z;
  }
  mat3 I;
  memset(&I, 0, sizeof I);
  for (int k = 0; k < n; ++k) {
    const vec3 r = v3(sites[k].body_pos[0], sites[k].body_pos[1], sites[k].body_pos[2]);
    const double m = sites[k].mass;
    const double r2 = vnorm2(r);
    I.a[0][0] += m * (r2 - r.x * r.x);
    I.a[1][1] += m * (r2 - r.y * r.y);
    I.a[2][2] += m * (r2 - r.z * r.z);
    I.a[0][1] -= m * r.x * r.y;
    I.a[0][2] -= m * r.x * r.z;
    I.a[1][2] -= m * r.y * r.z;
  }
  I.a[1][0] = I.a[0][1];
  I.a[2][0] = I.a[0][2];
  I.a[2][1] = I.a[1][2];
  double mom[3];
  mat3 axes;
  jacobi_eigen3(&I, mom, &axes);
  double scale = 0.0;
  for (int k = 0; k < 3; ++k) scale = (scale < mom[k]) ? mom[k] : scale; /* std::max({..,0}) */
  for (int k = 0; k < 3; ++k)
    if (mom[k] < 1e-12 * scale || mom[k] < 1e-300) mom[k] = 0.0;

  memset(sp, 0, sizeof *sp);
  sp->n_sites = n;
  sp->total_mass = mass;
  for (int k = 0; k < 3; ++k) sp->inertia_principal[k] = mom[k];
  for (int k = 0; k < n; ++k) {
    const double x = sites[k].body_pos[0], y = sites[k].body_pos[1], z = sites[k].body_pos[2];
    /* geom.hpp:90-94 mat_tvec */
    sites[k].body_pos[0] = axes.a[0][0] * x + axes.a[1][0] * y + axes.a[2][0] * z;
    sites[k].body_pos[1] = axes.a[0][1] * x + axes.a[1][1] * y + axes.a[2][1] * z;
    sites[k].body_pos[2] = axes.a[0][2] * x + axes.a[1][2] * y + axes.a[2][2] * z;
    sp->sites[k] = sites[k];
  }
  for (int k = 0; k < n; ++k) {
    sp->net_charge += sites[k].q;
    const double e = vnorm(v3(sites[k].body_pos[0], sites[k].body_pos[1], sites[k].body_pos[2]));
    if (sp->max_extent < e) sp->max_extent = e;
  }
  for (int k = 0; k < 3; ++k)
    if (sp->inertia_principal[k] > 0.0) ++sp->rotational_dof;
  return B2MD_OK;
}

/* ------------------------------------------------------- ewald.cpp:8-28 */
int oracle_ewald_tune(double delta, double cutoff, double box_length, double* alpha_out,
                      int* kmax_out) {
  if (!(delta > 0.0) || delta > 1e-2)
    return fail(B2MD_CONFIG_ERROR, "ewald_tune: accuracy must lie in (0, 1e-2]");
  if (cutoff <= 0.0 || box_length <= 0.0) return fail(B2MD_CONFIG_ERROR, "ewald_tune: bad geometry");
  double lo = 1e-6 / cutoff, hi = 40.0 / cutoff;
  if (erfc(lo * cutoff) < delta)
    return fail(B2MD_CONFIG_ERROR, "ewald_tune: accuracy infeasible for this cutoff");
  for (int it = 0; it < 200; ++it) {
    const double mid = 0.5 * (lo + hi);
    if (erfc(mid * cutoff) > delta) lo = mid; else hi = mid;
  }
  const double alpha = 0.5 * (lo + hi);
  const double x = sqrt(-log(delta));
  int kmax = (int)ceil(alpha * box_length * x / PI);
  if (kmax < 1) kmax = 1;
  *alpha_out = alpha;
  *kmax_out = kmax;
  return B2MD_OK;
}

/* --------------------------------------------------------- force field */

typedef struct { int a, b; double c12, c6; } lj_term;   /* potentials.hpp:80-83 */
typedef struct { int a, b; double qq; } q_term;         /* potentials.hpp:85-88 */
typedef struct { int nlj, nqq; lj_term lj[B2MD_MAX_SITES * B2MD_MAX_SITES];
                 q_term qq[B2MD_MAX_SITES * B2MD_MAX_SITES]; } pair_terms;
typedef struct { int nx, ny, nz; double kx, ky, kz, coeff; } kvec;  /* ewald.hpp:51-55 */

struct oracle_ff {
  int ns, n;
  b2md_species* species;
  int* counts;
  int* species_of;
  int* site_begin;
  int total_sites;
  double box, temperature;
  b2md_ff_options opts;
  /* PairTable potentials.cpp:35-83 */
  double rc, rc2, rf_factor, rf_r3inv, rf_shift, alpha;
  int single_lj_only;
  pair_terms* terms;
  double lrc_k;
  /* Ewald ewald.cpp:30-105 */
  int ewald;
  int kmax;
  double self_plus_intra;
  int nk;
  kvec* kv;
  char warning[256];
  /* per-evaluation scratch */
  double* off; /* site offsets, 3 per site */
};

static int species_of_molecule(const oracle_ff* ff, int mol) {
  int off = 0;
  for (int s = 0; s < ff->ns; ++s) {
    off += ff->counts[s];
    if (mol < off) return s;
  }
  return -1;
}

static int has_charges(const b2md_species* sp) {
  for (int k = 0; k < sp->n_sites; ++k)
    if (sp->sites[k].q != 0.0) return 1;
  return 0;
}

static double total_charge(const oracle_ff* ff) {
  double q = 0.0;
  for (int s = 0; s < ff->ns; ++s) q += ff->counts[s] * ff->species[s].net_charge;
  return q;
}

/* potentials.cpp:7-33 */
static int lj_lrc(const oracle_ff* ff, double cutoff, double* k_out) {
  if (cutoff <= 0.0) return fail(B2MD_CONFIG_ERROR, "lj_lrc: cutoff must be positive");
  double k = 0.0;
  int nt = 0;
  double sig[64], eps[64];
  long cnt[64];
  for (int s = 0; s < ff->ns; ++s)
    for (int q = 0; q < ff->species[s].n_sites; ++q) {
      const b2md_site* st = &ff->species[s].sites[q];
      if (st->kind != B2MD_SITE_CHARGE && st->epsilon > 0.0) {
        if (nt >= 64) return fail(B2MD_CONFIG_ERROR, "lj_lrc: too many site types");
        sig[nt] = st->sigma; eps[nt] = st->epsilon; cnt[nt] = ff->counts[s]; ++nt;
      }
    }
  for (int a = 0; a < nt; ++a)
    for (int b = 0; b < nt; ++b) {
      const double sigma = 0.5 * (sig[a] + sig[b]);
      const double e = sqrt(eps[a] * eps[b]);
      const double sr3 = sigma * sigma * sigma / (cutoff * cutoff * cutoff);
      const double sr9 = sr3 * sr3 * sr3;
      k += (8.0 * PI / 3.0) * (double)cnt[a] * (double)cnt[b] * e * sigma * sigma * sigma *
           (sr9 / 3.0 - sr3);
    }
  *k_out = k;
  return B2MD_OK;
}

/* model.cpp:244-268 */
static int validate(const oracle_ff* ff, int method) {
  int n = 0;
  for (int s = 0; s < ff->ns; ++s) n += ff->counts[s];
  if (n <= 0) return fail(B2MD_CONFIG_ERROR, "composition: no molecules");
  for (int s = 0; s < ff->ns; ++s)
    if (ff->counts[s] < 0) return fail(B2MD_CONFIG_ERROR, "composition: negative molecule count");
  if (ff->box <= 0.0) return fail(B2MD_CONFIG_ERROR, "composition: box length must be positive");
  if (ff->temperature <= 0.0)
    return fail(B2MD_CONFIG_ERROR, "composition: temperature must be positive");
  if (method == B2MD_METHOD_EWALD) {
    if (fabs(total_charge(ff)) > 1e-12)
      return fail(B2MD_CONFIG_ERROR, "ewald requires an electro-neutral system (net charge %f)",
                  total_charge(ff));
  } else if (method == B2MD_METHOD_REACTION_FIELD) {
    for (int s = 0; s < ff->ns; ++s)
      if (fabs(ff->species[s].net_charge) > 1e-12)
        return fail(B2MD_CONFIG_ERROR, "reaction_field requires neutral molecules");
  } else {
    for (int s = 0; s < ff->ns; ++s)
      if (has_charges(&ff->species[s]))
        return fail(B2MD_CONFIG_ERROR,
                    "species has point charges; choose electrostatics = reaction_field or ewald");
  }
  return B2MD_OK;
}

void oracle_ff_destroy(oracle_ff* ff) {
  if (!ff) return;
  free(ff->species); free(ff->counts); free(ff->species_of); free(ff->site_begin);
  free(ff->terms); free(ff->kv); free(ff->off);
  free(ff);
}

/* ForceField ctor parallel.cpp:55-72 -> PairTable potentials.cpp:35-83,
 * lj_lrc, validate, Ewald ewald.cpp:30-105 */
int oracle_ff_create(const b2md_composition* comp, const b2md_ff_options* opts, oracle_ff** out) {
  if (!comp || !opts || !out) return fail(B2MD_INVALID_ARGUMENT, "ff_create: null pointer");
  *out = NULL;
  oracle_ff* ff = (oracle_ff*)calloc(1, sizeof(oracle_ff));
  ff->ns = comp->n_species;
  ff->species = (b2md_species*)calloc(ff->ns > 0 ? ff->ns : 1, sizeof(b2md_species));
  ff->counts = (int*)calloc(ff->ns > 0 ? ff->ns : 1, sizeof(int));
  memcpy(ff->species, comp->species, sizeof(b2md_species) * ff->ns);
  memcpy(ff->counts, comp->counts, sizeof(int) * ff->ns);
  ff->box = comp->box_length;
  ff->temperature = comp->temperature;
  ff->opts = *opts;
  int rc;
  const double cutoff = opts->cutoff;
  const int method = opts->method;
  /* PairTable ctor */
  if (cutoff <= 0.0) { rc = fail(B2MD_CONFIG_ERROR, "pair table: cutoff must be positive"); goto bad; }
  if (cutoff > 0.5 * comp->box_length + 1e-12) {
    rc = fail(B2MD_CONFIG_ERROR, "pair table: cutoff %f exceeds half the box length %f", cutoff,
              0.5 * comp->box_length);
    goto bad;
  }
  ff->rc = cutoff;
  ff->rc2 = cutoff * cutoff;
  if (method == B2MD_METHOD_REACTION_FIELD) {
    const double e = opts->eps_rf;
    if (!(e > 1.0) && !isinf(e)) { rc = fail(B2MD_CONFIG_ERROR, "reaction field: epsilon_rf must exceed 1"); goto bad; }
    ff->rf_factor = isinf(e) ? 0.5 : (e - 1.0) / (2.0 * e + 1.0);  /* potentials.hpp:49-52 */
    ff->rf_r3inv = ff->rf_factor / (cutoff * cutoff * cutoff);
    ff->rf_shift = -(1.0 + ff->rf_factor) / cutoff;
  }
  const double alpha = (method == B2MD_METHOD_EWALD && opts->has_ewald) ? opts->ewald_alpha : 0.0;
  ff->alpha = alpha;
  if (method == B2MD_METHOD_EWALD && alpha <= 0.0) {
    rc = fail(B2MD_CONFIG_ERROR, "pair table: ewald method requires alpha > 0");
    goto bad;
  }
  ff->terms = (pair_terms*)calloc((size_t)ff->ns * ff->ns, sizeof(pair_terms));
  for (int sa = 0; sa < ff->ns; ++sa)
    for (int sb = 0; sb < ff->ns; ++sb) {
      pair_terms* t = &ff->terms[sa * ff->ns + sb];
      const b2md_species* A = &ff->species[sa];
      const b2md_species* B = &ff->species[sb];
      for (int ia = 0; ia < A->n_sites; ++ia)
        for (int ib = 0; ib < B->n_sites; ++ib) {
          const b2md_site* a = &A->sites[ia];
          const b2md_site* b = &B->sites[ib];
          if (a->kind != B2MD_SITE_CHARGE && b->kind != B2MD_SITE_CHARGE) {
            const double eps = sqrt(a->epsilon * b->epsilon);
            if (eps > 0.0) {
              const double sigma = 0.5 * (a->sigma + b->sigma);
              const double s3 = sigma * sigma * sigma;
              const double s6 = s3 * s3;
              lj_term lt = {ia, ib, 4.0 * eps * s6 * s6, 4.0 * eps * s6};
              t->lj[t->nlj++] = lt;
            }
          }
          if (method != B2MD_METHOD_NONE && a->q != 0.0 && b->q != 0.0) {
            q_term qt = {ia, ib, a->q * b->q};
            t->qq[t->nqq++] = qt;
          }
        }
    }
  ff->single_lj_only = 1;
  for (int s = 0; s < ff->ns; ++s)
    if (ff->species[s].n_sites != 1 || ff->species[s].sites[0].kind != B2MD_SITE_LJ)
      ff->single_lj_only = 0;
  /* lj_lrc */
  if ((rc = lj_lrc(ff, cutoff, &ff->lrc_k)) != B2MD_OK) goto bad;
  /* comp.validate */
  if (ff->ns <= 0) { rc = fail(B2MD_CONFIG_ERROR, "composition: no molecules"); goto bad; }
  if ((rc = validate(ff, method)) != B2MD_OK) goto bad;
  /* scene indexing (potentials.cpp:94-104) */
  ff->n = 0;
  for (int s = 0; s < ff->ns; ++s) ff->n += ff->counts[s];
  ff->species_of = (int*)malloc(sizeof(int) * ff->n);
  ff->site_begin = (int*)malloc(sizeof(int) * (ff->n + 1));
  ff->total_sites = 0;
  for (int i = 0; i < ff->n; ++i) {
    const int s = species_of_molecule(ff, i);
    ff->species_of[i] = s;
    ff->site_begin[i] = ff->total_sites;
    ff->total_sites += ff->species[s].n_sites;
  }
  ff->site_begin[ff->n] = ff->total_sites;
  ff->off = (double*)malloc(sizeof(double) * 3 * (ff->total_sites + 1));
  ff->opts.volume_derivatives = opts->volume_derivatives ? 1 : 0;
  if (method == B2MD_METHOD_EWALD) {
    if (!opts->has_ewald) { rc = fail(B2MD_CONFIG_ERROR, "force field: ewald method without ewald parameters"); goto bad; }
    if (opts->workers != 1) {
      rc = fail(B2MD_CONFIG_ERROR, "force field: ewald summation runs single-threaded (worker count must be 1)");
      goto bad;
    }
    /* Ewald ctor ewald.cpp:30-105 */
    ff->ewald = 1;
    ff->kmax = opts->ewald_kmax;
    if (alpha <= 0.0) { rc = fail(B2MD_CONFIG_ERROR, "ewald: alpha must be positive"); goto bad; }
    if (ff->kmax < 1) { rc = fail(B2MD_CONFIG_ERROR, "ewald: kmax must be at least 1"); goto bad; }
    if (fabs(total_charge(ff)) > 1e-12) { rc = fail(B2MD_CONFIG_ERROR, "ewald: system is not electro-neutral"); goto bad; }
    const double L = ff->box;
    const double tail = exp(-pow(PI * ff->kmax / (alpha * L), 2));
    if (tail > 1e-2)
      snprintf(ff->warning, sizeof ff->warning,
               "ewald: reciprocal truncation estimate %f at kmax = %d looks too coarse", tail, ff->kmax);
    double sum_q2 = 0.0, intra = 0.0;
    for (int s = 0; s < ff->ns; ++s) {
      const b2md_species* sp = &ff->species[s];
      const long n = ff->counts[s];
      int ch[B2MD_MAX_SITES], nch = 0;
      for (int k = 0; k < sp->n_sites; ++k)
        if (sp->sites[k].q != 0.0) ch[nch++] = k;
      for (int a = 0; a < nch; ++a) sum_q2 += n * sp->sites[ch[a]].q * sp->sites[ch[a]].q;
      double corr = 0.0;
      for (int a = 0; a < nch; ++a)
        for (int b = a + 1; b < nch; ++b) {
          const b2md_site* A = &sp->sites[ch[a]];
          const b2md_site* B = &sp->sites[ch[b]];
          const vec3 d = vsub(v3(A->body_pos[0], A->body_pos[1], A->body_pos[2]),
                              v3(B->body_pos[0], B->body_pos[1], B->body_pos[2]));
          const double r = vnorm(d);
          const double qq = A->q * B->q;
          if (r < 1e-12)
            corr += qq * 2.0 * alpha / sqrt(PI);
          else
            corr += qq * erf(alpha * r) / r;
        }
      intra += n * corr;
    }
    ff->self_plus_intra = -alpha / sqrt(PI) * sum_q2 - intra;
    const double two_pi_over_L = 2.0 * PI / L;
    const double volume = L * L * L;
    const int kmax = ff->kmax;
    int cap = 0;
    for (int nx = 0; nx <= kmax; ++nx) cap += (2 * kmax + 1) * (2 * kmax + 1);
    ff->kv = (kvec*)malloc(sizeof(kvec) * (cap + 1));
    ff->nk = 0;
    for (int nx = 0; nx <= kmax; ++nx) {
      const int ny_lo = (nx == 0) ? 0 : -kmax;
      for (int ny = ny_lo; ny <= kmax; ++ny) {
        const int nz_lo = (nx == 0 && ny == 0) ? 1 : -kmax;
        for (int nz = nz_lo; nz <= kmax; ++nz) {
          const long n2 = (long)nx * nx + (long)ny * ny + (long)nz * nz;
          if (n2 == 0 || n2 > (long)kmax * kmax) continue;
          kvec k;
          k.nx = nx; k.ny = ny; k.nz = nz;
          k.kx = two_pi_over_L * nx;
          k.ky = two_pi_over_L * ny;
          k.kz = two_pi_over_L * nz;
          const double k2 = k.kx * k.kx + k.ky * k.ky + k.kz * k.kz;
          k.coeff = 2.0 * (4.0 * PI / volume) * exp(-k2 / (4.0 * alpha * alpha)) / k2;
          ff->kv[ff->nk++] = k;
        }
      }
    }
    ff->opts.volume_derivatives = 0; /* parallel.cpp:68 */
  }
  *out = ff;
  return B2MD_OK;
bad:
  oracle_ff_destroy(ff);
  return rc;
}

const char* oracle_ff_warning(const oracle_ff* ff) { return ff ? ff->warning : ""; }
int oracle_ff_kvector_count(const oracle_ff* ff) { return ff ? ff->nk : 0; }
int oracle_ff_molecules(const oracle_ff* ff) { return ff ? ff->n : 0; }

/* build_scene site offsets, potentials.cpp:106-116 */
static void build_offsets(oracle_ff* ff, const double* orient) {
  for (int i = 0; i < ff->n; ++i) {
    const b2md_species* sp = &ff->species[ff->species_of[i]];
    const int base = ff->site_begin[i];
    const vec3 b0 = v3(sp->sites[0].body_pos[0], sp->sites[0].body_pos[1], sp->sites[0].body_pos[2]);
    if (sp->n_sites == 1 && vnorm2(b0) == 0.0) {
      store3(ff->off, base, v3(0, 0, 0));
    } else {
      const quat q = load4(orient, i);
      for (int k = 0; k < sp->n_sites; ++k) {
        const vec3 b = v3(sp->sites[k].body_pos[0], sp->sites[k].body_pos[1], sp->sites[k].body_pos[2]);
        store3(ff->off, base + k, rotate(q, b));
      }
    }
  }
}

/* EvalAccum potentials.hpp:144-166 */
typedef struct {
  double* force;
  double* torque;
  double u_lj, u_elec_real, u_rf, s1, s2, virial;
  long com_pairs;
} accum;

static long pair_base(long i, long n) { return i * n - i * (i + 1) / 2; }

/* unflatten_pair potentials.cpp:133-143 */
static void unflatten_pair(long p, int n, int* io, int* jo) {
  const long pc = (long)n * (n - 1) / 2;
  long i = (long)(n - 2 - floor((sqrt(8.0 * (pc - 1 - p) + 1.0) - 1.0) / 2.0));
  if (i < 0) i = 0;
  while (i > 0 && pair_base(i, n) > p) --i;
  while (pair_base(i + 1, n) <= p) ++i;
  *io = (int)i;
  *jo = (int)(p - pair_base(i, n)) + (int)i + 1;
}

static inline void acc_add(double* a, int i, vec3 f) {
  a[3 * i] += f.x; a[3 * i + 1] += f.y; a[3 * i + 2] += f.z;
}
static inline void acc_sub(double* a, int i, vec3 f) {
  a[3 * i] -= f.x; a[3 * i + 1] -= f.y; a[3 * i + 2] -= f.z;
}

/* potentials.cpp:148-181 */
static void range_single_site(oracle_ff* ff, const double* pos, long first, long last, accum* acc) {
  const int n = ff->n;
  const double box = ff->box;
  const double rc2 = ff->rc2;
  const int vderiv = ff->opts.volume_derivatives;
  int i, j;
  unflatten_pair(first, n, &i, &j);
  for (long p = first; p < last; ++p) {
    const vec3 rv = minimum_image(vsub(load3(pos, i), load3(pos, j)), box);
    const double r2 = vnorm2(rv);
    if (r2 < rc2) {
      const lj_term* t = &ff->terms[ff->species_of[i] * ff->ns + ff->species_of[j]].lj[0];
      const double inv_r2 = 1.0 / r2;
      const double ir6 = inv_r2 * inv_r2 * inv_r2;
      const double a12 = t->c12 * ir6 * ir6;
      const double a6 = t->c6 * ir6;
      acc->u_lj += a12 - a6;
      const double du_r = -12.0 * a12 + 6.0 * a6;
      const double fscale = -du_r * inv_r2;
      const vec3 f = vscale(fscale, rv);
      acc_add(acc->force, i, f);
      acc_sub(acc->force, j, f);
      acc->virial += vdot(rv, f);
      if (vderiv) {
        acc->s1 += du_r;
        acc->s2 += 156.0 * a12 - 42.0 * a6;
      }
      acc->com_pairs++;
    }
    if (++j == n) { ++i; j = i + 1; }
  }
}

/* potentials.cpp:185-293 */
static void evaluate_pair_range(oracle_ff* ff, const double* pos, long first, long last, accum* acc) {
  if (first >= last) return;
  if (ff->single_lj_only && ff->opts.method != B2MD_METHOD_EWALD) {
    range_single_site(ff, pos, first, last, acc);
    return;
  }
  const int n = ff->n;
  const double box = ff->box;
  const double rc2 = ff->rc2;
  const double rc = ff->rc;
  const int vderiv = ff->opts.volume_derivatives;
  const int method = ff->opts.method;
  const double alpha = ff->alpha;
  const double two_alpha_over_sqrt_pi = 2.0 * alpha / sqrt(PI);
  double reach[64];
  for (int s = 0; s < ff->ns && s < 64; ++s) reach[s] = ff->species[s].max_extent;
  int i, j;
  unflatten_pair(first, n, &i, &j);
  for (long p = first; p < last; ++p) {
    const vec3 R = minimum_image(vsub(load3(pos, i), load3(pos, j)), box);
    const double R2 = vnorm2(R);
    const int si = ff->species_of[i], sj = ff->species_of[j];
    const double rmax = rc + reach[si] + reach[sj];
    if (R2 < rmax * rmax) {
      const pair_terms* terms = &ff->terms[si * ff->ns + sj];
      const int base_i = ff->site_begin[i], base_j = ff->site_begin[j];
      double s1_pair = 0.0, s2_pair = 0.0;
      acc->com_pairs++;
      for (int q = 0; q < terms->nlj; ++q) {
        const lj_term* t = &terms->lj[q];
        const vec3 da = load3(ff->off, base_i + t->a);
        const vec3 db = load3(ff->off, base_j + t->b);
        const vec3 rv = vsub(vadd(R, da), db);
        const double r2 = vnorm2(rv);
        if (r2 >= rc2) continue;
        const double inv_r2 = 1.0 / r2;
        const double ir6 = inv_r2 * inv_r2 * inv_r2;
        const double a12 = t->c12 * ir6 * ir6;
        const double a6 = t->c6 * ir6;
        acc->u_lj += a12 - a6;
        const double du_r = -12.0 * a12 + 6.0 * a6;
        const double d2u_r2 = 156.0 * a12 - 42.0 * a6;
        const vec3 f = vscale(-du_r * inv_r2, rv);
        acc_add(acc->force, i, f);
        acc_sub(acc->force, j, f);
        acc_add(acc->torque, i, vcross(da, f));
        acc_sub(acc->torque, j, vcross(db, f));
        acc->virial += vdot(R, f);
        if (vderiv) {
          const double arr = vdot(rv, R) * inv_r2;
          s1_pair += du_r * arr;
          s2_pair += d2u_r2 * arr * arr + du_r * inv_r2 * (R2 - vdot(rv, R) * arr);
        }
      }
      for (int q = 0; q < terms->nqq; ++q) {
        const q_term* t = &terms->qq[q];
        const vec3 da = load3(ff->off, base_i + t->a);
        const vec3 db = load3(ff->off, base_j + t->b);
        const vec3 rv = vsub(vadd(R, da), db);
        const double r2 = vnorm2(rv);
        if (r2 >= rc2) continue;
        const double inv_r2 = 1.0 / r2;
        const double r = sqrt(r2);
        double u, du_r, d2u_r2;
        if (method == B2MD_METHOD_EWALD) {
          const double e = erfc(alpha * r) * t->qq / r;
          const double g = t->qq * two_alpha_over_sqrt_pi * exp(-alpha * alpha * r2);
          u = e;
          du_r = -(e + g);
          d2u_r2 = 0.0;
          acc->u_elec_real += u;
        } else {
          u = t->qq / r;
          du_r = -u;
          d2u_r2 = 2.0 * u;
          acc->u_elec_real += u;
          if (method == B2MD_METHOD_REACTION_FIELD) {
            const double rf = t->qq * ff->rf_r3inv * r2;
            acc->u_rf += rf + t->qq * ff->rf_shift;
            du_r += 2.0 * rf;
            d2u_r2 += 2.0 * rf;
          }
        }
        const vec3 f = vscale(-du_r * inv_r2, rv);
        acc_add(acc->force, i, f);
        acc_sub(acc->force, j, f);
        acc_add(acc->torque, i, vcross(da, f));
        acc_sub(acc->torque, j, vcross(db, f));
        acc->virial += vdot(R, f);
        if (vderiv && method != B2MD_METHOD_EWALD) {
          const double arr = vdot(rv, R) * inv_r2;
          s1_pair += du_r * arr;
          s2_pair += d2u_r2 * arr * arr + du_r * inv_r2 * (R2 - vdot(rv, R) * arr);
        }
      }
      acc->s1 += s1_pair;
      acc->s2 += s2_pair;
    }
    if (++j == n) { ++i; j = i + 1; }
  }
}

typedef struct { double re, im; } cplx;
static inline cplx cmul(cplx a, cplx b) {
  cplx r = {a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re};
  return r;
}
static inline cplx cconj(cplx a) { cplx r = {a.re, -a.im}; return r; }

/* Ewald::evaluate ewald.cpp:107-180 over k-vectors [k0, k1) */
static void ewald_evaluate(oracle_ff* ff, const double* pos, int k0, int k1, double* force,
                           double* torque, double* u_recip) {
  *u_recip = 0.0;
  int nq = 0;
  for (int m = 0; m < ff->n; ++m) {
    const b2md_species* sp = &ff->species[ff->species_of[m]];
    for (int k = 0; k < sp->n_sites; ++k)
      if (sp->sites[k].q != 0.0) ++nq;
  }
  if (nq == 0) return;
  int* mol = (int*)malloc(sizeof(int) * nq);
  vec3* poff = (vec3*)malloc(sizeof(vec3) * nq);
  vec3* ps = (vec3*)malloc(sizeof(vec3) * nq);
  double* q = (double*)malloc(sizeof(double) * nq);
  int a = 0;
  for (int m = 0; m < ff->n; ++m) {
    const b2md_species* sp = &ff->species[ff->species_of[m]];
    for (int k = 0; k < sp->n_sites; ++k)
      if (sp->sites[k].q != 0.0) {
        const vec3 off = load3(ff->off, ff->site_begin[m] + k);
        mol[a] = m;
        poff[a] = off;
        ps[a] = vadd(load3(pos, m), off);
        q[a] = sp->sites[k].q;
        ++a;
      }
  }
  const int kmax = ff->kmax;
  const double two_pi_over_L = 2.0 * PI / ff->box;
  const size_t stride = (size_t)(kmax + 1);
  cplx* ex = (cplx*)malloc(sizeof(cplx) * nq * stride);
  cplx* ey = (cplx*)malloc(sizeof(cplx) * nq * stride);
  cplx* ez = (cplx*)malloc(sizeof(cplx) * nq * stride);
  for (a = 0; a < nq; ++a) {
    const size_t base = (size_t)a * stride;
    const cplx one = {1.0, 0.0};
    ex[base] = ey[base] = ez[base] = one;
    const cplx fx = {cos(two_pi_over_L * ps[a].x), sin(two_pi_over_L * ps[a].x)};
    const cplx fy = {cos(two_pi_over_L * ps[a].y), sin(two_pi_over_L * ps[a].y)};
    const cplx fz = {cos(two_pi_over_L * ps[a].z), sin(two_pi_over_L * ps[a].z)};
    for (int k = 1; k <= kmax; ++k) {
      ex[base + k] = cmul(ex[base + k - 1], fx);
      ey[base + k] = cmul(ey[base + k - 1], fy);
      ez[base + k] = cmul(ez[base + k - 1], fz);
    }
  }
  cplx* site_phase = (cplx*)malloc(sizeof(cplx) * nq);
  for (int kk = k0; kk < k1; ++kk) {
    const kvec* kv = &ff->kv[kk];
    cplx S = {0.0, 0.0};
    for (a = 0; a < nq; ++a) {
      const size_t base = (size_t)a * stride;
      cplx e = ex[base + kv->nx];
      const cplx vy = ey[base + abs(kv->ny)];
      e = cmul(e, kv->ny >= 0 ? vy : cconj(vy));
      const cplx vz = ez[base + abs(kv->nz)];
      e = cmul(e, kv->nz >= 0 ? vz : cconj(vz));
      site_phase[a] = e;
      S.re += e.re * q[a];
      S.im += e.im * q[a];
    }
    *u_recip += 0.5 * kv->coeff * (S.re * S.re + S.im * S.im);
    const vec3 kvek = v3(kv->kx, kv->ky, kv->kz);
    for (a = 0; a < nq; ++a) {
      const double im = site_phase[a].im * S.re - site_phase[a].re * S.im;
      const vec3 f = vscale(q[a] * kv->coeff * im, kvek);
      acc_add(force, mol[a], f);
      acc_add(torque, mol[a], vcross(poff[a], f));
    }
  }
  free(site_phase); free(ex); free(ey); free(ez);
  free(mol); free(poff); free(ps); free(q);
}

/* ForceField::evaluate parallel.cpp:79-122 (W = 1) */
int oracle_evaluate(oracle_ff* ff, const double* pos, const double* orient, double* force,
                    double* torque, b2md_energy* energy, b2md_eval_stats* stats) {
  if (!ff || !pos || !orient) return fail(B2MD_INVALID_ARGUMENT, "evaluate: null pointer");
  const int n = ff->n;
  build_offsets(ff, orient);
  accum acc;
  memset(&acc, 0, sizeof acc);
  acc.force = (double*)calloc(3 * (size_t)n, sizeof(double));
  acc.torque = (double*)calloc(3 * (size_t)n, sizeof(double));
  evaluate_pair_range(ff, pos, 0, (long)n * (n - 1) / 2, &acc);
  b2md_energy e;
  memset(&e, 0, sizeof e);
  e.lj = acc.u_lj;
  e.elec_real = acc.u_elec_real;
  e.rf = acc.u_rf;
  const double volume = ff->box * ff->box * ff->box;
  e.lrc = ff->lrc_k / volume;                                           /* potentials.hpp:73 */
  if (ff->opts.volume_derivatives) {
    e.du_dv_explicit = acc.s1 / (3.0 * volume);                         /* potentials.hpp:64-66 */
    e.d2u_dv2_explicit = (acc.s2 - 2.0 * acc.s1) / (9.0 * volume * volume);
    e.du_dv_lrc = -ff->lrc_k / (volume * volume);                       /* potentials.hpp:74-75 */
    e.d2u_dv2_lrc = 2.0 * ff->lrc_k / (volume * volume * volume);
  }
  if (ff->ewald) {
    double u_recip;
    ewald_evaluate(ff, pos, 0, ff->nk, acc.force, acc.torque, &u_recip);
    e.elec_recip = u_recip;
    e.elec_self = ff->self_plus_intra;
  }
  if (force) memcpy(force, acc.force, sizeof(double) * 3 * n);
  if (torque) memcpy(torque, acc.torque, sizeof(double) * 3 * n);
  if (energy) *energy = e;
  if (stats) {
    stats->virial = acc.virial;
    stats->s1 = acc.s1;
    stats->s2 = acc.s2;
    stats->com_pairs = acc.com_pairs;
  }
  free(acc.force);
  free(acc.torque);
  return B2MD_OK;
}

int oracle_evaluate_shard(oracle_ff* ff, const double* pos, const double* orient, int row_begin,
                          int row_end, int k_begin, int k_end, double* force, double* torque,
                          double* sums) {
  if (!ff || !pos || !orient || !force || !torque || !sums)
    return fail(B2MD_INVALID_ARGUMENT, "evaluate_shard: null pointer");
  const int n = ff->n;
  build_offsets(ff, orient);
  accum acc;
  memset(&acc, 0, sizeof acc);
  acc.force = force;
  acc.torque = torque;
  memset(force, 0, sizeof(double) * 3 * n);
  memset(torque, 0, sizeof(double) * 3 * n);
  long i0 = (long)row_begin * 32, i1 = (long)row_end * 32;
  if (i0 > n) i0 = n;
  if (i1 > n) i1 = n;
  evaluate_pair_range(ff, pos, pair_base(i0, n), pair_base(i1, n), &acc);
  double u_recip = 0.0;
  if (ff->ewald && k_end > k_begin) ewald_evaluate(ff, pos, k_begin, k_end, force, torque, &u_recip);
  sums[0] = acc.u_lj; sums[1] = acc.u_elec_real; sums[2] = acc.u_rf; sums[3] = acc.s1;
  sums[4] = acc.s2; sums[5] = acc.virial; sums[6] = u_recip; sums[7] = (double)acc.com_pairs;
  return B2MD_OK;
}

int64_t oracle_pair_list(oracle_ff* ff, const double* pos, int32_t* pairs, int64_t capacity) {
  const int n = ff->n;
  const int single = ff->single_lj_only && ff->opts.method != B2MD_METHOD_EWALD;
  int64_t cnt = 0;
  for (int i = 0; i < n; ++i)
    for (int j = i + 1; j < n; ++j) {
      const vec3 R = minimum_image(vsub(load3(pos, i), load3(pos, j)), ff->box);
      const double R2 = vnorm2(R);
      int pass;
      if (single) {
        pass = R2 < ff->rc2;  /* potentials.cpp:156-158 */
      } else {                /* potentials.cpp:209-213 */
        const double rmax = ff->rc + ff->species[ff->species_of[i]].max_extent +
                            ff->species[ff->species_of[j]].max_extent;
        pass = R2 < rmax * rmax;
      }
      if (pass) {
        if (pairs && cnt < capacity) { pairs[2 * cnt] = i; pairs[2 * cnt + 1] = j; }
        ++cnt;
      }
    }
  return cnt;
}

/* model.cpp:279-286 */
void oracle_wrap(int n, double L, double* pos) {
  for (int i = 0; i < 3 * n; ++i) pos[i] -= L * floor(pos[i] / L);
}

/* engine.cpp:13-19 */
static void permute(int axis, const double q[4], double out[4]) {
  switch (axis) {
    case 1: out[0] = -q[1]; out[1] = q[0]; out[2] = q[3]; out[3] = -q[2]; break;
    case 2: out[0] = -q[2]; out[1] = -q[3]; out[2] = q[0]; out[3] = q[1]; break;
    default: out[0] = -q[3]; out[1] = q[2]; out[2] = -q[1]; out[3] = q[0]; break;
  }
}
static inline double dot4(const double a[4], const double b[4]) {
  return a[0] * b[0] + a[1] * b[1] + a[2] * b[2] + a[3] * b[3];
}

/* engine.cpp:28-59 NO_SQUISH free rotor */
static void free_rotate(double* orient, vec3* ang_mom, const double inertia[3], double dt) {
  double q[4] = {orient[0], orient[1], orient[2], orient[3]};
  double p[4] = {0, 0, 0, 0};
  for (int k = 1; k <= 3; ++k) {
    const double pi_k = vget(*ang_mom, k - 1);
    if (pi_k == 0.0) continue;
    double pq[4];
    permute(k, q, pq);
    for (int c = 0; c < 4; ++c) p[c] += 2.0 * pi_k * pq[c];
  }
  static const int axis_seq[5] = {3, 2, 1, 2, 3};
  const double dt_seq[5] = {0.5 * dt, 0.5 * dt, dt, 0.5 * dt, 0.5 * dt};
  for (int stage = 0; stage < 5; ++stage) {
    const int k = axis_seq[stage];
    const double ik = inertia[k - 1];
    if (ik <= 0.0) continue;
    double pq[4], pp[4];
    permute(k, q, pq);
    const double zeta = dot4(p, pq) / (4.0 * ik);
    const double c = cos(dt_seq[stage] * zeta);
    const double s = sin(dt_seq[stage] * zeta);
    permute(k, p, pp);
    for (int i = 0; i < 4; ++i) {
      q[i] = c * q[i] + s * pq[i];
      p[i] = c * p[i] + s * pp[i];
    }
  }
  for (int k = 1; k <= 3; ++k) {
    double pq[4];
    permute(k, q, pq);
    vset(ang_mom, k - 1, (inertia[k - 1] > 0.0) ? 0.5 * dot4(p, pq) : 0.0);
  }
  const double nrm = sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
  orient[0] = q[0] / nrm; orient[1] = q[1] / nrm; orient[2] = q[2] / nrm; orient[3] = q[3] / nrm;
}

/* engine.cpp:102-143 */
int oracle_step(oracle_ff* ff, double dt, int64_t nsteps, double* pos, double* orient, double* vel,
                double* ang_vel, double* force, double* torque, b2md_energy* energy,
                b2md_eval_stats* stats) {
  if (dt <= 0.0) return fail(B2MD_CONFIG_ERROR, "engine: time step must be positive");
  const int n = ff->n;
  const double half = 0.5 * dt;
  for (int64_t st = 0; st < nsteps; ++st) {
    for (int i = 0; i < n; ++i) {
      const b2md_species* sp = &ff->species[ff->species_of[i]];
      const double s = half / sp->total_mass;
      for (int k = 0; k < 3; ++k) vel[3 * i + k] += s * force[3 * i + k];
      if (sp->rotational_dof > 0) {
        const vec3 tb = rotate_inv(load4(orient, i), load3(torque, i));
        vec3 L = v3(0, 0, 0);
        for (int k = 0; k < 3; ++k) {
          const double ik = sp->inertia_principal[k];
          vset(&L, k, ik > 0.0 ? ik * ang_vel[3 * i + k] + half * vget(tb, k) : 0.0);
        }
        for (int k = 0; k < 3; ++k) pos[3 * i + k] += dt * vel[3 * i + k];
        free_rotate(orient + 4 * i, &L, sp->inertia_principal, dt);
        for (int k = 0; k < 3; ++k)
          ang_vel[3 * i + k] = sp->inertia_principal[k] > 0.0 ? vget(L, k) / sp->inertia_principal[k] : 0.0;
      } else {
        for (int k = 0; k < 3; ++k) pos[3 * i + k] += dt * vel[3 * i + k];
      }
    }
    oracle_wrap(n, ff->box, pos);
    int rc = oracle_evaluate(ff, pos, orient, force, torque, energy, stats);
    if (rc) return rc;
    for (int i = 0; i < n; ++i) {
      const b2md_species* sp = &ff->species[ff->species_of[i]];
      const double s = half / sp->total_mass;
      for (int k = 0; k < 3; ++k) vel[3 * i + k] += s * force[3 * i + k];
      if (sp->rotational_dof > 0) {
        const vec3 tb = rotate_inv(load4(orient, i), load3(torque, i));
        for (int k = 0; k < 3; ++k) {
          const double ik = sp->inertia_principal[k];
          if (ik > 0.0) ang_vel[3 * i + k] += half * vget(tb, k) / ik;
        }
      }
    }
    /* model.cpp:288-302 */
    for (int i = 0; i < n; ++i) {
      int ok = 1;
      for (int k = 0; k < 3; ++k)
        ok = ok && isfinite(pos[3 * i + k]) && isfinite(vel[3 * i + k]) && isfinite(ang_vel[3 * i + k]);
      ok = ok && isfinite(orient[4 * i]);
      if (!ok)
        return fail(B2MD_NUMERICAL_ERROR,
                    "engine step: non-finite state for molecule %d (pos %g %g %g, vel %g %g %g)", i,
                    pos[3 * i], pos[3 * i + 1], pos[3 * i + 2], vel[3 * i], vel[3 * i + 1], vel[3 * i + 2]);
    }
  }
  return B2MD_OK;
}

/* greenkubo.cpp:182-266 */
int oracle_heat_flux(oracle_ff* ff, const double* pos, const double* orient, const double* vel,
                     const double* ang_vel, const double* enthalpy, int n_enthalpy, double* jq) {
  if (!ff || !pos || !orient || !vel || !ang_vel || !jq || (n_enthalpy > 0 && !enthalpy))
    return fail(B2MD_INVALID_ARGUMENT, "heat_flux: null pointer");
  if (n_enthalpy != ff->ns) /* greenkubo.cpp:184-185 */
    return fail(B2MD_CONFIG_ERROR, "heat flux: partial molar enthalpy required for every component");
  const int n = ff->n;
  build_offsets(ff, orient);
  const double rc2 = ff->rc2;
  const int method = ff->opts.method;
  double* pair_u = (double*)calloc((size_t)n, sizeof(double));
  vec3* w_lab = (vec3*)malloc(sizeof(vec3) * (size_t)n);
  for (int i = 0; i < n; ++i) w_lab[i] = rotate(load4(orient, i), load3(ang_vel, i));
  vec3 transport = v3(0, 0, 0);
  for (int i = 0; i < n; ++i) {
    for (int j = i + 1; j < n; ++j) {
      const vec3 R = minimum_image(vsub(load3(pos, i), load3(pos, j)), ff->box);
      const pair_terms* terms = &ff->terms[ff->species_of[i] * ff->ns + ff->species_of[j]];
      const int bi = ff->site_begin[i], bj = ff->site_begin[j];
      double u_pair = 0.0;
      vec3 f_pair = v3(0, 0, 0), gamma_ij = v3(0, 0, 0), gamma_ji = v3(0, 0, 0);
      for (int q = 0; q < terms->nlj; ++q) {
        const lj_term* t = &terms->lj[q];
        const vec3 da = load3(ff->off, bi + t->a), db = load3(ff->off, bj + t->b);
        const vec3 rv = vsub(vadd(R, da), db);
        const double r2 = vnorm2(rv);
        if (r2 >= rc2) continue;
        const double inv_r2 = 1.0 / r2;
        const double ir6 = inv_r2 * inv_r2 * inv_r2;
        const double a12 = t->c12 * ir6 * ir6;
        const double a6 = t->c6 * ir6;
        const double u = a12 - a6, du_dr_r = -12.0 * a12 + 6.0 * a6;
        u_pair += u;
        const vec3 f = vscale(-du_dr_r * inv_r2, rv);
        f_pair = vadd(f_pair, f);
        gamma_ij = vadd(gamma_ij, vcross(da, f));
        gamma_ji = vsub(gamma_ji, vcross(db, f));
      }
      for (int q = 0; q < terms->nqq; ++q) {
        const q_term* t = &terms->qq[q];
        const vec3 da = load3(ff->off, bi + t->a), db = load3(ff->off, bj + t->b);
        const vec3 rv = vsub(vadd(R, da), db);
        const double r2 = vnorm2(rv);
        if (r2 >= rc2) continue;
        const double inv_r2 = 1.0 / r2;
        const double r = sqrt(r2);
        const double u_c = t->qq / r;
        double u = u_c, du_r = -u_c;
        if (method == B2MD_METHOD_REACTION_FIELD) {
          const double rf = t->qq * ff->rf_r3inv * r2;
          u += rf + t->qq * ff->rf_shift;
          du_r += 2.0 * rf;
        }
        u_pair += u;
        const vec3 f = vscale(-du_r * inv_r2, rv);
        f_pair = vadd(f_pair, f);
        gamma_ij = vadd(gamma_ij, vcross(da, f));
        gamma_ji = vsub(gamma_ji, vcross(db, f));
      }
      if (u_pair == 0.0 && f_pair.x == 0.0 && f_pair.y == 0.0 && f_pair.z == 0.0) continue;
      pair_u[i] += u_pair;
      pair_u[j] += u_pair;
      const vec3 vi = load3(vel, i), vj = load3(vel, j);
      transport = vadd(transport, vscale(0.5 * (vdot(f_pair, vi) + vdot(gamma_ij, w_lab[i]) +
                                                vdot(f_pair, vj) - vdot(gamma_ji, w_lab[j])),
                                         R));
    }
  }
  vec3 out = transport;
  for (int i = 0; i < n; ++i) {
    const b2md_species* sp = &ff->species[ff->species_of[i]];
    const vec3 w = load3(ang_vel, i), v = load3(vel, i);
    const double* I = sp->inertia_principal;
    const double e_kin = 0.5 * sp->total_mass * vnorm2(v) +
                         0.5 * (I[0] * w.x * w.x + I[1] * w.y * w.y + I[2] * w.z * w.z);
    out = vadd(out, vscale(e_kin + 0.5 * pair_u[i] - enthalpy[ff->species_of[i]], v));
  }
  jq[0] = out.x;
  jq[1] = out.y;
  jq[2] = out.z;
  free(pair_u);
  free(w_lab);
  return B2MD_OK;
}

/* ------------------------------------------------ RdfHistogram, structure.cpp */

struct oracle_rdf {
  const oracle_ff* ff;
  double bin_width, r_max;
  int bins, n_types;
  int* type_species; /* per type */
  int* type_site;
  int* type_of_site;       /* per (species, site), -1 for charge sites */
  int* species_type_begin; /* ns + 1 */
  uint64_t* counts;        /* n_pairs * bins */
  int64_t snapshots;
};

/* structure.cpp:10-36 */
int oracle_rdf_create(const oracle_ff* ff, double bin_width, double r_max, oracle_rdf** out) {
  if (!ff || !out) return fail(B2MD_INVALID_ARGUMENT, "rdf: null pointer");
  if (bin_width <= 0.0) return fail(B2MD_CONFIG_ERROR, "rdf: bin width must be positive");
  if (r_max > 0.5 * ff->box + 1e-12)
    return fail(B2MD_CONFIG_ERROR, "rdf: r_max exceeds half the box length");
  oracle_rdf* r = (oracle_rdf*)calloc(1, sizeof *r);
  r->ff = ff;
  r->bin_width = bin_width;
  r->r_max = r_max;
  r->bins = (int)ceil(r_max / bin_width);
  int total = 0;
  for (int s = 0; s < ff->ns; ++s) total += ff->species[s].n_sites;
  r->type_of_site = (int*)malloc(sizeof(int) * (size_t)(total > 0 ? total : 1));
  r->type_species = (int*)malloc(sizeof(int) * (size_t)(total > 0 ? total : 1));
  r->type_site = (int*)malloc(sizeof(int) * (size_t)(total > 0 ? total : 1));
  r->species_type_begin = (int*)malloc(sizeof(int) * (size_t)(ff->ns + 1));
  int k_all = 0;
  for (int s = 0; s < ff->ns; ++s) {
    r->species_type_begin[s] = k_all;
    const b2md_species* sp = &ff->species[s];
    for (int k = 0; k < sp->n_sites; ++k, ++k_all) {
      if (sp->sites[k].kind == B2MD_SITE_CHARGE) {
        r->type_of_site[k_all] = -1;
      } else {
        r->type_of_site[k_all] = r->n_types;
        r->type_species[r->n_types] = s;
        r->type_site[r->n_types] = k;
        ++r->n_types;
      }
    }
  }
  r->species_type_begin[ff->ns] = k_all;
  const int t = r->n_types;
  r->counts = (uint64_t*)calloc((size_t)(t * (t + 1) / 2) * (size_t)(r->bins > 0 ? r->bins : 1),
                                sizeof(uint64_t));
  *out = r;
  return B2MD_OK;
}

void oracle_rdf_destroy(oracle_rdf* r) {
  if (!r) return;
  free(r->type_species);
  free(r->type_site);
  free(r->type_of_site);
  free(r->species_type_begin);
  free(r->counts);
  free(r);
}

/* structure.hpp:51-54 */
static int rdf_pair_index(const oracle_rdf* r, int ta, int tb) {
  return ta * r->n_types - ta * (ta + 1) / 2 + tb;
}

/* structure.cpp:38-76 */
int oracle_rdf_accumulate(oracle_rdf* r, const double* pos, const double* orient) {
  if (!r || !pos || !orient) return fail(B2MD_INVALID_ARGUMENT, "rdf: null pointer");
  const oracle_ff* ff = r->ff;
  const int n = ff->n;
  const double r_max2 = r->r_max * r->r_max;
  int cap = 0;
  for (int m = 0; m < n; ++m) cap += ff->species[species_of_molecule(ff, m)].n_sites;
  vec3* site_pos = (vec3*)malloc(sizeof(vec3) * (size_t)(cap > 0 ? cap : 1));
  int* site_type = (int*)malloc(sizeof(int) * (size_t)(cap > 0 ? cap : 1));
  int* mol_begin = (int*)malloc(sizeof(int) * (size_t)(n + 1));
  int ns = 0;
  for (int m = 0; m < n; ++m) {
    mol_begin[m] = ns;
    const int s = species_of_molecule(ff, m);
    const b2md_species* sp = &ff->species[s];
    for (int k = 0; k < sp->n_sites; ++k) {
      const int t = r->type_of_site[r->species_type_begin[s] + k];
      if (t < 0) continue;
      const vec3 b = v3(sp->sites[k].body_pos[0], sp->sites[k].body_pos[1], sp->sites[k].body_pos[2]);
      site_pos[ns] = vadd(load3(pos, m), rotate(load4(orient, m), b));
      site_type[ns] = t;
      ++ns;
    }
  }
  mol_begin[n] = ns;
  for (int mi = 0; mi < n; ++mi) {
    for (int mj = mi + 1; mj < n; ++mj) {
      for (int a = mol_begin[mi]; a < mol_begin[mi + 1]; ++a) {
        for (int b = mol_begin[mj]; b < mol_begin[mj + 1]; ++b) {
          const vec3 d = minimum_image(vsub(site_pos[a], site_pos[b]), ff->box);
          const double d2 = vnorm2(d);
          if (d2 >= r_max2) continue;
          const int bin = (int)(sqrt(d2) / r->bin_width);
          if (bin >= r->bins) continue;
          const int ta = site_type[a] < site_type[b] ? site_type[a] : site_type[b];
          const int tb = site_type[a] < site_type[b] ? site_type[b] : site_type[a];
          ++r->counts[(size_t)rdf_pair_index(r, ta, tb) * (size_t)r->bins + (size_t)bin];
        }
      }
    }
  }
  ++r->snapshots;
  free(site_pos);
  free(site_type);
  free(mol_begin);
  return B2MD_OK;
}

int oracle_rdf_shape(const oracle_rdf* r, int* n_types, int* bins, int* n_pairs) {
  if (!r) return fail(B2MD_INVALID_ARGUMENT, "rdf: null pointer");
  if (n_types) *n_types = r->n_types;
  if (bins) *bins = r->bins;
  if (n_pairs) *n_pairs = r->n_types * (r->n_types + 1) / 2;
  return B2MD_OK;
}

int oracle_rdf_counts(const oracle_rdf* r, uint64_t* counts, int64_t* snapshots) {
  if (!r) return fail(B2MD_INVALID_ARGUMENT, "rdf: null pointer");
  const size_t nc = (size_t)(r->n_types * (r->n_types + 1) / 2) * (size_t)r->bins;
  if (counts) memcpy(counts, r->counts, sizeof(uint64_t) * nc);
  if (snapshots) *snapshots = r->snapshots;
  return B2MD_OK;
}

/* ------------------------------------------------------------- thermostat */

/* model.cpp:304-319 */
int oracle_kinetic_energy(const oracle_ff* ff, const double* vel, const double* ang_vel, double* out) {
  if (!ff || !vel || !ang_vel || !out) return fail(B2MD_INVALID_ARGUMENT, "kinetic_energy: null pointer");
  double kt = 0.0, kr = 0.0;
  for (int i = 0; i < ff->n; ++i) {
    const b2md_species* sp = &ff->species[species_of_molecule(ff, i)];
    kt += 0.5 * sp->total_mass * vnorm2(load3(vel, i));
  }
  for (int i = 0; i < ff->n; ++i) {
    const b2md_species* sp = &ff->species[species_of_molecule(ff, i)];
    const double* I = sp->inertia_principal;
    const vec3 w = load3(ang_vel, i);
    kr += 0.5 * (I[0] * w.x * w.x + I[1] * w.y * w.y + I[2] * w.z * w.z);
  }
  out[0] = kt;
  out[1] = kr;
  return B2MD_OK;
}

/* engine.cpp:145-160 with translational_dof / rotational_dof (model.cpp:321-330) */
int oracle_apply_thermostat(const oracle_ff* ff, double* vel, double* ang_vel) {
  double ke[2];
  int rc = oracle_kinetic_energy(ff, vel, ang_vel, ke);
  if (rc) return rc;
  const double T = ff->temperature;
  const int dof_t = 3 * ff->n - 3;
  if (ke[0] <= 0.0) return fail(B2MD_NUMERICAL_ERROR, "thermostat: zero translational kinetic energy");
  const double scale_t = sqrt(0.5 * dof_t * T / ke[0]);
  for (int i = 0; i < 3 * ff->n; ++i) vel[i] *= scale_t;
  int dof_r = 0;
  for (int s = 0; s < ff->ns; ++s) dof_r += ff->counts[s] * ff->species[s].rotational_dof;
  if (dof_r > 0) {
    if (ke[1] <= 0.0) return fail(B2MD_NUMERICAL_ERROR, "thermostat: zero rotational kinetic energy");
    const double scale_r = sqrt(0.5 * dof_r * T / ke[1]);
    for (int i = 0; i < 3 * ff->n; ++i) ang_vel[i] *= scale_r;
  }
  return B2MD_OK;
}
