// b200md context: device memory, launch sequences, CUDA graphs, host
// transfers, NCCL and the core of the C ABI declared in include/b200md.h
// (samplers.cu holds the heat flux, RDF, thermostat and checkpoint entries).
#include "ctx_internal.cuh"

using namespace b2md;

namespace b2md_host {

thread_local std::string g_err;

int set_err(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

NcclApi g_nccl;

int nccl_load() {
  if (g_nccl.loaded) return B2MD_OK;
  // an explicit library (the Python package points it at the NCCL its PyTorch
  // uses, so both share one), else one already in the process, else the system's
  void* h = nullptr;
  if (const char* path = std::getenv("B2MD_NCCL_LIBRARY")) h = dlopen(path, RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!h) return set_err(B2MD_CUDA_ERROR, std::string("NCCL not available: ") + dlerror());
  auto sym = [&](const char* name) { return dlsym(h, name); };
  g_nccl.GetUniqueId = reinterpret_cast<decltype(g_nccl.GetUniqueId)>(sym("ncclGetUniqueId"));
  g_nccl.CommInitRank = reinterpret_cast<decltype(g_nccl.CommInitRank)>(sym("ncclCommInitRank"));
  g_nccl.AllReduce = reinterpret_cast<decltype(g_nccl.AllReduce)>(sym("ncclAllReduce"));
  g_nccl.CommDestroy = reinterpret_cast<decltype(g_nccl.CommDestroy)>(sym("ncclCommDestroy"));
  g_nccl.GetErrorString = reinterpret_cast<decltype(g_nccl.GetErrorString)>(sym("ncclGetErrorString"));
  g_nccl.CommInitAll = reinterpret_cast<decltype(g_nccl.CommInitAll)>(sym("ncclCommInitAll"));
  g_nccl.GroupStart = reinterpret_cast<decltype(g_nccl.GroupStart)>(sym("ncclGroupStart"));
  g_nccl.GroupEnd = reinterpret_cast<decltype(g_nccl.GroupEnd)>(sym("ncclGroupEnd"));
  if (!g_nccl.GetUniqueId || !g_nccl.CommInitRank || !g_nccl.AllReduce || !g_nccl.CommDestroy ||
      !g_nccl.GetErrorString || !g_nccl.GroupStart || !g_nccl.GroupEnd)
    return set_err(B2MD_CUDA_ERROR, "NCCL: missing symbols");
  g_nccl.loaded = true;
  return B2MD_OK;
}

const char* kFamilyName[F_COUNT] = {"offsets",  "search", "force",   "ewald_tables", "ewald_sk",
                                    "ewald_force", "kick_kick_drift", "kick_drift", "kick", "allreduce",
                                    "heat_flux", "rdf", "cluster", "force_jsum", "nl_build"};

// AoS <-> SoA staging kernels (host layout Vec3 / Quat of include/tmd/geom.hpp)
static __global__ void k_aos_to_soa(const double* aos, int count, int width, double* d0, double* d1,
                             double* d2, double* d3) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= count) return;
  d0[i] = aos[size_t(i) * width];
  d1[i] = aos[size_t(i) * width + 1];
  d2[i] = aos[size_t(i) * width + 2];
  if (width == 4) d3[i] = aos[size_t(i) * width + 3];
}
static __global__ void k_soa_to_aos(double* aos, int count, int width, const double* d0, const double* d1,
                             const double* d2, const double* d3) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= count) return;
  aos[size_t(i) * width] = d0[i];
  aos[size_t(i) * width + 1] = d1[i];
  aos[size_t(i) * width + 2] = d2[i];
  if (width == 4) aos[size_t(i) * width + 3] = d3[i];
}

// Up to six AoS host arrays (pinned, device-accessible) <-> SoA device arrays
// in one launch: the transfer is the kernel's own PCIe / C2C traffic (no
// staging copy, one launch per direction).  grid.y = array.
struct AosBatch {
  const double* src[6];  // upload: host AoS
  double* dst[6];        // download: host AoS
  double* d[6][4];       // SoA components
  const int* err_src;    // download: device error flag copied to err_dst
  int* err_dst;          //   (pinned host) in the same launch, or nullptr
  int width[6];
  int n_arrays;
  int count;
};
static __global__ void k_aos_batch_upload(AosBatch b) {
  const int k = blockIdx.y, i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= b.count) return;
  const int w = b.width[k];
  const double* a = b.src[k] + size_t(i) * w;
  for (int c = 0; c < w; ++c) b.d[k][c][i] = a[c];
}
static __global__ void k_aos_batch_download(AosBatch b) {
  const int k = blockIdx.y, i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= b.count) return;
  const int w = b.width[k];
  double* a = b.dst[k] + size_t(i) * w;
  for (int c = 0; c < w; ++c) a[c] = b.d[k][c][i];
}

// Zero-copy variants for 16-byte-aligned pinned host arrays: the host array
// is read / written as a flat run of double2 (fully coalesced 16-byte PCIe
// transactions, ~47 GB/s measured, as fast as one DMA copy), each element's
// two doubles scattered to / gathered from their SoA components.  Flat
// element e of an array of width w is component e % w of molecule e / w.
static __global__ void k_aos_zero_copy_upload(AosBatch b) {
  const int k = blockIdx.y;
  const int w = b.width[k];
  const size_t ne = size_t(b.count) * w;
  const double2* __restrict__ src = reinterpret_cast<const double2*>(b.src[k]);
  for (size_t t = blockIdx.x * size_t(blockDim.x) + threadIdx.x; 2 * t < ne;
       t += size_t(gridDim.x) * blockDim.x) {
    const size_t e = 2 * t;
    if (e + 1 < ne) {
      const double2 v = src[t];
      b.d[k][e % w][e / w] = v.x;
      b.d[k][(e + 1) % w][(e + 1) / w] = v.y;
    } else {
      b.d[k][e % w][e / w] = b.src[k][e];
    }
  }
}
static __global__ void k_aos_zero_copy_download(AosBatch b) {
  const int k = blockIdx.y;
  const int w = b.width[k];
  const size_t ne = size_t(b.count) * w;
  double2* __restrict__ dst = reinterpret_cast<double2*>(b.dst[k]);
  if (b.err_dst && blockIdx.x == 0 && k == 0 && threadIdx.x == 0) *b.err_dst = *b.err_src;
  for (size_t t = blockIdx.x * size_t(blockDim.x) + threadIdx.x; 2 * t < ne;
       t += size_t(gridDim.x) * blockDim.x) {
    const size_t e = 2 * t;
    if (e + 1 < ne)
      dst[t] = make_double2(b.d[k][e % w][e / w], b.d[k][(e + 1) % w][(e + 1) / w]);
    else
      b.dst[k][e] = b.d[k][e % w][e / w];
  }
}

int n_total(const b2md_ctx* c) { return c->t.n * c->R; }

void drop_graphs(b2md_ctx* c) {
  if (c->step_graph) cudaGraphExecDestroy(c->step_graph);
  if (c->single_graph) cudaGraphExecDestroy(c->single_graph);
  if (c->prof_graph) cudaGraphExecDestroy(c->prof_graph);
  if (c->prof_template) cudaGraphDestroy(c->prof_template);
  c->prof_template = nullptr;
  for (cudaEvent_t e : c->cap_ev) cudaEventDestroy(e);
  c->cap_ev.clear();
  c->cap_fam.clear();
  c->cap_nodes.clear();
  c->step_graph = nullptr;
  c->single_graph = nullptr;
  c->prof_graph = nullptr;
}

void set_wrapped(b2md_ctx* c, bool w) {
  if (c->positions_wrapped != w) drop_graphs(c);
  c->positions_wrapped = w;
}

bool prof_on(const b2md_ctx* c, int fam) {
  return c->profile && (c->profile_level == 1 || (c->profile_level == 2 && (fam == F_SEARCH || fam == F_CLUSTER)) ||
                        (c->profile_level == 3 && fam == F_FORCE));
}

int prof_begin(b2md_ctx* c, int fam) {
  if (!prof_on(c, fam)) return B2MD_OK;
  c->prof_open = true;
  if (c->capturing_prof) {  // placeholder events; re-pointed before every launch
    cudaEvent_t e;
    CU(cudaEventCreate(&e));
    c->cap_ev.push_back(e);
    c->cap_fam.push_back(fam);
    // External: captured as an event-record node (plain records in a capture
    // only express dependencies)
    CU(cudaEventRecordWithFlags(e, c->stream, cudaEventRecordExternal));
    return B2MD_OK;
  }
  if (c->ev_used == c->ev_pool.size()) {
    cudaEvent_t a, b;
    CU(cudaEventCreate(&a));
    CU(cudaEventCreate(&b));
    c->ev_pool.push_back({a, b});
    c->ev_family.push_back(fam);
  }
  c->ev_family[c->ev_used] = fam;
  CU(cudaEventRecord(c->ev_pool[c->ev_used].first, c->stream));
  return B2MD_OK;
}

int prof_end(b2md_ctx* c) {
  if (!c->prof_open) return B2MD_OK;
  c->prof_open = false;
  if (c->capturing_prof) {
    cudaEvent_t e;
    CU(cudaEventCreate(&e));
    c->cap_ev.push_back(e);
    CU(cudaEventRecordWithFlags(e, c->stream, cudaEventRecordExternal));
    return B2MD_OK;
  }
  CU(cudaEventRecord(c->ev_pool[c->ev_used].second, c->stream));
  ++c->ev_used;
  return B2MD_OK;
}

int prof_harvest(b2md_ctx* c) {
  if (c->ev_used == 0) return B2MD_OK;
  CU(cudaStreamSynchronize(c->stream));
  for (size_t k = 0; k < c->ev_used; ++k) {
    float ms = 0.f;
    CU(cudaEventElapsedTime(&ms, c->ev_pool[k].first, c->ev_pool[k].second));
    c->prof_ms[c->ev_family[k]] += ms;
    c->prof_n[c->ev_family[k]] += 1;
  }
  c->ev_used = 0;
  return B2MD_OK;
}

int launch_offsets(b2md_ctx* c) {
  if (!c->t.any_offsets) return B2MD_OK;
  const int nt = n_total(c);
  PROF(c, F_OFFSETS, (k_offsets<<<(nt + 255) / 256, 256, 0, c->stream>>>(c->sys, c->st)));
  return B2MD_OK;
}

int launch_search(b2md_ctx* c) {
  if (c->n_super_tiles == 0) return B2MD_OK;
  SearchArgs a;
  a.s = c->sys;
  a.pos4 = c->st.pos4;
  a.mask = c->d_mask;
  a.super_tiles = c->d_super;
  a.fixpos = c->d_fixpos;
  a.rc2 = c->t.single_site_path ? c->t.rc2 : c->t.rmax2[0];
  const bool multi = c->t.ns > 1;
  {
    // certified fixed-point prefilter (kernels.cuh, search_tile_fix)
    const double L = c->t.box, two32 = 4294967296.0;
    const double rmax = std::sqrt(a.rc2);
    const double r2fix = a.rc2 * 1073741824.0 / (L * L);  // rmax^2 in (L/32768)^2 units
    const double dmax = std::ceil(rmax * 32768.0 / L) + 2.0;
    const double K = 3.0 * (2.0 * dmax + 1.0) + 64.0;   // |r2_fix - r2 (65536/L)^2| bound
    const double lo = std::floor(r2fix) - K;
    a.fix_ok = (!multi && c->use_fix_prefilter && rmax < 0.5 * L * (1.0 - 1e-3) && lo > 0.0 &&
                r2fix + K < 1.0e9) ? 1 : 0;
    a.fix_scale = two32 / L;
    a.fix_lo = lo > 0.0 ? uint32_t(lo) : 0u;
    a.fix_width = uint32_t(2.0 * K + 2.0);
    const double r2_32 = a.rc2 * two32 / (L * L);
    const double lo32 = std::floor(r2_32) - 8.0;
    a.fix_lo32 = lo32 > 0.0 ? uint32_t(lo32) : 0u;
    a.fix_w32 = 17u;
    if (!(r2_32 + 64.0 < two32) || lo32 <= 0.0) a.fix_ok = 0;
    a.cull = a.fix_ok && c->use_tile_cull ? 1 : 0;
    const double ru = rmax * two32 / L;
    a.cull_r2 = ru * ru * (1.0 + 1e-6);
  }
  dim3 grid(c->n_super_tiles, c->R);
  const int st = c->g.st;
  // generic path (mixtures, rmax >= L/2 (1 - 1e-3)) of small systems (few
  // tiles): RS = 4 warps per tile row
#define SEARCH_CASE(ST)                                                                  \
  case ST: {                                                                             \
    constexpr int RS = ST <= 2 ? 4 : 1;                                                  \
    if (multi)                                                                           \
      PROF(c, F_SEARCH, (k_search<ST, true, RS><<<grid, ST * 32 * RS, 0, c->stream>>>(a))); \
    else if (!a.fix_ok)                                                                  \
      PROF(c, F_SEARCH, (k_search<ST, false, RS><<<grid, ST * 32 * RS, 0, c->stream>>>(a))); \
    else                                                                                 \
      PROF(c, F_SEARCH, (k_search<ST, false><<<grid, ST * 32, 0, c->stream>>>(a)));      \
    break;                                                                               \
  }
  switch (st) {
    SEARCH_CASE(1)
    SEARCH_CASE(2)
    SEARCH_CASE(4)
    SEARCH_CASE(8)
    default:
      return set_err(B2MD_INVALID_ARGUMENT, "bad super-tile size");
  }
#undef SEARCH_CASE
  c->mask_valid = true;
  return B2MD_OK;
}

// The bit matrix of the current positions for its consumers (pair export,
// heat flux): the cluster walk does not build it.
int ensure_mask(b2md_ctx* c) {
  if (c->mask_valid) return B2MD_OK;
  return launch_search(c);
}

double* sums_ptr(b2md_ctx* c) { return c->d_fbuf + size_t(6) * n_total(c); }

ForceArgs force_args(b2md_ctx* c) {
  ForceArgs a;
  a.s = c->sys;
  a.st = c->st;
  a.mask = c->d_mask;
  a.cta_part = c->d_cta_part;
  a.ticket = c->d_ticket;
  a.sums = sums_ptr(c);
  a.c12 = 0.0;
  a.c6 = 0.0;
  a.c12x12 = 0.0;
  a.c6x6 = 0.0;
  if (!c->t.lj.empty() && !c->t.lj[0].empty()) {
    a.c12 = c->t.lj[0][0].c12;
    a.c6 = c->t.lj[0][0].c6;
    a.c12x12 = 12.0 * a.c12;
    a.c6x6 = 6.0 * a.c6;
  }
  a.rc2 = c->t.rc2;
  a.alpha = c->t.alpha;
  a.two_alpha_over_sqrt_pi = 2.0 * c->t.alpha / std::sqrt(3.14159265358979323846);
  a.rf_r3inv = c->t.rf_r3inv;
  a.rf_shift = c->t.rf_shift;
  // erfcx Chebyshev interpolation (kernels.cuh, erfcx_cheb): nodes in
  // u, t = t_lo + (u + 1)(1 - t_lo)/2, x = 2 (1/t - 1)
  {
    const int N = kErfcxDeg + 1;
    const double t_lo = 1.0 / (1.0 + 0.5 * kErfcxMax);
    double f[kErfcxDeg + 1];
    for (int k = 0; k < N; ++k) {
      const double u = std::cos(3.14159265358979323846 * (k + 0.5) / N);
      const double t = t_lo + 0.5 * (u + 1.0) * (1.0 - t_lo);
      const double x = 2.0 * (1.0 / t - 1.0);
      f[k] = std::erfc(x) * std::exp(x * x);
    }
    long double cheb[kErfcxDeg + 1];
    for (int j = 0; j < N; ++j) {
      long double sum = 0.0L;
      for (int k = 0; k < N; ++k)
        sum += static_cast<long double>(f[k]) * std::cos(3.14159265358979323846L * j * (k + 0.5L) / N);
      cheb[j] = (j == 0 ? 1.0L : 2.0L) * sum / N;
    }
    // Chebyshev -> monomial coefficients in u (T_{j+1} = 2 u T_j - T_{j-1},
    // extended precision): the series' coefficients fall off fast enough that
    // Horner's rule on the monomials is as accurate as Clenshaw's sum (both
    // 1.1e-14 of erfcx on [0, kErfcxMax)) at half the fp64 operations
    long double mono[kErfcxDeg + 1] = {}, tp[kErfcxDeg + 1] = {}, tc[kErfcxDeg + 1] = {};
    tp[0] = 1.0L;  // T_0
    tc[1] = 1.0L;  // T_1
    for (int k = 0; k < N; ++k) mono[k] = cheb[0] * tp[k] + cheb[1] * tc[k];
    for (int j = 1; j + 1 < N; ++j) {
      long double tn[kErfcxDeg + 1] = {};
      for (int k = 0; k < N; ++k) tn[k] = (k > 0 ? 2.0L * tc[k - 1] : 0.0L) - tp[k];
      for (int k = 0; k < N; ++k) {
        mono[k] += cheb[j + 1] * tn[k];
        tp[k] = tc[k];
        tc[k] = tn[k];
      }
    }
    for (int k = 0; k < N; ++k) a.erfcx_c[k] = static_cast<double>(mono[k]);
    a.erfcx_tlo = t_lo;
    a.erfcx_uscale = 2.0 / (1.0 - t_lo);
  }
  a.vderiv = c->t.vderiv ? 1 : 0;
  const int hh = hi32(0.5 * c->t.box);
  std::memcpy(&a.thr, &hh, 4);
  a.kick_dt = 0.0;
  a.rmax2 = c->t.rmax2.empty() ? c->t.rc2 : c->t.rmax2[0];
  a.error_mol = c->d_error;
  return a;
}

// The end-of-step half kick can run in the force kernel's row epilogue when
// a molecule's force is final there: no Ewald reciprocal term still to add
// and no cross-rank all-reduce.
bool kick_fusable(const b2md_ctx* c) {
  return c->engine && c->use_fused_kick && !(c->t.ewald && c->nq > 0) &&
         !(c->world > 1 && c->comm);
}

// k_force_rigid applies: a single species whose site pairs are all LJ terms
// in the PairTable's (ia, ib) order, no charges, 2 or 3 sites; returns the
// site count (0: not applicable)
int rigid_sites(const ModelTables& t) {
  if (t.single_site_path || t.ns != 1 || !t.qq[0].empty()) return 0;
  const int ns = t.species[0].n_sites;
  bool full = int(t.lj[0].size()) == ns * ns;
  for (int k = 0; full && k < ns * ns; ++k) full = t.lj[0][k].a == k / ns && t.lj[0][k].b == k % ns;
  return full && (ns == 2 || ns == 3) ? ns : 0;
}

// the once-per-pair block-pair tiles apply (k_force_rigid_tile): the rigid
// species k_force_rigid handles, records allocated
bool tile_path(const b2md_ctx* c) { return c->use_tile && c->d_trec && rigid_sites(c->t) > 0; }

// positions known to lie in [0, L) (set_state / step wrap them) and every
// listed pair's components far from L/2: the branch-free minimum image is exact
bool fast_min_image(const b2md_ctx* c) {
  if (!c->positions_wrapped) return false;
  const double h = 0.5 * c->t.box * (1.0 - 1.0 / 65536.0);
  for (double r2 : c->t.rmax2)
    if (!(r2 < h * h)) return false;
  return !(c->t.single_site_path && !(c->t.rc2 < h * h));
}

// The cluster walk (cluster.cuh) replaces search + bit-matrix walk for the
// single-site path; with b2md_set_shard / NCCL each rank walks its own
// contiguous range of i-groups (cluster_args).  Any positions:
// clusters with a member outside [0, L) are never culled, and the exact
// minimum image replaces the wrapped one when positions are not wrapped
// (same bits), so the hit sequence -- and the summation order -- is the same
// either way: restarts from unwrapped checkpoints stay bit-exact.
// CTAs of the cluster-pair walk: kGWarps i-groups of kGR slots each
int cpair_grid(const b2md_ctx* c) {
  const int groups = (c->t.n + kGR - 1) / kGR;
  return (groups + kGWarps - 1) / kGWarps;
}

bool cluster_path(const b2md_ctx* c) {
  return c->use_cluster && c->nc > 0 && c->t.single_site_path;
}

ClusterArgs cluster_args(const b2md_ctx* c) {
  ClusterArgs ca;
  ca.n = c->t.n;
  ca.nc = c->nc;
  ca.nsup = c->nsup;
  ca.fixpos = c->d_fixpos;
  ca.arcs = c->d_carc;
  ca.half = c->d_chalf;
  ca.sup_arcs = c->d_sarc;
  ca.sup_half = c->d_shalf;
  const double ru = std::sqrt(c->t.rc2) * 4294967296.0 / c->t.box;
  ca.lim = float(ru * ru * (1.0 + 1e-5));
  // row shard: contiguous i-group ranges (each a slab of the spatial order,
  // so the ranks' pair work is balanced); every row's force is complete on
  // its rank (both rows of a pair evaluate it), other rows are written 0
  const long groups = (c->t.n + kGR - 1) / kGR;
  ca.grp_begin = int(groups * c->rank / std::max(1, c->world));
  ca.grp_end = int(groups * (c->rank + 1) / std::max(1, c->world));
  ca.fixref = c->nl.fixref;
  ca.nl_ctl = c->nl.ctl;
  return ca;
}

bool nl_path(const b2md_ctx* c) { return cluster_path(c) && c->use_newton && c->nl.ctl; }

NListArgs nl_args(const b2md_ctx* c) {
  NListArgs nl = c->nl;
  nl.cbeg = int(long(c->nc) * c->rank / std::max(1, c->world));
  nl.cend = int(long(c->nc) * (c->rank + 1) / std::max(1, c->world));
  return nl;
}

// The once-per-pair list from the current cluster arcs (cluster.cuh): after
// every staging of positions (re-sort, evaluate, set_state, restore) and at
// the scheduled interval, always between a drift and a force evaluation.
int nl_build(b2md_ctx* c) {
  if (!nl_path(c)) return B2MD_OK;
  const ClusterArgs ca = cluster_args(c);
  const NListArgs nl = nl_args(c);
  const dim3 g((c->nc + kNLBuildWarps - 1) / kNLBuildWarps, c->R);
  const dim3 gp((c->nc * kNLParts + kNLBuildWarps - 1) / kNLBuildWarps, c->R);
  const int bs = kNLBuildWarps * 32;
  PROF(c, F_NL_BUILD, (k_nl_count<<<gp, bs, 0, c->stream>>>(ca, nl)));
  PROF(c, F_NL_BUILD, (k_nl_scan<<<c->R, kNLScanThreads, 0, c->stream>>>(nl, c->nc)));
  PROF(c, F_NL_BUILD, (k_nl_fill<<<gp, bs, 0, c->stream>>>(ca, nl)));
  if (nl.smap)
    PROF(c, F_NL_BUILD, (k_nl_zfill<<<g, bs, 0, c->stream>>>(nl, c->nc)));
  else
    PROF(c, F_NL_BUILD, (k_nl_inrec<<<g, bs, 0, c->stream>>>(nl, c->nc)));
  if (c->nl_member_gaps)
    PROF(c, F_NL_BUILD, (k_nl_gaps<<<dim3(c->n3_grid * 2, c->R), bs, 0, c->stream>>>(ca, nl)));
  c->steps_since_nl = 0;
  return B2MD_OK;
}

bool nl_due(const b2md_ctx* c) {
  return nl_path(c) && c->nl_interval > 0 && c->steps_since_nl >= c->nl_interval;
}

// Cluster arcs are derived wherever fixed-point positions are written: by
// the step's drift kernel (k_step_drift_arcs) and, here, after staging (a
// re-sort, evaluate / set_state / restore).
int launch_cluster_arcs(b2md_ctx* c) {
  if (!cluster_path(c)) return B2MD_OK;
  const ClusterArgs ca = cluster_args(c);
  PROF(c, F_CLUSTER, (k_cluster_arcs<<<c->R * c->nsup, kSC * kCS, 0, c->stream>>>(ca, c->R)));
  return nl_build(c);
}

int launch_cluster_force(b2md_ctx* c, bool kick) {
  const ClusterArgs ca = cluster_args(c);
  const int R = c->R;
  ForceArgs a = force_args(c);
  if (kick) a.kick_dt = c->dt;
  const bool w = fast_min_image(c), m = c->t.ns > 1, v = a.vderiv != 0;
  if (nl_path(c)) {
    const NListArgs nl = nl_args(c);
    ForceArgs aw = a;
    aw.kick_dt = 0.0;  // the rows are complete only after k_nl_reduce
    const dim3 ngrid(c->n3_grid, R);
#define NL_LAUNCH(M, W, V) \
  if (m == M && w == W && v == V) \
    PROF(c, F_FORCE, (k_force_nl<M, W, V><<<ngrid, kNLWarps * 32, 0, c->stream>>>(aw, ca, nl)));
    NL_LAUNCH(false, true, false)
    NL_LAUNCH(false, true, true)
    NL_LAUNCH(false, false, false)
    NL_LAUNCH(false, false, true)
    NL_LAUNCH(true, true, false)
    NL_LAUNCH(true, true, true)
    NL_LAUNCH(true, false, false)
    NL_LAUNCH(true, false, true)
#undef NL_LAUNCH
    PROF(c, F_JSUM, (k_nl_reduce<<<dim3((c->nc + kNLBuildWarps - 1) / kNLBuildWarps, R),
                                   kNLBuildWarps * 32, 0, c->stream>>>(a, ca, nl)));
    c->mask_valid = false;
    return B2MD_OK;
  }
  dim3 pgrid(cpair_grid(c), R);
#define CPAIR_LAUNCH(M, W, V) \
  if (m == M && w == W && v == V) \
    PROF(c, F_FORCE, (k_force_cpair<M, W, V><<<pgrid, kGWarps * 32, 0, c->stream>>>(a, ca)));
  CPAIR_LAUNCH(false, true, false)
  CPAIR_LAUNCH(false, true, true)
  CPAIR_LAUNCH(false, false, false)
  CPAIR_LAUNCH(false, false, true)
  CPAIR_LAUNCH(true, true, false)
  CPAIR_LAUNCH(true, true, true)
  CPAIR_LAUNCH(true, false, false)
  CPAIR_LAUNCH(true, false, true)
#undef CPAIR_LAUNCH
  c->mask_valid = false;
  return B2MD_OK;
}

int launch_tile_force(b2md_ctx* c, bool kick) {
  ForceArgs a = force_args(c);
  if (kick) a.kick_dt = c->dt;
  TileArgs ta;
  ta.rec = c->d_trec;
  ta.nb = c->tile_nb;
  ta.nbp = c->tile_nbp;
  ta.bp_begin = int(long(c->tile_nbp) * c->rank / std::max(1, c->world));
  ta.bp_end = int(long(c->tile_nbp) * (c->rank + 1) / std::max(1, c->world));
  ForceArgs aw = a;
  aw.kick_dt = 0.0;  // the molecules are complete only after k_rigid_reduce
  const bool w = fast_min_image(c);
  const dim3 grid((c->tile_nbp * kTileSplit + kTileWarps - 1) / kTileWarps, c->R);
  const int ns = rigid_sites(c->t);
  if (ns == 2 && w)
    PROF(c, F_FORCE, (k_force_rigid_tile<2, true><<<grid, kTileWarps * 32, 0, c->stream>>>(aw, ta)));
  else if (ns == 2)
    PROF(c, F_FORCE, (k_force_rigid_tile<2, false><<<grid, kTileWarps * 32, 0, c->stream>>>(aw, ta)));
  else if (w)
    PROF(c, F_FORCE, (k_force_rigid_tile<3, true><<<grid, kTileWarps * 32, 0, c->stream>>>(aw, ta)));
  else
    PROF(c, F_FORCE, (k_force_rigid_tile<3, false><<<grid, kTileWarps * 32, 0, c->stream>>>(aw, ta)));
  PROF(c, F_JSUM, (k_rigid_reduce<<<dim3(c->tile_nb, c->R), 192, 0, c->stream>>>(a, ta)));
  c->mask_valid = false;  // no partner search ran: the bit matrix is built on demand
  return B2MD_OK;
}

int launch_force(b2md_ctx* c, bool kick) {
  if (cluster_path(c)) return launch_cluster_force(c, kick);
  if (tile_path(c)) return launch_tile_force(c, kick);
  ForceArgs a = force_args(c);
  if (kick) a.kick_dt = c->dt;
  a.split = c->force_split;
  const bool w = fast_min_image(c);
  const bool sp = c->force_split > 1;
  dim3 grid(c->force_grid, c->R);
  const int bs = c->force_warps * 32;
#define FORCE_LAUNCH(K, ...)                                                              \
  do {                                                                                    \
    if (w && sp)                                                                          \
      PROF(c, F_FORCE, (K<__VA_ARGS__, true, true><<<grid, bs, 0, c->stream>>>(a)));      \
    else if (w)                                                                           \
      PROF(c, F_FORCE, (K<__VA_ARGS__, true, false><<<grid, bs, 0, c->stream>>>(a)));     \
    else if (sp)                                                                          \
      PROF(c, F_FORCE, (K<__VA_ARGS__, false, true><<<grid, bs, 0, c->stream>>>(a)));     \
    else                                                                                  \
      PROF(c, F_FORCE, (K<__VA_ARGS__, false, false><<<grid, bs, 0, c->stream>>>(a)));    \
  } while (0)
  // single species, every site pair an LJ term in (ia, ib) order, no charges
  const int rigid_ns = rigid_sites(c->t);
  if (c->t.single_site_path) {
    if (c->t.ns > 1)
      FORCE_LAUNCH(k_force_single, true);
    else
      FORCE_LAUNCH(k_force_single, false);
  } else if (rigid_ns == 2) {
    FORCE_LAUNCH(k_force_rigid, 2);
  } else if (rigid_ns == 3) {
    FORCE_LAUNCH(k_force_rigid, 3);
  } else if (c->t.method == B2MD_METHOD_EWALD) {
    FORCE_LAUNCH(k_force_multi, 2);
  } else if (c->t.method == B2MD_METHOD_REACTION_FIELD) {
    FORCE_LAUNCH(k_force_multi, 1);
  } else {
    FORCE_LAUNCH(k_force_multi, 0);
  }
#undef FORCE_LAUNCH
  return B2MD_OK;
}

EwaldArgs ewald_args(b2md_ctx* c) {
  EwaldArgs a;
  a.s = c->sys;
  a.st = c->st;
  a.nq = c->nq;
  a.kmax = c->t.kmax;
  a.nk = c->k_end - c->k_begin;
  a.k_begin = c->k_begin;
  a.q_mol = c->d_q_mol;
  a.q_site = c->d_q_site;
  a.q_val = c->d_q_val;
  a.mol_qbegin = c->d_mol_qbegin;
  a.kv = c->d_kv;
  a.tab = c->d_etab;
  a.S = c->d_S;
  a.uk = c->d_uk;
  a.ticket = c->d_ticket + c->R;
  a.sums = sums_ptr(c);
  a.nk_total = int(c->t.kv.size());
  a.two_pi_over_L = 2.0 * 3.14159265358979323846 / c->t.box;
  a.frec = nullptr;
  return a;
}

EwaldTiled ewald_tiled(b2md_ctx* c) {
  EwaldTiled et;
  et.Sp = c->d_ewSp;
  et.fq = c->d_ewfq;
  et.nchunks = (c->nq + kEwSkQ - 1) / kEwSkQ;
  return et;
}

// Ewald::evaluate (src/ewald.cpp:107-180): per-site phase tables, S(k) and
// U_recip (first part, stream st), then the forces/torques added onto the
// real-space ones (second part, after the real-space kernel on c->stream)
int launch_ewald_sk(b2md_ctx* c, cudaStream_t st) {
  EwaldArgs a = ewald_args(c);
  const int nt = c->nq * c->R;
  const bool prof = st == c->stream;  // profiling events live on c->stream
  if (prof)
    PROF(c, F_EWALD_TAB, (k_ewald_tables<<<(nt + 127) / 128, 128, 0, st>>>(a)));
  else
    k_ewald_tables<<<(nt + 127) / 128, 128, 0, st>>>(a);
  CU(cudaGetLastError());
  if (a.nk > 0 && c->ew_tiled) {
    const EwaldTiled et = ewald_tiled(c);
    const dim3 g(et.nchunks, c->R);
    const dim3 g2((a.nk + kEwSumK - 1) / kEwSumK, c->R);
    if (prof) {
      PROF(c, F_EWALD_SK, (k_ewald_sk_tiled<<<g, 256, 0, st>>>(a, et)));
      PROF(c, F_EWALD_SK, (k_ewald_sk_sum<<<g2, kEwSumK * 8, 0, st>>>(a, et)));
    } else {
      k_ewald_sk_tiled<<<g, 256, 0, st>>>(a, et);
      k_ewald_sk_sum<<<g2, kEwSumK * 8, 0, st>>>(a, et);
    }
    CU(cudaGetLastError());
  } else if (a.nk > 0) {
    if (prof)
      PROF(c, F_EWALD_SK, (k_ewald_sk<<<dim3(a.nk, c->R), 256, 0, st>>>(a)));
    else
      k_ewald_sk<<<dim3(a.nk, c->R), 256, 0, st>>>(a);
    CU(cudaGetLastError());
  } else {
    for (int r = 0; r < c->R; ++r)
      CU(cudaMemsetAsync(sums_ptr(c) + size_t(r) * kNumSums + kNumRowScalars, 0, sizeof(double),
                         st));
  }
  return B2MD_OK;
}

// side == false: after the real-space kernel on c->stream, added to its
// totals; side == true: on the Ewald branch stream beside it, written to
// d_frec (ewald_overlap: the end-of-step kick adds the two)
int launch_ewald_force(b2md_ctx* c, bool side) {
  EwaldArgs a = ewald_args(c);
  if (a.nk == 0) return B2MD_OK;
  if (c->ew_tiled) {
    const EwaldTiled et = ewald_tiled(c);
    PROF(c, F_EWALD_F, (k_ewald_force_tiled<<<dim3((c->nq + kEwFQ - 1) / kEwFQ, c->R),
                                              kEwFQ * kEwFParts, 0, c->stream>>>(a, et)));
    PROF(c, F_EWALD_F,
         (k_ewald_apply<<<dim3((c->t.n + 255) / 256, c->R), 256, 0, c->stream>>>(a, et)));
    return B2MD_OK;
  }
  // k-split: P warps per molecule so that molecules x P reach ~16 warps per SM
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device);
  int P = 1;
  while (P < 8 && long(c->t.n) * c->R * P < long(sms) * 16) P *= 2;
  if (const char* e = std::getenv("B2MD_EWALD_KPARTS")) P = std::max(1, std::min(8, std::atoi(e)));
  while (8 % P) --P;
  a.kparts = P;
  const int mpc = 8 / P;
  if (side) {
    a.frec = c->d_frec;
    k_ewald_force<<<dim3((c->t.n + mpc - 1) / mpc, c->R), 256, 0, c->stream2>>>(a);
    CU(cudaGetLastError());
    return B2MD_OK;
  }
  PROF(c, F_EWALD_F,
       (k_ewald_force<<<dim3((c->t.n + mpc - 1) / mpc, c->R), 256, 0, c->stream>>>(a)));
  return B2MD_OK;
}

int launch_ewald(b2md_ctx* c) {
  if (!c->t.ewald || c->nq == 0) return B2MD_OK;
  TRY(launch_ewald_sk(c, c->stream));
  return launch_ewald_force(c, false);
}

// The reciprocal forces can be computed beside the real-space kernel (they
// read S(k) and the phase tables only) when an end-of-step kick follows that
// adds them: step paths, one rank (the all-reduce unit is the force array),
// the gather form of the kernel, not while kernels are being timed.
bool ewald_overlap(const b2md_ctx* c) {
  return c->engine && c->t.ewald && c->nq > 0 && c->k_end > c->k_begin && !c->profile && c->stream2 &&
         c->d_frec && c->ew_overlap && !c->ew_tiled && !(c->world > 1 && c->comm);
}

int launch_allreduce(b2md_ctx* c) {
  if (c->world <= 1 || !c->comm) return B2MD_OK;
  TRY(prof_begin(c, F_ALLREDUCE));
  const size_t nt = size_t(n_total(c));
  if (c->t.any_offsets) {  // forces, torques and sums: one contiguous unit
    NC(g_nccl.AllReduce(c->d_fbuf, c->d_fbuf, 6 * nt + size_t(kNumSums) * c->R, ncclDouble, ncclSum,
                        c->comm, c->stream));
  } else {  // centred sites only: no torques (zero on every rank), forces + sums
    NC(g_nccl.GroupStart());
    NC(g_nccl.AllReduce(c->d_fbuf, c->d_fbuf, 3 * nt, ncclDouble, ncclSum, c->comm, c->stream));
    NC(g_nccl.AllReduce(c->d_fbuf + 6 * nt, c->d_fbuf + 6 * nt, size_t(kNumSums) * c->R, ncclDouble,
                        ncclSum, c->comm, c->stream));
    NC(g_nccl.GroupEnd());
  }
  TRY(prof_end(c));
  return B2MD_OK;
}

// Spatial order: molecules are assigned slots in column order of their
// (wrapped) positions (k_sort_keys), so 32-slot blocks stay thin lines and
// the search's tile cull stays effective as molecules diffuse.  Rebuilds perm / slot_of / sp_slot / sb_slot; the
// caller re-stages pos4, fixpos and the offsets before the next search.
// Results do not depend on the order beyond summation order (pair lists are
// exported in the reference's (i, j) order).
int resort(b2md_ctx* c) {
  NvtxRange nvtx_("b2md_resort");
  const int nt = n_total(c), n = c->t.n;
  const int g = (nt + 255) / 256;
  // columns of cross-section c^2 = 32 / (rho L) (about one 32-slot block
  // each: thin search tiles); for the cluster walk c = (kCS / rho)^(1/3), so
  // kCS consecutive slots make a compact cluster
  const double L = c->t.box, rho = double(n) / (L * L * L);
  const double side = c->use_cluster && c->nc > 0 ? std::cbrt(double(kCS) / rho)
                                                  : std::sqrt(32.0 / (rho * L));
  const int G = std::max(1, std::min(1024, int(L / side)));
  int cbits = 1;  // bits of the column index (< G^2)
  while ((1 << cbits) < G * G) ++cbits;
  k_sort_keys<<<g, 256, 0, c->stream>>>(c->st.px, c->st.py, c->st.pz, nt, n, L, G, cbits,
                                        c->d_keys[0], c->d_vals[0]);
  CU(cudaGetLastError());
  // (cfg3: 8 + 14 bits, three 8-bit radix passes instead of the five of a fixed 40-bit key)
  int end_bit = cbits + kSortXBits;
  while ((1 << (end_bit - cbits - kSortXBits)) < c->R) ++end_bit;
  size_t bytes = c->cub_bytes;
  CU(cub::DeviceRadixSort::SortPairs(c->d_cub, bytes, c->d_keys[0], c->d_keys[1], c->d_vals[0],
                                     c->d_vals[1], nt, 0, end_bit, c->stream));
  k_apply_order<<<g, 256, 0, c->stream>>>(c->d_vals[1], nt, n, c->d_species_of, c->d_tab,
                                          c->d_perm, c->d_slot_of, c->d_sp_slot,
                                          c->d_nsites_slot);
  CU(cudaGetLastError());
  bytes = c->cub_bytes;
  CU(cub::DeviceScan::ExclusiveSum(c->d_cub, bytes, c->d_nsites_slot, c->d_scan, nt, c->stream));
  k_site_starts<<<g, 256, 0, c->stream>>>(c->d_scan, nt, n, c->t.total_sites, c->d_sb_slot);
  CU(cudaGetLastError());
  c->steps_since_sort = 0;
  c->mask_valid = false;  // slot-indexed
  return B2MD_OK;
}

// resort + re-stage of what the integrator wrote in the old order
int resort_and_stage(b2md_ctx* c) {
  TRY(resort(c));
  TRY(launch_offsets(c));
  const int nt = n_total(c);
  k_stage_positions<<<(nt + 255) / 256, 256, 0, c->stream>>>(
      c->st.px, c->st.py, c->st.pz, nt, c->t.n, c->d_slot_of, c->t.box, 4294967296.0 / c->t.box,
      c->d_fixpos, c->st.pos4);
  CU(cudaGetLastError());
  TRY(launch_cluster_arcs(c));
  return B2MD_OK;
}

bool sort_due(const b2md_ctx* c) {
  return c->sort_interval > 0 && c->steps_since_sort >= c->sort_interval;
}

// ForceField::evaluate (src/parallel.cpp:79-122) on the device state.
int enqueue_forces(b2md_ctx* c, bool offsets, bool kick, bool recip_beside) {
  if (offsets) {  // evaluate / set_state path: the integrator did not refresh these
    TRY(launch_offsets(c));
    const int nt = n_total(c);
    k_stage_positions<<<(nt + 255) / 256, 256, 0, c->stream>>>(
        c->st.px, c->st.py, c->st.pz, nt, c->t.n, c->d_slot_of, c->t.box,
        4294967296.0 / c->t.box, c->d_fixpos, c->st.pos4);
    CU(cudaGetLastError());
    TRY(launch_cluster_arcs(c));
  }
  // the Ewald tables and S(k) only read positions: a parallel branch beside
  // the search and the real-space kernel (which overwrites the forces the
  // Ewald force kernel then adds to); serial while kernels are being timed
  const bool ewald = c->t.ewald && c->nq > 0;
  const bool fork = ewald && !c->profile && c->stream2;
  if (fork) {
    CU(cudaEventRecord(c->ev_fork, c->stream));
    CU(cudaStreamWaitEvent(c->stream2, c->ev_fork, 0));
    TRY(launch_ewald_sk(c, c->stream2));
    if (recip_beside) TRY(launch_ewald_force(c, true));
    CU(cudaEventRecord(c->ev_join, c->stream2));
  }
  if (!cluster_path(c) && !tile_path(c)) TRY(launch_search(c));
  TRY(launch_force(c, kick));
  if (fork) {
    CU(cudaStreamWaitEvent(c->stream, c->ev_join, 0));
    if (!recip_beside) TRY(launch_ewald_force(c, false));
  } else {
    TRY(launch_ewald(c));
  }
  TRY(launch_allreduce(c));
  return B2MD_OK;
}

StepArgs step_args(b2md_ctx* c) {
  StepArgs a;
  a.s = c->sys;
  a.st = c->st;
  a.dt = c->dt;
  a.error_mol = c->d_error;
  a.write_offsets = c->t.any_offsets ? 1 : 0;
  a.fixpos = c->d_fixpos;
  a.fix_scale = 4294967296.0 / c->t.box;
  return a;
}

// Engine::step (src/engine.cpp:102-143).  A run of k steps is issued as
//   kick_drift, [forces, kick+kick_drift] x (k-1), forces, kick
// where the bracket is one CUDA graph (the second half-kick of step s and the
// first of step s+1 share one launch), or, when the kick fuses into the force
// kernel (kick_fusable),
//   kick_drift, [forces+kick, kick_drift] x (k-1), forces+kick.
int launch_step_kernel(b2md_ctx* c, int fam, bool add_recip = false) {
  StepArgs a = step_args(c);
  if (add_recip) a.frec = c->d_frec;  // (F_KICK, F_KICK_KICK_DRIFT: the end-of-step kick)
  const int nt = n_total(c);
  // small CTAs: 16k molecules must still spread over all 148 SMs
  const int bs = 64, g = (nt + bs - 1) / bs;
  if (fam != F_KICK && cluster_path(c)) {  // slot-ordered, with the cluster arcs
    const ClusterArgs ca = cluster_args(c);
    if (fam == F_KICK_DRIFT)
      PROF(c, fam, (k_step_drift_arcs<false><<<c->R * c->nsup, kSC * kCS, 0, c->stream>>>(a, ca)));
    else
      PROF(c, fam, (k_step_drift_arcs<true><<<c->R * c->nsup, kSC * kCS, 0, c->stream>>>(a, ca)));
    return B2MD_OK;
  }
  if (fam == F_KICK_DRIFT)
    PROF(c, fam, (k_kick_drift<<<g, bs, 0, c->stream>>>(a)));
  else if (fam == F_KICK)
    PROF(c, fam, (k_kick<<<g, bs, 0, c->stream>>>(a)));
  else
    PROF(c, fam, (k_kick_kick_drift<<<g, bs, 0, c->stream>>>(a)));
  return B2MD_OK;
}

int enqueue_loop_body(b2md_ctx* c) {
  const bool fused = kick_fusable(c);
  const bool beside = !fused && ewald_overlap(c);
  TRY(enqueue_forces(c, false, fused, beside));
  TRY(launch_step_kernel(c, fused ? F_KICK_DRIFT : F_KICK_KICK_DRIFT, beside));
  return B2MD_OK;
}

// forces + the end-of-step half kick
int enqueue_forces_and_kick(b2md_ctx* c) {
  const bool fused = kick_fusable(c);
  const bool beside = !fused && ewald_overlap(c);
  TRY(enqueue_forces(c, false, fused, beside));
  if (!fused) TRY(launch_step_kernel(c, F_KICK, beside));
  return B2MD_OK;
}

int build_step_graph(b2md_ctx* c) {
  if (c->step_graph) return B2MD_OK;
  const bool prof = c->profile;
  c->profile = false;
  CU(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
  int rc = enqueue_loop_body(c);
  cudaGraph_t graph;
  cudaError_t e = cudaStreamEndCapture(c->stream, &graph);
  c->profile = prof;
  if (rc) return rc;
  CU(e);
  e = cudaGraphInstantiate(&c->step_graph, graph, 0);
  cudaGraphDestroy(graph);
  CU(e);
  return B2MD_OK;
}

int build_single_step_graph(b2md_ctx* c) {
  if (c->single_graph) return B2MD_OK;
  CU(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
  int rc = launch_step_kernel(c, F_KICK_DRIFT);
  if (!rc) rc = enqueue_forces_and_kick(c);
  cudaGraph_t graph;
  cudaError_t e = cudaStreamEndCapture(c->stream, &graph);
  if (rc) return rc;
  CU(e);
  e = cudaGraphInstantiate(&c->single_graph, graph, 0);
  cudaGraphDestroy(graph);
  CU(e);
  return B2MD_OK;
}

// One step as a graph with CUDA-event record nodes around every kernel
// family: per-kernel timing at graph-launch speed.  Before each launch the
// nodes are re-pointed at fresh events of the profiling pool.
int build_prof_graph(b2md_ctx* c) {
  if (c->prof_graph) return B2MD_OK;
  CU(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
  c->capturing_prof = true;
  int rc = launch_step_kernel(c, F_KICK_DRIFT);
  if (!rc) rc = enqueue_forces_and_kick(c);
  c->capturing_prof = false;
  cudaGraph_t graph;
  cudaError_t e = cudaStreamEndCapture(c->stream, &graph);
  if (rc) return rc;
  CU(e);
  size_t nn = 0;
  CU(cudaGraphGetNodes(graph, nullptr, &nn));
  std::vector<cudaGraphNode_t> nodes(nn);
  CU(cudaGraphGetNodes(graph, nodes.data(), &nn));
  c->cap_nodes.assign(c->cap_ev.size(), nullptr);
  for (cudaGraphNode_t node : nodes) {
    cudaGraphNodeType ty;
    CU(cudaGraphNodeGetType(node, &ty));
    if (ty != cudaGraphNodeTypeEventRecord) continue;
    cudaEvent_t ev;
    CU(cudaGraphEventRecordNodeGetEvent(node, &ev));
    for (size_t k = 0; k < c->cap_ev.size(); ++k)
      if (c->cap_ev[k] == ev) c->cap_nodes[k] = node;
  }
  for (cudaGraphNode_t node : c->cap_nodes)
    if (!node) {
      cudaGraphDestroy(graph);
      return set_err(B2MD_CUDA_ERROR, "profiling graph: event node not found");
    }
  e = cudaGraphInstantiate(&c->prof_graph, graph, 0);
  // instantiated nodes are addressed through the template graph's handles
  if (e == cudaSuccess) {
    c->prof_template = graph;
  } else {
    cudaGraphDestroy(graph);
  }
  CU(e);
  return B2MD_OK;
}

int launch_prof_graph(b2md_ctx* c) {
  TRY(build_prof_graph(c));
  for (size_t p = 0; 2 * p + 1 < c->cap_nodes.size(); ++p) {
    if (c->ev_used == c->ev_pool.size()) {
      cudaEvent_t a, b;
      CU(cudaEventCreate(&a));
      CU(cudaEventCreate(&b));
      c->ev_pool.push_back({a, b});
      c->ev_family.push_back(0);
    }
    c->ev_family[c->ev_used] = c->cap_fam[p];
    CU(cudaGraphExecEventRecordNodeSetEvent(c->prof_graph, c->cap_nodes[2 * p],
                                            c->ev_pool[c->ev_used].first));
    CU(cudaGraphExecEventRecordNodeSetEvent(c->prof_graph, c->cap_nodes[2 * p + 1],
                                            c->ev_pool[c->ev_used].second));
    ++c->ev_used;
  }
  CU(cudaGraphLaunch(c->prof_graph, c->stream));
  return B2MD_OK;
}

// A due re-sort runs between a step's drift and its force evaluation (so the
// bit matrix always matches the current slot order); that step is issued
// eagerly, all others as graphs.
int run_steps(b2md_ctx* c, int64_t nsteps) {
  c->state_in_box = true;  // every step's drift wraps before anything reads the positions
  const bool graphs = c->use_graphs && !c->profile;
  if (nsteps == 1 && c->use_graphs && !sort_due(c) && !nl_due(c)) {
    ++c->steps_since_sort;
    ++c->steps_since_nl;
    if (c->profile) return launch_prof_graph(c);
    TRY(build_single_step_graph(c));
    CU(cudaGraphLaunch(c->single_graph, c->stream));
    return B2MD_OK;
  }
  if (graphs) TRY(build_step_graph(c));
  TRY(launch_step_kernel(c, F_KICK_DRIFT));
  for (int64_t k = 0; k + 1 < nsteps; ++k) {
    if (sort_due(c))
      TRY(resort_and_stage(c));  // (rebuilds the list)
    else if (nl_due(c))
      TRY(nl_build(c));
    ++c->steps_since_sort;
    ++c->steps_since_nl;
    if (graphs)
      CU(cudaGraphLaunch(c->step_graph, c->stream));
    else
      TRY(enqueue_loop_body(c));
  }
  if (sort_due(c))
    TRY(resort_and_stage(c));
  else if (nl_due(c))
    TRY(nl_build(c));
  ++c->steps_since_sort;
  ++c->steps_since_nl;
  TRY(enqueue_forces_and_kick(c));
  return B2MD_OK;
}

// Host AoS <-> device SoA.  Every array has its own staging slot, so a
// sequence of transfers is queued without host synchronisation; callers
// synchronise once.
int upload_aos(b2md_ctx* c, int slot, const double* host, int width, double* d0, double* d1,
               double* d2, double* d3) {
  const int nt = n_total(c);
  double* stage = c->d_stage + size_t(slot) * 4 * nt;
  CU(cudaMemcpyAsync(stage, host, sizeof(double) * width * nt, cudaMemcpyHostToDevice, c->stream));
  k_aos_to_soa<<<(nt + 255) / 256, 256, 0, c->stream>>>(stage, nt, width, d0, d1, d2, d3);
  CU(cudaGetLastError());
  return B2MD_OK;
}

int download_aos(b2md_ctx* c, int slot, double* host, int width, const double* d0,
                 const double* d1, const double* d2, const double* d3) {
  const int nt = n_total(c);
  double* stage = c->d_stage + size_t(slot) * 4 * nt;
  k_soa_to_aos<<<(nt + 255) / 256, 256, 0, c->stream>>>(stage, nt, width, d0, d1, d2, d3);
  CU(cudaGetLastError());
  CU(cudaMemcpyAsync(host, stage, sizeof(double) * width * nt, cudaMemcpyDeviceToHost, c->stream));
  return B2MD_OK;
}

// EnergyBreakdown assembly (src/parallel.cpp:101-120)
void assemble(const b2md_ctx* c, const double* sums, b2md_energy* e, b2md_eval_stats* st) {
  const ModelTables& t = c->t;
  if (e) {
    std::memset(e, 0, sizeof *e);
    e->lj = sums[0];
    e->elec_real = sums[1];
    e->rf = sums[2];
    const double volume = t.box * t.box * t.box;
    e->lrc = t.lrc_k / volume;
    if (t.vderiv) {
      e->du_dv_explicit = sums[3] / (3.0 * volume);
      e->d2u_dv2_explicit = (sums[4] - 2.0 * sums[3]) / (9.0 * volume * volume);
      e->du_dv_lrc = -t.lrc_k / (volume * volume);
      e->d2u_dv2_lrc = 2.0 * t.lrc_k / (volume * volume * volume);
    }
    if (t.ewald) {
      e->elec_recip = sums[7];
      e->elec_self = t.self_plus_intra;
    }
  }
  if (st) {
    st->virial = sums[5];
    st->s1 = sums[3];
    st->s2 = sums[4];
    st->com_pairs = int64_t(sums[6]);
  }
}

// energy sums -> pinned host scratch (queued; read after the caller's sync)
int enqueue_scalars(b2md_ctx* c) {
  const size_t bytes = sizeof(double) * kNumSums * c->R;
  if (!c->h_sums_pinned) CU(cudaMallocHost(&c->h_sums_pinned, bytes));
  CU(cudaMemcpyAsync(c->h_sums_pinned, c->d_fbuf + size_t(6) * n_total(c), bytes,
                     cudaMemcpyDeviceToHost, c->stream));
  return B2MD_OK;
}

void assemble_all(b2md_ctx* c, b2md_energy* e, b2md_eval_stats* st) {
  for (int r = 0; r < c->R; ++r)
    assemble(c, c->h_sums_pinned + size_t(r) * kNumSums, e ? e + r : nullptr, st ? st + r : nullptr);
}

int download_scalars(b2md_ctx* c, b2md_energy* e, b2md_eval_stats* st) {
  if (!e && !st) return B2MD_OK;
  TRY(enqueue_scalars(c));
  CU(cudaStreamSynchronize(c->stream));
  assemble_all(c, e, st);
  return B2MD_OK;
}

// A host pointer the device can access directly (pinned / registered memory
// under unified addressing); nullptr for pageable memory.
const double* device_view(const double* host) {
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, host) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  return at.type == cudaMemoryTypeHost && at.devicePointer
             ? static_cast<const double*>(at.devicePointer) : nullptr;
}

struct AosSpec {
  const double* host;
  int width;
  double* d[4];
};

// Host AoS <-> device SoA for several arrays.  Pinned (device-accessible),
// 16-byte-aligned host arrays are moved by one zero-copy launch per
// direction (flat double2 PCIe transactions, at the link's bandwidth and with
// no per-array copy overheads: six DMA copies of cfg3's arrays take 69 us
// against 53 us); other host memory goes through the copy engines into the
// staging slots plus one batched conversion launch.
// flag: download only — also copy the device error flag into c->h_flag
// (deferred NumericalError of b2md_step_async, read after the caller's sync).
int move_arrays(b2md_ctx* c, const AosSpec* spec, int n, bool upload, bool flag = false) {
  if (flag && !c->h_flag) CU(cudaMallocHost(&c->h_flag, sizeof(int)));
  if (n == 0) {
    if (flag)
      CU(cudaMemcpyAsync(c->h_flag, c->d_error, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    return B2MD_OK;
  }
  const int nt = n_total(c);
  AosBatch b{};
  b.count = nt;
  b.n_arrays = n;
  bool direct = true;
  for (int k = 0; k < n && direct; ++k) {
    const double* v = device_view(spec[k].host);
    if (!v || reinterpret_cast<uintptr_t>(v) % 16 != 0) direct = false;
    b.src[k] = v;
    b.dst[k] = const_cast<double*>(v);
  }
  for (int k = 0; k < n; ++k) {
    b.width[k] = spec[k].width;
    for (int q = 0; q < 4; ++q) b.d[k][q] = spec[k].d[q];
  }
  const dim3 grid((nt + 255) / 256, n);
  if (direct) {
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device);
    const dim3 zgrid(std::max(1, std::min((nt * 2 + 255) / 256, sms * 4)), n);
    if (flag) {
      b.err_src = c->d_error;
      b.err_dst = c->h_flag;
    }
    if (upload)
      k_aos_zero_copy_upload<<<zgrid, 256, 0, c->stream>>>(b);
    else
      k_aos_zero_copy_download<<<zgrid, 256, 0, c->stream>>>(b);
    CU(cudaGetLastError());
    return B2MD_OK;
  }
  // staged: slot k of d_stage holds array k (4 nt doubles per slot).  (Side
  // copy streams and cached transfer graphs were measured: no gain — the
  // copies run at the link's bandwidth, cfg3 2.5 MB in ~48 us per direction.)
  for (int k = 0; k < n; ++k) {
    double* stage = c->d_stage + size_t(k) * 4 * nt;
    b.src[k] = stage;
    b.dst[k] = stage;
  }
  if (upload) {
    for (int k = 0; k < n; ++k)
      CU(cudaMemcpyAsync(c->d_stage + size_t(k) * 4 * nt, spec[k].host,
                         sizeof(double) * spec[k].width * nt, cudaMemcpyHostToDevice, c->stream));
    k_aos_batch_upload<<<grid, 256, 0, c->stream>>>(b);
    CU(cudaGetLastError());
  } else {
    k_aos_batch_download<<<grid, 256, 0, c->stream>>>(b);
    CU(cudaGetLastError());
    for (int k = 0; k < n; ++k)
      CU(cudaMemcpyAsync(const_cast<double*>(spec[k].host), c->d_stage + size_t(k) * 4 * nt,
                         sizeof(double) * spec[k].width * nt, cudaMemcpyDeviceToHost, c->stream));
    if (flag)
      CU(cudaMemcpyAsync(c->h_flag, c->d_error, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  }
  return B2MD_OK;
}

int upload_arrays(b2md_ctx* c, const AosSpec* spec, int n) { return move_arrays(c, spec, n, true); }
int download_arrays(b2md_ctx* c, const AosSpec* spec, int n) { return move_arrays(c, spec, n, false); }

int setup_shard(b2md_ctx* c) {
  int64_t cand = 0;
  shard_plan(c->t.n, int(c->t.kv.size()), c->world, c->rank, c->row_begin, c->row_end, c->k_begin,
             c->k_end, cand);
  // super tiles (SI, SJ), SI in this rank's super-tile rows, SI <= SJ
  std::vector<uint32_t> list;
  const int s0 = c->row_begin / c->g.st, s1 = (c->row_end + c->g.st - 1) / c->g.st;
  for (int si = s0; si < s1; ++si)
    for (int sj = si; sj < c->g.n_super; ++sj) list.push_back((uint32_t(si) << 16) | uint32_t(sj));
  // heaviest first: with spatially ordered molecules the tiles that survive
  // culling sit near the (periodic) diagonal; launching them first shortens
  // the tail.  The order does not affect results.
  const int ns = c->g.n_super;
  auto band = [ns](uint32_t code) {
    const int d = int(code & 0xffffu) - int(code >> 16);
    return std::min(d, ns - d);
  };
  std::stable_sort(list.begin(), list.end(),
                   [&](uint32_t x, uint32_t y) { return band(x) < band(y); });
  if (c->d_super) cudaFree(c->d_super);
  c->d_super = nullptr;
  TRY(dalloc(&c->d_super, list.size()));
  if (!list.empty())
    CU(cudaMemcpy(c->d_super, list.data(), sizeof(uint32_t) * list.size(), cudaMemcpyHostToDevice));
  c->n_super_tiles = int(list.size());
  // a fresh bit matrix: only this rank's tiles are ever written afterwards
  CU(cudaMemset(c->d_mask, 0, sizeof(uint32_t) * size_t(c->R) * c->g.n_pad * c->g.words));
  c->mask_valid = false;
  drop_graphs(c);
  return B2MD_OK;
}

int create_impl(int device, const b2md_composition* comp, const b2md_ff_options* opts, double dt,
                int R, b2md_ctx* c) {
  std::string err;
  if (int rc = build_tables(*comp, *opts, c->t, err)) return set_err(rc, err);
  const ModelTables& t = c->t;
  if (t.ns > kMaxSpecies) return set_err(B2MD_CONFIG_ERROR, "b200md: at most 8 species");
  size_t nlj = 0, nqq = 0;
  for (const auto& v : t.lj) nlj += v.size();
  for (const auto& v : t.qq) nqq += v.size();
  if (nlj > size_t(kMaxLjTerms) || nqq > size_t(kMaxQqTerms))
    return set_err(B2MD_CONFIG_ERROR, "b200md: too many site-site terms");
  if (R < 1) return set_err(B2MD_INVALID_ARGUMENT, "n_replicas must be >= 1");
  if (dt > 0.0) {
    c->engine = true;
    c->dt = dt;
  }
  c->R = R;
  c->device = device;
  c->warning = t.warning;
  int ndev = 0;
  CU(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev) return set_err(B2MD_CUDA_ERROR, "b200md: no such CUDA device");
  CU(cudaSetDevice(device));
  cudaDeviceGetAttribute(&c->sms, cudaDevAttrMultiProcessorCount, device);
  CU(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
  CU(cudaStreamCreateWithFlags(&c->stream2, cudaStreamNonBlocking));
  CU(cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming));
  CU(cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming));
  c->g = search_geometry(t.n);
  if (size_t(t.n) * size_t(t.n) > (size_t(1) << 32))
    return set_err(B2MD_CONFIG_ERROR, "b200md: too many molecules");

  // tables
  DevTables* h = new DevTables();
  std::memset(h, 0, sizeof(DevTables));
  h->ns = t.ns;
  for (int s = 0; s < t.ns; ++s) {
    const b2md_species& sp = t.species[s];
    DevSpecies& d = h->species[s];
    d.n_sites = sp.n_sites;
    d.rotational_dof = sp.rotational_dof;
    const double n2 = sp.sites[0].body_pos[0] * sp.sites[0].body_pos[0] +
                      sp.sites[0].body_pos[1] * sp.sites[0].body_pos[1] +
                      sp.sites[0].body_pos[2] * sp.sites[0].body_pos[2];
    d.centred = (sp.n_sites == 1 && n2 == 0.0) ? 1 : 0;
    d.total_mass = sp.total_mass;
    for (int k = 0; k < 3; ++k) d.inertia[k] = sp.inertia_principal[k];
    for (int k = 0; k < sp.n_sites; ++k)
      for (int x = 0; x < 3; ++x) d.body[k][x] = sp.sites[k].body_pos[x];
  }
  int lj_at = 0, qq_at = 0;
  for (int p = 0; p < t.ns * t.ns; ++p) {
    DevPairInfo& pi = h->pair[p];
    pi.lj_begin = lj_at;
    pi.lj_count = int(t.lj[p].size());
    for (const auto& term : t.lj[p]) h->lj[lj_at++] = {term.a, term.b, term.c12, term.c6};
    pi.qq_begin = qq_at;
    pi.qq_count = int(t.qq[p].size());
    for (const auto& term : t.qq[p]) h->qq[qq_at++] = {term.a, term.b, term.qq};
    pi.rmax2 = t.single_site_path ? t.rc2 : t.rmax2[p];
  }
  int rc = dalloc(&c->d_tab, 1);
  if (!rc) rc = cudaMemcpy(c->d_tab, h, sizeof(DevTables), cudaMemcpyHostToDevice) ? B2MD_CUDA_ERROR : 0;
  delete h;
  if (rc) return set_err(B2MD_CUDA_ERROR, "b200md: table upload failed");
  TRY(dalloc(&c->d_species_of, t.n));
  TRY(dalloc(&c->d_site_begin, t.n + 1));
  CU(cudaMemcpy(c->d_species_of, t.species_of.data(), sizeof(int) * t.n, cudaMemcpyHostToDevice));
  CU(cudaMemcpy(c->d_site_begin, t.site_begin.data(), sizeof(int) * (t.n + 1), cudaMemcpyHostToDevice));

  const size_t nt = size_t(t.n) * R;
  TRY(dalloc(&c->d_state, 13 * nt));
  TRY(dalloc(&c->d_fbuf, 6 * nt + size_t(kNumSums) * R));
  TRY(dalloc(&c->d_off, size_t(t.total_sites) * R));
  // + two clusters: the cluster walk stages whole clusters (and a pad cluster)
  TRY(dalloc(&c->d_pos4, nt + 2 * kCS));
  CU(cudaMemset(c->d_pos4, 0, sizeof(double4) * (nt + 2 * kCS)));
  TRY(dalloc(&c->d_stage, 6 * 4 * nt));
  TRY(dalloc(&c->d_mask, size_t(R) * c->g.n_pad * c->g.words));
  TRY(dalloc(&c->d_fixpos, nt));
  {
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    // row split: two warps per row for the general multi-site kernel
    // (charge terms: erfc / exp per site pair) when its rows do not fill the
    // resident warps (16 per SM at 128 registers).  Measured (steps/s): cfg2
    // S=1 4.2k, S=2 5.0k, S=4 4.7k; the LJ-only walks lose at any split
    // (cfg0 S=4 -23%, cfg1 S=2 -17%, cfg4 S=2 -18%: duplicated expansion
    // outweighs the extra warps).
    const bool multi_kernel = !t.single_site_path && rigid_sites(t) == 0;
    const long resident = long(sms) * 16;
    int S = multi_kernel && long(t.n) * R < resident ? 2 : 1;
    if (const char* e = std::getenv("B2MD_FORCE_SPLIT")) S = std::max(1, std::min(kForceWarps, std::atoi(e)));
    while (kForceWarps % S) --S;
    c->force_split = S;
    const int rpc = kForceWarps / S;
    const int rows_grid = (t.n + rpc - 1) / rpc;
    c->force_grid = std::max(1, std::min(rows_grid, sms * 4));
    // re-sort only where the search's tile cull can use the order: single
    // species (fixed-point path) and a COM radius well below L/2
    const double rmax = std::sqrt(t.single_site_path ? t.rc2 : t.rmax2[0]);
    c->sort_interval = (t.ns == 1 && rmax < 0.3 * t.box) ? 100 : 0;
    // cluster walk (single-site path) where its cull pays: a cutoff well
    // below L/2 (cfg0's rc = 0.45 L culls nothing; measured 24.6k vs 32k
    // steps/s there); compact clusters need a fresher order than search
    // tiles.  B2MD_CLUSTER=0 disables it, =2 forces it (tests, measurement).
    int cl_mode = 1;
    if (const char* e = std::getenv("B2MD_CLUSTER")) cl_mode = std::atoi(e);
    if (t.single_site_path && (cl_mode == 2 || (cl_mode == 1 && rmax < 0.3 * t.box))) {
      c->nc = (t.n + kCS - 1) / kCS;
      if (rmax < 0.3 * t.box) c->sort_interval = 40;
    }
    if (const char* e = std::getenv("B2MD_SORT_INTERVAL")) c->sort_interval = std::max(0, std::atoi(e));
    // tuning knobs (measurement only): warps per CTA, CTAs per replica
    if (const char* e = std::getenv("B2MD_FORCE_WARPS"))
      c->force_warps = std::max(1, std::min(kForceWarps, std::atoi(e)));
    if (const char* e = std::getenv("B2MD_FORCE_GRID")) c->force_grid = std::max(1, std::atoi(e));
    // the fused kick runs on each row's lane 0: it pays for small systems
    // (one launch less), but lengthens every warp's critical path when warps
    // own several rows (measured: cfg0/cfg1 +3-7%, cfg3/cfg4 -2-4%)
    c->use_fused_kick = size_t(t.n) * R < 4096;
    // the cluster-pair walk ends with 4 rows per warp written by 4 lanes:
    // the kick costs those lanes a few loads, not a serial row epilogue
    if (c->nc > 0) c->use_fused_kick = true;
    if (const char* e = std::getenv("B2MD_FUSED_KICK")) c->use_fused_kick = std::atoi(e) != 0;
  }
  // per-CTA scalar partials of the widest force grid: the row walks, the
  // both-rows cluster walk (kGWarps groups per CTA) and the once-per-pair
  // walk (down to one cluster per CTA)
  {
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device);
    TRY(dalloc(&c->d_cta_part, size_t(R) * kNumRowScalars *
                                   std::max({c->force_grid, c->nc > 0 ? cpair_grid(c) : 0,
                                             c->nc > 0 ? sms * kNLMinBlocks * 8 : 0,
                                             (((c->t.n + 31) / 32) * ((c->t.n + 31) / 32 + 1) / 2 *
                                                  kTileSplit + kTileWarps - 1) / kTileWarps})));
  }
  if (c->nc > 0) {
    c->nsup = (c->nc + kSC - 1) / kSC;
    TRY(dalloc(&c->d_carc, size_t(R) * c->nc));
    TRY(dalloc(&c->d_chalf, size_t(R) * c->nc));
    TRY(dalloc(&c->d_sarc, size_t(R) * c->nsup));
    TRY(dalloc(&c->d_shalf, size_t(R) * c->nsup));
    // once-per-pair list: worst-case capacity (every cluster pair listed),
    // 192 B of record per entry; beyond 8 GB the both-rows walk runs
    if (const char* e = std::getenv("B2MD_NEWTON")) c->use_newton = std::atoi(e) != 0;
    const size_t nc = size_t(c->nc);
    // every cluster pair once, plus < kB padding entries per owner
    const size_t max_ent = (nc * (nc + 1) / 2 + nc * kB + kB - 1) / kB * kB;
    if (size_t(R) * max_ent * kRecP * sizeof(double) > (size_t(8) << 30))
      c->use_newton = false;
    if (c->use_newton) {
      // the end-of-step kick runs in k_nl_reduce (its inputs fetched ahead of
      // the record loop); B2MD_FUSED_KICK=0: with the next step's drift
      // (k_step_drift_arcs<true>) / a k_kick launch at the end of a run
      c->use_fused_kick = true;
      if (const char* e = std::getenv("B2MD_FUSED_KICK")) c->use_fused_kick = std::atoi(e) != 0;
      NListArgs& nl = c->nl;
      int sms = 148;
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device);
      c->n3_grid = sms * kNLMinBlocks;
      // (measurement) more CTAs than resident slots: the hardware deals them as slots free up
      if (const char* e = std::getenv("B2MD_NL_GRIDMUL"))
        c->n3_grid *= std::max(1, std::min(8, std::atoi(e)));
      nl.max_ent = int(max_ent);
      TRY(dalloc(&nl.rec, size_t(R) * max_ent * kRecP));
      TRY(dalloc(&nl.rstamp, size_t(R) * max_ent));
      TRY(dalloc(&nl.irec, size_t(R) * (max_ent / kB) * kRecD));
      TRY(dalloc(&nl.ocnt, size_t(R) * nc));
      TRY(dalloc(&nl.ocp, size_t(R) * nc * kNLParts));
      TRY(dalloc(&nl.icp, size_t(R) * nc * kNLParts));
      TRY(dalloc(&nl.icnt, size_t(R) * nc));
      TRY(dalloc(&nl.ebase, size_t(R) * (nc + 1)));
      TRY(dalloc(&nl.ibase, size_t(R) * (nc + 1)));
      TRY(dalloc(&nl.ent, size_t(R) * max_ent));
      TRY(dalloc(&nl.in_src, size_t(R) * max_ent));
      // dense [owner][receiver] slot map up to 256 MB (nc <= 8k clusters on one replica)
      if (size_t(R) * nc * nc * sizeof(int) <= (size_t(256) << 20)) TRY(dalloc(&nl.smap, size_t(R) * nc * nc));
      TRY(dalloc(&nl.fixref, size_t(R) * c->t.n));
      TRY(dalloc(&nl.ctl, size_t(R) * kNLCtl));
      // stale until the first build; epoch 1 (the stamps start at 0)
      std::vector<int> ctl(size_t(R) * kNLCtl, 0);
      for (int r = 0; r < R; ++r) {
        ctl[size_t(r) * kNLCtl + kNLOverflow] = 1;
        ctl[size_t(r) * kNLCtl + kNLEpoch] = 1;
      }
      CU(cudaMemcpy(nl.ctl, ctl.data(), sizeof(int) * ctl.size(), cudaMemcpyHostToDevice));
      // skin and scheduled rebuild interval (B2MD_NL_SKIN, B2MD_NL_INTERVAL)
      c->nl_skin = 1.0;
      c->nl_interval = 15;
      if (const char* e = std::getenv("B2MD_NL_SKIN")) c->nl_skin = std::max(0.0, std::atof(e));
      if (const char* e = std::getenv("B2MD_NL_INTERVAL")) c->nl_interval = std::max(0, std::atoi(e));
      // member-pair build gaps (k_nl_gaps); 0: the arcs' bound only (measurement)
      if (const char* e = std::getenv("B2MD_NL_GAPS")) c->nl_member_gaps = std::atoi(e) != 0;
      const double rs = (std::sqrt(c->t.rc2) + c->nl_skin) * 4294967296.0 / c->t.box;
      nl.lim_build = float(rs * rs * (1.0 + 1e-5));
      nl.skin_half = float(0.5 * c->nl_skin * 4294967296.0 / c->t.box + 64.0);
      nl.rc_fix = float(std::sqrt(c->t.rc2) * 4294967296.0 / c->t.box);
      const double du = 0.5 * c->nl_skin * 4294967296.0 / c->t.box;
      const float d2s = float(du * du * (1.0 - 1e-4));
      std::memcpy(&nl.d2_stale, &d2s, sizeof d2s);
    }
  }
  if (rigid_sites(c->t) > 0) {
    if (const char* e = std::getenv("B2MD_TILE")) c->use_tile = std::atoi(e) != 0;
    if (c->use_tile) {
      c->tile_nb = (c->t.n + 31) / 32;
      c->tile_nbp = c->tile_nb * (c->tile_nb + 1) / 2;
      TRY(dalloc(&c->d_trec, size_t(R) * c->tile_nbp * kTileSplit * 2 * 32 * 6));
    }
  }
  TRY(dalloc(&c->d_ticket, size_t(2) * R));
  TRY(dalloc(&c->d_flux, size_t(kNumSums) * R));
  TRY(dalloc(&c->d_ke, R));
  TRY(dalloc(&c->d_thermo_err, R));
  CU(cudaMemset(c->d_thermo_err, 0, sizeof(int) * R));
  {
    // spatial-order tables, identity until the first resort
    TRY(dalloc(&c->d_perm, nt));
    TRY(dalloc(&c->d_slot_of, nt));
    TRY(dalloc(&c->d_sp_slot, nt));
    TRY(dalloc(&c->d_sb_slot, nt));
    TRY(dalloc(&c->d_nsites_slot, nt));
    TRY(dalloc(&c->d_scan, nt));
    TRY(dalloc(&c->d_keys[0], nt));
    TRY(dalloc(&c->d_keys[1], nt));
    TRY(dalloc(&c->d_vals[0], nt));
    TRY(dalloc(&c->d_vals[1], nt));
    std::vector<int> ident(nt), sp(nt), sb(nt);
    for (size_t g = 0; g < nt; ++g) {
      const int i = int(g % t.n);
      ident[g] = i;
      sp[g] = t.species_of[i];
      sb[g] = t.site_begin[i];
    }
    CU(cudaMemcpy(c->d_perm, ident.data(), sizeof(int) * nt, cudaMemcpyHostToDevice));
    CU(cudaMemcpy(c->d_slot_of, ident.data(), sizeof(int) * nt, cudaMemcpyHostToDevice));
    CU(cudaMemcpy(c->d_sp_slot, sp.data(), sizeof(int) * nt, cudaMemcpyHostToDevice));
    CU(cudaMemcpy(c->d_sb_slot, sb.data(), sizeof(int) * nt, cudaMemcpyHostToDevice));
    size_t b1 = 0, b2 = 0;
    CU(cub::DeviceRadixSort::SortPairs(nullptr, b1, c->d_keys[0], c->d_keys[1], c->d_vals[0],
                                       c->d_vals[1], int(nt), 0, 52));
    CU(cub::DeviceScan::ExclusiveSum(nullptr, b2, c->d_nsites_slot, c->d_scan, int(nt)));
    c->cub_bytes = std::max(b1, b2);
    CU(cudaMalloc(&c->d_cub, c->cub_bytes));
  }
  TRY(dalloc(&c->d_error, 1));
  const int big = INT_MAX;
  CU(cudaMemcpy(c->d_error, &big, sizeof(int), cudaMemcpyHostToDevice));
  double* s = c->d_state;
  c->st.px = s + 0 * nt;
  c->st.py = s + 1 * nt;
  c->st.pz = s + 2 * nt;
  c->st.qw = s + 3 * nt;
  c->st.qx = s + 4 * nt;
  c->st.qy = s + 5 * nt;
  c->st.qz = s + 6 * nt;
  c->st.vx = s + 7 * nt;
  c->st.vy = s + 8 * nt;
  c->st.vz = s + 9 * nt;
  c->st.wx = s + 10 * nt;
  c->st.wy = s + 11 * nt;
  c->st.wz = s + 12 * nt;
  c->st.fx = c->d_fbuf + 0 * nt;
  c->st.fy = c->d_fbuf + 1 * nt;
  c->st.fz = c->d_fbuf + 2 * nt;
  c->st.tx = c->d_fbuf + 3 * nt;
  c->st.ty = c->d_fbuf + 4 * nt;
  c->st.tz = c->d_fbuf + 5 * nt;
  c->st.off = c->d_off;
  c->st.pos4 = c->d_pos4;

  c->sys.n = t.n;
  c->sys.R = R;
  c->sys.total_sites = t.total_sites;
  c->sys.n_pad = c->g.n_pad;
  c->sys.words = c->g.words;
  c->sys.ns = t.ns;
  c->sys.species_of = c->d_species_of;
  c->sys.site_begin = c->d_site_begin;
  c->sys.tab = c->d_tab;
  c->sys.perm = c->d_perm;
  c->sys.slot_of = c->d_slot_of;
  c->sys.sp_slot = c->d_sp_slot;
  c->sys.sb_slot = c->d_sb_slot;
  MinImage& mi = c->sys.mi;
  mi.L = t.box;
  mi.negL = -t.box;
  mi.hi_lo = hi32(0.5 * t.box);
  mi.hi_hi = mi.hi_lo + 1;
  mi.hi_max = hi32(1.5 * t.box) - 1;

  // Ewald
  if (t.ewald) {
    c->nq = int(t.charged.size());
    std::vector<int> qm, qs, qb(t.n + 1, 0);
    std::vector<double> qv;
    for (const auto& ch : t.charged) {
      qm.push_back(ch.mol);
      qs.push_back(ch.site);
      qv.push_back(ch.q);
      qb[ch.mol + 1]++;
    }
    for (int m = 0; m < t.n; ++m) qb[m + 1] += qb[m];
    TRY(dalloc(&c->d_q_mol, c->nq));
    TRY(dalloc(&c->d_q_site, c->nq));
    TRY(dalloc(&c->d_q_val, c->nq));
    TRY(dalloc(&c->d_mol_qbegin, t.n + 1));
    if (c->nq) {
      CU(cudaMemcpy(c->d_q_mol, qm.data(), sizeof(int) * c->nq, cudaMemcpyHostToDevice));
      CU(cudaMemcpy(c->d_q_site, qs.data(), sizeof(int) * c->nq, cudaMemcpyHostToDevice));
      CU(cudaMemcpy(c->d_q_val, qv.data(), sizeof(double) * c->nq, cudaMemcpyHostToDevice));
    }
    CU(cudaMemcpy(c->d_mol_qbegin, qb.data(), sizeof(int) * (t.n + 1), cudaMemcpyHostToDevice));
    std::vector<DevKVec> kv;
    for (const auto& k : t.kv) kv.push_back({k.kx, k.ky, k.kz, k.coeff, k.nx, k.ny, k.nz, 0});
    TRY(dalloc(&c->d_kv, kv.size()));
    if (!kv.empty())
      CU(cudaMemcpy(c->d_kv, kv.data(), sizeof(DevKVec) * kv.size(), cudaMemcpyHostToDevice));
    TRY(dalloc(&c->d_etab, size_t(R) * 3 * (t.kmax + 1) * std::max(c->nq, 1)));
    TRY(dalloc(&c->d_S, size_t(R) * std::max<size_t>(kv.size(), 1)));
    TRY(dalloc(&c->d_uk, size_t(R) * std::max<size_t>(kv.size(), 1)));
    // tiled S(k) / forces (kernels.cuh): chunk partials and per-charge forces
    // (measured on cfg2: equal to the gather form -- 6.33k vs 6.38k steps/s --
    // so the gather form stays the default; B2MD_EWALD_TILED=1 selects it)
    c->ew_tiled = false;
    if (const char* e = std::getenv("B2MD_EWALD_TILED")) c->ew_tiled = t.kmax + 1 <= kEwMaxK && std::atoi(e) != 0;
    if (c->ew_tiled) {
      const size_t nch = (size_t(std::max(c->nq, 1)) + kEwSkQ - 1) / kEwSkQ;
      TRY(dalloc(&c->d_ewSp, size_t(R) * nch * std::max<size_t>(kv.size(), 1)));
      TRY(dalloc(&c->d_ewfq, size_t(R) * std::max(c->nq, 1) * 3));
    }
    // reciprocal forces / torques written beside the real-space kernel in the
    // step paths (ewald_overlap; B2MD_EWALD_OVERLAP=0: after it, added in place)
    if (c->nq > 0) TRY(dalloc(&c->d_frec, size_t(6) * R * t.n));
    if (const char* e = std::getenv("B2MD_EWALD_OVERLAP")) c->ew_overlap = std::atoi(e) != 0;
  }
  c->rank = 0;
  c->world = 1;
  TRY(setup_shard(c));
  CU(cudaDeviceSynchronize());
  return B2MD_OK;
}

void free_ctx(b2md_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  drop_graphs(c);
  for (auto& e : c->ev_pool) {
    cudaEventDestroy(e.first);
    cudaEventDestroy(e.second);
  }
  if (c->comm) g_nccl.CommDestroy(c->comm);
  if (c->h_sums_pinned) cudaFreeHost(c->h_sums_pinned);
  if (c->h_flag) cudaFreeHost(c->h_flag);
  void* ptrs[] = {c->d_tab,   c->d_species_of, c->d_site_begin, c->d_state, c->d_fbuf, c->d_off,
                  c->d_stage, c->d_mask,       c->d_cta_part, c->d_ticket, c->d_fixpos, c->d_pos4,   c->d_super, c->d_error, c->d_q_mol,
                  c->d_q_site, c->d_q_val,     c->d_mol_qbegin, c->d_kv,    c->d_etab,  c->d_S,
                  c->d_uk,    c->d_flux,  c->d_perm, c->d_slot_of, c->d_sp_slot, c->d_sb_slot,
                  c->d_nsites_slot, c->d_scan, c->d_keys[0], c->d_keys[1], c->d_vals[0],
                  c->d_vals[1], c->d_cub, c->d_ke, c->d_thermo_err, c->d_carc,
                  c->d_chalf, c->d_sarc, c->d_shalf, c->d_trec, c->d_ewSp, c->d_ewfq, c->d_frec, c->nl.rec, c->nl.irec,
                  c->nl.ocnt, c->nl.icnt, c->nl.ebase, c->nl.ibase, c->nl.ent,
                  c->nl.in_src, c->nl.fixref, c->nl.rstamp, c->nl.smap, c->nl.ocp, c->nl.icp,
                  c->nl.ctl};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  if (c->stream) cudaStreamDestroy(c->stream);
  if (c->stream2) cudaStreamDestroy(c->stream2);
  if (c->ev_fork) cudaEventDestroy(c->ev_fork);
  if (c->ev_join) cudaEventDestroy(c->ev_join);
  delete c;
  cudaGetLastError();  // (a context that failed to create leaves no error behind)
}

int check_error_flag(b2md_ctx* c) {
  int flag = INT_MAX;
  CU(cudaMemcpyAsync(&flag, c->d_error, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  CU(cudaStreamSynchronize(c->stream));
  c->async_pending = false;
  return error_from_flag(c, flag);
}

// The NumericalError of check_finite (model.cpp:288-302) for a device error
// flag value already on the host (INT_MAX: none).
int error_from_flag(b2md_ctx* c, int flag) {
  if (flag == INT_MAX) return B2MD_OK;
  const int r = flag / c->t.n, i = flag % c->t.n;
  double v[6];
  const size_t nt = n_total(c);
  const double* srcs[6] = {c->st.px + flag, c->st.py + flag, c->st.pz + flag,
                           c->st.vx + flag, c->st.vy + flag, c->st.vz + flag};
  for (int k = 0; k < 6; ++k) CU(cudaMemcpy(&v[k], srcs[k], sizeof(double), cudaMemcpyDeviceToHost));
  (void)nt;
  char buf[512];
  std::snprintf(buf, sizeof buf,
                "engine step: non-finite state for molecule %d (pos %g %g %g, vel %g %g %g)%s", i,
                v[0], v[1], v[2], v[3], v[4], v[5], c->R > 1 ? " in replica" : "");
  std::string msg = buf;
  if (c->R > 1) msg += " " + std::to_string(r);
  return set_err(B2MD_NUMERICAL_ERROR, msg);
}

}  // namespace b2md_host

using namespace b2md_host;

// ============================================================== C ABI
extern "C" {

const char* b2md_last_error(void) { return g_err.c_str(); }
int b2md_abi_version(void) { return B2MD_ABI_VERSION; }

int b2md_build_species(const b2md_site* sites, int n_sites, b2md_species* out) {
  if (!sites || !out) return set_err(B2MD_INVALID_ARGUMENT, "build_species: null pointer");
  std::string err;
  if (int rc = build_species(sites, n_sites, *out, err)) return set_err(rc, err);
  return B2MD_OK;
}

int b2md_ewald_tune(double delta, double cutoff, double box_length, double* alpha, int* kmax) {
  if (!alpha || !kmax) return set_err(B2MD_INVALID_ARGUMENT, "ewald_tune: null pointer");
  std::string err;
  if (int rc = ewald_tune(delta, cutoff, box_length, *alpha, *kmax, err)) return set_err(rc, err);
  return B2MD_OK;
}

int b2md_ewald_kvector_count(int kmax, int* count) {
  if (!count || kmax < 0) return set_err(B2MD_INVALID_ARGUMENT, "kvector_count: bad argument");
  *count = count_kvectors(kmax);
  return B2MD_OK;
}

int b2md_shard_plan(int n_molecules, int n_kvectors, int world, int rank, int* row_begin,
                    int* row_end, int* k_begin, int* k_end, int64_t* candidate_pairs) {
  if (n_molecules < 1 || world < 1 || rank < 0 || rank >= world || !row_begin || !row_end ||
      !k_begin || !k_end || !candidate_pairs)
    return set_err(B2MD_INVALID_ARGUMENT, "shard_plan: bad argument");
  shard_plan(n_molecules, n_kvectors, world, rank, *row_begin, *row_end, *k_begin, *k_end,
             *candidate_pairs);
  return B2MD_OK;
}

int b2md_create(int device, const b2md_composition* comp, const b2md_ff_options* opts, double dt,
                int n_replicas, b2md_ctx** out) {
  NvtxRange nvtx_("b2md_create");
  if (!comp || !opts || !out) return set_err(B2MD_INVALID_ARGUMENT, "create: null pointer");
  *out = nullptr;
  b2md_ctx* c = new b2md_ctx();
  int rc = create_impl(device, comp, opts, dt, n_replicas, c);
  if (rc) {
    const std::string keep = g_err;
    free_ctx(c);
    g_err = keep;
    return rc;
  }
  *out = c;
  return B2MD_OK;
}

void b2md_destroy(b2md_ctx* ctx) { free_ctx(ctx); }

const char* b2md_warning(const b2md_ctx* ctx) { return ctx ? ctx->warning.c_str() : ""; }

int b2md_evaluate(b2md_ctx* c, const double* pos, const double* orient, double* force,
                  double* torque, b2md_energy* energy, b2md_eval_stats* stats) {
  NvtxRange nvtx_("b2md_evaluate");
  if (!c || !pos) return set_err(B2MD_INVALID_ARGUMENT, "evaluate: null pointer");
  CU(cudaSetDevice(c->device));
  TRY(upload_aos(c, 0, pos, 3, c->st.px, c->st.py, c->st.pz, nullptr));
  if (orient) {
    TRY(upload_aos(c, 1, orient, 4, c->st.qw, c->st.qx, c->st.qy, c->st.qz));
  } else if (c->t.any_offsets) {
    return set_err(B2MD_INVALID_ARGUMENT, "evaluate: orientations required for multi-site species");
  }
  set_wrapped(c, false);
  c->state_in_box = false;
  if (c->sort_interval > 0) TRY(resort(c));
  TRY(enqueue_forces(c, true));
  if (force) TRY(download_aos(c, 4, force, 3, c->st.fx, c->st.fy, c->st.fz, nullptr));
  if (torque) TRY(download_aos(c, 5, torque, 3, c->st.tx, c->st.ty, c->st.tz, nullptr));
  TRY(download_scalars(c, energy, stats));
  CU(cudaStreamSynchronize(c->stream));
  c->state_valid = false;  // velocities not set: not an engine state
  return B2MD_OK;
}

int b2md_set_state(b2md_ctx* c, const double* pos, const double* orient, const double* vel,
                   const double* ang_vel) {
  NvtxRange nvtx_("b2md_set_state");
  if (!c || !pos || !orient || !vel || !ang_vel)
    return set_err(B2MD_INVALID_ARGUMENT, "set_state: null pointer");
  CU(cudaSetDevice(c->device));
  TRY(upload_aos(c, 0, pos, 3, c->st.px, c->st.py, c->st.pz, nullptr));
  TRY(upload_aos(c, 1, orient, 4, c->st.qw, c->st.qx, c->st.qy, c->st.qz));
  TRY(upload_aos(c, 2, vel, 3, c->st.vx, c->st.vy, c->st.vz, nullptr));
  TRY(upload_aos(c, 3, ang_vel, 3, c->st.wx, c->st.wy, c->st.wz, nullptr));
  const int nt = n_total(c);
  // state_.wrap() (engine.cpp:96): px, py, pz are contiguous
  k_wrap<<<(3 * nt + 255) / 256, 256, 0, c->stream>>>(c->st.px, 3 * nt, c->t.box);
  CU(cudaGetLastError());
  set_wrapped(c, true);
  c->state_in_box = true;
  const int big = INT_MAX;
  CU(cudaMemcpyAsync(c->d_error, &big, sizeof(int), cudaMemcpyHostToDevice, c->stream));
  if (c->sort_interval > 0) TRY(resort(c));
  TRY(enqueue_forces(c, true));
  CU(cudaStreamSynchronize(c->stream));
  c->state_valid = true;
  return B2MD_OK;
}

int b2md_step(b2md_ctx* c, int64_t nsteps) {
  NvtxRange nvtx_("b2md_step");
  if (!c) return set_err(B2MD_INVALID_ARGUMENT, "step: null context");
  if (!c->engine) return set_err(B2MD_CONFIG_ERROR, "engine: time step must be positive");
  if (!c->state_valid) return set_err(B2MD_CONFIG_ERROR, "engine: set_state must precede step");
  if (nsteps <= 0) return B2MD_OK;
  CU(cudaSetDevice(c->device));
  TRY(run_steps(c, nsteps));
  return check_error_flag(c);
}

int b2md_step_async(b2md_ctx* c, int64_t nsteps) {
  NvtxRange nvtx_("b2md_step_async");
  if (!c) return set_err(B2MD_INVALID_ARGUMENT, "step: null context");
  if (!c->engine) return set_err(B2MD_CONFIG_ERROR, "engine: time step must be positive");
  if (!c->state_valid) return set_err(B2MD_CONFIG_ERROR, "engine: set_state must precede step");
  if (nsteps <= 0) return B2MD_OK;
  CU(cudaSetDevice(c->device));
  TRY(run_steps(c, nsteps));
  c->async_pending = true;
  return B2MD_OK;
}

int b2md_sync(b2md_ctx* c) {
  NvtxRange nvtx_("b2md_sync");
  if (!c) return set_err(B2MD_INVALID_ARGUMENT, "sync: null context");
  CU(cudaSetDevice(c->device));
  return check_error_flag(c);
}

int b2md_upload_state(b2md_ctx* c, const double* pos, const double* orient, const double* vel,
                      const double* ang_vel, const double* force, const double* torque) {
  NvtxRange nvtx_("b2md_upload_state");
  if (!c) return set_err(B2MD_INVALID_ARGUMENT, "upload_state: null context");
  CU(cudaSetDevice(c->device));
  AosSpec spec[6];
  int n = 0;
  if (pos) spec[n++] = {pos, 3, {c->st.px, c->st.py, c->st.pz, nullptr}};
  if (orient) spec[n++] = {orient, 4, {c->st.qw, c->st.qx, c->st.qy, c->st.qz}};
  if (vel) spec[n++] = {vel, 3, {c->st.vx, c->st.vy, c->st.vz, nullptr}};
  if (ang_vel) spec[n++] = {ang_vel, 3, {c->st.wx, c->st.wy, c->st.wz, nullptr}};
  if (force) spec[n++] = {force, 3, {c->st.fx, c->st.fy, c->st.fz, nullptr}};
  if (torque) spec[n++] = {torque, 3, {c->st.tx, c->st.ty, c->st.tz, nullptr}};
  TRY(upload_arrays(c, spec, n));
  if (pos) c->mask_valid = false;
  // steps wrap before every evaluation, so step-time forces may use the fast
  // path; the uploaded positions themselves are taken as given (no wrap), so
  // consumers of the current state (heat flux) use the exact minimum image
  // until a step has wrapped them
  set_wrapped(c, true);
  if (pos) c->state_in_box = false;
  c->state_valid = true;
  return B2MD_OK;
}

int b2md_get_state(b2md_ctx* c, double* pos, double* orient, double* vel, double* ang_vel,
                   double* force, double* torque, b2md_energy* energy, b2md_eval_stats* stats) {
  NvtxRange nvtx_("b2md_get_state");
  if (!c) return set_err(B2MD_INVALID_ARGUMENT, "get_state: null context");
  CU(cudaSetDevice(c->device));
  AosSpec spec[6];
  int n = 0;
  if (pos) spec[n++] = {pos, 3, {c->st.px, c->st.py, c->st.pz, nullptr}};
  if (orient) spec[n++] = {orient, 4, {c->st.qw, c->st.qx, c->st.qy, c->st.qz}};
  if (vel) spec[n++] = {vel, 3, {c->st.vx, c->st.vy, c->st.vz, nullptr}};
  if (ang_vel) spec[n++] = {ang_vel, 3, {c->st.wx, c->st.wy, c->st.wz, nullptr}};
  if (force) spec[n++] = {force, 3, {c->st.fx, c->st.fy, c->st.fz, nullptr}};
  if (torque) spec[n++] = {torque, 3, {c->st.tx, c->st.ty, c->st.tz, nullptr}};
  // after b2md_step_async the error flag rides along with the arrays, so the
  // step's NumericalError is reported here without a sync of its own
  const bool flag = c->async_pending;
  TRY(move_arrays(c, spec, n, false, flag));
  if (energy || stats) TRY(enqueue_scalars(c));
  CU(cudaStreamSynchronize(c->stream));  // one sync for arrays, sums and flag
  if (energy || stats) assemble_all(c, energy, stats);
  if (flag) {
    c->async_pending = false;
    return error_from_flag(c, *c->h_flag);
  }
  return B2MD_OK;
}

int b2md_set_search_options(b2md_ctx* c, int fix_prefilter, int tile_cull) {
  if (!c) return set_err(B2MD_INVALID_ARGUMENT, "set_search_options: null context");
  c->use_fix_prefilter = fix_prefilter != 0;
  c->use_tile_cull = tile_cull != 0;
  drop_graphs(c);  // launch arguments are baked into the graphs
  return B2MD_OK;
}

int b2md_set_step_options(b2md_ctx* c, int fused_kick) {
  if (!c) return set_err(B2MD_INVALID_ARGUMENT, "set_step_options: null context");
  c->use_fused_kick = fused_kick != 0;
  drop_graphs(c);
  return B2MD_OK;
}

int b2md_set_sort_interval(b2md_ctx* c, int steps) {
  if (!c || steps < 0) return set_err(B2MD_INVALID_ARGUMENT, "set_sort_interval: bad argument");
  c->sort_interval = steps;
  return B2MD_OK;
}

int b2md_get_sort_interval(const b2md_ctx* c, int* steps, int* steps_since_sort) {
  if (!c) return set_err(B2MD_INVALID_ARGUMENT, "get_sort_interval: null context");
  if (steps) *steps = c->sort_interval;
  if (steps_since_sort) *steps_since_sort = c->steps_since_sort;
  return B2MD_OK;
}

int b2md_nlist_info(b2md_ctx* c, int replica, int64_t info[8]) {
  if (!c || !info || replica < 0 || replica >= c->R)
    return set_err(B2MD_INVALID_ARGUMENT, "nlist_info: bad argument");
  for (int k = 0; k < 8; ++k) info[k] = 0;
  if (!nl_path(c)) return B2MD_OK;
  int ctl[kNLCtl];
  CU(cudaMemcpyAsync(ctl, c->nl.ctl + size_t(replica) * kNLCtl, sizeof ctl, cudaMemcpyDeviceToHost,
                     c->stream));
  CU(cudaStreamSynchronize(c->stream));
  info[0] = 1;
  info[1] = ctl[kNLEntries];
  info[2] = ctl[kNLIncoming];
  info[3] = (ctl[kNLOverflow] != 0 || unsigned(ctl[kNLD2]) > c->nl.d2_stale) ? 1 : 0;
  info[4] = ctl[kNLEpoch] - 1;
  info[5] = c->steps_since_nl;
  info[6] = c->nl_interval;
  info[7] = int64_t(std::llround(c->nl_skin * 1e6));
  return B2MD_OK;
}

int b2md_pair_list(b2md_ctx* c, int replica, int32_t* pairs, int64_t capacity, int64_t* n_pairs) {
  NvtxRange nvtx_("b2md_pair_list");
  if (!c || !n_pairs) return set_err(B2MD_INVALID_ARGUMENT, "pair_list: null pointer");
  if (replica < 0 || replica >= c->R) return set_err(B2MD_INVALID_ARGUMENT, "pair_list: bad replica");
  CU(cudaSetDevice(c->device));
  const int n = c->t.n;
  TRY(ensure_mask(c));
  const uint32_t* mask = c->d_mask + size_t(replica) * c->g.n_pad * c->g.words;
  const int* perm = c->d_perm + size_t(replica) * n;
  int64_t* d_cnt = nullptr;
  CU(cudaMalloc(&d_cnt, sizeof(int64_t) * (n + 1)));
  k_pair_count<<<(n + 255) / 256, 256, 0, c->stream>>>(mask, perm, n, c->g.words, d_cnt);
  std::vector<int64_t> cnt(n + 1, 0);
  cudaError_t e = cudaMemcpyAsync(cnt.data(), d_cnt, sizeof(int64_t) * n, cudaMemcpyDeviceToHost, c->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
  if (e != cudaSuccess) {
    cudaFree(d_cnt);
    return set_err(B2MD_CUDA_ERROR, cudaGetErrorString(e));
  }
  // exclusive scan of the per-row counts
  int64_t total = 0;
  for (int i = 0; i < n; ++i) {
    const int64_t v = cnt[i];
    cnt[i] = total;
    total += v;
  }
  *n_pairs = total;
  if (pairs && total > 0) {
    if (capacity < total) {
      cudaFree(d_cnt);
      return set_err(B2MD_INVALID_ARGUMENT, "pair_list: capacity too small");
    }
    int32_t* d_pairs = nullptr;
    e = cudaMalloc(&d_pairs, sizeof(int32_t) * 2 * total);
    if (e == cudaSuccess) e = cudaMemcpyAsync(d_cnt, cnt.data(), sizeof(int64_t) * n, cudaMemcpyHostToDevice, c->stream);
    if (e == cudaSuccess) {
      k_pair_fill<<<(n + 255) / 256, 256, 0, c->stream>>>(mask, perm, n, c->g.words, d_cnt, d_pairs);
      e = cudaGetLastError();
    }
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(pairs, d_pairs, sizeof(int32_t) * 2 * total, cudaMemcpyDeviceToHost, c->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
    cudaFree(d_pairs);
    if (e != cudaSuccess) {
      cudaFree(d_cnt);
      return set_err(B2MD_CUDA_ERROR, cudaGetErrorString(e));
    }
    // each row i's partners j came in slot order: sort them (reference order)
    for (int i = 0; i < n; ++i) {
      const int64_t b = cnt[i], en = i + 1 < n ? cnt[i + 1] : total;
      std::vector<int32_t> js;
      js.reserve(size_t(en - b));
      for (int64_t q = b; q < en; ++q) js.push_back(pairs[2 * q + 1]);
      std::sort(js.begin(), js.end());
      for (int64_t q = b; q < en; ++q) pairs[2 * q + 1] = js[size_t(q - b)];
    }
  }
  cudaFree(d_cnt);
  return B2MD_OK;
}

int b2md_nccl_unique_id(char id[128]) {
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  ncclUniqueId u;
  TRY(nccl_load());
  NC(g_nccl.GetUniqueId(&u));
  std::memcpy(id, &u, 128);
  return B2MD_OK;
}

int b2md_attach_nccl(b2md_ctx* c, const char id[128], int rank, int world) {
  if (!c || !id || world < 1 || rank < 0 || rank >= world)
    return set_err(B2MD_INVALID_ARGUMENT, "attach_nccl: bad argument");
  CU(cudaSetDevice(c->device));
  if (world > 1) TRY(nccl_load());
  if (c->comm) {
    g_nccl.CommDestroy(c->comm);
    c->comm = nullptr;
  }
  if (world > 1) {
    ncclUniqueId u;
    std::memcpy(&u, id, 128);
    NC(g_nccl.CommInitRank(&c->comm, world, u, rank));
  }
  c->rank = rank;
  c->world = world;
  TRY(setup_shard(c));
  return B2MD_OK;
}

int b2md_set_shard(b2md_ctx* c, int rank, int world) {
  if (!c || world < 1 || rank < 0 || rank >= world)
    return set_err(B2MD_INVALID_ARGUMENT, "set_shard: bad argument");
  CU(cudaSetDevice(c->device));
  if (c->comm) {
    g_nccl.CommDestroy(c->comm);
    c->comm = nullptr;
  }
  c->rank = rank;
  c->world = world;
  TRY(setup_shard(c));
  return B2MD_OK;
}

void* b2md_stream(b2md_ctx* c) { return c ? reinterpret_cast<void*>(c->stream) : nullptr; }

int b2md_profile_enable(b2md_ctx* c, int enable) {
  if (!c) return set_err(B2MD_INVALID_ARGUMENT, "profile_enable: null context");
  TRY(prof_harvest(c));
  if (enable != c->profile_level || (enable != 0) != c->profile) drop_graphs(c);
  c->profile = enable != 0;
  if (enable) c->profile_level = enable;
  if (c->profile)
    for (int f = 0; f < F_COUNT; ++f) {
      c->prof_ms[f] = 0.0;
      c->prof_n[f] = 0;
    }
  return B2MD_OK;
}

int b2md_kernel_times(b2md_ctx* c, int max_rows, char (*names)[32], double* total_ms,
                      int64_t* launches, int* n_rows) {
  if (!c || !n_rows) return set_err(B2MD_INVALID_ARGUMENT, "kernel_times: null pointer");
  TRY(prof_harvest(c));
  int k = 0;
  for (int f = 0; f < F_COUNT && k < max_rows; ++f) {
    if (c->prof_n[f] == 0) continue;
    if (names) std::snprintf(names[k], 32, "%s", kFamilyName[f]);
    if (total_ms) total_ms[k] = c->prof_ms[f];
    if (launches) launches[k] = c->prof_n[f];
    ++k;
  }
  *n_rows = k;
  return B2MD_OK;
}

int b2md_set_graphs(b2md_ctx* c, int enable) {
  if (!c) return set_err(B2MD_INVALID_ARGUMENT, "set_graphs: null context");
  c->use_graphs = enable != 0;
  return B2MD_OK;
}

int b2md_measure_fp64_peak(int device, double* gflops) {
  if (!gflops) return set_err(B2MD_INVALID_ARGUMENT, "measure_fp64_peak: null pointer");
  CU(cudaSetDevice(device));
  int sms = 0;
  CU(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
  const int blocks = sms * 8, threads = 256, iters = 20000;
  double* out = nullptr;
  CU(cudaMalloc(&out, sizeof(double) * blocks * threads));
  cudaEvent_t e0, e1;
  CU(cudaEventCreate(&e0));
  CU(cudaEventCreate(&e1));
  k_dfma_peak<<<blocks, threads>>>(out, 200, 1.0000001, 1e-7);
  CU(cudaEventRecord(e0));
  for (int r = 0; r < 5; ++r) k_dfma_peak<<<blocks, threads>>>(out, iters, 1.0000001, 1e-7);
  CU(cudaEventRecord(e1));
  CU(cudaEventSynchronize(e1));
  float ms = 0.f;
  CU(cudaEventElapsedTime(&ms, e0, e1));
  *gflops = 5.0 * blocks * threads * double(iters) * 8 * 2 / (double(ms) * 1e6);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(out);
  return B2MD_OK;
}

}  // extern "C"
