// b200md samplers and state I/O on the device: the Green-Kubo heat flux,
// RDF histograms, the thermostat and kinetic energies, and the checkpoint
// state block (C ABI of include/b200md.h).
#include "ctx_internal.cuh"
#include "rdf.cuh"

using namespace b2md;

namespace b2md_host {

// heat_flux (src/greenkubo.cpp:182-266) over the current mask, site offsets
// and packed positions (valid after set_state / step / evaluate), then the
// cross-rank sum of the per-replica 3-vectors.
// single species, centred LJ only: the cluster walk (no partner search)
bool flux_cluster(const b2md_ctx* c) {
  return cluster_path(c) && c->t.ns == 1 && c->t.qq[0].empty();
}

int launch_heat_flux(b2md_ctx* c, const double* enthalpy) {
  FluxArgs a;
  a.f = force_args(c);
  for (int k = 0; k < kMaxSpecies; ++k) a.enthalpy[k] = k < c->t.ns ? enthalpy[k] : 0.0;
  a.out = c->d_flux;
  // the generic walk visits every row on every rank: rank 0 adds the
  // kinetic term; the cluster walk visits only this rank's rows (disjoint
  // over ranks), so each rank adds it for its own rows
  a.kinetic = (c->rank == 0 || flux_cluster(c)) ? 1 : 0;
  // positions after a raw upload / restore may lie outside [0, L)
  const bool w = fast_min_image(c) && c->state_in_box;
  if (flux_cluster(c)) {
    const ClusterArgs ca = cluster_args(c);
    dim3 pgrid(cpair_grid(c), c->R);
    if (w)
      PROF(c, F_HEAT_FLUX, (k_heat_flux_cpair<true><<<pgrid, kGWarps * 32, 0, c->stream>>>(a, ca)));
    else
      PROF(c, F_HEAT_FLUX, (k_heat_flux_cpair<false><<<pgrid, kGWarps * 32, 0, c->stream>>>(a, ca)));
    if (c->world > 1 && c->comm)
      NC(g_nccl.AllReduce(c->d_flux, c->d_flux, size_t(kNumSums) * c->R, ncclDouble, ncclSum,
                          c->comm, c->stream));
    return B2MD_OK;
  }
  const bool offs = c->t.any_offsets;
  const bool one = c->t.ns == 1;
  dim3 grid(c->force_grid, c->R);
  const int bs = c->force_warps * 32;
  const int m = c->t.method == B2MD_METHOD_EWALD ? 2 : (c->t.method == B2MD_METHOD_REACTION_FIELD ? 1 : 0);
#define FLUX_K(M, O, W)                                                                       \
  do {                                                                                        \
    if (one)                                                                                  \
      PROF(c, F_HEAT_FLUX, (k_heat_flux<M, O, W, true><<<grid, bs, 0, c->stream>>>(a)));      \
    else                                                                                      \
      PROF(c, F_HEAT_FLUX, (k_heat_flux<M, O, W, false><<<grid, bs, 0, c->stream>>>(a)));     \
  } while (0)
#define FLUX_CASE(M)                  \
  case M:                             \
    if (offs && w)                    \
      FLUX_K(M, true, true);          \
    else if (offs)                    \
      FLUX_K(M, true, false);         \
    else if (w)                       \
      FLUX_K(M, false, true);         \
    else                              \
      FLUX_K(M, false, false);        \
    break;
  switch (m) {
    FLUX_CASE(0)
    FLUX_CASE(1)
    FLUX_CASE(2)
  }
#undef FLUX_K
#undef FLUX_CASE
  if (c->world > 1 && c->comm)
    NC(g_nccl.AllReduce(c->d_flux, c->d_flux, size_t(kNumSums) * c->R, ncclDouble, ncclSum, c->comm,
                     c->stream));
  return B2MD_OK;
}

int download_flux(b2md_ctx* c, double* jq) {
  std::vector<double> h(size_t(kNumSums) * c->R);
  CU(cudaMemcpyAsync(h.data(), c->d_flux, sizeof(double) * h.size(), cudaMemcpyDeviceToHost,
                     c->stream));
  CU(cudaStreamSynchronize(c->stream));
  for (int r = 0; r < c->R; ++r)
    for (int k = 0; k < 3; ++k) jq[3 * r + k] = h[size_t(r) * kNumSums + k];
  return B2MD_OK;
}

int check_enthalpy(const b2md_ctx* c, const double* enthalpy, int n_enthalpy, const double* jq) {
  if (!jq || (n_enthalpy > 0 && !enthalpy))
    return set_err(B2MD_INVALID_ARGUMENT, "heat_flux: null pointer");
  // greenkubo.cpp:184-185
  if (n_enthalpy != c->t.ns)
    return set_err(B2MD_CONFIG_ERROR,
                   "heat flux: partial molar enthalpy required for every component");
  return B2MD_OK;
}

}  // namespace b2md_host

using namespace b2md_host;

int b2md_heat_flux(b2md_ctx* c, const double* enthalpy, int n_enthalpy, double* jq) {
  NvtxRange nvtx_("b2md_heat_flux");
  if (!c) return set_err(B2MD_INVALID_ARGUMENT, "heat_flux: null context");
  TRY(check_enthalpy(c, enthalpy, n_enthalpy, jq));
  if (!c->state_valid)
    return set_err(B2MD_CONFIG_ERROR, "heat_flux: set_state must precede heat_flux");
  CU(cudaSetDevice(c->device));
  if (!flux_cluster(c)) TRY(ensure_mask(c));  // (the cluster walk's arcs are current)
  TRY(launch_heat_flux(c, enthalpy));
  return download_flux(c, jq);
}

int b2md_heat_flux_state(b2md_ctx* c, const double* pos, const double* orient, const double* vel,
                         const double* ang_vel, const double* enthalpy, int n_enthalpy,
                         double* jq) {
  NvtxRange nvtx_("b2md_heat_flux_state");
  if (!c) return set_err(B2MD_INVALID_ARGUMENT, "heat_flux: null context");
  if (!pos || !orient || !vel || !ang_vel)
    return set_err(B2MD_INVALID_ARGUMENT, "heat_flux: null pointer");
  TRY(check_enthalpy(c, enthalpy, n_enthalpy, jq));
  CU(cudaSetDevice(c->device));
  TRY(upload_aos(c, 0, pos, 3, c->st.px, c->st.py, c->st.pz, nullptr));
  TRY(upload_aos(c, 1, orient, 4, c->st.qw, c->st.qx, c->st.qy, c->st.qz));
  TRY(upload_aos(c, 2, vel, 3, c->st.vx, c->st.vy, c->st.vz, nullptr));
  TRY(upload_aos(c, 3, ang_vel, 3, c->st.wx, c->st.wy, c->st.wz, nullptr));
  set_wrapped(c, false);  // the reference takes the positions as given
  c->state_in_box = false;
  if (c->sort_interval > 0)
    TRY(resort_and_stage(c));
  else {
    TRY(launch_offsets(c));
    const int nt = n_total(c);
    k_stage_positions<<<(nt + 255) / 256, 256, 0, c->stream>>>(
        c->st.px, c->st.py, c->st.pz, nt, c->t.n, c->d_slot_of, c->t.box,
        4294967296.0 / c->t.box, c->d_fixpos, c->st.pos4);
    CU(cudaGetLastError());
    TRY(launch_cluster_arcs(c));
  }
  if (!flux_cluster(c)) TRY(launch_search(c));
  TRY(launch_heat_flux(c, enthalpy));
  TRY(download_flux(c, jq));
  c->state_valid = false;  // forces not evaluated: not an engine state
  return B2MD_OK;
}

// ------------------------------------------------------------ thermostat
// model.cpp:321-330
int dof_trans(const b2md_ctx* c) { return 3 * c->t.n - 3; }
int dof_rot(const b2md_ctx* c) {
  int dof = 0;
  for (int m = 0; m < c->t.n; ++m) dof += c->t.species[c->t.species_of[m]].rotational_dof;
  return dof;
}

int launch_kinetic(b2md_ctx* c) {
  k_kinetic<<<c->R, kKeThreads, 0, c->stream>>>(c->sys, c->st, c->d_ke);
  CU(cudaGetLastError());
  return B2MD_OK;
}

// Engine::apply_thermostat (engine.cpp:145-160) on every replica, on the stream
int launch_thermostat(b2md_ctx* c) {
  TRY(launch_kinetic(c));
  ThermoArgs a;
  a.s = c->sys;
  a.st = c->st;
  a.ke = c->d_ke;
  a.err = c->d_thermo_err;
  a.temperature = c->t.temperature;
  a.dof_t = dof_trans(c);
  a.dof_r = dof_rot(c);
  const int nt = n_total(c);
  k_thermostat<<<(nt + 255) / 256, 256, 0, c->stream>>>(a);
  CU(cudaGetLastError());
  return B2MD_OK;
}

int check_thermostat(b2md_ctx* c) {
  std::vector<int> err(c->R, 0);
  CU(cudaMemcpyAsync(err.data(), c->d_thermo_err, sizeof(int) * c->R, cudaMemcpyDeviceToHost,
                     c->stream));
  CU(cudaStreamSynchronize(c->stream));
  for (int r = 0; r < c->R; ++r)
    if (err[r]) {
      CU(cudaMemset(c->d_thermo_err, 0, sizeof(int) * c->R));
      return set_err(B2MD_NUMERICAL_ERROR, err[r] == 1
                                               ? "thermostat: zero translational kinetic energy"
                                               : "thermostat: zero rotational kinetic energy");
    }
  return B2MD_OK;
}

int b2md_kinetic_energy(b2md_ctx* c, double* ke_trans, double* ke_rot) {
  NvtxRange nvtx_("b2md_kinetic_energy");
  if (!c) return set_err(B2MD_INVALID_ARGUMENT, "kinetic_energy: null context");
  CU(cudaSetDevice(c->device));
  TRY(launch_kinetic(c));
  std::vector<double2> ke(c->R);
  CU(cudaMemcpyAsync(ke.data(), c->d_ke, sizeof(double2) * c->R, cudaMemcpyDeviceToHost, c->stream));
  CU(cudaStreamSynchronize(c->stream));
  for (int r = 0; r < c->R; ++r) {
    if (ke_trans) ke_trans[r] = ke[r].x;
    if (ke_rot) ke_rot[r] = ke[r].y;
  }
  return B2MD_OK;
}

int b2md_apply_thermostat(b2md_ctx* c) {
  NvtxRange nvtx_("b2md_apply_thermostat");
  if (!c) return set_err(B2MD_INVALID_ARGUMENT, "apply_thermostat: null context");
  if (!c->state_valid) return set_err(B2MD_CONFIG_ERROR, "engine: set_state must precede step");
  CU(cudaSetDevice(c->device));
  TRY(launch_thermostat(c));
  return check_thermostat(c);
}

// Engine::run's thermostatted loop (engine.cpp:273-296): steps numbered
// done+1 .. done+nsteps of the current phase, the rescale after every step
// whose number is a multiple of `interval` (<= 0: none).
int b2md_step_thermostat(b2md_ctx* c, int64_t nsteps, int interval, int64_t done) {
  NvtxRange nvtx_("b2md_step_thermostat");
  if (!c) return set_err(B2MD_INVALID_ARGUMENT, "step: null context");
  if (!c->engine) return set_err(B2MD_CONFIG_ERROR, "engine: time step must be positive");
  if (!c->state_valid) return set_err(B2MD_CONFIG_ERROR, "engine: set_state must precede step");
  if (nsteps <= 0) return B2MD_OK;
  CU(cudaSetDevice(c->device));
  if (interval <= 0) {
    TRY(run_steps(c, nsteps));
    return check_error_flag(c);
  }
  for (int64_t k = 0; k < nsteps;) {
    const int64_t step_no = done + k;                      // steps already taken
    const int64_t to_next = interval - step_no % interval;  // steps to the next rescale
    const int64_t chunk = std::min<int64_t>(to_next, nsteps - k);
    TRY(run_steps(c, chunk));
    k += chunk;
    if ((done + k) % interval == 0) TRY(launch_thermostat(c));
  }
  TRY(check_error_flag(c));
  return check_thermostat(c);
}

// ------------------------------------------------------ checkpoint state
// The device-resident part of Engine::checkpoint_bytes (engine.cpp:432-441):
// u32 n, f64 box_length, then 13 f64 per molecule, little-endian (the
// ByteWriter of checkpoint.hpp:15-38 writes raw host bytes; x86-64 and the
// GPU hosts here are little-endian).
size_t b2md_state_block_size(const b2md_ctx* c) { return c ? 12 + size_t(104) * c->t.n : 0; }

int b2md_save_state_block(b2md_ctx* c, int replica, uint8_t* buf, size_t cap) {
  NvtxRange nvtx_("b2md_save_state_block");
  if (!c || !buf) return set_err(B2MD_INVALID_ARGUMENT, "save_state_block: null pointer");
  if (replica < 0 || replica >= c->R)
    return set_err(B2MD_INVALID_ARGUMENT, "save_state_block: bad replica");
  const int n = c->t.n;
  if (cap < b2md_state_block_size(c))
    return set_err(B2MD_INVALID_ARGUMENT, "save_state_block: buffer too small");
  CU(cudaSetDevice(c->device));
  const uint32_t nn = uint32_t(n);
  const double box = c->t.box;
  std::memcpy(buf, &nn, 4);
  std::memcpy(buf + 4, &box, 8);
  k_pack_state<<<(n + 255) / 256, 256, 0, c->stream>>>(c->st, n, replica, c->d_stage);
  CU(cudaGetLastError());
  CU(cudaMemcpyAsync(buf + 12, c->d_stage, sizeof(double) * 13 * n, cudaMemcpyDeviceToHost,
                     c->stream));
  CU(cudaStreamSynchronize(c->stream));
  return B2MD_OK;
}

int b2md_restore_state_block(b2md_ctx* c, int replica, const uint8_t* buf, size_t len) {
  NvtxRange nvtx_("b2md_restore_state_block");
  if (!c || !buf) return set_err(B2MD_INVALID_ARGUMENT, "restore_state_block: null pointer");
  if (replica < 0 || replica >= c->R)
    return set_err(B2MD_INVALID_ARGUMENT, "restore_state_block: bad replica");
  // ByteReader::need (checkpoint.hpp:87-91) and engine.cpp:479-480
  auto truncated = [&](size_t need, size_t at) {
    return set_err(B2MD_IO_ERROR, "checkpoint: truncated or corrupted data (need " +
                                      std::to_string(need) + " bytes at offset " +
                                      std::to_string(at) + ")");
  };
  if (len < 4) return truncated(4, 0);
  uint32_t nn = 0;
  std::memcpy(&nn, buf, 4);
  if (int(nn) != c->t.n) return set_err(B2MD_IO_ERROR, "checkpoint: molecule count mismatch");
  if (len < 12) return truncated(8, 4);
  double box = 0.0;
  std::memcpy(&box, buf + 4, 8);
  if (box != c->t.box)  // the context's tables are built for the composition's box
    return set_err(B2MD_IO_ERROR, "checkpoint: box length does not match the composition");
  const int n = c->t.n;
  for (int i = 0; i < n; ++i)
    if (len < 12 + size_t(104) * (i + 1)) {
      const size_t at = 12 + size_t(104) * i;
      return truncated(8, at + ((len - at) / 8) * 8);
    }
  CU(cudaSetDevice(c->device));
  CU(cudaMemcpyAsync(c->d_stage, buf + 12, sizeof(double) * 13 * n, cudaMemcpyHostToDevice,
                     c->stream));
  k_unpack_state<<<(n + 255) / 256, 256, 0, c->stream>>>(c->st, n, replica, c->d_stage);
  CU(cudaGetLastError());
  // restore_dynamic ends with compute_forces() (engine.cpp:540): no wrap
  set_wrapped(c, false);
  const int big = INT_MAX;
  CU(cudaMemcpyAsync(c->d_error, &big, sizeof(int), cudaMemcpyHostToDevice, c->stream));
  if (c->sort_interval > 0) TRY(resort(c));
  TRY(enqueue_forces(c, true));
  CU(cudaStreamSynchronize(c->stream));
  set_wrapped(c, true);  // steps wrap before every later evaluation
  c->state_in_box = false;  // restored as given (no wrap) until a step wraps
  c->state_valid = true;
  return B2MD_OK;
}

// ---------------------------------------------------------------- RDF
// tmd::RdfHistogram (include/tmd/structure.hpp:29-67) over a context: one
// histogram per replica, accumulated on the device (rdf.cuh).
struct b2md_rdf {
  b2md_ctx* ctx = nullptr;
  double bin_width = 0.0, r_max = 0.0;
  int bins = 0, n_types = 0, n_pairs = 0, S = 0;
  std::vector<int> type_species, type_site;
  std::vector<int64_t> snapshots;  // per replica
  int* d_site_mol = nullptr;
  int* d_site_k = nullptr;
  int* d_site_type = nullptr;
  double4* d_sites = nullptr;
  uint4* d_fix = nullptr;
  unsigned long long* d_counts = nullptr;
};

namespace {

void rdf_free(b2md_rdf* h) {
  if (!h) return;
  void* ptrs[] = {h->d_site_mol, h->d_site_k, h->d_site_type, h->d_sites, h->d_fix, h->d_counts};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  delete h;
}

// structure.cpp:38-76 on the context's device positions / orientations
int rdf_launch(b2md_rdf* h) {
  b2md_ctx* c = h->ctx;
  for (auto& s : h->snapshots) ++s;
  if (h->S == 0 || h->n_pairs == 0 || h->bins == 0) return B2MD_OK;
  RdfArgs a;
  a.s = c->sys;
  a.px = c->st.px;
  a.py = c->st.py;
  a.pz = c->st.pz;
  a.qw = c->st.qw;
  a.qx = c->st.qx;
  a.qy = c->st.qy;
  a.qz = c->st.qz;
  a.site_mol = h->d_site_mol;
  a.site_k = h->d_site_k;
  a.site_type = h->d_site_type;
  a.S = h->S;
  a.n_types = h->n_types;
  a.bins = h->bins;
  a.n_pairs = h->n_pairs;
  a.rmax2 = h->r_max * h->r_max;  // structure.cpp:41
  a.bin_width = h->bin_width;
  a.sites = h->d_sites;
  a.fix = h->d_fix;
  a.counts = h->d_counts;
  a.L = c->t.box;
  {
    // fp32 fast-path margins (rdf.cuh, k_rdf_pairs): relative 2e-6 on d2
    // (bound 5.4e-7: nine fp32 roundings) plus the fixed-point quantisation
    // (<= 1 unit of L/2^32 per axis: |dd| <= sqrt(3) units, 4 taken); the
    // thresholds' own fp32 rounding is covered by the extra 1e-6
    const double L = c->t.box, unit = L / 4294967296.0;
    const double r2 = a.rmax2, rm = h->r_max, dd = 4.0 * unit;
    a.scale = float(unit);
    a.rmax2_lo = float((r2 * (1.0 - 2e-6) - 2.0 * rm * dd) * (1.0 - 1e-6));
    a.rmax2_hi = float((r2 * (1.0 + 2e-6) + 2.0 * rm * dd + dd * dd) * (1.0 + 1e-6));
    a.inv_bw_f = float(1.0 / h->bin_width);
    a.bin_abs = float(2.0 * dd / h->bin_width + 1e-6);
  }
  const int total = h->S * c->R;
  k_rdf_stage<<<(total + 255) / 256, 256, 0, c->stream>>>(a);
  CU(cudaGetLastError());
  a.inv_bw = 1.0 / h->bin_width;
  // tile side: the largest of 256 / 128 / 64 that still gives ~2 CTAs per SM
  const int nc = h->n_pairs * h->bins;
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device);
  auto ctas = [&](int t) {
    const long nb = (h->S + t - 1) / t;
    return nb * (nb + 1) / 2 * c->R;
  };
  const int T = ctas(256) >= 2 * sms ? 256 : (ctas(128) >= 2 * sms ? 128 : 64);
  const int nb = (h->S + T - 1) / T;
  const dim3 grid(nb, nb, c->R);
  // a per-CTA shared histogram pays when the tile's pairs outnumber its counters
  const bool shared = nc <= kRdfSharedCounters && T * T >= 4 * nc;
  const size_t sm = shared ? sizeof(unsigned) * nc : 0;
#define RDF_LAUNCH(TT)                                                                   \
  if (shared)                                                                            \
    PROF(c, F_RDF, (k_rdf_pairs<TT, true><<<grid, TT, sm, c->stream>>>(a)));             \
  else                                                                                   \
    PROF(c, F_RDF, (k_rdf_pairs<TT, false><<<grid, TT, 0, c->stream>>>(a)));
  if (T == 256) {
    RDF_LAUNCH(256)
  } else if (T == 128) {
    RDF_LAUNCH(128)
  } else {
    RDF_LAUNCH(64)
  }
#undef RDF_LAUNCH
  return B2MD_OK;
}

}  // namespace

int b2md_rdf_create(b2md_ctx* c, double bin_width, double r_max, b2md_rdf** out) {
  if (!c || !out) return set_err(B2MD_INVALID_ARGUMENT, "rdf: null pointer");
  // structure.cpp:12-14
  if (bin_width <= 0.0) return set_err(B2MD_CONFIG_ERROR, "rdf: bin width must be positive");
  if (r_max > 0.5 * c->t.box + 1e-12)
    return set_err(B2MD_CONFIG_ERROR, "rdf: r_max exceeds half the box length");
  CU(cudaSetDevice(c->device));
  auto* h = new b2md_rdf;
  h->ctx = c;
  h->bin_width = bin_width;
  h->r_max = r_max;
  h->bins = static_cast<int>(std::ceil(r_max / bin_width));
  // structure.cpp:17-32: types in (species, site) order, charge sites skipped
  std::vector<int> type_of(c->t.ns * B2MD_MAX_SITES, -1);
  for (int s = 0; s < c->t.ns; ++s) {
    const b2md_species& sp = c->t.species[s];
    for (int k = 0; k < sp.n_sites; ++k) {
      if (sp.sites[k].kind == B2MD_SITE_CHARGE) continue;
      type_of[s * B2MD_MAX_SITES + k] = h->n_types++;
      h->type_species.push_back(s);
      h->type_site.push_back(k);
    }
  }
  h->n_pairs = h->n_types * (h->n_types + 1) / 2;
  std::vector<int> site_mol, site_k, site_type;
  for (int m = 0; m < c->t.n; ++m) {
    const int s = c->t.species_of[m];
    for (int k = 0; k < c->t.species[s].n_sites; ++k) {
      const int t = type_of[s * B2MD_MAX_SITES + k];
      if (t < 0) continue;
      site_mol.push_back(m);
      site_k.push_back(k);
      site_type.push_back(t);
    }
  }
  h->S = static_cast<int>(site_mol.size());
  h->snapshots.assign(c->R, 0);
  int rc = B2MD_OK;
  const size_t nc = size_t(h->n_pairs) * h->bins * c->R;
  if (h->S > 0) {
    rc = dalloc(&h->d_site_mol, h->S);
    if (!rc) rc = dalloc(&h->d_site_k, h->S);
    if (!rc) rc = dalloc(&h->d_site_type, h->S);
    if (!rc) rc = dalloc(&h->d_sites, size_t(h->S) * c->R);
    if (!rc) rc = dalloc(&h->d_fix, size_t(h->S) * c->R);
    if (!rc) {
      cudaMemcpy(h->d_site_mol, site_mol.data(), sizeof(int) * h->S, cudaMemcpyHostToDevice);
      cudaMemcpy(h->d_site_k, site_k.data(), sizeof(int) * h->S, cudaMemcpyHostToDevice);
      cudaMemcpy(h->d_site_type, site_type.data(), sizeof(int) * h->S, cudaMemcpyHostToDevice);
    }
  }
  if (!rc && nc > 0) {
    rc = dalloc(&h->d_counts, nc);
    if (!rc && cudaMemset(h->d_counts, 0, sizeof(unsigned long long) * nc) != cudaSuccess)
      rc = set_err(B2MD_CUDA_ERROR, "rdf: memset failed");
  }
  if (rc) {
    rdf_free(h);
    return rc;
  }
  *out = h;
  return B2MD_OK;
}

void b2md_rdf_destroy(b2md_rdf* h) {
  if (h && h->ctx) cudaSetDevice(h->ctx->device);
  rdf_free(h);
}

int b2md_rdf_shape(const b2md_rdf* h, int* n_types, int* bins, int* n_pairs) {
  if (!h) return set_err(B2MD_INVALID_ARGUMENT, "rdf: null handle");
  if (n_types) *n_types = h->n_types;
  if (bins) *bins = h->bins;
  if (n_pairs) *n_pairs = h->n_pairs;
  return B2MD_OK;
}

int b2md_rdf_types(const b2md_rdf* h, int* species, int* site) {
  if (!h) return set_err(B2MD_INVALID_ARGUMENT, "rdf: null handle");
  for (int t = 0; t < h->n_types; ++t) {
    if (species) species[t] = h->type_species[t];
    if (site) site[t] = h->type_site[t];
  }
  return B2MD_OK;
}

int b2md_rdf_accumulate(b2md_rdf* h) {
  NvtxRange nvtx_("b2md_rdf_accumulate");
  if (!h) return set_err(B2MD_INVALID_ARGUMENT, "rdf: null handle");
  CU(cudaSetDevice(h->ctx->device));
  return rdf_launch(h);
}

int b2md_rdf_accumulate_state(b2md_rdf* h, const double* pos, const double* orient) {
  NvtxRange nvtx_("b2md_rdf_accumulate_state");
  if (!h || !pos || !orient) return set_err(B2MD_INVALID_ARGUMENT, "rdf: null pointer");
  b2md_ctx* c = h->ctx;
  CU(cudaSetDevice(c->device));
  TRY(upload_aos(c, 0, pos, 3, c->st.px, c->st.py, c->st.pz, nullptr));
  TRY(upload_aos(c, 1, orient, 4, c->st.qw, c->st.qx, c->st.qy, c->st.qz));
  c->state_valid = false;  // positions replaced: not an engine state any more
  TRY(rdf_launch(h));
  CU(cudaStreamSynchronize(c->stream));
  return B2MD_OK;
}

int b2md_rdf_counts(const b2md_rdf* h, int replica, uint64_t* counts, int64_t* snapshots) {
  if (!h) return set_err(B2MD_INVALID_ARGUMENT, "rdf: null handle");
  if (replica < 0 || replica >= h->ctx->R) return set_err(B2MD_INVALID_ARGUMENT, "rdf: bad replica");
  b2md_ctx* c = h->ctx;
  CU(cudaSetDevice(c->device));
  const size_t nc = size_t(h->n_pairs) * h->bins;
  if (counts && nc > 0) {
    CU(cudaMemcpyAsync(counts, h->d_counts + replica * nc, sizeof(uint64_t) * nc,
                       cudaMemcpyDeviceToHost, c->stream));
    CU(cudaStreamSynchronize(c->stream));
  }
  if (snapshots) *snapshots = h->snapshots[replica];
  return B2MD_OK;
}

int b2md_rdf_set_counts(b2md_rdf* h, int replica, const uint64_t* counts, int64_t snapshots) {
  if (!h) return set_err(B2MD_INVALID_ARGUMENT, "rdf: null handle");
  if (replica < 0 || replica >= h->ctx->R) return set_err(B2MD_INVALID_ARGUMENT, "rdf: bad replica");
  b2md_ctx* c = h->ctx;
  CU(cudaSetDevice(c->device));
  const size_t nc = size_t(h->n_pairs) * h->bins;
  if (nc > 0) {
    if (counts)
      CU(cudaMemcpyAsync(h->d_counts + replica * nc, counts, sizeof(uint64_t) * nc,
                         cudaMemcpyHostToDevice, c->stream));
    else
      CU(cudaMemsetAsync(h->d_counts + replica * nc, 0, sizeof(uint64_t) * nc, c->stream));
    CU(cudaStreamSynchronize(c->stream));
  }
  h->snapshots[replica] = snapshots;
  return B2MD_OK;
}

