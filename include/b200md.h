/*
 * b200md.h — C ABI of the B200-native force/energy/partner-search/step path.
 *
 * This is the drop-in boundary for the hot path of the reference `tmd` library
 * (ms2 2.0 restatement, /root/reference/proj).  Every entry point below replaces
 * one reference interface; the reference declaration it stands in for is cited
 * as include/tmd/<file>:<line> or src/<file>:<line>.
 *
 * Conventions
 *  - Plain C: POD structs, raw pointers and sizes, no torch / CUDA types.
 *  - Every call returns an `int` status (B2MD_OK == 0).  On failure the
 *    message is available from b2md_last_error() (thread-local).  The status
 *    codes mirror the reference exception hierarchy (include/tmd/error.hpp:8-30):
 *    ModelError, ConfigError, IoError, NumericalError.  A C++ shim rethrows them
 *    (see INTEGRATION.md).
 *  - Host arrays use the reference's AoS layouts: Vec3 = 3 doubles (x,y,z)
 *    (include/tmd/geom.hpp:9-11), Quat = 4 doubles (w,x,y,z)
 *    (include/tmd/geom.hpp:37-38).  On the device the state is SoA.
 *  - Molecules are ordered by species (include/tmd/model.hpp:66-68).
 *  - There is no CPU fallback: a context needs a CUDA device; creating one
 *    without a device fails with B2MD_CUDA_ERROR.  Pure host helpers
 *    (species building, tuning, shard plans) work without a GPU.
 */
#ifndef B200MD_H
#define B200MD_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define B2MD_ABI_VERSION 1
#define B2MD_MAX_SITES 16

/* status codes (include/tmd/error.hpp:8-30) */
enum {
  B2MD_OK = 0,
  B2MD_MODEL_ERROR = 1,      /* tmd::ModelError */
  B2MD_CONFIG_ERROR = 2,     /* tmd::ConfigError */
  B2MD_IO_ERROR = 3,         /* tmd::IoError */
  B2MD_NUMERICAL_ERROR = 4,  /* tmd::NumericalError */
  B2MD_CUDA_ERROR = 5,       /* device / driver failure (no reference analogue) */
  B2MD_INVALID_ARGUMENT = 6  /* bad pointer / size at the C boundary */
};

/* tmd::SiteKind (include/tmd/model.hpp:16) */
enum { B2MD_SITE_LJ = 0, B2MD_SITE_CHARGE = 1, B2MD_SITE_DUMMY = 2 };

/* tmd::ElectrostaticsMethod (include/tmd/model.hpp:52) */
enum { B2MD_METHOD_NONE = 0, B2MD_METHOD_REACTION_FIELD = 1, B2MD_METHOD_EWALD = 2 };

/* tmd::Site (include/tmd/model.hpp:18-25) */
typedef struct {
  int32_t kind;
  int32_t pad_;
  double body_pos[3];
  double sigma;
  double epsilon;
  double q;
  double mass;
} b2md_site;

/* tmd::MoleculeSpecies after build_species (include/tmd/model.hpp:29-40) */
typedef struct {
  int32_t n_sites;
  int32_t rotational_dof;
  b2md_site sites[B2MD_MAX_SITES];
  double total_mass;
  double inertia_principal[3];
  double net_charge;
  double max_extent;
} b2md_species;

/* tmd::SystemComposition (include/tmd/model.hpp:54-72) */
typedef struct {
  int32_t n_species;
  int32_t pad_;
  const b2md_species* species; /* n_species entries, already built */
  const int32_t* counts;       /* n_species entries */
  double box_length;
  double temperature;
} b2md_composition;

/* tmd::ForceFieldOptions (include/tmd/parallel.hpp:45-52) + tmd::EwaldParams
 * (include/tmd/ewald.hpp:15-18).  `workers` is accepted for interface parity;
 * the reference's ewald+workers!=1 rejection (src/parallel.cpp:65-66) is kept. */
typedef struct {
  double cutoff;
  int32_t method;
  int32_t has_ewald;
  double eps_rf;         /* +inf = conducting boundary */
  double ewald_alpha;
  int32_t ewald_kmax;
  int32_t workers;
  int32_t volume_derivatives; /* 1 = accumulate s1/s2 (forced 0 for ewald) */
  int32_t pad_;
} b2md_ff_options;

/* tmd::EnergyBreakdown (include/tmd/energy.hpp:9-25) */
typedef struct {
  double lj;
  double elec_real;
  double elec_recip;
  double elec_self;
  double rf;
  double lrc;
  double du_dv_explicit;
  double du_dv_lrc;
  double d2u_dv2_explicit;
  double d2u_dv2_lrc;
} b2md_energy;

/* per-evaluation scalar outputs beyond EnergyBreakdown: the molecular virial
 * (include/tmd/model.hpp:86) and the raw volume-derivative sums s1, s2
 * (include/tmd/potentials.hpp:54-58). */
typedef struct {
  double virial;
  double s1;
  double s2;
  int64_t com_pairs;     /* molecule pairs passing the COM partner search */
} b2md_eval_stats;

typedef struct b2md_ctx b2md_ctx;

/* ---------------------------------------------------------------- host-only */

const char* b2md_last_error(void);
int b2md_abi_version(void);

/* tmd::build_species (src/model.cpp:68-129): re-centre on the COM, rotate into
 * the principal frame (Jacobi, src/model.cpp:12-60), zero tiny moments. */
int b2md_build_species(const b2md_site* sites, int n_sites, b2md_species* out);

/* tmd::ewald_tune (src/ewald.cpp:8-28) */
int b2md_ewald_tune(double delta, double cutoff, double box_length, double* alpha, int* kmax);

/* number of Ewald k-vectors of the reference's half-space rule
 * (src/ewald.cpp:77-104) */
int b2md_ewald_kvector_count(int kmax, int* count);

/* Row-block shard plan for `world` ranks: the i<j tile triangle (32-molecule
 * tiles) is cut into contiguous tile rows with balanced candidate-pair counts,
 * the GPU analogue of the reference's static split of the flat pair index
 * (src/parallel.cpp:84-91).  Outputs the tile-row range [row_begin,row_end)
 * and the k-vector range [k_begin,k_end) owned by `rank`. */
int b2md_shard_plan(int n_molecules, int n_kvectors, int world, int rank, int* row_begin,
                    int* row_end, int* k_begin, int* k_end, int64_t* candidate_pairs);

/* ------------------------------------------------------------- device paths */

/* tmd::ForceField::ForceField (src/parallel.cpp:55-72).  Validates exactly as
 * the reference (PairTable ctor src/potentials.cpp:35-51, comp.validate
 * src/model.cpp:244-268, Ewald ctor src/ewald.cpp:30-35).  `n_replicas`
 * independent systems of the same composition are held and stepped together
 * (1 for a plain ForceField).  `dt` > 0 makes the context an Engine
 * (src/engine.cpp:63-66); dt <= 0 gives a force-field-only context. */
int b2md_create(int device, const b2md_composition* comp, const b2md_ff_options* opts, double dt,
                int n_replicas, b2md_ctx** out);
void b2md_destroy(b2md_ctx* ctx);

/* non-empty when Ewald parameters look too coarse (src/ewald.cpp:41-44) */
const char* b2md_warning(const b2md_ctx* ctx);

/* tmd::ForceField::evaluate(SystemState&) (src/parallel.cpp:79-122) with host
 * buffers: positions (n*3, NOT wrapped — exactly like the reference) and
 * orientations (n*4) in, forces/torques (n*3), energy and stats out.  For
 * n_replicas > 1 all arrays are replica-major and energy/stats hold one entry
 * per replica.  Any output pointer may be NULL. */
int b2md_evaluate(b2md_ctx* ctx, const double* pos, const double* orient, double* force,
                  double* torque, b2md_energy* energy, b2md_eval_stats* stats);

/* tmd::Engine::set_state (src/engine.cpp:91-98): upload, wrap, compute forces. */
int b2md_set_state(b2md_ctx* ctx, const double* pos, const double* orient, const double* vel,
                   const double* ang_vel);

/* tmd::Engine::step (src/engine.cpp:102-143), `nsteps` times, device
 * resident.  Returns B2MD_NUMERICAL_ERROR like check_finite
 * (src/model.cpp:288-302); the state then holds the end of the failing step. */
int b2md_step(b2md_ctx* ctx, int64_t nsteps);

/* Enqueue `nsteps` steps without waiting (device-resident step loop);
 * b2md_sync waits for them and reports a NumericalError like b2md_step, and
 * so does the next b2md_get_state (its download carries the error flag, so
 * upload -> step_async -> get_state costs one host round trip). */
int b2md_step_async(b2md_ctx* ctx, int64_t nsteps);
int b2md_sync(b2md_ctx* ctx);

/* Raw upload of a complete dynamic state including the cached forces and
 * torques of that state — no wrap, no force evaluation (the data part of
 * tmd::Engine::restore_dynamic, src/engine.cpp:520-540).  NULL keeps the
 * device copy of that array.  The call is asynchronous on the context's
 * stream: pinned (device-accessible) host buffers are read by the device
 * AFTER it returns, so they must stay valid and unmodified until the next
 * synchronising call on the context (b2md_sync, b2md_get_state, b2md_step).
 * Pageable buffers are staged before it returns. */
int b2md_upload_state(b2md_ctx* ctx, const double* pos, const double* orient, const double* vel,
                      const double* ang_vel, const double* force, const double* torque);

/* tmd::Engine::state() (include/tmd/engine.hpp:60): download.  NULL skips. */
int b2md_get_state(b2md_ctx* ctx, double* pos, double* orient, double* vel, double* ang_vel,
                   double* force, double* torque, b2md_energy* energy, b2md_eval_stats* stats);

/* COM partner search of the current device state (src/potentials.cpp:156-158
 * single-site, src/potentials.cpp:209-213 multi-site): the i<j molecule pairs
 * passing the test, as (i,j) int32 pairs sorted by i then j.  With
 * pairs == NULL only the count is returned.  `replica` selects the system. */
int b2md_pair_list(b2md_ctx* ctx, int replica, int32_t* pairs, int64_t capacity,
                   int64_t* n_pairs);

/* Partner-search strategy (results are identical; for tests and
 * measurement).  fix_prefilter: the certified fixed-point prefilter of the
 * single-species path (else the exact fp64 test on every candidate);
 * tile_cull: skip 32x32 tiles whose molecule blocks' bounding arcs are
 * further apart than the COM radius (fixed-point path only).  Both default 1. */
int b2md_set_search_options(b2md_ctx* ctx, int fix_prefilter, int tile_cull);

/* Spatial ordering: internally molecules occupy slots in column order of
 * their wrapped positions (thin x-lines of ~32 molecules, for the search's
 * tile cull) (re-sorted by every set_state / evaluate and every
 * `steps` steps; 0 keeps the input order).  Only summation order changes;
 * every output is indexed as the input and pair lists keep the reference's
 * (i, j) order.  Default: 100 for a single species with COM radius < 0.3 L
 * (where the tile cull can use it), else 0. */
int b2md_set_sort_interval(b2md_ctx* ctx, int steps);
/* The current interval and the steps taken since the last re-sort (a step
 * re-sorts when steps_since_sort >= steps > 0). */
int b2md_get_sort_interval(const b2md_ctx* ctx, int* steps, int* steps_since_sort);

/* The once-per-pair cluster-pair list of the single-site cluster path
 * (the default walk of single-site systems with rc < 0.3 L;
 * no reference counterpart: diagnostics for tests and measurement).  info[0] = 1 when the list path is active (else all 0),
 * info[1] = entries (owned cluster pairs) of `replica`, info[2] = incoming
 * record slots, info[3] = 1 when the list is stale (a molecule moved more than
 * skin / 2 since the build: the exact per-step walk runs until the next
 * build), info[4] = evaluations since the context was created, info[5] = steps
 * since the last build, info[6] = scheduled build interval, info[7] = the
 * skin in units of 1e-6 length.  Synchronises the context's stream. */
int b2md_nlist_info(b2md_ctx* ctx, int replica, int64_t info[8]);

/* Step structure (same results bit for bit; for tests and measurement):
 * fused_kick = 1 runs the end-of-step half kick (engine.cpp:131-142) in the
 * force kernel's row epilogue whenever a molecule's force is final there (no
 * Ewald reciprocal term, no multi-GPU all-reduce).  Default: 1 below 4096
 * molecules in total (one launch less per step), 0 above (the epilogue kick
 * lengthens warps that own several rows). */
int b2md_set_step_options(b2md_ctx* ctx, int fused_kick);

/* Green-Kubo heat flux J_q (tmd::heat_flux, include/tmd/greenkubo.hpp:93,
 * src/greenkubo.cpp:182-266) of the context's current device state: the
 * state set_state / step left (Engine::run samples it every n_ext steps,
 * src/engine.cpp:235-238).  `enthalpy` holds one partial molar enthalpy per
 * species; n_enthalpy != species count is B2MD_CONFIG_ERROR, as the
 * reference throws ConfigError.  Writes jq[3 * n_replicas].  Charge terms are
 * bare Coulomb (+ reaction field), the reference's choice, under every
 * method.  Under NCCL sharding every rank calls it (collective) and gets the
 * full sum. */
int b2md_heat_flux(b2md_ctx* ctx, const double* enthalpy, int n_enthalpy, double* jq);

/* Same, of a host state (the reference's free-function form: positions taken
 * as given, no wrap).  Overwrites the device state; step needs a new
 * set_state afterwards.  pos/orient/vel/ang_vel: AoS, n_replicas systems. */
int b2md_heat_flux_state(b2md_ctx* ctx, const double* pos, const double* orient,
                         const double* vel, const double* ang_vel, const double* enthalpy,
                         int n_enthalpy, double* jq);

/* Thermostat and kinetic energies (src/engine.cpp:145-160, src/model.cpp:
 * 304-330).  kinetic_energy: kinetic_energy_trans / _rot of every replica
 * (fixed-order device reduction).  apply_thermostat: Engine::apply_thermostat
 * (isokinetic rescale to the composition's temperature) on every replica;
 * B2MD_NUMERICAL_ERROR "thermostat: zero translational (rotational) kinetic
 * energy" as the reference throws.  step_thermostat: Engine::run's loop —
 * steps numbered done+1 .. done+nsteps of the phase, the rescale after each
 * step whose number is a multiple of `interval` (<= 0: none). */
int b2md_kinetic_energy(b2md_ctx* ctx, double* ke_trans, double* ke_rot);
int b2md_apply_thermostat(b2md_ctx* ctx);
int b2md_step_thermostat(b2md_ctx* ctx, int64_t nsteps, int interval, int64_t done);

/* Checkpoint state block: the device-resident part of
 * tmd::Engine::checkpoint_bytes (src/engine.cpp:432-441) — u32 n, f64
 * box_length, then per molecule pos.xyz, orient.wxyz, vel.xyz, ang_vel.xyz
 * (13 x f64), little-endian; 12 + 104 n bytes.  save packs replica `replica`
 * on the device.  restore is restore_dynamic's state part (engine.cpp:
 * 479-491) followed by its compute_forces() (engine.cpp:540; no wrap), for
 * one replica; the other replicas keep their state.  Errors as the
 * reference: B2MD_IO_ERROR "checkpoint: molecule count mismatch", the
 * ByteReader's "checkpoint: truncated or corrupted data (need N bytes at
 * offset M)"; a box length different from the composition's is also
 * B2MD_IO_ERROR.  The rest of the container (header, counters, RNG,
 * statistics, samplers) is host data: paper_1507_07548_b200/checkpoint.py. */
size_t b2md_state_block_size(const b2md_ctx* ctx);
int b2md_save_state_block(b2md_ctx* ctx, int replica, uint8_t* buf, size_t cap);
int b2md_restore_state_block(b2md_ctx* ctx, int replica, const uint8_t* buf, size_t len);

/* Radial distribution histograms: tmd::RdfHistogram (include/tmd/structure.hpp:
 * 29-67, src/structure.cpp:10-76) over a context's composition, one histogram
 * per replica, accumulated on the device.  Sampling sites are every LJ and
 * dummy site (charge-only sites skipped); site types are numbered in
 * (species, site) order; counts are uint64 [pair][bin] with pair(ta <= tb) =
 * ta*T - ta(ta+1)/2 + tb, exactly the reference's (integer, bit-exact).
 * create fails like the constructor: bin_width <= 0 or r_max > L/2 (+1e-12)
 * is B2MD_CONFIG_ERROR.  finalize / first_minimum / solvation_number are
 * host arithmetic on these counts (structure.cpp:78-194). */
typedef struct b2md_rdf b2md_rdf;
int b2md_rdf_create(b2md_ctx* ctx, double bin_width, double r_max, b2md_rdf** out);
void b2md_rdf_destroy(b2md_rdf* rdf);
int b2md_rdf_shape(const b2md_rdf* rdf, int* n_types, int* bins, int* n_pairs);
int b2md_rdf_types(const b2md_rdf* rdf, int* species, int* site);
/* accumulate (structure.cpp:38-76) of the context's device state, every replica */
int b2md_rdf_accumulate(b2md_rdf* rdf);
/* ... of host positions / orientations (AoS, n_replicas systems, as given);
 * replaces the context's device state (an Engine needs a new set_state). */
int b2md_rdf_accumulate_state(b2md_rdf* rdf, const double* pos, const double* orient);
int b2md_rdf_counts(const b2md_rdf* rdf, int replica, uint64_t* counts, int64_t* snapshots);
/* restore counts (RdfHistogram::deserialize, structure.cpp:142-153); NULL zeroes */
int b2md_rdf_set_counts(b2md_rdf* rdf, int replica, const uint64_t* counts, int64_t snapshots);

/* Multi-GPU row sharding (one process per GPU).  b2md_nccl_unique_id fills a
 * 128-byte ncclUniqueId on the root; every rank then calls b2md_attach_nccl
 * with the broadcast id.  After attaching, each rank evaluates only its shard
 * of the tile triangle and k-vectors and one packed ncclAllReduce(sum, f64)
 * over NVLink combines forces, torques and energy sums every evaluation. */
int b2md_nccl_unique_id(char id[128]);
int b2md_attach_nccl(b2md_ctx* ctx, const char id[128], int rank, int world);

/* One process driving `ndev` GPUs: the single-process
 * counterpart of one rank per GPU, for a caller shaped like the reference's
 * Engine, which owns the whole computation in one process
 * (src/engine.cpp:100-143) and splits it only over in-process workers
 * (src/parallel.cpp:84-95).  One context per device (b2md_create on
 * devices[k], or device k when devices is NULL), one NCCL communicator per
 * device from ncclCommInitAll; context k is rank k of an ndev-way row shard
 * (as after b2md_attach_nccl).  Group calls run the per-context call on one
 * worker thread per device, so every device's collectives are in flight
 * together, and return the first failure.  Every context holds the whole
 * replicated state; b2md_group_get_state reads rank 0's.  b2md_group_context
 * gives a rank's context for per-device calls (streams, profiling); do not
 * step a group's contexts one by one from a single thread (the all-reduce of
 * one device would wait for the others). */
typedef struct b2md_group b2md_group;
int b2md_create_group(int ndev, const int* devices, const b2md_composition* comp,
                      const b2md_ff_options* opts, double dt, int n_replicas, b2md_group** out);
void b2md_destroy_group(b2md_group* group);
int b2md_group_size(const b2md_group* group);
b2md_ctx* b2md_group_context(b2md_group* group, int rank);
int b2md_group_set_state(b2md_group* group, const double* pos, const double* orient,
                         const double* vel, const double* ang_vel);
int b2md_group_step(b2md_group* group, int64_t nsteps);
int b2md_group_step_async(b2md_group* group, int64_t nsteps);
int b2md_group_sync(b2md_group* group);
int b2md_group_get_state(b2md_group* group, double* pos, double* orient, double* vel,
                         double* ang_vel, double* force, double* torque, b2md_energy* energy,
                         b2md_eval_stats* stats);

/* Restrict the context to rank `rank`'s shard of a `world`-way split
 * WITHOUT a communicator: evaluations then return that rank's partial forces,
 * torques and sums (what each rank holds before the all-reduce).  For tests
 * of the decomposition on one device; b2md_attach_nccl is the production path. */
int b2md_set_shard(b2md_ctx* ctx, int rank, int world);

/* Opaque cudaStream_t of the context (for event timing by the caller).  Every
 * call's work is ordered on this stream; Ewald systems fork the tables and
 * S(k) onto an internal second stream and join it back within the same call,
 * so events recorded on this stream bracket the whole evaluation. */
void* b2md_stream(b2md_ctx* ctx);

/* Per-kernel CUDA-event timing of the device step (bench instrumentation).
 * enable = 1 records an event pair around every launch of each kernel
 * family, enable = 2 only around the partner search, enable = 3 only around
 * the force walk (one family at a time: least perturbation); 0 turns it off.  Single steps run as a CUDA graph whose
 * event-record nodes are re-pointed at fresh events before every launch.
 * b2md_kernel_times returns {name, total_ms, launches} rows. */
int b2md_profile_enable(b2md_ctx* ctx, int enable);
int b2md_kernel_times(b2md_ctx* ctx, int max_rows, char (*names)[32], double* total_ms,
                      int64_t* launches, int* n_rows);

/* Use a CUDA graph for the device step loop (default on). */
int b2md_set_graphs(b2md_ctx* ctx, int enable);

/* Measured FP64 (DFMA) peak of the device, GFLOP/s, from a short
 * microbenchmark (roofline denominator). */
int b2md_measure_fp64_peak(int device, double* gflops);

#ifdef __cplusplus
}
#endif

#endif /* B200MD_H */
