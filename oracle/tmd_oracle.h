/*
 * tmd_oracle.h — CPU oracle for the b200md parity tests.  TEST INFRASTRUCTURE
 * ONLY: nothing on the product path (paper_1507_07548_b200/, include/) may
 * link or call it.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs use it, as the checker.
 *
 * A plain-C restatement of the reference `tmd` force/energy/partner-search
 * and integrator path (/root/reference/proj), serial (the reference with
 * workers = 1).  Each function cites the reference file:line it restates and
 * keeps the reference's floating-point operation order; compiled without FMA
 * contraction (-ffp-contract=off, no -march) it reproduces the reference bit
 * for bit.  Parity is pinned twice: (1) against the real reference compiled
 * from /root/reference into oracle/_ref (tests/test_oracle_pins.py, bitwise),
 * (2) against the known-answer values of the reference's own tests and the
 * committed golden vectors under tests/golden/ (generated from oracle/_ref by
 * tests/golden/make_golden.py).
 *
 * The model structs are the C-ABI's POD types (include/b200md.h).
 */
#ifndef TMD_ORACLE_H
#define TMD_ORACLE_H

#include "../include/b200md.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct oracle_ff oracle_ff;

const char* oracle_last_error(void);

int oracle_build_species(const b2md_site* sites, int n_sites, b2md_species* out);
int oracle_ewald_tune(double delta, double cutoff, double box_length, double* alpha, int* kmax);

int oracle_ff_create(const b2md_composition* comp, const b2md_ff_options* opts, oracle_ff** out);
void oracle_ff_destroy(oracle_ff* ff);
const char* oracle_ff_warning(const oracle_ff* ff);
int oracle_ff_kvector_count(const oracle_ff* ff);
int oracle_ff_molecules(const oracle_ff* ff);

/* ForceField::evaluate, serial (src/parallel.cpp:79-122, W = 1). */
int oracle_evaluate(oracle_ff* ff, const double* pos, const double* orient, double* force,
                    double* torque, b2md_energy* energy, b2md_eval_stats* stats);

/* Shard of an evaluation: molecule pairs with i in [row_begin*32,
 * row_end*32) (a contiguous flat-index range of src/potentials.cpp:133-143)
 * and k-vectors [k_begin, k_end).  Outputs raw partial sums: force, torque,
 * and sums[8] = {u_lj, u_elec_real, u_rf, s1, s2, virial, u_recip, com_pairs}. */
int oracle_evaluate_shard(oracle_ff* ff, const double* pos, const double* orient, int row_begin,
                          int row_end, int k_begin, int k_end, double* force, double* torque,
                          double* sums);

/* COM partner search (src/potentials.cpp:156-158 / 209-213): i<j pairs in
 * flat order.  Returns the count; writes up to `capacity` (i,j) pairs. */
int64_t oracle_pair_list(oracle_ff* ff, const double* pos, int32_t* pairs, int64_t capacity);

/* Engine::set_state's wrap (src/model.cpp:279-286) */
void oracle_wrap(int n, double box_length, double* pos);

/* Engine::step x nsteps (src/engine.cpp:102-143).  force/torque must hold the
 * forces of the incoming state (as Engine keeps them cached). */
int oracle_step(oracle_ff* ff, double dt, int64_t nsteps, double* pos, double* orient, double* vel,
                double* ang_vel, double* force, double* torque, b2md_energy* energy,
                b2md_eval_stats* stats);

/* heat_flux (src/greenkubo.cpp:182-266): J_q of the given state;
 * `enthalpy` holds one partial molar enthalpy per species. */
int oracle_heat_flux(oracle_ff* ff, const double* pos, const double* orient, const double* vel,
                     const double* ang_vel, const double* enthalpy, int n_enthalpy, double* jq);

/* kinetic_energy_trans / _rot (src/model.cpp:304-319): out[2] */
int oracle_kinetic_energy(const oracle_ff* ff, const double* vel, const double* ang_vel, double* out);
/* Engine::apply_thermostat (src/engine.cpp:145-160), in place */
int oracle_apply_thermostat(const oracle_ff* ff, double* vel, double* ang_vel);

/* RdfHistogram (include/tmd/structure.hpp:29-67, src/structure.cpp:10-76):
 * integer site-pair histograms per unordered site-type pair. */
typedef struct oracle_rdf oracle_rdf;
int oracle_rdf_create(const oracle_ff* ff, double bin_width, double r_max, oracle_rdf** out);
void oracle_rdf_destroy(oracle_rdf* rdf);
/* structure.cpp:38-76 */
int oracle_rdf_accumulate(oracle_rdf* rdf, const double* pos, const double* orient);
int oracle_rdf_shape(const oracle_rdf* rdf, int* n_types, int* bins, int* n_pairs);
/* counts[pair * bins + bin] */
int oracle_rdf_counts(const oracle_rdf* rdf, uint64_t* counts, int64_t* snapshots);

#ifdef __cplusplus
}
#endif

#endif
