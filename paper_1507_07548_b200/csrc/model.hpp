// Host-side model tables of the b200md force field: everything the reference
// computes once in the ForceField constructor (src/parallel.cpp:55-72) —
// PairTable (src/potentials.cpp:35-83), LJ long-range correction
// (src/potentials.cpp:7-33), composition validation (src/model.cpp:244-268)
// and the Ewald constants/k-vectors (src/ewald.cpp:30-105) — plus the
// species builder (src/model.cpp:68-129) and the multi-GPU shard plan.
// Compiled with -ffp-contract=off so every constant is bit-identical to the
// reference's (the device kernels then see exactly the reference's c12, c6,
// rmax^2, Ewald coefficients).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "../../include/b200md.h"

namespace b2md {

struct LjTerm {
  int a, b;
  double c12, c6;
};

struct QTerm {
  int a, b;
  double qq;
};

struct KVec {
  int nx, ny, nz;
  double kx, ky, kz, coeff;
};

struct ChargedSite {
  int mol;   // molecule index within a replica
  int site;  // global site index within a replica (site_begin[mol] + k)
  double q;
};

struct ModelTables {
  // composition
  int ns = 0;
  int n = 0;            // molecules per replica
  int total_sites = 0;  // sites per replica
  double box = 0.0, temperature = 0.0;
  std::vector<b2md_species> species;
  std::vector<int> counts;
  std::vector<int> species_of;  // per molecule
  std::vector<int> site_begin;  // per molecule + 1
  bool any_rigid = false;       // some species has rotational dof
  bool any_offsets = false;     // some species has non-centred sites
  // PairTable
  int method = B2MD_METHOD_NONE;
  double rc = 0.0, rc2 = 0.0;
  double rf_factor = 0.0, rf_r3inv = 0.0, rf_shift = 0.0;
  double alpha = 0.0;
  bool single_lj_only = false;
  bool single_site_path = false;  // evaluate_range_single_site applies
  bool vderiv = true;
  std::vector<std::vector<LjTerm>> lj;  // [sa*ns+sb]
  std::vector<std::vector<QTerm>> qq;   // [sa*ns+sb]
  std::vector<double> rmax2;            // [sa*ns+sb] COM search radius^2
  double lrc_k = 0.0;
  // Ewald
  bool ewald = false;
  int kmax = 0;
  double self_plus_intra = 0.0;
  std::vector<KVec> kv;
  std::vector<ChargedSite> charged;  // per replica, molecule order
  std::string warning;
};

// Returns B2MD_OK or an error code with `err` set (reference exception text).
int build_tables(const b2md_composition& comp, const b2md_ff_options& opts, ModelTables& out,
                 std::string& err);

int build_species(const b2md_site* sites, int n, b2md_species& out, std::string& err);
int ewald_tune(double delta, double cutoff, double box, double& alpha, int& kmax, std::string& err);
int count_kvectors(int kmax);

// Tile-row shard plan (32-molecule tiles, i<j triangle).
void shard_plan(int n_molecules, int n_kvectors, int world, int rank, int& row_begin, int& row_end,
                int& k_begin, int& k_end, int64_t& candidates);

}  // namespace b2md
