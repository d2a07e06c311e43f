// Internal to libb200md (not installed): the context struct and the host
// helpers shared by context.cu (setup, launch sequences, graphs, transfers,
// NCCL, the core C ABI) and samplers.cu (heat flux, RDF, thermostat,
// checkpoint state).
#pragma once

#include <cuda_runtime.h>
#include <nccl.h>
#include <nvtx3/nvToolsExt.h>
#include <dlfcn.h>
#include <algorithm>
#include <cub/cub.cuh>
#include <cstdlib>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <string>
#include <vector>
#include "../../include/b200md.h"
#include "kernels.cuh"
#include "rdf.cuh"
#include "cluster.cuh"
#include "model.hpp"
#include "search_geometry.hpp"

// NVTX range over one C-ABI call (header-only NVTX3: free unless a tool such as
// nsys / ncu --nvtx attaches): the tracing hook of SURVEY 5
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

namespace b2md_host {
using namespace b2md;

int set_err(int code, const std::string& msg);

// (a failed call's error is consumed here, so a non-sticky error -- e.g. an
// invalid device number -- is not reported again by a later launch check)
#define CU(expr)                                                                          \
  do {                                                                                    \
    cudaError_t e_ = (expr);                                                              \
    if (e_ != cudaSuccess) {                                                              \
      cudaGetLastError();                                                                 \
      return set_err(B2MD_CUDA_ERROR, std::string("CUDA error: ") + cudaGetErrorString(e_) + \
                                          " at " #expr);                                  \
    }                                                                                     \
  } while (0)

// NCCL is resolved at first multi-GPU use (dlopen), not linked: a process
// that loads another NCCL first (e.g. PyTorch's bundled one) keeps it.
struct NcclApi {
  bool loaded = false;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;  // b2md_create_group
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};
extern NcclApi g_nccl;
int nccl_load();

#define NC(expr)                                                                        \
  do {                                                                                  \
    ncclResult_t r_ = (expr);                                                           \
    if (r_ != ncclSuccess)                                                              \
      return set_err(B2MD_CUDA_ERROR, std::string("NCCL error: ") +                     \
                                          g_nccl.GetErrorString(r_) + " at " #expr);    \
  } while (0)

#define TRY(expr)          \
  do {                     \
    int rc_ = (expr);      \
    if (rc_) return rc_;   \
  } while (0)

inline int hi32(double x) {
  int64_t b;
  std::memcpy(&b, &x, 8);
  return int(b >> 32);
}

template <typename T>
int dalloc(T** p, size_t count) {
  if (count == 0) count = 1;
  CU(cudaMalloc(reinterpret_cast<void**>(p), count * sizeof(T)));
  CU(cudaMemset(*p, 0, count * sizeof(T)));
  return B2MD_OK;
}

enum Family { F_OFFSETS, F_SEARCH, F_FORCE, F_EWALD_TAB, F_EWALD_SK, F_EWALD_F, F_KICK_KICK_DRIFT,
              F_KICK_DRIFT, F_KICK, F_ALLREDUCE, F_HEAT_FLUX, F_RDF, F_CLUSTER, F_JSUM, F_NL_BUILD,
              F_COUNT };
extern const char* kFamilyName[F_COUNT];

}  // namespace b2md_host

using namespace b2md;  // device types of the context (kernels.cuh, model.hpp)

struct b2md_ctx {
  int device = 0;
  int sms = 148;  // streaming multiprocessors of the device
  cudaStream_t stream = nullptr;
  // Ewald tables + S(k) run on stream2 beside the real-space kernel (fork /
  // join events; captured into the step graphs as parallel branches)
  cudaStream_t stream2 = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  ModelTables t;
  SearchGeometry g;
  int R = 1;
  double dt = 0.0;
  bool engine = false;
  bool state_valid = false;
  bool positions_wrapped = false;  // step-time positions lie in [0, L) (the drift wraps first)
  bool state_in_box = false;       // the CURRENT device positions lie in [0, L)
                                   // (false after a raw upload / restore until a step wraps)
  // device tables
  DevTables* d_tab = nullptr;
  int* d_species_of = nullptr;
  int* d_site_begin = nullptr;
  // state
  double* d_state = nullptr;  // px..wz (13 arrays of R*n)
  double* d_fbuf = nullptr;   // fx fy fz tx ty tz (6*R*n) + sums (R*kNumSums): allreduce unit
  double4* d_off = nullptr;   // R * total_sites site offsets
  double4* d_pos4 = nullptr;  // R * n packed positions
  double* d_stage = nullptr;  // AoS staging: 6 slots of 4*R*n (one per array, no reuse waits)
  uint32_t* d_mask = nullptr;
  uint4* d_fixpos = nullptr;  // fixed-point positions (search prefilter, cluster arcs)
  bool mask_valid = false;    // d_mask holds the current positions' partners
  // cluster walk of the single-site path (cluster.cuh)
  bool use_cluster = true;
  int nc = 0, nsup = 0;       // clusters, super-clusters per replica
  uint4* d_carc = nullptr;    // R * nc arc centres
  float4* d_chalf = nullptr;  // R * nc arc half extents
  uint4* d_sarc = nullptr;    // R * nsup
  float4* d_shalf = nullptr;  // R * nsup
  // once-per-pair cluster-pair list (k_force_nl + k_nl_reduce, cluster.cuh)
  bool nl_member_gaps = true;  // k_nl_gaps after every list build
  bool use_newton = true;      // once-per-pair list on the cluster path (B2MD_NEWTON=0: both-rows walk)
  NListArgs nl{};              // device arrays of the list (null: not allocated)
  double nl_skin = 0.0;        // list skin (length units)
  int nl_interval = 0;         // steps between scheduled builds (0: only at staging / re-sort)
  int64_t steps_since_nl = 0;
  int n3_grid = 0;             // persistent CTAs per replica of k_force_nl
  // rigid single-species LJ molecules: once-per-pair block-pair tiles
  // (k_force_rigid_tile + k_rigid_reduce; B2MD_TILE=0: search + k_force_rigid)
  bool use_tile = false;
  double* d_trec = nullptr;    // R * nbp * kTileSplit * 2 * 32 * 6
  int tile_nb = 0, tile_nbp = 0;
  double* d_cta_part = nullptr;  // force-kernel per-CTA scalar partials
  unsigned* d_ticket = nullptr;   // 2 * R: force, ewald
  int force_grid = 1;
  int force_warps = kForceWarps;  // warps per CTA of the partner walks
  int force_split = 1;            // warps per row in the force walks (1, 2, 4, 8)
  uint32_t* d_super = nullptr;
  int n_super_tiles = 0;
  int* d_error = nullptr;
  StateDev st{};
  SysDev sys{};
  // ewald
  int nq = 0;
  int* d_q_mol = nullptr;
  int* d_q_site = nullptr;
  double* d_q_val = nullptr;
  int* d_mol_qbegin = nullptr;
  DevKVec* d_kv = nullptr;
  double2* d_etab = nullptr;
  double2* d_S = nullptr;
  double* d_uk = nullptr;
  bool ew_tiled = false;        // tiled S(k) / force kernels (B2MD_EWALD_TILED=0: gather form)
  double2* d_ewSp = nullptr;    // R * chunks * nk: S(k) partials
  double* d_ewfq = nullptr;     // R * nq * 3: reciprocal force per charge
  double* d_frec = nullptr;     // 6 * R * n: reciprocal forces / torques (ewald_overlap)
  bool ew_overlap = true;       // k_ewald_force beside the real-space kernel in step paths
  double* d_flux = nullptr;  // R * kNumSums: heat flux totals
  double2* d_ke = nullptr;    // R: (kinetic_energy_trans, kinetic_energy_rot)
  int* d_thermo_err = nullptr;  // R: thermostat failure code (0 ok)
  // spatial order (resort): slot tables and radix-sort buffers
  int* d_perm = nullptr;
  int* d_slot_of = nullptr;
  int* d_sp_slot = nullptr;
  int* d_sb_slot = nullptr;
  int* d_nsites_slot = nullptr;
  int* d_scan = nullptr;
  unsigned long long* d_keys[2] = {nullptr, nullptr};
  int* d_vals[2] = {nullptr, nullptr};
  void* d_cub = nullptr;
  size_t cub_bytes = 0;
  int sort_interval = 100;  // steps between re-sorts (0: keep the input order)
  int64_t steps_since_sort = 0;
  // sharding
  int rank = 0, world = 1;
  int row_begin = 0, row_end = 0, k_begin = 0, k_end = 0;
  ncclComm_t comm = nullptr;
  // graphs
  bool use_graphs = true;
  bool use_fix_prefilter = true;
  bool use_tile_cull = true;
  bool use_fused_kick = true;  // end-of-step half kick inside the force kernel
  cudaGraphExec_t step_graph = nullptr;  // forces + fused kick/kick-drift
  cudaGraphExec_t single_graph = nullptr;  // one whole step
  cudaGraphExec_t prof_graph = nullptr;    // one whole step with event-record nodes
  cudaGraph_t prof_template = nullptr;      // its template (owns the node handles)
  bool capturing_prof = false;
  std::vector<cudaEvent_t> cap_ev;          // placeholder events captured into prof_graph
  std::vector<int> cap_fam;                 // kernel family of each captured event pair
  std::vector<cudaGraphNode_t> cap_nodes;   // the event-record node of each placeholder
  // profiling
  bool profile = false;
  int profile_level = 1;   // 1: every kernel family, 2: the partner search only, 3: the force walk only
  bool prof_open = false;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev_pool;
  size_t ev_used = 0;
  std::vector<int> ev_family;
  double prof_ms[b2md_host::F_COUNT] = {};
  int64_t prof_n[b2md_host::F_COUNT] = {};
  // host scratch
  std::vector<double> h_sums;
  double* h_sums_pinned = nullptr;  // energy sums read-back (cudaMallocHost)
  int* h_flag = nullptr;            // error flag read-back (cudaMallocHost)
  bool async_pending = false;       // b2md_step_async not yet checked

  std::string warning;
};

namespace b2md_host {

// context.cu helpers used by samplers.cu
int n_total(const b2md_ctx* c);
void drop_graphs(b2md_ctx* c);
void set_wrapped(b2md_ctx* c, bool w);
int prof_begin(b2md_ctx* c, int fam);
int prof_end(b2md_ctx* c);
int launch_offsets(b2md_ctx* c);
int launch_search(b2md_ctx* c);
int ensure_mask(b2md_ctx* c);
bool cluster_path(const b2md_ctx* c);
int cpair_grid(const b2md_ctx* c);
ClusterArgs cluster_args(const b2md_ctx* c);
int launch_cluster_arcs(b2md_ctx* c);
int nl_build(b2md_ctx* c);
ForceArgs force_args(b2md_ctx* c);
bool fast_min_image(const b2md_ctx* c);
int resort(b2md_ctx* c);
int resort_and_stage(b2md_ctx* c);
int enqueue_forces(b2md_ctx* c, bool offsets, bool kick = false, bool recip_beside = false);
int run_steps(b2md_ctx* c, int64_t nsteps);
int upload_aos(b2md_ctx* c, int slot, const double* host, int width, double* d0, double* d1,
               double* d2, double* d3);
int check_error_flag(b2md_ctx* c);
int error_from_flag(b2md_ctx* c, int flag);

#define PROF(ctx, fam, launch)      \
  do {                              \
    TRY(prof_begin(ctx, fam));      \
    launch;                         \
    CU(cudaGetLastError());         \
    TRY(prof_end(ctx));             \
  } while (0)

}  // namespace b2md_host
