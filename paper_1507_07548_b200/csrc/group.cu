// One process, N GPUs: b2md_create_group and the group calls (include/b200md.h).
//
// The reference is a single process: Engine::step calls ForceField::evaluate
// (src/engine.cpp:100-143), whose only split is the static partition of the
// flat pair index over in-process workers (src/parallel.cpp:84-95).  The
// group is the B200 form of that split for a caller that owns all GPUs in one
// process: one context per device (the full replicated state, its row shard
// of the pair work), one NCCL communicator per device from ncclCommInitAll,
// and the packed all-reduce of every evaluation over NVLink.  Every group call
// runs the per-device call on a persistent worker thread per device, so the
// collectives of all devices are in flight together (a single host thread
// issuing them one device after the other would wait on itself), and reports
// the first failure.
#include <condition_variable>
#include <functional>
#include <mutex>
#include <thread>

#include "ctx_internal.cuh"

namespace b2md_host {
int setup_shard(b2md_ctx* c);
}
using namespace b2md_host;

struct b2md_group {
  std::vector<b2md_ctx*> ctx;
  // worker pool: worker k runs task(k) for every posted generation
  std::vector<std::thread> workers;
  std::mutex mu;
  std::condition_variable cv_go, cv_done;
  std::function<int(int)> task;
  uint64_t gen = 0;
  int pending = 0;
  bool quit = false;
  std::vector<int> rc;
  std::vector<std::string> err;

  void worker(int k) {
    uint64_t seen = 0;
    for (;;) {
      std::function<int(int)> t;
      {
        std::unique_lock<std::mutex> lk(mu);
        cv_go.wait(lk, [&] { return quit || gen != seen; });
        if (quit) return;
        seen = gen;
        t = task;
      }
      const int r = t(k);
      std::string e = r ? b2md_last_error() : std::string();
      std::lock_guard<std::mutex> lk(mu);
      rc[k] = r;
      err[k] = e;
      if (--pending == 0) cv_done.notify_all();
    }
  }

  // run f(k) on every device's worker; the first failure (lowest rank) wins
  int run(std::function<int(int)> f) {
    {
      std::unique_lock<std::mutex> lk(mu);
      task = std::move(f);
      pending = int(ctx.size());
      ++gen;
    }
    cv_go.notify_all();
    std::unique_lock<std::mutex> lk(mu);
    cv_done.wait(lk, [&] { return pending == 0; });
    for (size_t k = 0; k < ctx.size(); ++k)
      if (rc[k]) return set_err(rc[k], "device " + std::to_string(ctx[k]->device) + ": " + err[k]);
    return B2MD_OK;
  }

  ~b2md_group() {
    {
      std::lock_guard<std::mutex> lk(mu);
      quit = true;
    }
    cv_go.notify_all();
    for (auto& w : workers) w.join();
    for (b2md_ctx* c : ctx) b2md_destroy(c);
  }
};

extern "C" {

int b2md_create_group(int ndev, const int* devices, const b2md_composition* comp,
                      const b2md_ff_options* opts, double dt, int n_replicas, b2md_group** out) {
  NvtxRange nvtx_("b2md_create_group");
  if (!out || !comp || !opts || ndev < 1)
    return set_err(B2MD_INVALID_ARGUMENT, "create_group: bad argument");
  *out = nullptr;
  std::vector<int> dev(ndev);
  for (int k = 0; k < ndev; ++k) dev[k] = devices ? devices[k] : k;
  auto* g = new b2md_group();
  for (int k = 0; k < ndev; ++k) {
    b2md_ctx* c = nullptr;
    const int rc = b2md_create(dev[k], comp, opts, dt, n_replicas, &c);
    if (rc) {
      const std::string keep = b2md_last_error();
      delete g;
      return set_err(rc, keep);
    }
    g->ctx.push_back(c);
  }
  if (ndev > 1) {
    int rc = nccl_load();
    if (!rc && !g_nccl.CommInitAll) rc = set_err(B2MD_CUDA_ERROR, "NCCL: ncclCommInitAll missing");
    std::vector<ncclComm_t> comms(ndev, nullptr);
    if (!rc) {
      const ncclResult_t r = g_nccl.CommInitAll(comms.data(), ndev, dev.data());
      if (r != ncclSuccess)
        rc = set_err(B2MD_CUDA_ERROR, std::string("NCCL error: ") + g_nccl.GetErrorString(r) +
                                          " at ncclCommInitAll");
    }
    for (int k = 0; k < ndev && !rc; ++k) {
      b2md_ctx* c = g->ctx[k];
      c->comm = comms[k];
      c->rank = k;
      c->world = ndev;
      if (cudaSetDevice(c->device) != cudaSuccess) rc = set_err(B2MD_CUDA_ERROR, "create_group: device");
      if (!rc) rc = setup_shard(c);
    }
    if (rc) {
      const std::string keep = b2md_last_error();
      delete g;
      return set_err(rc, keep);
    }
  }
  g->rc.assign(ndev, 0);
  g->err.assign(ndev, std::string());
  for (int k = 0; k < ndev; ++k) g->workers.emplace_back([g, k] { g->worker(k); });
  *out = g;
  return B2MD_OK;
}

void b2md_destroy_group(b2md_group* g) { delete g; }

int b2md_group_size(const b2md_group* g) { return g ? int(g->ctx.size()) : 0; }

b2md_ctx* b2md_group_context(b2md_group* g, int rank) {
  if (!g || rank < 0 || rank >= int(g->ctx.size())) return nullptr;
  return g->ctx[rank];
}

int b2md_group_set_state(b2md_group* g, const double* pos, const double* orient, const double* vel,
                         const double* ang_vel) {
  if (!g) return set_err(B2MD_INVALID_ARGUMENT, "group_set_state: null group");
  return g->run([&](int k) { return b2md_set_state(g->ctx[k], pos, orient, vel, ang_vel); });
}

int b2md_group_step(b2md_group* g, int64_t nsteps) {
  if (!g) return set_err(B2MD_INVALID_ARGUMENT, "group_step: null group");
  return g->run([&](int k) { return b2md_step(g->ctx[k], nsteps); });
}

int b2md_group_step_async(b2md_group* g, int64_t nsteps) {
  if (!g) return set_err(B2MD_INVALID_ARGUMENT, "group_step_async: null group");
  return g->run([&](int k) { return b2md_step_async(g->ctx[k], nsteps); });
}

int b2md_group_sync(b2md_group* g) {
  if (!g) return set_err(B2MD_INVALID_ARGUMENT, "group_sync: null group");
  return g->run([&](int k) { return b2md_sync(g->ctx[k]); });
}

int b2md_group_get_state(b2md_group* g, double* pos, double* orient, double* vel, double* ang_vel,
                         double* force, double* torque, b2md_energy* energy,
                         b2md_eval_stats* stats) {
  if (!g) return set_err(B2MD_INVALID_ARGUMENT, "group_get_state: null group");
  // every device holds the whole (replicated) state after the all-reduce;
  // the others are synchronised so no step is left in flight
  return g->run([&](int k) {
    return k == 0 ? b2md_get_state(g->ctx[0], pos, orient, vel, ang_vel, force, torque, energy, stats)
                  : b2md_sync(g->ctx[k]);
  });
}

}  // extern "C"
