// Several GPUs in one process behind the C-ABI (eik_solve_multi): fsm_solve
// (classic_solvers.cpp:128-158) as strip-Jacobi over row strips, one device
// per strip (SURVEY.md 8(b) "n_gpus plus device list", 8(e) option A).
//
// Device d owns rows [n d / P, n (d+1) / P) plus a frozen ghost row on each
// side (exit nodes of its local plan whose values are overwritten).  Round k:
// every device sweeps its strip once in direction k mod 4 (the exact
// wavefront kernel, eik_plan_sweep), then each strip's edge rows go into its
// neighbours' ghost rows by peer copies over NVLink (cudaMemcpyPeerAsync:
// one process drives every device, so no communicator is needed), and the
// change flags are OR-ed on the host.  The run stops after the first round
// in which no strip changed: that round read ghost rows equal to the
// post-round state, so the field is the discrete fixed point fsm_solve
// converges to.  With one device it IS fsm_solve (eik_solve).  Per device:
// its strip's F, C and u only (1/P of the grid).  The multi-process variant
// (one rank per GPU, NCCL over torch.distributed) is distributed.py.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <condition_variable>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "eik_internal.h"
#include "eik_plan.h"
#include "eikonal_b200.h"

namespace eikb200 {

eik_plan* plan_create(const eik_problem* p, const eik_cells* c, int32_t method, bool defer_upload,
                      cudaStream_t stream, const cudaEvent_t* events);
int plan_prepare(eik_plan* P);
int plan_sweep(eik_plan* P, int64_t first_sweep, int count, int* changed);
int plan_rows_async(eik_plan* P, int64_t row0, int64_t nrows, double* dev_buf, bool to_plan,
                    cudaStream_t stream);
void plan_free(eik_plan* P);
int64_t fmm_node_updates(const eik_grid& g, const int64_t* exits, int64_t n_exit);

namespace {

constexpr double kInfM = __builtin_huge_val();

class Barrier {
 public:
  explicit Barrier(int n) : n_(n) {}
  void wait() {
    std::unique_lock<std::mutex> lk(mu_);
    const int gen = gen_;
    if (++count_ == n_) {
      count_ = 0;
      ++gen_;
      cv_.notify_all();
    } else {
      cv_.wait(lk, [&] { return gen != gen_; });
    }
  }

 private:
  std::mutex mu_;
  std::condition_variable cv_;
  int n_, count_ = 0, gen_ = 0;
};

struct Strip {
  int device = 0;
  int64_t r0 = 0, r1 = 0, nl = 0;  // global rows [r0, r1); local rows 0..nl-1
  std::vector<double> F;            // local speed (ghost rows: 1)
  std::vector<int64_t> exits;
  std::vector<double> cost;
  eik_plan* plan = nullptr;
  cudaStream_t stream = nullptr;
  double* recv = nullptr;           // [2][m] on the strip's device: the neighbours' edge rows land
                                    // here, then go into the ghost rows through plan_rows_async,
                                    // which marks what they change for the next sweep launch
  int changed[2] = {0, 0};  // by round parity: a fast thread writes round k+1's
                            // flag while a slow one still reads round k's
  int rc = EIK_OK;
  std::string msg;
  double* row(int64_t local) const { return plan->dU + local * plan->pitch + kPad; }
};

}  // namespace

int solve_multi(const eik_problem* p, int32_t method, const int32_t* devices, int32_t n_dev,
                eik_output* out) {
  const int64_t m = p->grid.m, n = p->grid.n;
  if (n_dev > n) return fail(EIK_ERR_CONFIG, "more devices than grid rows");
  if (p->speed_on_device) return fail(EIK_ERR_NOT_IMPL, "eik_solve_multi takes a host speed array");
  if (out->u_on_device) return fail(EIK_ERR_NOT_IMPL, "eik_solve_multi writes a host u");
  const auto t0 = std::chrono::steady_clock::now();
  std::vector<Strip> S(n_dev);
  for (int d = 0; d < n_dev; ++d) {
    Strip& s = S[d];
    s.device = devices[d];
    s.r0 = n * d / n_dev;
    s.r1 = n * (d + 1) / n_dev;
    s.nl = s.r1 - s.r0 + 2;
    s.F.assign((size_t)s.nl * m, 1.0);
    std::memcpy(s.F.data() + m, p->speed + s.r0 * m, sizeof(double) * (size_t)(s.r1 - s.r0) * m);
    for (int64_t i = 0; i < m; ++i) {  // ghost row 0 (frozen)
      s.exits.push_back(i);
      s.cost.push_back(0.0);
    }
    const int64_t* lo = std::lower_bound(p->exit_nodes, p->exit_nodes + p->n_exit, s.r0 * m);
    const int64_t* hi = std::lower_bound(p->exit_nodes, p->exit_nodes + p->n_exit, s.r1 * m);
    for (const int64_t* e = lo; e < hi; ++e) {
      s.exits.push_back(*e - (s.r0 - 1) * m);
      s.cost.push_back(p->exit_cost[e - p->exit_nodes]);
    }
    for (int64_t i = 0; i < m; ++i) {  // ghost row nl-1
      s.exits.push_back((s.nl - 1) * m + i);
      s.cost.push_back(0.0);
    }
  }
  Barrier bar(n_dev);
  int64_t rounds = 0;
  const int64_t limit = 4 * (m + n) + 16;
  std::vector<double> inf_row((size_t)m, kInfM);
  auto worker = [&](int d) {
    Strip& s = S[d];
    auto fail_here = [&](int rc) {
      s.rc = rc;
      s.msg = eik_last_error();
    };
    if (cudaSetDevice(s.device) != cudaSuccess || cudaStreamCreateWithFlags(&s.stream, cudaStreamNonBlocking) != cudaSuccess) {
      s.rc = EIK_ERR_CUDA;
      s.msg = "cannot use device " + std::to_string(s.device);
    }
    for (int e : {d - 1, d + 1})  // NVLink peer access to the neighbouring devices
      if (s.rc == EIK_OK && e >= 0 && e < n_dev && S[e].device != s.device) {
        int ok = 0;
        cudaDeviceCanAccessPeer(&ok, s.device, S[e].device);
        if (ok && cudaDeviceEnablePeerAccess(S[e].device, 0) != cudaSuccess) cudaGetLastError();
      }
    if (s.rc == EIK_OK) {
      eik_problem lp{};
      lp.grid = {m, s.nl, p->grid.h, p->grid.x0, p->grid.y0 + (double)(s.r0 - 1) * p->grid.h};
      lp.speed = s.F.data();
      lp.exit_nodes = s.exits.data();
      lp.exit_cost = s.cost.data();
      lp.n_exit = (int64_t)s.exits.size();
      s.plan = plan_create(&lp, nullptr, EIK_FSM, false, nullptr, nullptr);
      if (!s.plan) fail_here(eik_last_status() ? eik_last_status() : EIK_ERR_CUDA);
      else if (int rc = plan_prepare(s.plan)) fail_here(rc);
      else {  // off-grid beyond the domain edges: +inf ghost rows until exchanged
        cudaMemcpy(s.row(0), inf_row.data(), sizeof(double) * m, cudaMemcpyHostToDevice);
        cudaMemcpy(s.row(s.nl - 1), inf_row.data(), sizeof(double) * m, cudaMemcpyHostToDevice);
        if (cudaMalloc(&s.recv, sizeof(double) * 2 * m) != cudaSuccess) {
          s.rc = EIK_ERR_CUDA;
          s.msg = "cannot allocate the ghost-row receive buffer";
        }
      }
      s.F.clear();
      s.F.shrink_to_fit();
    }
    bar.wait();
    bool failed = false;
    for (const Strip& o : S) failed = failed || o.rc != EIK_OK;
    for (int64_t k = 0; !failed; ++k) {
      if (d == 0 && k >= limit) {
        s.rc = EIK_ERR_BUDGET;
        s.msg = "strip-Jacobi FSM did not converge within the round budget";
      }
      int ch = 0;
      if (s.rc == EIK_OK) {
        if (int rc = plan_sweep(s.plan, k, 1, &ch)) fail_here(rc);
      }
      s.changed[k & 1] = ch;
      bar.wait();  // every strip swept round k
      // edge rows into the neighbours' ghost rows (device to device)
      // (into their receive buffers: slot 0 = their lower ghost row's new
      // values, slot 1 = their upper one's)
      if (s.rc == EIK_OK && d > 0 && S[d - 1].recv)
        cudaMemcpyPeerAsync(S[d - 1].recv + m, S[d - 1].device, s.row(1), s.device,
                            sizeof(double) * m, s.stream);
      if (s.rc == EIK_OK && d + 1 < n_dev && S[d + 1].recv)
        cudaMemcpyPeerAsync(S[d + 1].recv, S[d + 1].device, s.row(s.nl - 2), s.device,
                            sizeof(double) * m, s.stream);
      if (s.rc == EIK_OK && cudaStreamSynchronize(s.stream) != cudaSuccess) {
        s.rc = EIK_ERR_CUDA;
        s.msg = "peer copy of strip edge rows failed";
      }
      bar.wait();  // every receive buffer holds round k's edges
      if (s.rc == EIK_OK && d > 0 && S[d - 1].rc == EIK_OK)
        if (int rc = plan_rows_async(s.plan, 0, 1, s.recv, true, s.stream)) fail_here(rc);
      if (s.rc == EIK_OK && d + 1 < n_dev && S[d + 1].rc == EIK_OK)
        if (int rc = plan_rows_async(s.plan, s.nl - 1, 1, s.recv + m, true, s.stream)) fail_here(rc);
      if (s.rc == EIK_OK && cudaStreamSynchronize(s.stream) != cudaSuccess) {
        s.rc = EIK_ERR_CUDA;
        s.msg = "ghost row update failed";
      }
      bar.wait();  // ghost rows hold round k's edges
      bool any = false;
      for (const Strip& o : S) {
        any = any || o.changed[k & 1];
        failed = failed || o.rc != EIK_OK;
      }
      if (d == 0) rounds = k + 1;
      if (!any) break;
    }
  };
  std::vector<std::thread> th;
  for (int d = 0; d < n_dev; ++d) th.emplace_back(worker, d);
  for (auto& t : th) t.join();
  int rc = EIK_OK;
  std::string msg;
  for (const Strip& s : S)
    if (rc == EIK_OK && s.rc != EIK_OK) {
      rc = s.rc;
      msg = "device " + std::to_string(s.device) + ": " + s.msg;
    }
  if (rc == EIK_OK && out->u) {
    for (const Strip& s : S) {
      cudaSetDevice(s.device);
      const cudaError_t e = cudaMemcpy2D(out->u + s.r0 * m, sizeof(double) * m, s.row(1),
                                         sizeof(double) * s.plan->pitch, sizeof(double) * m,
                                         s.r1 - s.r0, cudaMemcpyDeviceToHost);
      if (e != cudaSuccess) {
        rc = EIK_ERR_CUDA;
        msg = std::string("gather: ") + cudaGetErrorString(e);
        break;
      }
    }
  }
  for (Strip& s : S) {
    if (s.plan) {
      cudaSetDevice(s.device);
      if (s.recv) cudaFree(s.recv);
      plan_free(s.plan);
    }
    if (s.stream) cudaStreamDestroy(s.stream);
  }
  if (rc) return fail(rc, msg);
  const int64_t M = m * n;
  out->sweeps = rounds;
  out->node_updates = rounds * (M - p->n_exit);
  out->heap_removals = 0;
  if (method == EIK_FMM) {  // the FMM row: the fixed point, fmm_solve's counters
    out->sweeps = 0;
    out->node_updates = fmm_node_updates(p->grid, p->exit_nodes, p->n_exit);
    out->heap_removals = M - p->n_exit;
  }
  out->device_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  out->rounds = rounds;
  out->grid_ctas = n_dev;
  return EIK_OK;
}

}  // namespace eikb200
