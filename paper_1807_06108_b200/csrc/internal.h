// internal.h -- context object shared by the C-ABI host code and the
// per-system engines.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

#include "../../include/jmppi.h"
#include "kernels.cuh"

namespace jm {

struct RolloutCall {
  const double* x0 = nullptr;
  const double* u_nom = nullptr;
  uint64_t seed = 0, iteration = 0;
  const uint64_t* seeds = nullptr;  // batched trials: one master seed per grid.y slice (nseeds <= kMaxSeeds)
  int nseeds = 0;
  const uint64_t* iteration_dev = nullptr;
  double* const* costs_dev = nullptr;
  const void* eps_in = nullptr;
  const void* jump_in = nullptr;
  double* costs = nullptr;
  double* states = nullptr;
  int64_t* diverged = nullptr;
  LoopState* loop = nullptr;
  const unsigned long long* push_peers = nullptr;  // peer-memory exchange (write_record)
  int push_rank = 0, push_world = 0;
};

struct EngineBase {
  virtual ~EngineBase() = default;
  // occupancy-derived launch shape; sets ctx->grid/ntiles/smem
  virtual cudaError_t configure(jm_ctx* c) = 0;
  virtual cudaError_t rollout(jm_ctx* c, const RolloutCall& rc) = 0;
  virtual cudaError_t noise(jm_ctx* c, NoiseArgs& na) = 0;
  // combine records -> u_new (+ diagnostics); loop != null: the last CTA also
  // runs the plant step and writes the shifted sequence to u_nom_next
  virtual cudaError_t finalize(jm_ctx* c, FinArgs f, LoopState* loop, double* u_nom_next) = 0;
};

EngineBase* make_engine_integrator(int cost_kind, int precision, int n);
EngineBase* make_engine_cartpole(int cost_kind, int precision);
EngineBase* make_engine_quadrotor(int cost_kind, int precision);
EngineBase* make_engine_linear(int cost_kind, int precision, int n, int m);

}  // namespace jm

struct jm_ctx {
  jm_model_desc model{};
  jm_cost_desc cost{};
  jm_mppi_desc mppi{};
  int device = 0;
  int num_sms = 148;
  cudaStream_t stream = nullptr;
  cudaStream_t own_stream = nullptr;
  int N = 0, M = 0, Q = 0, T = 0, K = 0, TM = 0, rec_stride = 0;
  int block = 128, grid = 1, ntiles = 1;
  int ws = 0;              // warp-specialised Philox rollout: block of 2*block threads
  int eps_smem = 0;        // Philox main kernel keeps the eps scratch in shared memory
  int fast = 0;            // non-trace launches use rollout_fast (rollout_fast.cuh)
  int spt = 1;             // rollout_fast: samples per thread (2 = packed f32x2)
  int jw_fast = 0;         // rollout_fast: jump window (steps)
  size_t fast_smem = 0;    // rollout_fast: dynamic shared memory
  size_t main_smem = 0;    // dynamic smem of the Philox main kernel
  size_t smem = 0;
  size_t real_size = 4;
  double Ld[16] = {0}, Lj[16] = {0}, Lp[16] = {0};  // chol(c Sigma_D), chol(Sigma_J), chol(Sigma_D)
  uint32_t jthr = 0;      // sampler jump threshold (0 = no jumps)
  uint32_t jthr_plant = 0;
  int poisson = 0;            // jm_jump_process == JM_JUMPS_POISSON
  jm::CountTable cnt{};         // zero-truncated count thresholds (philox.cuh slot 4)
  uint32_t cnt_plant[jm::kMaxCount + 1] = {};  // plant: n = #{k : u24 < cnt_plant[k]}
  uint32_t* d_gap = nullptr;  // jump-gap survival table (philox.cuh), gap_n = T + 1 entries
  int gap_n = 0;
  int jw_slab = 0;             // jump window of the slab-staged (single-wave, non-WS) rollout
  float gap_inv = 0.f;        // 1 / log2(1 - p)
  int jw_len = 32;            // jump window of the rollout kernels (steps)
  jm::EngineBase* eng = nullptr;
  // device workspace
  void* d_scratch = nullptr;      // per-CTA eps_combined slabs (Philox mode)
  void* d_hbm_eps = nullptr;      // HBM-mode input staging (host API)
  void* d_hbm_jump = nullptr;
  double* d_costs = nullptr;      // K
  double* d_weights = nullptr;    // K
  double* d_wsum = nullptr;       // weight normaliser block sums
  double* d_records = nullptr;    // grid * rec_stride
  double* d_small = nullptr;      // x0 | u_nom | u_new | norms | mapping | u_init | record
  double* h_big = nullptr;        // pinned 2K doubles: costs | weights
  double* d_states = nullptr;     // trace
  int64_t* d_div = nullptr;
  size_t states_cap = 0;
  // pinned staging for the host API
  double* h_small = nullptr;
  jm::DiagOut* d_diag() const { return reinterpret_cast<jm::DiagOut*>(d_small + off_diag()); }
  int32_t* d_status() const { return reinterpret_cast<int32_t*>(d_small + off_status()); }
  // closed loop
  jm::LoopState* d_loop = nullptr;
  double* d_loop_unom = nullptr;
  double* d_loop_unew = nullptr;
  // single-GPU closed loop: the CTA records travel through the same epoch-flag
  // buffer as the multi-GPU exchange (world 1), so the finalize merges them as
  // the rollout's CTAs finish instead of after the whole grid
  double* d_self_push = nullptr;                 // jm_peer_buffer_doubles(ctx, 1)
  unsigned long long* d_self_base = nullptr;     // {d_self_push}
  double* d_hist = nullptr;       // states | controls
  int64_t* d_hist_jumps = nullptr;
  uint64_t* d_hist_t = nullptr;   // t_start | t_end
  uint64_t* d_tl = nullptr;       // tuning timeline (JM_TIMELINE=1): loop_cap x kTlSlots stamps
  int loop_cap = 0;
  int launch_trials = 1;  // grid.y of the rollout / finalize launches (batched trials)
  void* d_lin_f = nullptr;  // Linear model: [A | G] as float (rollout in fp32)
  void* d_lin_d = nullptr;  //               and as double (fp64 rollout, the plant)
  unsigned int* d_counter = nullptr;  // finalize last-CTA counter
  std::vector<double*> stash;        // device weight buffers (K doubles)
  std::vector<int> stash_free;
  void* d_flush = nullptr;         // L2 flush buffer (bench)
  size_t flush_cap = 0;
  cudaGraph_t graph = nullptr;
  // graphs of one drop-in iteration (H2D..D2H), one per master seed (the seed is a
  // kernel parameter), most recent last
  std::vector<std::pair<uint64_t, cudaGraphExec_t>> iter_execs;
  uint64_t loop_seed = 0;  // master seed the loop graph was captured with
  cudaGraphExec_t graph_exec = nullptr;
  std::string err;
  std::string variant;  // rollout kernel variant the launcher picked (jm_kernel_name)

  // d_small / h_small layout (doubles):
  //   inputs  [x0:16][u_nom:TM][mapping:16][u_init:16]   (x0 slots 13..15 of
  //           the graph path: stash pointer, seed, iteration as raw 64-bit words)
  //   outputs [u_new:TM][norms:T][diag:4][status:2][u_shift:TM]
  //   [record:rec_stride]  (this context's reduced record)
  size_t off_x0() const { return 0; }
  size_t off_unom() const { return 16; }
  size_t off_map() const { return 16 + (size_t)TM; }
  size_t off_uinit() const { return off_map() + 16; }
  size_t off_unew() const { return off_uinit() + 16; }
  size_t off_norms() const { return off_unew() + (size_t)TM; }
  size_t off_diag() const { return off_norms() + (size_t)T; }
  size_t off_status() const { return off_diag() + 4; }
  size_t off_ushift() const { return off_status() + 2; }
  size_t off_rec() const { return off_ushift() + (size_t)TM; }
  size_t small_doubles() const { return off_rec() + (size_t)rec_stride; }
};
