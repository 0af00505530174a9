// engine.cuh -- per-(system, precision) launcher: packs the plugin
// descriptors into kernel parameters, picks the launch shape and launches the
// templated kernels.
#pragma once
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <type_traits>
#include <utility>

#include "internal.h"
#include "finalize.cuh"
#include "rollout_fast.cuh"

namespace jm {

template <typename Real>
void fill_cartpole(const jm_model_desc& md, SysParams<Real>& sp) {
  const double mc = md.params[0], mp = md.params[1], l = md.params[2], g = md.params[3];
  sp.mp[0] = Real(mc);
  sp.mp[1] = Real(mp);
  sp.mp[2] = Real(l);
  sp.mp[3] = Real(g);
  sp.mp[4] = Real(1.0 / l);
}

template <typename Real>
void fill_quadrotor(const jm_model_desc& md, SysParams<Real>& sp) {
  const double mass = md.params[0], ixx = md.params[2], iyy = md.params[3], izz = md.params[4],
               g = md.params[5];
  sp.mp[0] = Real(1.0 / mass);
  sp.mp[1] = Real(g);
  sp.mp[2] = Real((iyy - izz) / ixx);
  sp.mp[3] = Real((izz - ixx) / iyy);
  sp.mp[4] = Real((ixx - iyy) / izz);
  sp.mp[5] = Real(1.0 / ixx);
  sp.mp[6] = Real(1.0 / iyy);
  sp.mp[7] = Real(1.0 / izz);
}

// cost weights enter as sqrt(w), sqrt(w) * target (systems.cuh)
template <typename Real>
void fill_cost(const jm_cost_desc& cd, int n, SysParams<Real>& sp) {
  for (int i = 0; i < 12; ++i) {
    sp.sw[i] = Real(0);
    sp.swt[i] = Real(0);
  }
  if (cd.kind == JM_COST_DIAG_QUADRATIC) {
    for (int i = 0; i < n; ++i) {
      const double s = std::sqrt(cd.weights[i]);
      sp.sw[i] = Real(s);
      sp.swt[i] = Real(s * cd.target[i]);
    }
  } else {
    for (int i = 0; i < 4; ++i) sp.sw[i] = Real(std::sqrt(cd.weights[i]));
    if (cd.kind == JM_COST_QUADROTOR_HOVER) {
      const double s = std::sqrt(cd.weights[0]);
      for (int i = 0; i < 3; ++i) sp.swt[i] = Real(s * cd.target[i]);
    }
  }
  sp.term_scale = Real(cd.terminal_scale);
}

template <class Dyn, class Cost, typename Real>
class Engine final : public EngineBase {
  using Sys = System<Dyn, Cost>;
  static constexpr int N = Dyn::N, M = Dyn::M;

 public:
  template <typename R>
  static void fill_sys(const jm_ctx* c, SysParams<R>& sp) {
    for (auto& v : sp.mp) v = R(0);
    if constexpr (std::is_same<Dyn, Cartpole>::value) fill_cartpole<R>(c->model, sp);
    if constexpr (std::is_same<Dyn, Quadrotor>::value) fill_quadrotor<R>(c->model, sp);
    fill_cost<R>(c->cost, N, sp);
    fill_trig(sp.tk);
    sp.ext = reinterpret_cast<const R*>(std::is_same<R, float>::value ? c->d_lin_f : c->d_lin_d);
  }

  int q_of(const jm_ctx* c) const { return c->model.jump_channel == JM_JUMP_STATE ? Dyn::QJ : M; }
  // dynamic smem of a rollout launch (kernels.cuh smem_plan)
  // (jump-mark staging: 32 lanes x W steps x q per warp; marks_warps = the warps running jump windows)
  size_t plan_bytes(const jm_ctx* c, int tile, int marks_warps, int W, int nring, bool scr) const {
    const int nmarks = c->jthr ? marks_warps * 32 * W * q_of(c) : 0;
    return smem_plan(c->TM, c->T * (2 * M + 1), tile, nmarks, nring, scr ? c->TM * tile : 0, c->gap_n,
                     (int)sizeof(Real))
        .total;
  }

  template <bool PH, bool TR, int JM>
  static const void* kfn() {
    return reinterpret_cast<const void*>(&rollout_kernel<Sys, Real, PH, TR, JM>);
  }
  // the warp-specialised kernel's shared memory (its sparse epilogue's chunk scratch included)
  size_t ws_bytes(const jm_ctx* c, int tile, int W) const {
    const int nmarks = c->jthr ? tile * W * q_of(c) : 0;
    const int chunk = ws_chunk(tile, regen_items(c->T, 4 / Pad<M>::value));
    return smem_plan(c->TM, c->T * (2 * M + 1), tile, nmarks, ws_ring(c, tile), chunk * c->TM, c->gap_n,
                     (int)sizeof(Real))
        .total;
  }

  // (the dynamic-smem attribute is per FUNCTION, shared by every context of this
  // engine type: it is raised to the device's opt-in maximum -- a bound, not a
  // reservation -- so one context's configure never shrinks another's launch)
  static cudaError_t raise_smem(const void* f, int optin) {
    cudaFuncAttributes fa{};
    cudaError_t e = cudaFuncGetAttributes(&fa, f);
    if (e != cudaSuccess) return e;
    return cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, optin - (int)fa.sharedSizeBytes);
  }
  // the TRACE kernels (rollout_kernel: per-step states for return_rollouts)
  template <int JM>
  cudaError_t set_attrs(int optin) {
    const void* fns[2] = {kfn<true, true, JM>(), kfn<false, true, JM>()};
    for (const void* f : fns) {
      cudaError_t e = raise_smem(f, optin);
      if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
  }

  // the product (non-trace) kernel, rollout_fast: SPT samples per thread
  // (2: packed f32x2, for the BASELINE systems in fp32)
  static constexpr bool kPackable = std::is_same<Real, float>::value &&
                                    (std::is_same<Dyn, Cartpole>::value || std::is_same<Dyn, Quadrotor>::value);
  // (QUAD: the eps'eps term of the modified cost is formed -- c != 1, the general
  // channel, or fed noise, whose non-finite values must still poison the cost)
  // (LDIAG: diagonal-Cholesky form, instantiated where it pays -- packed Philox kernels, m > 1)
  #ifdef JM_NO_LDIAG
  static constexpr bool kDiagForm = false;
#else
  static constexpr bool kDiagForm = kPackable && M > 1;
#endif
  template <bool PH, int JM, int SPT, bool QUAD, bool LDIAG = false>
  static auto fast_kern() {
    if constexpr (SPT == 2 && kPackable)
      return &rollout_fast<Sys, Real, PH, JM, 2, kPackedThreads, QUAD, LDIAG && PH && kDiagForm>;
    else
      return &rollout_fast<Sys, Real, PH, JM, 1, 512, QUAD>;
  }
  template <bool PH, int JM, int SPT>
  static const void* fast_fn_q(bool quad, bool ldiag = false) {
    if constexpr (PH && SPT == 2 && kDiagForm) {
      if (ldiag)
        return quad ? reinterpret_cast<const void*>(fast_kern<PH, JM, SPT, true, true>())
                    : reinterpret_cast<const void*>(fast_kern<PH, JM, SPT, false, true>());
    }
    return quad ? reinterpret_cast<const void*>(fast_kern<PH, JM, SPT, true>())
                : reinterpret_cast<const void*>(fast_kern<PH, JM, SPT, false>());
  }
  // the diffusion factor's strict lower triangle is all zero
  static bool ld_diag(const jm_ctx* c) {
    for (int i = 0; i < M; ++i)
      for (int j = 0; j < i; ++j)
        if (c->Ld[i * M + j] != 0.0) return false;
    return true;
  }
  static const void* fast_fn_rt(bool ph, int jm, int spt, bool quad, bool ldiag) {
    if (ph) {
      if (jm) return spt == 2 ? fast_fn_q<true, 1, 2>(quad, ldiag) : fast_fn_q<true, 1, 1>(quad);
      return spt == 2 ? fast_fn_q<true, 0, 2>(quad, ldiag) : fast_fn_q<true, 0, 1>(quad);
    }
    if (jm) return spt == 2 ? fast_fn_q<false, 1, 2>(true) : fast_fn_q<false, 1, 1>(true);
    return spt == 2 ? fast_fn_q<false, 0, 2>(true) : fast_fn_q<false, 0, 1>(true);
  }
  static bool fast_quad(const jm_ctx* c) {
    return c->mppi.noise_source != JM_NOISE_PHILOX || c->cost.general_channel || c->cost.c != 1.0;
  }
  // steps per regeneration item (kernel GS) and the fast kernel's shared memory
  int fast_gs(bool philox) const { return philox ? 4 / Pad<M>::value : (M >= 3 ? 1 : 4); }
  size_t fast_bytes(const jm_ctx* c, int tile, int spt, int W, bool philox) const {
    const int nb = regen_items(c->T, fast_gs(philox));
    const size_t mbytes = (philox && c->jthr) ? fast_marks_bytes(tile, tile / spt / 32, W, q_of(c), (int)sizeof(Real)) : 0;
    return fast_plan(c->TM, c->T * (2 * M + 1), tile, tile / spt, nb, mbytes, c->gap_n, (int)sizeof(Real)).total;
  }

  // warp-specialised kernel (Philox, non-trace): block = 2 x tile
  static constexpr int kWsMaxThreads = (N <= 4) ? 1024 : 512;
  static constexpr int kWsBufs = 6;  // ring depth: slack for the producers' jump-window bursts
  template <int JM>
  static auto ws_kern() {
    return &rollout_kernel_ws<Sys, Real, JM, kWsMaxThreads, kWsBufs>;
  }
  int ws_ring(const jm_ctx* c, int tile) const {
    const int gw = (c->model.jump_channel == JM_JUMP_STATE) ? WsShape<Sys, 1>::GW : WsShape<Sys, 0>::GW;
    return kWsBufs * gw * tile;
  }

  // Launch shape.  K <= num_sms * 512: one CTA per SM, every SM gets the
  // same sample count (a latency-bound horizon loop gains nothing from
  // stacking CTAs on few SMs).  Larger K: 256-sample tiles, grid = SMs x
  // occupancy, tiles grid-strided.  Philox path, single wave: the per-CTA
  // eps scratch the epilogue reads is kept in shared memory when it fits, and
  // tiles of <= kWsMaxTile samples run the warp-specialised kernel (measured:
  // it wins only where a few warps per SM leave the issue slots idle).
  // (measured: cartpole tiles of 128 run 20.9 us without WS vs 26.3 with it, 64 tie;
  // the quadrotor's longer chain still wins with WS at 128: 79.6 vs 83.8 us)
  static constexpr int kWsMaxTile = (N <= 4) ? 64 : 128;
  cudaError_t configure(jm_ctx* c) override {
    const bool philox = c->mppi.noise_source == JM_NOISE_PHILOX;
    static const int ws_env = std::getenv("JM_WS") ? std::atoi(std::getenv("JM_WS")) : -1;  // A/B: 0 off, 1 on
    static const int spt_env = std::getenv("JM_SPT") ? std::atoi(std::getenv("JM_SPT")) : 0;  // A/B: 1 or 2
    int block = c->mppi.block_threads;
    const int K = c->K, sms = c->num_sms;
    // samples per thread of the product kernel: packed pairs need an even K
    // (adjacent HBM columns) and tiles of whole 64-sample warp pairs
    // default (measured, DESIGN 6): pairs where the kernel is issue-bound (multi-wave, HBM
    // mode); one sample per thread in the latency-bound single wave (more warps in flight)
    const bool want2 = spt_env ? spt_env == 2 : (!philox || K > sms * kRolloutMaxThreads);
    int spt = (kPackable && want2 && K % 2 == 0 && (block <= 0 || block % 64 == 0)) ? 2 : 1;
    if (block <= 0) {
      if (K <= sms * kRolloutMaxThreads) {
        const int per = (K + sms - 1) / sms;
        block = std::max(32 * spt, ((per + 32 * spt - 1) / (32 * spt)) * (32 * spt));
      } else {
        block = (spt == 2 ? kPackedThreads : 256) * spt;
      }
    }
    const bool ws = philox && 2 * block <= kWsMaxThreads && (ws_env < 0 ? block <= kWsMaxTile : ws_env == 1);
    c->block = block;
    c->ws = ws;
    const int threads = ws ? 2 * block : block;
    const int nring = ws ? ws_ring(c, block) : 0;
    const int mwarps = block / 32;  // warps running jump windows (the producers under WS)
    int optin = 0;
    cudaError_t e = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, c->device);
    if (e != cudaSuccess) return e;
    c->ntiles = (K + block - 1) / block;
    // jump window: the longest (fewer window passes) whose staging fits
    // (128-bit event masks: windows up to 128 steps); single wave: the whole SM,
    // multi-wave: two CTAs per SM must still fit (the occupancy 256-thread tiles need)
    const size_t cap = (size_t)optin - 2048;  // (static shared memory of the rollout kernels: < 2 KB)
    const size_t cap_ws = (size_t)optin - 8192;  // (the WS kernel's static regeneration list: up to 6 KB)
    const size_t budget = ws ? cap_ws : (c->ntiles <= sms ? cap : std::min(cap, (size_t)optin / 2 - 2048));
    int W = std::min(128, (c->T + 3) / 4 * 4);
    while (W > 8 && (ws ? ws_bytes(c, block, W) : plan_bytes(c, block, mwarps, W, 0, false)) > budget) W -= 4;
    c->jw_len = W;
    c->eps_smem = 0;
    const size_t msmem = ws ? ws_bytes(c, block, W) : 0;              // the warp-specialised kernel
    const size_t smem = plan_bytes(c, block, mwarps, W, 0, false);  // trace kernels
    const bool fast = !ws;  // the product kernel (Philox without warp specialisation, and HBM)
    c->fast = fast;
    c->spt = spt;
    size_t fsmem = 0;
    int WF = 0;
    if (fast) {
      // multi-wave: two CTAs per SM must fit; single wave: the whole SM
      const size_t fbudget = (c->ntiles <= sms) ? cap : std::min(cap, (size_t)optin / 2 - 2048);
      WF = std::min(128, (c->T + 3) / 4 * 4);
      // (JM_JW_NOCAP=1, tests: windows as long as the memory allows whatever the rate, so a warp's
      // window overflows its mark table and the halve-and-redo path runs)
      static const bool jw_nocap = std::getenv("JM_JW_NOCAP") != nullptr && std::atoi(std::getenv("JM_JW_NOCAP")) != 0;
      if (philox && c->jthr && marks_indexed(q_of(c)) && !jw_nocap) WF = std::min(WF, marks_window_cap(c->jthr, spt));
      static const int jw_env = std::getenv("JM_JW") ? std::atoi(std::getenv("JM_JW")) : 0;  // A/B: window length
      if (jw_env >= 4) WF = std::min(WF, jw_env / 4 * 4);
      while (WF > 8 && fast_bytes(c, block, spt, WF, philox) > fbudget) WF -= 4;
      (void)budget;
      fsmem = fast_bytes(c, block, spt, WF, philox);
      if (fsmem > cap) return cudaErrorInvalidConfiguration;
    }
    c->jw_fast = WF;
    c->fast_smem = fsmem;
    const void* fn = nullptr;
    const bool sj = c->model.jump_channel == JM_JUMP_STATE;
    e = sj ? set_attrs<1>(optin) : set_attrs<0>(optin);
    if (e != cudaSuccess) return e;
    if (ws) fn = sj ? reinterpret_cast<const void*>(ws_kern<1>()) : reinterpret_cast<const void*>(ws_kern<0>());
    if (fast) fn = fast_fn_rt(philox, sj ? 1 : 0, spt, fast_quad(c), ld_diag(c));
    e = raise_smem(fn, optin);
    if (e != cudaSuccess) return e;
    int occ = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, fast ? block / spt : threads, fast ? fsmem : msmem);
    if (e != cudaSuccess) return e;
    if (occ < 1) return cudaErrorInvalidConfiguration;
    c->smem = smem;
    c->main_smem = msmem;
    c->grid = std::min(c->ntiles, occ * sms);
    // the non-trace kernel this context launches (jm_kernel_name; ncu -k regex:rollout_kernel)
    c->variant = std::string(ws ? "rollout_kernel_ws" : "rollout_fast") + "/" + (philox ? "philox" : "hbm") + "/" +
                 (ws ? "ws" : (c->ntiles <= sms ? "single_wave" : "multi_wave")) + "/" +
                 (sizeof(Real) == 4 ? "f32" : "f64") + (fast ? "/spt" + std::to_string(spt) : "");
    if (c->grid > kMaxRecords) c->grid = kMaxRecords;
    const size_t fsm = finalize_smem_bytes(kMaxRecords);
    return cudaFuncSetAttribute(reinterpret_cast<const void*>(&finalize_kernel<Dyn>),
                                cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fsm);
  }

  RolloutArgs<Real> make_args(const jm_ctx* c, const RolloutCall& rc) const {
    RolloutArgs<Real> a{};
    const double dt = c->mppi.dt, lam = c->cost.lambda_, cc = c->cost.c;
    a.K = c->K;
    a.T = c->T;
    a.TM = c->TM;
    a.ntiles = c->ntiles;
    a.sample_offset = c->mppi.sample_offset;
    a.dt = Real(dt);
    a.sdt = Real(std::sqrt(dt));
    a.inv_lam = Real(1.0 / c->mppi.lambda_);  // weights use cfg.lambda_ (controller.py:157)
    a.cq = Real(0.5 * lam * (1.0 - 1.0 / cc));  // costs.py:519 times dt/dt
    a.lam_sdt = Real(lam * std::sqrt(dt));       // lambda u eps / sqrt(dt) * dt
    for (int i = 0; i < 16; ++i) {
      a.R[i] = Real(c->cost.R[i]);
      a.calb[i] = Real(c->cost.cal_b[i]);
      a.bb[i] = Real(c->cost.bb[i]);
      a.Ld[i] = Real(c->Ld[i]);
      a.Lj[i] = Real(c->Lj[i]);
    }
    for (int j = 0; j < 4; ++j) {
      a.u_lo[j] = Real(c->model.u_lo[j]);
      a.u_hi[j] = Real(c->model.u_hi[j]);
      a.mu_j[j] = Real(c->mppi.mark_mean[j]);
    }
    a.has_limits = c->model.has_limits;
    a.general = c->cost.general_channel;
    a.jump_on = c->jthr != 0;
    a.gap_thr = c->d_gap;
    a.gap_n = c->gap_n;
    a.gap_inv = c->gap_inv;
    a.poisson = c->poisson;
    a.cnt = c->cnt;
    a.jw_len = c->jw_len;
    a.jscale = Real(c->model.jump_scale_unit ? 1.0 : std::sqrt(dt));
    fill_sys<Real>(c, a.sp);
    for (int i = 0; i < kMaxSeeds; ++i) a.seeds[i] = (rc.seeds && i < rc.nseeds) ? rc.seeds[i] : rc.seed;
    a.iteration = rc.iteration;
    a.iteration_dev = rc.iteration_dev;
    a.x0 = rc.x0;
    a.u_nom = rc.u_nom;
    a.eps_in = reinterpret_cast<const Real*>(rc.eps_in);
    a.jump_in = reinterpret_cast<const Real*>(rc.jump_in);
    a.eps_out = reinterpret_cast<Real*>(c->d_scratch);
    a.eps_smem = c->eps_smem;
    a.costs = rc.costs;
    a.costs_dev = rc.costs_dev;
    a.states = rc.states;
    a.diverged = rc.diverged;
    a.records = c->d_records;
    a.rec_stride = c->rec_stride;
    a.loop = rc.loop;
    a.push_peers = rc.push_peers;
    a.push_rank = rc.push_rank;
    a.push_world = rc.push_world;
    return a;
  }

  template <typename... KArgs, typename... Args>
  static cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                                Args&&... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    static const bool no_pdl = std::getenv("JM_NO_PDL") != nullptr;  // debugging switch
    cfg.attrs = attr;
    cfg.numAttrs = no_pdl ? 0 : 1;
    return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
  }

  template <bool PH, int JM, int SPT>
  cudaError_t launch_fast(jm_ctx* c, const RolloutArgs<Real>& a) {
    RolloutArgs<Real> b = a;
    b.jw_len = c->jw_fast;
    dim3 grid(c->grid, c->launch_trials), block(c->block / SPT);
    if constexpr (PH && SPT == 2 && kDiagForm) {
      if (ld_diag(c)) {
        if (fast_quad(c))
          return launch_pdl(fast_kern<PH, JM, SPT, true, true>(), grid, block, c->fast_smem, c->stream, b);
        return launch_pdl(fast_kern<PH, JM, SPT, false, true>(), grid, block, c->fast_smem, c->stream, b);
      }
    }
    if (fast_quad(c)) return launch_pdl(fast_kern<PH, JM, SPT, true>(), grid, block, c->fast_smem, c->stream, b);
    if constexpr (PH) return launch_pdl(fast_kern<PH, JM, SPT, false>(), grid, block, c->fast_smem, c->stream, b);
    return cudaErrorInvalidValue;
  }

  template <int JM>
  cudaError_t launch(jm_ctx* c, const RolloutArgs<Real>& a, bool philox, bool trace) {
    dim3 grid(c->grid, c->launch_trials), block(c->block);
    if (!trace && c->fast) {
      if (philox) return c->spt == 2 ? launch_fast<true, JM, 2>(c, a) : launch_fast<true, JM, 1>(c, a);
      return c->spt == 2 ? launch_fast<false, JM, 2>(c, a) : launch_fast<false, JM, 1>(c, a);
    }
    if (philox && !trace && c->ws)
      return launch_pdl(ws_kern<JM>(), grid, dim3(2 * c->block), c->main_smem, c->stream, a);
    if (!trace) return cudaErrorInvalidValue;  // (every non-trace launch is fast or WS)
    RolloutArgs<Real> b = a;
    b.eps_smem = 0;
    if (philox) return launch_pdl(rollout_kernel<Sys, Real, true, true, JM>, grid, block, c->smem, c->stream, b);
    return launch_pdl(rollout_kernel<Sys, Real, false, true, JM>, grid, block, c->smem, c->stream, b);
  }

  cudaError_t rollout(jm_ctx* c, const RolloutCall& rc) override {
    const RolloutArgs<Real> a = make_args(c, rc);
    const bool philox = c->mppi.noise_source == JM_NOISE_PHILOX;
    const bool trace = rc.states != nullptr;
    if (c->model.jump_channel == JM_JUMP_STATE) return launch<1>(c, a, philox, trace);
    return launch<0>(c, a, philox, trace);
  }

  cudaError_t noise(jm_ctx* c, NoiseArgs& na) override {
    const int block = 128;
    const int grid = (c->K + block - 1) / block;
    if (c->model.jump_channel == JM_JUMP_STATE)
      noise_kernel<M, 1, Dyn::QJ, Real><<<grid, block, 0, c->stream>>>(na);
    else
      noise_kernel<M, 0, Dyn::QJ, Real><<<grid, block, 0, c->stream>>>(na);
    return cudaGetLastError();
  }

  PlantArgs plant_args(const jm_ctx* c, LoopState* loop, const double* u_new, double* u_nom) const {
    PlantArgs p{};
    fill_sys<double>(c, p.sp);
    const double dt = c->mppi.dt;
    p.dt = dt;
    p.sdt = std::sqrt(dt);
    p.jscale = c->model.jump_scale_unit ? 1.0 : std::sqrt(dt);
    for (int i = 0; i < 16; ++i) {
      p.Lp[i] = c->Lp[i];
      p.Lj[i] = c->Lj[i];
    }
    for (int j = 0; j < 4; ++j) {
      p.mu_j[j] = c->mppi.mark_mean[j];
      p.u_lo[j] = c->model.u_lo[j];
      p.u_hi[j] = c->model.u_hi[j];
    }
    p.jthr = c->jthr_plant;
    p.poisson = c->poisson;
    for (int i = 0; i <= kMaxCount; ++i) p.cnt0[i] = c->cnt_plant[i];
    p.q = c->Q;
    p.jmode = c->model.jump_channel;
    p.has_limits = c->model.has_limits;
    p.T = c->T;
    p.M = M;
    p.loop = loop;
    p.u_new = u_new;
    p.u_nom = u_nom;
    return p;
  }

  cudaError_t finalize(jm_ctx* c, FinArgs f, LoopState* loop, double* u_nom_next) override {
    if (f.nrec > kMaxRecords) return cudaErrorInvalidValue;
    f.loop = loop;
    if (!f.counter) f.counter = c->d_counter;
    const PlantArgs p = plant_args(c, loop, f.u_new, u_nom_next);
    // the column-parallel finalize wherever no cross-GPU exchange is involved
    static const bool no_cols = std::getenv("JM_FIN_ONE_CTA") != nullptr;  // A/B: the one-CTA merge
    if (!no_cols && f.rec_out == nullptr && f.push_peers == nullptr && (f.wait_flags == nullptr || f.wait_gpu)) {
      f.cols = fincol_width(M);
      const int g = (c->TM + f.cols - 1) / f.cols;
      // a plain launch, not a programmatic dependent one: resident early beside the
      // rollout's CTAs, the finalize's CTAs measured 0.5 us slower per cfg1 step
      // (tools/ab1.sh; JM_FIN_PDL=1 restores the early launch)
      static const bool fin_pdl = std::getenv("JM_FIN_PDL") != nullptr;
      if (!fin_pdl) {
        finalize_cols<Dyn><<<dim3(g, c->launch_trials), dim3(fincol_threads(f.nrec)), 0, c->stream>>>(f, p);
        return cudaGetLastError();
      }
      return launch_pdl(finalize_cols<Dyn>, dim3(g, c->launch_trials), dim3(fincol_threads(f.nrec)), 0, c->stream,
                        f, p);
    }
    f.cols = fin_cols(M);
    const int fgrid = (c->TM + f.cols - 1) / f.cols;
    return launch_pdl(finalize_kernel<Dyn>, dim3(fgrid, c->launch_trials), dim3(kFinThreads), finalize_smem_bytes(f.nrec), c->stream,
                      f, p);
  }

};

}  // namespace jm
