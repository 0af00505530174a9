// kernels.cuh -- the sm_100a kernels of one MPC iteration.
//
//   rollout_kernel   K1 (in-register Philox noise, or the HBM wire-format
//                    reader) + K2 fused rollout/modified cost + the per-CTA
//                    half of K3/K4 (online-softmax partials: rho, Z, sum w^2,
//                    N[t,j] = sum_k w_k eps[k,t,j]).  Reference:
//                    controller.py:118-158, noise.py:129-161,
//                    dynamics.py:87-135, costs.py:80-111.
//   finalize_kernel  K3/K4/K5 across CTAs (or across GPUs): log-sum-exp merge
//                    of the partial records, u_new = u_nom + N/(Z sqrt dt)
//                    (@ mapping^T), diagnostics (controller.py:62-78,
//                    :157-169); in the closed loop its last CTA also runs K7,
//                    the plant step + warm-start shift (harness.py:131-150).
//   noise_kernel     K1 in write mode (sample_noise_batch on device).
//   weights_*_kernel / shift_kernel (api.cu only): controller.py:62-71, :96-100.
// All reductions are fixed-order (no float atomics): results are bitwise
// reproducible run to run for a given launch configuration, and the noise is
// independent of it.
#pragma once
#include <cuda_runtime.h>
#include <math_constants.h>

#include <cstdint>
#include <type_traits>

#include "philox.cuh"
#include "systems.cuh"

namespace jm {

constexpr int kFinCols = 128;      // finalize: column capacity of a CTA; it owns fin_cols(m) <= 128 of them
// columns per finalize CTA: a multiple of m, so a CTA holds whole steps (mapping rows, per-step norms)
__host__ __device__ __forceinline__ int fin_cols(int m) { return (kFinCols / m) * m; }
#ifndef JM_FIN_THREADS
#define JM_FIN_THREADS 1024
#endif
constexpr int kFinThreads = JM_FIN_THREADS;  // finalize: its warps split the records
constexpr int kMaxRecords = 4096;
constexpr int kRolloutMaxThreads = 512;
// Master seeds travel in the kernel parameters, one per grid.y slice (batched
// trials), indexed by the CTA-uniform blockIdx.y: the Philox round keys
// (seed + r * golden-ratio constants) then live in uniform registers, computed
// once per kernel, and the rounds' key XORs read them as uniform operands --
// no per-thread key schedule in the hot loop.
constexpr int kMaxSeeds = 128;

// Device-resident closed-loop controller state (ControllerState +
// the plant state of run_trial).
struct LoopState {
  double x[12];            // plant state
  double u_init[4];        // MppiConfig.u_init
  uint64_t seed;           // master_seed
  uint64_t iteration;      // ControllerState.iteration_index (RNG stream id)
  int32_t step;            // control step k
  int32_t max_steps;
  int32_t halted;          // 1 after divergence / no viable rollout / max_steps
  int32_t status;          // jm_status
  int32_t diverged_at;     // step index or -1
  int32_t sampler_jumps;   // the controller's sampler draws jumps ("new" variant; "old": 0, harness.py:218-221)
  // history buffers (device)
  double* hist_states;     // (max_steps+1) * n
  double* hist_controls;   // max_steps * m
  int64_t* hist_jumps;     // max_steps
  uint64_t* t_start;       // max_steps, %globaltimer ns
  uint64_t* t_end;         // max_steps
  uint64_t* tl;            // tuning timeline (JM_TIMELINE=1): kTlSlots %globaltimer stamps per step, or null
  double* unom;            // nominal sequences, 2 x T*m: step k reads parity k & 1 and the finalize writes
                           // the warm-started (shifted) sequence for step k + 1 into the other parity, so
                           // no finalize CTA overwrites columns another CTA has yet to read
};

// the nominal sequence a closed-loop step reads (parity = step & 1) / writes for the next step
__device__ __forceinline__ double* loop_unom(const LoopState* L, int step, int TM) {
  return L->unom + (size_t)(step & 1) * TM;
}

// Timeline slots of one control step (jm_loop_timeline; tuning only, off unless
// JM_TIMELINE is set when the loop is initialised)
enum : int {
  kTlRollEntry = 0,    // rollout CTA 0 entry (before the grid dependency wait)
  kTlRollWait = 1,     // rollout CTA 0 past the wait
  kTlRollHorizon = 2,  // rollout CTA 0 after the prologue (first step about to run)
  kTlRollHorizonEndMin = 3,  // first CTA to finish its horizon
  kTlRollHorizonEndMax = 4,  // last CTA to finish its horizon
  kTlRollEndMax = 5,   // last CTA to write its record
  kTlFinEntry = 6,     // finalize CTA 0 entry
  kTlFinWait = 7,      // finalize CTA 0 past the wait
  kTlFinMerged = 8,    // finalize CTA 0: update computed (before the plant)
  kTlFinEnd = 9,       // finalize: plant + shift done
  kTlSlots = 12
};
struct DiagOut {
  double min_cost, ess, normaliser;
  int64_t n_finite;
};

__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// a step's stamp row (null when the timeline is off), read once by the stamping thread
__device__ __forceinline__ unsigned long long* tl_row(const LoopState* L, int step) {
  return (L != nullptr && L->tl != nullptr) ? reinterpret_cast<unsigned long long*>(L->tl) + (size_t)step * kTlSlots
                                            : nullptr;
}
__device__ __forceinline__ void tl_put(unsigned long long* row, int slot, uint64_t t) {
  if (row != nullptr) row[slot] = t;
}
__device__ __forceinline__ void tl_put(unsigned long long* row, int slot) { tl_put(row, slot, globaltimer()); }
__device__ __forceinline__ void tl_max(unsigned long long* row, int slot) {
  if (row != nullptr) atomicMax(row + slot, (unsigned long long)globaltimer());
}

// Programmatic dependent launch (sm_90+): a kernel launched with
// cudaLaunchAttributeProgrammaticStreamSerialization may start while its
// predecessor runs; grid_dep_wait() blocks until the predecessor grid has
// completed and its writes are visible.
__device__ __forceinline__ void grid_dep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void grid_dep_launch() { asm volatile("griddepcontrol.launch_dependents;" :::); }

// System-scope acquire / release on the 32-bit epoch flags of the peer-memory
// record exchange (peers write them over NVLink).
__device__ __forceinline__ uint32_t ld_acquire_sys(const unsigned int* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(unsigned int* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// GPU scope: the single-GPU (world 1) use of the same exchange -- a system-scope
// fence per CTA costs microseconds the record hand-off does not need there
__device__ __forceinline__ uint32_t ld_acquire_gpu(const unsigned int* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_gpu(unsigned int* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
  return v;
}
template <typename T>
__device__ __forceinline__ T warp_min(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(0xFFFFFFFFu, v, o));
  return v;
}

// exact warp minimum of doubles (no NaNs) on the integer reduction unit: an
// order-preserving 64-bit key, min of the high words, then of the low words
// among the lanes holding that high word -- two REDUX instead of five rounds of
// 64-bit shuffles
__device__ __forceinline__ double warp_min_redux(double v) {
  unsigned long long b = (unsigned long long)__double_as_longlong(v);
  b ^= (b >> 63) ? ~0ull : (1ull << 63);
  const uint32_t hi = (uint32_t)(b >> 32), lo = (uint32_t)b;
  const uint32_t mh = __reduce_min_sync(0xFFFFFFFFu, hi);
  const uint32_t ml = __reduce_min_sync(0xFFFFFFFFu, hi == mh ? lo : 0xFFFFFFFFu);
  unsigned long long k = ((unsigned long long)mh << 32) | ml;
  k ^= (k >> 63) ? (1ull << 63) : ~0ull;
  return __longlong_as_double((long long)k);
}

template <typename Real>
__device__ __forceinline__ Real r_inf();
template <>
__device__ __forceinline__ float r_inf<float>() { return CUDART_INF_F; }
template <>
__device__ __forceinline__ double r_inf<double>() { return CUDART_INF; }

template <typename Real>
__device__ __forceinline__ Real r_exp(Real v);
template <>
__device__ __forceinline__ float r_exp<float>(float v) { return expf(v); }
template <>
__device__ __forceinline__ double r_exp<double>(double v) { return exp(v); }

template <typename Real>
struct RolloutArgs {
  int K, T, TM, ntiles;
  long long sample_offset;
  Real dt, sdt, inv_lam, cq, lam_sdt;  // cq = 0.5*lam*(1-1/c); lam_sdt = lam*sqrt(dt)
  Real R[16];
  int general;      // CostModel.control_channel == False: cal_b in the step table, eps' bb eps per step
  Real calb[16];    // m x m row-major (costs.py:112-124)
  Real bb[16];
  Real u_lo[4], u_hi[4];
  int has_limits;
  int jump_on;      // sampler draws jumps (jump_sampling_enabled && nu > 0)
  const uint32_t* gap_thr;  // jump-gap survival table (philox.cuh), gap_n = T + 1 entries
  int gap_n;
  float gap_inv;    // 1 / log2(1 - p)
  int poisson;      // jump_process = poisson: an event carries n >= 1 arrivals (philox.cuh slot 4)
  CountTable cnt;
  int jw_len;       // jump window (steps, multiple of 4 in [8, 32])
  Real jscale;      // state-jump scale (1 or sqrt dt)
  Real Ld[16];      // chol(c * Sigma_D), m x m row-major
  Real Lj[16];      // chol(Sigma_J), q x q row-major
  Real mu_j[4];     // mark mean
  SysParams<Real> sp;
  uint64_t iteration;
  const uint64_t* iteration_dev;  // graph-replayed drop-in call: iteration staged in device memory
  uint64_t seeds[kMaxSeeds];      // master seed of grid.y slice b (batched trials; [0] otherwise)
  const double* x0;
  const double* u_nom;
  const Real* eps_in;    // HBM mode: step-major eps_combined
  const Real* jump_in;   // HBM mode, state jumps: step-major ind*mark
  Real* eps_out;         // Philox mode: per-CTA eps_combined scratch [cta][t*m+j][lane]
  int eps_smem;          // Philox, single wave: the scratch lives in shared memory instead
  double* costs;         // K
  double* const* costs_dev;  // graph-replayed drop-in call: costs go to the buffer named in device memory
  double* states;        // trace: K*(T+1)*n
  int64_t* diverged;     // trace: K
  double* records;       // gridDim.x * rec_stride
  int rec_stride;
  LoopState* loop;
  // peer-memory exchange (jm_loop_rollout_push): the CTA's record goes straight
  // into every rank's symmetric buffer instead of `records`
  const unsigned long long* push_peers;
  int push_rank, push_world;
};

// ---------------------------------------------------------------- noise
// Diffusion normals of one 4-step group for sample kg: z[s*MP + j] for step
// t0+s (normal index i = t*MP + j, Philox block i>>2, lane i&3).
template <int MP>
__device__ __forceinline__ void group_normals(const StreamKey& sk, uint32_t t0, uint32_t kg, float* z) {
#pragma unroll
  for (int b = 0; b < MP; ++b) {
    const P4 r = draw(sk, kSlotDiffusion, (t0 * MP >> 2) + b, kg);
    box_muller(r.x, r.y, z[4 * b + 0], z[4 * b + 1]);
    box_muller(r.z, r.w, z[4 * b + 2], z[4 * b + 3]);
  }
}

// eps = L z (lower triangular, fixed fma order so every kernel that
// regenerates a draw gets the same bits).
template <int M, typename Real>
__device__ __forceinline__ void apply_chol(const Real* L, const float* z, Real* eps) {
#pragma unroll
  for (int j = 0; j < M; ++j) {
    Real acc = L[j * M] * Real(z[0]);
#pragma unroll
    for (int l = 1; l <= j; ++l) acc = fma(L[j * M + l], Real(z[l]), acc);
    eps[j] = acc;
  }
}

template <typename Real>
__device__ __forceinline__ Real radd(Real a, Real b);  // uncontracted add / mul: every kernel
template <>                                            // (and the oracle) rounds them alike
__device__ __forceinline__ float radd<float>(float a, float b) { return __fadd_rn(a, b); }
template <>
__device__ __forceinline__ double radd<double>(double a, double b) { return __dadd_rn(a, b); }
template <typename Real>
__device__ __forceinline__ Real rmul(Real a, Real b);
template <>
__device__ __forceinline__ float rmul<float>(float a, float b) { return __fmul_rn(a, b); }
template <>
__device__ __forceinline__ double rmul<double>(double a, double b) { return __dmul_rn(a, b); }

// marks = mu + Lj z
template <int Q, typename Real>
__device__ __forceinline__ void apply_marks(const Real* Lj, const Real* mu, const float* z, Real* mk) {
  Real c[Q];
  apply_chol<Q, Real>(Lj, z, c);
#pragma unroll
  // (an uncontracted add: c[0] is a bare product, and a compiler free to fuse mu + L z into one
  // fma in some inlining contexts and not in others would give the sampler, the rollout's mark
  // pass and the regeneration marks that differ in the last bit)
  for (int i = 0; i < Q; ++i) mk[i] = radd<Real>(mu[i], c[i]);
}

template <int Q>
struct Pad {
  static constexpr int value = (Q == 3) ? 4 : Q;
};

// ---------------------------------------------------------------- per-tile weighting
// Online softmax of one tile into the CTA accumulator (K3/K4 partials):
// rho_new = min(rho_acc, min_tile S); w_k = exp(-(S_k - rho_new)/lambda);
// Z, sum w^2, n_finite and N[r] += sum_k w_k eps[r,k] (rescaled by
// exp(-(rho_new - rho_acc)/lambda)).  Every thread of the CTA calls it; Sf holds
// the thread's SPT costs (+inf for none), cols their tile columns.
template <typename Real, int SPT, int RPW>
__device__ __forceinline__ void tile_epilogue(const Real* Sf, const int* cols, int nk, const Real* src,
                                              size_t rstride, int TM, Real inv_lam, Real* sw, double* Nacc,
                                              double (*s_red)[32], double* s_acc, double* s_bc) {
  (void)s_bc;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  // tile minimum: warp minimum on the REDUX unit (NaN costs count as +inf,
  // they get weight 0 either way), partials in shared memory, one barrier,
  // then every warp reduces the partials itself -- no serial thread-0 pass
  Real mloc = r_inf<Real>();
#pragma unroll
  for (int u = 0; u < SPT; ++u) mloc = fmin(mloc, Sf[u]);
  const double m = warp_min_redux(double(mloc));
  if (lane == 0) s_red[0][warp] = m;
  __syncthreads();
  const double mm = warp_min_redux(lane < nwarps ? s_red[0][lane] : CUDART_INF);
  const double rho_prev = s_acc[0];
  const double rho_new = fmin(rho_prev, mm);
  if (rho_new == CUDART_INF) return;  // no finite cost yet in this CTA (uniform)
  // rescale of the CTA's earlier tiles (multi-tile CTAs): one exp per warp
  double scale_old = 0.0;
  if (rho_prev != CUDART_INF) {
    const double e = lane == 0 ? exp((rho_new - rho_prev) * double(inv_lam)) : 0.0;
    scale_old = __shfl_sync(0xFFFFFFFFu, e, 0);
  }
  double z1 = 0.0, z2 = 0.0;
  int nf = 0;
#pragma unroll
  for (int u = 0; u < SPT; ++u) {
    const bool fin = Sf[u] < r_inf<Real>();
    const Real w = fin ? r_exp<Real>(-(Sf[u] - Real(rho_new)) * inv_lam) : Real(0);
    if (cols[u] >= 0) sw[cols[u]] = w;
    z1 += double(w);
    z2 += double(w) * double(w);
    nf += fin ? 1 : 0;
  }
  z1 = warp_sum(z1);
  z2 = warp_sum(z2);
  nf = __reduce_add_sync(0xFFFFFFFFu, nf);
  if (lane == 0) {
    s_red[1][warp] = z1;
    s_red[2][warp] = z2;
    s_red[3][warp] = double(nf);
  }
  __syncthreads();  // sw[] and the partials are complete; s_acc[0] has been read by every thread
  if (warp == nwarps - 1 && lane == 0) {  // the last warp has the fewest row blocks below
    double a1 = 0.0, a2 = 0.0, a3 = 0.0;
    for (int w2 = 0; w2 < nwarps; ++w2) {
      a1 += s_red[1][w2];
      a2 += s_red[2][w2];
      a3 += s_red[3][w2];
    }
    s_acc[0] = rho_new;
    s_acc[1] = s_acc[1] * scale_old + a1;
    s_acc[2] = s_acc[2] * scale_old * scale_old + a2;
    s_acc[3] += a3;
  }
  // N[r] += sum_k w_k eps[r, k] over the tile: a warp takes RPW rows, lanes
  // over k (RPW x 4 independent loads in flight per lane: 16 rows for the
  // small systems' global scratch, whose loads are L2/HBM latency-bound; the
  // quadrotor keeps 8, 16 spills its horizon loop), then one
  // transposing butterfly reduces the RPW row partials across the lanes
  // (9 shuffles for 8 rows instead of 40) -- fixed order, deterministic
  // row blocks in reverse horizon order: a global slab's late rows were
  // written last and are the ones still in L2 (the slabs of all resident
  // tiles exceed it), so they are read before the other CTAs' writes evict them
  const int nblk = (TM + RPW - 1) / RPW;
  for (int bi = warp; bi < nblk; bi += nwarps) {
    const int r0 = (nblk - 1 - bi) * RPW;
    Real acc[RPW];
#pragma unroll
    for (int i = 0; i < RPW; ++i) acc[i] = Real(0);
#pragma unroll 4
    for (int kk = lane; kk < nk; kk += 32) {
      const Real wk = sw[kk];
#pragma unroll
      for (int i = 0; i < RPW; ++i)
        if (r0 + i < TM) acc[i] = fma(wk, src[(size_t)(r0 + i) * rstride + kk], acc[i]);  // 0 * inf = NaN like controller.py:78
    }
    // stages off = 16, 8, ...: lanes split the rows (the upper half of the lane bit keeps the upper rows)
#pragma unroll
    for (int n = RPW / 2, off = 16; n >= 1; n >>= 1, off >>= 1) {
      const bool up = (lane & off) != 0;
#pragma unroll
      for (int i = 0; i < n; ++i) {
        const Real send = up ? acc[i] : acc[i + n];
        const Real keep = up ? acc[i + n] : acc[i];
        acc[i] = keep + __shfl_xor_sync(0xFFFFFFFFu, send, off);
      }
    }
    // the G = 32/RPW lanes sharing lane / G hold partials of row (lane / G) % RPW; finish across them
    constexpr int G = 32 / RPW;
#pragma unroll
    for (int off = G / 2; off >= 1; off >>= 1) acc[0] += __shfl_xor_sync(0xFFFFFFFFu, acc[0], off);
    const int row = r0 + ((lane / G) & (RPW - 1));
    if ((lane & (G - 1)) == 0 && row < TM) Nacc[row] = Nacc[row] * scale_old + double(acc[0]);
  }
  __syncthreads();
}

// ---------------------------------------------------------------- shared memory plan
// One layout for both rollout kernels and the host launcher (engine.cuh):
//   Nacc (TM doubles) | marks (nmarks Real) | step table (T*(2m+1) Real) |
//   sw (tile Real) | ring (WS only) | eps scratch (single wave) | gap table (uint32)
struct SmemPlan {
  size_t nacc, marks, tab, sw, ring, scr, gap, total;
};
__host__ __device__ __forceinline__ size_t al16(size_t x) { return (x + 15) & ~(size_t)15; }
__host__ __device__ __forceinline__ SmemPlan smem_plan(int TM, int tabn, int tile, int nmarks, int nring, int nscr,
                                                       int ngap, int rs) {
  SmemPlan p;
  size_t o = 0;
  p.nacc = o;
  o = al16(o + sizeof(double) * (size_t)TM);
  p.marks = o;
  o = al16(o + (size_t)rs * nmarks);
  p.tab = o;
  o = al16(o + (size_t)rs * tabn);
  p.sw = o;
  o = al16(o + (size_t)rs * tile);
  p.ring = o;
  o = al16(o + (size_t)rs * nring);
  p.scr = o;
  o = al16(o + (size_t)rs * nscr);
  p.gap = o;
  o = al16(o + sizeof(uint32_t) * (size_t)ngap);
  p.total = o;
  return p;
}

// ---------------------------------------------------------------- jump windows
// Jump events come from each sample's JumpClock (philox.cuh).  Per window of
// W <= 32 steps a warp (a) advances every lane's clock through the window
// (one uniform per event) into a bit mask, and (b) generates the marks of all
// its events cooperatively: the warp's events form one list (lane-major,
// then time order) and lane j produces entries j, j+32, ... -- the
// Philox + Box-Muller + Cholesky work of a mark is done once, by one lane,
// instead of by the whole warp every time any lane jumps.  Marks land in a
// dense per-warp buffer wd[(s*Q + i)*32 + lane] (zero where no event), so a
// step adds its staged value with one conflict-free shared-memory load and
// no branch.  State jumps (JM = 1) are staged pre-scaled (jscale * mark).

// Mark of jump event e: mu + Lj z, or -- Poisson counts -- the sum of the
// event's n arrivals' iid N(mu, Sigma_J) marks, n mu + sqrt(n) Lj z (n = 1
// leaves the single-mark value untouched).
template <int Q, int QP, typename Real>
__device__ __forceinline__ void mark_of(const StreamKey& sk, uint32_t kg, uint32_t e, const Real* Lj, const Real* mu,
                                        Real* mk, bool poisson, const CountTable& ct) {
  float z[QP];
  event_mark_normals<QP>(sk, kg, e, z);
  apply_marks<Q, Real>(Lj, mu, z, mk);
  if (poisson) {
    const int n = event_count(sk, kg, e, ct);
    if (n > 1) {
      Real c[Q];
      apply_chol<Q, Real>(Lj, z, c);
      const Real rn = Real(n), sn = sqrt(rn);
#pragma unroll
      for (int i = 0; i < Q; ++i) mk[i] = fma(sn, c[i], rn * mu[i]);
    }
  }
}

// Event masks of a window: 32-bit (W <= 32) or 128-bit (W <= 128) words.
struct Mask128 {
  uint64_t lo, hi;
};
__device__ __forceinline__ void mask_set(uint32_t& m, int b) { m |= 1u << b; }
__device__ __forceinline__ void mask_set(Mask128& m, int b) {
  const uint64_t bit = 1ull << (b & 63);
  if (b < 64)
    m.lo |= bit;
  else
    m.hi |= bit;
}
__device__ __forceinline__ void mask_pop(uint32_t& m) { m &= m - 1u; }
__device__ __forceinline__ void mask_pop(Mask128& m) {
  if (m.lo)
    m.lo &= m.lo - 1ull;
  else
    m.hi &= m.hi - 1ull;
}
__device__ __forceinline__ int mask_low(uint32_t m) { return __ffs((int)m) - 1; }
__device__ __forceinline__ int mask_low(const Mask128& m) {
  return m.lo ? __ffsll((long long)m.lo) - 1 : 64 + __ffsll((long long)m.hi) - 1;
}
__device__ __forceinline__ uint32_t mask_shfl(uint32_t m, int L) { return __shfl_sync(0xFFFFFFFFu, m, L); }
__device__ __forceinline__ Mask128 mask_shfl(const Mask128& m, int L) {
  return Mask128{__shfl_sync(0xFFFFFFFFu, m.lo, L), __shfl_sync(0xFFFFFFFFu, m.hi, L)};
}

// Called by all 32 lanes of a warp whose samples kg are consecutive by lane.
// Staging layout: entry (step s of the window, component i, lane L) at
// wd[(s * RQ + i) * CS + L] -- a per-warp buffer (RQ = Q, CS = 32), or the
// rows of the CTA's shared-memory eps slab that steps w0.. have not written
// yet (RQ = m, CS = tile; the step reads its mark there just before storing
// its eps_combined over it).  MaskT: 32- or 128-bit event masks (W <= 32 / 128).
template <int Q, int QP, int JM, typename Real, typename MaskT = Mask128, int RQ = Q, bool ZERO = true>
__device__ __forceinline__ void jump_window(JumpClock& c, int w0, int wend, int W, const StreamKey& sk, uint32_t kg,
                                            const GapSampler& gs, const Real* Lj, const Real* mu, Real jscale,
                                            Real* wd, bool poisson, const CountTable& ct, int CS = 32) {
  const int lane = threadIdx.x & 31;
  MaskT mask{};
  const uint32_t e0 = c.e;
  int n = 0;
  while (__any_sync(0xFFFFFFFFu, c.tj < wend)) {
    if (c.tj < wend) {
      mask_set(mask, c.tj - w0);
      ++n;
      clock_next(c, sk, kg, gs);
    }
  }
  int inc = n;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xFFFFFFFFu, inc, o);
    if (lane >= o) inc += v;
  }
  const int off = inc - n;
  const int tot = __shfl_sync(0xFFFFFFFFu, inc, 31);
  __syncwarp();  // the previous window's marks have been read
  // (only the window's steps: the slab has no rows past the horizon; a slab
  // zeroed in the prologue needs none)
  if (ZERO)
    for (int t = 0; t < wend - w0; ++t)
#pragma unroll
      for (int i = 0; i < Q; ++i) wd[(t * RQ + i) * CS + lane] = Real(0);
  __syncwarp();
  for (int j0 = 0; j0 < tot; j0 += 32) {
    const int j = j0 + lane;
    int L = 0;  // owner lane of entry j: the last lane with off <= j
#pragma unroll
    for (int bb = 16; bb > 0; bb >>= 1) {
      const int oc = __shfl_sync(0xFFFFFFFFu, off, L + bb);
      if (oc <= j) L += bb;
    }
    const int k = j - __shfl_sync(0xFFFFFFFFu, off, L);
    const uint32_t eL = __shfl_sync(0xFFFFFFFFu, e0, L) + (uint32_t)k;
    MaskT mL = mask_shfl(mask, L);
    if (j < tot) {
      for (int r = 0; r < k; ++r) mask_pop(mL);  // the owner's k-th event step
      const int s = mask_low(mL);
      Real mk[Q];
      mark_of<Q, QP, Real>(sk, kg - (uint32_t)lane + (uint32_t)L, eL, Lj, mu, mk, poisson, ct);
#pragma unroll
      for (int i = 0; i < Q; ++i) wd[(s * RQ + i) * CS + L] = (JM == 1) ? rmul<Real>(jscale, mk[i]) : mk[i];
    }
  }
  __syncwarp();
}

// ---------------------------------------------------------------- rollout
// Common prologue: per-step table (clamped u, controller.py:128, hoisted into
//   udt = u dt, a_t = 1/2 u'Ru dt, b_t = lambda u sqrt(dt)   (costs.py:98-111 times dt)),
// accumulator reset and the gap table copy.
template <int M, typename Real>
__device__ __forceinline__ void rollout_prologue(const RolloutArgs<Real>& a, const double* u_nom, Real* tab,
                                                 double* Nacc, double* s_acc, uint32_t* S) {
  constexpr int TS = 2 * M + 1;
  const int T = a.T;
  // read-only (.nc) loads, unrolled: the loop's global reads are issued
  // together instead of one round trip per iteration
#pragma unroll 4
  for (int t = threadIdx.x; t < T; t += blockDim.x) {
    Real u[M];
#pragma unroll
    for (int j = 0; j < M; ++j) {
      Real v = Real(u_nom[t * M + j]);  // (plain load: written by the previous step's finalize)
      if (a.has_limits) v = fmin(fmax(v, a.u_lo[j]), a.u_hi[j]);
      u[j] = v;
    }
    Real uru = Real(0);
#pragma unroll
    for (int j = 0; j < M; ++j)
#pragma unroll
      for (int l = 0; l < M; ++l) uru += u[j] * a.R[j * M + l] * u[l];
#pragma unroll
    for (int j = 0; j < M; ++j) {
      tab[t * TS + j] = u[j] * a.dt;
      Real cu = u[j];
      if (a.general) {  // lambda u' calB eps = lambda (calB' u) . eps (costs.py:116-117)
        cu = Real(0);
#pragma unroll
        for (int i = 0; i < M; ++i) cu = fma(u[i], a.calb[i * M + j], cu);
      }
      tab[t * TS + M + 1 + j] = a.lam_sdt * cu;
    }
    tab[t * TS + M] = Real(0.5) * uru * a.dt;
  }
  for (int r = threadIdx.x; r < a.TM; r += blockDim.x) Nacc[r] = 0.0;
#pragma unroll 4
  for (int i = threadIdx.x; i < a.gap_n; i += blockDim.x) S[i] = __ldg(a.gap_thr + i);
  if (threadIdx.x == 0) {
    s_acc[0] = CUDART_INF;
    s_acc[1] = 0.0;
    s_acc[2] = 0.0;
    s_acc[3] = 0.0;
  }
}

// eps' eps, or eps' bb eps for the general channel (costs.py:118-121); eps'eps
// formed first (costs.py:101/:514), so an overflowing eps gives NaN even when c = 1
template <int M, typename Real, bool GEN>
__device__ __forceinline__ Real noise_quad(const RolloutArgs<Real>& a, const Real* eps) {
  Real quad = eps[0] * eps[0];
#pragma unroll
  for (int j = 1; j < M; ++j) quad = fma(eps[j], eps[j], quad);
  if (GEN) {
    quad = Real(0);
#pragma unroll
    for (int i = 0; i < M; ++i) {
      Real t = Real(0);
#pragma unroll
      for (int j = 0; j < M; ++j) t = fma(a.bb[i * M + j], eps[j], t);
      quad = fma(eps[i], t, quad);
    }
  }
  return quad;
}

// Batched trials (jm_batch_loop_host): blockIdx.y is the trial; its loop
// state, nominal controls, records and eps slabs are the trial-th slices.
//
// Peer-memory exchange: every rank's symmetric buffer (world W, grid G,
// record stride rs) is [parity 0: W*G records][parity 1: W*G records][W*G
// uint32 epoch flags].  A CTA stores its record into slot rank*G + cta of
// parity (epoch & 1) of EVERY rank's buffer -- peer pointers, so the stores
// travel over NVLink/NVSwitch as soon as the CTA's tile is done, overlapping
// the slower CTAs -- then raises its flag there to the epoch (release after a
// system-scope fence).  Double buffering by parity: a rank runs at most one
// control step ahead of the slowest peer (its next push needs its own
// finalize, which waited for every peer's records).
template <typename Real>
__device__ __forceinline__ void write_record(const RolloutArgs<Real>& a, const double* s_acc, const double* Nacc) {
  if (a.push_peers != nullptr) {
    const uint32_t epoch = (uint32_t)a.loop->step + 1u;
    const int W = a.push_world, G = gridDim.x, slot = a.push_rank * G + blockIdx.x;
    const size_t off = ((size_t)(epoch & 1u) * W * G + slot) * a.rec_stride;
    for (int p = 0; p < W; ++p) {
      double* dst = reinterpret_cast<double*>(a.push_peers[p]) + off;
      if (threadIdx.x == 0) {
        dst[0] = s_acc[0];
        dst[1] = s_acc[1];
        dst[2] = s_acc[2];
        dst[3] = s_acc[3];
      }
      for (int r = threadIdx.x; r < a.TM; r += blockDim.x) dst[4 + r] = Nacc[r];
    }
    if (W == 1) {  // the local buffer: GPU-scope release is enough
      __threadfence();
      __syncthreads();
      if (threadIdx.x == 0)
        st_release_gpu(reinterpret_cast<unsigned int*>(reinterpret_cast<double*>(a.push_peers[0]) +
                                                       2 * (size_t)G * a.rec_stride) + slot,
                       epoch);
      return;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence_system();
      for (int p = 0; p < W; ++p)
        st_release_sys(reinterpret_cast<unsigned int*>(reinterpret_cast<double*>(a.push_peers[p]) +
                                                       2 * (size_t)W * G * a.rec_stride) + slot,
                       epoch);
    }
    return;
  }
  double* rec = a.records + ((size_t)blockIdx.y * gridDim.x + blockIdx.x) * a.rec_stride;
  if (threadIdx.x == 0) {
    rec[0] = s_acc[0];
    rec[1] = s_acc[1];
    rec[2] = s_acc[2];
    rec[3] = s_acc[3];
  }
  for (int r = threadIdx.x; r < a.TM; r += blockDim.x) rec[4 + r] = Nacc[r];
}

// One sample per thread.  JM = 0: control-channel jumps (marks folded into
// eps_combined, q = m); JM = 1: state-space jumps on Dyn::jump_row (q =
// Dyn::QJ, eps_combined = eps_d).  PHILOX: noise drawn in registers (else the
// HBM wire format); TRACE: per-step states + divergence steps (host API).
// (a 64-register cap via 2 blocks/SM measured slower: parameter reloads)
template <class Sys, typename Real>
struct RolloutMinBlocks {
  static constexpr int value = 1;
};

// SCR_SMEM (Philox, non-trace, single wave): the eps scratch is a
// shared-memory array (compile-time, so its stores / epilogue loads are
// STS / LDS with 32-bit addresses).
template <class Sys, typename Real, bool PHILOX, bool TRACE, int JM, bool SCR_SMEM = false>
__global__ void __launch_bounds__(kRolloutMaxThreads, (RolloutMinBlocks<Sys, Real>::value))
    rollout_kernel(const RolloutArgs<Real> a) {
  using Dyn = typename Sys::Dyn;
  using Cost = typename Sys::Cost;
  constexpr int N = Sys::N, M = Sys::M;
  constexpr int MP = Pad<M>::value;
  constexpr int Q = (JM == 0) ? M : Dyn::QJ;
  constexpr int QP = Pad<Q>::value;
  constexpr int TS = 2 * M + 1;

  extern __shared__ double smem_d[];
  __shared__ double s_red[4][32];
  __shared__ double s_acc[4];  // rho, Z, W2, nfinite of this CTA
  __shared__ double s_bc[2];

  const int TM = a.TM, T = a.T, K = a.K;
  const int tileK = blockDim.x, nwarps = blockDim.x >> 5;
  static_assert(!SCR_SMEM || (PHILOX && !TRACE), "shared-memory scratch: Philox main kernel only");
  constexpr bool in_smem = SCR_SMEM;
  // SCR_SMEM: jump marks are staged in the eps slab itself (no separate buffer)
  const SmemPlan sp_ = smem_plan(TM, T * TS, tileK, (a.jump_on && !SCR_SMEM) ? nwarps * 32 * a.jw_len * Q : 0, 0,
                                 in_smem ? TM * tileK : 0, a.gap_n, (int)sizeof(Real));
  (void)nwarps;
  char* const sb = reinterpret_cast<char*>(smem_d);
  double* Nacc = reinterpret_cast<double*>(sb + sp_.nacc);
  Real* tab = reinterpret_cast<Real*>(sb + sp_.tab);
  Real* sw = reinterpret_cast<Real*>(sb + sp_.sw);
  uint32_t* Sg = reinterpret_cast<uint32_t*>(sb + sp_.gap);
  Real* const wd = reinterpret_cast<Real*>(sb + sp_.marks) + (threadIdx.x >> 5) * 32 * a.jw_len * Q;
  Real* const scr = in_smem ? reinterpret_cast<Real*>(sb + sp_.scr)
                            : a.eps_out + ((size_t)blockIdx.y * gridDim.x + blockIdx.x) * TM * tileK;
#ifdef JM_ROLL_STAMPS  // tuning builds: CTA 0's phase clocks land in costs[0..6] (costs requested)
  long long rts[8];
  int rn = 0;
  rts[rn++] = clock64();
#define ROLL_STAMP() (rts[rn++] = clock64())
#else
#define ROLL_STAMP() ((void)0)
#endif

  grid_dep_wait();    // u_nom / x / iteration come from the previous control step
  grid_dep_launch();  // (after the wait: the finalize's pre-wait prologue reads the
                      // plant state the previous finalize wrote) let the finalize
                      // grid get resident while the horizon runs
  LoopState* L = a.loop ? a.loop + blockIdx.y : nullptr;
  if (L != nullptr && L->halted) return;
  const uint64_t iter = L ? L->iteration : (a.iteration_dev ? *a.iteration_dev : a.iteration);
  const double* x0 = L ? L->x : a.x0;
  if (L != nullptr && blockIdx.x == 0 && threadIdx.x == 0) L->t_start[L->step] = globaltimer();
  ROLL_STAMP();
  rollout_prologue<M, Real>(a, L ? loop_unom(L, L->step, TM) : a.u_nom + (size_t)blockIdx.y * TM, tab, Nacc, s_acc, Sg);
  if (SCR_SMEM && a.jump_on) {  // the slab rows double as the jump-mark staging: zero them once, 16 B a store
    float4* z4 = reinterpret_cast<float4*>(scr);
    const int n4 = (int)((size_t)TM * tileK * sizeof(Real) / 16);
    for (int i = threadIdx.x; i < n4; i += blockDim.x) z4[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
  __syncthreads();
  ROLL_STAMP();

  // loop-invariant parameters, pinned in registers
  SysParams<Real> sp = a.sp;
#pragma unroll
  for (int i = 0; i < 10; ++i) pin(sp.mp[i]);
#pragma unroll
  for (int i = 0; i < N; ++i) {
    pin(sp.sw[i]);
    pin(sp.swt[i]);
  }
  if (SCR_SMEM) {  // (the multi-wave kernels run at the 128-register cap: no room to pin them)
#pragma unroll
    for (int i = 0; i < 3; ++i) pin(sp.tk[i]);
  }
  Real Ld[M * M], Lj[Q * Q], mu[Q];
#pragma unroll
  for (int i = 0; i < M * M; ++i) {
    Ld[i] = a.Ld[i];
    pin(Ld[i]);
  }
#pragma unroll
  for (int i = 0; i < Q * Q; ++i) Lj[i] = a.Lj[i];
#pragma unroll
  for (int i = 0; i < Q; ++i) mu[i] = a.mu_j[i];
  Real dt = a.dt, sdt = a.sdt, cq = a.cq, jscale = a.jscale;
  pin(dt);
  pin(sdt);
  pin(cq);
  const GapSampler gs{Sg, T, a.gap_inv};
  const int JW = a.jw_len;
  const bool jumps = PHILOX && a.jump_on && (L == nullptr || L->sampler_jumps);

  const StreamKey sk = make_stream_key(a.seeds[blockIdx.y], iter);
  double* const costs_out = gridDim.y > 1 ? nullptr : (a.costs_dev ? *a.costs_dev : a.costs);

  // the general-channel cost (costs.py:112-124) as a compile-time variant of the tile loop:
  // a runtime branch inside the step would be predicated and cost the control-channel path
  auto tiles = [&](auto gen_tag) {
  constexpr bool GEN = decltype(gen_tag)::value;
  for (int tile = blockIdx.x; tile < a.ntiles; tile += gridDim.x) {
    const int base = tile * tileK;
    const int kl = base + threadIdx.x;
    const bool act = kl < K;
    const uint32_t kg = (uint32_t)(a.sample_offset + kl);
    Real* ep = scr + threadIdx.x;  // Philox scratch: row (t*M+j) of this sample's column
    Real x[N];
    Real S = Real(0);
    int dstep = -1;
#pragma unroll
    for (int i = 0; i < N; ++i) x[i] = Real(x0[i]);
    if (TRACE && act) {
#pragma unroll
      for (int i = 0; i < N; ++i) a.states[((size_t)kl * (T + 1)) * N + i] = double(x[i]);
    }
    JumpClock clk;
    const Real* wl = wd + (threadIdx.x & 31);  // this lane's staged marks, advanced per step
    int wnext = 0;                             // first step of the next jump window
    if (jumps) clock_start(clk, sk, kg, gs);

    // one horizon step t with its final eps_combined and state jump
    auto step = [&](const int t, const Real* eps, const Real* sj, const bool has_sj) {
      // modified running cost on x_t (controller.py:140-142):
      // q dt + 1/2 u'Ru dt + lambda sqrt(dt) u'eps + 1/2 lambda (1-1/c) eps'eps
      // (eps'eps formed first, as costs.py:101/:514, so an overflowing eps
      // gives NaN even when c = 1)
      const auto ax = Dyn::template aux<Real, SCR_SMEM || !PHILOX>(x, sp);
      const Real qv = Cost::template q<Dyn, Real>(x, ax, sp);
      const Real* st = tab + t * TS;
      Real inc = fma(qv, dt, st[M]);
      const Real quad = noise_quad<M, Real, GEN>(a, eps);
#pragma unroll
      for (int j = 0; j < M; ++j) inc = fma(st[M + 1 + j], eps[j], inc);
      S += fma(cq, quad, inc);
      // Euler step (dynamics.py:130-135 / :115-129 with B = G)
      Real xold[N];
      if (TRACE) {
#pragma unroll
        for (int i = 0; i < N; ++i) xold[i] = x[i];
      }
      Real v[M];
#pragma unroll
      for (int j = 0; j < M; ++j) v[j] = fma(eps[j], sdt, st[j]);
      Dyn::template advance<Real>(x, ax, v, dt, sp);
      if (JM == 1 && has_sj) {
#pragma unroll
        for (int i = 0; i < Q; ++i) x[Dyn::jump_row(i)] = radd<Real>(x[Dyn::jump_row(i)], sj[i]);  // x + H (ind * mark)
      }
      if (TRACE) {
        // divergence mask, controller.py:144-151
        bool fin = true;
#pragma unroll
        for (int i = 0; i < N; ++i) fin = fin && isfinite(x[i]);
        if (dstep >= 0 || !fin) {
          if (dstep < 0) dstep = t;
#pragma unroll
          for (int i = 0; i < N; ++i) x[i] = xold[i];
        }
        if (act) {
#pragma unroll
          for (int i = 0; i < N; ++i) a.states[((size_t)kl * (T + 1) + t + 1) * N + i] = double(x[i]);
        }
      }
    };
    // noise of step t (sub-step s2 of its group) from the group buffers, then the step
    auto noisy_step = [&](const int t, const int s2, const float* zz, const float* zzm) {
      Real eps[M];
      Real sj[Q];
      bool has_sj = false;
      if (PHILOX) {
        apply_chol<M, Real>(Ld, zz + s2 * MP, eps);
        if (jumps) {
          // staged marks: the separate buffer, or this step's own slab rows (SCR_SMEM)
          const Real* mrow = SCR_SMEM ? ep : wl;
          const int mcs = SCR_SMEM ? tileK : 32;
          if (JM == 0) {
#pragma unroll
            for (int j = 0; j < M; ++j) eps[j] = radd<Real>(eps[j], mrow[j * mcs]);  // eps_c = eps_d + eps_j (noise.py:156-157)
          } else {
#pragma unroll
            for (int i = 0; i < Q; ++i) sj[i] = mrow[i * mcs];  // jscale * ind * mark
            has_sj = true;
          }
          if (!SCR_SMEM) wl += Q * 32;
        }
#pragma unroll
        for (int j = 0; j < M; ++j) ep[(size_t)j * tileK] = eps[j];
        ep += (size_t)M * tileK;
      } else {
        // HBM wire format, prefetched one group ahead into zz / zzm
#pragma unroll
        for (int j = 0; j < M; ++j) eps[j] = reinterpret_cast<const Real*>(zz)[s2 * M + j];
        if (JM == 1 && a.jump_in != nullptr) {
#pragma unroll
          for (int i = 0; i < Q; ++i) sj[i] = jscale * reinterpret_cast<const Real*>(zzm)[s2 * Q + i];
          has_sj = true;
        }
      }
      step(t, eps, sj, has_sj);
    };
    // Diffusion noise of group g+1 is drawn while group g steps (software
    // pipeline: it is independent of the state, so it fills the dynamics
    // chain's latency); full groups carry no per-step horizon checks.  HBM
    // mode reuses the group buffers as raw storage for the loaded noise.
    constexpr int ZW = PHILOX ? 4 * MP : (4 * M * (int)sizeof(Real) + 3) / 4;
    constexpr int ZMW = (4 * Q * (int)sizeof(Real) + 3) / 4;
    // rows of this sample's column: one running pointer per tensor (advanced by
    // a row per step) instead of a 64-bit index product per load; rows past the
    // horizon are clamped to T-1 (only the last two groups can reach them)
    const int kcol = act ? kl : 0;
    const Real* pe = PHILOX ? nullptr : a.eps_in + kcol;
    const Real* pj = (PHILOX || JM != 1 || a.jump_in == nullptr) ? nullptr : a.jump_in + kcol;
    const size_t rowe = (size_t)M * K, rowj = (size_t)Q * K;
    auto load_group = [&](const int g0, float* zz, float* zzm) {
      Real* ze = reinterpret_cast<Real*>(zz);
      Real* zj = reinterpret_cast<Real*>(zzm);
      if (g0 + 4 <= T) {
        const Real* qe = pe + (size_t)g0 * rowe;
#pragma unroll
        for (int s2 = 0; s2 < 4; ++s2) {
#pragma unroll
          for (int j = 0; j < M; ++j) ze[s2 * M + j] = __ldg(qe + (size_t)j * K);
          qe += rowe;
        }
        if (JM == 1 && pj != nullptr) {
          const Real* qj = pj + (size_t)g0 * rowj;
#pragma unroll
          for (int s2 = 0; s2 < 4; ++s2) {
#pragma unroll
            for (int i = 0; i < Q; ++i) zj[s2 * Q + i] = __ldg(qj + (size_t)i * K);
            qj += rowj;
          }
        }
      } else {
#pragma unroll
        for (int s2 = 0; s2 < 4; ++s2) {
          const int t = min(g0 + s2, T - 1);
#pragma unroll
          for (int j = 0; j < M; ++j) ze[s2 * M + j] = __ldg(pe + (size_t)t * rowe + (size_t)j * K);
          if (JM == 1 && pj != nullptr) {
#pragma unroll
            for (int i = 0; i < Q; ++i) zj[s2 * Q + i] = __ldg(pj + (size_t)t * rowj + (size_t)i * K);
          }
        }
      }
    };
    float z[ZW];
    float zm[ZMW];  // HBM mode: jump rows of the current group
    float z1[PHILOX ? 1 : ZW], zm1[PHILOX ? 1 : ZMW];  // HBM mode: the next group (loads run two groups ahead)
    if (PHILOX) {
      group_normals<MP>(sk, 0u, kg, z);
    } else {
      load_group(0, z, zm);
      load_group(4, z1, zm1);
    }
    for (int t0 = 0; t0 < T; t0 += 4) {
      if (jumps && t0 == wnext) {
        wnext = t0 + JW;
        if (SCR_SMEM) {
          jump_window<Q, QP, JM, Real, Mask128, M, false>(clk, t0, min(wnext, T), JW, sk, kg, gs, Lj, mu, jscale,
                                                    scr + (size_t)t0 * M * tileK + (threadIdx.x & ~31), a.poisson != 0,
                                                    a.cnt, tileK);
        } else {
          jump_window<Q, QP, JM, Real>(clk, t0, min(wnext, T), JW, sk, kg, gs, Lj, mu, jscale, wd, a.poisson != 0,
                                       a.cnt);
          wl = wd + (threadIdx.x & 31);
        }
      }
      if (t0 + 4 <= T) {
        float zn[ZW], zmn[ZMW];
        if (PHILOX)
          group_normals<MP>(sk, (uint32_t)(t0 + 4), kg, zn);
        else
          load_group(t0 + 8, zn, zmn);  // (clamped inside the horizon)
#pragma unroll
        for (int s2 = 0; s2 < 4; ++s2) noisy_step(t0 + s2, s2, z, zm);
        if (PHILOX) {
#pragma unroll
          for (int i = 0; i < ZW; ++i) z[i] = zn[i];
        } else {
#pragma unroll
          for (int i = 0; i < ZW; ++i) {
            z[i] = z1[i];
            z1[i] = zn[i];
          }
#pragma unroll
          for (int i = 0; i < ZMW; ++i) {
            zm[i] = zm1[i];
            zm1[i] = zmn[i];
          }
        }
      } else {
#pragma unroll
        for (int s2 = 0; s2 < 4; ++s2)
          if (t0 + s2 < T) noisy_step(t0 + s2, s2, z, zm);
      }
    }
    // Once non-finite, an Euler state x += dx stays non-finite, so the final
    // state decides divergence (the reference checks every step).
    bool fin = true;
#pragma unroll
    for (int i = 0; i < N; ++i) fin = fin && isfinite(x[i]);
    if (TRACE) {
      fin = dstep < 0;
      if (act) a.diverged[kl] = dstep;
    }
    if (fin) {
      const auto ax = Dyn::template aux<Real, SCR_SMEM || !PHILOX>(x, sp);
      S += sp.term_scale * Cost::template q<Dyn, Real>(x, ax, sp);  // controller.py:155
    } else {
      S = r_inf<Real>();
    }
    if (act && costs_out) costs_out[kl] = double(S);
    const Real Sf = act ? S : r_inf<Real>();
    const int col = threadIdx.x;
    ROLL_STAMP();
#ifdef JM_ROLL_STAMPS
    __syncthreads();
    ROLL_STAMP();
#endif
    // ---- per-CTA online softmax over this tile (K3/K4 partials) ----
    tile_epilogue<Real, 1, (SCR_SMEM || N > 4) ? 8 : 16>(&Sf, &col, min(tileK, K - base), PHILOX ? scr : a.eps_in + base,
                           PHILOX ? (size_t)tileK : (size_t)K, TM, a.inv_lam, sw, Nacc, s_red, s_acc, s_bc);
    ROLL_STAMP();
  }
  };
  if (a.general)
    tiles(std::true_type{});
  else
    tiles(std::false_type{});
  __syncthreads();
  write_record(a, s_acc, Nacc);
#ifdef JM_ROLL_STAMPS
  ROLL_STAMP();
  double* const co = a.costs_dev ? *a.costs_dev : a.costs;
  if (co && blockIdx.x == 0 && threadIdx.x == 0)
    for (int i = 1; i < rn; ++i) co[i - 1] = double(rts[i] - rts[0]);
#endif
}

// ---------------------------------------------------------------- plant + shift (closed loop)
struct PlantArgs {
  SysParams<double> sp;
  double dt, sdt, jscale;
  double Lp[16];   // chol(Sigma_D)  (plant: Sigma_D, not c*Sigma_D; harness.py:123)
  double Lj[16];   // chol(Sigma_J)
  double mu_j[4];
  uint32_t jthr;   // plant always has jumps (harness.py:138)
  int poisson;     // Poisson arrivals: n = #{k : u24 < cnt0[k]} (cnt0[0] = the event threshold)
  uint32_t cnt0[kMaxCount + 1];
  int q, jmode, has_limits, T, M;
  double u_lo[4], u_hi[4];
  LoopState* loop;
  const double* u_new;
  double* u_nom;
};

// The plant step, split so that everything that does not depend on u_new
// (the LoopState fields, the plant noise draws) is done before the finalize
// kernel waits for the rollout grid.
struct PlantPre {
  double x[12];
  double aux[6];  // Dyn::aux<double>(x): the plant state's trig, computed before the wait
  double ed[4];   // L_D z  (Sigma_D, harness.py:137)
  double mk[4];   // mu + L_J z', drawn every step (harness.py:139)
  int k;
  int jump;       // U < nu dt (harness.py:138); Poisson: the arrival count
};

template <class Dyn>
__device__ void plant_prepare(const PlantArgs& a, PlantPre& pre) {
  constexpr int N = Dyn::N, M = Dyn::M;
  const LoopState* L = a.loop + blockIdx.y;
  const int k = L->step;
  pre.k = k;
  for (int i = 0; i < N; ++i) pre.x[i] = L->x[i];
  {
    const auto ax = Dyn::template aux<double>(pre.x, a.sp);
    static_assert(sizeof(ax) <= sizeof(pre.aux), "plant trig");
    memcpy(pre.aux, &ax, sizeof(ax));
  }
  const StreamKey sk = make_stream_key(L->seed, 0);
  P4 r = draw(sk, kSlotPlant, 3u * k + 0u, 0u);
  float z[4];
  box_muller(r.x, r.y, z[0], z[1]);
  box_muller(r.z, r.w, z[2], z[3]);
  double ed[M];
  apply_chol<M, double>(a.Lp, z, ed);
  for (int j = 0; j < M; ++j) pre.ed[j] = ed[j];
  const P4 ju = draw(sk, kSlotPlant, 3u * k + 1u, 0u);
  if (a.poisson) {
    int n = 0;
    for (int i = 0; i <= kMaxCount; ++i) n += (ju.x >> 8) < a.cnt0[i] ? 1 : 0;
    pre.jump = n;
  } else {
    pre.jump = ju.x < a.jthr ? 1 : 0;
  }
  r = draw(sk, kSlotPlant, 3u * k + 2u, 0u);
  box_muller(r.x, r.y, z[0], z[1]);
  box_muller(r.z, r.w, z[2], z[3]);
  for (int i = 0; i < 4; ++i) {
    double acc = 0.0;
    for (int l = 0; l <= i && i < a.q; ++l) acc = fma(a.Lj[i * a.q + l], double(z[l]), acc);
    pre.mk[i] = (i < a.q) ? a.mu_j[i] + acc : 0.0;
    if (pre.jump > 1 && i < a.q) pre.mk[i] = fma(sqrt(double(pre.jump)), acc, double(pre.jump) * a.mu_j[i]);
  }
}

// One plant step from u_new[0] and the warm-start shift; run by one CTA after
// u_new is complete.
// u_src: the finished control sequence (shared memory when the finalize is a
// single CTA, else a.u_new in global memory, read past L1).
// The plant state update of one control step (one thread): x <- Euler step from
// the clamped u0 with the prepared noise (harness.py:137-148), history, and the
// divergence check; returns false when the plant diverged (loop halted).
template <class Dyn>
__device__ bool plant_advance(const PlantArgs& a, const PlantPre& pre, const double* u0, LoopState* L) {
  constexpr int N = Dyn::N, M = Dyn::M;
  const int k = pre.k;
  {
    const bool jump = pre.jump != 0;
    double x[N];
    for (int i = 0; i < N; ++i) x[i] = pre.x[i];
    typename Dyn::template Aux<double> ax;
    memcpy(&ax, pre.aux, sizeof(ax));  // (computed before the grid dependency wait)
    double v[M];
    for (int j = 0; j < M; ++j) {
      const double e = (jump && a.jmode == 0) ? pre.ed[j] + pre.mk[j] : pre.ed[j];
      v[j] = fma(e, a.sdt, u0[j] * a.dt);
    }
    Dyn::template advance<double>(x, ax, v, a.dt, a.sp);
    if (jump && a.jmode == 1) {
#pragma unroll
      for (int i = 0; i < Dyn::QJ; ++i) x[Dyn::jump_row(i)] += a.jscale * pre.mk[i];
    }
    bool fin = true;
    for (int i = 0; i < N; ++i) fin = fin && isfinite(x[i]);
    for (int j = 0; j < M; ++j) L->hist_controls[(size_t)k * M + j] = u0[j];
    L->hist_jumps[k] = pre.jump;
    if (!fin) {  // StateDivergedError -> trial failure (harness.py:144-148)
      L->halted = 1;
      L->status = 7;
      L->diverged_at = k;
      return false;
    }
    for (int i = 0; i < N; ++i) {
      L->x[i] = x[i];
      L->hist_states[(size_t)(k + 1) * N + i] = x[i];
    }
    return true;
  }
}

// One plant step from u_new[0] and the warm-start shift; run by one CTA after
// u_new is complete.
// u_src: the finished control sequence (shared memory when the finalize is a
// single CTA, else a.u_new in global memory, read past L1).
template <class Dyn>
__device__ void plant_finish(const PlantArgs& a, const PlantPre& pre, const double* u_src, bool u_src_global) {
  constexpr int M = Dyn::M;
  LoopState* L = a.loop + blockIdx.y;
  double* const u_nom = loop_unom(L, pre.k + 1, a.T * M);  // the next step's parity
  __shared__ int s_ok;
  if (threadIdx.x == 0) {
    L->t_end[pre.k] = globaltimer();
    double u0[M];
    for (int j = 0; j < M; ++j) {
      double v = u_src_global ? __ldcg(u_src + j) : u_src[j];
      if (a.has_limits) v = fmin(fmax(v, a.u_lo[j]), a.u_hi[j]);  // harness.py:136
      u0[j] = v;
    }
    s_ok = plant_advance<Dyn>(a, pre, u0, L) ? 1 : 0;
  }
  __syncthreads();
  if (!s_ok) return;
  const int TM = a.T * M;
  for (int i = threadIdx.x; i < TM; i += blockDim.x)
    u_nom[i] = (i < TM - M) ? (u_src_global ? __ldcg(u_src + i + M) : u_src[i + M])
                              : L->u_init[i - (TM - M)];  // warm_start_shift
  __syncthreads();
  if (threadIdx.x == 0) {
    tl_put(tl_row(L, L->step), kTlFinEnd);
    L->iteration += 1;  // ControllerState(..., k+1, cfg) (harness.py:150)
    L->step += 1;
    if (L->step >= L->max_steps) L->halted = 1;
  }
}

// ---------------------------------------------------------------- finalize
// -DJM_FIN_STAMPS (tuning builds only): thread 0 records clock64() at the phase
// boundaries and writes the cycles since kernel entry into a.norms[0..] (the
// drop-in call returns them as per_step_update_norm)
#ifdef JM_FIN_STAMPS
#define FIN_STAMP() (fin_ts[fin_nts++] = clock64())
#else
#define FIN_STAMP() ((void)0)
#endif
struct FinArgs {
  const double* rec;
  int nrec, rec_stride, TM, M;
  int cols;  // columns per CTA, fin_cols(M)
  double inv_lam, inv_sdt;
  const double* u_nom;
  const double* mapping;  // m x m or null
  double* u_new;
  double* norms;          // T or null
  DiagOut* diag;          // or null
  int32_t* status;        // or null
  double* rec_out;        // reduce mode: write the merged record instead of finalizing
  LoopState* loop;
  unsigned int* counter;  // last-CTA-done counter (closed loop / shift output)
  const double* u_init;   // optional: u_shift = warm_start_shift(u_new, u_init)
  double* u_shift;
  volatile int32_t* done; // optional: set to 1 (system-scope fence first) once every output is written
  // peer-memory exchange (jm_loop_finish_peers): before merging, wait until the
  // nrec (= world x grid) flags reach this step's epoch (L->step + 1); records
  // of epoch parity e & 1 start at rec + (e & 1) * nrec * rec_stride
  const unsigned int* wait_flags;
  int wait_gpu;     // the flags are released at GPU scope (single-GPU use of the exchange)
  int wait_nflags;  // flags to wait on (0: nrec)
  // two-level exchange (jm_loop_reduce_push): reduce mode stores the merged
  // record into slot push_rank of parity (epoch & 1) of every peer buffer
  // ([2 parities x push_world records][flags]) and raises flag
  // push_rank * gridDim.x + blockIdx.x there (one per column block);
  // epoch = push_loop->step + 1
  const unsigned long long* push_peers;
  int push_rank, push_world;
  const LoopState* push_loop;
};

// reduce mode: write this CTA's part of the merged record (the head from
// CTA 0, columns [c0, c0 + kFinCols)) into rec_out, or into every peer's
// buffer followed by this CTA's flag release
__device__ __forceinline__ void fin_emit_record(const FinArgs& a, int c0, double rho, double Z, double W2, double NF,
                                                const double* cols) {
  const int tid = threadIdx.x;
  const int ncol = min(a.cols, a.TM - c0);
  if (a.push_peers == nullptr) {
    if (blockIdx.x == 0 && tid == 0) {
      a.rec_out[0] = rho;
      a.rec_out[1] = Z;
      a.rec_out[2] = W2;
      a.rec_out[3] = NF;
    }
    if (tid < ncol) a.rec_out[4 + c0 + tid] = cols ? cols[tid] : 0.0;
    return;
  }
  const uint32_t epoch = (uint32_t)a.push_loop->step + 1u;
  const int W = a.push_world;
  const size_t off = ((size_t)(epoch & 1u) * W + a.push_rank) * a.rec_stride;
  for (int p = 0; p < W; ++p) {
    double* dst = reinterpret_cast<double*>(a.push_peers[p]) + off;
    if (blockIdx.x == 0 && tid == 0) {
      dst[0] = rho;
      dst[1] = Z;
      dst[2] = W2;
      dst[3] = NF;
    }
    if (tid < ncol) dst[4 + c0 + tid] = cols ? cols[tid] : 0.0;
  }
  __syncthreads();
  if (tid == 0) {
    const int slot = a.push_rank * gridDim.x + blockIdx.x;
    if (W == 1) {
      __threadfence();
    } else {
      __threadfence_system();
    }
    for (int p = 0; p < W; ++p) {
      unsigned int* flags =
          reinterpret_cast<unsigned int*>(reinterpret_cast<double*>(a.push_peers[p]) + 2 * (size_t)W * a.rec_stride);
      if (W == 1)
        st_release_gpu(flags + slot, epoch);
      else
        st_release_sys(flags + slot, epoch);
    }
  }
}

inline size_t finalize_smem_bytes(int nrec) {
  return sizeof(double) * ((size_t)nrec + (size_t)(kFinThreads / 32) * (kFinCols + 1));
}

template <class Dyn>
__global__ void __launch_bounds__(kFinThreads) finalize_kernel(const FinArgs a, const PlantArgs p) {
  extern __shared__ double fsm[];
  constexpr int NW = kFinThreads / 32;
  static_assert(NW <= 32 && (NW & (NW - 1)) == 0, "block reductions: one partial per lane");
  double* se = fsm;                 // e_b = exp(-(rho_b - rho)/lambda), per record
  double* part = fsm + a.nrec;      // [NW][kFinCols + 1] (padded: conflict-free column reads)
  __shared__ double s_red[4][NW];
  __shared__ double s_delta[kFinCols];
  __shared__ double s_unew[kFinCols];  // this CTA's u_new columns (single CTA: the whole sequence)
  __shared__ int s_last;
  __shared__ PlantPre s_pre;
  // batched trials: blockIdx.y selects the trial's records, controls, counter and loop state
  const int trial = blockIdx.y;
  const double* recs = a.rec + (size_t)trial * a.nrec * a.rec_stride;
  const double* const unom = a.u_nom ? a.u_nom + (size_t)trial * a.TM : nullptr;
  double* const unew = a.u_new ? a.u_new + (size_t)trial * a.TM : nullptr;
  unsigned int* const counter = a.counter ? a.counter + trial : nullptr;
  LoopState* L = a.loop ? a.loop + trial : nullptr;
  const double* const unom_in = L ? loop_unom(L, L->step, a.TM) : unom;  // (read before the wait: stable)
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
#ifdef JM_FIN_STAMPS
  long long fin_ts[12];
  int fin_nts = 0;
  FIN_STAMP();
#endif
  // closed loop: LoopState reads and the plant noise do not depend on the
  // rollout, so they run before the grid dependency resolves; so do the
  // nominal controls (written by the previous step's shift / the input copy,
  // both complete before this step's rollout released us) and `halted`
  if (L != nullptr && tid == kFinThreads - 1) plant_prepare<Dyn>(p, s_pre);
  // (the two-level reduce runs without a loop of its own: it stops with the loop it pushes for,
  // so a halted rank no longer re-pushes stale records and raises peers' flags)
  const bool halted = (L != nullptr && L->halted) || (a.push_loop != nullptr && a.push_loop->halted);
  const int c0 = blockIdx.x * a.cols;
  const bool reduce_mode = a.rec_out != nullptr || a.push_peers != nullptr;
  const double unom_c = (!reduce_mode && tid < a.cols && c0 + tid < a.TM) ? unom_in[c0 + tid] : 0.0;
  const uint64_t t_entry = globaltimer();
  grid_dep_wait();
  if (halted) return;
  if (blockIdx.x == 0 && tid == 0 && L != nullptr) {
    unsigned long long* const row = tl_row(L, L->step);
    tl_put(row, kTlFinEntry, t_entry);
    tl_put(row, kTlFinWait);
  }
  const int rs = a.rec_stride;
  FIN_STAMP();
  if (a.wait_flags != nullptr) {  // every rank's CTA records arrive over NVLink (write_record)
    const uint32_t epoch = (uint32_t)L->step + 1u;
    // a peer that never pushes (a dead rank) must not hang the GPU: after 30 s
    // the loop halts with JM_ERR_CUDA instead
    __shared__ int s_timeout;
    if (tid == 0) s_timeout = 0;
    __syncthreads();
    const uint64_t t_begin = globaltimer();
    const int nflags = a.wait_nflags > 0 ? a.wait_nflags : a.nrec;
    for (int r = tid; r < nflags; r += kFinThreads)
      while ((a.wait_gpu ? ld_acquire_gpu(a.wait_flags + r) : ld_acquire_sys(a.wait_flags + r)) < epoch) {
        if (!a.wait_gpu) __nanosleep(32);
        if (globaltimer() - t_begin > 30ull * 1000000000ull) {
          s_timeout = 1;
          break;
        }
      }
    __syncthreads();
    if (s_timeout) {
      if (tid == 0) {
        L->status = 5;  // JM_ERR_CUDA
        L->halted = 1;
      }
      return;
    }
    __threadfence();
    recs += (size_t)(epoch & 1u) * a.nrec * rs;
  }
  // global rho (controller.py:69: min over finite costs) and the rescaled
  // sums in one pass over the record heads (<= 1024 records: one per thread,
  // held in registers).  Block reductions: warp partials -> shared memory ->
  // one barrier -> every warp reduces the 32 partials itself (fixed order, so
  // all warps agree bit for bit), instead of warp 0 + a broadcast barrier.
  double h0 = CUDART_INF, h1 = 0.0, h2 = 0.0, h3 = 0.0;
  const bool one_pass = a.nrec <= kFinThreads;
  double m = CUDART_INF;
  if (one_pass) {
    if (tid < a.nrec) {
      const double* r = recs + (size_t)tid * rs;
      h0 = r[0];
      h1 = r[1];
      h2 = r[2];
      h3 = r[3];
    }
    m = h0;
  } else {
    for (int b = tid; b < a.nrec; b += kFinThreads) m = fmin(m, recs[(size_t)b * rs]);
  }
  // the column pass below reads every record's N block: start those lines
  // towards L1 now (after the head loads are issued), under the reductions
  {
    constexpr int CPL = kFinCols / 32;
    for (int b = warp; b < a.nrec; b += NW) {
      const double* r = recs + (size_t)b * rs + 4;
#pragma unroll
      for (int i = 0; i < CPL; ++i) {
        const int c = c0 + lane + 32 * i;
        if (c < a.TM && lane + 32 * i < a.cols && ((c & 15) == 0 || c == c0 + lane)) asm volatile("prefetch.global.L1 [%0];" ::"l"(r + c));
      }
    }
  }
  m = warp_min_redux(m);
  if (lane == 0) s_red[0][warp] = m;
  __syncthreads();
  const double rho = warp_min_redux(lane < NW ? s_red[0][lane] : CUDART_INF);
  FIN_STAMP();
  double z = 0.0, w2 = 0.0, nf = 0.0;
  if (one_pass) {
    if (tid < a.nrec) {
      const double e = (h0 == CUDART_INF || rho == CUDART_INF) ? 0.0 : exp(-(h0 - rho) * a.inv_lam);
      se[tid] = e;
      z = h1 * e;
      w2 = h2 * e * e;
      nf = h3;
    }
  } else {
    for (int b = tid; b < a.nrec; b += kFinThreads) {
      const double* r = recs + (size_t)b * rs;
      const double e = (r[0] == CUDART_INF || rho == CUDART_INF) ? 0.0 : exp(-(r[0] - rho) * a.inv_lam);
      se[b] = e;
      z += r[1] * e;
      w2 += r[2] * e * e;
      nf += r[3];
    }
  }
  z = warp_sum(z);
  w2 = warp_sum(w2);
  nf = warp_sum(nf);
  if (lane == 0) {
    s_red[1][warp] = z;
    s_red[2][warp] = w2;
    s_red[3][warp] = nf;
  }
  __syncthreads();
  const double Z = warp_sum(lane < NW ? s_red[1][lane] : 0.0), W2 = warp_sum(lane < NW ? s_red[2][lane] : 0.0),
               NF = warp_sum(lane < NW ? s_red[3][lane] : 0.0);
  FIN_STAMP();
  if (rho == CUDART_INF) {  // controller.py:66-67
    if (blockIdx.x == 0 && tid == 0) {
      if (a.status) *a.status = 3;  // JM_ERR_NO_VIABLE
      if (a.diag) *a.diag = DiagOut{CUDART_INF, 0.0, 0.0, 0};
      if (L) {
        L->status = 3;
        L->halted = 1;
      }
      if (a.done != nullptr) {  // the caller only reads the status in this case
        __threadfence_system();
        *a.done = 1;
      }
    }
    if (reduce_mode) {
      fin_emit_record(a, c0, CUDART_INF, 0.0, 0.0, 0.0, nullptr);
      return;
    }
    for (int c = c0 + tid; c < min(c0 + a.cols, a.TM); c += kFinThreads) unew[c] = unom_in[c];
    return;
  }
  // columns: warps split records (several in flight), lanes split columns
  constexpr int CPL = kFinCols / 32;
  double acc[CPL];
#pragma unroll
  for (int i = 0; i < CPL; ++i) acc[i] = 0.0;
#pragma unroll 4
  for (int b = warp; b < a.nrec; b += NW) {
    const double* r = recs + (size_t)b * rs + 4;
    const double e = se[b];
#pragma unroll
    for (int i = 0; i < CPL; ++i) {
      const int c = c0 + lane + 32 * i;
      if (c < a.TM && lane + 32 * i < a.cols) acc[i] = fma(r[c], e, acc[i]);
    }
  }
#pragma unroll
  for (int i = 0; i < CPL; ++i) part[warp * (kFinCols + 1) + lane + 32 * i] = acc[i];
  __syncthreads();
  FIN_STAMP();
  // cross-warp column sums: thread c adds the NW warp partials of column c
  // (consecutive columns: conflict-free) in four interleaved chains, then
  // combines them -- fixed order, no 64-bit shuffle rounds
  if (tid < kFinCols) {
    double v0 = 0.0, v1 = 0.0, v2 = 0.0, v3 = 0.0;
#pragma unroll
    for (int w = 0; w < NW; w += 4) {
      v0 += part[(w + 0) * (kFinCols + 1) + tid];
      if (w + 1 < NW) v1 += part[(w + 1) * (kFinCols + 1) + tid];
      if (w + 2 < NW) v2 += part[(w + 2) * (kFinCols + 1) + tid];
      if (w + 3 < NW) v3 += part[(w + 3) * (kFinCols + 1) + tid];
    }
    s_delta[tid] = (v0 + v1) + (v2 + v3);
  }
  __syncthreads();
  FIN_STAMP();
  if (reduce_mode) {
    fin_emit_record(a, c0, rho, Z, W2, NF, s_delta);
    return;
  }
  // delta = N / (Z sqrt(dt))  (controller.py:158), then mapping (:159-160)
  const double scale = a.inv_sdt / Z;
  double out = 0.0;
  const int c = c0 + tid;
  const int M = a.M;
  if (tid < a.cols && c < a.TM) {
    const int j = c % M, cb = tid - j;
    if (a.mapping) {
      for (int l = 0; l < M; ++l) out = fma(a.mapping[j * M + l], s_delta[cb + l] * scale, out);
    } else {
      out = s_delta[tid] * scale;
    }
  }
  __syncthreads();
  if (tid < a.cols && c < a.TM) {
    s_delta[tid] = out;
    const double un = unom_c + out;  // u_nom + delta, unclamped (controller.py:161)
    s_unew[tid] = un;
    unew[c] = un;
  }
  __syncthreads();
  FIN_STAMP();
  if (a.norms) {  // per_step_update_norm (controller.py:168)
    const int tl = tid, t = c0 / M + tl;
    if (tl < a.cols / M && t * M < a.TM) {
      double s2 = 0.0;
      for (int j = 0; j < M; ++j) s2 += s_delta[tl * M + j] * s_delta[tl * M + j];
      a.norms[t] = sqrt(s2);
    }
  }
  if (blockIdx.x == 0 && tid == 0) {
    if (a.status) *a.status = 0;
    if (a.diag) *a.diag = DiagOut{rho, Z * Z / W2, Z, (int64_t)NF};  // ESS = 1/sum w^2 (:167)
  }
  if (a.u_shift != nullptr && gridDim.x == 1) {  // warm_start_shift of this iteration's result
    const int TM = a.TM, Mm = a.M;
    for (int i = tid; i < TM; i += kFinThreads)
      a.u_shift[i] = (i < TM - Mm) ? s_unew[i + Mm] : a.u_init[i - (TM - Mm)];
#ifdef JM_FIN_STAMPS
    FIN_STAMP();
    __syncthreads();
    if (tid == 0 && a.norms)
      for (int i = 1; i < fin_nts; ++i) a.norms[i - 1] = double(fin_ts[i] - fin_ts[0]);
#endif
    if (a.done != nullptr) {
      __syncthreads();
      if (tid == 0) {
        __threadfence_system();
        *a.done = 1;
      }
    }
  } else if (a.u_shift != nullptr) {
    __threadfence();
    __syncthreads();
    if (tid == 0) s_last = (atomicAdd(counter, 1u) == gridDim.x - 1) ? 1 : 0;
    __syncthreads();
    if (s_last) {
      __threadfence();
      const int TM = a.TM, Mm = a.M;
      for (int i = tid; i < TM; i += kFinThreads)
        a.u_shift[i] = (i < TM - Mm) ? __ldcg(unew + i + Mm) : a.u_init[i - (TM - Mm)];
      if (tid == 0) *counter = 0u;
      if (a.done != nullptr) {
        __syncthreads();
        if (tid == 0) {
          __threadfence_system();
          *a.done = 1;
        }
      }
    }
  }
  if (L != nullptr) {
    if (blockIdx.x == 0 && tid == 0) tl_put(tl_row(L, L->step), kTlFinMerged);
    grid_dep_launch();  // the next control step's rollout may become resident
    if (gridDim.x == 1) {
      plant_finish<Dyn>(p, s_pre, s_unew, false);
      return;
    }
    // several CTAs: the last one to finish runs the plant step + shift
    __threadfence();
    __syncthreads();
    if (tid == 0) s_last = (atomicAdd(counter, 1u) == gridDim.x - 1) ? 1 : 0;
    __syncthreads();
    if (s_last) {
      __threadfence();
      plant_finish<Dyn>(p, s_pre, unew, true);
      if (tid == 0) *counter = 0u;
    }
  }
}

// ---------------------------------------------------------------- noise (write mode)
struct NoiseArgs {
  int K, T, q, jump_on;
  const uint32_t* gap_thr;  // jump-gap survival table (device), T + 1 entries
  float gap_inv;
  int poisson;
  CountTable cnt;
  long long sample_offset;
  uint64_t seed, iteration;
  double Ld[16], Lj[16], mu_j[4];
  // sample-major float64 outputs (host API mirror of sample_noise_batch)
  double* eps_d;
  int64_t* ind;
  double* eps_j;
  double* eps_c;
  // step-major Real outputs (HBM-mode inputs)
  void* eps_c_sm;
  void* jump_sm;
};

// One thread per sample, its jump clock advanced step by step (a utility
// path: the rollout kernels use the cooperative windows instead; both give
// the same events and marks).
template <int M, int JM, int QJ, typename Real>
__global__ void __launch_bounds__(256) noise_kernel(const NoiseArgs a) {
  constexpr int MP = Pad<M>::value;
  constexpr int Q = (JM == 0) ? M : QJ;
  constexpr int QP = Pad<Q>::value;
  const int kl = blockIdx.x * blockDim.x + threadIdx.x;
  if (kl >= a.K) return;
  const uint32_t kg = (uint32_t)(a.sample_offset + kl);
  const StreamKey sk = make_stream_key(a.seed, a.iteration);
  Real Ld[M * M], Lj[Q * Q], mu[Q];
#pragma unroll
  for (int i = 0; i < M * M; ++i) Ld[i] = Real(a.Ld[i]);
#pragma unroll
  for (int i = 0; i < Q * Q; ++i) Lj[i] = Real(a.Lj[i]);
#pragma unroll
  for (int i = 0; i < Q; ++i) mu[i] = Real(a.mu_j[i]);
  const int T = a.T, K = a.K;
  JumpClock clk;
  const GapSampler gs{a.gap_thr, T, a.gap_inv};
  if (a.jump_on) clock_start(clk, sk, kg, gs);
  for (int t0 = 0; t0 < T; t0 += 4) {
    float z[4 * MP];
    group_normals<MP>(sk, (uint32_t)t0, kg, z);
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      const int t = t0 + s;
      if (t >= T) break;
      Real ed[M], ec[M], mk[Q];
      apply_chol<M, Real>(Ld, z + s * MP, ed);
      const bool jump = a.jump_on && t == clk.tj;
      int count = 0;
#pragma unroll
      for (int i = 0; i < Q; ++i) mk[i] = Real(0);
      if (jump) {
        mark_of<Q, QP, Real>(sk, kg, clk.e, Lj, mu, mk, a.poisson != 0, a.cnt);
        count = a.poisson ? event_count(sk, kg, clk.e, a.cnt) : 1;
        clock_next(clk, sk, kg, gs);
      }
#pragma unroll
      for (int j = 0; j < M; ++j) ec[j] = ed[j];
      if (JM == 0 && jump) {
#pragma unroll
        for (int j = 0; j < M; ++j) ec[j] = radd<Real>(ec[j], mk[(j < Q) ? j : 0]);
      }
      const size_t row = (size_t)kl * T + t;
      if (a.eps_d)
#pragma unroll
        for (int j = 0; j < M; ++j) a.eps_d[row * M + j] = double(ed[j]);
      if (a.ind) a.ind[row] = count;  // indicator, or the Poisson arrival count
      if (a.eps_j)
#pragma unroll
        for (int i = 0; i < Q; ++i) a.eps_j[row * Q + i] = jump ? double(mk[i]) : 0.0;
      if (a.eps_c)
#pragma unroll
        for (int j = 0; j < M; ++j) a.eps_c[row * M + j] = double(ec[j]);
      if (a.eps_c_sm)
#pragma unroll
        for (int j = 0; j < M; ++j) reinterpret_cast<Real*>(a.eps_c_sm)[(size_t)(t * M + j) * K + kl] = ec[j];
      if (JM == 1 && a.jump_sm)
#pragma unroll
        for (int i = 0; i < Q; ++i)
          reinterpret_cast<Real*>(a.jump_sm)[(size_t)(t * Q + i) * K + kl] = jump ? mk[i] : Real(0);
    }
  }
}

#ifdef JM_COMMON_KERNELS  // non-template kernels: defined in api.cu only
// ---------------------------------------------------------------- weights
// Output weights = compute_weights (controller.py:62-71) of the returned
// float64 costs: w = exp(-(S - rho)/lambda) normalised by its own float64 sum
// (fixed-order: per-block shuffle trees, then the block sums in order), so they
// sum to 1 to rounding in both compute precisions.
constexpr int kWThreads = 256;
__global__ void weights_exp_kernel(const double* costs, const DiagOut* diag, double inv_lam, int K, double* w,
                                   double* block_sums) {
  __shared__ double s[kWThreads / 32];
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  double e = 0.0;
  if (k < K) {
    const double c = costs[k];
    e = isfinite(c) ? exp(-(c - diag->min_cost) * inv_lam) : 0.0;
    w[k] = e;
  }
  e = warp_sum(e);
  if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = e;
  __syncthreads();
  if (threadIdx.x < 32) {
    double v = threadIdx.x < (kWThreads / 32) ? s[threadIdx.x] : 0.0;
    v = warp_sum(v);
    if (threadIdx.x == 0) block_sums[blockIdx.x] = v;
  }
}

__global__ void weights_norm_kernel(const double* block_sums, int nblocks, int K, double* w) {
  __shared__ double s_z;
  if (threadIdx.x < 32) {
    double z = 0.0;
    for (int b = threadIdx.x; b < nblocks; b += 32) z += block_sums[b];
    z = warp_sum(z);
    if (threadIdx.x == 0) s_z = z;
  }
  __syncthreads();
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < K && s_z > 0.0) w[k] /= s_z;
}

// ---------------------------------------------------------------- zero-copy staging
// The drop-in graph moves its ~1-2 KB input/output blocks with one CTA reading /
// writing pinned host memory directly (UVA) instead of DMA memcpy nodes.
__global__ void copy_block_kernel(const double* __restrict__ src, double* __restrict__ dst, int n) {
  grid_dep_launch();  // the rollout may launch and wait in griddepcontrol.wait meanwhile
  for (int i = threadIdx.x; i < n; i += blockDim.x) dst[i] = src[i];
}

// ---------------------------------------------------------------- shift
__global__ void shift_kernel(const double* u, const double* u_init, int T, int M, double* out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int TM = T * M;
  if (i >= TM) return;
  out[i] = (i < TM - M) ? u[i + M] : u_init[i - (TM - M)];
}

// ---------------------------------------------------------------- microbenchmarks
__global__ void mb_ffma_kernel(float* out, int iters, float b, float c) {
  float a0 = threadIdx.x * 1e-7f, a1 = a0 + 1e-7f, a2 = a0 + 2e-7f, a3 = a0 + 3e-7f;
  float a4 = a0 + 4e-7f, a5 = a0 + 5e-7f, a6 = a0 + 6e-7f, a7 = a0 + 7e-7f;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      a0 = fmaf(a0, b, c); a1 = fmaf(a1, b, c); a2 = fmaf(a2, b, c); a3 = fmaf(a3, b, c);
      a4 = fmaf(a4, b, c); a5 = fmaf(a5, b, c); a6 = fmaf(a6, b, c); a7 = fmaf(a7, b, c);
    }
  }
  const float s = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
  if (s == 12345.678f) out[blockIdx.x] = s;
}

__global__ void mb_mufu_kernel(float* out, int iters) {
  float a0 = threadIdx.x * 1e-9f, a1 = a0 + 1e-9f, a2 = a0 + 2e-9f, a3 = a0 + 3e-9f;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a0));
      asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a1));
      asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a2));
      asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a3));
    }
  }
  const float s = a0 + a1 + a2 + a3;
  if (s == 12345.678f) out[blockIdx.x] = s;
}

__global__ void mb_dfma_kernel(double* out, int iters, double b, double c) {
  double a0 = threadIdx.x * 1e-7, a1 = a0 + 1e-7, a2 = a0 + 2e-7, a3 = a0 + 3e-7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
    }
  }
  const double s = a0 + a1 + a2 + a3;
  if (s == 12345.678) out[blockIdx.x] = s;
}
#endif  // JM_COMMON_KERNELS

}  // namespace jm
