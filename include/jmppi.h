/*
 * jmppi.h -- C ABI of the B200-native sampled-trajectory core of jump-diffusion
 * MPPI (arXiv 1807.06108).
 *
 * The reference (`jump_mppi`, pure Python/numpy) has no FFI.  Its "operator
 * API" for this hot path is the Python controller/plugin contract; every entry
 * point below names the reference function it replaces (paths relative to
 * /root/reference/pkg/src/jump_mppi/).  A Python maintainer binds this header
 * with ctypes; the package `paper_1807_06108_b200` is that
 * binding plus the drop-in mirror of the reference API.
 *
 * Conventions
 *  - Plain C: no torch / CUDA types in signatures.  Streams are passed as
 *    `void*` (a cudaStream_t; NULL = the context's own stream).
 *  - `*_host` entry points take HOST buffers and do every host<->device copy
 *    themselves (the drop-in path).  `*_dev` entry points take DEVICE pointers
 *    and only enqueue work on the stream (the device-resident path used by the
 *    closed loop, the bench and the multi-GPU shard driver).
 *  - Controls, states and diagnostics cross the boundary as float64 (the
 *    reference's dtype).  Bulk per-sample noise tensors are in the context's
 *    compute precision ("Real": float for JM_F32, double for JM_F64).
 *  - Noise tensor wire format ("step-major", the layout of the reference's
 *    step-major copies, controller.py:123-125, transposed so that K is the
 *    contiguous axis): eps[(t*m + j)*K + k], jump[(t*q + i)*K + k].
 *  - Every function returns a jm_status; jm_last_error() gives the message.
 *    Status -> reference exception mapping is documented per code.
 */
#ifndef JMPPI_H
#define JMPPI_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define JM_ABI_VERSION 5
#define JM_MAX_STATE 12
#define JM_MAX_CONTROL 4
#define JM_MAX_JUMP 4

typedef enum {
  JM_OK = 0,
  JM_ERR_CONFIG = 1,       /* -> ConfigError          (types.py:23-28, :116-121)       */
  JM_ERR_VALUE = 2,        /* -> ValueError           (noise.py:148-149 zero-one law)   */
  JM_ERR_NO_VIABLE = 3,    /* -> ControllerError("no viable rollout") (controller.py:66-67) */
  JM_ERR_NOISE = 4,        /* -> NoiseError           (noise.py:63-68, non-PD covariance) */
  JM_ERR_CUDA = 5,         /* CUDA runtime failure (no reference analogue)              */
  JM_ERR_UNSUPPORTED = 6,  /* plugin / shape this build has no kernel for              */
  JM_ERR_DIVERGED = 7      /* -> StateDivergedError  (dynamics.py:29-33), plant only    */
} jm_status;

typedef enum { JM_MODEL_INTEGRATOR = 0, JM_MODEL_CARTPOLE = 1, JM_MODEL_QUADROTOR = 2, JM_MODEL_LINEAR = 3 } jm_model_kind;
typedef enum {
  JM_COST_DIAG_QUADRATIC = 0,   /* q = sum_i w_i (x_i - x*_i)^2 (conftest quadratic_q, BASELINE cartpole) */
  JM_COST_CARTPOLE_SWINGUP = 1, /* CartpoleStateCost, costs.py:149-168                                  */
  JM_COST_QUADROTOR_HOVER = 2   /* QuadrotorStateCost, costs.py:171-190                                 */
} jm_cost_kind;
typedef enum {
  JM_JUMP_CONTROL = 0,  /* B = H = G, marks folded into eps_combined (dynamics.py:274-283, noise.py:156-157) */
  JM_JUMP_STATE = 1     /* H = constant state selector; eps_combined = eps_d           */
} jm_jump_channel;
typedef enum { JM_NOISE_PHILOX = 0, JM_NOISE_HBM = 1 } jm_noise_source;
typedef enum { JM_F32 = 0, JM_F64 = 1 } jm_precision;
/* Jump arrivals per (sample, step): the reference's zero-one law (an indicator
 * U < nu dt, noise.py:151), or Poisson(nu dt) counts whose marks add up
 * (compound Poisson; BASELINE north star "Poisson jump counts per step"). */
typedef enum { JM_JUMPS_BERNOULLI = 0, JM_JUMPS_POISSON = 1 } jm_jump_process;

/* Replaces the DynamicsModel plugin (dynamics.py:45-65) built by
 * cartpole_dynamics (:264-284) / quadrotor_dynamics (:389-409). */
typedef struct {
  int32_t kind;               /* jm_model_kind */
  int32_t state_dim;          /* n */
  int32_t control_dim;        /* m */
  int32_t has_limits;         /* control_limits is not None (dynamics.py:55, :61-65) */
  double params[8];           /* cartpole: mc, mp, l, g (:196-199); quadrotor: mass, arm, ixx, iyy, izz, g (:298-301) */
  double u_lo[JM_MAX_CONTROL];
  double u_hi[JM_MAX_CONTROL];
  int32_t jump_channel;       /* jm_jump_channel */
  int32_t jump_dim;           /* q (== m for JM_JUMP_CONTROL) */
  int32_t jump_rows[JM_MAX_JUMP]; /* JM_JUMP_STATE: state rows hit by the jump (H selector) */
  int32_t jump_scale_unit;    /* 1: O(1) jump increment ("unit", dynamics.py:111); 0: sqrt(dt) */
  /* JM_MODEL_LINEAR: a generic linear plugin f(x) = A x, G constant, B = H = G
   * (a DynamicsModel with drift = A @ x and constant control/diffusion/jump
   * matrices, noise_through_controls=True); (n, m) in {(2,1), (4,1), (4,2), (6,3)} */
  int32_t pad_lin_;
  double lin_A[JM_MAX_STATE * JM_MAX_STATE]; /* row-major n x n */
  double lin_G[JM_MAX_STATE * JM_MAX_CONTROL]; /* row-major n x m */
} jm_model_desc;

/* Replaces the CostModel plugin (costs.py:28-56) with its state/terminal cost
 * callables (costs.py:149-201). */
typedef struct {
  int32_t kind;               /* jm_cost_kind */
  int32_t pad_;
  double weights[JM_MAX_STATE];  /* swing-up: w_pos, w_vel, w_angle, w_avel; hover: w_pos, w_vel, w_att, w_rate; diag: per-state */
  double target[JM_MAX_STATE];   /* hover: waypoint (3); diag: x* (n) */
  double terminal_scale;      /* ScaledTerminalCost.scale (costs.py:193-201) */
  double R[JM_MAX_CONTROL * JM_MAX_CONTROL]; /* control_cost_matrix, row-major m x m */
  double lambda_;             /* CostModel.lambda_ */
  double c;                   /* CostModel.c */
  /* CostModel.control_channel == False (costs.py:50-54, :112-124): the
   * correction matrices of the modified running cost.  The noise enters
   * through B with as many components as controls (p = m). */
  int32_t general_channel;    /* 0: control channel (cal_b = bb = I) */
  int32_t pad2_;
  double cal_b[JM_MAX_CONTROL * JM_MAX_CONTROL]; /* G' Sigma^-1 B, row-major m x p */
  double bb[JM_MAX_CONTROL * JM_MAX_CONTROL];    /* B' Sigma^-1 B, row-major p x p */
} jm_cost_desc;

/* Replaces MppiConfig (types.py:57-87) plus the sampler extensions the
 * BASELINE configs need (mark mean, Poisson arrival counts). */
typedef struct {
  double lambda_, c, dt, nu;
  int32_t horizon;            /* T = horizon_n */
  int32_t samples;            /* K = samples_m handled by this context (the local shard) */
  int32_t control_dim;        /* m */
  int32_t jump_enabled;       /* jump_sampling_enabled (types.py:76) */
  double sigma_d[JM_MAX_CONTROL * JM_MAX_CONTROL]; /* m x m, row-major */
  double sigma_j[JM_MAX_JUMP * JM_MAX_JUMP];       /* q x q, row-major */
  double mark_mean[JM_MAX_JUMP];                   /* 0 in the reference (noise.py:150-155) */
  int32_t precision;          /* jm_precision */
  int32_t noise_source;       /* jm_noise_source */
  int64_t sample_offset;      /* global index of local sample 0 (multi-GPU shards) */
  int32_t block_threads;      /* 0 = auto */
  int32_t jump_process;       /* jm_jump_process: arrivals per jump step */
} jm_mppi_desc;

/* UpdateDiagnostics scalars (controller.py:48-53). */
typedef struct {
  double min_cost;            /* rho = min over finite costs */
  double ess;                 /* 1 / sum w^2 */
  double normaliser;          /* Z = sum exp(-(S-rho)/lambda) */
  int64_t n_finite;           /* samples with finite cost */
} jm_diag;

typedef struct jm_ctx jm_ctx;

int jm_abi_version(void);
const char* jm_last_error(const jm_ctx* ctx);   /* NULL ctx -> thread-global last error */
int jm_device_count(int* out);

/* Construction: validates the config (types.py:90-121: lambda>0, c>=1, dt>0,
 * nu>=0, nu*dt<0.1, SPD covariances), factors c*Sigma_D and Sigma_J
 * (noise.py:63-68, :143-145), allocates device workspace for K samples. */
int jm_create(const jm_model_desc* model, const jm_cost_desc* cost, const jm_mppi_desc* mppi,
              int device, jm_ctx** out);
int jm_destroy(jm_ctx* ctx);
/* stream: a cudaStream_t; NULL = the context's own non-blocking stream (the
 * legacy default stream 0 cannot be selected: pass an explicit stream). */
int jm_set_stream(jm_ctx* ctx, void* stream);
/* size in doubles of one weighting record: 4 + T*m (rho, Z, sum w^2, n_finite, N[T*m]) */
int jm_record_doubles(const jm_ctx* ctx, int64_t* out);

/* ---- one MPC iteration: replaces mppi_iteration (controller.py:103-181) ----
 * x0 (n), u_nom (T*m) float64.  eps_c / jump: NULL in Philox mode; in HBM
 * mode the step-major noise tensors described above (jump only for
 * JM_JUMP_STATE).  mapping: m x m or NULL (controller.py:159-160).
 * Outputs (any may be NULL except u_new): u_new (T*m) = u_nom + delta;
 * costs (K); weights (K); step_norms (T) = per_step_update_norm;
 * states (K*(T+1)*n) + diverged_step (K, -1 if alive) = return_rollouts. */
int jm_iteration_host(jm_ctx* ctx, const double* x0, const double* u_nom, uint64_t seed,
                      uint64_t iteration, const void* eps_c, const void* jump,
                      const double* mapping, double* u_new, double* costs, double* weights,
                      double* step_norms, double* states, int64_t* diverged_step, jm_diag* diag,
                      const double* u_init, double* u_shift, uint64_t* weights_stash);
/* Extra outputs of jm_iteration_host:
 *  u_init (m) + u_shift (T*m): warm_start_shift(u_new, u_init) (controller.py:96-100)
 *    computed by the same finalize kernel;
 *  weights_stash: the per-sample costs stay in a device buffer identified by
 *    the returned handle; jm_stash_fetch forms the weights from them with the
 *    iteration's min_cost and normaliser (jm_diag) and downloads them;
 *    jm_stash_release frees the slot -- the drop-in API's lazy
 *    UpdateDiagnostics.weights. */
int jm_stash_fetch(jm_ctx* ctx, uint64_t handle, double min_cost, double normaliser, double* host);
int jm_stash_release(jm_ctx* ctx, uint64_t handle);

/* The drop-in call in its compact form (jump_mppi.mppi_iteration followed by
 * warm_start_shift, controller.py:103-181 + :96-100, Philox noise, no
 * mapping): the same work as jm_iteration_host(..., u_init, u_shift,
 * weights_stash) with one output block
 *   out = [u_new (T*m) | step_norms (T) | min_cost, ess, normaliser, n_finite
 *          (int64 bits) | status, pad (2 words) | u_shift (T*m)]
 * (jm_dropin_doubles() doubles), so a binding passes 4 pointers. */
int jm_iteration_dropin(jm_ctx* ctx, const double* x0, const double* u_nom, const double* u_init,
                        uint64_t seed, uint64_t iteration, double* out, uint64_t* weights_stash);
int64_t jm_dropin_doubles(const jm_ctx* ctx);

/* Upload x0 (n) and u_nom (T*m) into the context's device inputs (used by
 * jm_bench_iteration; jm_iteration_host does this itself). */
int jm_upload_inputs(jm_ctx* ctx, const double* x0, const double* u_nom);

/* Device-resident split of the same iteration (all pointers device memory).
 * 1) rollout: K1 noise + K2 fused rollout/cost + per-CTA K3/K4 partials.
 *    iteration_dev may be NULL (then `iteration` is used).  */
int jm_rollout_dev(jm_ctx* ctx, const double* x0_dev, const double* u_nom_dev, uint64_t seed,
                   uint64_t iteration, const uint64_t* iteration_dev, const void* eps_c_dev,
                   const void* jump_dev, double* costs_dev, double* states_dev,
                   int64_t* diverged_dev);
/* 2) reduce the per-CTA partials into one record (for the cross-GPU exchange). */
int jm_reduce_dev(jm_ctx* ctx, double* record_dev);
/* 3) combine nrec records (NULL = this context's own CTA partials) and apply
 *    the update; diag_dev receives a jm_diag, status_dev an int32 jm_status. */
int jm_finalize_dev(jm_ctx* ctx, const double* records_dev, int32_t nrec, const double* u_nom_dev,
                    const double* mapping_dev, double* u_new_dev, double* step_norms_dev,
                    jm_diag* diag_dev, int32_t* status_dev);
/* 4) per-sample weights from costs + the final record (controller.py:62-71). */
int jm_weights_dev(jm_ctx* ctx, const double* costs_dev, const jm_diag* diag_dev, double* weights_dev);

/* warm_start_shift (controller.py:96-100) on device: out[t] = u[t+1], out[T-1] = u_init. */
int jm_shift_dev(jm_ctx* ctx, const double* u_dev, const double* u_init_dev, double* out_dev);

/* warm_start_shift (controller.py:96-100) on host buffers (device kernel). */
int jm_shift_host(int device, int32_t T, int32_t m, const double* u, const double* u_init,
                  double* out);

/* compute_weights (controller.py:62-71) on device, float64, host buffers.
 * Returns JM_ERR_NO_VIABLE if no cost is finite. */
int jm_compute_weights_host(int device, int64_t K, const double* costs, double lambda_,
                            double* weights);
/* update_controls (controller.py:81-93): weights of costs (K), then
 * u_new = u_nom + (sum_k w_k eps[k]) / sqrt(dt) (@ mapping^T) with eps the
 * stacked eps_combined (K, T, m) sample-major float64 host, as the reference
 * stacks them (controller.py:89). */
int jm_update_controls_host(int device, int64_t K, int32_t T, int32_t m, const double* costs,
                            const double* eps_c, double lambda_, double dt, const double* u_nom,
                            const double* mapping, double* u_new, double* weights);

/* sample_noise_batch (noise.py:129-161) with the on-device Philox stream:
 * eps_d/eps_j/eps_c (K*T*m, sample-major like the reference, float64 host),
 * indicators (K*T int64).  Any output may be NULL. */
int jm_sample_noise_host(jm_ctx* ctx, uint64_t seed, uint64_t iteration, double* eps_d,
                         int64_t* indicators, double* eps_j, double* eps_c);
/* Same, device-resident, step-major, Real-typed (feeds HBM mode). */
int jm_sample_noise_dev(jm_ctx* ctx, uint64_t seed, uint64_t iteration, void* eps_c_dev,
                        void* jump_dev);

/* ---- closed loop on device: replaces run_trial's loop body (harness.py:131-150)
 * Per control step: iteration, u0 = clamp(u_new[0]), plant noise from the plant
 * stream (Sigma_D, not c*Sigma_D; harness.py:123,137-139), Euler step with
 * divergence check, warm_start_shift, iteration += 1.  Captured once into a
 * CUDA graph and replayed.  Host outputs: states ((steps+1)*n), controls
 * (steps*m), jumps (steps), step_ns (steps, device-clock time per iteration),
 * *diverged_at (-1 if none), *status (jm_status of the loop). */
int jm_closed_loop_host(jm_ctx* ctx, const double* x0, const double* u_init, uint64_t seed,
                        int32_t steps, double* states, double* controls, int64_t* jumps,
                        double* step_ns, int32_t* diverged_at, int32_t* status);

/* Device-resident closed loop for the bench / shard driver: the context owns
 * one loop (plant state, warm-started nominal sequence, histories of up to
 * max_steps steps) and one captured CUDA graph of a control step.
 * init uploads x0/u_init (host) and captures; step enqueues one graph launch
 * (no host sync); read synchronises and returns the plant state. */
int jm_loop_init(jm_ctx* ctx, const double* x0, const double* u_init, uint64_t seed,
                 uint64_t first_iteration, int32_t max_steps);
int jm_loop_step(jm_ctx* ctx);
int jm_loop_read(jm_ctx* ctx, double* x_out, uint64_t* iteration_out, int32_t* step_out,
                 int32_t* halted_out, int32_t* status_out);
/* Raw loop histories of the first `steps` control steps: states ((steps+1)*n),
 * controls (steps*m), jumps (steps); synchronises the context's stream. */
int jm_loop_history(jm_ctx* ctx, int32_t steps, double* states, double* controls, int64_t* jumps);
/* Tuning instrumentation: %globaltimer stamps (ns) of the first `steps` loop steps,
 * 12 per step (kernel entries / grid-dependency waits / horizon ends of the rollout
 * and finalize kernels, kernels.cuh kTl*); JM_ERR_UNSUPPORTED unless the
 * environment had JM_TIMELINE set when jm_loop_init ran. */
int jm_loop_timeline(jm_ctx* ctx, int32_t steps, uint64_t* out);

/* Closed-loop control step split around a cross-GPU exchange (one process per
 * GPU, samples sharded by mppi.sample_offset): stage 1 = rollout of the local
 * shard + reduction into one weighting record; stage 2 = merge nrec gathered
 * records (rank order), update, plant step, shift.  Both enqueue on the
 * context's stream (jm_set_stream: share it with the collective). */
int jm_loop_rollout(jm_ctx* ctx, double* record_dev);
int jm_loop_finish(jm_ctx* ctx, const double* records_dev, int32_t nrec);

/* Batched closed-loop trials (run_batch, harness.py:197-233, with the process
 * pool replaced by a trial dimension on the GPU): `trials` (<= 128) independent
 * run_trial loops of `steps` control steps, trial b from x0[b*n..] with
 * master seed seeds[b], all advanced by the same two launches per control
 * step (grid.y = trial).  sampler_jumps[b] = 0 makes trial b's sampler draw
 * no jumps -- the "old" controller variant (jump_sampling_enabled = False,
 * harness.py:218-221) -- so both variants of a paired batch run as ONE batch
 * (NULL: every trial as the context's config says).  Each trial's outputs equal a jm_closed_loop_host
 * run with its seed, bit for bit.  Outputs are trial-major:
 * states (trials, steps+1, n), controls (trials, steps, m), jumps (trials,
 * steps), step_ns (trials, steps), diverged_at / status (trials); any may be
 * NULL.  A trial halts on its own (divergence, no viable rollout) without
 * stopping the others. */
int jm_batch_loop_host(jm_ctx* ctx, int32_t trials, const double* x0, const double* u_init,
                       const uint64_t* seeds, const int32_t* sampler_jumps, int32_t steps, double* states,
                       double* controls, int64_t* jumps, double* step_ns, int32_t* diverged_at, int32_t* status);

/* Peer-memory record exchange -- the multi-GPU step without a collective.
 * Every rank owns a symmetric buffer (e.g. torch.distributed._symmetric_memory)
 * of jm_peer_buffer_doubles(ctx, world) doubles, zeroed before the first step,
 * whose base addresses on all ranks (device-addressable peer pointers over
 * NVLink) are in peer_bases_dev (world entries, device memory).
 * jm_loop_rollout_push: the rollout kernel's CTAs store their weighting
 * records straight into every rank's buffer (slot rank x grid + cta) and raise
 * their epoch flags there -- the exchange is fused into the compute kernel and
 * overlaps its slower CTAs.  jm_loop_finish_peers: the finalize waits on its
 * own buffer's flags on the device, merges the world x grid records in rank
 * order, updates, steps the plant and shifts.  Stream-ordered, no host wait,
 * graph-capturable; the epoch is the loop's step counter. */
int64_t jm_peer_buffer_doubles(const jm_ctx* ctx, int32_t world);
int jm_loop_rollout_push(jm_ctx* ctx, const unsigned long long* peer_bases_dev, int32_t rank, int32_t world);
int jm_loop_finish_peers(jm_ctx* ctx, const double* my_buffer_dev, int32_t world);
/* Two-level form of the same exchange (large worlds, where merging world x grid
 * CTA records outgrows the finalize): the rollout, then a reduce of this rank's
 * CTA records into ONE record (the NCCL transport's jm_loop_rollout reduce,
 * bit for bit) stored into slot `rank` of every peer buffer with its epoch
 * flags; the finish waits on world x ceil(T*m/128) flags and merges `world`
 * records.  Same buffer (jm_peer_buffer_doubles(ctx, world) doubles, zeroed).
 * Replaces the same reference step as jm_loop_rollout_push/_finish_peers. */
int jm_loop_rollout_reduce_push(jm_ctx* ctx, const unsigned long long* peer_bases_dev, int32_t rank, int32_t world);
int jm_loop_finish_reduced_peers(jm_ctx* ctx, const double* my_buffer_dev, int32_t world);

/* ---- measurement helpers ---- */
/* Time `steps` closed-loop control steps (jm_loop_init first) with CUDA events
 * on the context's stream; before each step a cudaMemsetAsync of flush_bytes
 * (> L2) evicts the L2.  use_graph=2: all steps captured into ONE graph
 * (flush, event, step kernels, event per step -- the device-resident loop
 * without per-step host launches); use_graph=1: one graph launch per step;
 * use_graph=0: direct launches, step_ms and rollout_ms (the rollout kernel
 * alone).  Either output may be NULL. */
int jm_bench_loop(jm_ctx* ctx, int32_t steps, int64_t flush_bytes, int32_t use_graph, double* step_ms,
                  double* rollout_ms);
/* Time `reps` device-resident iterations (rollout + finalize, no host copies)
 * from the context's current x0/u_nom; HBM mode first fills device noise
 * tensors from the Philox sampler.  iter_ms / rollout_ms per rep; with
 * rollout_ms NULL no event separates the two kernels (the timed path keeps
 * the programmatic-dependent-launch overlap). */
int jm_bench_iteration(jm_ctx* ctx, int32_t reps, int64_t flush_bytes, double* iter_ms, double* rollout_ms);
/* FP32 FFMA and MUFU throughput microbenchmarks (the roofline denominators
 * SURVEY 8(d) asks to measure): returns TFLOP/s and Tops/s. */
int jm_microbench(int device, double* fp32_tflops, double* mufu_tops, double* fp64_tflops);
/* The non-trace rollout kernel variant this context launches (the one the bench
 * times): "<kernel>/<noise>/<shape>/<precision>", e.g.
 * "rollout_kernel/philox/single_wave_smem/f32" (ncu -k regex:<kernel>). */
const char* jm_kernel_name(const jm_ctx* ctx);
/* Cumulative bytes this process has moved host->device / device->host through the
 * library (explicit copies and the drop-in graph's zero-copy blocks); bench.py's
 * e2e h2d/d2h_bytes_per_step are differences of these counters. */
int jm_transfer_bytes(int64_t* h2d, int64_t* d2h);
/* Number of kernel launches one jm_iteration_host / loop step enqueues. */
int jm_launches_per_iteration(const jm_ctx* ctx, int32_t* iteration, int32_t* loop_step);

#ifdef __cplusplus
}
#endif
#endif /* JMPPI_H */
