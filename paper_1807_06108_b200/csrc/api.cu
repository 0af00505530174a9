// api.cu -- the extern "C" boundary (include/jmppi.h).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>
#include <atomic>
#include <chrono>

#define JM_COMMON_KERNELS
#include "internal.h"

using jm::DiagOut;
using jm::LoopState;

namespace {

thread_local std::string g_err;

// host<->device copy counters (jm_transfer_bytes): every explicit copy the library issues goes
// through these wrappers; the drop-in graph's zero-copy blocks are counted in dropin_launch
std::atomic<long long> g_h2d{0}, g_d2h{0};
inline void count_xfer(size_t n, cudaMemcpyKind k) {
  if (k == cudaMemcpyHostToDevice) g_h2d += (long long)n;
  if (k == cudaMemcpyDeviceToHost) g_d2h += (long long)n;
}
inline cudaError_t xferAsync(void* d, const void* s, size_t n, cudaMemcpyKind k, cudaStream_t st) {
  count_xfer(n, k);
  return cudaMemcpyAsync(d, s, n, k, st);
}
inline cudaError_t xferSync(void* d, const void* s, size_t n, cudaMemcpyKind k) {
  count_xfer(n, k);
  return cudaMemcpy(d, s, n, k);
}

int fail(jm_ctx* c, int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  if (c) c->err = buf;
  return code;
}

#define CK(expr)                                                                          \
  do {                                                                                    \
    cudaError_t e_ = (expr);                                                              \
    if (e_ != cudaSuccess)                                                                \
      return fail(ctx, JM_ERR_CUDA, "%s: %s (%s:%d)", #expr, cudaGetErrorString(e_), __FILE__, \
                  __LINE__);                                                              \
  } while (0)

// Lower Cholesky of an n x n row-major matrix (reads the lower triangle, like
// numpy.linalg.cholesky / LAPACK potrf 'L'; noise.py:63-68).
bool cholesky(const double* A, int n, double* L) {
  for (int i = 0; i < 16; ++i) L[i] = 0.0;
  for (int i = 0; i < n; ++i) {
    for (int j = 0; j <= i; ++j) {
      double s = A[i * n + j];
      for (int k = 0; k < j; ++k) s -= L[i * n + k] * L[j * n + k];
      if (i == j) {
        if (!(s > 0.0) || !std::isfinite(s)) return false;
        L[i * n + i] = std::sqrt(s);
      } else {
        L[i * n + j] = s / L[j * n + j];
      }
    }
  }
  return true;
}

uint32_t jump_threshold(double p) {
  // jump iff (word >> 8) * 2^-24 < p  <=>  word < ceil(p 2^24) << 8
  if (!(p > 0.0)) return 0u;
  double thr = std::ceil(p * 16777216.0);
  if (thr > 16777215.0) thr = 16777215.0;
  return ((uint32_t)thr) << 8;
}

// Per-step probability of a jump event: the zero-one law's nu dt, or
// P(N >= 1) = 1 - exp(-nu dt) for Poisson(nu dt) arrivals.
double event_probability(double nu_dt, bool poisson) { return poisson ? -std::expm1(-nu_dt) : nu_dt; }

// Poisson(lam) tail P(N > k) as the forward sum of the next 40 pmf terms
// (the oracle restates this exact order, oracle/philox_stream.py).
double poisson_tail(double lam, int k) {
  double term = std::exp(-lam);
  for (int j = 1; j <= k; ++j) term *= lam / j;
  double s = 0.0;
  for (int j = k + 1; j <= k + 40; ++j) {
    term *= lam / j;
    s += term;
  }
  return s;
}

// Count thresholds: event arrivals n = 1 + #{k : u24 < c[k-1]},
// c[k-1] = floor(2^24 P(N > k) / P(N >= 1)); plant arrivals (no conditioning)
// n = #{k : u24 < p[k]}, p[0] = ceil(P(N >= 1) 2^24) (the event threshold),
// p[k] = floor(2^24 P(N > k)).
void count_tables(double lam, jm::CountTable* ev, uint32_t* plant) {
  const double p1 = -std::expm1(-lam);
  for (int k = 1; k <= jm::kMaxCount; ++k) {
    const double t = poisson_tail(lam, k);
    ev->c[k - 1] = p1 > 0.0 ? (uint32_t)std::floor(t / p1 * 16777216.0) : 0u;
    plant[k] = (uint32_t)std::floor(t * 16777216.0);
  }
  plant[0] = jump_threshold(p1) >> 8;
}

// Survival table of the geometric jump gaps (philox.cuh, slot 1):
// S[0] = 2^24, S[g] = floor(S[g-1] (2^24 - q) / 2^24), q = ceil(p 2^24), g <= T;
// *inv = 1 / log2((2^24 - q) / 2^24) for the sampler's first guess.
std::vector<uint32_t> gap_table(double p, int T, float* inv) {
  const double qd = p > 0.0 ? std::min(std::ceil(p * 16777216.0), 16777216.0) : 0.0;
  const uint64_t keep = (1ull << 24) - (uint64_t)qd;
  std::vector<uint32_t> S((size_t)T + 1, 0u);
  S[0] = 1u << 24;
  for (int g = 1; g <= T; ++g) S[g] = (uint32_t)(((uint64_t)S[g - 1] * keep) >> 24);
  *inv = (float)(1.0 / std::log2((double)keep / 16777216.0));
  return S;
}

template <typename T>
cudaError_t dalloc(T** p, size_t count) {
  *p = nullptr;
  if (count == 0) return cudaSuccess;
  return cudaMalloc(reinterpret_cast<void**>(p), count * sizeof(T));
}

void dfree(void* p) {
  if (p) cudaFree(p);
}

// ---------------------------------------------------------------- update_controls kernels
// compute_weights (controller.py:62-71): one CTA, fixed-order reduction.
__global__ void cw_kernel(const double* costs, int64_t K, double inv_lam, double* w, double* out2) {
  __shared__ double s[1024];
  __shared__ double s_rho;
  const int tid = threadIdx.x;
  double m = CUDART_INF;
  for (int64_t k = tid; k < K; k += blockDim.x) {
    const double c = costs[k];
    if (isfinite(c)) m = fmin(m, c);
  }
  s[tid] = m;
  __syncthreads();
  if (tid == 0) {
    double mm = CUDART_INF;
    for (int i = 0; i < (int)blockDim.x; ++i) mm = fmin(mm, s[i]);
    s_rho = mm;
  }
  __syncthreads();
  const double rho = s_rho;
  double z = 0.0;
  for (int64_t k = tid; k < K; k += blockDim.x) {
    const double c = costs[k];
    const double e = (isfinite(c) && rho != CUDART_INF) ? exp(-(c - rho) * inv_lam) : 0.0;
    w[k] = e;
    z += e;
  }
  __syncthreads();
  s[tid] = z;
  __syncthreads();
  if (tid == 0) {
    double zz = 0.0;
    for (int i = 0; i < (int)blockDim.x; ++i) zz += s[i];
    out2[0] = rho;
    out2[1] = zz;
  }
  __syncthreads();
  const double Z = out2[1];
  for (int64_t k = tid; k < K; k += blockDim.x) w[k] = (Z > 0.0) ? w[k] / Z : 0.0;
}

// _weighted_noise_average + update (controller.py:74-93): column r of the
// stacked (K, T*m) eps, fixed k order.
__global__ void wavg_kernel(const double* w, const double* eps, int64_t K, int TM, int M,
                            double inv_sdt, const double* u_nom, const double* mapping,
                            double* u_new) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t * M >= TM) return;
  double d[4] = {0, 0, 0, 0};
  for (int64_t k = 0; k < K; ++k) {
    const double wk = w[k];
    for (int j = 0; j < M; ++j) d[j] = fma(wk, eps[k * TM + t * M + j], d[j]);
  }
  for (int j = 0; j < M; ++j) {
    double out = 0.0;
    if (mapping) {
      for (int l = 0; l < M; ++l) out += (d[l] * inv_sdt) * mapping[j * M + l];
    } else {
      out = d[j] * inv_sdt;
    }
    u_new[t * M + j] = u_nom[t * M + j] + out;
  }
}

jm::FinArgs fin_args(const jm_ctx* ctx, const double* records, int nrec) {
  jm::FinArgs f{};
  f.rec = records ? records : ctx->d_records;
  f.nrec = records ? nrec : ctx->grid;
  f.rec_stride = ctx->rec_stride;
  f.TM = ctx->TM;
  f.M = ctx->M;
  f.cols = jm::fin_cols(ctx->M);
  f.inv_lam = 1.0 / ctx->mppi.lambda_;
  f.inv_sdt = 1.0 / std::sqrt(ctx->mppi.dt);
  return f;
}

// weights of `costs` into `w` (2 launches; scratch = ctx->d_wsum)
cudaError_t launch_weights(jm_ctx* ctx, const double* costs, const DiagOut* diag, double* w) {
  const int b = jm::kWThreads, g = (ctx->K + b - 1) / b;
  jm::weights_exp_kernel<<<g, b, 0, ctx->stream>>>(costs, diag, 1.0 / ctx->mppi.lambda_, ctx->K, w, ctx->d_wsum);
  jm::weights_norm_kernel<<<g, b, 0, ctx->stream>>>(ctx->d_wsum, g, ctx->K, w);
  return cudaGetLastError();
}

int rollout_and_finalize(jm_ctx* ctx, const jm::RolloutCall& rc, const double* mapping_dev,
                         double* weights_dev, bool want_shift) {
  CK(ctx->eng->rollout(ctx, rc));
  jm::FinArgs f = fin_args(ctx, nullptr, 0);
  f.u_nom = rc.u_nom;
  f.mapping = mapping_dev;
  f.u_new = ctx->d_small + ctx->off_unew();
  f.norms = ctx->d_small + ctx->off_norms();
  f.diag = ctx->d_diag();
  f.status = ctx->d_status();
  if (want_shift) {
    f.u_init = ctx->d_small + ctx->off_uinit();
    f.u_shift = ctx->d_small + ctx->off_ushift();
  }
  CK(ctx->eng->finalize(ctx, f, nullptr, nullptr));
  if (weights_dev) CK(launch_weights(ctx, ctx->d_costs, ctx->d_diag(), weights_dev));
  return JM_OK;
}

int stash_acquire(jm_ctx* ctx, uint64_t* handle) {
  if (ctx->stash_free.empty()) {
    double* b = nullptr;
    CK(dalloc(&b, (size_t)ctx->K));
    ctx->stash.push_back(b);
    ctx->stash_free.push_back((int)ctx->stash.size() - 1);
  }
  const int i = ctx->stash_free.back();
  ctx->stash_free.pop_back();
  *handle = (uint64_t)i + 1;
  return JM_OK;
}

// One drop-in iteration as a static CUDA graph: a one-CTA copy of the staged
// input block from pinned host memory (zero-copy reads), the rollout (costs
// straight into the stash buffer named in the block), and the finalize
// (+shift), which writes its outputs straight into the pinned host block and
// raises a done word there last -- the host spins on that word instead of a
// stream synchronisation.  Weights are formed from the stashed costs when
// first read (jm_stash_fetch).  seed / iteration / stash pointer travel in the
// staged block (x0 slots 13 and 15), so replays need no parameter updates; the master
// seed is a kernel parameter (uniform-register Philox keys): one graph per seed, a few
// kept (a controller keeps its seed: run_trial, the CLI bench loop).
constexpr size_t kIterGraphs = 8;
// the drop-in iteration's three launches on ctx->stream: one-CTA zero-copy read of the staged
// input block, rollout (costs straight into the stash buffer the block names), finalize
// writing its outputs and the done word into the pinned block
cudaError_t enqueue_dropin_iteration(jm_ctx* ctx, uint64_t seed) {
  double* ds = ctx->d_small;
  double* hs = ctx->h_small;
  uint64_t* words = reinterpret_cast<uint64_t*>(ds + ctx->off_x0());
  jm::copy_block_kernel<<<1, 256, 0, ctx->stream>>>(hs, ds, (int)ctx->off_unew());
  cudaError_t e = cudaGetLastError();
  jm::RolloutCall rc;
  rc.x0 = ds + ctx->off_x0();
  rc.u_nom = ds + ctx->off_unom();
  rc.seed = seed;
  rc.iteration_dev = words + 15;
  rc.costs_dev = reinterpret_cast<double* const*>(words + 13);  // costs straight into the stash buffer
  if (e == cudaSuccess) e = ctx->eng->rollout(ctx, rc);
  if (e == cudaSuccess) {
    jm::FinArgs f = fin_args(ctx, nullptr, 0);
    f.u_nom = rc.u_nom;
    f.u_new = hs + ctx->off_unew();  // zero-copy outputs (UVA: pinned host memory is device-addressable)
    f.norms = hs + ctx->off_norms();
    f.diag = reinterpret_cast<jm::DiagOut*>(hs + ctx->off_diag());
    f.status = reinterpret_cast<int32_t*>(hs + ctx->off_status());
    f.u_init = ds + ctx->off_uinit();
    f.u_shift = hs + ctx->off_ushift();
    f.done = reinterpret_cast<int32_t*>(hs + ctx->off_status()) + 1;
    e = ctx->eng->finalize(ctx, f, nullptr, nullptr);
  }
  return e;
}

int capture_iteration_graph(jm_ctx* ctx, uint64_t seed, cudaGraphExec_t* out) {
  auto& v = ctx->iter_execs;
  for (size_t i = 0; i < v.size(); ++i)
    if (v[i].first == seed) {
      *out = v[i].second;
      if (i + 1 != v.size()) std::rotate(v.begin() + i, v.begin() + i + 1, v.end());  // most recent last
      return JM_OK;
    }
  if (v.size() >= kIterGraphs) {
    cudaGraphExecDestroy(v.front().second);
    v.erase(v.begin());
  }
  cudaStream_t saved = ctx->stream;
  ctx->stream = ctx->own_stream;
  CK(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal));
  cudaError_t e = enqueue_dropin_iteration(ctx, seed);
  cudaGraph_t g = nullptr;
  cudaError_t e2 = cudaStreamEndCapture(ctx->stream, &g);
  ctx->stream = saved;
  CK(e);
  CK(e2);
  cudaGraphExec_t ge = nullptr;
  cudaError_t e3 = cudaGraphInstantiate(&ge, g, 0);
  cudaGraphDestroy(g);
  CK(e3);
  v.emplace_back(seed, ge);
  *out = ge;
  return JM_OK;
}

// The drop-in graph launch: stage the inputs in the pinned block, replay the
// iteration graph, spin on the done word; outputs are left in the pinned block
// (h_small from off_unew on).
int dropin_launch(jm_ctx* ctx, const double* x0, const double* u_nom, const double* u_init, uint64_t seed,
                  uint64_t iteration, uint64_t* weights_stash) {
  // JM_DROPIN_DIRECT=1 (tuning): three stream launches instead of one graph launch
  static const bool direct = std::getenv("JM_DROPIN_DIRECT") != nullptr && std::atoi(std::getenv("JM_DROPIN_DIRECT")) != 0;
  cudaGraphExec_t ge = nullptr;
  int r = direct ? JM_OK : capture_iteration_graph(ctx, seed, &ge);
  if (r != JM_OK) return r;
  uint64_t handle = 0;
  r = stash_acquire(ctx, &handle);
  if (r != JM_OK) return r;
  double* hs = ctx->h_small;
  std::memcpy(hs + ctx->off_x0(), x0, sizeof(double) * ctx->N);
  std::memcpy(hs + ctx->off_unom(), u_nom, sizeof(double) * ctx->TM);
  std::memcpy(hs + ctx->off_uinit(), u_init, sizeof(double) * ctx->M);
  uint64_t* words = reinterpret_cast<uint64_t*>(hs + ctx->off_x0());
  words[13] = reinterpret_cast<uint64_t>(ctx->stash[handle - 1]);
  words[15] = iteration;
  volatile int32_t* st = reinterpret_cast<volatile int32_t*>(hs + ctx->off_status());
  st[0] = 0;
  st[1] = 0;  // done word, raised by the finalize after its last output
  if (direct)
    CK(enqueue_dropin_iteration(ctx, seed));
  else
    CK(cudaGraphLaunch(ge, ctx->stream));
  // (zero-copy over PCIe: copy_block_kernel reads [x0|u_nom|mapping|u_init], the finalize
  // writes [u_new|norms|diag|status|u_shift] into the pinned block)
  g_h2d += (long long)(sizeof(double) * ctx->off_unew());
  g_d2h += (long long)(sizeof(double) * (ctx->off_rec() - ctx->off_unew()));
  // spin on the done word (a stream synchronisation wakes the host several
  // microseconds later); fall back to the synchronisation after 2 s so a
  // faulting launch still reports its error
  const auto t_spin = std::chrono::steady_clock::now();
  while (st[1] == 0) {
    if (std::chrono::steady_clock::now() - t_spin > std::chrono::seconds(2)) {
      CK(cudaStreamSynchronize(ctx->stream));
      if (st[1] == 0) return fail(ctx, JM_ERR_CUDA, "drop-in iteration graph finished without its done word");
      break;
    }
  }
  std::atomic_thread_fence(std::memory_order_acquire);
  if (st[0] == JM_ERR_NO_VIABLE) {
    ctx->stash_free.push_back((int)handle - 1);
    return fail(ctx, JM_ERR_NO_VIABLE, "no viable rollout");
  }
  *weights_stash = handle;
  return JM_OK;
}

int ensure_trace(jm_ctx* ctx) {
  const size_t need = (size_t)ctx->K * (ctx->T + 1) * ctx->N;
  if (ctx->states_cap >= need) return JM_OK;
  dfree(ctx->d_states);
  dfree(ctx->d_div);
  ctx->d_states = nullptr;
  ctx->d_div = nullptr;
  CK(dalloc(&ctx->d_states, need));
  CK(dalloc(&ctx->d_div, (size_t)ctx->K));
  ctx->states_cap = need;
  return JM_OK;
}

// one control step of the closed loop on ctx->stream: rollout, then finalize
// whose last CTA runs the plant step + shift (2 launches)
cudaError_t loop_step_launches(jm_ctx* ctx, cudaEvent_t mid) {
  jm::RolloutCall rc;
  rc.u_nom = ctx->d_loop_unom;
  rc.costs = ctx->d_costs;
  rc.loop = ctx->d_loop;
  rc.seed = ctx->loop_seed;  // the loop's master seed (a kernel parameter)
  // opt-in (JM_SELF_PUSH=1): measured 46.2 vs 43.4 us per cfg1 step -- the 147
  // CTAs finish within ~1 us of each other, so merging behind the flags
  // overlaps little and the per-record flag polls lengthen each warp's chain
  static const bool self_push_env = std::getenv("JM_SELF_PUSH") != nullptr;
  const bool self_push = self_push_env && ctx->d_self_push != nullptr && mid == nullptr;
  if (self_push) {  // records + epoch flags into the world-1 exchange buffer
    rc.push_peers = ctx->d_self_base;
    rc.push_rank = 0;
    rc.push_world = 1;
  }
  cudaError_t e = ctx->eng->rollout(ctx, rc);
  if (e == cudaSuccess && mid) e = cudaEventRecord(mid, ctx->stream);
  if (e != cudaSuccess) return e;
  jm::FinArgs f = self_push ? fin_args(ctx, ctx->d_self_push, ctx->grid) : fin_args(ctx, nullptr, 0);
  if (self_push)
    f.wait_flags = reinterpret_cast<const unsigned int*>(ctx->d_self_push + 2 * (size_t)ctx->grid * ctx->rec_stride);
  f.wait_gpu = self_push ? 1 : 0;
  f.u_nom = ctx->d_loop_unom;
  f.u_new = ctx->d_loop_unew;
  return ctx->eng->finalize(ctx, f, ctx->d_loop, ctx->d_loop_unom);
}

int capture_loop_graph(jm_ctx* ctx) {
  if (ctx->graph_exec) return JM_OK;
  cudaStream_t saved = ctx->stream;
  ctx->stream = ctx->own_stream;
  CK(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal));
  cudaError_t e1 = loop_step_launches(ctx, nullptr);
  cudaGraph_t g = nullptr;
  cudaError_t e4 = cudaStreamEndCapture(ctx->stream, &g);
  ctx->stream = saved;
  CK(e1);
  CK(e4);
  ctx->graph = g;
  CK(cudaGraphInstantiate(&ctx->graph_exec, g, 0));
  return JM_OK;
}

}  // namespace

extern "C" {

int jm_abi_version(void) { return JM_ABI_VERSION; }

const char* jm_last_error(const jm_ctx* ctx) { return ctx ? ctx->err.c_str() : g_err.c_str(); }

int jm_device_count(int* out) {
  jm_ctx* ctx = nullptr;
  CK(cudaGetDeviceCount(out));
  return JM_OK;
}

int jm_create(const jm_model_desc* model, const jm_cost_desc* cost, const jm_mppi_desc* mppi,
              int device, jm_ctx** out) {
  jm_ctx* ctx = nullptr;
  if (!model || !cost || !mppi || !out) return fail(nullptr, JM_ERR_VALUE, "null argument");
  *out = nullptr;
  const jm_mppi_desc& p = *mppi;
  // MppiConfig invariants (types.py:90-113)
  if (!(p.lambda_ > 0)) return fail(nullptr, JM_ERR_CONFIG, "invalid configuration: lambda must be positive");
  if (!(p.c >= 1.0)) return fail(nullptr, JM_ERR_CONFIG, "invalid configuration: c must be at least 1");
  if (!(p.dt > 0)) return fail(nullptr, JM_ERR_CONFIG, "invalid configuration: dt must be positive");
  if (!(p.nu >= 0)) return fail(nullptr, JM_ERR_CONFIG, "invalid configuration: nu must be nonnegative");
  if (p.horizon < 1) return fail(nullptr, JM_ERR_CONFIG, "invalid configuration: horizon_n must be a positive integer");
  if (p.samples < 1) return fail(nullptr, JM_ERR_CONFIG, "invalid configuration: samples_m must be a positive integer");
  if (!(cost->lambda_ > 0)) return fail(nullptr, JM_ERR_CONFIG, "invalid configuration: cost lambda must be positive");
  if (!(cost->c >= 1.0)) return fail(nullptr, JM_ERR_CONFIG, "invalid configuration: cost c must be at least 1");
  const int m = model->control_dim, n = model->state_dim;
  for (int i = 0; i < JM_MAX_STATE; ++i)
    if (!(cost->weights[i] >= 0.0))  // nonnegative state costs (costs.py:37)
      return fail(nullptr, JM_ERR_CONFIG, "invalid configuration: cost weights must be nonnegative");
  if (m != p.control_dim) return fail(nullptr, JM_ERR_CONFIG, "control_dim mismatch between model (%d) and config (%d)", m, p.control_dim);
  if (p.jump_process != JM_JUMPS_BERNOULLI && p.jump_process != JM_JUMPS_POISSON)
    return fail(nullptr, JM_ERR_CONFIG, "invalid configuration: jump_process must be bernoulli or poisson");
  if (p.jump_enabled && !(p.nu * p.dt < 0.1))  // noise.py:148-149
    return fail(nullptr, JM_ERR_VALUE, "zero-one jump law violated (nu*dt = %g)", p.nu * p.dt);

  ctx = new jm_ctx();
  ctx->model = *model;
  ctx->cost = *cost;
  ctx->mppi = p;
  ctx->device = device;
  ctx->N = n;
  ctx->M = m;
  ctx->T = p.horizon;
  ctx->K = p.samples;
  ctx->TM = ctx->T * m;
  ctx->Q = model->jump_channel == JM_JUMP_CONTROL ? m : model->jump_dim;
  ctx->rec_stride = 4 + ctx->TM + (ctx->TM & 1);
  ctx->real_size = p.precision == JM_F64 ? 8 : 4;
  ctx->block = p.block_threads > 0 ? p.block_threads : 128;
  if (ctx->block % 32 != 0 || ctx->block > 256) {
    delete ctx;
    return fail(nullptr, JM_ERR_CONFIG, "block_threads must be a multiple of 32 and <= 256");
  }
  // factors (noise.py:143, :150; harness.py:123-124)
  double cs[16];
  for (int i = 0; i < m * m; ++i) cs[i] = p.c * p.sigma_d[i];
  if (!cholesky(cs, m, ctx->Ld)) {
    delete ctx;
    return fail(nullptr, JM_ERR_NOISE, "covariance factorization failed for c*sigma_d");
  }
  if (!cholesky(p.sigma_d, m, ctx->Lp)) {
    delete ctx;
    return fail(nullptr, JM_ERR_NOISE, "covariance factorization failed for sigma_d");
  }
  if (!cholesky(p.sigma_j, ctx->Q, ctx->Lj)) {
    delete ctx;
    return fail(nullptr, JM_ERR_NOISE, "covariance factorization failed for sigma_j");
  }
  ctx->poisson = p.jump_process == JM_JUMPS_POISSON;
  const double p_event = event_probability(p.nu * p.dt, ctx->poisson);
  ctx->jthr = p.jump_enabled ? jump_threshold(p_event) : 0u;
  ctx->jthr_plant = jump_threshold(p_event);
  if (ctx->poisson) count_tables(p.nu * p.dt, &ctx->cnt, ctx->cnt_plant);

  // plugin -> kernel family
  switch (model->kind) {
    case JM_MODEL_INTEGRATOR:
      if (n != m) break;
      ctx->eng = jm::make_engine_integrator(cost->kind, p.precision, n);
      break;
    case JM_MODEL_CARTPOLE:
      if (n != 4 || m != 1) break;
      ctx->eng = jm::make_engine_cartpole(cost->kind, p.precision);
      break;
    case JM_MODEL_QUADROTOR:
      if (n != 12 || m != 4) break;
      ctx->eng = jm::make_engine_quadrotor(cost->kind, p.precision);
      break;
    case JM_MODEL_LINEAR:
      if (model->jump_channel != JM_JUMP_CONTROL) break;  // B = H = G
      ctx->eng = jm::make_engine_linear(cost->kind, p.precision, n, m);
      break;
    default:
      break;
  }
  if (!ctx->eng) {
    delete ctx;
    return fail(nullptr, JM_ERR_UNSUPPORTED, "no kernel for model kind %d (n=%d, m=%d) with cost kind %d",
                model->kind, n, m, cost->kind);
  }
  if (model->jump_channel == JM_JUMP_STATE) {
    // the state-jump selector rows are compiled into each model
    const int expect_q = model->kind == JM_MODEL_CARTPOLE ? 1 : (model->kind == JM_MODEL_QUADROTOR ? 3 : n);
    bool ok = ctx->Q == expect_q;
    for (int i = 0; ok && i < ctx->Q; ++i) {
      const int row = model->kind == JM_MODEL_CARTPOLE ? 3 : (model->kind == JM_MODEL_QUADROTOR ? 3 + i : i);
      ok = model->jump_rows[i] == row;
    }
    if (!ok) {
      delete ctx->eng;
      delete ctx;
      return fail(nullptr, JM_ERR_UNSUPPORTED,
                  "state-jump selector not supported for this model (cartpole: row 3; quadrotor: rows 3,4,5)");
    }
  }

  cudaError_t e = cudaSetDevice(device);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, device);
  if (e == cudaSuccess && model->kind == JM_MODEL_LINEAR) {  // [A | G] for the Linear engine
    std::vector<double> ag((size_t)n * n + (size_t)n * m);
    for (int i = 0; i < n * n; ++i) ag[i] = model->lin_A[i];
    for (int i = 0; i < n * m; ++i) ag[(size_t)n * n + i] = model->lin_G[i];
    std::vector<float> agf(ag.begin(), ag.end());
    e = cudaMalloc(&ctx->d_lin_d, sizeof(double) * ag.size());
    if (e == cudaSuccess) e = cudaMalloc(&ctx->d_lin_f, sizeof(float) * agf.size());
    if (e == cudaSuccess) e = xferSync(ctx->d_lin_d, ag.data(), sizeof(double) * ag.size(), cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = xferSync(ctx->d_lin_f, agf.data(), sizeof(float) * agf.size(), cudaMemcpyHostToDevice);
  }
  if (e == cudaSuccess && ctx->jthr) {
    const std::vector<uint32_t> S = gap_table(p_event, ctx->T, &ctx->gap_inv);
    ctx->gap_n = (int)S.size();
    e = cudaMalloc(&ctx->d_gap, S.size() * sizeof(uint32_t));
    if (e == cudaSuccess) e = xferSync(ctx->d_gap, S.data(), S.size() * sizeof(uint32_t), cudaMemcpyHostToDevice);
  }
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&ctx->own_stream, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = ctx->eng->configure(ctx);
  ctx->stream = ctx->own_stream;
  if (e == cudaSuccess && p.noise_source == JM_NOISE_PHILOX)
    e = cudaMalloc(&ctx->d_scratch, (size_t)ctx->grid * ctx->TM * ctx->block * ctx->real_size);
  if (e == cudaSuccess) e = dalloc(&ctx->d_costs, (size_t)ctx->K);
  if (e == cudaSuccess) e = dalloc(&ctx->d_weights, (size_t)ctx->K);
  if (e == cudaSuccess) e = dalloc(&ctx->d_wsum, (size_t)(ctx->K + jm::kWThreads - 1) / jm::kWThreads);
  if (e == cudaSuccess) e = dalloc(&ctx->d_records, (size_t)ctx->grid * ctx->rec_stride);
  if (e == cudaSuccess) e = dalloc(&ctx->d_small, ctx->small_doubles());
  if (e == cudaSuccess) e = dalloc(&ctx->d_counter, 1);
  if (e == cudaSuccess) e = cudaMemsetAsync(ctx->d_counter, 0, sizeof(unsigned int), ctx->stream);
  if (e == cudaSuccess) e = cudaMallocHost(&ctx->h_small, ctx->small_doubles() * sizeof(double));
  if (e == cudaSuccess) e = cudaMallocHost(&ctx->h_big, 2 * (size_t)ctx->K * sizeof(double));
  if (e == cudaSuccess) e = cudaMemsetAsync(ctx->d_small, 0, ctx->small_doubles() * sizeof(double), ctx->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
  if (e != cudaSuccess) {
    const std::string msg = cudaGetErrorString(e);
    jm_destroy(ctx);
    return fail(nullptr, JM_ERR_CUDA, "jm_create: %s", msg.c_str());
  }
  *out = ctx;
  return JM_OK;
}

int jm_destroy(jm_ctx* ctx) {
  if (!ctx) return JM_OK;
  cudaSetDevice(ctx->device);
  if (ctx->own_stream) cudaStreamSynchronize(ctx->own_stream);
  if (ctx->graph_exec) cudaGraphExecDestroy(ctx->graph_exec);
  if (ctx->graph) cudaGraphDestroy(ctx->graph);
  for (auto& pe : ctx->iter_execs) cudaGraphExecDestroy(pe.second);
  dfree(ctx->d_scratch);
  dfree(ctx->d_gap);
  dfree(ctx->d_lin_f);
  dfree(ctx->d_lin_d);
  dfree(ctx->d_hbm_eps);
  dfree(ctx->d_hbm_jump);
  dfree(ctx->d_costs);
  dfree(ctx->d_weights);
  dfree(ctx->d_wsum);
  dfree(ctx->d_records);
  dfree(ctx->d_small);
  dfree(ctx->d_counter);
  for (double* b : ctx->stash) dfree(b);
  dfree(ctx->d_states);
  dfree(ctx->d_div);
  dfree(ctx->d_loop);
  dfree(ctx->d_loop_unom);
  dfree(ctx->d_loop_unew);
  dfree(ctx->d_self_push);
  dfree(ctx->d_self_base);
  dfree(ctx->d_hist);
  dfree(ctx->d_hist_jumps);
  dfree(ctx->d_hist_t);
  dfree(ctx->d_tl);
  dfree(ctx->d_flush);
  if (ctx->h_small) cudaFreeHost(ctx->h_small);
  if (ctx->h_big) cudaFreeHost(ctx->h_big);
  if (ctx->own_stream) cudaStreamDestroy(ctx->own_stream);
  delete ctx->eng;
  delete ctx;
  return JM_OK;
}

int jm_set_stream(jm_ctx* ctx, void* stream) {
  if (!ctx) return fail(nullptr, JM_ERR_VALUE, "null context");
  ctx->stream = stream ? reinterpret_cast<cudaStream_t>(stream) : ctx->own_stream;
  return JM_OK;
}

int jm_record_doubles(const jm_ctx* ctx, int64_t* out) {
  if (!ctx || !out) return fail(nullptr, JM_ERR_VALUE, "null argument");
  *out = ctx->rec_stride;
  return JM_OK;
}

int jm_iteration_host(jm_ctx* ctx, const double* x0, const double* u_nom, uint64_t seed,
                      uint64_t iteration, const void* eps_c, const void* jump,
                      const double* mapping, double* u_new, double* costs, double* weights,
                      double* step_norms, double* states, int64_t* diverged_step, jm_diag* diag,
                      const double* u_init, double* u_shift, uint64_t* weights_stash) {
  if (!ctx || !x0 || !u_nom || !u_new) return fail(ctx, JM_ERR_VALUE, "null argument");
  if ((u_init == nullptr) != (u_shift == nullptr)) return fail(ctx, JM_ERR_VALUE, "u_init and u_shift go together");
  CK(cudaSetDevice(ctx->device));
  const bool hbm = ctx->mppi.noise_source == JM_NOISE_HBM;
  if (hbm && !eps_c) return fail(ctx, JM_ERR_VALUE, "HBM noise mode needs eps_combined");
  if (hbm && ctx->model.jump_channel == JM_JUMP_STATE && ctx->jthr && !jump)
    return fail(ctx, JM_ERR_VALUE, "HBM noise mode with state jumps needs the jump tensor");
  const int N = ctx->N, M = ctx->M, TM = ctx->TM, T = ctx->T, K = ctx->K;
  double* hs = ctx->h_small;
  double* ds = ctx->d_small;
  static const bool iter_graph = std::getenv("JM_NO_ITER_GRAPH") == nullptr;
  if (iter_graph && !hbm && !mapping && !costs && !weights && !states && !diverged_step && u_shift && weights_stash) {
    // the drop-in fast path: one graph launch
    const int r = dropin_launch(ctx, x0, u_nom, u_init, seed, iteration, weights_stash);
    if (r != JM_OK) return r;
    const DiagOut* dg = reinterpret_cast<const DiagOut*>(hs + ctx->off_diag());
    std::memcpy(u_new, hs + ctx->off_unew(), sizeof(double) * TM);
    std::memcpy(u_shift, hs + ctx->off_ushift(), sizeof(double) * TM);
    if (step_norms) std::memcpy(step_norms, hs + ctx->off_norms(), sizeof(double) * T);
    if (diag) {
      diag->min_cost = dg->min_cost;
      diag->ess = dg->ess;
      diag->normaliser = dg->normaliser;
      diag->n_finite = dg->n_finite;
    }
    return JM_OK;
  }
  std::memcpy(hs + ctx->off_x0(), x0, sizeof(double) * N);
  std::memcpy(hs + ctx->off_unom(), u_nom, sizeof(double) * TM);
  if (mapping) std::memcpy(hs + ctx->off_map(), mapping, sizeof(double) * M * M);
  if (u_init) std::memcpy(hs + ctx->off_uinit(), u_init, sizeof(double) * M);
  CK(xferAsync(ds, hs, sizeof(double) * ctx->off_unew(), cudaMemcpyHostToDevice, ctx->stream));
  jm::RolloutCall rc;
  rc.x0 = ds + ctx->off_x0();
  rc.u_nom = ds + ctx->off_unom();
  rc.seed = seed;
  rc.iteration = iteration;
  rc.costs = ctx->d_costs;
  if (hbm) {
    const size_t eb = (size_t)TM * K * ctx->real_size;
    if (!ctx->d_hbm_eps) CK(cudaMalloc(&ctx->d_hbm_eps, eb));
    CK(xferAsync(ctx->d_hbm_eps, eps_c, eb, cudaMemcpyHostToDevice, ctx->stream));
    rc.eps_in = ctx->d_hbm_eps;
    if (jump && ctx->model.jump_channel == JM_JUMP_STATE) {
      const size_t jb = (size_t)T * ctx->Q * K * ctx->real_size;
      if (!ctx->d_hbm_jump) CK(cudaMalloc(&ctx->d_hbm_jump, jb));
      CK(xferAsync(ctx->d_hbm_jump, jump, jb, cudaMemcpyHostToDevice, ctx->stream));
      rc.jump_in = ctx->d_hbm_jump;
    }
  }
  const bool trace = states != nullptr || diverged_step != nullptr;
  if (trace) {
    const int r = ensure_trace(ctx);
    if (r != JM_OK) return r;
    rc.states = ctx->d_states;
    rc.diverged = ctx->d_div;
  }
  double* wdev = weights ? ctx->d_weights : nullptr;
  uint64_t handle = 0;
  if (weights_stash && !costs && !weights) {  // keep this iteration's costs; weights are formed on fetch
    const int rs = stash_acquire(ctx, &handle);
    if (rs != JM_OK) return rs;
    rc.costs = ctx->stash[handle - 1];
  }
  const int r = rollout_and_finalize(ctx, rc, mapping ? ds + ctx->off_map() : nullptr, wdev, u_shift != nullptr);
  if (r != JM_OK) return r;
  if (weights_stash && !handle) {
    const int rs = stash_acquire(ctx, &handle);
    if (rs != JM_OK) return rs;
    CK(xferAsync(ctx->stash[handle - 1], ctx->d_costs, sizeof(double) * K, cudaMemcpyDeviceToDevice,
                       ctx->stream));
  }
  const size_t out_n = ctx->off_rec() - ctx->off_unew();
  CK(xferAsync(hs + ctx->off_unew(), ds + ctx->off_unew(), sizeof(double) * out_n,
                     cudaMemcpyDeviceToHost, ctx->stream));
  if (costs) CK(xferAsync(ctx->h_big, ctx->d_costs, sizeof(double) * K, cudaMemcpyDeviceToHost, ctx->stream));
  if (weights)
    CK(xferAsync(ctx->h_big + K, wdev, sizeof(double) * K, cudaMemcpyDeviceToHost, ctx->stream));
  if (states)
    CK(xferAsync(states, ctx->d_states, sizeof(double) * (size_t)K * (T + 1) * N,
                       cudaMemcpyDeviceToHost, ctx->stream));
  if (diverged_step)
    CK(xferAsync(diverged_step, ctx->d_div, sizeof(int64_t) * K, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  const int32_t status = *reinterpret_cast<int32_t*>(hs + ctx->off_status());
  const DiagOut* dg = reinterpret_cast<const DiagOut*>(hs + ctx->off_diag());
  if (costs) std::memcpy(costs, ctx->h_big, sizeof(double) * K);
  if (status == JM_ERR_NO_VIABLE) {
    if (handle) ctx->stash_free.push_back((int)handle - 1);
    return fail(ctx, JM_ERR_NO_VIABLE, "no viable rollout");
  }
  if (weights_stash) *weights_stash = handle;
  if (u_shift) std::memcpy(u_shift, hs + ctx->off_ushift(), sizeof(double) * TM);
  std::memcpy(u_new, hs + ctx->off_unew(), sizeof(double) * TM);
  if (step_norms) std::memcpy(step_norms, hs + ctx->off_norms(), sizeof(double) * T);
  if (weights) std::memcpy(weights, ctx->h_big + K, sizeof(double) * K);
  if (diag) {
    diag->min_cost = dg->min_cost;
    diag->ess = dg->ess;
    diag->normaliser = dg->normaliser;
    diag->n_finite = dg->n_finite;
  }
  return JM_OK;
}

int jm_upload_inputs(jm_ctx* ctx, const double* x0, const double* u_nom) {
  if (!ctx || !x0 || !u_nom) return fail(ctx, JM_ERR_VALUE, "null argument");
  CK(cudaSetDevice(ctx->device));
  std::memcpy(ctx->h_small + ctx->off_x0(), x0, sizeof(double) * ctx->N);
  std::memcpy(ctx->h_small + ctx->off_unom(), u_nom, sizeof(double) * ctx->TM);
  CK(xferAsync(ctx->d_small, ctx->h_small, sizeof(double) * ctx->off_map(), cudaMemcpyHostToDevice,
                     ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  return JM_OK;
}

int jm_iteration_dropin(jm_ctx* ctx, const double* x0, const double* u_nom, const double* u_init,
                        uint64_t seed, uint64_t iteration, double* out, uint64_t* weights_stash) {
  if (!ctx || !x0 || !u_nom || !u_init || !out || !weights_stash) return fail(ctx, JM_ERR_VALUE, "null argument");
  if (ctx->mppi.noise_source == JM_NOISE_HBM) return fail(ctx, JM_ERR_VALUE, "HBM noise mode needs jm_iteration_host");
  CK(cudaSetDevice(ctx->device));
  const int r = dropin_launch(ctx, x0, u_nom, u_init, seed, iteration, weights_stash);
  if (r != JM_OK) return r;
  std::memcpy(out, ctx->h_small + ctx->off_unew(), sizeof(double) * (size_t)jm_dropin_doubles(ctx));
  return JM_OK;
}

int jm_transfer_bytes(int64_t* h2d, int64_t* d2h) {
  if (h2d) *h2d = (int64_t)g_h2d.load();
  if (d2h) *d2h = (int64_t)g_d2h.load();
  return JM_OK;
}

int64_t jm_dropin_doubles(const jm_ctx* ctx) { return ctx ? (int64_t)(ctx->off_rec() - ctx->off_unew()) : 0; }

int jm_stash_fetch(jm_ctx* ctx, uint64_t handle, double min_cost, double normaliser, double* host) {
  if (!ctx || !host || handle == 0 || handle > ctx->stash.size()) return fail(ctx, JM_ERR_VALUE, "bad stash handle");
  CK(cudaSetDevice(ctx->device));
  // weights of the stashed costs (controller.py:62-71) with that iteration's rho and Z
  DiagOut* dd = reinterpret_cast<DiagOut*>(ctx->d_small + ctx->off_rec());  // scratch slot
  DiagOut hd{min_cost, 0.0, normaliser, 0};
  CK(xferAsync(dd, &hd, sizeof(hd), cudaMemcpyHostToDevice, ctx->stream));
  CK(launch_weights(ctx, ctx->stash[handle - 1], dd, ctx->d_weights));
  CK(xferAsync(host, ctx->d_weights, sizeof(double) * ctx->K, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  return JM_OK;
}

int jm_stash_release(jm_ctx* ctx, uint64_t handle) {
  if (!ctx || handle == 0 || handle > ctx->stash.size()) return fail(ctx, JM_ERR_VALUE, "bad stash handle");
  ctx->stash_free.push_back((int)handle - 1);
  return JM_OK;
}

int jm_rollout_dev(jm_ctx* ctx, const double* x0_dev, const double* u_nom_dev, uint64_t seed,
                   uint64_t iteration, const uint64_t* iteration_dev, const void* eps_c_dev,
                   const void* jump_dev, double* costs_dev, double* states_dev, int64_t* diverged_dev) {
  if (!ctx || !x0_dev || !u_nom_dev) return fail(ctx, JM_ERR_VALUE, "null argument");
  if (ctx->mppi.noise_source == JM_NOISE_HBM && !eps_c_dev)
    return fail(ctx, JM_ERR_VALUE, "HBM noise mode needs eps_combined");
  CK(cudaSetDevice(ctx->device));
  jm::RolloutCall rc;
  rc.x0 = x0_dev;
  rc.u_nom = u_nom_dev;
  rc.seed = seed;
  rc.iteration = iteration;
  rc.iteration_dev = iteration_dev;
  rc.eps_in = eps_c_dev;
  rc.jump_in = ctx->model.jump_channel == JM_JUMP_STATE ? jump_dev : nullptr;
  rc.costs = costs_dev ? costs_dev : ctx->d_costs;
  rc.states = states_dev;
  rc.diverged = diverged_dev;
  if ((states_dev == nullptr) != (diverged_dev == nullptr))
    return fail(ctx, JM_ERR_VALUE, "states and diverged buffers go together");
  CK(ctx->eng->rollout(ctx, rc));
  return JM_OK;
}

int jm_reduce_dev(jm_ctx* ctx, double* record_dev) {
  if (!ctx || !record_dev) return fail(ctx, JM_ERR_VALUE, "null argument");
  CK(cudaSetDevice(ctx->device));
  jm::FinArgs f = fin_args(ctx, nullptr, 0);
  f.rec_out = record_dev;
  CK(ctx->eng->finalize(ctx, f, nullptr, nullptr));
  return JM_OK;
}

int jm_finalize_dev(jm_ctx* ctx, const double* records_dev, int32_t nrec, const double* u_nom_dev,
                    const double* mapping_dev, double* u_new_dev, double* step_norms_dev,
                    jm_diag* diag_dev, int32_t* status_dev) {
  if (!ctx || !u_nom_dev || !u_new_dev) return fail(ctx, JM_ERR_VALUE, "null argument");
  if (records_dev && (nrec < 1 || nrec > jm::kMaxRecords)) return fail(ctx, JM_ERR_VALUE, "bad record count");
  CK(cudaSetDevice(ctx->device));
  jm::FinArgs f = fin_args(ctx, records_dev, nrec);
  f.u_nom = u_nom_dev;
  f.mapping = mapping_dev;
  f.u_new = u_new_dev;
  f.norms = step_norms_dev;
  f.diag = reinterpret_cast<DiagOut*>(diag_dev);
  f.status = status_dev;
  CK(ctx->eng->finalize(ctx, f, nullptr, nullptr));
  return JM_OK;
}

int jm_weights_dev(jm_ctx* ctx, const double* costs_dev, const jm_diag* diag_dev, double* weights_dev) {
  if (!ctx || !costs_dev || !diag_dev || !weights_dev) return fail(ctx, JM_ERR_VALUE, "null argument");
  CK(cudaSetDevice(ctx->device));
  CK(launch_weights(ctx, costs_dev, reinterpret_cast<const DiagOut*>(diag_dev), weights_dev));
  return JM_OK;
}

int jm_shift_dev(jm_ctx* ctx, const double* u_dev, const double* u_init_dev, double* out_dev) {
  if (!ctx || !u_dev || !u_init_dev || !out_dev) return fail(ctx, JM_ERR_VALUE, "null argument");
  CK(cudaSetDevice(ctx->device));
  const int b = 128, g = (ctx->TM + b - 1) / b;
  jm::shift_kernel<<<g, b, 0, ctx->stream>>>(u_dev, u_init_dev, ctx->T, ctx->M, out_dev);
  CK(cudaGetLastError());
  return JM_OK;
}

int jm_shift_host(int device, int32_t T, int32_t m, const double* u, const double* u_init, double* out) {
  jm_ctx* ctx = nullptr;
  if (T < 1 || m < 1 || !u || !u_init || !out) return fail(nullptr, JM_ERR_VALUE, "bad arguments");
  CK(cudaSetDevice(device));
  // per-thread device scratch, grown on demand (no allocation per call)
  thread_local int s_dev = -1;
  thread_local size_t s_cap = 0;
  thread_local double* s_buf = nullptr;
  const int TM = T * m;
  const size_t need = 2 * (size_t)TM + (size_t)m;
  if (s_dev != device || s_cap < need) {
    if (s_buf && s_dev == device) dfree(s_buf);
    s_buf = nullptr;
    CK(dalloc(&s_buf, need));
    s_dev = device;
    s_cap = need;
  }
  double *d_u = s_buf, *d_o = s_buf + TM, *d_i = s_buf + 2 * TM;
  CK(xferSync(d_u, u, sizeof(double) * TM, cudaMemcpyHostToDevice));
  CK(xferSync(d_i, u_init, sizeof(double) * m, cudaMemcpyHostToDevice));
  jm::shift_kernel<<<(TM + 127) / 128, 128>>>(d_u, d_i, T, m, d_o);
  CK(cudaGetLastError());
  CK(xferSync(out, d_o, sizeof(double) * TM, cudaMemcpyDeviceToHost));
  return JM_OK;
}

int jm_compute_weights_host(int device, int64_t K, const double* costs, double lambda_, double* weights) {
  jm_ctx* ctx = nullptr;
  if (K < 1 || !costs || !weights) return fail(nullptr, JM_ERR_VALUE, "bad arguments");
  CK(cudaSetDevice(device));
  double *d_c = nullptr, *d_w = nullptr, *d_o = nullptr;
  CK(dalloc(&d_c, (size_t)K));
  CK(dalloc(&d_w, (size_t)K));
  CK(dalloc(&d_o, 2));
  CK(xferSync(d_c, costs, sizeof(double) * K, cudaMemcpyHostToDevice));
  cw_kernel<<<1, 1024>>>(d_c, K, 1.0 / lambda_, d_w, d_o);
  CK(cudaGetLastError());
  double o[2];
  CK(xferSync(weights, d_w, sizeof(double) * K, cudaMemcpyDeviceToHost));
  CK(xferSync(o, d_o, sizeof(o), cudaMemcpyDeviceToHost));
  dfree(d_c);
  dfree(d_w);
  dfree(d_o);
  if (o[0] == INFINITY) return fail(nullptr, JM_ERR_NO_VIABLE, "no viable rollout");
  return JM_OK;
}

int jm_update_controls_host(int device, int64_t K, int32_t T, int32_t m, const double* costs,
                            const double* eps_c, double lambda_, double dt, const double* u_nom,
                            const double* mapping, double* u_new, double* weights) {
  jm_ctx* ctx = nullptr;
  if (K < 1 || T < 1 || m < 1 || m > 4 || !costs || !eps_c || !u_nom || !u_new)
    return fail(nullptr, JM_ERR_VALUE, "bad arguments");
  CK(cudaSetDevice(device));
  const int TM = T * m;
  double *d_c, *d_w, *d_o, *d_e, *d_u, *d_n, *d_m = nullptr;
  CK(dalloc(&d_c, (size_t)K));
  CK(dalloc(&d_w, (size_t)K));
  CK(dalloc(&d_o, 2));
  CK(dalloc(&d_e, (size_t)K * TM));
  CK(dalloc(&d_u, (size_t)TM));
  CK(dalloc(&d_n, (size_t)TM));
  CK(xferSync(d_c, costs, sizeof(double) * K, cudaMemcpyHostToDevice));
  CK(xferSync(d_e, eps_c, sizeof(double) * K * TM, cudaMemcpyHostToDevice));
  CK(xferSync(d_u, u_nom, sizeof(double) * TM, cudaMemcpyHostToDevice));
  if (mapping) {
    CK(dalloc(&d_m, (size_t)m * m));
    CK(xferSync(d_m, mapping, sizeof(double) * m * m, cudaMemcpyHostToDevice));
  }
  cw_kernel<<<1, 1024>>>(d_c, K, 1.0 / lambda_, d_w, d_o);
  CK(cudaGetLastError());
  wavg_kernel<<<(T + 127) / 128, 128>>>(d_w, d_e, K, TM, m, 1.0 / std::sqrt(dt), d_u, d_m, d_n);
  CK(cudaGetLastError());
  double o[2];
  CK(xferSync(o, d_o, sizeof(o), cudaMemcpyDeviceToHost));
  CK(xferSync(u_new, d_n, sizeof(double) * TM, cudaMemcpyDeviceToHost));
  if (weights) CK(xferSync(weights, d_w, sizeof(double) * K, cudaMemcpyDeviceToHost));
  for (double* p : {d_c, d_w, d_o, d_e, d_u, d_n, d_m}) dfree(p);
  if (o[0] == INFINITY) return fail(nullptr, JM_ERR_NO_VIABLE, "no viable rollout");
  return JM_OK;
}

static jm::NoiseArgs noise_args(const jm_ctx* ctx, uint64_t seed, uint64_t iteration) {
  jm::NoiseArgs na{};
  na.K = ctx->K;
  na.T = ctx->T;
  na.q = ctx->Q;
  na.jump_on = ctx->jthr != 0;
  na.gap_thr = ctx->d_gap;
  na.gap_inv = ctx->gap_inv;
  na.poisson = ctx->poisson;
  na.cnt = ctx->cnt;
  na.sample_offset = ctx->mppi.sample_offset;
  na.seed = seed;
  na.iteration = iteration;
  for (int i = 0; i < 16; ++i) {
    na.Ld[i] = ctx->Ld[i];
    na.Lj[i] = ctx->Lj[i];
  }
  for (int i = 0; i < 4; ++i) na.mu_j[i] = ctx->mppi.mark_mean[i];
  return na;
}

int jm_sample_noise_host(jm_ctx* ctx, uint64_t seed, uint64_t iteration, double* eps_d,
                         int64_t* indicators, double* eps_j, double* eps_c) {
  if (!ctx) return fail(nullptr, JM_ERR_VALUE, "null context");
  CK(cudaSetDevice(ctx->device));
  const size_t KT = (size_t)ctx->K * ctx->T;
  double *d_ed = nullptr, *d_ej = nullptr, *d_ec = nullptr;
  int64_t* d_ind = nullptr;
  if (eps_d) CK(dalloc(&d_ed, KT * ctx->M));
  if (eps_j) CK(dalloc(&d_ej, KT * ctx->Q));
  if (eps_c) CK(dalloc(&d_ec, KT * ctx->M));
  if (indicators) CK(dalloc(&d_ind, KT));
  jm::NoiseArgs na = noise_args(ctx, seed, iteration);
  na.eps_d = d_ed;
  na.eps_j = d_ej;
  na.eps_c = d_ec;
  na.ind = d_ind;
  CK(ctx->eng->noise(ctx, na));
  if (eps_d) CK(xferAsync(eps_d, d_ed, sizeof(double) * KT * ctx->M, cudaMemcpyDeviceToHost, ctx->stream));
  if (eps_j) CK(xferAsync(eps_j, d_ej, sizeof(double) * KT * ctx->Q, cudaMemcpyDeviceToHost, ctx->stream));
  if (eps_c) CK(xferAsync(eps_c, d_ec, sizeof(double) * KT * ctx->M, cudaMemcpyDeviceToHost, ctx->stream));
  if (indicators) CK(xferAsync(indicators, d_ind, sizeof(int64_t) * KT, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  for (void* p : {(void*)d_ed, (void*)d_ej, (void*)d_ec, (void*)d_ind}) dfree(p);
  return JM_OK;
}

int jm_sample_noise_dev(jm_ctx* ctx, uint64_t seed, uint64_t iteration, void* eps_c_dev, void* jump_dev) {
  if (!ctx || !eps_c_dev) return fail(ctx, JM_ERR_VALUE, "null argument");
  CK(cudaSetDevice(ctx->device));
  jm::NoiseArgs na = noise_args(ctx, seed, iteration);
  na.eps_c_sm = eps_c_dev;
  na.jump_sm = ctx->model.jump_channel == JM_JUMP_STATE ? jump_dev : nullptr;
  CK(ctx->eng->noise(ctx, na));
  return JM_OK;
}

int jm_loop_init(jm_ctx* ctx, const double* x0, const double* u_init, uint64_t seed,
                 uint64_t first_iteration, int32_t max_steps) {
  if (!ctx || !x0 || !u_init || max_steps < 1) return fail(ctx, JM_ERR_VALUE, "bad arguments");
  if (ctx->mppi.noise_source != JM_NOISE_PHILOX)
    return fail(ctx, JM_ERR_UNSUPPORTED, "the device closed loop samples its own (Philox) noise");
  CK(cudaSetDevice(ctx->device));
  const int N = ctx->N, M = ctx->M, TM = ctx->TM;
  if (max_steps > ctx->loop_cap || (ctx->graph_exec && seed != ctx->loop_seed)) {  // (re)capture
    if (ctx->graph_exec) cudaGraphExecDestroy(ctx->graph_exec);
    if (ctx->graph) cudaGraphDestroy(ctx->graph);
    ctx->graph_exec = nullptr;
    ctx->graph = nullptr;
  }
  ctx->loop_seed = seed;
  if (max_steps > ctx->loop_cap) {
    dfree(ctx->d_hist);
    dfree(ctx->d_hist_jumps);
    dfree(ctx->d_hist_t);
    dfree(ctx->d_tl);
    ctx->d_tl = nullptr;
    if (!ctx->d_loop) {
      CK(dalloc(reinterpret_cast<char**>(&ctx->d_loop), sizeof(LoopState)));
      CK(dalloc(&ctx->d_loop_unom, 2 * (size_t)TM));  // two parities (LoopState::unom)
      CK(dalloc(&ctx->d_loop_unew, (size_t)TM));
      if (ctx->grid <= jm::kMaxRecords) {
        CK(dalloc(&ctx->d_self_push, (size_t)jm_peer_buffer_doubles(ctx, 1)));
        CK(dalloc(&ctx->d_self_base, 1));
        const unsigned long long base = reinterpret_cast<unsigned long long>(ctx->d_self_push);
        CK(xferSync(ctx->d_self_base, &base, sizeof(base), cudaMemcpyHostToDevice));
      }
    }
    CK(dalloc(&ctx->d_hist, (size_t)(max_steps + 1) * N + (size_t)max_steps * M));
    CK(dalloc(&ctx->d_hist_jumps, (size_t)max_steps));
    CK(dalloc(&ctx->d_hist_t, 2 * (size_t)max_steps));
    ctx->loop_cap = max_steps;
  }
  LoopState h{};
  for (int i = 0; i < N; ++i) h.x[i] = x0[i];
  for (int j = 0; j < M; ++j) h.u_init[j] = u_init[j];
  h.seed = seed;
  h.iteration = first_iteration;
  h.step = 0;
  h.max_steps = max_steps;
  h.halted = 0;
  h.status = 0;
  h.diverged_at = -1;
  h.sampler_jumps = 1;
  h.hist_states = ctx->d_hist;
  h.hist_controls = ctx->d_hist + (size_t)(ctx->loop_cap + 1) * N;
  h.hist_jumps = ctx->d_hist_jumps;
  h.t_start = ctx->d_hist_t;
  h.t_end = ctx->d_hist_t + ctx->loop_cap;
  static const bool timeline = std::getenv("JM_TIMELINE") != nullptr;
  if (timeline && !ctx->d_tl) CK(dalloc(&ctx->d_tl, (size_t)ctx->loop_cap * jm::kTlSlots));
  if (ctx->d_tl) CK(cudaMemsetAsync(ctx->d_tl, 0, sizeof(uint64_t) * (size_t)ctx->loop_cap * jm::kTlSlots, ctx->own_stream));
  h.tl = ctx->d_tl;
  h.unom = ctx->d_loop_unom;
  std::vector<double> unom((size_t)TM);
  for (int t = 0; t < ctx->T; ++t)
    for (int j = 0; j < M; ++j) unom[(size_t)t * M + j] = u_init[j];  // initial_controller_state (controller.py:56-59)
  cudaStream_t s = ctx->own_stream;
  // the last-CTA ticket of a previous run may have been left mid-count (a finalize CTA
  // that timed out on a dead peer returns without taking its ticket)
  CK(cudaMemsetAsync(ctx->d_counter, 0, sizeof(unsigned int), s));
  if (ctx->d_self_push)  // epochs restart at 1: clear the flags of the previous run
    CK(cudaMemsetAsync(ctx->d_self_push, 0, sizeof(double) * (size_t)jm_peer_buffer_doubles(ctx, 1), s));
  CK(xferAsync(ctx->d_loop, &h, sizeof(h), cudaMemcpyHostToDevice, s));
  CK(xferAsync(ctx->d_loop_unom, unom.data(), sizeof(double) * TM, cudaMemcpyHostToDevice, s));
  CK(xferAsync(ctx->d_hist, x0, sizeof(double) * N, cudaMemcpyHostToDevice, s));
  CK(cudaStreamSynchronize(s));
  return capture_loop_graph(ctx);
}

int jm_loop_rollout(jm_ctx* ctx, double* record_dev) {
  if (!ctx || !ctx->d_loop || !record_dev) return fail(ctx, JM_ERR_VALUE, "loop not initialised");
  CK(cudaSetDevice(ctx->device));
  jm::RolloutCall rc;
  rc.u_nom = ctx->d_loop_unom;
  rc.costs = ctx->d_costs;
  rc.loop = ctx->d_loop;
  rc.seed = ctx->loop_seed;  // the loop's master seed (a kernel parameter)
  CK(ctx->eng->rollout(ctx, rc));
  jm::FinArgs f = fin_args(ctx, nullptr, 0);
  f.rec_out = record_dev;
  CK(ctx->eng->finalize(ctx, f, nullptr, nullptr));
  return JM_OK;
}

int jm_loop_finish(jm_ctx* ctx, const double* records_dev, int32_t nrec) {
  if (!ctx || !ctx->d_loop || !records_dev || nrec < 1 || nrec > jm::kMaxRecords)
    return fail(ctx, JM_ERR_VALUE, "bad arguments");
  CK(cudaSetDevice(ctx->device));
  jm::FinArgs f = fin_args(ctx, records_dev, nrec);
  f.u_nom = ctx->d_loop_unom;
  f.u_new = ctx->d_loop_unew;
  CK(ctx->eng->finalize(ctx, f, ctx->d_loop, ctx->d_loop_unom));
  return JM_OK;
}

int64_t jm_peer_buffer_doubles(const jm_ctx* ctx, int32_t world) {
  if (!ctx || world < 1) return 0;
  const int64_t n = (int64_t)world * ctx->grid;                      // one record per rank x CTA
  return 2 * n * ctx->rec_stride + (n + 1) / 2;                      // 2 parities + uint32 flags
}

int jm_loop_rollout_push(jm_ctx* ctx, const unsigned long long* peer_bases_dev, int32_t rank, int32_t world) {
  if (!ctx || !ctx->d_loop || !peer_bases_dev || world < 1 || rank < 0 || rank >= world ||
      (int64_t)world * ctx->grid > jm::kMaxRecords)
    return fail(ctx, JM_ERR_VALUE, "bad arguments (world x grid must be <= %d records)", jm::kMaxRecords);
  CK(cudaSetDevice(ctx->device));
  jm::RolloutCall rc;
  rc.u_nom = ctx->d_loop_unom;
  rc.loop = ctx->d_loop;
  rc.seed = ctx->loop_seed;  // the loop's master seed (a kernel parameter)
  rc.push_peers = peer_bases_dev;
  rc.push_rank = rank;
  rc.push_world = world;
  CK(ctx->eng->rollout(ctx, rc));
  return JM_OK;
}

int jm_loop_finish_peers(jm_ctx* ctx, const double* my_buffer_dev, int32_t world) {
  if (!ctx || !ctx->d_loop || !my_buffer_dev || world < 1 || (int64_t)world * ctx->grid > jm::kMaxRecords)
    return fail(ctx, JM_ERR_VALUE, "bad arguments");
  CK(cudaSetDevice(ctx->device));
  const int nrec = world * ctx->grid;
  jm::FinArgs f = fin_args(ctx, my_buffer_dev, nrec);
  f.u_nom = ctx->d_loop_unom;
  f.u_new = ctx->d_loop_unew;
  f.wait_flags = reinterpret_cast<const unsigned int*>(my_buffer_dev + 2 * (size_t)nrec * ctx->rec_stride);
  CK(ctx->eng->finalize(ctx, f, ctx->d_loop, ctx->d_loop_unom));
  return JM_OK;
}

int jm_loop_rollout_reduce_push(jm_ctx* ctx, const unsigned long long* peer_bases_dev, int32_t rank, int32_t world) {
  const int ncb = ctx ? (ctx->TM + jm::fin_cols(ctx->M) - 1) / jm::fin_cols(ctx->M) : 0;
  if (!ctx || !ctx->d_loop || !peer_bases_dev || world < 1 || rank < 0 || rank >= world || ncb > ctx->grid)
    return fail(ctx, JM_ERR_VALUE, "bad arguments");
  CK(cudaSetDevice(ctx->device));
  jm::RolloutCall rc;
  rc.u_nom = ctx->d_loop_unom;
  rc.costs = ctx->d_costs;
  rc.loop = ctx->d_loop;
  rc.seed = ctx->loop_seed;  // the loop's master seed (a kernel parameter)
  CK(ctx->eng->rollout(ctx, rc));
  jm::FinArgs f = fin_args(ctx, nullptr, 0);  // reduce this rank's CTA records ...
  f.push_peers = peer_bases_dev;              // ... into slot `rank` of every peer buffer
  f.push_rank = rank;
  f.push_world = world;
  f.push_loop = ctx->d_loop;
  CK(ctx->eng->finalize(ctx, f, nullptr, nullptr));
  return JM_OK;
}

int jm_loop_finish_reduced_peers(jm_ctx* ctx, const double* my_buffer_dev, int32_t world) {
  if (!ctx || !ctx->d_loop || !my_buffer_dev || world < 1 || world > jm::kMaxRecords)
    return fail(ctx, JM_ERR_VALUE, "bad arguments");
  CK(cudaSetDevice(ctx->device));
  const int ncb = (ctx->TM + jm::fin_cols(ctx->M) - 1) / jm::fin_cols(ctx->M);
  jm::FinArgs f = fin_args(ctx, my_buffer_dev, world);
  f.u_nom = ctx->d_loop_unom;
  f.u_new = ctx->d_loop_unew;
  f.wait_flags = reinterpret_cast<const unsigned int*>(my_buffer_dev + 2 * (size_t)world * ctx->rec_stride);
  f.wait_nflags = world * ncb;
  CK(ctx->eng->finalize(ctx, f, ctx->d_loop, ctx->d_loop_unom));
  return JM_OK;
}

int jm_loop_step(jm_ctx* ctx) {
  if (!ctx || !ctx->graph_exec) return fail(ctx, JM_ERR_VALUE, "loop not initialised");
  CK(cudaGraphLaunch(ctx->graph_exec, ctx->own_stream));
  return JM_OK;
}

int jm_loop_read(jm_ctx* ctx, double* x_out, uint64_t* iteration_out, int32_t* step_out,
                 int32_t* halted_out, int32_t* status_out) {
  if (!ctx || !ctx->d_loop) return fail(ctx, JM_ERR_VALUE, "loop not initialised");
  CK(cudaSetDevice(ctx->device));
  LoopState h{};
  CK(xferAsync(&h, ctx->d_loop, sizeof(h), cudaMemcpyDeviceToHost, ctx->own_stream));
  CK(cudaStreamSynchronize(ctx->own_stream));
  if (x_out) std::memcpy(x_out, h.x, sizeof(double) * ctx->N);
  if (iteration_out) *iteration_out = h.iteration;
  if (step_out) *step_out = h.step;
  if (halted_out) *halted_out = h.halted;
  if (status_out) *status_out = h.status;
  return JM_OK;
}

int jm_loop_timeline(jm_ctx* ctx, int32_t steps, uint64_t* out) {
  if (!ctx || !out || steps < 1 || steps > ctx->loop_cap) return fail(ctx, JM_ERR_VALUE, "bad arguments");
  if (!ctx->d_tl) return fail(ctx, JM_ERR_UNSUPPORTED, "loop timeline off (set JM_TIMELINE=1 before jm_loop_init)");
  CK(cudaStreamSynchronize(ctx->stream));
  CK(xferSync(out, ctx->d_tl, sizeof(uint64_t) * (size_t)steps * jm::kTlSlots, cudaMemcpyDeviceToHost));
  return JM_OK;
}

int jm_loop_history(jm_ctx* ctx, int32_t steps, double* states, double* controls, int64_t* jumps) {
  if (!ctx || !ctx->d_loop || steps < 0 || steps > ctx->loop_cap) return fail(ctx, JM_ERR_VALUE, "bad arguments");
  CK(cudaSetDevice(ctx->device));
  CK(cudaStreamSynchronize(ctx->stream));
  CK(cudaStreamSynchronize(ctx->own_stream));
  const int N = ctx->N, M = ctx->M;
  if (states) CK(xferSync(states, ctx->d_hist, sizeof(double) * (size_t)(steps + 1) * N, cudaMemcpyDeviceToHost));
  if (controls)
    CK(xferSync(controls, ctx->d_hist + (size_t)(ctx->loop_cap + 1) * N, sizeof(double) * (size_t)steps * M,
                  cudaMemcpyDeviceToHost));
  if (jumps) CK(xferSync(jumps, ctx->d_hist_jumps, sizeof(int64_t) * (size_t)steps, cudaMemcpyDeviceToHost));
  return JM_OK;
}

int jm_closed_loop_host(jm_ctx* ctx, const double* x0, const double* u_init, uint64_t seed,
                        int32_t steps, double* states, double* controls, int64_t* jumps,
                        double* step_ns, int32_t* diverged_at, int32_t* status) {
  int r = jm_loop_init(ctx, x0, u_init, seed, 0, steps);
  if (r != JM_OK) return r;
  for (int s = 0; s < steps; ++s) {
    r = jm_loop_step(ctx);
    if (r != JM_OK) return r;
  }
  LoopState h{};
  CK(xferAsync(&h, ctx->d_loop, sizeof(h), cudaMemcpyDeviceToHost, ctx->own_stream));
  const int N = ctx->N, M = ctx->M;
  std::vector<double> hs((size_t)(steps + 1) * N), hc((size_t)steps * M);
  std::vector<int64_t> hj((size_t)steps);
  std::vector<uint64_t> ht(2 * (size_t)ctx->loop_cap);
  CK(xferAsync(hs.data(), ctx->d_hist, sizeof(double) * hs.size(), cudaMemcpyDeviceToHost, ctx->own_stream));
  CK(xferAsync(hc.data(), ctx->d_hist + (size_t)(ctx->loop_cap + 1) * N, sizeof(double) * hc.size(),
                     cudaMemcpyDeviceToHost, ctx->own_stream));
  CK(xferAsync(hj.data(), ctx->d_hist_jumps, sizeof(int64_t) * hj.size(), cudaMemcpyDeviceToHost, ctx->own_stream));
  CK(xferAsync(ht.data(), ctx->d_hist_t, sizeof(uint64_t) * ht.size(), cudaMemcpyDeviceToHost, ctx->own_stream));
  CK(cudaStreamSynchronize(ctx->own_stream));
  // steps actually executed (h.step), then the reference's post-divergence fill
  // (harness.py:144-148): states[k+1:] = states[k], controls[k+1:] = 0.
  const int done = h.step;
  const int last = (h.diverged_at >= 0) ? h.diverged_at : done;  // last valid state row
  for (int k = 0; k <= steps; ++k) {
    const int src = std::min(k, last);
    if (states)
      for (int i = 0; i < N; ++i) states[(size_t)k * N + i] = hs[(size_t)src * N + i];
  }
  for (int k = 0; k < steps; ++k) {
    const bool valid = (h.diverged_at >= 0) ? k <= h.diverged_at : k < done;
    if (controls)
      for (int j = 0; j < M; ++j) controls[(size_t)k * M + j] = valid ? hc[(size_t)k * M + j] : 0.0;
    if (jumps) jumps[k] = valid ? hj[k] : 0;
    if (step_ns) step_ns[k] = valid ? double(ht[ctx->loop_cap + k] - ht[k]) : 0.0;
  }
  if (diverged_at) *diverged_at = h.diverged_at;
  if (status) *status = h.status;
  if (h.status == JM_ERR_NO_VIABLE) return fail(ctx, JM_ERR_NO_VIABLE, "no viable rollout");
  return JM_OK;
}

int jm_batch_loop_host(jm_ctx* ctx, int32_t trials, const double* x0, const double* u_init,
                       const uint64_t* seeds, const int32_t* sampler_jumps, int32_t steps, double* states,
                       double* controls, int64_t* jumps, double* step_ns, int32_t* diverged_at, int32_t* status) {
  if (!ctx || !x0 || !u_init || !seeds || trials < 1 || steps < 1) return fail(ctx, JM_ERR_VALUE, "bad arguments");
  if (ctx->mppi.noise_source != JM_NOISE_PHILOX)
    return fail(ctx, JM_ERR_UNSUPPORTED, "the device closed loop samples its own (Philox) noise");
  if (trials > jm::kMaxSeeds)
    return fail(ctx, JM_ERR_VALUE, "at most %d trials per batch (the master seeds are kernel parameters)", jm::kMaxSeeds);
  CK(cudaSetDevice(ctx->device));
  const int N = ctx->N, M = ctx->M, TM = ctx->TM, B = trials;
  const size_t S = (size_t)steps;
  // trial-major device buffers for this run
  jm::LoopState* d_loop = nullptr;
  double *d_unom = nullptr, *d_unew = nullptr, *d_hs = nullptr, *d_hc = nullptr, *d_rec = nullptr;
  double* d_scr = nullptr;
  int64_t* d_hj = nullptr;
  uint64_t* d_ht = nullptr;
  unsigned int* d_cnt = nullptr;
  cudaError_t e = dalloc(reinterpret_cast<char**>(&d_loop), sizeof(jm::LoopState) * (size_t)B);
  if (e == cudaSuccess) e = dalloc(&d_unom, 2 * (size_t)B * TM);  // per trial: two parities
  if (e == cudaSuccess) e = dalloc(&d_unew, (size_t)B * TM);
  if (e == cudaSuccess) e = dalloc(&d_hs, (size_t)B * (S + 1) * N);
  if (e == cudaSuccess) e = dalloc(&d_hc, (size_t)B * S * M);
  if (e == cudaSuccess) e = dalloc(&d_hj, (size_t)B * S);
  if (e == cudaSuccess) e = dalloc(&d_ht, (size_t)B * 2 * S);
  if (e == cudaSuccess) e = dalloc(&d_rec, (size_t)B * ctx->grid * ctx->rec_stride);
  if (e == cudaSuccess) e = dalloc(&d_cnt, (size_t)B);
  if (e == cudaSuccess) e = cudaMemset(d_cnt, 0, sizeof(unsigned int) * B);
  // (the batch runs the product kernels only: no eps slabs -- their sparse epilogue regenerates noise)
  std::vector<jm::LoopState> hl((size_t)B);
  std::vector<double> unom((size_t)B * 2 * TM, 0.0), hs0((size_t)B * (S + 1) * N, 0.0);
  for (int b = 0; b < B && e == cudaSuccess; ++b) {
    jm::LoopState& h = hl[b];
    h = jm::LoopState{};
    for (int i = 0; i < N; ++i) h.x[i] = x0[(size_t)b * N + i];
    for (int j = 0; j < M; ++j) h.u_init[j] = u_init[j];
    h.seed = seeds[b];
    h.sampler_jumps = sampler_jumps ? (sampler_jumps[b] != 0) : 1;
    h.iteration = 0;
    h.max_steps = steps;
    h.diverged_at = -1;
    h.hist_states = d_hs + (size_t)b * (S + 1) * N;
    h.hist_controls = d_hc + (size_t)b * S * M;
    h.hist_jumps = d_hj + (size_t)b * S;
    h.t_start = d_ht + (size_t)b * 2 * S;
    h.t_end = h.t_start + S;
    h.unom = d_unom + (size_t)b * 2 * TM;
    for (int t = 0; t < ctx->T; ++t)
      for (int j = 0; j < M; ++j) unom[(size_t)b * 2 * TM + (size_t)t * M + j] = u_init[j];  // controller.py:56-59
    for (int i = 0; i < N; ++i) hs0[(size_t)b * (S + 1) * N + i] = x0[(size_t)b * N + i];
  }
  cudaStream_t s = ctx->own_stream;
  if (e == cudaSuccess) e = xferAsync(d_loop, hl.data(), sizeof(jm::LoopState) * B, cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess) e = xferAsync(d_unom, unom.data(), sizeof(double) * unom.size(), cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess) e = xferAsync(d_hs, hs0.data(), sizeof(double) * hs0.size(), cudaMemcpyHostToDevice, s);
  // one control step of every trial = the two loop kernels with grid.y = B, captured once
  cudaGraph_t g = nullptr;
  cudaGraphExec_t ge = nullptr;
  if (e == cudaSuccess) {
    cudaStream_t saved_stream = ctx->stream;
    double* saved_rec = ctx->d_records;
    void* saved_scr = ctx->d_scratch;
    ctx->stream = s;
    ctx->d_records = d_rec;
    if (d_scr) ctx->d_scratch = d_scr;
    ctx->launch_trials = B;
    e = cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
    if (e == cudaSuccess) {
      jm::RolloutCall rc;
      rc.u_nom = d_unom;
      rc.loop = d_loop;
      rc.seeds = seeds;  // trial b's master seed is the kernels' seeds[b] (blockIdx.y = b)
      rc.nseeds = B;
      cudaError_t e1 = ctx->eng->rollout(ctx, rc);
      if (e1 == cudaSuccess) {
        jm::FinArgs f = fin_args(ctx, nullptr, 0);
        f.u_nom = d_unom;
        f.u_new = d_unew;
        f.counter = d_cnt;
        e1 = ctx->eng->finalize(ctx, f, d_loop, d_unom);
      }
      const cudaError_t e2 = cudaStreamEndCapture(s, &g);
      e = e1 != cudaSuccess ? e1 : e2;
    }
    ctx->launch_trials = 1;
    ctx->d_records = saved_rec;
    ctx->d_scratch = saved_scr;
    ctx->stream = saved_stream;
  }
  if (e == cudaSuccess) e = cudaGraphInstantiate(&ge, g, 0);
  for (int k = 0; k < steps && e == cudaSuccess; ++k) e = cudaGraphLaunch(ge, s);
  std::vector<double> hs((size_t)B * (S + 1) * N), hc((size_t)B * S * M);
  std::vector<int64_t> hj((size_t)B * S);
  std::vector<uint64_t> ht((size_t)B * 2 * S);
  if (e == cudaSuccess) e = xferAsync(hl.data(), d_loop, sizeof(jm::LoopState) * B, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = xferAsync(hs.data(), d_hs, sizeof(double) * hs.size(), cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = xferAsync(hc.data(), d_hc, sizeof(double) * hc.size(), cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = xferAsync(hj.data(), d_hj, sizeof(int64_t) * hj.size(), cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = xferAsync(ht.data(), d_ht, sizeof(uint64_t) * ht.size(), cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (ge) cudaGraphExecDestroy(ge);
  if (g) cudaGraphDestroy(g);
  for (void* ptr : {(void*)d_loop, (void*)d_unom, (void*)d_unew, (void*)d_hs, (void*)d_hc, (void*)d_hj, (void*)d_ht,
                    (void*)d_rec, (void*)d_cnt, (void*)d_scr})
    dfree(ptr);
  CK(e);
  // per trial: the reference's post-divergence fill (harness.py:144-148), as jm_closed_loop_host
  for (int b = 0; b < B; ++b) {
    const jm::LoopState& h = hl[b];
    const int done = h.step;
    const int last = (h.diverged_at >= 0) ? h.diverged_at : done;
    for (int k = 0; k <= steps; ++k) {
      const int src = std::min(k, last);
      if (states)
        for (int i = 0; i < N; ++i)
          states[((size_t)b * (S + 1) + k) * N + i] = hs[((size_t)b * (S + 1) + src) * N + i];
    }
    for (int k = 0; k < steps; ++k) {
      const bool valid = (h.diverged_at >= 0) ? k <= h.diverged_at : k < done;
      if (controls)
        for (int j = 0; j < M; ++j)
          controls[((size_t)b * S + k) * M + j] = valid ? hc[((size_t)b * S + k) * M + j] : 0.0;
      if (jumps) jumps[(size_t)b * S + k] = valid ? hj[(size_t)b * S + k] : 0;
      if (step_ns)
        step_ns[(size_t)b * S + k] = valid ? double(ht[(size_t)b * 2 * S + S + k] - ht[(size_t)b * 2 * S + k]) : 0.0;
    }
    if (diverged_at) diverged_at[b] = h.diverged_at;
    if (status) status[b] = h.status;
  }
  return JM_OK;
}

int jm_microbench(int device, double* fp32_tflops, double* mufu_tops, double* fp64_tflops) {
  jm_ctx* ctx = nullptr;
  CK(cudaSetDevice(device));
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
  float* d_out = nullptr;
  CK(dalloc(&d_out, (size_t)sms * 64));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  const int blocks = sms * 8, threads = 256;
  float best = 0.f;
  auto timeit = [&](auto launch) -> float {
    launch();  // warm-up (clocks ramp)
    launch();
    cudaEventRecord(e0);
    launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    return ms;
  };
  const int it_f = 8192, it_m = 2048, it_d = 2048;
  float ms = timeit([&] { jm::mb_ffma_kernel<<<blocks, threads>>>(d_out, it_f, 0.9999f, 1e-7f); });
  CK(cudaGetLastError());
  best = ms;
  if (fp32_tflops) *fp32_tflops = (double)blocks * threads * it_f * 32.0 * 2.0 / (best * 1e-3) / 1e12;
  ms = timeit([&] { jm::mb_mufu_kernel<<<blocks, threads>>>(d_out, it_m); });
  CK(cudaGetLastError());
  if (mufu_tops) *mufu_tops = (double)blocks * threads * it_m * 16.0 / (ms * 1e-3) / 1e12;
  ms = timeit([&] { jm::mb_dfma_kernel<<<blocks, threads>>>(reinterpret_cast<double*>(d_out), it_d, 0.9999, 1e-7); });
  CK(cudaGetLastError());
  if (fp64_tflops) *fp64_tflops = (double)blocks * threads * it_d * 16.0 * 2.0 / (ms * 1e-3) / 1e12;
  CK(cudaDeviceSynchronize());
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  dfree(d_out);
  return JM_OK;
}

static int ensure_flush(jm_ctx* ctx, int64_t bytes) {
  if (bytes <= 0 || (size_t)bytes <= ctx->flush_cap) return JM_OK;
  dfree(ctx->d_flush);
  ctx->d_flush = nullptr;
  ctx->flush_cap = 0;
  CK(cudaMalloc(&ctx->d_flush, (size_t)bytes));
  ctx->flush_cap = (size_t)bytes;
  return JM_OK;
}

static int loop_direct(jm_ctx* ctx, cudaEvent_t mid) {
  cudaStream_t saved = ctx->stream;
  ctx->stream = ctx->own_stream;
  cudaError_t e = loop_step_launches(ctx, mid);
  ctx->stream = saved;
  CK(e);
  return JM_OK;
}

int jm_bench_loop(jm_ctx* ctx, int32_t steps, int64_t flush_bytes, int32_t use_graph, double* step_ms,
                  double* rollout_ms) {
  if (!ctx || !ctx->graph_exec || steps < 1) return fail(ctx, JM_ERR_VALUE, "loop not initialised");
  CK(cudaSetDevice(ctx->device));
  int r = ensure_flush(ctx, flush_bytes);
  if (r != JM_OK) return r;
  cudaStream_t s = ctx->own_stream;
  std::vector<cudaEvent_t> ev(3 * (size_t)steps);
  for (auto& e : ev) CK(cudaEventCreate(&e));
  if (use_graph == 2) {
    // the whole timed run as ONE graph (the device-resident loop as deployed:
    // no host launch per control step); per step: L2 flush, event, the two
    // step kernels, event -- the flush stays outside each step's event pair
    cudaStream_t saved = ctx->stream;
    ctx->stream = s;
    cudaGraph_t g = nullptr;
    cudaGraphExec_t ge = nullptr;
    cudaError_t e = cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
    for (int i = 0; e == cudaSuccess && i < steps; ++i) {
      if (flush_bytes > 0) e = cudaMemsetAsync(ctx->d_flush, i & 0xFF, (size_t)flush_bytes, s);
      if (e == cudaSuccess) e = cudaEventRecordWithFlags(ev[3 * i], s, cudaEventRecordExternal);
      if (e == cudaSuccess) e = loop_step_launches(ctx, nullptr);
      if (e == cudaSuccess) e = cudaEventRecordWithFlags(ev[3 * i + 2], s, cudaEventRecordExternal);
    }
    const cudaError_t e2 = cudaStreamEndCapture(s, &g);
    ctx->stream = saved;
    if (e == cudaSuccess) e = e2;
    if (e == cudaSuccess) e = cudaGraphInstantiate(&ge, g, 0);
    if (e == cudaSuccess) e = cudaGraphLaunch(ge, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (ge) cudaGraphExecDestroy(ge);
    if (g) cudaGraphDestroy(g);
    CK(e);
    for (int i = 0; i < steps; ++i) {
      float a = 0.f;
      CK(cudaEventElapsedTime(&a, ev[3 * i], ev[3 * i + 2]));
      if (step_ms) step_ms[i] = a;
      if (rollout_ms) rollout_ms[i] = 0.0;
    }
    for (auto& ee : ev) cudaEventDestroy(ee);
    return JM_OK;
  }
  for (int i = 0; i < steps; ++i) {
    if (flush_bytes > 0) CK(cudaMemsetAsync(ctx->d_flush, i & 0xFF, (size_t)flush_bytes, s));
    CK(cudaEventRecord(ev[3 * i], s));
    if (use_graph) {
      CK(cudaGraphLaunch(ctx->graph_exec, s));
    } else {
      r = loop_direct(ctx, ev[3 * i + 1]);
      if (r != JM_OK) return r;
    }
    CK(cudaEventRecord(ev[3 * i + 2], s));
  }
  CK(cudaStreamSynchronize(s));
  for (int i = 0; i < steps; ++i) {
    float a = 0.f, b = 0.f;
    CK(cudaEventElapsedTime(&a, ev[3 * i], ev[3 * i + 2]));
    if (step_ms) step_ms[i] = a;
    if (rollout_ms) {
      if (!use_graph) CK(cudaEventElapsedTime(&b, ev[3 * i], ev[3 * i + 1]));
      rollout_ms[i] = use_graph ? 0.0 : b;
    }
  }
  for (auto& e : ev) cudaEventDestroy(e);
  return JM_OK;
}

int jm_bench_iteration(jm_ctx* ctx, int32_t reps, int64_t flush_bytes, double* iter_ms, double* rollout_ms) {
  if (!ctx || reps < 1) return fail(ctx, JM_ERR_VALUE, "bad arguments");
  CK(cudaSetDevice(ctx->device));
  int r = ensure_flush(ctx, flush_bytes);
  if (r != JM_OK) return r;
  const bool hbm = ctx->mppi.noise_source == JM_NOISE_HBM;
  jm::RolloutCall rc;
  rc.x0 = ctx->d_small + ctx->off_x0();
  rc.u_nom = ctx->d_small + ctx->off_unom();
  rc.seed = 1;
  rc.iteration = 0;
  rc.costs = ctx->d_costs;
  if (hbm) {
    const size_t eb = (size_t)ctx->TM * ctx->K * ctx->real_size;
    if (!ctx->d_hbm_eps) CK(cudaMalloc(&ctx->d_hbm_eps, eb));
    const bool sj = ctx->model.jump_channel == JM_JUMP_STATE;
    if (sj && !ctx->d_hbm_jump) CK(cudaMalloc(&ctx->d_hbm_jump, (size_t)ctx->T * ctx->Q * ctx->K * ctx->real_size));
    jm::NoiseArgs na = noise_args(ctx, 1, 0);
    na.eps_c_sm = ctx->d_hbm_eps;
    na.jump_sm = sj ? ctx->d_hbm_jump : nullptr;
    CK(ctx->eng->noise(ctx, na));
    rc.eps_in = ctx->d_hbm_eps;
    rc.jump_in = sj ? ctx->d_hbm_jump : nullptr;
  }
  cudaStream_t s = ctx->stream;
  std::vector<cudaEvent_t> ev(3 * (size_t)reps);
  for (auto& e : ev) CK(cudaEventCreate(&e));
  for (int i = 0; i < reps; ++i) {
    rc.iteration = (uint64_t)i;
    if (flush_bytes > 0) CK(cudaMemsetAsync(ctx->d_flush, i & 0xFF, (size_t)flush_bytes, s));
    CK(cudaEventRecord(ev[3 * i], s));
    CK(ctx->eng->rollout(ctx, rc));
    if (rollout_ms) CK(cudaEventRecord(ev[3 * i + 1], s));  // (an event between the kernels defeats PDL)
    jm::FinArgs f = fin_args(ctx, nullptr, 0);
    f.u_nom = rc.u_nom;
    f.u_new = ctx->d_small + ctx->off_unew();
    f.norms = ctx->d_small + ctx->off_norms();
    f.diag = ctx->d_diag();
    f.status = ctx->d_status();
    CK(ctx->eng->finalize(ctx, f, nullptr, nullptr));
    CK(cudaEventRecord(ev[3 * i + 2], s));
  }
  CK(cudaStreamSynchronize(s));
  for (int i = 0; i < reps; ++i) {
    float a = 0.f, b = 0.f;
    CK(cudaEventElapsedTime(&a, ev[3 * i], ev[3 * i + 2]));
    if (rollout_ms) CK(cudaEventElapsedTime(&b, ev[3 * i], ev[3 * i + 1]));
    if (iter_ms) iter_ms[i] = a;
    if (rollout_ms) rollout_ms[i] = b;
  }
  for (auto& e : ev) cudaEventDestroy(e);
  return JM_OK;
}

const char* jm_kernel_name(const jm_ctx* ctx) { return ctx ? ctx->variant.c_str() : ""; }

int jm_launches_per_iteration(const jm_ctx* ctx, int32_t* iteration, int32_t* loop_step) {
  if (!ctx) return fail(nullptr, JM_ERR_VALUE, "null context");
  if (iteration) *iteration = 2;  // rollout + finalize (+1 weights kernel when weights are requested)
  if (loop_step) *loop_step = 2;  // rollout + finalize (whose last CTA runs the plant step + shift)
  return JM_OK;
}

}  // extern "C"
