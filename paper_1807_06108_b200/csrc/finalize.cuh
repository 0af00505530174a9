// finalize.cuh -- the column-parallel finalize of one MPC iteration.
//
// Replaces controller.py:62-78 + :157-169 across the rollout's CTA records
// (log-sum-exp merge -> rho, Z, sum w^2, n_finite, N[t, j]), the update
// u_new = u_nom + N / (Z sqrt dt) (@ mapping^T), the diagnostics, the warm
// start shift (controller.py:96-100) and, in the closed loop, the plant step
// of run_trial (harness.py:131-150).
//
// finalize_kernel (kernels.cuh) merges every record in ONE CTA: a chain of
// dependent L2 round trips through ~120 KB of record columns on one SM (cfg1:
// 5 us from the rollout's completion to the update, tools/timeline.py).
// Here CTA b owns the columns [b*cw, (b+1)*cw) of the sequence -- whole steps,
// cw a multiple of m -- plus an m-column halo (the shifted sequence needs
// u_new[c + m]), and one thread per record: every thread issues all its loads
// (head + its columns) at once, one block minimum, one block sum of
// (Z, sum w^2, n_finite, N[cw + m]) in a fixed tree order (deterministic), and
// the CTA writes its columns.  The CTA holding column 0 runs the plant step;
// the last CTA to finish (a ticket) advances the loop's step / iteration
// counters or raises the drop-in call's done word.  The loop's nominal
// sequence is double-buffered by step parity (LoopState::unom), so no CTA's
// shifted writes race another CTA's reads.
//
// Used for the single-GPU loop, batched trials and the drop-in / host
// iteration; the multi-GPU exchanges (reduce mode, peer flags) keep
// finalize_kernel.
#pragma once
#include "kernels.cuh"

namespace jm {

constexpr int kFinColsMax = 12;  // columns + halo per CTA (quadrotor: 2 steps x 4 + 4)

// columns per CTA: whole steps (cartpole 4, quadrotor 8 = two steps, m = 2: 4, m = 3: 6), plus an
// m-column halo: at most kFinColsMax
__host__ __device__ __forceinline__ int fincol_width(int m) { return m == 4 ? 8 : (m == 3 ? 6 : 4); }
__host__ __device__ __forceinline__ int fincol_threads(int nrec) {
  const int t = (nrec + 31) / 32 * 32;
  return t < 32 ? 32 : (t > 512 ? 512 : t);
}

template <class Dyn>
__global__ void __launch_bounds__(512) finalize_cols(const FinArgs a, const PlantArgs p) {
  constexpr int N = Dyn::N, M = Dyn::M;
  const int trial = blockIdx.y;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
  const int TM = a.TM, cw = a.cols, rs = a.rec_stride;
  const int c0 = blockIdx.x * cw;
  const int ncol = min(cw, TM - c0);
  const int ntot = min(cw + M, TM - c0);  // this CTA's columns + the shift's halo
  const double* recs = a.rec + (size_t)trial * a.nrec * rs;  // (flag mode: parity slot added below)
  LoopState* L = a.loop ? a.loop + trial : nullptr;
  unsigned int* const counter = a.counter + trial;
  __shared__ double s_min[32];
  __shared__ double s_part[32][kFinColsMax + 3];
  __shared__ double s_sum[kFinColsMax + 3];
  __shared__ double s_un[kFinColsMax];
  __shared__ int s_last;
  __shared__ PlantPre s_pre;

  // before the grid dependency resolves: the loop state (stable until this
  // grid's last CTA advances it), the plant's noise, the nominal columns
  const uint64_t t_entry = globaltimer();
  const bool halted = L != nullptr && L->halted;
  const int step = L ? L->step : 0;
  unsigned long long* const tlr = (blockIdx.x == 0 && tid == 0) ? tl_row(L, step) : nullptr;  // (tuning timeline)
  const double* unom = L ? loop_unom(L, step, TM) : a.u_nom + (size_t)trial * TM;
  double* const unew = a.u_new ? a.u_new + (size_t)trial * TM : nullptr;
  if (L != nullptr && !halted && blockIdx.x == 0 && tid == (int)blockDim.x - 1) plant_prepare<Dyn>(p, s_pre);
  const double un_c = (tid < ntot) ? unom[c0 + tid] : 0.0;
  // touch this thread's record lines before the wait (address translation and the L2
  // lines' home: the first accesses after the rollout's completion otherwise pay
  // ~3k cycles; the data itself is read after the wait)
  if (tid < a.nrec) {
    const double* r = recs + (size_t)tid * rs;
    asm volatile("prefetch.global.L2 [%0];" ::"l"(r));
    asm volatile("prefetch.global.L2 [%0];" ::"l"(r + 4 + c0));
  }
  if (a.wait_flags != nullptr) {
    // world-1 record exchange (jm_loop_rollout_push layout): every rollout CTA raised its
    // record's epoch flag (release, GPU scope) -- wait for the flags instead of the whole
    // grid's completion; the rollout's reads of the loop state precede its record
    if (halted) return;
    const uint32_t epoch = (uint32_t)step + 1u;
    for (int r = tid; r < a.nrec; r += blockDim.x)
      while (ld_acquire_gpu(a.wait_flags + r) < epoch) {
      }
    __syncthreads();
    recs += (size_t)(epoch & 1u) * a.nrec * rs;
  } else {
    grid_dep_wait();
  }
  if (halted) return;
  tl_put(tlr, kTlFinEntry, t_entry);
  tl_put(tlr, kTlFinWait);

  // one record per thread (more than 1024 records: a strided loop): all loads at once
  double h0 = CUDART_INF, h1 = 0.0, h2 = 0.0, h3 = 0.0, col[kFinColsMax];
#pragma unroll
  for (int j = 0; j < kFinColsMax; ++j) col[j] = 0.0;
  double m = CUDART_INF;
  const bool one = a.nrec <= (int)blockDim.x;
  if (one) {
    if (tid < a.nrec) {
      const double* r = recs + (size_t)tid * rs;
      h0 = __ldcg(r);  // (L2: written by the rollout's CTAs on other SMs)
      h1 = __ldcg(r + 1);
      h2 = __ldcg(r + 2);
      h3 = __ldcg(r + 3);
#pragma unroll
      for (int j = 0; j < kFinColsMax; ++j)
        if (j < ntot) col[j] = __ldcg(r + 4 + c0 + j);
    }
    m = h0;
  } else {
    for (int b = tid; b < a.nrec; b += blockDim.x) m = fmin(m, recs[(size_t)b * rs]);
  }
  // global rho (controller.py:69: min over finite costs); every warp reduces the partials
  m = warp_min_redux(m);
  if (lane == 0) s_min[warp] = m;
  __syncthreads();
  const double rho = warp_min_redux(lane < nwarps ? s_min[lane] : CUDART_INF);
  // e_b = exp(-(rho_b - rho) / lambda): the log-sum-exp rescale of each record
  double z = 0.0, w2 = 0.0, nf = 0.0, acc[kFinColsMax];
#pragma unroll
  for (int j = 0; j < kFinColsMax; ++j) acc[j] = 0.0;
  if (rho != CUDART_INF) {
    if (one) {
      if (tid < a.nrec) {
        const double e = (h0 == CUDART_INF) ? 0.0 : exp(-(h0 - rho) * a.inv_lam);
        z = h1 * e;
        w2 = h2 * e * e;
        nf = h3;
#pragma unroll
        for (int j = 0; j < kFinColsMax; ++j) acc[j] = col[j] * e;  // 0 * inf = NaN like controller.py:78
      }
    } else {
      for (int b = tid; b < a.nrec; b += blockDim.x) {
        const double* r = recs + (size_t)b * rs;
        const double e = (r[0] == CUDART_INF) ? 0.0 : exp(-(r[0] - rho) * a.inv_lam);
        z = fma(r[1], e, z);
        w2 = fma(r[2], e * e, w2);
        nf += r[3];
#pragma unroll
        for (int j = 0; j < kFinColsMax; ++j)
          if (j < ntot) acc[j] = fma(r[4 + c0 + j], e, acc[j]);
      }
    }
  }
  // block sums of (Z, sum w^2, n_finite, N[ntot]): warp butterflies, then the
  // warp partials in warp order (fixed: bitwise reproducible)
  z = warp_sum(z);
  w2 = warp_sum(w2);
  nf = warp_sum(nf);
#pragma unroll
  for (int j = 0; j < kFinColsMax; ++j)
    if (j < ntot) acc[j] = warp_sum(acc[j]);
  if (lane == 0) {
    s_part[warp][0] = z;
    s_part[warp][1] = w2;
    s_part[warp][2] = nf;
#pragma unroll
    for (int j = 0; j < kFinColsMax; ++j) s_part[warp][3 + j] = acc[j];
  }
  __syncthreads();
  if (tid < ntot + 3) {
    double s = 0.0;
    for (int w = 0; w < nwarps; ++w) s += s_part[w][tid];
    s_sum[tid] = s;
  }
  __syncthreads();
  const double Z = s_sum[0], W2 = s_sum[1], NF = s_sum[2];
  const bool viable = rho != CUDART_INF;
  // delta = N / (Z sqrt dt) (controller.py:158), then the mapping (:159-160); the
  // CTA holds whole steps, so a step's m columns are all here
  if (tid < ntot) {
    double out = 0.0;
    if (viable) {
      const double scale = a.inv_sdt / Z;
      const int j = (c0 + tid) % M, cb = tid - j;
      if (a.mapping) {
        for (int l = 0; l < M; ++l) out = fma(a.mapping[j * M + l], s_sum[3 + cb + l] * scale, out);
      } else {
        out = s_sum[3 + tid] * scale;
      }
    }
    s_un[tid] = un_c + out;  // u_nom + delta, unclamped (controller.py:161); no viable rollout: u_nom
    if (tid < ncol && unew) unew[c0 + tid] = un_c + out;
    s_part[0][tid] = out;  // (delta, for the norms)
  }
  __syncthreads();
  tl_put(tlr, kTlFinMerged);
  if (a.norms && viable && tid < ncol / M) {  // per_step_update_norm (controller.py:168)
    double s2 = 0.0;
    for (int j = 0; j < M; ++j) s2 += s_part[0][tid * M + j] * s_part[0][tid * M + j];
    a.norms[c0 / M + tid] = sqrt(s2);
  }
  // warm_start_shift (controller.py:96-100): the loop's next nominal (the other
  // parity) or the drop-in call's u_shift
  double* const shift_out = L ? loop_unom(L, step + 1, TM) : a.u_shift;
  if (shift_out && tid < ncol) {
    const int c = c0 + tid;
    const double* ui = L ? L->u_init : a.u_init;
    shift_out[c] = (c < TM - M) ? s_un[tid + M] : ui[c - (TM - M)];
  }
  if (blockIdx.x == 0 && tid == 0) {
    if (a.status) *a.status = viable ? 0 : 3;  // JM_ERR_NO_VIABLE (controller.py:66-67)
    if (a.diag) *a.diag = viable ? DiagOut{rho, Z * Z / W2, Z, (int64_t)NF} : DiagOut{CUDART_INF, 0.0, 0.0, 0};
  }
  if (L != nullptr) {
    grid_dep_launch();  // the next control step's rollout may become resident
    if (blockIdx.x == 0) {
      // the plant step from u_new[0] (harness.py:136-148)
      if (tid == 0) {
        L->t_end[step] = globaltimer();
        if (!viable) {  // ControllerError("no viable rollout") ends the trial
          L->status = 3;
          L->halted = 1;
        } else {
          double u0[M];
          for (int j = 0; j < M; ++j) {
            double v = s_un[j];
            if (p.has_limits) v = fmin(fmax(v, p.u_lo[j]), p.u_hi[j]);  // harness.py:136
            u0[j] = v;
          }
          plant_advance<Dyn>(p, s_pre, u0, L);
        }
      }
    }
  }
  // the last CTA to finish: the loop's counters / the drop-in call's done word
  if (L != nullptr || a.done != nullptr) {
    __syncthreads();
    if (tid == 0) {
      unsigned int ticket;
      if (a.done != nullptr) {
        __threadfence_system();  // this CTA's outputs (pinned host memory) before the ticket
        ticket = atomicAdd(counter, 1u);
      } else {
        // one acquire-release atomic instead of a sequentially consistent fence + a relaxed one
        // (the fence was 25% of this kernel's stall samples): our writes are released, the last
        // CTA acquires the others' (L->halted from the plant CTA)
        asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], 1;" : "=r"(ticket) : "l"(counter) : "memory");
      }
      s_last = (ticket == gridDim.x - 1) ? 1 : 0;
      if (s_last) {
        if (a.done != nullptr) __threadfence();
        *counter = 0u;  // (read again by the next launch only)
        if (L != nullptr) {
          tl_put(tl_row(L, step), kTlFinEnd);
          if (!L->halted) {
            L->iteration += 1;  // ControllerState(..., k+1, cfg) (harness.py:150)
            L->step += 1;
            if (L->step >= L->max_steps) L->halted = 1;
          }
        }
        if (a.done != nullptr) {
          __threadfence_system();
          *a.done = 1;
        }
      }
    }
  }
}

}  // namespace jm
