// rollout_fast.cuh -- the product rollout kernel (non-trace: Philox or HBM noise).
//
// Replaces controller.py:118-158 (sample_noise_batch, the T-step loop of
// modified cost + step_unchecked, the per-CTA half of compute_weights and the
// weighted noise sum) for every launch that does not return trajectories.
// Differences from rollout_kernel (kernels.cuh, kept for the TRACE path):
//
//  * No eps slab.  The weighted sum N[t,j] = sum_k w_k eps[k,t,j] needs eps
//    again once the weights are known; instead of storing every sample's
//    T*m noise values (a 179 KB shared slab at cfg1, 240 MB of L2/HBM slabs at
//    cfg3) the epilogue REGENERATES the noise of the samples that carry
//    weight.  With lambda = 1 and costs spread over 1e2..1e4 a tile has
//    1-3 samples within (S - rho)/lambda <= 55 of its minimum
//    (tools/weight_sparsity.py, B200: 0.4-1% of a tile at cfg1/cfg2/cfg3);
//    the others' weights, < e^-55 = 1.3e-24 of the tile's best, are dropped
//    from N (their sum over K <= 2^24 samples changes N by < 1e-16
//    relative) but not from Z, sum w^2 or the finite count.  Regeneration is
//    exact: the same Philox blocks, Box-Muller, Cholesky product and jump
//    marks (jump clock walked from t = 0) as the rollout, so N is the dense
//    sum minus the negligible terms.  HBM mode re-reads the fed columns of
//    those samples instead, and also revisits non-finite-cost samples with
//    weight 0 so a non-finite fed eps still turns N into NaN as the
//    reference's einsum does (controller.py:78).
//  * SPT = 2 samples per thread in packed f32x2 registers (vec2.cuh): one
//    FFMA2/FMUL2/FADD2 issue slot for both samples' dynamics, cost and
//    sincos.  Noise: per sample, per Philox block (4 normals: 4 cartpole
//    steps, 1 quadrotor step), one block pipelined ahead.
//  * Jump-mark staging buffer cleared per event (each lane zeroes the entries
//    of its previous window's events) instead of per window row.
//  * c = 1 (cq = 0) with Philox noise: the eps'eps term is fma(0, quad, inc) =
//    inc exactly (finite noise), so it is not formed (QUAD = false).
#pragma once
#include "kernels.cuh"

namespace jm {

#ifndef JM_PACKED_THREADS
#define JM_PACKED_THREADS 256
#endif
constexpr int kPackedThreads = JM_PACKED_THREADS;  // threads per CTA of the two-samples-per-thread kernels (2 CTAs per SM)
#ifndef JM_HBM_DEPTH
#define JM_HBM_DEPTH 2
#endif
constexpr int kHbmDepth = JM_HBM_DEPTH;  // HBM mode: noise groups in flight ahead of the one being consumed
constexpr float kSparseCut = 55.0f;  // (S - rho) / lambda above which N drops the sample (w < e^-55)

template <int SPT, typename Real>
struct VecOf {
  using type = Real;
};
template <>
struct VecOf<2, float> {
  using type = F2;
};

// build V from SPT per-sample scalars / read half u of V
__device__ __forceinline__ float vpack(const float* s, std::integral_constant<int, 1>) { return s[0]; }
__device__ __forceinline__ double vpack(const double* s, std::integral_constant<int, 1>) { return s[0]; }
__device__ __forceinline__ F2 vpack(const float* s, std::integral_constant<int, 2>) { return F2(s[0], s[1]); }
template <typename V, typename R>
__device__ __forceinline__ V vcast(R s) {
  return V(scalar_t<V>(s));
}

// uncontracted add / mul on every arithmetic type (marks, jump increments:
// the rollout and the regeneration round them alike)
__device__ __forceinline__ float vadd(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ double vadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ F2 vadd(F2 a, F2 b) { return a + b; }
// eps_d + eps_j (control-channel marks): two scalar __fadd_rn, not one packed add.  The f32x2 add
// -- the __fadd2_rn builtin, and inline `add.rn.f32x2` alike -- was fused with the packed multiply
// before it (eps = L z, then + mark became one FFMA2), moving eps_c by an ulp against the sampler's
// scalar sum on most events (tests/test_gpu_fullsize.py
// test_philox_and_hbm_kernels_agree_control_channel_jumps pins it).  The state-jump sum x + H mark
// keeps vadd: what precedes it is an fma, which cannot absorb an add.
__device__ __forceinline__ float vadd_exact(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ double vadd_exact(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ F2 vadd_exact(F2 a, F2 b) { return F2(__fadd_rn(a.v.x, b.v.x), __fadd_rn(a.v.y, b.v.y)); }
// jscale * mark of the fed-noise path, per half for the same reason (the Philox path stages rmul(jscale, mark))
__device__ __forceinline__ float vmul_exact(float s, float a) { return __fmul_rn(s, a); }
__device__ __forceinline__ double vmul_exact(double s, double a) { return __dmul_rn(s, a); }
__device__ __forceinline__ F2 vmul_exact(float s, F2 a) { return F2(__fmul_rn(s, a.v.x), __fmul_rn(s, a.v.y)); }

// eps = L z, fixed fma order (apply_chol in kernels.cuh: the same operations per sample)
template <int M, typename V, typename S>
__device__ __forceinline__ void chol_v(const S* L, const V* z, V* eps) {
#pragma unroll
  for (int j = 0; j < M; ++j) {
    V acc = L[j * M] * z[0];
#pragma unroll
    for (int l = 1; l <= j; ++l) acc = fma(L[j * M + l], z[l], acc);
    eps[j] = acc;
  }
}

// one Philox block of diffusion normals (4 words -> 4 normals)
__device__ __forceinline__ void block_normals(const StreamKey& sk, uint32_t b, uint32_t kg, float* z) {
  const P4 r = draw(sk, kSlotDiffusion, b, kg);
  box_muller(r.x, r.y, z[0], z[1]);
  box_muller(r.z, r.w, z[2], z[3]);
}

// box_muller (philox.cuh) of two samples at once: its FADD / FFMA / FMULs packed,
// the MUFU steps per half -- every operation per half as the scalar form, so the
// normals are bit-identical (the regeneration draws them with the scalar form)
__device__ __forceinline__ void box_muller2(uint32_t a0, uint32_t a1, uint32_t b0, uint32_t b1, F2& z0, F2& z1) {
  const F2 u1 = 2.0f - F2(__uint_as_float(0x3F800000u | (a0 >> 9)), __uint_as_float(0x3F800000u | (a1 >> 9)));
  const F2 ang = fma(F2(__uint_as_float(0x3F800000u | (b0 >> 9)), __uint_as_float(0x3F800000u | (b1 >> 9))),
                     6.2831853071795865f, -9.4247779607693797f);
  float l0, l1, r0, r1;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(l0) : "f"(u1.v.x));
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(l1) : "f"(u1.v.y));
  const F2 rr = -1.3862943611198906f * F2(l0, l1);
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r0) : "f"(rr.v.x));
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r1) : "f"(rr.v.y));
  float s0, c0, s1, c1;
  __sincosf(ang.v.x, &s0, &c0);
  __sincosf(ang.v.y, &s1, &c1);
  const F2 r(r0, r1);
  z0 = r * F2(c0, c1);
  z1 = r * F2(s0, s1);
}

// the block's normals of this thread's SPT samples, as V
__device__ __forceinline__ void block_normals_v(const StreamKey& sk, uint32_t b, const uint32_t* kg, float* z) {
  block_normals(sk, b, kg[0], z);
}
__device__ __forceinline__ void block_normals_v(const StreamKey& sk, uint32_t b, const uint32_t* kg, double* z) {
  float f[4];
  block_normals(sk, b, kg[0], f);
#pragma unroll
  for (int i = 0; i < 4; ++i) z[i] = double(f[i]);
}
__device__ __forceinline__ void block_normals_v(const StreamKey& sk, uint32_t b, const uint32_t* kg, F2* z) {
  const P4 r0 = draw(sk, kSlotDiffusion, b, kg[0]);
  const P4 r1 = draw(sk, kSlotDiffusion, b, kg[1]);
  box_muller2(r0.x, r1.x, r0.y, r1.y, z[0], z[1]);
  box_muller2(r0.z, r1.z, r0.w, r1.w, z[2], z[3]);
}

// ---------------------------------------------------------------- mark staging, two forms
// Dense (q = 1): one Real per (step, sample) of the window, zero where no event.
// Indexed (q >= 2): one BYTE per (step, thread) -- 0, or the entry of the warp's compact mark
// table holding the q values of that step's event for each of the thread's SPT samples (zero
// for a sample without one; entry 0 is all zero), laid out [i][half] so a step still reads
// each component of both halves with one load -- a window costs tile / SPT x W bytes instead
// of tile x W x q Reals and reaches ~10 times further for the same shared memory (quadrotor,
// q = 3, two CTAs per SM: 128 steps instead of 12; each window costs a clock pass, a prefix
// scan and a cooperative mark pass of fixed latency).  A warp's window holds at most
// kMarkCap - 1 entries; the launch sizes W from nu dt so that is ~1.6x the expected count,
// and a window that still overflows is halved and redone from the saved clocks (exact for
// any rate: one step of a warp has at most 32 entries).
constexpr int kMarkCap = 256;
__host__ __device__ constexpr bool marks_indexed(int q) { return q >= 2; }
__host__ __device__ __forceinline__ size_t fast_marks_bytes(int tile, int nwarps, int W, int q, int rs) {
  if (W <= 0) return 0;
  if (!marks_indexed(q)) return (size_t)rs * tile * W * q;
  const int spt = tile / (nwarps * 32);
  return (((size_t)nwarps * 32 * W + 15) & ~(size_t)15) + (size_t)rs * nwarps * kMarkCap * q * spt;
}
// the longest indexed window whose expected event count per warp stays below ~5/8 of the table
// (p = nu dt as jthr / 2^32; spt samples per lane)
__host__ __device__ __forceinline__ int marks_window_cap(uint32_t jthr, int spt) {
  const double ev_per_step = 32.0 * spt * (double)jthr / 4294967296.0;  // (jthr = ceil(p 2^24) << 8)
  const double w = 160.0 / (ev_per_step > 1e-12 ? ev_per_step : 1e-12);
  return w >= 128.0 ? 128 : (w < 4.0 ? 4 : ((int)w & ~3));
}

// ---------------------------------------------------------------- jump windows (clearing form)
// jump_window (kernels.cuh) with (a) the owner lane's sample at kg + (L - lane)
// * kstride (two samples per thread: the even / odd samples of a warp form one
// 32-lane window each), (b) a buffer that stays zero outside event entries:
// each lane first clears the entries of its previous window's events (prev),
// instead of the warp zeroing every row of the window.
// Entry (s, i, L) at wd[((s * Q + i) * 32 + L) * ES]: ES = SPT interleaves the
// two halves of a thread (one 8-byte load reads both samples' marks).
template <int Q, int QP, int JM, int ES, typename Real>
__device__ __forceinline__ void jump_window_c(JumpClock& c, Mask128& prev, int w0, int wend, const StreamKey& sk,
                                              uint32_t kg, int kstride, const GapSampler& gs, const Real* Lj,
                                              const Real* mu, Real jscale, Real* wd, bool poisson,
                                              const CountTable& ct) {
  const int lane = threadIdx.x & 31;
  Mask128 mask{};
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
  for (Mask128 m = prev; m.lo | m.hi; mask_pop(m)) {
    const int s = mask_low(m);
#pragma unroll
    for (int i = 0; i < Q; ++i) wd[((s * Q + i) * 32 + lane) * ES] = Real(0);
  }
  prev = mask;
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
    Mask128 mL = mask_shfl(mask, L);
    if (j < tot) {
      for (int r = 0; r < k; ++r) mask_pop(mL);
      const int s = mask_low(mL);
      Real mk[Q];
      mark_of<Q, QP, Real>(sk, kg + (uint32_t)((L - lane) * kstride), eL, Lj, mu, mk, poisson, ct);
#pragma unroll
      for (int i = 0; i < Q; ++i) wd[((s * Q + i) * 32 + L) * ES] = (JM == 1) ? rmul<Real>(jscale, mk[i]) : mk[i];
    }
  }
  __syncwarp();
}

// ---------------------------------------------------------------- jump window, indexed staging
// The events of [w0, wend) of one sample: its clock advanced past the window, the event
// steps as a mask relative to w0; returns their number.
__device__ __forceinline__ int window_events(JumpClock& c, int w0, int wend, const StreamKey& sk, uint32_t kg,
                                             const GapSampler& gs, Mask128& mask) {
  mask = Mask128{0ull, 0ull};
  int n = 0;
  while (__any_sync(0xFFFFFFFFu, c.tj < wend)) {
    if (c.tj < wend) {
      mask_set(mask, c.tj - w0);
      ++n;
      clock_next(c, sk, kg, gs);
    }
  }
  return n;
}

// One window of a warp's 32 threads x SPT samples (lane's samples kg0 + u) in ONE cooperative
// pass: the (thread, step) pairs with an event on either sample form one list (by lane, then
// time), lane j computes entry j's mark(s) into table entry 1 + j -- tabw[((1 + j) * Q + i) *
// SPT + u], zero for a sample without an event at that step -- and stores that byte at
// ib[(step - w0) * 32 + lane].  Returns the window's end (<= wend_max; shorter only after an
// overflow, a multiple of `gran` steps past w0).
__device__ __forceinline__ int mask_count_below(const Mask128& m, int s) {  // set bits below bit s
  const uint64_t lo = s >= 64 ? m.lo : (m.lo & ((1ull << s) - 1ull));
  const uint64_t hi = s >= 64 ? (m.hi & ((1ull << (s - 64)) - 1ull)) : 0ull;
  return __popcll(lo) + __popcll(hi);
}
__device__ __forceinline__ bool mask_test(const Mask128& m, int s) {
  return ((s >= 64 ? m.hi >> (s - 64) : m.lo >> s) & 1ull) != 0ull;
}

template <int Q, int QP, int JM, int SPT, typename Real>
__device__ __forceinline__ int jump_window_idx(JumpClock* c, Mask128& prev, int w0, int wend_max, int gran,
                                               const StreamKey& sk, uint32_t kg0, const GapSampler& gs,
                                               const Real* Lj, const Real* mu, Real jscale, uint8_t* ib, Real* tabw,
                                               bool poisson, const CountTable& ct) {
  const int lane = threadIdx.x & 31;
  int wend = wend_max;
  Mask128 mask[SPT], um;
  uint32_t e0[SPT];
  int nl, inc, tot;
  for (;;) {
    JumpClock saved[SPT];
    um = Mask128{0ull, 0ull};
#pragma unroll
    for (int u = 0; u < SPT; ++u) {
      saved[u] = c[u];
      e0[u] = c[u].e;
      window_events(c[u], w0, wend, sk, kg0 + (uint32_t)u, gs, mask[u]);
      um.lo |= mask[u].lo;
      um.hi |= mask[u].hi;
    }
    nl = __popcll(um.lo) + __popcll(um.hi);
    inc = nl;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xFFFFFFFFu, inc, o);
      if (lane >= o) inc += v;
    }
    tot = __shfl_sync(0xFFFFFFFFu, inc, 31);
    if (tot < kMarkCap) break;  // (uniform)
    // overflow: redo a window half as long from the saved clocks
#pragma unroll
    for (int u = 0; u < SPT; ++u) c[u] = saved[u];
    const int half = ((wend - w0) / 2 / gran) * gran;
    wend = w0 + (half > gran ? half : gran);
  }
  const int off = inc - nl;
  __syncwarp();  // the previous window's bytes have been read
  for (Mask128 m = prev; m.lo | m.hi; mask_pop(m)) ib[mask_low(m) * 32 + lane] = 0;
  prev = um;
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
    Mask128 mL[SPT];
    uint32_t eL[SPT];
    Mask128 uL{0ull, 0ull};
#pragma unroll
    for (int u = 0; u < SPT; ++u) {
      mL[u] = mask_shfl(mask[u], L);
      eL[u] = __shfl_sync(0xFFFFFFFFu, e0[u], L);
      uL.lo |= mL[u].lo;
      uL.hi |= mL[u].hi;
    }
    if (j < tot) {
      for (int r = 0; r < k; ++r) mask_pop(uL);
      const int sidx = mask_low(uL);
      Real* const ent = tabw + (size_t)(1 + j) * Q * SPT;
#pragma unroll
      for (int u = 0; u < SPT; ++u) {
        Real mk[Q];
#pragma unroll
        for (int i = 0; i < Q; ++i) mk[i] = Real(0);
        if (mask_test(mL[u], sidx))
          mark_of<Q, QP, Real>(sk, kg0 + (uint32_t)((L - lane) * SPT + u),
                               eL[u] + (uint32_t)mask_count_below(mL[u], sidx), Lj, mu, mk, poisson, ct);
#pragma unroll
        for (int i = 0; i < Q; ++i) ent[i * SPT + u] = (JM == 1) ? rmul<Real>(jscale, mk[i]) : mk[i];
      }
      ib[sidx * 32 + L] = (uint8_t)(1 + j);
    }
  }
  __syncwarp();
  return wend;
}

// ---------------------------------------------------------------- regeneration
// eps_combined of sample kg over the steps of Philox block b (4 / MP steps) into
// out[t * M + j] -- the rollout's own draws: block_normals, the same Cholesky
// fma order, control-channel marks added with an uncontracted add.
template <int M, int MP, int Q, int QP, int JM, typename Real>
__device__ __forceinline__ void regen_philox(const RolloutArgs<Real>& a, const StreamKey& sk, const GapSampler& gs,
                                             uint32_t kg, int b, const Real* Ld, const Real* Lj, const Real* mu,
                                             bool jumps, Real* out) {
  constexpr int SB = 4 / MP;
  const int t0 = b * SB;
  float z[4];
  block_normals(sk, (uint32_t)b, kg, z);
  JumpClock clk;
  const bool marks = JM == 0 && jumps;
  if (marks) {
    clock_start(clk, sk, kg, gs);
    while (clk.tj < t0) clock_next(clk, sk, kg, gs);
  }
#pragma unroll
  for (int s2 = 0; s2 < SB; ++s2) {
    const int t = t0 + s2;
    if (t >= a.T) break;
    Real eps[M];
    apply_chol<M, Real>(Ld, z + s2 * MP, eps);
    if (marks && clk.tj == t) {
      Real mk[Q];
      mark_of<Q, QP, Real>(sk, kg, clk.e, Lj, mu, mk, a.poisson != 0, a.cnt);
#pragma unroll
      for (int j = 0; j < M; ++j) eps[j] = radd<Real>(eps[j], mk[(j < Q) ? j : 0]);
      clock_next(clk, sk, kg, gs);
    }
#pragma unroll
    for (int j = 0; j < M; ++j) out[t * M + j] = eps[j];
  }
}

// ---------------------------------------------------------------- sparse tile epilogue
// Online softmax of one tile into the CTA accumulator (the per-CTA half of
// compute_weights + _weighted_noise_average, controller.py:62-78):
// rho_new = min(rho_acc, min_tile S); w_k = exp(-(S_k - rho_new)/lambda);
// Z, sum w^2 and n_finite over every sample; N[r] += w_k eps[r, k] over the
// samples with (S_k - rho_new)/lambda <= kSparseCut, whose eps rows
// regen(col, item, row_out) rewrites (nb items of ipt steps per sample) into a
// chunk scratch, summed in list order (fixed: deterministic).  Every thread
// calls it; Sf/cols hold its SPT samples (+inf / -1 for none).
struct SparseSmem {
  double (*s_red)[32];
  double* s_acc;
  int* s_cnt;
  int* sig_col;
  float* sig_w;  // weights as float (the fp32 kernels' w; fp64 kernels round the weight of a
  double* sig_wd;  // ... or as double)
  void* scratch;
  int chunk;     // samples per regeneration chunk
};

template <int SPT, typename Real, class Regen>
__device__ __forceinline__ void sparse_epilogue(const Real* Sf, const int* cols, int TM, Real inv_lam, double* Nacc,
                                                const SparseSmem& sm, int nb, bool keep_nonfinite, Regen regen) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  const int nthreads = blockDim.x;
  Real mloc = r_inf<Real>();
#pragma unroll
  for (int u = 0; u < SPT; ++u) mloc = fmin(mloc, Sf[u]);
  const double m = warp_min_redux(double(mloc));
  if (lane == 0) sm.s_red[0][warp] = m;
  __syncthreads();
  const double mm = warp_min_redux(lane < nwarps ? sm.s_red[0][lane] : CUDART_INF);
  const double rho_prev = sm.s_acc[0];
  const double rho_new = fmin(rho_prev, mm);
  if (rho_new == CUDART_INF) return;  // no finite cost yet in this CTA (uniform)
  double scale_old = 0.0;
  if (rho_prev != CUDART_INF) {
    const double e = lane == 0 ? exp((rho_new - rho_prev) * double(inv_lam)) : 0.0;
    scale_old = __shfl_sync(0xFFFFFFFFu, e, 0);
  }
  double z1 = 0.0, z2 = 0.0;
  int nf = 0, cnt = 0;
  Real w[SPT];
  bool sig[SPT];
  uint32_t bal[SPT];
#pragma unroll
  for (int u = 0; u < SPT; ++u) {
    const bool fin = Sf[u] < r_inf<Real>();
    const Real d = (Sf[u] - Real(rho_new)) * inv_lam;
    w[u] = fin ? r_exp<Real>(-d) : Real(0);
    z1 += double(w[u]);
    z2 += double(w[u]) * double(w[u]);
    nf += fin ? 1 : 0;
    sig[u] = cols[u] >= 0 && (fin ? d <= Real(kSparseCut) : keep_nonfinite);
    bal[u] = __ballot_sync(0xFFFFFFFFu, sig[u]);
    cnt += __popc(bal[u]);
  }
  z1 = warp_sum(z1);
  z2 = warp_sum(z2);
  nf = __reduce_add_sync(0xFFFFFFFFu, nf);
  if (lane == 0) {
    sm.s_red[1][warp] = z1;
    sm.s_red[2][warp] = z2;
    sm.s_red[3][warp] = double(nf);
    sm.s_cnt[warp] = cnt;
  }
  __syncthreads();  // partials and counts complete; s_acc[0] has been read by every thread
  if (warp == nwarps - 1 && lane == 0) {
    double a1 = 0.0, a2 = 0.0, a3 = 0.0;
    for (int w2 = 0; w2 < nwarps; ++w2) {
      a1 += sm.s_red[1][w2];
      a2 += sm.s_red[2][w2];
      a3 += sm.s_red[3][w2];
    }
    sm.s_acc[0] = rho_new;
    sm.s_acc[1] = sm.s_acc[1] * scale_old + a1;
    sm.s_acc[2] = sm.s_acc[2] * scale_old * scale_old + a2;
    sm.s_acc[3] += a3;
  }
  // the list of weighted samples: warp order, then sample slot u, then lane
  int off = 0, nsig = 0;
  for (int w2 = 0; w2 < nwarps; ++w2) {
    const int c = sm.s_cnt[w2];
    off += (w2 < warp) ? c : 0;
    nsig += c;
  }
  const uint32_t below = (1u << lane) - 1u;
#pragma unroll
  for (int u = 0; u < SPT; ++u) {
    if (sig[u]) {
      const int p = off + __popc(bal[u] & below);
      sm.sig_col[p] = cols[u];
      if constexpr (sizeof(Real) == 4)
        sm.sig_w[p] = float(w[u]);
      else
        sm.sig_wd[p] = double(w[u]);
    }
    off += __popc(bal[u]);
  }
  // the earlier tiles' N relative to the new minimum (multi-tile CTAs)
  if (scale_old != 1.0)
    for (int r = threadIdx.x; r < TM; r += nthreads) Nacc[r] = (rho_prev == CUDART_INF) ? 0.0 : Nacc[r] * scale_old;
  __syncthreads();  // the list is complete
  Real* scr = reinterpret_cast<Real*>(sm.scratch);
  for (int c0 = 0; c0 < nsig; c0 += sm.chunk) {
    const int nc = min(sm.chunk, nsig - c0);
    for (int it = threadIdx.x; it < nc * nb; it += nthreads) {
      const int si = it / nb;
      regen(sm.sig_col[c0 + si], it - si * nb, scr + (size_t)si * TM);
    }
    __syncthreads();
    for (int r = threadIdx.x; r < TM; r += nthreads) {
      double acc = 0.0;
      for (int si = 0; si < nc; ++si) {
        const double wk = (sizeof(Real) == 4) ? double(sm.sig_w[c0 + si]) : sm.sig_wd[c0 + si];
        acc = fma(wk, double(scr[(size_t)si * TM + r]), acc);  // 0 * inf = NaN like controller.py:78
      }
      Nacc[r] += acc;
    }
    __syncthreads();
  }
}

// regeneration items per sample: Philox blocks (4 / MP steps each), or HBM groups of GS steps
__host__ __device__ __forceinline__ int regen_items(int T, int steps_per_item) {
  return (T + steps_per_item - 1) / steps_per_item;
}

// ---------------------------------------------------------------- rollout, warp-specialised
// Philox, non-trace.  The block is 2C threads: warps [0, C/32) are consumers
// (one sample each: dynamics + modified cost), warps [C/32, 2C/32) producers
// (thread C+c draws the noise of consumer c's sample).  Per 4-step group a
// producer writes eps_combined (and the state-jump increments, JM = 1) into
// a shared-memory ring of NBUF slots; full/empty handshakes are named barriers
// (bar.arrive / bar.sync over all 2C threads).  Used for small tiles, where
// a few warps per SM cannot hide the dynamics chain's latency: moving the
// noise to other warps roughly doubles the warps in flight (measured: a win
// up to ~128 samples per SM, a loss above, where the +30% instructions of
// the hand-off dominate).  Same noise bits as rollout_fast; the
// same sparse epilogue (the weighted samples' noise regenerated by all 2C
// threads, no eps slab).
__device__ __forceinline__ void named_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void named_arrive(int id, int n) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}

template <class Sys, int JM>
struct WsShape {
  static constexpr int M = Sys::M;
  static constexpr int Q = (JM == 0) ? M : Sys::Dyn::QJ;
  static constexpr int GW = 4 * M + (JM == 1 ? 4 * Q : 0);  // Reals per sample per group
};

// regeneration chunk of the WS kernel: samples per pass of its 2C threads over nb items each
__host__ __device__ __forceinline__ int ws_chunk(int C, int nb) {
  const int c = (2 * C) / nb;
  return c < 1 ? 1 : (c > C ? C : c);
}

template <class Sys, typename Real, int JM, int MAXT, int kWsBuf>
__global__ void __launch_bounds__(MAXT) rollout_kernel_ws(const RolloutArgs<Real> a) {
  using Dyn = typename Sys::Dyn;
  using Cost = typename Sys::Cost;
  constexpr int N = Sys::N, M = Sys::M;
  constexpr int MP = Pad<M>::value;
  constexpr int Q = (JM == 0) ? M : Dyn::QJ;
  constexpr int QP = Pad<Q>::value;
  constexpr int TS = 2 * M + 1;
  constexpr int GW = WsShape<Sys, JM>::GW;

  extern __shared__ double smem_d[];
  __shared__ double s_red[4][32];
  __shared__ double s_acc[4];
  __shared__ int s_cnt[32];
  __shared__ int s_sigc[MAXT / 2];
  __shared__ double s_sigw[MAXT / 2];

  const int TM = a.TM, T = a.T, K = a.K;
  const int C = blockDim.x >> 1;  // samples per tile
  const int nitems = regen_items(T, 4 / MP);  // regeneration items (Philox blocks) per sample
  const int chunk = ws_chunk(C, nitems);
  const SmemPlan sp_ = smem_plan(TM, T * TS, C, a.jump_on ? (C >> 5) * 32 * a.jw_len * Q : 0, kWsBuf * GW * C,
                                 chunk * TM, a.gap_n, (int)sizeof(Real));
  char* const sb = reinterpret_cast<char*>(smem_d);
  double* Nacc = reinterpret_cast<double*>(sb + sp_.nacc);
  Real* tab = reinterpret_cast<Real*>(sb + sp_.tab);
  Real* ring = reinterpret_cast<Real*>(sb + sp_.ring);  // [slot][w][c]
  uint32_t* Sg = reinterpret_cast<uint32_t*>(sb + sp_.gap);
  const SparseSmem sm{s_red, s_acc, s_cnt, s_sigc, reinterpret_cast<float*>(s_sigw), s_sigw, sb + sp_.scr, chunk};

  grid_dep_wait();
  grid_dep_launch();
  LoopState* L = a.loop ? a.loop + blockIdx.y : nullptr;
  if (L != nullptr && L->halted) return;
  const uint64_t iter = L ? L->iteration : (a.iteration_dev ? *a.iteration_dev : a.iteration);
  const double* x0 = L ? L->x : a.x0;
  if (L != nullptr && blockIdx.x == 0 && threadIdx.x == 0) L->t_start[L->step] = globaltimer();
  rollout_prologue<M, Real>(a, L ? loop_unom(L, L->step, TM) : a.u_nom + (size_t)blockIdx.y * TM, tab, Nacc, s_acc, Sg);
  __syncthreads();

  const bool producer = (int)threadIdx.x >= C;
  const int c = producer ? (int)threadIdx.x - C : (int)threadIdx.x;
  const int G = (T + 3) >> 2;
  const int nb = 2 * C;
  double* const costs_out = gridDim.y > 1 ? nullptr : (a.costs_dev ? *a.costs_dev : a.costs);

  for (int tile = blockIdx.x; tile < a.ntiles; tile += gridDim.x) {
    const int base = tile * C;
    const int kl = base + c;
    const bool act = kl < K;
    Real Sf = r_inf<Real>();
    if (producer) {
      const StreamKey sk = make_stream_key(a.seeds[blockIdx.y], iter);
      const uint32_t kg = (uint32_t)(a.sample_offset + kl);
      Real Ld[M * M], Lj[Q * Q], mu[Q];
#pragma unroll
      for (int i = 0; i < M * M; ++i) Ld[i] = a.Ld[i];
#pragma unroll
      for (int i = 0; i < Q * Q; ++i) Lj[i] = a.Lj[i];
#pragma unroll
      for (int i = 0; i < Q; ++i) mu[i] = a.mu_j[i];
      const Real jscale = a.jscale;
      const GapSampler gs{Sg, T, a.gap_inv};
      const int JW = a.jw_len;
      const bool jumps = a.jump_on && (L == nullptr || L->sampler_jumps);
      Real* const wd = reinterpret_cast<Real*>(sb + sp_.marks) + (c >> 5) * 32 * JW * Q;
      JumpClock clk;
      const Real* wl = wd + (c & 31);
      int wnext = 0;
      if (jumps) clock_start(clk, sk, kg, gs);
      // the producers' horizon, unswitched on the sampler's jump flag
      auto produce = [&](auto jtag) {
        constexpr bool J = decltype(jtag)::value;
        for (int g = 0; g < G; ++g) {
          const int slot = g % kWsBuf;
          const int t0 = 4 * g;
          if (J && t0 == wnext) {
            wnext = t0 + JW;
            jump_window<Q, QP, JM, Real>(clk, t0, min(wnext, T), JW, sk, kg, gs, Lj, mu, jscale, wd, a.poisson != 0,
                                         a.cnt);
            wl = wd + (c & 31);
          }
          float z[4 * MP];
          group_normals<MP>(sk, (uint32_t)t0, kg, z);
          Real eps[4][M], sj[4][Q];
  #pragma unroll
          for (int s = 0; s < 4; ++s) {
            apply_chol<M, Real>(Ld, z + s * MP, eps[s]);
  #pragma unroll
            for (int i = 0; i < Q; ++i) sj[s][i] = Real(0);
            if constexpr (J) {  // staged marks (zero where no event, and past T)
              if (JM == 0) {
  #pragma unroll
                for (int j = 0; j < M; ++j) eps[s][j] = radd<Real>(eps[s][j], wl[j * 32]);  // noise.py:156-157
              } else {
  #pragma unroll
                for (int i = 0; i < Q; ++i) sj[s][i] = wl[i * 32];
              }
              wl += Q * 32;
            }
          }
          if (g >= kWsBuf) named_sync(1 + kWsBuf + slot, nb);  // slot drained by the consumers
          Real* rs = ring + (size_t)slot * GW * C + c;
  #pragma unroll
          for (int s = 0; s < 4; ++s) {
  #pragma unroll
            for (int j = 0; j < M; ++j) rs[(s * M + j) * C] = eps[s][j];
            if (JM == 1) {
  #pragma unroll
              for (int i = 0; i < Q; ++i) rs[(4 * M + s * Q + i) * C] = sj[s][i];
            }
          }
          named_arrive(1 + slot, nb);  // slot full
        }
      };
      if (jumps)
        produce(std::true_type{});
      else
        produce(std::false_type{});
    } else {
      SysParams<Real> sp = a.sp;
#pragma unroll
      for (int i = 0; i < 10; ++i) pin(sp.mp[i]);
#pragma unroll
      for (int i = 0; i < N; ++i) {
        pin(sp.sw[i]);
        pin(sp.swt[i]);
      }
#pragma unroll
      for (int i = 0; i < 3; ++i) pin(sp.tk[i]);
      Real dt = a.dt, sdt = a.sdt, cq = a.cq;
      pin(dt);
      pin(sdt);
      pin(cq);
      Real x[N];
#pragma unroll
      for (int i = 0; i < N; ++i) x[i] = Real(x0[i]);
      Real S = Real(0);
      // the consumers' horizon, unswitched on the general-channel flag (a uniform run-time branch
      // inside the step would split the 4-step group's basic block)
      auto consume = [&](auto gtag) {
        constexpr bool GEN = decltype(gtag)::value;
        auto step = [&](const int t, const Real* eps, const Real* sj) {
          const auto ax = Dyn::template aux<Real, true>(x, sp);
          const Real qv = Cost::template q<Dyn, Real>(x, ax, sp);
          const Real* st = tab + t * TS;
          Real inc = fma(qv, dt, st[M]);
          const Real quad = noise_quad<M, Real, GEN>(a, eps);
  #pragma unroll
          for (int j = 0; j < M; ++j) inc = fma(st[M + 1 + j], eps[j], inc);
          S += fma(cq, quad, inc);  // costs.py:98-111 times dt
          Real v[M];
  #pragma unroll
          for (int j = 0; j < M; ++j) v[j] = fma(eps[j], sdt, st[j]);
          Dyn::template advance<Real>(x, ax, v, dt, sp);  // dynamics.py:130-135
          if (JM == 1) {
  #pragma unroll
            for (int i = 0; i < Q; ++i) x[Dyn::jump_row(i)] = radd<Real>(x[Dyn::jump_row(i)], sj[i]);  // x + H (ind * mark)
          }
        };
        for (int g = 0; g < G; ++g) {
          const int slot = g % kWsBuf;
          named_sync(1 + slot, nb);
          const Real* rs = ring + (size_t)slot * GW * C + c;
          Real e[4 * M], jv[(JM == 1) ? 4 * Q : 1];
  #pragma unroll
          for (int i = 0; i < 4 * M; ++i) e[i] = rs[i * C];
          if (JM == 1) {
  #pragma unroll
            for (int i = 0; i < 4 * Q; ++i) jv[i] = rs[(4 * M + i) * C];
          }
          if (g < G - kWsBuf) named_arrive(1 + kWsBuf + slot, nb);
          const int t0 = 4 * g;
          if (t0 + 4 <= T) {
  #pragma unroll
            for (int s = 0; s < 4; ++s) step(t0 + s, e + s * M, jv + (JM == 1 ? s * Q : 0));
          } else {
  #pragma unroll
            for (int s = 0; s < 4; ++s)
              if (t0 + s < T) step(t0 + s, e + s * M, jv + (JM == 1 ? s * Q : 0));
          }
        }
      };
      if (a.general)
        consume(std::true_type{});
      else
        consume(std::false_type{});
      bool fin = true;
#pragma unroll
      for (int i = 0; i < N; ++i) fin = fin && isfinite(x[i]);
      if (fin) {
        const auto ax = Dyn::template aux<Real, true>(x, sp);
        S += sp.term_scale * Cost::template q<Dyn, Real>(x, ax, sp);  // controller.py:155
      } else {
        S = r_inf<Real>();
      }
      if (act && costs_out) costs_out[kl] = double(S);
      Sf = act ? S : r_inf<Real>();
    }
    const int col = (producer || !act) ? -1 : c;
    {
      const StreamKey sk = make_stream_key(a.seeds[blockIdx.y], iter);
      const GapSampler gs{Sg, T, a.gap_inv};
      const bool jumps = a.jump_on && (L == nullptr || L->sampler_jumps);
      Real Ld[M * M], Lj[Q * Q], mu[Q];
#pragma unroll
      for (int i = 0; i < M * M; ++i) Ld[i] = a.Ld[i];
#pragma unroll
      for (int i = 0; i < Q * Q; ++i) Lj[i] = a.Lj[i];
#pragma unroll
      for (int i = 0; i < Q; ++i) mu[i] = a.mu_j[i];
      sparse_epilogue<1, Real>(&Sf, &col, TM, a.inv_lam, Nacc, sm, nitems, false, [&](int cc, int b, Real* out) {
        regen_philox<M, MP, Q, QP, JM, Real>(a, sk, gs, (uint32_t)(a.sample_offset + base + cc), b, Ld, Lj, mu, jumps,
                                             out);
      });
    }
  }
  __syncthreads();
  write_record(a, s_acc, Nacc);
}


// ---------------------------------------------------------------- shared memory plan (fast kernel)
//   Nacc (TM doubles) | mark staging (fast_marks_bytes) | step table (T x (2m+1) Real) |
//   sig_col (tile int) | sig_w (tile double) | scratch (chunk x TM Real) | gap table (uint32)
struct FastPlan {
  size_t nacc, marks, tab, sigc, sigw, scr, gap, total;
  int chunk;
};
__host__ __device__ __forceinline__ FastPlan fast_plan(int TM, int tabn, int tile, int nthreads, int nb, size_t mbytes,
                                                       int ngap, int rs) {
  FastPlan p;
  p.chunk = nthreads / nb > 1 ? nthreads / nb : 1;
  if (p.chunk > tile) p.chunk = tile;
  size_t o = 0;
  p.nacc = o;
  o = al16(o + sizeof(double) * (size_t)TM);
  p.marks = o;
  o = al16(o + mbytes);
  p.tab = o;
  o = al16(o + (size_t)rs * tabn);
  p.sigc = o;
  o = al16(o + sizeof(int) * (size_t)tile);
  p.sigw = o;
  o = al16(o + sizeof(double) * (size_t)tile);
  p.scr = o;
  o = al16(o + (size_t)rs * p.chunk * TM);
  p.gap = o;
  o = al16(o + sizeof(uint32_t) * (size_t)ngap);
  p.total = o;
  return p;
}


// ---------------------------------------------------------------- the kernel
// QUAD = false: the c = 1 Philox case, the eps'eps term dropped (fma(0, quad,
// inc) = inc exactly for finite noise); true: the term formed, eps' eps or, for
// the general channel (costs.py:118-121, a rare plugin: a uniform branch),
// eps' bb eps.  Separate kernels, so each carries one copy of the tile loop.
// LDIAG: the diffusion Cholesky factor is diagonal (independent input channels, every BASELINE
// config): eps_j = L_jj z_j, m multiplies instead of m (m + 1) / 2 multiply-adds -- the same
// value as the dense product, whose off-diagonal terms add exact zeros.
template <class Sys, typename Real, bool PHILOX, int JM, int SPT, int MAXT, bool QUAD, bool LDIAG = false>
__global__ void __launch_bounds__(MAXT, (SPT == 2 ? 2 : 1)) rollout_fast(const RolloutArgs<Real> a) {
  using Dyn = typename Sys::Dyn;
  using Cost = typename Sys::Cost;
  using V = typename VecOf<SPT, Real>::type;
  static_assert(SPT == 1 || std::is_same<Real, float>::value, "two samples per thread: fp32 only");
  constexpr int N = Sys::N, M = Sys::M;
  constexpr int MP = Pad<M>::value;
  constexpr int Q = (JM == 0) ? M : Dyn::QJ;
  constexpr int QP = Pad<Q>::value;
  constexpr int TS = 2 * M + 1;
  // steps per noise group: one Philox block (4 normals); HBM mode: 4 steps of
  // the small systems, one quadrotor step (its loads are 7 words a step)
  constexpr int GS = PHILOX ? 4 / MP : (M >= 3 ? 1 : 4);

  extern __shared__ double smem_d[];
  __shared__ double s_red[4][32];
  __shared__ double s_acc[4];
  __shared__ int s_cnt[32];

  const int TM = a.TM, T = a.T, K = a.K;
  const int nthreads = blockDim.x, nwarps = nthreads >> 5;
  const int tileK = SPT * nthreads;
  const int nb = regen_items(T, GS);
  constexpr bool IDX = PHILOX && marks_indexed(Q);  // indexed mark staging (q >= 2)
  static_assert(!IDX || GS * 32 < kMarkCap, "one group of steps must fit the mark table");
  // (the plan depends on kernel parameters only: nothing is read from memory before the
  // prefetches below are in flight)
  const bool stage = PHILOX && a.jump_on;
  const FastPlan pl = fast_plan(TM, T * TS, tileK, nthreads, nb,
                                stage ? fast_marks_bytes(tileK, nwarps, a.jw_len, Q, (int)sizeof(Real)) : 0, a.gap_n,
                                (int)sizeof(Real));
  char* const sb = reinterpret_cast<char*>(smem_d);
  double* Nacc = reinterpret_cast<double*>(sb + pl.nacc);
  Real* tab = reinterpret_cast<Real*>(sb + pl.tab);
  uint32_t* Sg = reinterpret_cast<uint32_t*>(sb + pl.gap);
  Real* const marks = reinterpret_cast<Real*>(sb + pl.marks);
  SparseSmem sm{s_red, s_acc, s_cnt, reinterpret_cast<int*>(sb + pl.sigc), reinterpret_cast<float*>(sb + pl.sigw),
                reinterpret_cast<double*>(sb + pl.sigw), sb + pl.scr, pl.chunk};

  const uint64_t t_entry = globaltimer();
  if (a.loop != nullptr) {
    // closed loop: pull the lines the prologue reads one after another (LoopState, then the
    // nominal sequence of the parity LoopState::step selects -- both parities sit at
    // u_nom + trial * 2 TM) into L2 side by side, so a cold start pays one DRAM round trip
    // instead of two dependent ones (an L2 prefetch of lines the previous step's finalize is
    // still writing is harmless: L2 is the point of coherence)
    const char* lp = reinterpret_cast<const char*>(a.loop + blockIdx.y);
    const char* up = reinterpret_cast<const char*>(a.u_nom + (size_t)blockIdx.y * 2 * TM);
    const int nl = (2 * TM * (int)sizeof(double) + 127) / 128;
    const int i = (int)threadIdx.x;
    if (i < 2)
      asm volatile("prefetch.global.L2 [%0];" ::"l"(lp + 128 * i));
    else if (i - 2 < nl)
      asm volatile("prefetch.global.L2 [%0];" ::"l"(up + 128 * (i - 2)));
  }
  // indexed staging: bytes [warp][step][lane][half], then the warps' mark tables
  uint8_t* const ibw = reinterpret_cast<uint8_t*>(marks) + (size_t)(threadIdx.x >> 5) * 32 * a.jw_len;
  Real* const tabw =
      reinterpret_cast<Real*>(reinterpret_cast<char*>(marks) + (((size_t)nthreads * a.jw_len + 15) & ~(size_t)15)) +
      (size_t)(threadIdx.x >> 5) * kMarkCap * Q * SPT;
  if (stage) {  // the mark staging is zero outside event entries (jump_window_c / jump_window_idx); zeroed
                // before the grid wait: shared memory is ours, and the stores overlap the prefetches'
                // (and, in the closed loop, the previous finalize's) latency
    const size_t zb = IDX ? (size_t)nthreads * a.jw_len : (size_t)SPT * nwarps * 32 * a.jw_len * Q * sizeof(Real);
    const int n4 = (int)((zb + 15) / 16);
    float4* z4 = reinterpret_cast<float4*>(marks);
    for (int i = threadIdx.x; i < n4; i += nthreads) z4[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (IDX && (threadIdx.x & 31) < Q * SPT) tabw[threadIdx.x & 31] = Real(0);  // entry 0: no event
  }
  grid_dep_wait();    // u_nom / x / iteration come from the previous control step
  grid_dep_launch();  // let the finalize grid get resident while the horizon runs
  LoopState* L = a.loop ? a.loop + blockIdx.y : nullptr;
  if (L != nullptr && L->halted) return;
  // (batched old/new variants: the "old" trials' sampler draws no jumps)
  const bool jumps = stage && (L == nullptr || L->sampler_jumps);
  const uint64_t iter = L ? L->iteration : (a.iteration_dev ? *a.iteration_dev : a.iteration);
  const double* x0 = L ? L->x : a.x0;
  // timeline row (tuning: JM_TIMELINE), read by each CTA's stamping thread only
  unsigned long long* const tlr = (threadIdx.x == 0) ? tl_row(L, L ? L->step : 0) : nullptr;
  if (L != nullptr && blockIdx.x == 0 && threadIdx.x == 0) {
    L->t_start[L->step] = globaltimer();
    tl_put(tlr, kTlRollEntry, t_entry);
    tl_put(tlr, kTlRollWait);
  }
  rollout_prologue<M, Real>(a, L ? loop_unom(L, L->step, TM) : a.u_nom + (size_t)blockIdx.y * TM, tab, Nacc, s_acc, Sg);
  __syncthreads();

  using S = Real;  // parameter type (scalar_t<V>)
  SysParams<S> sp = a.sp;
#pragma unroll
  for (int i = 0; i < 10; ++i) pin(sp.mp[i]);
#pragma unroll
  for (int i = 0; i < N; ++i) {
    pin(sp.sw[i]);
    pin(sp.swt[i]);
  }
  S Ld[M * M], Lj[Q * Q], mu[Q];
#pragma unroll
  for (int i = 0; i < M * M; ++i) {
    Ld[i] = a.Ld[i];
    pin(Ld[i]);
  }
#pragma unroll
  for (int i = 0; i < Q * Q; ++i) Lj[i] = a.Lj[i];
#pragma unroll
  for (int i = 0; i < Q; ++i) mu[i] = a.mu_j[i];
  S dt = a.dt, sdt = a.sdt, cq = a.cq;
  const S jscale = a.jscale;
  pin(dt);
  pin(sdt);
  pin(cq);
  const GapSampler gs{Sg, T, a.gap_inv};
  const int JW = a.jw_len;
  const StreamKey sk = make_stream_key(a.seeds[blockIdx.y], iter);
  double* const costs_out = gridDim.y > 1 ? nullptr : (a.costs_dev ? *a.costs_dev : a.costs);
  const int lane = threadIdx.x & 31;
  if (blockIdx.x == 0) tl_put(tlr, kTlRollHorizon);
  Real* wdu[SPT];
#pragma unroll
  for (int u = 0; u < SPT; ++u) wdu[u] = marks + (size_t)(threadIdx.x >> 5) * SPT * 32 * JW * Q + u;
  Mask128 prev[SPT];
#pragma unroll
  for (int u = 0; u < SPT; ++u) prev[u] = Mask128{0ull, 0ull};

  {
    for (int tile = blockIdx.x; tile < a.ntiles; tile += gridDim.x) {
      const int base = tile * tileK;
      int col[SPT], kl[SPT];
      bool act[SPT];
      uint32_t kg[SPT];
#pragma unroll
      for (int u = 0; u < SPT; ++u) {
        col[u] = SPT * (int)threadIdx.x + u;
        kl[u] = base + col[u];
        act[u] = kl[u] < K;
        kg[u] = (uint32_t)(a.sample_offset + kl[u]);
      }
      V x[N];
#pragma unroll
      for (int i = 0; i < N; ++i) x[i] = vcast<V>(x0[i]);
      V Sacc = vcast<V>(0.0);
      JumpClock clk[SPT];
      const Real* wl[SPT];
      const uint8_t* il = ibw + lane;
      int wnext = 0;
#pragma unroll
      for (int u = 0; u < SPT; ++u) {
        wl[u] = wdu[u] + lane * SPT;
        if (jumps) clock_start(clk[u], sk, kg[u], gs);
      }

      // one horizon step t with its eps_combined and state-jump increment
      // (gen: the general-channel form eps' bb eps, a compile-time tag -- a uniform run-time branch
      // here would split every step's basic block)
      auto step = [&](auto gen, const int t, const V* eps, const V* sj, const bool has_sj) {
        const auto ax = Dyn::template aux<V, true>(x, sp);
        const V qv = Cost::template q<Dyn, V>(x, ax, sp);
        const Real* st = tab + t * TS;
        V inc = fma(qv, dt, st[M]);
#pragma unroll
        for (int j = 0; j < M; ++j) inc = fma(st[M + 1 + j], eps[j], inc);
        if constexpr (!QUAD) {
          Sacc += inc;
        } else {
          V quad = eps[0] * eps[0];
#pragma unroll
          for (int j = 1; j < M; ++j) quad = fma(eps[j], eps[j], quad);
          if constexpr (decltype(gen)::value) {  // eps' bb eps (costs.py:118-121)
            quad = vcast<V>(0.0);
#pragma unroll
            for (int i = 0; i < M; ++i) {
              V tq = vcast<V>(0.0);
#pragma unroll
              for (int j = 0; j < M; ++j) tq = fma(a.bb[i * M + j], eps[j], tq);
              quad = fma(eps[i], tq, quad);
            }
          }
          Sacc += fma(cq, quad, inc);
        }
        V v[M];
#pragma unroll
        for (int j = 0; j < M; ++j) v[j] = fma(eps[j], sdt, st[j]);
        Dyn::template advance<V>(x, ax, v, dt, sp);
        if (JM == 1 && has_sj) {
#pragma unroll
          for (int i = 0; i < Q; ++i) x[Dyn::jump_row(i)] = vadd(x[Dyn::jump_row(i)], sj[i]);
        }
      };

      if constexpr (PHILOX) {
        // the horizon, unswitched on the sampler's jumps (a uniform run-time flag): each form is
        // straight-line per noise group, so the next group's Philox block overlaps the dynamics
        auto horizon = [&](auto jtag, auto gtag) {
          constexpr bool J = decltype(jtag)::value;
          V z[4], zn[4];
          block_normals_v(sk, 0u, kg, z);
          auto noisy = [&](const int t, const int s2, const V* zz) {
            V eps[M], sj[Q];
            bool has_sj = false;
            if constexpr (LDIAG) {
  #pragma unroll
              for (int j = 0; j < M; ++j) eps[j] = Ld[j * M + j] * zz[s2 * MP + j];
            } else {
              chol_v<M>(Ld, zz + s2 * MP, eps);
            }
            if constexpr (J) {
              V mv[Q];  // the staged marks of both halves: one load (interleaved pairs)
              if constexpr (IDX) {
                // the step's table entry (0: none) of this thread, then its samples' marks
              const uint32_t ii = *il;
              il += 32;
#pragma unroll
              for (int i = 0; i < Q; ++i) {
                if constexpr (SPT == 2)
                  mv[i] = F2(*reinterpret_cast<const float2*>(tabw + (ii * Q + i) * 2));
                else
                  mv[i] = tabw[ii * Q + i];
              }
              } else {
  #pragma unroll
                for (int i = 0; i < Q; ++i) {
                  if constexpr (SPT == 2)
                    mv[i] = F2(*reinterpret_cast<const float2*>(wl[0] + i * 32 * SPT));
                  else
                    mv[i] = wl[0][i * 32];
                }
                wl[0] += Q * 32 * SPT;
              }
              if (JM == 0) {
  #pragma unroll
                for (int j = 0; j < M; ++j) eps[j] = vadd_exact(eps[j], mv[j]);  // noise.py:156-157
              } else {
  #pragma unroll
                for (int i = 0; i < Q; ++i) sj[i] = mv[i];
                has_sj = true;
              }
            }
            step(gtag, t, eps, sj, has_sj);
          };
          // outer loop: one jump window (the whole horizon without jumps); inner loop: its noise
          // groups, nothing but the groups -- the window code stays out of the hot loop's live ranges
          for (int w0 = 0; w0 < T;) {
            int wend = T;
            if constexpr (J) {
              if constexpr (IDX) {
                wend = jump_window_idx<Q, QP, JM, SPT, Real>(clk, prev[0], w0, min(w0 + JW, T), GS, sk, kg[0], gs, Lj, mu,
                                                             jscale, ibw, tabw, a.poisson != 0, a.cnt);
                il = ibw + lane;
              } else {
                wend = min(w0 + JW, T);
#pragma unroll
                for (int u = 0; u < SPT; ++u) {
                  jump_window_c<Q, QP, JM, SPT, Real>(clk[u], prev[u], w0, wend, sk, kg[u], SPT, gs, Lj, mu, jscale,
                                                      wdu[u], a.poisson != 0, a.cnt);
                  wl[u] = wdu[u] + lane * SPT;
                }
              }
            }
            // (windows start on group boundaries: the group index form lets the compiler see
            // t0 = GS g, so the step table's rows of a group are read with vector loads)
            int g = w0 / GS;
            // two groups per trip, the normal buffers z / zn swapping roles (no register copies;
            // the BASELINE systems in fp32 -- elsewhere the longer body only adds register pressure)
            if constexpr (std::is_same<Real, float>::value && Dyn::kPairGroups) {
              for (; (g + 2) * GS <= wend; g += 2) {
                const int t0 = g * GS;
                block_normals_v(sk, (uint32_t)(g + 1), kg, zn);
#pragma unroll
                for (int s2 = 0; s2 < GS; ++s2) noisy(t0 + s2, s2, z);
                block_normals_v(sk, (uint32_t)(g + 2), kg, z);  // (one spare block at the horizon's end)
#pragma unroll
                for (int s2 = 0; s2 < GS; ++s2) noisy(t0 + GS + s2, s2, zn);
              }
            }
            for (; (g + 1) * GS <= wend; ++g) {  // (the window's odd group; every group of the other systems)
              const int t0 = g * GS;
              block_normals_v(sk, (uint32_t)(g + 1), kg, zn);
#pragma unroll
              for (int s2 = 0; s2 < GS; ++s2) noisy(t0 + s2, s2, z);
#pragma unroll
              for (int i = 0; i < 4; ++i) z[i] = zn[i];
            }
            const int t0 = g * GS;
            if (t0 < wend) {  // (the horizon's last, partial group: wend == T)
#pragma unroll
              for (int s2 = 0; s2 < GS; ++s2)
                if (t0 + s2 < T) noisy(t0 + s2, s2, z);
            }
            w0 = wend;
          }
        };
        // (the general-channel form exists only in the QUAD kernels)
        const bool gen = QUAD && a.general;
        if (jumps) {
          if (gen) {
            if constexpr (QUAD) horizon(std::true_type{}, std::true_type{});
          } else {
            horizon(std::true_type{}, std::false_type{});
          }
        } else {
          if (gen) {
            if constexpr (QUAD) horizon(std::false_type{}, std::true_type{});
          } else {
            horizon(std::false_type{}, std::false_type{});
          }
        }
      } else {
        // HBM wire format eps[(t*M + j)*K + k], jump[(t*Q + i)*K + k]: a thread's
        // SPT samples are adjacent columns (one 8-byte load for both), groups
        // of GS steps loaded two groups ahead
        constexpr int EW = GS * M * SPT, JWD = (JM == 1) ? GS * Q * SPT : 1;
        const bool hj = JM == 1 && a.jump_in != nullptr;
        const int kc = act[0] ? kl[0] : 0;
        const Real* pe = a.eps_in + kc;
        const Real* pj = hj ? a.jump_in + kc : nullptr;
        const size_t rowe = (size_t)M * K, rowj = (size_t)Q * K;
        auto load = [&](const Real* p) -> V {
          if constexpr (SPT == 2) {
            const float2 v2 = __ldg(reinterpret_cast<const float2*>(p));
            return F2(v2);
          } else {
            return V(__ldg(p));
          }
        };
        // the horizon, unswitched on whether a jump tensor was fed (a uniform run-time flag)
        auto horizon = [&](auto jtag, auto gtag) {
          constexpr bool HJ = decltype(jtag)::value;
          auto load_group = [&](int g0, V* ze, V* zj) {
  #pragma unroll
            for (int s2 = 0; s2 < GS; ++s2) {
              const int t = min(g0 + s2, T - 1);
  #pragma unroll
              for (int j = 0; j < M; ++j) ze[s2 * M + j] = load(pe + (size_t)t * rowe + (size_t)j * K);
              if (JM == 1) {
  #pragma unroll
                for (int i = 0; i < Q; ++i) zj[s2 * Q + i] = HJ ? load(pj + (size_t)t * rowj + (size_t)i * K) : vcast<V>(0.0);
              }
            }
          };
          constexpr int GE = GS * M, GJ = (JM == 1) ? GS * Q : 1;
          (void)EW;
          (void)JWD;
          // a ring of kHbmDepth + 1 register buffers, the group loop unrolled over the ring so
          // a buffer's role is a compile-time index (no register rotation moves): group g runs
          // from buffer g % NB while group g + kHbmDepth is loaded into the buffer group g - 1
          // has just released
          // (fp64, the strict-parity precision: one group ahead -- its buffers are twice the registers)
          constexpr int DEPTH = sizeof(Real) == 8 ? 1 : kHbmDepth;
          constexpr int NB = DEPTH + 1;
          V eb[NB][GE], jb[NB][GJ];
  #pragma unroll
          for (int d = 0; d < DEPTH; ++d) load_group(d * GS, eb[d], jb[d]);
          for (int t0 = 0; t0 < T; t0 += NB * GS) {
  #pragma unroll
            for (int r = 0; r < NB; ++r) {
              const int tg = t0 + r * GS;
              if (tg < T) {
                load_group(tg + DEPTH * GS, eb[(r + DEPTH) % NB], jb[(r + DEPTH) % NB]);  // (clamped inside the horizon)
  #pragma unroll
                for (int s2 = 0; s2 < GS; ++s2) {
                  if (GS == 1 || tg + s2 < T) {
                    V sj[Q];
                    if (JM == 1) {
  #pragma unroll
                      for (int i = 0; i < Q; ++i) sj[i] = vmul_exact(jscale, jb[r][s2 * Q + i]);  // (a bare packed product could fuse into the add)
                    }
                    step(gtag, tg + s2, eb[r] + s2 * M, sj, JM == 1 && HJ);
                  }
                }
              }
            }
          }
        };
        const bool gen = QUAD && a.general;
        if (hj) {
          if (gen) {
            if constexpr (QUAD) horizon(std::true_type{}, std::true_type{});
          } else {
            horizon(std::true_type{}, std::false_type{});
          }
        } else {
          if (gen) {
            if constexpr (QUAD) horizon(std::false_type{}, std::true_type{});
          } else {
            horizon(std::false_type{}, std::false_type{});
          }
        }
      }
      if (tlr != nullptr) {  // (timeline: the first and the last CTA to finish the horizon)
        tl_max(tlr, kTlRollHorizonEndMax);
        atomicMax(tlr + kTlRollHorizonEndMin, ~(unsigned long long)globaltimer());
      }
      // Once non-finite, an Euler state x += dx stays non-finite, so the final
      // state decides divergence (the reference checks every step).
      Real Sf[SPT];
      int cols[SPT];
      {
        const auto ax = Dyn::template aux<V, true>(x, sp);
        const V term = Cost::template q<Dyn, V>(x, ax, sp);
#pragma unroll
        for (int u = 0; u < SPT; ++u) {
          bool fin = true;
#pragma unroll
          for (int i = 0; i < N; ++i) fin = fin && isfinite(half_of(x[i], u));
          const Real Su = fin ? fma(sp.term_scale, Real(half_of(term, u)), Real(half_of(Sacc, u)))  // controller.py:155
                              : r_inf<Real>();
          if (act[u] && costs_out) costs_out[kl[u]] = double(Su);
          Sf[u] = act[u] ? Su : r_inf<Real>();
          cols[u] = act[u] ? col[u] : -1;
        }
      }
      // ---- per-CTA online softmax over this tile (K3/K4 partials), sparse N
      if constexpr (PHILOX) {
        sparse_epilogue<SPT, Real>(Sf, cols, TM, a.inv_lam, Nacc, sm, nb, false, [&](int c, int b, Real* out) {
          regen_philox<M, MP, Q, QP, JM, Real>(a, sk, gs, (uint32_t)(a.sample_offset + base + c), b, Ld, Lj, mu, jumps,
                                               out);
        });
      } else {
        sparse_epilogue<SPT, Real>(Sf, cols, TM, a.inv_lam, Nacc, sm, nb, true, [&](int c, int b, Real* out) {
          const int k = base + c;
#pragma unroll
          for (int s2 = 0; s2 < GS; ++s2) {
            const int t = b * GS + s2;
            if (t < T) {
#pragma unroll
              for (int j = 0; j < M; ++j) out[t * M + j] = a.eps_in[(size_t)(t * M + j) * K + k];
            }
          }
        });
      }
    }
  }
  __syncthreads();
  write_record(a, s_acc, Nacc);
  tl_max(tlr, kTlRollEndMax);
}

}  // namespace jm
