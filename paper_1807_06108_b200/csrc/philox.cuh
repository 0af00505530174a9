// philox.cuh -- counter-based noise for the sampled-trajectory core.
//
// Replaces the reference's numpy Philox4x64 + ziggurat draws
// (jump_mppi/noise.py:38-51 RngStream, :129-161 sample_noise_batch).  Bit
// parity with numpy is not a goal (RNG values are never pinned by
// the reference tests); what is kept is the *contract*:
//   * a stream is keyed on (master_seed, stream_id = iteration index), so the
//     noise of an iteration does not depend on scheduling, block size or GPU
//     count (the sample index in the counter is GLOBAL);
//   * Gaussian draws use counter slots independent of the jump draws, so
//     jump_sampling_enabled=False and nu=0 give bit-identical eps_d
//     (noise.py:114-115, tests/test_noise.py:149-154, acceptance P2);
//   * zero-one jump law per (sample, step) with probability nu*dt
//     (noise.py:151), realised as the equivalent renewal process: the gaps
//     between jump steps are geometric, so one uniform is drawn per EVENT
//     instead of per step (nu*dt ~ 0.01 in every BASELINE config); marks are
//     drawn only for events (noise.py:152-155).
//
// Counter layout (Philox4x32-10, Salmon et al. SC'11):
//   key  = (seed lo32, seed hi32)
//   ctr  = (block, sample, iteration lo32, slot<<24 | iteration hi32 & 0xffffff)
//   slot 0: diffusion normals, normal index i = t*MP + j, block = i>>2, lane = i&3
//   slot 1: jump gaps, event e: word e&3 of block e>>2, u = word>>8 (24 bits);
//           gap G_e = max{g in [0,T] : u < S[g]} with the integer survival
//           table S[0] = 2^24, S[g] = floor(S[g-1] * (2^24 - q) / 2^24),
//           q = ceil(nu dt 2^24) (so P(G >= g) = S[g]/2^24 = (1-p)^g up to
//           2^-24 roundings); event steps t_0 = G_0, t_e = t_{e-1} + 1 + G_e
//   slot 2: marks of event e, normal index e*QP + i (QP = q, 3 padded to 4),
//           block = index>>2, lane = index&3
//   slot 3: closed-loop plant, block = 3*step + {0 diffusion, 1 uniform, 2 marks}
//   slot 4: Poisson arrival counts (jump_process = poisson), event e: word e&3
//           of block e>>2, u = word>>8; n = 1 + #{k in 1..8 : u < C[k]} with
//           C[k] = floor(2^24 P(N > k | N >= 1)), N ~ Poisson(nu dt) (the
//           event steps themselves come from slot 1 with p = 1 - exp(-nu dt))
// Normals: Box-Muller on pairs of words with 23-bit mantissa uniforms.
// The CPU emulation of this exact mapping is oracle/philox_stream.py.
#pragma once
#include <cmath>
#include <cstdint>

namespace jm {

struct P4 {
  uint32_t x, y, z, w;
};

enum : uint32_t { kSlotDiffusion = 0, kSlotJumpUniform = 1, kSlotMark = 2, kSlotPlant = 3, kSlotCount = 4 };

__host__ __device__ __forceinline__ P4 philox4x32_10(P4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
#ifdef __CUDA_ARCH__
    const uint32_t lo0 = 0xD2511F53u * c.x, hi0 = __umulhi(0xD2511F53u, c.x);
    const uint32_t lo1 = 0xCD9E8D57u * c.z, hi1 = __umulhi(0xCD9E8D57u, c.z);
#else
    const uint64_t p0 = (uint64_t)0xD2511F53u * c.x, p1 = (uint64_t)0xCD9E8D57u * c.z;
    const uint32_t lo0 = (uint32_t)p0, hi0 = (uint32_t)(p0 >> 32);
    const uint32_t lo1 = (uint32_t)p1, hi1 = (uint32_t)(p1 >> 32);
#endif
    c = P4{hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0};
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  return c;
}

// Per-launch stream key: (seed, iteration) -> key words + the two upper
// counter words (slot is or-ed in by draw()).
struct StreamKey {
  uint32_t k0, k1, c2, c3;
};

__host__ __device__ __forceinline__ StreamKey make_stream_key(uint64_t seed, uint64_t iteration) {
  StreamKey s;
  s.k0 = (uint32_t)seed;
  s.k1 = (uint32_t)(seed >> 32);
  s.c2 = (uint32_t)iteration;
  s.c3 = (uint32_t)(iteration >> 32) & 0xFFFFFFu;
  return s;
}

__host__ __device__ __forceinline__ P4 draw(const StreamKey& s, uint32_t slot, uint32_t block,
                                            uint32_t sample) {
  return philox4x32_10(P4{block, sample, s.c2, s.c3 | (slot << 24)}, s.k0, s.k1);
}

// Jump clock of one sample: step and index of its next jump event.
struct JumpClock {
  int tj;      // step of the next event (>= T: none left in the horizon)
  uint32_t e;  // index of that event
  P4 w;        // gap words of block e >> 2
};

__host__ __device__ __forceinline__ uint32_t p4_word(const P4& w, uint32_t i) {
  return i == 0 ? w.x : (i == 1 ? w.y : (i == 2 ? w.z : w.w));
}

// Geometric gap G = max{g in [0, T] : u < S[g]} over the survival table
// S[0..T].  A float estimate log2(u / 2^24) / log2(1 - p) lands on G or next
// to it; the integer comparisons against S make the result exact (and
// identical to the oracle's count), whatever the estimate's rounding.
struct GapSampler {
  const uint32_t* S;  // survival table, T + 1 entries
  int T;
  float inv_l2keep;   // 1 / log2(1 - p) (< 0; -0 when p = 1)
};

__host__ __device__ __forceinline__ int jump_gap(const GapSampler& gs, uint32_t u24) {
#ifdef __CUDA_ARCH__
  float l;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(l) : "f"((float)u24 + 0.5f));
  int g = __float2int_rz((l - 24.0f) * gs.inv_l2keep);  // saturating
#else
  int g = (int)std::fmin((std::log2((double)u24 + 0.5) - 24.0) * gs.inv_l2keep, (double)gs.T);
#endif
  g = g < 0 ? 0 : (g > gs.T ? gs.T : g);
  while (g > 0 && u24 >= gs.S[g]) --g;
  while (g < gs.T && u24 < gs.S[g + 1]) ++g;
  return g;
}

__host__ __device__ __forceinline__ void clock_start(JumpClock& c, const StreamKey& sk, uint32_t kg,
                                                     const GapSampler& gs) {
  c.e = 0;
  c.w = draw(sk, kSlotJumpUniform, 0u, kg);
  c.tj = jump_gap(gs, c.w.x >> 8);
}

__host__ __device__ __forceinline__ void clock_next(JumpClock& c, const StreamKey& sk, uint32_t kg,
                                                    const GapSampler& gs) {
  c.e += 1;
  if ((c.e & 3u) == 0u) c.w = draw(sk, kSlotJumpUniform, c.e >> 2, kg);
  c.tj += 1 + jump_gap(gs, p4_word(c.w, c.e & 3u) >> 8);
}

// Compound-Poisson arrivals per jump step (BASELINE "Poisson jump counts per
// step"): thresholds of the zero-truncated count distribution, zero-padded;
// all zero = Bernoulli (one arrival per event, the reference's zero-one law).
constexpr int kMaxCount = 8;
struct CountTable {
  uint32_t c[kMaxCount];  // c[k-1] = floor(2^24 P(N > k | N >= 1)), k = 1..8
};

__host__ __device__ __forceinline__ int event_count(const StreamKey& sk, uint32_t kg, uint32_t e,
                                                    const CountTable& ct) {
  const uint32_t u = p4_word(draw(sk, kSlotCount, e >> 2, kg), e & 3u) >> 8;
  int n = 1;
#pragma unroll
  for (int k = 0; k < kMaxCount; ++k) n += u < ct.c[k] ? 1 : 0;
  return n;
}

#ifdef __CUDACC__
// Box-Muller on two words.  u1 in (0,1], angle uniform in [-pi, pi).
// Resolution: both uniforms keep the top 23 bits of their word, so u1 >= 2^-23
// and |z| <= sqrt(-2 ln 2^-23) = 5.65: the normal's tails beyond 5.65 sigma
// (two-sided mass 1.6e-8, about one draw in 6e7; ~100 of the 6.6e9 draws of a
// cfg1 iteration would have landed there) are folded onto the 2^23-point grid
// below it, and the angle takes 2^23 values.  The reference's ziggurat has no
// such cut; the moment / frequency tests (tests/test_gpu_api.py, G-stat in
// tests/test_gpu_f32_gate.py) bound the effect on the control statistics.
// MUFU lg2/sqrt/sin/cos: noise quality only needs ~1e-6 relative accuracy;
// the fp64 kernels consume the very same float normals (cast), so both
// precisions see identical noise for a given (seed, iteration).
__device__ __forceinline__ void box_muller(uint32_t a, uint32_t b, float& z0, float& z1) {
  const float u1 = 2.0f - __uint_as_float(0x3F800000u | (a >> 9));        // (0, 1]
  const float ang = __fmaf_rn(__uint_as_float(0x3F800000u | (b >> 9)),     // [1,2) -> [-pi,pi)
                              6.2831853071795865f, -9.4247779607693797f);
  // u1 >= 2^-23 and -2 ln u1 is 0 or >= ~2e-7: no subnormal operands, so the
  // .ftz forms are exact equivalents without the subnormal fix-up instructions
  float l2, r;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(l2) : "f"(u1));
  const float rr = __fmul_rn(-1.3862943611198906f, l2);  // -2 ln u1
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(rr));
  float sn, cs;
  __sincosf(ang, &sn, &cs);
  z0 = __fmul_rn(r, cs);
  z1 = __fmul_rn(r, sn);
}

// Mark normals of event e (QP of them, QP in {1, 2, 4}: never straddles a
// Philox block); only the Box-Muller pair(s) holding them are evaluated.
template <int QP>
__device__ __forceinline__ void event_mark_normals(const StreamKey& sk, uint32_t kg, uint32_t e, float* z) {
  const uint32_t i0 = e * QP;
  const P4 r = draw(sk, kSlotMark, i0 >> 2, kg);
  if (QP == 4) {
    box_muller(r.x, r.y, z[0], z[1]);
    box_muller(r.z, r.w, z[2], z[3]);
  } else {
    const bool hi = (i0 & 2u) != 0u;
    float a, b;
    box_muller(hi ? r.z : r.x, hi ? r.w : r.y, a, b);
    if (QP == 2) {
      z[0] = a;
      z[1] = b;
    } else {
      z[0] = (i0 & 1u) ? b : a;
    }
  }
}
#endif

}  // namespace jm
