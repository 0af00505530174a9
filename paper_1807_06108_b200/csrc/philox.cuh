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
//   * zero-one jump law: one uniform per (sample, step) vs nu*dt
//     (noise.py:151); marks drawn only for jump events (noise.py:152-155).
//
// Counter layout (Philox4x32-10, Salmon et al. SC'11):
//   key  = (seed lo32, seed hi32)
//   ctr  = (block, sample, iteration lo32, slot<<24 | iteration hi32 & 0xffffff)
//   slot 0: diffusion normals, normal index i = t*MP + j, block = i>>2, lane = i&3
//   slot 1: jump uniforms, block = t>>2, word = t&3, jump iff word < thr<<8
//   slot 2: marks, normal index t*QP + i (QP = q, 3 padded to 4), block = index>>2
//           (drawn only for 4-step groups / blocks that hold a jump event)
//   slot 3: closed-loop plant, block = 3*step + {0 diffusion, 1 uniform, 2 marks}
// Normals: Box-Muller on pairs of words with 23-bit mantissa uniforms.
// The CPU emulation of this exact mapping is oracle/philox_stream.py.
#pragma once
#include <cstdint>

namespace jm {

struct P4 {
  uint32_t x, y, z, w;
};

enum : uint32_t { kSlotDiffusion = 0, kSlotJumpUniform = 1, kSlotMark = 2, kSlotPlant = 3 };

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

#ifdef __CUDACC__
// Box-Muller on two words.  u1 in (0,1], angle uniform in [-pi, pi).
// MUFU lg2/sqrt/sin/cos: noise quality only needs ~1e-6 relative accuracy;
// the fp64 kernels consume the very same float normals (cast), so both
// precisions see identical noise for a given (seed, iteration).
__device__ __forceinline__ void box_muller(uint32_t a, uint32_t b, float& z0, float& z1) {
  const float u1 = 2.0f - __uint_as_float(0x3F800000u | (a >> 9));        // (0, 1]
  const float ang = __fmaf_rn(__uint_as_float(0x3F800000u | (b >> 9)),     // [1,2) -> [-pi,pi)
                              6.2831853071795865f, -9.4247779607693797f);
  const float rr = __fmul_rn(-1.3862943611198906f, __log2f(u1));          // -2 ln u1
  float r;
  asm("sqrt.approx.f32 %0, %1;" : "=f"(r) : "f"(rr));
  float sn, cs;
  __sincosf(ang, &sn, &cs);
  z0 = __fmul_rn(r, cs);
  z1 = __fmul_rn(r, sn);
}
#endif

}  // namespace jm
