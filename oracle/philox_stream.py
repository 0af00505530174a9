"""CPU emulation of the device noise stream (csrc/philox.cuh).

TEST INFRASTRUCTURE ONLY.  Philox4x32-10 (Salmon, Moraes, Dror, Shaw, SC'11;
the Random123 reference algorithm -- restated here from the published round
function, pinned by the Random123 known-answer vectors in
tests/test_oracle_golden.py) with the repo's counter layout and Box-Muller
mapping.  Integer outputs (Philox words, jump indicators) are bit-exact with
the device; normals agree to ~1e-6 relative (the device uses MUFU
lg2/sqrt/sin/cos approximations, this emulation float64 libm).
"""

from __future__ import annotations

import math

import numpy as np

M0, M1 = np.uint64(0xD2511F53), np.uint64(0xCD9E8D57)
W0, W1 = np.uint32(0x9E3779B9), np.uint32(0xBB67AE85)
MASK = np.uint64(0xFFFFFFFF)

SLOT_DIFFUSION, SLOT_JUMP_UNIFORM, SLOT_MARK, SLOT_PLANT, SLOT_COUNT = 0, 1, 2, 3, 4
MAX_COUNT = 8


def philox4x32_10(c0, c1, c2, c3, k0, k1):
    """Vectorised Philox4x32-10 on uint32 arrays; returns 4 uint32 arrays."""
    c0, c1, c2, c3 = (np.asarray(v, dtype=np.uint32) for v in (c0, c1, c2, c3))
    c0, c1, c2, c3 = np.broadcast_arrays(c0, c1, c2, c3)
    k0 = np.uint32(k0)
    k1 = np.uint32(k1)
    with np.errstate(over="ignore"):
        for _ in range(10):
            p0 = M0 * c0.astype(np.uint64)
            p1 = M1 * c2.astype(np.uint64)
            hi0, lo0 = (p0 >> np.uint64(32)).astype(np.uint32), (p0 & MASK).astype(np.uint32)
            hi1, lo1 = (p1 >> np.uint64(32)).astype(np.uint32), (p1 & MASK).astype(np.uint32)
            c0, c1, c2, c3 = hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0
            k0 = np.uint32(k0 + W0)
            k1 = np.uint32(k1 + W1)
    return c0, c1, c2, c3


def stream_key(seed: int, iteration: int):
    seed, iteration = int(seed), int(iteration)
    return (seed & 0xFFFFFFFF, (seed >> 32) & 0xFFFFFFFF, iteration & 0xFFFFFFFF,
            (iteration >> 32) & 0xFFFFFF)


def draw(key, slot, block, sample):
    k0, k1, c2, c3 = key
    c3s = np.uint32(c3 | (slot << 24))
    return philox4x32_10(block, sample, np.uint32(c2), c3s, k0, k1)


def _f32_from_bits(bits):
    return np.asarray(bits, dtype=np.uint32).view(np.float32)


def box_muller(a, b):
    """Device mapping: u1 = 2 - [1,2) in (0,1], angle = [1,2)*2pi - 3pi."""
    one = np.uint32(0x3F800000)
    u1 = (np.float32(2.0) - _f32_from_bits(one | (np.asarray(a, np.uint32) >> np.uint32(9)))).astype(np.float64)
    f = _f32_from_bits(one | (np.asarray(b, np.uint32) >> np.uint32(9))).astype(np.float64)
    ang = np.float32(f * np.float64(np.float32(6.2831853071795865)) + np.float64(np.float32(-9.4247779607693797)))
    r = np.sqrt(-2.0 * np.log(u1))
    ang = np.asarray(ang, dtype=np.float64)
    return r * np.cos(ang), r * np.sin(ang)


def gap_table(p: float, T: int):
    """Survival table of the geometric jump gaps (csrc/philox.cuh slot 1, api.cu gap_table):
    S[0] = 2^24, S[g] = floor(S[g-1] (2^24 - q) / 2^24), q = ceil(p 2^24); exact integers."""
    q = min(int(np.ceil(p * 16777216.0)), 16777216) if p > 0 else 0
    S = [1 << 24]
    for _ in range(T):
        S.append((S[-1] * ((1 << 24) - q)) >> 24)
    return np.array(S, dtype=np.int64)


def jump_gap(S, u24):
    """G = max{g in [0, T] : u < S[g]} (S decreasing, S[0] = 2^24 > u)."""
    return np.sum(np.asarray(u24, np.int64)[..., None] < S[None, 1:], axis=-1)


def jump_events(key, k, T, p):
    """Per-sample jump steps from the renewal clock: list over events e of
    (event index e, step array (K,), alive mask (K,) where step < T)."""
    S = gap_table(p, T)
    K = k.shape[0]
    t = np.full(K, -1, dtype=np.int64)
    out = []
    e = 0
    while True:
        w = draw(key, SLOT_JUMP_UNIFORM, np.uint32(e >> 2), k[:, 0])
        u24 = (w[e & 3] >> np.uint32(8)).astype(np.int64)
        t = t + 1 + jump_gap(S, u24)
        alive = t < T
        if not alive.any():
            return out
        out.append((e, t.copy(), alive))
        e += 1


def event_probability(nu_dt: float, poisson: bool = False) -> float:
    """Per-step probability of a jump event: nu dt (zero-one law, noise.py:151) or
    P(N >= 1) = 1 - exp(-nu dt) for Poisson(nu dt) arrivals (api.cu event_probability)."""
    return -math.expm1(-nu_dt) if poisson else nu_dt


def poisson_tail(lam: float, k: int) -> float:
    """P(N > k), N ~ Poisson(lam): the forward sum of the next 40 pmf terms in the
    device library's order (api.cu poisson_tail), so both round alike."""
    term = math.exp(-lam)
    for j in range(1, k + 1):
        term *= lam / j
    s = 0.0
    for j in range(k + 1, k + 41):
        term *= lam / j
        s += term
    return s


def count_tables(lam: float):
    """(event, plant) count thresholds of philox.cuh slot 4 / the plant draw:
    event arrivals n = 1 + #{k : u24 < ev[k-1]}, ev[k-1] = floor(2^24 P(N > k) / P(N >= 1));
    plant arrivals n = #{k : u24 < pl[k]}, pl[0] = ceil(P(N >= 1) 2^24), pl[k] = floor(2^24 P(N > k))."""
    p1 = -math.expm1(-lam)
    ev, pl = [], [jump_threshold(p1) >> 8]
    for k in range(1, MAX_COUNT + 1):
        t = poisson_tail(lam, k)
        ev.append(int(math.floor(t / p1 * 16777216.0)) if p1 > 0 else 0)
        pl.append(int(math.floor(t * 16777216.0)))
    return np.array(ev, dtype=np.int64), np.array(pl, dtype=np.int64)


def event_counts(key, k, e, ev):
    """Arrival counts of event e for samples k (slot 4, word e&3 of block e>>2)."""
    w = draw(key, SLOT_COUNT, np.uint32(e >> 2), k)
    u = (w[e & 3] >> np.uint32(8)).astype(np.int64)
    return 1 + np.sum(u[..., None] < np.asarray(ev, np.int64)[None, :], axis=-1)


def jump_threshold(p: float) -> int:
    if not p > 0:
        return 0
    thr = min(int(np.ceil(p * 16777216.0)), 16777215)
    return thr << 8


def device_noise(seed, iteration, K, T, m, q, Ld, Lj, mark_mean, jthr, jump_channel="control",
                 sample_offset=0, counts=None):
    """(eps_d, ind, eps_j, eps_c) as the device sampler draws them (float64).

    Ld (m x m) = chol(c Sigma_D), Lj (q x q) = chol(Sigma_J), jthr from
    jump_threshold(event_probability(nu dt)) (0 = no jumps; the renewal clock's
    per-step probability is its quantised ceil(p 2^24) / 2^24).  counts: the
    event table of count_tables(nu dt) for Poisson arrivals (ind = n, the mark
    the sum of n marks, n mu + sqrt(n) Lj z); None = one arrival per event."""
    key = stream_key(seed, iteration)
    MP = 4 if m == 3 else m
    k = (np.arange(K, dtype=np.int64) + sample_offset).astype(np.uint32)[:, None]
    # diffusion normals: index i = t*MP + j, block i>>2
    nblk = (T * MP + 3) // 4
    blocks = np.arange(nblk, dtype=np.uint32)[None, :]
    w = draw(key, SLOT_DIFFUSION, blocks, k)
    z01 = box_muller(w[0], w[1])
    z23 = box_muller(w[2], w[3])
    z = np.stack([z01[0], z01[1], z23[0], z23[1]], axis=-1).reshape(K, nblk * 4)[:, : T * MP]
    z = z.reshape(K, T, MP)[:, :, :m]
    eps_d = np.einsum("jl,ktl->ktj", np.tril(Ld), z)
    ind = np.zeros((K, T), dtype=np.int64)
    eps_j = np.zeros((K, T, q))
    if jthr:
        # jump steps from the renewal clock; marks of event e: normals e*QP + i (slot 2)
        p = (jthr >> 8) / 16777216.0  # the quantised per-step probability the table is built from
        QP = 4 if q == 3 else q
        for e, t, alive in jump_events(key, k, T, p):
            rows = np.nonzero(alive)[0]
            cols = t[rows]
            n = event_counts(key, k[rows, 0], e, counts) if counts is not None else np.ones(rows.size, np.int64)
            ind[rows, cols] = n
            idx = np.int64(e * QP) + np.arange(q)[None, :]
            blk = np.broadcast_to((idx >> 2).astype(np.uint32), (rows.size, q))
            mw = draw(key, SLOT_MARK, blk, k[rows, 0][:, None])
            a01 = box_muller(mw[0], mw[1])
            a23 = box_muller(mw[2], mw[3])
            allz = np.stack([a01[0], a01[1], a23[0], a23[1]], axis=-1)  # (events, q, 4)
            zz = np.take_along_axis(allz, np.broadcast_to((idx & 3)[..., None], (rows.size, q, 1)), axis=-1)[..., 0]
            nn = n.astype(float)[:, None]
            eps_j[rows, cols] = np.where(nn > 1, nn * np.asarray(mark_mean, float)[:q] + np.sqrt(nn) * (zz @ np.tril(Lj).T),
                                         np.asarray(mark_mean, float)[:q] + zz @ np.tril(Lj).T)
    eps_c = eps_d + eps_j if jump_channel == "control" else eps_d.copy()
    return eps_d, ind, eps_j, eps_c
