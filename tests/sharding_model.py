"""Ant sharding across ranks — the host-side contract the C
engine (aco_gpu.cu: aco_gpu_create / do_update / finish_stats) implements.

* Rank r of G owns the contiguous global ants [r*S, min(m, (r+1)*S)),
  S = ceil(m / G).  The RNG is keyed by the GLOBAL ant id (rng.hpp:54-55,
  engine.hpp:101-103), so every tour is independent of G.
* Deterministic (scatter-to-gather) deposit: ranks all-gather their
  per-city successor/predecessor tables and w_k = 1/C_k in shard-major
  layout ([shard][city][S]); every rank then folds contributions per cell in
  ascending global ant order — bit-identical to G = 1 (pheromone.hpp:133-148).
* Atomic deposit: each rank scatters its ants into a zeroed delta, delta is
  all-reduced (sum), then tau = fl(fl(tau * (1 - rho)) + delta) — within the
  1e-5 relative tolerance of deposit_accumulate (pheromone.hpp:195-208).
* Iteration stats, all on the device (no host round trip): the iteration
  best and its lowest global ant (the reference's tie rule,
  engine.hpp:117-129) come from ONE all-reduce MIN of the packed key
  (length << shift) | global ant, shift = ceil(log2 m), whenever every
  possible tour length fits (n * max_d < 2^(62 - shift)); otherwise from two
  MINs, the length and then the lowest ant among ranks holding it.  Lengths
  are summed by an all-reduce SUM; the owning rank contributes its best tour
  and the others zeros to an all-reduce MAX, which replicates the winning
  tour; best-so-far updates on strict improvement (engine.hpp:151-154).

TEST SUPPORT: the CPU model of that protocol used by
tests/test_multirank_gloo.py (the product path is aco_gpu.cu).
"""
from __future__ import annotations

INF = 2**63 - 1


def key_shift(m: int) -> int:
    """Bits of the ant field (aco_gpu_create: smallest s >= 1 with 2^s >= m)."""
    s = 1
    while (1 << s) < m:
        s += 1
    return s


def two_stage(m: int, n: int, max_d: int) -> bool:
    s = key_shift(m)
    return s >= 62 or n * max(max_d, 1) >= (1 << (62 - s))


def shard_size(m: int, world: int) -> int:
    return -(-m // world)


def shard_range(m: int, world: int, rank: int):
    s = shard_size(m, world)
    return min(m, rank * s), min(m, (rank + 1) * s)


def owner_of(ant: int, m: int, world: int) -> int:
    return ant // shard_size(m, world)


def stats_key(best_length: int, best_local_ant: int, ant_begin: int, shift: int) -> int:
    """Stage-1 MIN key of a shard's iteration best (k_shard_key); shift == 0
    is the two-stage protocol's length-only key."""
    if shift == 0:
        return best_length
    return (best_length << shift) | (ant_begin + best_local_ant)


def stage2_ant(best_length: int, best_local_ant: int, ant_begin: int, global_len: int) -> int:
    """Two-stage protocol, k_shard_ant: candidate ant or +inf (then MIN)."""
    return ant_begin + best_local_ant if best_length == global_len else INF


def unpack_key(key: int, shift: int):
    """(best length, global ant) of a reduced packed key."""
    return key >> shift, key & ((1 << shift) - 1)
