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
* Iteration stats, all on the device (no host round trip): one all-reduce
  MIN of the packed key (best length << 24 | global ant) gives the best
  length and its lowest global ant (the reference's tie rule,
  engine.hpp:117-129); all-reduce SUM of the int64 lengths; the owning rank
  contributes its best tour and the others zeros to an all-reduce MAX,
  which replicates the winning tour; best-so-far updates on strict
  improvement (engine.hpp:151-154).
"""
from __future__ import annotations

KEY_SHIFT = 24  # global ant ids < 2**24


def shard_size(m: int, world: int) -> int:
    return -(-m // world)


def shard_range(m: int, world: int, rank: int):
    s = shard_size(m, world)
    return min(m, rank * s), min(m, (rank + 1) * s)


def owner_of(ant: int, m: int, world: int) -> int:
    return ant // shard_size(m, world)


def stats_key(best_length: int, best_local_ant: int, ant_begin: int) -> int:
    """Packed MIN key of a shard's iteration best (k_shard_key)."""
    return (best_length << KEY_SHIFT) | (ant_begin + best_local_ant)


def unpack_key(key: int):
    """(best length, global ant) of a reduced key."""
    return key >> KEY_SHIFT, key & ((1 << KEY_SHIFT) - 1)
