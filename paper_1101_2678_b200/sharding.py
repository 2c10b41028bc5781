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
* Iteration stats: all-reduce MIN of the best length, then MIN of the global
  ant index among the ranks holding it (the reference's lowest-index tie
  rule, engine.hpp:117-129), all-reduce SUM of the int64 lengths; the owner
  broadcasts the best tour when it strictly improves best-so-far.
"""
from __future__ import annotations


def shard_size(m: int, world: int) -> int:
    return -(-m // world)


def shard_range(m: int, world: int, rank: int):
    s = shard_size(m, world)
    return min(m, rank * s), min(m, (rank + 1) * s)


def owner_of(ant: int, m: int, world: int) -> int:
    return ant // shard_size(m, world)
