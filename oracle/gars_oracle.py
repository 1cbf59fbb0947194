"""oracle/gars_oracle.py — TEST INFRASTRUCTURE ONLY (the checker, never the
product path).  Pure-Python restatement of GARS for parity tests of
include/janus/gars.hpp (through the C ABI janus_gars_*).

Follows the reference SPEC (module "gars") and PAPER.md
Algorithm 1:
  * pack_and_shuffle: sort by atoms descending, ties by id ascending
    (SPEC.md:514); each graph to the micro-batch of minimum current total,
    ties to the lowest index; shuffle each micro-batch with
    ONE SplitMix64(seed) stream, micro-batch 0 first, descending Fisher-Yates
    (rng.hpp:29-34); tag comm_free iff max <= total / d_gp
    (PAPER.md:724-730).
  * assign_gp_bins, greedy sequential baseline
    (PAPER.md:917-918), synth_dataset inverse CDF,
    balance_stats.
Parity is pinned to the SPEC's worked examples (tests/test_gars.py).
"""
from __future__ import annotations

import math

M64 = (1 << 64) - 1


class SplitMix64:
    """reference rng.hpp:11-38."""

    def __init__(self, seed: int):
        self.s = seed & M64

    def next(self) -> int:
        self.s = (self.s + 0x9E3779B97F4A7C15) & M64
        z = self.s
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
        return z ^ (z >> 31)

    def next_below(self, n: int) -> int:
        return 0 if n <= 1 else self.next() % n

    def next_double(self) -> float:
        return (self.next() >> 11) * 2.0 ** -53

    def shuffle(self, v: list) -> None:
        for i in range(len(v), 1, -1):
            j = self.next_below(i)
            v[i - 1], v[j] = v[j], v[i - 1]


def tag_of(sizes, d_gp: int) -> int:
    """0 = comm_free, 1 = dist."""
    return 0 if max(sizes) * d_gp <= sum(sizes) else 1


def pack_and_shuffle(atoms, n_mb: int, d_gp: int, seed: int):
    """-> list of (graph ids in shuffled order, tag)."""
    order = sorted(range(len(atoms)), key=lambda i: (-atoms[i], i))
    groups = [[] for _ in range(n_mb)]
    load = [0] * n_mb
    for i in order:
        j = min(range(n_mb), key=lambda k: (load[k], k))
        groups[j].append(i)
        load[j] += atoms[i]
    rng = SplitMix64(seed)
    out = []
    for g in groups:
        rng.shuffle(g)
        out.append((g, tag_of([atoms[i] for i in g], d_gp) if g else 0))
    return out


def assign_gp_bins(sizes, d_gp: int):
    load = [0] * d_gp
    bins = []
    for a in sizes:
        b = min(range(d_gp), key=lambda k: (load[k], k))
        bins.append(b)
        load[b] += a
    return bins


def greedy_sequential(atoms, n_mb: int):
    budget = -(-sum(atoms) // n_mb)
    groups = [[] for _ in range(n_mb)]
    tot = [0] * n_mb
    j = 0
    for i, a in enumerate(atoms):
        if j + 1 < n_mb and groups[j] and tot[j] + a > budget:
            j += 1
        groups[j].append(i)
        tot[j] += a
    return groups


def synth_sizes(n: int, seed: int, stats=(85, 53, 213, 427, 905)):
    q = [0.0, 0.5, 0.9, 0.99, 1.0]
    v = [1.0, stats[1], stats[2], stats[3], stats[4]]
    rng = SplitMix64(seed)
    out = []
    for _ in range(n):
        u = rng.next_double()
        k = 0
        while k < 3 and u >= q[k + 1]:
            k += 1
        t = (u - q[k]) / (q[k + 1] - q[k])
        x = v[k] + t * (v[k + 1] - v[k])
        out.append(int(min(stats[4], max(1.0, float(round(x))))))
    return out


def balance_stats(totals):
    m = sum(totals) / len(totals)
    return m, math.sqrt(sum((t - m) ** 2 for t in totals) / len(totals))
