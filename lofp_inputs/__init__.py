"""Seeded synthetic inputs for the LOFP path sum (shared by the oracle side and the CUDA side).

This module holds NO arithmetic of the method: it only draws circuits (mode pairs and
angles) and Fock patterns.  Both ``oracle/`` and ``paper_2510_26408_b200`` consume what
it produces; neither is imported here.

Conventions (readings R3, R10-R13):
  * Modes are 0-based.  A "Clements-style" mesh of depth D on M modes has, in layer l
    (1-based), the nearest-neighbour pairs (0,1),(2,3),... when l is odd and
    (1,2),(3,4),... when l is even (the parity the worked example of P:164 fixes;
    BASELINE.json configs[0] "15 BS" for M=6, D=6).
  * Angles: ``numpy.random.default_rng(seed)``; for l = 1..D, for each pair top to
    bottom, theta ~ U[0, pi/2) then phi ~ U[0, 2 pi) (BASELINE.json configs; P:80 states
    phi in [0, pi], the configs widen it).
  * Output batches are drawn from ``default_rng([seed, 1])`` i.i.d. (duplicates allowed).
"""
from __future__ import annotations

import itertools
import math
from dataclasses import dataclass, field

import numpy as np


def clements_pairs(M: int, D: int):
    """Mode pairs of each layer of the brickwork mesh (layer 1 couples (0,1),(2,3),...)."""
    layers = []
    for l in range(1, D + 1):
        start = 0 if l % 2 == 1 else 1
        layers.append([(a, a + 1) for a in range(start, M - 1, 2)])
    return layers


def clements_mesh(M: int, D: int, seed: int):
    """Layers of (mode_a, mode_b, theta, phi) with angles drawn as described above."""
    rng = np.random.default_rng(seed)
    out = []
    for pairs in clements_pairs(M, D):
        layer = []
        for a, b in pairs:
            theta = float(rng.uniform(0.0, math.pi / 2))
            phi = float(rng.uniform(0.0, 2 * math.pi))
            layer.append((a, b, theta, phi))
        out.append(layer)
    return out


def random_nn_circuit(M: int, D: int, rng, fill: float = 1.0, reverse_prob: float = 0.0):
    """Random nearest-neighbour circuit with partially filled layers (test inputs).

    Each layer picks disjoint adjacent pairs greedily from a random start; every pair is
    kept with probability ``fill``; a kept pair is listed as (b, a) with probability
    ``reverse_prob`` (port 1 = the lower mode).
    """
    layers = []
    for _ in range(D):
        layer = []
        k = int(rng.integers(0, 2))
        while k + 1 < M:
            if rng.random() < fill:
                a, b = k, k + 1
                if rng.random() < reverse_prob:
                    a, b = b, a
                layer.append((a, b, float(rng.uniform(0, math.pi / 2)), float(rng.uniform(0, 2 * math.pi))))
                k += 2
            else:
                k += 1
        layers.append(layer)
    return layers


def random_nonlocal_circuit(M: int, D: int, rng, fill: float = 0.8, reverse_prob: float = 0.3):
    """Random circuit with non-local pairs (test inputs for NEXT-4, "non-local
    connections"): each layer pairs a random subset of the modes with each other, any
    distance apart (disjoint pairs, crossings allowed)."""
    layers = []
    for _ in range(D):
        modes = list(rng.permutation(M))
        layer = []
        while len(modes) >= 2:
            a, b = int(modes.pop()), int(modes.pop())
            if rng.random() < fill:
                if rng.random() < reverse_prob:
                    a, b = b, a
                layer.append((a, b, float(rng.uniform(0, math.pi / 2)), float(rng.uniform(0, 2 * math.pi))))
        layers.append(layer)
    return layers


def all_outputs(M: int, N: int) -> np.ndarray:
    """All occupation patterns of N photons in M modes, lexicographically descending."""
    rows = []

    def rec(prefix, left, modes_left):
        if modes_left == 1:
            rows.append(prefix + [left])
            return
        for v in range(left, -1, -1):
            rec(prefix + [v], left - v, modes_left - 1)

    if M == 0:
        return np.zeros((0, 0), dtype=np.int32)
    rec([], N, M)
    return np.array(rows, dtype=np.int32)


def uniform_subsets(M: int, n: int, B: int, rng) -> np.ndarray:
    """B i.i.d. collision-free patterns, uniform over the n-subsets of M modes."""
    out = np.zeros((B, M), dtype=np.int32)
    if B == 0:
        return out
    idx = np.argsort(rng.random((B, M)), axis=1)[:, :n]
    np.put_along_axis(out, idx, 1, axis=1)
    return out


def bounded_patterns(M: int, N: int, cap: int, B: int, rng) -> np.ndarray:
    """B i.i.d. patterns uniform over {t : sum t = N, 0 <= t_i <= cap} (reading R12)."""
    cnt = [[0] * (N + 1) for _ in range(M + 1)]
    cnt[M][0] = 1
    for i in range(M - 1, -1, -1):
        for r in range(N + 1):
            cnt[i][r] = sum(cnt[i + 1][r - v] for v in range(0, min(cap, r) + 1))
    total = cnt[0][N]
    out = np.zeros((B, M), dtype=np.int32)
    for b in range(B):
        r = N
        for i in range(M):
            u = int(rng.integers(0, cnt[i][r]))
            for v in range(0, min(cap, r) + 1):
                w = cnt[i + 1][r - v]
                if u < w:
                    out[b, i] = v
                    r -= v
                    break
                u -= w
    return out, total


def displaced_patterns(M: int, sources, d: int, B: int, rng):
    """B i.i.d. collision-free patterns o_1 < ... < o_n with |o_i - s_i| <= d, uniform over
    all such sorted placements (reading R13).  Returns (batch, number of patterns)."""
    s = list(sources)
    n = len(s)
    # cnt[i][p]: number of ways to place photons i..n-1 given photon i sits at mode p
    cnt = [dict() for _ in range(n + 1)]
    for i in range(n - 1, -1, -1):
        for p in range(max(0, s[i] - d), min(M - 1, s[i] + d) + 1):
            if i == n - 1:
                cnt[i][p] = 1
            else:
                cnt[i][p] = sum(w for q, w in cnt[i + 1].items() if q > p)
    total = sum(cnt[0].values())
    out = np.zeros((B, M), dtype=np.int32)
    for b in range(B):
        prev = -1
        for i in range(n):
            opts = sorted((p, w) for p, w in cnt[i].items() if p > prev)
            tot = sum(w for _, w in opts)
            u = int(rng.integers(0, tot))
            for p, w in opts:
                if u < w:
                    out[b, p] = 1
                    prev = p
                    break
                u -= w
    return out, total


@dataclass
class Config:
    """One BASELINE.json configuration: circuit, input state and the literal output draw."""
    index: int
    M: int
    D: int
    N: int
    seed: int
    S: np.ndarray
    batch: int
    desc: str
    layers: list = field(default_factory=list)

    def draw_outputs(self, B: int | None = None, stream: int = 1) -> np.ndarray:
        """The literal output batch of the config (BASELINE.json), rows i.i.d."""
        B = self.batch if B is None else B
        rng = np.random.default_rng([self.seed, stream])
        if self.index == 0:
            return all_outputs(self.M, self.N)
        if self.index in (1, 2):
            return uniform_subsets(self.M, self.N, B, rng)
        if self.index == 3:
            return bounded_patterns(self.M, self.N, 2, B, rng)[0]
        if self.index == 4:
            src = [i for i in range(self.M) if self.S[i] > 0]
            return displaced_patterns(self.M, src, 4, B, rng)[0]
        raise ValueError(self.index)


def _cfg(index, M, D, seed, occ, batch, desc):
    S = np.zeros(M, dtype=np.int32)
    for m, v in occ:
        S[m] = v
    return Config(index=index, M=M, D=D, N=int(S.sum()), seed=seed, S=S, batch=batch, desc=desc,
                  layers=clements_mesh(M, D, seed))


def config(index: int) -> Config:
    """BASELINE.json configs[index] as concrete inputs."""
    if index == 0:
        return _cfg(0, 6, 6, 0, [(0, 1), (1, 1), (2, 1)], 56, "m=6 n=3 D=6, all 56 outputs")
    if index == 1:
        return _cfg(1, 16, 4, 1, [(m, 1) for m in range(0, 16, 2)], 1024,
                    "m=16 n=8 D=4, 1024 uniform 8-subsets")
    if index == 2:
        return _cfg(2, 32, 6, 2, [(m, 1) for m in range(16)], 4096,
                    "m=32 n=16 D=6, 4096 uniform 16-subsets")
    if index == 3:
        return _cfg(3, 24, 8, 3, [(m, 2) for m in range(0, 24, 4)], 2048,
                    "m=24 n=12 D=8 bunched, 2048 patterns <=2/mode")
    if index == 4:
        return _cfg(4, 64, 4, 4, [(m, 1) for m in range(0, 48, 2)], 16384,
                    "m=64 n=24 D=4, 16384 displacement<=4 patterns")
    raise ValueError(f"no config {index}")


def paper_correctness_inputs():
    """The four 6-mode inputs of the paper's correctness check, with their depths."""
    return [((1, 1, 1, 1, 1, 1), 3), ((0, 0, 4, 0, 0, 4), 4), ((2, 0, 3, 0, 0, 3), 5), ((2, 0, 0, 2, 0, 2), 6)]
