"""Write the seeded output batches of every BASELINE.json config to data/cfg{i}.npz.

The draws come from ``lofp_inputs`` (no method arithmetic); the only other calls are to
``oracle/`` (structural reachability and exact path counts), so every stored value is
written by this committed script from the oracle alone (no CUDA involvement).

Stored per config:
  T_literal, P_literal : the literal batch of BASELINE.json (stream 1) and its exact
                         number of valid paths per output (0 = structural zero).
  T_cond, P_cond       : the measured batch (configs 2-4, reading R14): draws
                         from stream 2 kept iff structurally reachable and
                         P(T) <= P_CAP, until the batch is full.
  draws                : how many stream-2 candidates were drawn to fill T_cond.
  T_hero, P_hero       : configs[4] only: the 8 largest-P reachable outputs of 32768
                         uncapped stream-3 draws (single-output scaling).

usage: python scripts/make_batches.py [config indices...]
"""
from __future__ import annotations

import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import lofp_inputs as li  # noqa: E402
import oracle  # noqa: E402

P_CAP = 10 ** 9


def counts_u64(c, T):
    cnt = oracle.count_paths(c.M, c.layers, c.S, T)
    if any(x is None for x in cnt):
        raise RuntimeError("path counter state limit hit")
    if any(x >= 2 ** 64 for x in cnt):
        raise RuntimeError("path count overflows uint64")
    return np.array(cnt, dtype=np.uint64)


def conditioned(c, chunk):
    rng = np.random.default_rng([c.seed, 2])
    keepT, keepP = [], []
    have, draws = 0, 0
    t0 = time.time()
    while have < c.batch:
        if c.index in (1, 2):
            T = li.uniform_subsets(c.M, c.N, chunk, rng)
        elif c.index == 3:
            T = li.bounded_patterns(c.M, c.N, 2, chunk, rng)[0]
        else:
            src = [i for i in range(c.M) if c.S[i] > 0]
            T = li.displaced_patterns(c.M, src, 4, chunk, rng)[0]
        draws += chunk
        r = oracle.reachable(c.M, c.layers, c.S, T)
        cand = T[r]
        if len(cand):
            P = counts_u64(c, cand)
            ok = P <= P_CAP
            # keep draw order; stop exactly at the batch size
            for t, p in zip(cand[ok], P[ok]):
                if have < c.batch:
                    keepT.append(t)
                    keepP.append(p)
                    have += 1
        print(f"  cfg{c.index}: {draws} draws, {have} kept ({time.time() - t0:.0f}s)", flush=True)
    # exact draw count: recount the position of the last kept draw is not needed for the
    # experiment; report the candidates drawn (a multiple of chunk)
    return np.array(keepT, dtype=np.uint8), np.array(keepP, dtype=np.uint64), draws


def hero(c, n=8, chunks=8, chunk=4096):
    """Uncapped single-output scaling sample: the n largest-P structurally
    reachable outputs among chunks x chunk draws of stream 3 (same distribution as the
    conditioned batch, no path cap)."""
    rng = np.random.default_rng([c.seed, 3])
    src = [i for i in range(c.M) if c.S[i] > 0]
    Ts, Ps = [], []
    for _ in range(chunks):
        T = li.displaced_patterns(c.M, src, 4, chunk, rng)[0]
        cand = T[oracle.reachable(c.M, c.layers, c.S, T)]
        if len(cand):
            Ts.append(cand)
            Ps.append(counts_u64(c, cand))
    T, P = np.concatenate(Ts), np.concatenate(Ps)
    top = np.argsort(P.astype(np.float64), kind="stable")[::-1][:n]
    return T[top].astype(np.uint8), P[top], chunks * chunk


def main(which):
    os.makedirs(os.path.join(ROOT, "data"), exist_ok=True)
    for i in which:
        c = li.config(i)
        t0 = time.time()
        T = c.draw_outputs()
        P = counts_u64(c, T)
        out = dict(T_literal=T.astype(np.uint8), P_literal=P, cap=np.uint64(P_CAP))
        if i in (2, 3, 4):
            chunk = {2: 1 << 20, 3: 4096, 4: 4096}[i]
            Tc, Pc, draws = conditioned(c, chunk)
            out.update(T_cond=Tc, P_cond=Pc, draws=np.int64(draws))
        if i == 4:
            Th, Ph, hd = hero(c)
            out.update(T_hero=Th, P_hero=Ph, hero_draws=np.int64(hd))
        path = os.path.join(ROOT, "data", f"cfg{i}.npz")
        np.savez_compressed(path, **out)
        msg = f"cfg{i}: literal {len(T)} (sum P = {int(P.astype(object).sum()):.3e})"
        if "P_cond" in out:
            msg += f", conditioned {len(out['P_cond'])} (sum P = {int(out['P_cond'].astype(object).sum()):.3e})"
        print(msg + f" [{time.time() - t0:.0f}s] -> {path}", flush=True)


if __name__ == "__main__":
    main([int(a) for a in sys.argv[1:]] or [0, 1, 2, 3, 4])
