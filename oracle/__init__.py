"""CPU oracle for the LOFP path sum — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product path
(``paper_2510_26408_b200``) never imports it, and this package imports nothing from
the product path.  The arithmetic lives in ``lofp_oracle.c`` (long double, written
from PAPER.md; see its header for the passage each function follows); this module
only marshals numpy arrays through ctypes.

A circuit is given as ``layers``: a list of D layers, each a list of
``(mode_a, mode_b, theta, phi)`` tuples; ``mode_a`` is BS port 1.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "lofp_oracle.c")
_LIB_PATH = os.path.join(_HERE, "liblofp_oracle.so")
_lib = None

_i32p = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(dtype=np.uint64, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(dtype=np.uint8, flags="C_CONTIGUOUS")


def build(force: bool = False) -> str:
    """Compile the oracle (plain gcc, -O2, OpenMP, no fast-math)."""
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(_SRC):
        tmp = _LIB_PATH + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-shared", "-fPIC", "-std=gnu11",
                               "-o", tmp, _SRC, "-lquadmath", "-lm"])
        os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB_PATH)
        c_int, c_long, c_double = ctypes.c_int, ctypes.c_long, ctypes.c_double
        lib.oracle_bs_element.argtypes = [c_double, c_double, c_int, c_int, c_int, c_int, _f64p]
        lib.oracle_bs_element.restype = None
        lib.oracle_naive_permanent.argtypes = [c_int, _f64p, _f64p]
        lib.oracle_ryser_permanent.argtypes = [c_int, _f64p, _f64p]
        circ = [c_int, c_int, _i32p, _i32p, _i32p]
        lib.oracle_circuit_unitary.argtypes = circ + [_f64p, _f64p, _f64p]
        lib.oracle_amplitude_permanent.argtypes = circ + [_f64p, _f64p, _i32p, c_long, _i32p, c_int, c_int, _f64p]
        lib.oracle_path_sum.argtypes = circ + [_f64p, _f64p, _i32p, c_long, _i32p, c_int, c_int, _f64p, _u64p]
        lib.oracle_path_sum_gates.argtypes = circ + [_f64p, _f64p, _i32p, c_long, _i32p, c_int, c_int, c_int,
                                                     _i32p, _i32p, _f64p, _f64p, _f64p, _u64p]
        lib.oracle_cone_sets.argtypes = circ + [c_int, c_int, _i32p, _i32p]
        lib.oracle_reachable.argtypes = circ + [_i32p, c_long, _i32p, c_int, _u8p]
        lib.oracle_count_paths.argtypes = circ + [_i32p, c_long, _i32p, c_int, c_long, _u64p, _i32p]
        _lib = lib
    return _lib


def _flatten(layers):
    bpl = np.array([len(l) for l in layers], dtype=np.int32)
    flat = [bs for l in layers for bs in l]
    ma = np.array([b[0] for b in flat], dtype=np.int32)
    mb = np.array([b[1] for b in flat], dtype=np.int32)
    th = np.array([b[2] for b in flat], dtype=np.float64)
    ph = np.array([b[3] for b in flat], dtype=np.float64)
    if len(bpl) == 0:
        bpl = np.zeros(1, dtype=np.int32)
    for a in (ma, mb, th, ph):
        if a.size == 0:
            a.resize(1, refcheck=False)
    return bpl, ma, mb, th, ph


def _state(x, M):
    a = np.ascontiguousarray(np.asarray(x, dtype=np.int32))
    if a.shape[-1] != M:
        raise ValueError("occupation vector length must equal the number of modes")
    return a


def _batch(T, M):
    a = np.ascontiguousarray(np.asarray(T, dtype=np.int32))
    if a.ndim == 1:
        a = a[None, :]
    if a.shape[1] != M:
        raise ValueError("output rows must have one entry per mode")
    return a


def _check(rc, what):
    if rc != 0:
        raise ValueError(f"oracle {what} failed with code {rc}")


def bs_element(theta, phi, x1, x2, y1, y2) -> complex:
    """<y1,y2|BS(theta,phi)|x1,x2> by Appendix A (reading R1)."""
    out = np.zeros(2)
    _load().oracle_bs_element(float(theta), float(phi), int(x1), int(x2), int(y1), int(y2), out)
    return complex(out[0], out[1])


def permanent(A, method: str = "ryser") -> complex:
    A = np.ascontiguousarray(np.asarray(A, dtype=np.complex128))
    n = A.shape[0]
    a = np.ascontiguousarray(A.view(np.float64).reshape(-1))
    if a.size == 0:
        a = np.zeros(2)
    out = np.zeros(2)
    fn = _load().oracle_naive_permanent if method == "naive" else _load().oracle_ryser_permanent
    _check(fn(n, a, out), "permanent")
    return complex(out[0], out[1])


def circuit_unitary(M, layers) -> np.ndarray:
    """U = U_D ... U_1, U[out, in]."""
    bpl, ma, mb, th, ph = _flatten(layers)
    out = np.zeros(M * M * 2)
    _check(_load().oracle_circuit_unitary(M, len(layers), bpl, ma, mb, th, ph, out), "circuit_unitary")
    return out.view(np.complex128).reshape(M, M)


def amplitudes_permanent(M, layers, S, T, method: str = "ryser", threads: int = 0) -> np.ndarray:
    """Per(U[T,S]) / sqrt(prod S! prod T!) for every row of T."""
    bpl, ma, mb, th, ph = _flatten(layers)
    S = _state(S, M)
    T = _batch(T, M)
    out = np.zeros(T.shape[0] * 2)
    rc = _load().oracle_amplitude_permanent(M, len(layers), bpl, ma, mb, th, ph, S, T.shape[0], T,
                                             1 if method == "naive" else 0, threads, out)
    _check(rc, "amplitude_permanent")
    return out.view(np.complex128)


PRUNE_NONE, PRUNE_CONE, PRUNE_BOX = 0, 1, 2


def path_sum(M, layers, S, T, prune: int = PRUNE_BOX, threads: int = 0, return_leaves: bool = False,
             gates=()):
    """Eq. (1) for every row of T; optionally the number of valid paths summed.

    ``gates``: photon-number-preserving phase gates, tuples
    ``(mode, after_layer, a, b)`` multiplying every path by exp(i (a n + b n^2)), n = the
    photons in ``mode`` after layer ``after_layer`` (0 = on the input).
    """
    bpl, ma, mb, th, ph = _flatten(layers)
    S = _state(S, M)
    T = _batch(T, M)
    B = T.shape[0]
    out = np.zeros(B * 2)
    leaves = np.zeros(max(B, 1), dtype=np.uint64)
    G = len(gates)
    gm = np.array([g[0] for g in gates] or [0], dtype=np.int32)
    gl = np.array([g[1] for g in gates] or [0], dtype=np.int32)
    ga = np.array([g[2] for g in gates] or [0.0], dtype=np.float64)
    gb = np.array([g[3] for g in gates] or [0.0], dtype=np.float64)
    rc = _load().oracle_path_sum_gates(M, len(layers), bpl, ma, mb, th, ph, S, B, T, prune, threads, G,
                                       gm, gl, ga, gb, out, leaves)
    _check(rc, "path_sum")
    amps = out.view(np.complex128)
    return (amps, leaves[:B].copy()) if return_leaves else amps


def cone_sets(M, layers, m, j):
    """Past (input) and future (output) light cones of waveguide (mode m, segment j)."""
    bpl, ma, mb, th, ph = _flatten(layers)
    past = np.zeros(M, dtype=np.int32)
    fut = np.zeros(M, dtype=np.int32)
    _check(_load().oracle_cone_sets(M, len(layers), bpl, ma, mb, m, j, past, fut), "cone_sets")
    return past.astype(bool), fut.astype(bool)


def reachable(M, layers, S, T, threads: int = 0) -> np.ndarray:
    """Structural reachability of every row of T (reading R5)."""
    bpl, ma, mb, th, ph = _flatten(layers)
    S = _state(S, M)
    T = _batch(T, M)
    out = np.zeros(max(T.shape[0], 1), dtype=np.uint8)
    _check(_load().oracle_reachable(M, len(layers), bpl, ma, mb, S, T.shape[0], T, threads, out), "reachable")
    return out[: T.shape[0]].astype(bool)


def count_paths(M, layers, S, T, threads: int = 0, max_states: int = 1 << 22) -> list:
    """Exact number of valid paths (terms of eq. (1)) for every row of T (reading R6).

    Returns Python ints (counts may exceed 2**64); None where the state space limit was hit.
    """
    bpl, ma, mb, th, ph = _flatten(layers)
    S = _state(S, M)
    T = _batch(T, M)
    B = T.shape[0]
    out = np.zeros(max(B, 1) * 2, dtype=np.uint64)
    st = np.zeros(max(B, 1), dtype=np.int32)
    _check(_load().oracle_count_paths(M, len(layers), bpl, ma, mb, S, B, T, threads, max_states, out, st),
           "count_paths")
    res = []
    for q in range(B):
        if st[q] != 0:
            res.append(None)
        else:
            res.append(int(out[2 * q]) | (int(out[2 * q + 1]) << 64))
    return res


def tvd(p, q) -> float:
    """Total variation distance."""
    return 0.5 * float(np.sum(np.abs(np.asarray(p) - np.asarray(q))))
