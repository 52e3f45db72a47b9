"""Python binding of liblofp (include/lofp.h): argument marshalling only.

Every step of the path sum runs in the CUDA library; PyTorch is used here only for
device memory (the output buffer) and the current CUDA stream.  There is no CPU
fallback: if liblofp.so is missing this module raises on import.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("LOFP_LIB") or os.path.join(_HERE, "liblofp.so")

LOFP_OK, LOFP_E_INVALID_ARG, LOFP_E_UNSUPPORTED, LOFP_E_CUDA, LOFP_E_OOM, LOFP_E_BAD_OUTPUT = range(6)


class lofp_bs(ctypes.Structure):
    _fields_ = [("mode_a", ctypes.c_int32), ("mode_b", ctypes.c_int32),
                ("theta", ctypes.c_double), ("phi", ctypes.c_double)]


class lofp_gate(ctypes.Structure):
    _fields_ = [("mode", ctypes.c_int32), ("after_layer", ctypes.c_int32),
                ("a", ctypes.c_double), ("b", ctypes.c_double)]


class lofp_run_stats(ctypes.Structure):
    _fields_ = [("batch", ctypes.c_int64), ("feasible", ctypes.c_int64), ("paths", ctypes.c_int64),
                ("cmuls", ctypes.c_int64), ("units", ctypes.c_int64), ("subsplits", ctypes.c_int64),
                ("pairs", ctypes.c_int64), ("elements", ctypes.c_int64), ("unsupported", ctypes.c_int64),
                ("bad_rows", ctypes.c_int64), ("check_errors", ctypes.c_int64), ("max_states", ctypes.c_int64),
                ("max_list", ctypes.c_int64), ("table_entries", ctypes.c_int64), ("terms", ctypes.c_int64),
                ("over_budget", ctypes.c_int64), ("generic", ctypes.c_int64),
                ("phase_cycles", ctypes.c_int64 * 8), ("tile_cycles", ctypes.c_int64 * 2),
                ("grid_blocks", ctypes.c_int32), ("block_threads", ctypes.c_int32),
                ("launches", ctypes.c_int32), ("mode", ctypes.c_int32),
                ("units_ms", ctypes.c_float), ("total_ms", ctypes.c_float),
                ("contract_deferred", ctypes.c_int64)]


EXPORTS = ["lofp_create", "lofp_create_ex", "lofp_amplitudes", "lofp_amplitudes_counted", "lofp_amplitudes_contract",
           "lofp_distribution", "lofp_set_path_budget", "lofp_amplitudes_host",
           "lofp_destroy", "lofp_status_string", "lofp_last_error", "lofp_stats"]


def _load():
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} is not built: run `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = ctypes.CDLL(LIB_PATH)
    P = ctypes.c_void_p
    lib.lofp_create.argtypes = [ctypes.c_int32, ctypes.c_int32, ctypes.POINTER(ctypes.c_int32),
                                ctypes.POINTER(lofp_bs), ctypes.POINTER(P)]
    lib.lofp_create.restype = ctypes.c_int
    lib.lofp_create_ex.argtypes = [ctypes.c_int32, ctypes.c_int32, ctypes.POINTER(ctypes.c_int32),
                                   ctypes.POINTER(lofp_bs), ctypes.c_int32, ctypes.POINTER(lofp_gate),
                                   ctypes.POINTER(P)]
    lib.lofp_create_ex.restype = ctypes.c_int
    lib.lofp_amplitudes.argtypes = [P, ctypes.POINTER(ctypes.c_int32), ctypes.c_int64, P, P, P]
    lib.lofp_amplitudes.restype = ctypes.c_int
    lib.lofp_amplitudes_counted.argtypes = [P, ctypes.POINTER(ctypes.c_int32), ctypes.c_int64, P, P, P, P]
    lib.lofp_amplitudes_counted.restype = ctypes.c_int
    lib.lofp_amplitudes_contract.argtypes = [P, ctypes.POINTER(ctypes.c_int32), ctypes.c_int64, P, P, P, P]
    lib.lofp_amplitudes_contract.restype = ctypes.c_int
    lib.lofp_distribution.argtypes = [P, ctypes.POINTER(ctypes.c_int32), ctypes.c_int64, P, P,
                                      ctypes.POINTER(ctypes.c_int64), ctypes.c_int32, P]
    lib.lofp_distribution.restype = ctypes.c_int
    lib.lofp_set_path_budget.argtypes = [P, ctypes.c_uint64]
    lib.lofp_set_path_budget.restype = ctypes.c_int
    lib.lofp_amplitudes_host.argtypes = [P, ctypes.POINTER(ctypes.c_int32), ctypes.c_int64, P, P]
    lib.lofp_amplitudes_host.restype = ctypes.c_int
    lib.lofp_destroy.argtypes = [P]
    lib.lofp_destroy.restype = None
    lib.lofp_status_string.argtypes = [ctypes.c_int]
    lib.lofp_status_string.restype = ctypes.c_char_p
    lib.lofp_last_error.argtypes = [P]
    lib.lofp_last_error.restype = ctypes.c_char_p
    lib.lofp_stats.argtypes = [P, ctypes.POINTER(lofp_run_stats)]
    lib.lofp_stats.restype = ctypes.c_int
    return lib


_lib = _load()


class LofpError(RuntimeError):
    def __init__(self, status: int, msg: str):
        self.status = status
        super().__init__(f"{_lib.lofp_status_string(status).decode()}: {msg}")


def _occ(S, M):
    s = np.ascontiguousarray(np.asarray(S, dtype=np.int32))
    if s.shape != (M,):
        raise ValueError(f"input occupation must have {M} entries")
    return s


class Circuit:
    """A mesh of beam splitters: ``layers`` is a list of layers, each a list of
    ``(mode_a, mode_b, theta, phi)`` (mode_a = BS port 1).  ``gates``: optional phase
    gates ``(mode, after_layer, a, b)`` multiplying |n> of that mode by exp(i (a n + b n^2))
    (P:338)."""

    def __init__(self, modes: int, layers, gates=()):
        self.modes = int(modes)
        self.layers = [list(l) for l in layers]
        self.gates = [tuple(g) for g in gates]
        flat = [bs for l in self.layers for bs in l]
        bpl = (ctypes.c_int32 * max(len(self.layers), 1))(*[len(l) for l in self.layers])
        arr = (lofp_bs * max(len(flat), 1))(*[lofp_bs(int(a), int(b), float(t), float(p)) for a, b, t, p in flat])
        garr = (lofp_gate * max(len(self.gates), 1))(*[lofp_gate(int(m), int(j), float(a), float(b))
                                                        for m, j, a, b in self.gates])
        h = ctypes.c_void_p()
        st = _lib.lofp_create_ex(self.modes, len(self.layers), bpl, arr, len(self.gates), garr, ctypes.byref(h))
        if st != LOFP_OK:
            raise LofpError(st, "lofp_create failed")
        self._h = h
        self.device_index = None  # the CUDA device the context lives on (set on first use)
        try:
            import torch
            if torch.cuda.is_available():
                self.device_index = torch.cuda.current_device()
        except ImportError:
            pass

    def close(self):
        if getattr(self, "_h", None):
            _lib.lofp_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, st):
        if st != LOFP_OK:
            raise LofpError(st, _lib.lofp_last_error(self._h).decode())

    def _out(self, T, out):
        import torch
        if T.dtype != torch.int32 or not T.is_cuda or T.dim() != 2 or T.shape[1] != self.modes:
            raise ValueError("T must be an int32 CUDA tensor of shape [B, modes]")
        if self.device_index is not None and T.device.index != self.device_index:
            raise ValueError(f"T is on {T.device}, the circuit on cuda:{self.device_index}")
        B = T.shape[0]
        if out is None:
            out = torch.empty((B, 2), dtype=torch.float64, device=T.device)
        elif (out.dtype != torch.float64 or tuple(out.shape) != (B, 2) or not out.is_contiguous()
              or out.device != T.device):
            raise ValueError("out must be a contiguous float64 tensor [B, 2] on T's device")
        return out

    def amplitudes(self, S, T, out=None, counts=None, stream=None):
        """<T_b|U_P|S> for every row of the int32 CUDA tensor T [B, M] -> complex128 CUDA [B].

        ``counts``: optional int64 CUDA tensor [B] receiving the number of path products
        formed per output (= the exact number of valid paths).  Runs on ``stream``
        (default: torch's current stream); the result is ready when that stream is.
        """
        import torch
        T = T.contiguous()
        out = self._out(T, out)
        B = T.shape[0]
        s = _occ(S, self.modes)
        strm = (stream or torch.cuda.current_stream(T.device)).cuda_stream
        sp = s.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))
        with torch.cuda.device(T.device):
            if counts is None:
                st = _lib.lofp_amplitudes(self._h, sp, B, ctypes.c_void_p(T.data_ptr()),
                                          ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(strm))
            else:
                if counts.dtype != torch.int64 or counts.numel() != B or not counts.is_cuda or \
                        counts.device != T.device or not counts.is_contiguous():
                    raise ValueError("counts must be a contiguous int64 CUDA tensor [B] on T's device")
                st = _lib.lofp_amplitudes_counted(self._h, sp, B, ctypes.c_void_p(T.data_ptr()),
                                                  ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(counts.data_ptr()),
                                                  ctypes.c_void_p(strm))
        self._check(st)
        return torch.view_as_complex(out)

    def contract(self, S, T, out=None, counts=None, stream=None):
        """The same amplitudes by the strip tensor contraction: work per output
        scales with the light-cone state space, not the number of paths.  ``counts``
        (optional int64 CUDA tensor [B]) receives the exact number of valid paths."""
        import torch
        T = T.contiguous()
        out = self._out(T, out)
        B = T.shape[0]
        s = _occ(S, self.modes)
        strm = (stream or torch.cuda.current_stream(T.device)).cuda_stream
        cp = None
        if counts is not None:
            if counts.dtype != torch.int64 or counts.numel() != B or counts.device != T.device or \
                    not counts.is_contiguous():
                raise ValueError("counts must be a contiguous int64 CUDA tensor [B] on T's device")
            cp = ctypes.c_void_p(counts.data_ptr())
        with torch.cuda.device(T.device):
            st = _lib.lofp_amplitudes_contract(self._h, s.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), B,
                                               ctypes.c_void_p(T.data_ptr()), ctypes.c_void_p(out.data_ptr()),
                                               cp, ctypes.c_void_p(strm))
        self._check(st)
        return torch.view_as_complex(out)

    def distribution(self, S, method: str = "contract", device=None, stream=None):
        """Every output pattern of sum(S) photons and its amplitude, computed in one
        call: returns (T int32 CUDA [count, M], amplitudes complex128 CUDA [count])."""
        import torch
        s = _occ(S, self.modes)
        sp = s.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))
        dev = torch.device("cuda", self.device_index if device is None else device)
        n = ctypes.c_int64(0)
        _lib.lofp_distribution(self._h, sp, 0, None, None, ctypes.byref(n), 0, None)  # count only
        count = int(n.value)
        if count <= 0:
            self._check(_lib.lofp_distribution(self._h, sp, 0, None, None, ctypes.byref(n), 0, None))
        T = torch.empty((count, self.modes), dtype=torch.int32, device=dev)
        out = torch.empty((count, 2), dtype=torch.float64, device=dev)
        strm = (stream or torch.cuda.current_stream(dev)).cuda_stream
        with torch.cuda.device(dev):
            st = _lib.lofp_distribution(self._h, sp, count, ctypes.c_void_p(T.data_ptr()),
                                        ctypes.c_void_p(out.data_ptr()), ctypes.byref(n),
                                        0 if method == "contract" else 1, ctypes.c_void_p(strm))
        self._check(st)
        return T, torch.view_as_complex(out)

    def set_path_budget(self, max_paths_per_output: int = 0):
        """Skip (NaN) outputs with more valid paths than this in path-sum calls; 0 = no limit."""
        self._check(_lib.lofp_set_path_budget(self._h, int(max_paths_per_output)))

    def amplitudes_host(self, S, T) -> np.ndarray:
        """End-to-end call with host buffers (numpy in, numpy out)."""
        s = _occ(S, self.modes)
        t = np.ascontiguousarray(np.asarray(T, dtype=np.int32))
        if t.ndim != 2 or t.shape[1] != self.modes:
            raise ValueError("T must have shape [B, modes]")
        out = np.empty((t.shape[0], 2), dtype=np.float64)
        st = _lib.lofp_amplitudes_host(self._h, s.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), t.shape[0],
                                       ctypes.c_void_p(t.ctypes.data), ctypes.c_void_p(out.ctypes.data))
        self._check(st)
        return out.view(np.complex128)[:, 0]

    def stats(self) -> dict:
        st = lofp_run_stats()
        rc = _lib.lofp_stats(self._h, ctypes.byref(st))
        if rc not in (LOFP_OK, LOFP_E_BAD_OUTPUT):
            self._check(rc)
        d = {k: getattr(st, k) for k, _ in lofp_run_stats._fields_}
        d["phase_cycles"] = list(st.phase_cycles)
        d["tile_cycles"] = list(st.tile_cycles)
        d["status"] = rc
        return d
