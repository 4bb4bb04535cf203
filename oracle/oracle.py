"""ctypes bindings for the CPU checkers -- TEST INFRASTRUCTURE ONLY.

* ``Oracle``    -> oracle/liboracle.so, our C restatement (tf_oracle.c) of the
  reference arithmetic (proj/include/tilefabric/{common,tilemath,reference}.hpp).
* ``Reference`` -> oracle/_ref/libtfref.so, the reference headers compiled
  unmodified (oracle/Makefile).  It pins the restatement and is the CPU
  baseline arm of bench.py.

Parity status: pinned.  tests/test_oracle_golden.py checks the restatement
bit-for-bit against the reference build and against the golden values in
tests/golden/ (which were produced by the reference's own code; see
tests/golden/make_golden.py).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_F = np.ctypeslib.ndpointer(dtype=np.float32, flags="C_CONTIGUOUS")
_U64 = np.ctypeslib.ndpointer(dtype=np.uint64, flags="C_CONTIGUOUS")


def build() -> None:
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def _load(path: str) -> C.CDLL:
    if not os.path.exists(path):
        build()
    return C.CDLL(path)


class Oracle:
    """Restated reference math (tf_oracle.c)."""

    def __init__(self) -> None:
        L = self.lib = _load(os.path.join(HERE, "liboracle.so"))
        L.tfo_uniform_reals.argtypes = [C.c_uint64, C.c_size_t, _F]
        L.tfo_gemm.argtypes = [_F, _F, C.c_size_t, C.c_size_t, C.c_size_t, _F]
        L.tfo_gemm_rows.argtypes = [_F, _F, C.c_size_t, C.c_size_t, C.c_size_t, C.c_size_t, _F]
        L.tfo_attention.argtypes = [_F, _F, _F, C.c_size_t, C.c_size_t, C.c_size_t, C.c_float, _F, _F]
        L.tfo_attention_partial_wire.argtypes = [_F, _F, _F, C.c_int, C.c_int, C.c_size_t, C.c_float, _F]
        L.tfo_attention_partial_wire.restype = C.c_longlong
        L.tfo_combine_wire.argtypes = [_F, _F, C.c_int, C.c_int]
        L.tfo_finalize_wire.argtypes = [_F, C.c_int, C.c_int, _F]
        L.tfo_finalize_wire.restype = C.c_int
        L.tfo_neutral_wire.argtypes = [_F, C.c_int, C.c_int]
        L.tfo_fd_world.argtypes = [_F, _F, _F, C.c_int, C.c_int, C.c_size_t, C.c_float, C.c_int, _F, _F, _F]
        L.tfo_fd_world.restype = C.c_int
        L.tfo_max_head_relative_error.argtypes = [_F, _F, C.c_int, C.c_int]
        L.tfo_max_head_relative_error.restype = C.c_double
        L.tfo_fnv1a64.argtypes = [C.c_void_p, C.c_size_t]
        L.tfo_fnv1a64.restype = C.c_uint64
        L.tfo_round_bf16.argtypes = [_F, C.c_size_t, C.c_void_p, C.c_void_p]

    # common.hpp:132-140
    def uniform_reals(self, seed: int, n: int) -> np.ndarray:
        out = np.empty(n, np.float32)
        self.lib.tfo_uniform_reals(seed, n, out)
        return out

    # ag_gemm.hpp:71-83 -- A (m x k) first, then B (k x n), one stream
    def ag_problem(self, seed: int, m: int, n: int, k: int):
        v = self.uniform_reals(seed, m * k + k * n)
        return v[: m * k].reshape(m, k).copy(), v[m * k:].reshape(k, n).copy()

    # flash_decode.hpp:90-106 -- q, then K, then V
    def fd_problem(self, seed: int, heads: int, d: int, L: int):
        hd = heads * d
        v = self.uniform_reals(seed, hd + 2 * hd * L)
        q = v[:hd].reshape(heads, d).copy()
        k = v[hd: hd + hd * L].reshape(heads, L, d).copy()
        vv = v[hd + hd * L:].reshape(heads, L, d).copy()
        return q, k, vv, np.float32(1.0 / np.sqrt(np.float32(d)))

    def gemm(self, a: np.ndarray, b: np.ndarray) -> np.ndarray:
        m, k = a.shape
        n = b.shape[1]
        c = np.empty((m, n), np.float32)
        self.lib.tfo_gemm(np.ascontiguousarray(a, np.float32).ravel(),
                          np.ascontiguousarray(b, np.float32).ravel(), m, n, k, c.ravel())
        return c

    def gemm_rows(self, a: np.ndarray, b: np.ndarray, rows) -> np.ndarray:
        """Full-K reference rows for a sampled row set."""
        rows = np.asarray(rows)
        return self.gemm(np.ascontiguousarray(a[rows]), b)

    def attention(self, q, k, v, scale) -> np.ndarray:
        h, L, d = k.shape
        out = np.empty((h, d), np.float32)
        scratch = np.empty(L, np.float32)
        self.lib.tfo_attention(_c(q), _c(k), _c(v), h, d, L, float(scale), out.ravel(), scratch)
        return out

    def partial_wire(self, q, k, v, scale) -> np.ndarray:
        h, L, d = k.shape
        wire = np.empty((h, d + 2), np.float32)
        bad = self.lib.tfo_attention_partial_wire(_c(q), _c(k), _c(v), h, d, L, float(scale), wire.ravel())
        if bad:
            raise FloatingPointError(f"non-finite score at flat index {bad - 1}")
        return wire

    def neutral_wire(self, heads: int, d: int) -> np.ndarray:
        w = np.empty((heads, d + 2), np.float32)
        self.lib.tfo_neutral_wire(w.ravel(), heads, d)
        return w

    def combine_wire(self, acc: np.ndarray, x: np.ndarray) -> np.ndarray:
        acc = np.ascontiguousarray(acc, np.float32).copy()
        h, d2 = acc.shape
        self.lib.tfo_combine_wire(acc.ravel(), _c(x), h, d2 - 2)
        return acc

    def finalize_wire(self, acc: np.ndarray) -> np.ndarray:
        h, d2 = acc.shape
        out = np.empty((h, d2 - 2), np.float32)
        rc = self.lib.tfo_finalize_wire(_c(acc), h, d2 - 2, out.ravel())
        if rc:
            raise ZeroDivisionError(f"finalize: head {rc - 1} has an empty normalizer")
        return out

    def fd_world(self, q, k, v, scale, world: int):
        """fd::run_fused's math (flash_decode.hpp:140-180, 348-423): per-source
        wire rows (the inbox, W x H x (d+2)) and the folded output (H x d)."""
        h, L, d = k.shape
        wires = np.empty((world + 1, h, d + 2), np.float32)
        scratch = np.empty(2 * h * (L // world) * d, np.float32)
        out = np.empty((h, d), np.float32)
        rc = self.lib.tfo_fd_world(_c(q), _c(k), _c(v), h, d, L, float(scale), world,
                                   wires.ravel(), scratch, out.ravel())
        if rc:
            raise ArithmeticError(f"tfo_fd_world rc={rc}")
        return wires[:world].copy(), out

    def head_rel_err(self, a, b) -> float:
        a = np.ascontiguousarray(a, np.float32)
        b = np.ascontiguousarray(b, np.float32)
        h, d = a.shape[-2], a.shape[-1]
        a2 = a.reshape(-1, d)
        b2 = b.reshape(-1, d)
        return float(self.lib.tfo_max_head_relative_error(a2.ravel(), b2.ravel(), a2.shape[0], d))

    def fnv(self, arr: np.ndarray) -> str:
        arr = np.ascontiguousarray(arr)
        return "%016x" % self.lib.tfo_fnv1a64(arr.ctypes.data, arr.nbytes)

    def round_bf16(self, x: np.ndarray):
        """RNE to bf16: returns (fp32 widened copy, uint16 bits)."""
        x = np.ascontiguousarray(x, np.float32)
        f = np.empty_like(x)
        u = np.empty(x.shape, np.uint16)
        self.lib.tfo_round_bf16(x.ravel(), x.size, f.ctypes.data, u.ctypes.data)
        return f, u


def _c(x) -> np.ndarray:
    return np.ascontiguousarray(x, np.float32).ravel()


class Reference:
    """The reference headers themselves (oracle/_ref/libtfref.so)."""

    PATH = os.path.join(HERE, "_ref", "libtfref.so")

    @classmethod
    def available(cls) -> bool:
        return os.path.exists(cls.PATH)

    def __init__(self) -> None:
        L = self.lib = C.CDLL(self.PATH)
        L.tfr_last_error.restype = C.c_char_p
        L.tfr_uniform_reals.argtypes = [C.c_uint64, C.c_size_t, _F]
        L.tfr_ag_run.argtypes = [C.c_int, C.c_uint64, C.c_size_t, C.c_size_t, C.c_size_t,
                                 C.c_size_t, C.c_size_t, C.c_size_t, C.c_int, C.c_int64,
                                 C.c_void_p, C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_double)]
        L.tfr_ag_run_inputs.argtypes = [C.c_int, _F, _F, C.c_size_t, C.c_size_t, C.c_size_t,
                                        C.c_size_t, C.c_size_t, C.c_size_t, C.c_int, C.c_void_p,
                                        C.POINTER(C.c_double), C.POINTER(C.c_double)]
        L.tfr_fd_run.argtypes = [C.c_int, C.c_uint64, C.c_int, C.c_int, C.c_size_t, C.c_int,
                                 C.c_int64, C.c_void_p, C.c_void_p, C.POINTER(C.c_double),
                                 C.POINTER(C.c_double)]
        L.tfr_fd_run_inputs.argtypes = [C.c_int, _F, _F, _F, C.c_int, C.c_int, C.c_size_t,
                                        C.c_float, C.c_int, C.c_void_p, C.POINTER(C.c_double),
                                        C.POINTER(C.c_double)]
        L.tfr_gemm.argtypes = [_F, _F, C.c_size_t, C.c_size_t, C.c_size_t, _F]
        L.tfr_attention.argtypes = [_F, _F, _F, C.c_size_t, C.c_size_t, C.c_size_t, C.c_float, _F]
        L.tfr_attention_partial_wire.argtypes = [_F, _F, _F, C.c_int, C.c_int, C.c_size_t, C.c_float, _F]
        L.tfr_combine_wire.argtypes = [_F, _F, C.c_int, C.c_int]
        L.tfr_finalize_wire.argtypes = [_F, C.c_int, C.c_int, _F]
        L.tfr_max_head_relative_error.argtypes = [_F, _F, C.c_int, C.c_int]
        L.tfr_max_head_relative_error.restype = C.c_double
        L.tfr_hardware_concurrency.restype = C.c_uint

    def _check(self, rc: int) -> None:
        if rc:
            raise RuntimeError(f"reference rc={rc}: {self.lib.tfr_last_error().decode()}")

    def uniform_reals(self, seed: int, n: int) -> np.ndarray:
        out = np.empty(n, np.float32)
        self._check(self.lib.tfr_uniform_reals(seed, n, out))
        return out

    def ag_run(self, variant: int, seed: int, m: int, n: int, k: int, world: int,
               tiles=(16, 16, 16), launch_cost_ns: int = 0):
        """ag::run_{baseline,pull,push}(make_problem(seed, m, n, k, tiles));
        returns (C per rank [W, m, n], flag counts per rank or None, makespan_ns, post_ns)."""
        c = np.empty((world, m, n), np.float32)
        kw = k // world
        n_kb = (kw + tiles[2] - 1) // tiles[2]
        flags = np.zeros((world, world * n_kb), np.uint64) if variant == 2 else None
        ms, post = C.c_double(), C.c_double()
        self._check(self.lib.tfr_ag_run(variant, seed, m, n, k, *tiles, world, launch_cost_ns,
                                        c.ctypes.data, flags.ctypes.data if flags is not None else None,
                                        C.byref(ms), C.byref(post)))
        return c, flags, ms.value, post.value

    def ag_run_inputs(self, variant: int, a, b, world: int, tiles=(16, 16, 16)):
        m, k = a.shape
        n = b.shape[1]
        c = np.empty((m, n), np.float32)
        ms, post = C.c_double(), C.c_double()
        self._check(self.lib.tfr_ag_run_inputs(variant, _c(a), _c(b), m, n, k, *tiles, world,
                                               c.ctypes.data, C.byref(ms), C.byref(post)))
        return c, ms.value, post.value

    def fd_run(self, variant: int, seed: int, heads: int, d: int, L: int, world: int,
               launch_cost_ns: int = 0):
        out = np.empty((world, heads, d), np.float32)
        flags = np.zeros((world, world), np.uint64)
        ms, post = C.c_double(), C.c_double()
        self._check(self.lib.tfr_fd_run(variant, seed, heads, d, L, world, launch_cost_ns,
                                        out.ctypes.data, flags.ctypes.data, C.byref(ms), C.byref(post)))
        return out, flags, ms.value, post.value

    def fd_run_inputs(self, variant: int, q, k, v, scale, world: int):
        h, L, d = k.shape
        out = np.empty((h, d), np.float32)
        ms, post = C.c_double(), C.c_double()
        self._check(self.lib.tfr_fd_run_inputs(variant, _c(q), _c(k), _c(v), h, d, L, float(scale),
                                               world, out.ctypes.data, C.byref(ms), C.byref(post)))
        return out, ms.value, post.value

    def gemm(self, a, b) -> np.ndarray:
        m, k = a.shape
        n = b.shape[1]
        c = np.empty((m, n), np.float32)
        self._check(self.lib.tfr_gemm(_c(a), _c(b), m, n, k, c.ravel()))
        return c

    def attention(self, q, k, v, scale) -> np.ndarray:
        h, L, d = k.shape
        out = np.empty((h, d), np.float32)
        self._check(self.lib.tfr_attention(_c(q), _c(k), _c(v), h, d, L, float(scale), out.ravel()))
        return out

    def partial_wire(self, q, k, v, scale) -> np.ndarray:
        h, L, d = k.shape
        w = np.empty((h, d + 2), np.float32)
        self._check(self.lib.tfr_attention_partial_wire(_c(q), _c(k), _c(v), h, d, L, float(scale), w.ravel()))
        return w

    def combine_wire(self, acc, x) -> np.ndarray:
        acc = np.ascontiguousarray(acc, np.float32).copy()
        h, d2 = acc.shape
        self._check(self.lib.tfr_combine_wire(acc.ravel(), _c(x), h, d2 - 2))
        return acc

    def head_rel_err(self, a, b) -> float:
        d = a.shape[-1]
        a2 = np.ascontiguousarray(a, np.float32).reshape(-1, d)
        b2 = np.ascontiguousarray(b, np.float32).reshape(-1, d)
        return float(self.lib.tfr_max_head_relative_error(a2.ravel(), b2.ravel(), a2.shape[0], d))
