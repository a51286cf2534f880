"""CPU oracle for the Burger permutation-map hot path -- TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` leg may import this package.  The
product path (``paper_quant_ph_0308158_b200``) never imports it, and this
package never imports the product path: they share no code.

* ``qsim_oracle.c``  -- plain single-threaded C: step map (P:L43 2(b)),
  composite walk (readings R1/R2), materialised build, apply, fused, sampled
  walk and the paper's "basic accumulation method".
* ``dense.py``       -- textbook dense 2^M x 2^M matrices built from Kronecker
  products of 2x2 blocks (M <= 4), the brute-force pin the north star names.

Gate lists are numpy ``uint8`` arrays of shape (n, 4): kind, target,
control0, control1 (see ``workloads``); this module re-reads them on its own.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "qsim_oracle.c")
_LIB_PATH = os.path.join(_HERE, "libqsim_oracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile the oracle with plain ``gcc -O2`` (no OpenMP, no intrinsics)."""
    if force or not os.path.exists(_LIB_PATH) or (
            os.path.getmtime(_LIB_PATH) < os.path.getmtime(_SRC)):
        tmp = _LIB_PATH + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c99", "-fPIC", "-shared",
                               "-o", tmp, _SRC])
        os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB_PATH)
        u8p = ctypes.POINTER(ctypes.c_uint8)
        lib.oracle_step.restype = ctypes.c_uint64
        lib.oracle_step.argtypes = [u8p, ctypes.c_uint64]
        lib.oracle_walk.restype = ctypes.c_uint64
        lib.oracle_walk.argtypes = [u8p, ctypes.c_int32, ctypes.c_uint64]
        lib.oracle_build.restype = None
        lib.oracle_build.argtypes = [u8p, ctypes.c_int32, ctypes.c_uint64,
                                     ctypes.c_uint64, ctypes.c_void_p]
        lib.oracle_apply.restype = None
        lib.oracle_apply.argtypes = [ctypes.c_void_p, ctypes.c_uint64,
                                     ctypes.c_int32, ctypes.c_void_p,
                                     ctypes.c_void_p]
        lib.oracle_fused.restype = None
        lib.oracle_fused.argtypes = [u8p, ctypes.c_int32, ctypes.c_uint64,
                                     ctypes.c_uint64, ctypes.c_int32,
                                     ctypes.c_void_p, ctypes.c_void_p]
        lib.oracle_walk_many.restype = None
        lib.oracle_walk_many.argtypes = [u8p, ctypes.c_int32, ctypes.c_void_p,
                                         ctypes.c_uint64, ctypes.c_void_p]
        lib.oracle_build_signed.restype = None
        lib.oracle_build_signed.argtypes = [u8p, ctypes.c_int32, ctypes.c_uint64,
                                            ctypes.c_uint64, ctypes.c_void_p, ctypes.c_void_p]
        lib.oracle_apply_signed.restype = None
        lib.oracle_apply_signed.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint64,
                                            ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p]
        lib.oracle_walk_signed.restype = ctypes.c_uint64
        lib.oracle_walk_signed.argtypes = [u8p, ctypes.c_int32, ctypes.c_uint64,
                                           ctypes.POINTER(ctypes.c_int)]
        lib.oracle_kron_element.restype = None
        lib.oracle_kron_element.argtypes = [ctypes.c_void_p, ctypes.c_int32, ctypes.c_uint64,
                                            ctypes.c_void_p, ctypes.c_void_p]
        lib.oracle_fused_kron.restype = None
        lib.oracle_fused_kron.argtypes = [u8p, ctypes.c_int32, ctypes.c_int32, ctypes.c_void_p,
                                          ctypes.c_uint64, ctypes.c_uint64, ctypes.c_void_p]
        lib.oracle_accumulate.restype = None
        lib.oracle_accumulate.argtypes = [u8p, ctypes.c_int32, ctypes.c_int32,
                                          ctypes.c_int32, ctypes.c_void_p]
        _lib = lib
    return _lib


def _gates_arg(gates):
    g = np.ascontiguousarray(np.asarray(gates, dtype=np.uint8).reshape(-1, 4))
    ptr = g.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8))
    return g, ptr, int(g.shape[0])


def _elem_bytes(arr: np.ndarray) -> int:
    if arr.dtype == np.complex64:
        return 8
    if arr.dtype == np.complex128:
        return 16
    raise TypeError(f"state dtype must be complex64/complex128, got {arr.dtype}")


def step(gate, x: int) -> int:
    """One wiring-diagram step on one address, P:L43 2(b)."""
    g, ptr, _ = _gates_arg(gate)
    return int(_load().oracle_step(ptr, x))


def walk(gates, i: int) -> int:
    """perm[i] = f_1(f_2(...f_n(i))) (readings R1, R2)."""
    g, ptr, n = _gates_arg(gates)
    return int(_load().oracle_walk(ptr, n, i))


def build_map(gates, M: int, start: int = 0, count: int | None = None) -> np.ndarray:
    """Materialised composite gather permutation, uint32, entries [start, start+count)."""
    N = 1 << M
    if count is None:
        count = N - start
    g, ptr, n = _gates_arg(gates)
    perm = np.empty(count, dtype=np.uint32)
    _load().oracle_build(ptr, n, start, count, perm.ctypes.data)
    return perm


def build_map_signed(gates, M: int, start: int = 0, count: int | None = None):
    """(perm, signs): phased permutation (reading R17); bit r % 32 of
    signs[r // 32] is 1 when row start + r holds -1."""
    N = 1 << M
    if count is None:
        count = N - start
    g, ptr, n = _gates_arg(gates)
    perm = np.empty(count, dtype=np.uint32)
    signs = np.empty(max((count + 31) // 32, 1), dtype=np.uint32)
    _load().oracle_build_signed(ptr, n, start, count, perm.ctypes.data, signs.ctypes.data)
    return perm, signs


def walk_signed(gates, i: int):
    g, ptr, n = _gates_arg(gates)
    s = ctypes.c_int()
    x = _load().oracle_walk_signed(ptr, n, i, ctypes.byref(s))
    return int(x), int(s.value)


def apply_map_signed(perm: np.ndarray, signs: np.ndarray, k1: np.ndarray) -> np.ndarray:
    """k2[i] = sign[i] * k1[perm[i]] (IEEE negation for -1)."""
    perm = np.ascontiguousarray(perm, dtype=np.uint32)
    signs = np.ascontiguousarray(signs, dtype=np.uint32)
    k1 = np.ascontiguousarray(k1)
    k2 = np.empty(perm.shape[0], dtype=k1.dtype)
    _load().oracle_apply_signed(perm.ctypes.data, signs.ctypes.data, perm.shape[0],
                                _elem_bytes(k1), k1.ctypes.data, k2.ctypes.data)
    return k2


def apply_map(perm: np.ndarray, k1: np.ndarray) -> np.ndarray:
    """k2[i] = k1[perm[i]] (reading R2), bytes copied."""
    perm = np.ascontiguousarray(perm, dtype=np.uint32)
    k1 = np.ascontiguousarray(k1)
    k2 = np.empty(perm.shape[0], dtype=k1.dtype)
    _load().oracle_apply(perm.ctypes.data, perm.shape[0], _elem_bytes(k1),
                         k1.ctypes.data, k2.ctypes.data)
    return k2


def run_fused(gates, k1: np.ndarray, start: int = 0, count: int | None = None) -> np.ndarray:
    """k2[start:start+count] with the map recomputed per entry."""
    k1 = np.ascontiguousarray(k1)
    if count is None:
        count = k1.shape[0] - start
    g, ptr, n = _gates_arg(gates)
    out = np.empty(count, dtype=k1.dtype)
    _load().oracle_fused(ptr, n, start, count, _elem_bytes(k1), k1.ctypes.data,
                         out.ctypes.data)
    return out


def walk_many(gates, idx) -> np.ndarray:
    """perm at the sampled output indices idx (uint64)."""
    idx = np.ascontiguousarray(np.asarray(idx, dtype=np.uint64))
    g, ptr, n = _gates_arg(gates)
    out = np.empty(idx.shape[0], dtype=np.uint64)
    _load().oracle_walk_many(ptr, n, idx.ctypes.data, idx.shape[0], out.ctypes.data)
    return out


def accumulate(gates, k1: np.ndarray) -> np.ndarray:
    """The paper's "basic accumulation method": gate-by-gate swaps."""
    k = np.array(k1, copy=True, order="C")
    M = int(k.shape[0]).bit_length() - 1
    assert (1 << M) == k.shape[0]
    g, ptr, n = _gates_arg(gates)
    _load().oracle_accumulate(ptr, n, M, _elem_bytes(k), k.ctypes.data)
    return k


def _qubits_arg(qubits) -> np.ndarray:
    """(M, 2) complex array -> 4M doubles: re/im of q_j(0), q_j(1), j = 1..M."""
    q = np.asarray(qubits, dtype=np.complex128).reshape(-1, 2)
    return np.ascontiguousarray(q.view(np.float64).reshape(-1))


def kron_element(qubits, i: int) -> complex:
    """k_1(i) = q_M(b_M) ... q_1(b_1) (Appendix 1), double precision."""
    q = _qubits_arg(qubits)
    M = q.shape[0] // 4
    re, im = ctypes.c_double(), ctypes.c_double()
    _load().oracle_kron_element(q.ctypes.data, M, i, ctypes.byref(re), ctypes.byref(im))
    return complex(re.value, im.value)


def fused_kron(gates, qubits, start: int = 0, count: int | None = None) -> np.ndarray:
    """k2[i] = k_1(perm[i]) with k_1 generated on the fly (complex128)."""
    q = _qubits_arg(qubits)
    M = q.shape[0] // 4
    if count is None:
        count = (1 << M) - start
    g, ptr, n = _gates_arg(gates)
    out = np.empty(count, dtype=np.complex128)
    _load().oracle_fused_kron(ptr, n, M, q.ctypes.data, start, count, out.ctypes.data)
    return out
