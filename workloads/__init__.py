"""Seeded synthetic inputs for the five BASELINE.json configs.

Input generation only -- shared by the tests, bench.py and smoke(), and
holding none of the method's arithmetic (no address map, no gather).  The
readings it implements (gate RNG, gate mix, ripple cascade, state seeds and
normalisation) are R6-R10 in DESIGN.md.

Gate lists are numpy uint8 arrays of shape (n, 4): (kind, target, c0, c1)
with kind 0 NOT, 1 CNOT, 2 CCNOT (Toffoli); bits are 0-based (bit b is
address bit a(b+1), a(1) the LSB); unused control slots hold 255.
Row 0 is Step 1 (applied first).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

NOT, CNOT, CCNOT = 0, 1, 2
Z, CZ, CCZ, SWAP = 3, 4, 5, 6      # phased permutations
UNUSED = 255
_NCTRL = {NOT: 0, CNOT: 1, CCNOT: 2, Z: 0, CZ: 1, CCZ: 2, SWAP: 1}

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "stategen.c")
_LIB_PATH = os.path.join(_HERE, "libqsim_gen.so")
_lib = None


# --------------------------------------------------------------------------
# gates
# --------------------------------------------------------------------------
def gate(kind: int, target: int, *controls: int) -> np.ndarray:
    """(kind, target, c0, c1); SWAP(a, b) is gate(SWAP, a, b)."""
    assert len(controls) == _NCTRL[kind], (kind, controls)
    c = list(controls) + [UNUSED] * (2 - len(controls))
    return np.array([kind, target, c[0], c[1]], dtype=np.uint8)


def gates_array(rows) -> np.ndarray:
    rows = [np.asarray(r, dtype=np.uint8) for r in rows]
    if not rows:
        return np.zeros((0, 4), dtype=np.uint8)
    return np.stack(rows).astype(np.uint8)


def random_gates(n: int, nbits: int, seed: int) -> np.ndarray:
    """Reading R6/R7: numpy PCG64 default_rng(seed); per gate kind ~ i.i.d.
    uniform over {NOT, CNOT, CCNOT}, then 1+kind distinct bits drawn
    uniformly from 0..nbits-1, the first being the target."""
    rng = np.random.default_rng(seed)
    rows = []
    for _ in range(n):
        kind = int(rng.integers(3))
        bits = rng.choice(nbits, size=1 + kind, replace=False)
        rows.append(gate(kind, int(bits[0]), *[int(b) for b in bits[1:]]))
    return gates_array(rows)


def random_gates_ext(n: int, nbits: int, seed: int,
                     kinds=(NOT, CNOT, CCNOT, Z, CZ, CCZ, SWAP)) -> np.ndarray:
    """Test circuits over the extended gate set: kind uniform over `kinds`,
    then 1 + (#controls) distinct bits, the first being the target."""
    rng = np.random.default_rng(seed)
    rows = []
    for _ in range(n):
        kind = int(kinds[int(rng.integers(len(kinds)))])
        bits = rng.choice(nbits, size=1 + _NCTRL[kind], replace=False)
        rows.append(gate(kind, int(bits[0]), *[int(b) for b in bits[1:]]))
    return gates_array(rows)


def ripple_gates(M: int, n: int) -> np.ndarray:
    """Reading R9: per j = 1..M-2 the block [CNOT(a(j) -> a(j+1)),
    CCNOT(a(j), a(j+1) -> a(j+2))] (arrow = control -> target), the pass
    repeated and truncated to n gates.  Deterministic, no RNG."""
    block = []
    for j0 in range(M - 2):                    # j = j0 + 1, 0-based bits
        block.append(gate(CNOT, j0 + 1, j0))
        block.append(gate(CCNOT, j0 + 2, j0, j0 + 1))
    rows = []
    while len(rows) < n:
        rows.extend(block[: n - len(rows)])
    return gates_array(rows)


def worked_step() -> np.ndarray:
    """P:L43 2(b): "In Step 1, a(1) is the target bit and a(2) is the
    controlling bit" -> CNOT(target bit 0, control bit 1)."""
    return gate(CNOT, 0, 1)


# --------------------------------------------------------------------------
# states
# --------------------------------------------------------------------------
def _load():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH) or (
                os.path.getmtime(_LIB_PATH) < os.path.getmtime(_SRC)):
            build()
        lib = ctypes.CDLL(_LIB_PATH)
        lib.gen_sumsq.restype = ctypes.c_double
        lib.gen_sumsq.argtypes = [ctypes.c_uint64, ctypes.c_int32, ctypes.c_uint64]
        lib.gen_fill.restype = None
        lib.gen_fill.argtypes = [ctypes.c_uint64, ctypes.c_int32, ctypes.c_double,
                                 ctypes.c_int32, ctypes.c_uint64, ctypes.c_uint64,
                                 ctypes.c_void_p]
        lib.gen_tagged.restype = None
        lib.gen_tagged.argtypes = [ctypes.c_int32, ctypes.c_uint64, ctypes.c_uint64,
                                   ctypes.c_void_p]
        _lib = lib
    return _lib


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB_PATH) or (
            os.path.getmtime(_LIB_PATH) < os.path.getmtime(_SRC)):
        tmp = _LIB_PATH + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c99", "-fopenmp", "-ffp-contract=off",
                               "-fPIC", "-shared", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


GAUSS, POLAR = 0, 1
_ELEM = {"c64": 8, "c128": 16}
NP_DTYPE = {"c64": np.complex64, "c128": np.complex128}


@dataclass(frozen=True)
class StateSpec:
    """Reading R10: counter-based generator keyed by state_seed; normalised."""
    M: int
    dtype: str          # "c64" | "c128"
    mode: int           # GAUSS | POLAR
    seed: int

    @property
    def N(self) -> int:
        return 1 << self.M

    def scale(self) -> float:
        return 1.0 / float(np.sqrt(_load().gen_sumsq(self.seed, self.mode, self.N)))


def fill_state(spec: StateSpec, out_ptr: int, start: int = 0, count: int | None = None,
               scale: float | None = None) -> None:
    """Write entries [start, start+count) of the normalised state to host memory."""
    if count is None:
        count = spec.N - start
    if scale is None:
        scale = spec.scale()
    _load().gen_fill(spec.seed, spec.mode, scale, _ELEM[spec.dtype], start, count, out_ptr)


def make_state(spec: StateSpec, start: int = 0, count: int | None = None,
               scale: float | None = None) -> np.ndarray:
    if count is None:
        count = spec.N - start
    out = np.empty(count, dtype=NP_DTYPE[spec.dtype])
    fill_state(spec, out.ctypes.data, start, count, scale)
    return out


def tagged_state(dtype: str, N: int, start: int = 0) -> np.ndarray:
    out = np.empty(N, dtype=NP_DTYPE[dtype])
    _load().gen_tagged(_ELEM[dtype], start, N, out.ctypes.data)
    return out


def fill_tagged(dtype: str, out_ptr: int, start: int, count: int) -> None:
    _load().gen_tagged(_ELEM[dtype], start, count, out_ptr)


def random_qubits(M: int, seed: int, dtype: str = "c64") -> np.ndarray:
    """M normalised qubits [q_j(0), q_j(1)] (Appendix 1), row j-1 = q_j:
    i.i.d. Gaussian complex pairs scaled to |q(0)|^2 + |q(1)|^2 = 1, rounded
    to the state dtype (the rounded values are the input both sides use)."""
    rng = np.random.default_rng(seed)
    z = rng.standard_normal((M, 2)) + 1j * rng.standard_normal((M, 2))
    z /= np.sqrt((np.abs(z) ** 2).sum(axis=1, keepdims=True))
    return z.astype(NP_DTYPE[dtype])


def basis_qubits(M: int, bit: int, dtype: str = "c64") -> np.ndarray:
    """Every qubit |bit>: [1, 0] for |0>, [0, 1] for |1> (P:L87 uses all |1>)."""
    q = np.zeros((M, 2), dtype=NP_DTYPE[dtype])
    q[:, bit] = 1
    return q


# --------------------------------------------------------------------------
# the five BASELINE.json configs (cfg1..cfg5 = configs[0..4])
# --------------------------------------------------------------------------
@dataclass(frozen=True)
class Config:
    name: str
    M: int
    dtype: str
    modes: tuple
    description: str
    gate_seed: int | None
    state: StateSpec

    def gates(self) -> np.ndarray:
        if self.name == "cfg1":                       # reading R8
            return gates_array([worked_step()] + list(random_gates(8, 3, 0)))
        if self.name == "cfg4":                       # reading R9
            return ripple_gates(30, 256)
        n = {"cfg2": 64, "cfg3": 256, "cfg5": 64}[self.name]
        return random_gates(n, self.M, self.gate_seed)

    @property
    def N(self) -> int:
        return 1 << self.M


CONFIGS = {
    "cfg1": Config("cfg1", 3, "c64", ("build", "apply", "fused"),
                   "M=3: worked step CNOT(t=a(1), c=a(2)) + 8 random gates (seed 0); "
                   "c64 |a|~U(0,1], arg~U(0,2pi), normalised", 0,
                   StateSpec(3, "c64", POLAR, 1000)),
    "cfg2": Config("cfg2", 20, "c64", ("build", "apply", "fused"),
                   "M=20: 64 random NOT/CNOT/CCNOT over bits 0..19 (seed 1); "
                   "c64 Gaussian normalised", 1, StateSpec(20, "c64", GAUSS, 1001)),
    "cfg3": Config("cfg3", 26, "c128", ("build", "apply"),
                   "M=26: 256 random gates over bits 0..25 (seed 2); c128 Gaussian "
                   "normalised; materialised map then gather", 2,
                   StateSpec(26, "c128", GAUSS, 1002)),
    "cfg4": Config("cfg4", 30, "c64", ("build", "apply", "fused"),
                   "M=30: 256-gate ripple cascade; c64 Gaussian normalised; fused vs "
                   "materialised", None, StateSpec(30, "c64", GAUSS, 1003)),
    "cfg5": Config("cfg5", 32, "c64", ("build", "apply", "fused"),
                   "M=32: 64 random gates over bits 0..31 (seed 4); c64 Gaussian "
                   "normalised; materialised and fused", 4,
                   StateSpec(32, "c64", GAUSS, 1004)),
}
