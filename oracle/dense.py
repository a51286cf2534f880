"""Dense brute-force matrices for tiny M -- TEST INFRASTRUCTURE (see oracle/).

The north star asks for "brute-force dense 2^M x 2^M matrix products for
M <= 4".  These matrices are assembled the textbook way, from Kronecker
products of 2x2 blocks -- not from the address bit-trick in qsim_oracle.c --
so that a wrong sign, index or transposition in either construction shows up
as a disagreement.

Ordering (Appendix 1): a state is q_M (x) ... (x) q_1, so the factor
for address bit a(j) (0-based bit j-1) is the (M-j)-th factor from the left,
and a(1) is the LSB.

Controlled-X on target t with control set C:
    U = I - P_C + P_C X_t,   P_C = prod_{c in C} |1><1|_c
which for C = {} is X_t (NOT), for |C| = 1 the CNOT and for |C| = 2 the
Toffoli.  Each step matrix is real, non-negative, symmetric, with one unity
per row.  The composite is U_n ... U_1 with Step 1 applied first
(reading R1) and k2 = U k1.
"""
from __future__ import annotations

import numpy as np

_I2 = np.eye(2)
_X = np.array([[0.0, 1.0], [1.0, 0.0]])
_P1 = np.array([[0.0, 0.0], [0.0, 1.0]])


def _on_bits(M: int, factors: dict) -> np.ndarray:
    """Kronecker product with factors[b] on 0-based bit b (identity elsewhere)."""
    out = np.ones((1, 1))
    for b in range(M - 1, -1, -1):          # q_M first, q_1 last
        out = np.kron(out, factors.get(b, _I2))
    return out


_P0 = np.array([[1.0, 0.0], [0.0, 0.0]])
_S01 = np.array([[0.0, 1.0], [0.0, 0.0]])   # |0><1|
_S10 = np.array([[0.0, 0.0], [1.0, 0.0]])   # |1><0|


def step_matrix(gate, M: int) -> np.ndarray:
    """Bit-flip kinds 0-2: I - P_C + P_C X_t.  Phase kinds 3-5 (Z, CZ, CCZ):
    I - 2 P_{C + t} (diagonal, -1 where the target and all controls are 1).
    SWAP (6) on bits (t, c0): |00><00| + |11><11| + |01><10| + |10><01|."""
    kind, target, c0, c1 = (int(v) for v in gate)
    if kind <= 2:
        controls = [c0, c1][:kind]
        proj = _on_bits(M, {c: _P1 for c in controls})            # P_C
        flip = _on_bits(M, {**{c: _P1 for c in controls}, target: _X})  # P_C X_t
        return np.eye(1 << M) - proj + flip
    if kind <= 5:
        controls = [c0, c1][:kind - 3]
        return np.eye(1 << M) - 2 * _on_bits(M, {**{c: _P1 for c in controls}, target: _P1})
    a, b = target, c0
    return (_on_bits(M, {a: _P0, b: _P0}) + _on_bits(M, {a: _P1, b: _P1})
            + _on_bits(M, {a: _S01, b: _S10}) + _on_bits(M, {a: _S10, b: _S01}))


def composite_matrix(gates, M: int) -> np.ndarray:
    """U = U_n ... U_1 (Step 1 first)."""
    U = np.eye(1 << M)
    for g in np.asarray(gates, dtype=np.uint8).reshape(-1, 4):
        U = step_matrix(g, M) @ U
    return U


def perm_of(U: np.ndarray) -> np.ndarray:
    """Column index of the single unity in each row (gather form, reading R2)."""
    assert np.all((U == 0) | (U == 1)) and np.all(U.sum(axis=1) == 1)
    return np.argmax(U, axis=1).astype(np.uint32)


def signed_perm_of(U: np.ndarray):
    """(column, value) of the single non-zero of each row of a phased
    permutation (values +-1)."""
    assert np.all(np.isin(U, (-1.0, 0.0, 1.0))) and np.all(np.abs(U).sum(axis=1) == 1)
    cols = np.argmax(np.abs(U), axis=1)
    return cols.astype(np.uint32), U[np.arange(U.shape[0]), cols]
