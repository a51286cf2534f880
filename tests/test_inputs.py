"""Input reproducibility (CPU only): the seeded gate lists and states that
every parity test and the bench use must not drift silently.

* SURVEY.md Appendix A.1 / A.2 pin the first gates and the NOT / CNOT / CCNOT
  counts of each BASELINE.json config under readings R6-R9; they
  were computed there with numpy 2.3.5, independently of this repository.
* tests/golden/inputs_sha256.txt (written by tests/golden/make_inputs_sha.py,
  which calls only workloads/) records the numpy version and the SHA-256 of
  every generated gate list and of a state prefix: a numpy upgrade that
  changes Generator streams, or an edit of workloads/stategen.c, fails here
  instead of silently changing every config.
"""
import hashlib
import os

import numpy as np
import pytest

import workloads as wl

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
NOT, CNOT, CCNOT = wl.NOT, wl.CNOT, wl.CCNOT


def _g(kind, t, *c):
    return tuple(int(x) for x in wl.gate(kind, t, *c))


def _rows(gates):
    return [tuple(int(x) for x in r) for r in gates]


def test_cfg1_gate_list_appendix_A1():
    """the worked step then 8 gates from seed 0."""
    want = [_g(CNOT, 0, 1), _g(CCNOT, 1, 2, 0), _g(NOT, 0), _g(NOT, 0), _g(CCNOT, 0, 2, 1),
            _g(CCNOT, 0, 2, 1), _g(CCNOT, 1, 0, 2), _g(CNOT, 2, 1), _g(CCNOT, 1, 2, 0)]
    assert _rows(wl.CONFIGS["cfg1"].gates()) == want


@pytest.mark.parametrize("name, first, counts", [
    ("cfg2", [_g(CNOT, 9, 15), _g(NOT, 2), _g(CCNOT, 4, 17, 6), _g(NOT, 16)], (16, 24, 24)),
    ("cfg3", [_g(CCNOT, 6, 7, 2), _g(CNOT, 2, 8), _g(CCNOT, 24, 17, 4), _g(CNOT, 6, 5)], (89, 93, 74)),
    ("cfg5", [_g(CCNOT, 28, 27, 16), _g(CCNOT, 14, 19, 2), _g(CNOT, 18, 24), _g(CCNOT, 26, 17, 6)],
     (23, 22, 19)),
])
def test_random_configs_appendix_A2(name, first, counts):
    """first four gates and kind counts (reading R6/R7)."""
    g = wl.CONFIGS[name].gates()
    assert _rows(g[:4]) == first
    kinds = g[:, 0]
    assert tuple(int((kinds == k).sum()) for k in (NOT, CNOT, CCNOT)) == counts
    M = wl.CONFIGS[name].M
    for r in g:                               # distinct bits, all below M
        bits = [int(r[1])] + [int(c) for c in r[2:2 + int(r[0])]]
        assert len(set(bits)) == len(bits) and max(bits) < M
        assert all(int(c) == wl.UNUSED for c in r[2 + int(r[0]):])


def test_cfg4_ripple_appendix_A2():
    """SURVEY App. A.2 / reading R9: 56-gate block repeated to 256 gates."""
    g = wl.CONFIGS["cfg4"].gates()
    assert len(g) == 256
    assert _rows(g[:4]) == [_g(CNOT, 1, 0), _g(CCNOT, 2, 0, 1), _g(CNOT, 2, 1), _g(CCNOT, 3, 1, 2)]
    assert _rows(g[-2:]) == [_g(CNOT, 16, 15), _g(CCNOT, 17, 15, 16)]
    assert int((g[:, 0] == CNOT).sum()) == 128 and int((g[:, 0] == CCNOT).sum()) == 128
    assert np.array_equal(g[:56], g[56:112])


def _sha_rows():
    with open(os.path.join(GOLDEN, "inputs_sha256.txt")) as f:
        return dict(ln.split(None, 1) for ln in f if ln.strip() and not ln.startswith("#"))


def test_recorded_numpy_version_and_gate_list_hashes():
    rec = _sha_rows()
    for name, cfg in wl.CONFIGS.items():
        h = hashlib.sha256(np.ascontiguousarray(cfg.gates(), dtype=np.uint8).tobytes()).hexdigest()
        assert rec[f"gates_{name}"].strip() == h, (
            f"{name} gate list changed (recorded with numpy {rec['numpy'].strip()}, "
            f"running numpy {np.__version__})")


@pytest.mark.parametrize("name", ["cfg1", "cfg2", "cfg3", "cfg4", "cfg5"])
def test_recorded_state_prefix_hashes(name):
    """The counter-based state generator (reading R10): the first 2^12 entries
    (scaled by the config's normalisation) are byte-identical to the record."""
    rec = _sha_rows()
    spec = wl.CONFIGS[name].state
    n = min(spec.N, 1 << 12)
    scale = float.fromhex(rec[f"scale_{name}"].strip())
    st = wl.make_state(spec, 0, n, scale=scale)
    assert hashlib.sha256(st.tobytes()).hexdigest() == rec[f"state_{name}"].strip()
    if spec.M <= 26:                              # the scale itself (cfg5: 2^32 draws, skipped)
        assert spec.scale() == scale
