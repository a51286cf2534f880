"""Writes tests/golden/inputs_sha256.txt: the numpy version, the SHA-256 of
every config's generated gate list, the normalisation scale of each state and
the SHA-256 of its first 2^12 entries.  Calls only workloads/ (no method
arithmetic, never the CUDA path).

    python tests/golden/make_inputs_sha.py
"""
import hashlib
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import numpy as np  # noqa: E402
import workloads as wl  # noqa: E402

lines = ["# Written by tests/golden/make_inputs_sha.py (workloads/ only).",
         "# Gate lists: readings R6-R9 (numpy default_rng); states: reading R10.",
         f"numpy {np.__version__}"]
for name, cfg in wl.CONFIGS.items():
    g = np.ascontiguousarray(cfg.gates(), dtype=np.uint8)
    lines.append(f"gates_{name} {hashlib.sha256(g.tobytes()).hexdigest()}")
for name, cfg in wl.CONFIGS.items():
    spec = cfg.state
    scale = spec.scale()
    st = wl.make_state(spec, 0, min(spec.N, 1 << 12), scale=scale)
    lines.append(f"scale_{name} {float(scale).hex()}")
    lines.append(f"state_{name} {hashlib.sha256(st.tobytes()).hexdigest()}")
with open(os.path.join(HERE, "inputs_sha256.txt"), "w") as f:
    f.write("\n".join(lines) + "\n")
print("\n".join(lines))
