"""Writes the regression fixtures in this directory that are not printed in
the paper.  It calls only oracle/ and workloads/ (never the CUDA path).

    python tests/golden/make_golden.py
"""
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import oracle  # noqa: E402
import workloads as wl  # noqa: E402

cfg = wl.CONFIGS["cfg1"]
perm = oracle.build_map(cfg.gates(), cfg.M)
with open(os.path.join(HERE, "cfg1_perm.txt"), "w") as f:
    f.write("# Written by tests/golden/make_golden.py from oracle.build_map (oracle only).\n")
    f.write("# cfg1 = BASELINE.json configs[0]: worked step CNOT(t=a(1), c=a(2)) [P:L43]\n")
    f.write("# followed by 8 random gates (seed 0, reading R8).  Gather permutation perm[0..7].\n")
    f.write("# Cross-checked in tests against the dense Kronecker product (oracle/dense.py).\n")
    f.write(" ".join(str(int(v)) for v in perm) + "\n")
print(perm)
