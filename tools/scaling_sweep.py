"""Per-bit scaling sweep on one B200 (Figure 4 analogue).

The paper reports run time growing "roughly x3.4 per bit ... from M = 30 to
31" on NCSA modi4 with up to 64 threads.  This times the hot path
for M = 20..32 on 64 random NOT/CNOT/CCNOT gates (seed 4, the cfg5 recipe
over M bits) and complex64 Gaussian states, and prints a CSV with the
growth factor per added bit.

    python tools/scaling_sweep.py [--mmin 20] [--mmax 32] [--kron-max 40] > profiles/rNN_scaling.csv

A second table times the input generated on the fly (Appendix 1): the whole
2^M output for M <= 32, and for 32 < M <= --kron-max the 2^32-entry portion
[0, 2^32) with the whole output extrapolated as 2^(M-32) such portions (the
"continuous portions" of P:L13; nothing of size 2^M is ever stored).
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_quant_ph_0308158_b200 as q  # noqa: E402
import workloads as wl  # noqa: E402
from tools.sweep_apply import timeit  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mmin", type=int, default=20)
    ap.add_argument("--mmax", type=int, default=32)
    ap.add_argument("--kron-max", type=int, default=40)
    ap.add_argument("--tune", default="none", choices=["none", "measure", "patient"],
                    help="qsim_plan_tune_ex effort per M (outside the timings)")
    args = ap.parse_args()
    print("M,entries,map_gather_ms,build_ms,apply_ms,fused_ms,entries_per_s,growth_per_bit,"
          "plan_natural")
    prev = None
    for M in range(args.mmin, args.mmax + 1):
        N = 1 << M
        gates = wl.random_gates(64, M, 4)
        spec = wl.StateSpec(M, "c64", wl.GAUSS, 1004)
        host = torch.empty(N * 8, dtype=torch.uint8, pin_memory=True)
        wl.fill_state(spec, host.data_ptr())
        k1 = host.to("cuda")
        del host
        k2 = torch.empty_like(k1)
        perm = torch.empty(N, dtype=torch.int32, device="cuda")
        ws = q.workspace()
        plan = q.plan_create(gates, M, "c64")
        if args.tune != "none" and not (plan.flags & 1):
            q.plan_tune(plan, gates, perm, k1, k2, ws,
                        effort=q.TUNE_MEASURE if args.tune == "measure" else q.TUNE_PATIENT)
        t_mg = timeit(lambda: q.map_gather_planned(plan, gates, perm, k1, k2, ws))
        t_b = timeit(lambda: q.build_map(gates, M, perm))
        t_a = timeit(lambda: q.apply_map_planned(plan, perm, k1, k2, ws))
        t_f = timeit(lambda: q.run_fused_planned(plan, gates, k1, k2, ws))
        growth = "" if prev is None else f"{t_mg / prev:.3f}"
        print(f"{M},{N},{t_mg:.4f},{t_b:.4f},{t_a:.4f},{t_f:.4f},{N / t_mg * 1e3:.4e},{growth},"
              f"{int(plan.flags & 1)}", flush=True)
        prev = t_mg
        del k1, k2, perm
        torch.cuda.empty_cache()
    print()
    print("M,portion_entries,kron_portion_ms,kron_full_ms_extrapolated,entries_per_s,growth_per_bit,kernel")
    prev = None
    out = torch.empty(1 << min(args.kron_max, 32), dtype=torch.complex64, device="cuda")
    for M in range(args.mmin, args.kron_max + 1):
        count = 1 << min(M, 32)
        gates = wl.random_gates(64, M, 4)
        qb = wl.random_qubits(M, 2040, "c64")
        t = timeit(lambda: q.run_fused_kron(gates, M, qb, out, start=0, count=count, dtype="c64"))
        full = t * (1 << max(M - 32, 0))
        growth = "" if prev is None else f"{full / prev:.3f}"
        print(f"{M},{count},{t:.4f},{full:.4f},{count / t * 1e3:.4e},{growth},{q.last_kernel()}",
              flush=True)
        prev = full


if __name__ == "__main__":
    main()
