"""A/B (experiment): on-the-fly input with direct stores vs CTA-staged TMA bulk
stores (QSIM_KRON_STAGE 0 / 1 / 2), cfg5's circuit at M = 32 and the M = 40
portion; outputs compared byte for byte with the direct-store kernel."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402
import paper_quant_ph_0308158_b200 as q  # noqa: E402
import workloads as wl  # noqa: E402

for M in (32, 40):
    gates = wl.CONFIGS["cfg5"].gates() if M == 32 else wl.random_gates(64, M, 4)
    qb = wl.random_qubits(M, 2040, "c64")
    count = 1 << 32
    start = 0 if M == 32 else (1 << (M - 1)) - count // 2
    ref = torch.empty(count, dtype=torch.complex64, device="cuda")
    out = torch.empty_like(ref)
    for stage in os.environ.get("STAGES", "0,1,2").split(","):
        os.environ["QSIM_KRON_STAGE"] = stage
        dst = ref if stage == "0" else out
        dst.zero_()
        times = []
        for i in range(8):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            q.run_fused_kron(gates, M, qb, dst, start=start, count=count, dtype="c64")
            b.record()
            torch.cuda.synchronize()
            times.append(a.elapsed_time(b))
        same = True if stage == "0" else bool(torch.equal(ref.view(torch.int64), out.view(torch.int64)))
        print(json.dumps({"M": M, "stage": stage, "ms_best": min(times[2:]),
                          "ms_med": sorted(times[2:])[3], "bytes_equal_to_direct": same,
                          "kernel": q.last_kernel()}), flush=True)
