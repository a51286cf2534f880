"""Experiment: a wider search over the runtime part of the traversal order
(counter bits 10..31, a kernel parameter -- no recompiles) than
qsim_plan_tune's stage 3 (which only moves one tail bit into the 10 positions
above the cover).  Moves: swap any two counter positions in 10..31 (this also
exchanges the CTA's warp-level cover bits 10..12 with tail bits).  Hill
climbing on cfg5 map+gather, one timed call per screen, re-timed (best of 5)
before a move is accepted.  Prints the path and the final A/B."""
import json
import os
import random
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import paper_quant_ph_0308158_b200 as q  # noqa: E402
import workloads as wl  # noqa: E402


def main():
    budget_s = float(os.environ.get("TC_BUDGET_S", "240"))
    dev = torch.device("cuda:0")
    cfg = wl.CONFIGS["cfg5"]
    gates, M, N = cfg.gates(), cfg.M, cfg.N
    k1 = torch.empty(N * 8, dtype=torch.uint8, device=dev)
    stage = torch.empty(1 << 30, dtype=torch.uint8, pin_memory=True)
    scale = cfg.state.scale()
    chunk = (1 << 30) // 8
    for s0 in range(0, N, chunk):  # the bench's Gaussian state (power depends on the data)
        wl.fill_state(cfg.state, stage.data_ptr(), s0, chunk, scale=scale)
        k1[s0 * 8:(s0 + chunk) * 8].copy_(stage)
    del stage
    k2 = torch.empty_like(k1)
    perm = torch.empty(N, dtype=torch.int32, device=dev)
    ws = q.workspace(dev)
    plan = q.plan_create(gates, M, "c64")
    tuned = json.load(open(os.path.join(ROOT, "profiles", "r02_tuned_plan_cfg5.json")))
    for k, v in enumerate(tuned["sigma"]):
        plan.sigma[k] = v
    plan.chunk_log2, plan.fused_chunk_log2 = tuned["chunk_log2"], tuned["fused_chunk_log2"]
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def timed(sig, reps):
        for k in range(32):
            plan.sigma[k] = sig[k]
        best = 1e30
        for _ in range(reps):
            a.record()
            q.map_gather_planned(plan, gates, perm, k1, k2, ws)
            b.record()
            b.synchronize()
            best = min(best, a.elapsed_time(b))
        return best

    cur = list(tuned["sigma"])
    timed(cur, 2)
    cur_t = timed(cur, 5)
    start_t = cur_t
    print(json.dumps({"start_ms": cur_t, "sigma": cur}), flush=True)
    rng = random.Random(12345)
    t0 = time.time()
    evals = accepted = 0
    while time.time() - t0 < budget_s:
        i, j = rng.sample(range(10, 32), 2)
        cand = list(cur)
        cand[i], cand[j] = cand[j], cand[i]
        t = timed(cand, 1)
        evals += 1
        if t < cur_t * 0.995:
            t5 = timed(cand, 5)
            if t5 < cur_t * 0.995:
                cur, cur_t = cand, t5
                accepted += 1
                print(json.dumps({"accepted": [i, j], "ms": t5, "evals": evals}), flush=True)
    # final A/B, interleaved
    ab = {"start": [], "final": []}
    for _ in range(5):
        ab["start"].append(timed(tuned["sigma"], 3))
        ab["final"].append(timed(cur, 3))
    print(json.dumps({"evals": evals, "accepted": accepted, "start_ms": start_t, "final_ms": cur_t,
                      "ab_start_min": min(ab["start"]), "ab_final_min": min(ab["final"]),
                      "sigma": cur}), flush=True)
    # parity of the final order: sampled outputs vs a fresh build_map (same library)
    for k in range(32):
        plan.sigma[k] = cur[k]
    q.map_gather_planned(plan, gates, perm, k1, k2, ws)
    ref = torch.empty_like(perm)
    q.build_map(gates, M, ref)
    torch.cuda.synchronize()
    idx = torch.randint(0, N, (1 << 22,), device=dev)
    print(json.dumps({"perm_equal_on_samples": bool(torch.equal(perm[idx], ref[idx]))}), flush=True)


if __name__ == "__main__":
    main()
