"""Experiment driver for first_touch.cu (NOT the product path): cfg5 planned
apply with / without whole-line loads by each k1 line's first reader.
Prints one JSON line per variant (CUDA-event ms, best and median of reps)."""
import ctypes
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import paper_quant_ph_0308158_b200 as q  # noqa: E402
import workloads as wl  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def tabs(sigma, M=32):
    fwd = np.zeros((4, 256), np.uint32)
    inv = np.zeros((4, 256), np.uint32)
    sinv = [0] * 32
    for k in range(M):
        sinv[sigma[k]] = k
    for b in range(4):
        for v in range(256):
            f = i = 0
            for j in range(8):
                if (v >> j) & 1:
                    f |= 1 << sigma[8 * b + j]
                    i |= 1 << sinv[8 * b + j]
            fwd[b, v], inv[b, v] = f, i
    return np.concatenate([fwd.ravel(), inv.ravel()])


def main():
    reps = int(os.environ.get("FT_REPS", "5"))
    modes = [int(x) for x in os.environ.get("FT_MODES", "0,1,2,3,4").split(",")]
    lib = ctypes.CDLL(os.path.join(HERE, "libft.so"))
    dev = torch.device("cuda:0")
    cfg = wl.CONFIGS["cfg5"]
    gates, M, N = cfg.gates(), cfg.M, cfg.N
    k1 = torch.empty(N * 2, dtype=torch.float32, device=dev).normal_()
    k2 = torch.empty_like(k1)
    perm = torch.empty(N, dtype=torch.int32, device=dev)
    ws = q.workspace(dev)
    q.build_map(gates, M, perm)
    plan = q.plan_create(gates, M, "c64")
    torch.cuda.synchronize()
    if os.environ.get("FT_NOTUNE") == "1":  # the tuned cfg5 plan recorded in profiles/
        tuned = json.load(open(os.path.join(ROOT, "profiles", "r02_tuned_plan_cfg5.json")))
        for k, v in enumerate(tuned["sigma"]):
            plan.sigma[k] = v
        plan.chunk_log2, plan.fused_chunk_log2 = tuned["chunk_log2"], tuned["fused_chunk_log2"]
    else:
        q.plan_tune(plan, gates, perm, k1, k2, ws)
    q.build_map(gates, M, perm)
    torch.cuda.synchronize()
    sigma = list(plan.sigma)
    print(json.dumps({"sigma": sigma, "chunk_log2": plan.chunk_log2}), flush=True)
    t = torch.from_numpy(tabs(sigma).view(np.int32)).to(dev)
    inv = torch.empty(N, dtype=torch.int32, device=dev)
    bitmap = torch.empty(N // 32, dtype=torch.int32, device=dev)
    sink = torch.zeros(4, dtype=torch.int32, device=dev)
    ticket = torch.zeros(4, dtype=torch.int64, device=dev)
    cnt = torch.zeros(4, dtype=torch.int64, device=dev)
    st = torch.cuda.current_stream().cuda_stream
    assert lib.ft_inv(ctypes.c_void_p(perm.data_ptr()), ctypes.c_void_p(inv.data_ptr()), ctypes.c_uint64(N),
                      ctypes.c_void_p(st)) == 0

    def ev_time(fn):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        fn()
        torch.cuda.synchronize()
        ts = []
        for _ in range(reps):
            a.record()
            fn()
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        return min(ts), float(np.median(ts))

    # reference result: the library's planned apply
    jit = ev_time(lambda: q.apply_map_planned(plan, perm, k1, k2, ws))
    print(json.dumps({"variant": "qsim_apply_map_planned (library)", "ms_best": jit[0], "ms_med": jit[1]}),
          flush=True)
    if os.environ.get("FT_LIB") == "1":
        for name, fn in (("run_fused_planned", lambda: q.run_fused_planned(plan, gates, k1, k2, ws)),
                         ("map_gather_planned", lambda: q.map_gather_planned(plan, gates, perm, k1, k2, ws))):
            r = ev_time(fn)
            print(json.dumps({"variant": name + " (library)", "ms_best": r[0], "ms_med": r[1]}), flush=True)
        q.build_map(gates, M, perm)
        q.apply_map_planned(plan, perm, k1, k2, ws)
    idx = torch.randint(0, N, (1 << 20,), device=dev)
    want = k2.view(torch.int64)[idx].clone()

    for fm in (0, 1):
        assert lib.ft_flags(ctypes.c_void_p(perm.data_ptr()), ctypes.c_void_p(inv.data_ptr()),
                            ctypes.c_void_p(t.data_ptr()), ctypes.c_void_p(bitmap.data_ptr()), ctypes.c_uint64(N),
                            fm, plan.chunk_log2, ctypes.c_void_p(cnt.data_ptr()), ctypes.c_void_p(st)) == 0
        torch.cuda.synchronize()
        nflag = int(cnt[0])
        cnt.zero_()
        for mode in modes:
            if fm == 1 and mode < 2:
                continue
            k2.zero_()

            def run():
                rc = lib.ft_gather(mode, ctypes.c_uint64(N), plan.chunk_log2, ctypes.c_void_p(ticket.data_ptr()),
                                   ctypes.c_void_p(k1.data_ptr()), ctypes.c_void_p(k2.data_ptr()),
                                   ctypes.c_void_p(perm.data_ptr()), ctypes.c_void_p(bitmap.data_ptr()),
                                   ctypes.c_void_p(t.data_ptr()), ctypes.c_void_p(sink.data_ptr()), 148,
                                   ctypes.c_void_p(st))
                assert rc == 0, rc
            r = ev_time(run)
            ok = bool(torch.equal(k2.view(torch.int64)[idx], want))
            print(json.dumps({"variant": f"ft mode {mode}", "flags": ["min counter", "min chunk"][fm],
                              "flagged": nflag, "ms_best": r[0], "ms_med": r[1], "k2_ok": ok}), flush=True)


if __name__ == "__main__":
    t0 = time.time()
    main()
    print(json.dumps({"wall_s": time.time() - t0}))
