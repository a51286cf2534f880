import os, sys
sys.path.insert(0, '/root/repo')
import torch, ctypes
import paper_quant_ph_0308158_b200 as q
import workloads as wl
M=24; g = wl.random_gates(64, M, 4)
N=1<<M
k1 = torch.arange(N, dtype=torch.int64, device='cuda').view(torch.uint8)
k2 = torch.empty_like(k1); perm = torch.empty(N, dtype=torch.int32, device='cuda'); ws = q.workspace()
plan = q.plan_create(g, M, 'c64'); plan.flags &= ~1
q.build_map(g, M, perm); torch.cuda.synchronize()
for v in sys.argv[1:]:
    os.environ['QSIM_PF'] = v
    for name, fn in [('ap', lambda: q.apply_map_planned(plan, perm, k1, k2, ws)), ('fu', lambda: q.run_fused_planned(plan, g, k1, k2, ws))]:
        try:
            fn(); torch.cuda.synchronize(); print(v, name, 'ok', q.last_kernel())
        except Exception as e:
            print(v, name, 'ERR', e, q.lib().qsim_last_error().decode(), q.last_kernel())
