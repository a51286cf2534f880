timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "pairs or linear or planned" > gpurun_out/pytest_pairs.log 2>&1
{
for m in map_gather fused; do QSIM_PLAN_PAIRS=1 python tools/diag_planned.py cfg5 $m | tail -1 | sed "s/^/pairs /"; done
} > gpurun_out/diag10.log 2>&1
