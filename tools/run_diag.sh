timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "linear or planned" > gpurun_out/pytest_lt.log 2>&1
{
for m in map_gather fused; do python tools/diag_planned.py cfg5 $m | tail -1; QSIM_NO_LINEAR=1 python tools/diag_planned.py cfg5 $m | tail -1 | sed "s/^/nolin /"; done
} > gpurun_out/diag8.log 2>&1
