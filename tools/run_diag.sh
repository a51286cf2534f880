timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "local or structured or planned" > gpurun_out/pytest_local.log 2>&1
{
for c in low:10 low:13; do for m in map_gather fused; do python tools/diag_planned.py $c $m | tail -1; done; done
} > gpurun_out/diag18.log 2>&1
