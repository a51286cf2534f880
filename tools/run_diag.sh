timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pytest_parity.log 2>&1
{
python tools/diag_planned.py cfg5 apply | tail -1
python tools/diag_planned.py cfg4 apply | tail -1
} > gpurun_out/diag12.log 2>&1
