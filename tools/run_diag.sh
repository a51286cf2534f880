timeout 900 python -m pytest tests/test_gpu_kron.py tests/test_gpu_phased.py -q -x > gpurun_out/pytest_kron.log 2>&1
{ python tools/bench_kron.py 32; python tools/bench_kron.py 40 32; python tools/bench_kron.py 32 32 c128; } > gpurun_out/diag13.log 2>&1
