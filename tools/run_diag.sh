timeout 900 python -m pytest tests/test_gpu_kron.py -q -x > gpurun_out/pytest_kron.log 2>&1
{ for rc in 1 2 4 8 16; do QSIM_KRON_COPIES=$rc python tools/bench_kron.py 32 | sed "s/^/rc=$rc /"; QSIM_KRON_COPIES=$rc python tools/bench_kron.py 40 32 | sed "s/^/rc=$rc /"; done; python tools/bench_kron.py 32 32 c128; } > gpurun_out/diag14.log 2>&1
