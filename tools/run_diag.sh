{
for gb in 8 9 10 11; do QSIM_KRON_GROUP_BITS=$gb python tools/bench_kron.py 32; QSIM_KRON_GROUP_BITS=$gb python tools/bench_kron.py 40 32; done
python tools/bench_kron.py 32 32 c128; python tools/bench_kron.py 26 26 c128
} > gpurun_out/diag9.log 2>&1
