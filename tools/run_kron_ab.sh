# A/B of the in-thread output bits (QSIM_THREAD_BITS=0: J = 5..9, no fast path)
for lay in 0 1; do
  export QSIM_THREAD_BITS=$lay
  timeout 120 python tools/bench_kron.py 32
  timeout 120 python tools/bench_kron.py 32 32 c64 8
  timeout 120 python tools/bench_kron.py 32 32 c64 6
  timeout 120 python tools/bench_kron.py 32 31 c128
  timeout 120 python tools/bench_kron.py 40 32
  timeout 120 python tools/bench_kron.py 30 30 c64 3
  timeout 120 python tools/bench_build.py 32
  timeout 120 python tools/bench_build.py 32 8
  timeout 120 python tools/bench_build.py 32 6
  timeout 120 python tools/bench_build.py 30 3
done
