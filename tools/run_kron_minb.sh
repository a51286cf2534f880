for mb in 1 2 3 4; do
  export QSIM_KRON_MINB=$mb
  echo "minb=$mb"
  timeout 120 python tools/bench_kron.py 32
  timeout 120 python tools/bench_kron.py 40 32
  timeout 120 python tools/bench_kron.py 32 31 c128
done
