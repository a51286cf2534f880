# on-the-fly input: transposed (default) vs affine (QSIM_KRON_AFFINE=1) in-thread fast path
for af in 0 1; do
  export QSIM_KRON_AFFINE=$af
  echo "affine=$af"
  timeout 120 python tools/bench_kron.py 32
  timeout 120 python tools/bench_kron.py 32 32 c64 8
  timeout 120 python tools/bench_kron.py 32 32 c64 6
  timeout 120 python tools/bench_kron.py 32 31 c128
  timeout 120 python tools/bench_kron.py 40 32
  timeout 120 python tools/bench_kron.py 30 30 c64 3
done
QSIM_KRON_AFFINE=1 timeout 900 python -m pytest tests/test_gpu_kron.py -q -x 2>&1 | tail -2
