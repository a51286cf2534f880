# build kernel: QSIM_BUILD_THREAD_BITS=0 (J = 5..9, transpose) vs =1 (default: in-thread affine fast path when |V| <= 6 and affine)
for bt in 0 1; do
  export QSIM_BUILD_THREAD_BITS=$bt
  timeout 120 python tools/bench_build.py 32
  timeout 120 python tools/bench_build.py 32 8
  timeout 120 python tools/bench_build.py 32 6
  timeout 120 python tools/bench_build.py 32 5
  timeout 120 python tools/bench_build.py 30 3
  timeout 120 python tools/bench_build.py 31
done
