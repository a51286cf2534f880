# build kernel on seeds whose in-thread bits are high: default vs QSIM_BUILD_THREAD_BITS=0
for bt in 0 1; do
  export QSIM_BUILD_THREAD_BITS=$bt
  for sd in 7 11 4; do timeout 120 python tools/bench_build.py 32 $sd; done
done
