# on-the-fly input and build across circuits (M = 32, 64 random gates, seeds 4..11)
for sd in 4 5 6 7 8 9 10 11; do
  timeout 120 python tools/bench_kron.py 32 32 c64 $sd
  timeout 120 python tools/bench_build.py 32 $sd
done
