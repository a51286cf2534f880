timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "tune" > gpurun_out/pytest_tune.log 2>&1
timeout 1200 python tools/seed_sweep.py --M 32 --seeds 4,5,6,7,8,9 --tune > gpurun_out/seed32t.csv 2>&1
timeout 900 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/bench_t.json 2> gpurun_out/bench_t.err
