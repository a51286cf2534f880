timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1
timeout 600 python tools/all_configs.py > gpurun_out/all_configs2.jsonl 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_lb.json 2> gpurun_out/bench_lb.err
