timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "planned or staged" > gpurun_out/pytest_planned.log 2>&1
{
for T in 11 12 13 14; do for c in 15 16 17; do QSIM_PLAN_COVER_BITS=$T python tools/diag_planned.py cfg5 map_gather chunk=$c | tail -1 | sed "s/^/T=$T /"; done; done
for c in 16 17; do python tools/diag_planned.py cfg5 fused chunk=$c | tail -1; done
for m in map_gather fused apply; do for o in natural sigma; do python tools/diag_planned.py cfg3 $m order=$o | tail -1; done; done
} > gpurun_out/diag5.log 2>&1
