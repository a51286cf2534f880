{
for r in 4 5 6 8; do for T in 13 15; do for m in map_gather fused; do QSIM_PLAN_RUN_BITS=$r QSIM_PLAN_COVER_BITS=$T python tools/diag_planned.py cfg5 $m | tail -1 | sed "s/^/run=$r T=$T /"; done; done; done
} > gpurun_out/diag7.log 2>&1
