# cover granule A/B (QSIM_PLAN_GRANULE_BYTES: 32 = sector, the default; 64; 128 = L1 line)
{
for gb in 32 64 128; do
  for T in 12 13 14; do
    for m in map_gather fused; do
      QSIM_PLAN_GRANULE_BYTES=$gb QSIM_PLAN_COVER_BITS=$T QSIM_PLAN_COVER_FIXED=1 timeout 120 python tools/diag_planned.py cfg5 $m | tail -1 | sed "s/^/granule=$gb T=$T /"
    done
  done
done
} > gpurun_out/diag_granule.log 2>&1
