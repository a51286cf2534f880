# cover-bit order from counter bit 5 (QSIM_PLAN_COVER_ORDER=2: lanes unchanged, commonest sector-mate differences on the thread bits)
{
for co in 0 2; do
  for sd in 4 6 8 5; do
    for m in map_gather fused; do
      QSIM_PLAN_COVER_ORDER=$co timeout 120 python tools/diag_planned.py seed:$sd $m | tail -1 | sed "s/^/order=$co /"
    done
  done
done
} > gpurun_out/diag_order2.log 2>&1
