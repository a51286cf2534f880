# cover-bit order inside the cover (QSIM_PLAN_COVER_ORDER=1: commonest sector-mate difference bits on lanes / thread bits)
{
for co in 0 1; do
  for sd in 4 6 8; do
    for m in map_gather fused; do
      QSIM_PLAN_COVER_ORDER=$co timeout 120 python tools/diag_planned.py seed:$sd $m | tail -1 | sed "s/^/order=$co /"
    done
  done
done
} > gpurun_out/diag_order.log 2>&1
