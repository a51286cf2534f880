# reads-only time (QSIM_DEBUG_STORE=none, results invalid): sector-cover plan vs linear traversal
{
for env in "QSIM_DEBUG_STORE=none" "QSIM_DEBUG_STORE=none QSIM_PLAN_LINEAR=1 QSIM_PLAN_COVER_FIXED=1" "QSIM_PLAN_LINEAR=1 QSIM_PLAN_COVER_FIXED=1"; do
  env $env timeout 120 python tools/diag_planned.py cfg5 fused | tail -1 | sed "s/^/$env /"
done
} > gpurun_out/diag_lt2.log 2>&1
