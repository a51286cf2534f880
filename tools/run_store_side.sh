# timing-only experiment (results invalid under QSIM_DEBUG_STORE): how much of the
# fused / map+gather step is the k2 store pattern?  seq = k2 in counter order, none = no k2
for ds in "" seq none; do
  for m in fused map_gather; do
    QSIM_DEBUG_STORE=$ds timeout 120 python tools/diag_planned.py cfg5 $m | tail -1 | sed "s/^/store=${ds:-plan} /"
  done
done
