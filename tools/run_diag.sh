{
for q in "" ".L2::64B" ".L2::128B" ".L2::256B"; do
  for m in map_gather fused; do QSIM_JIT_LDQ="$q" python tools/diag_planned.py cfg5 $m | tail -1 | sed "s/^/ldq=$q /"; done
done
} > gpurun_out/diag23.log 2>&1
