{
for m in map_gather fused apply; do
python tools/diag_planned.py cfg5 $m | tail -1 | sed "s/^/hint=0 /"
QSIM_JIT_K1_HINT=1 python tools/diag_planned.py cfg5 $m | tail -1 | sed "s/^/hint=1 /"
done
} > gpurun_out/diag16.log 2>&1
