{
for m in map_gather fused; do
python tools/diag_planned.py cfg5 $m | tail -1 | sed "s/^/st=.cs /"
QSIM_JIT_STORE="" python tools/diag_planned.py cfg5 $m | tail -1 | sed "s/^/st=wb /"
QSIM_JIT_STORE=".cg" python tools/diag_planned.py cfg5 $m | tail -1 | sed "s/^/st=.cg /"
QSIM_JIT_STORE=".L1::no_allocate" python tools/diag_planned.py cfg5 $m | tail -1 | sed "s/^/st=noalloc /"
done
} > gpurun_out/diag15.log 2>&1
