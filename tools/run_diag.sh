# tile order inside a chunk (QSIM_JIT_TILE_ROT = r: the tile's low r bits pick the block)
{
for r in 0 1 2; do
  for m in map_gather fused; do
    QSIM_JIT_TILE_ROT=$r timeout 120 python tools/diag_planned.py cfg5 $m | tail -1 | sed "s/^/rot=$r /"
  done
  QSIM_JIT_TILE_ROT=$r timeout 120 python tools/diag_planned.py cfg5 map_gather chunk=16 | tail -1 | sed "s/^/rot=$r /"
done
} > gpurun_out/diag_rot.log 2>&1
