# compute-sanitizer over tools/sanitize_cases.py with every tool, plus the
# staged small-box fallbacks and the Ax layer pieces / sub-slabs.
#   bash tools/sanitize_all.sh OUT.md
out=$1
{
echo "# compute-sanitizer over every kernel"
echo
echo 'Command: `compute-sanitizer --tool T python tools/sanitize_cases.py` on one B200 (odd sizes, slab/window launches, residual epilogue, main-axis and z-layered Ax with texture fills, Siddon, matched staged (4-CTA 8-plane and 3-CTA 14-plane variants, x-major views in the transposed frame and in their own frame, zero-on-flush) incl. a 2 KB box budget that forces the half-depth and global fallbacks, fine-detector lane strides, FDK staged + direct path, TV-GD (r01 tiled pair and the marching gradient / fused / step passes, paired and single-voxel), ROF (marching and r01)).'
echo
echo "| tool | result | cases completed |"
echo "|---|---|---|"
run() {  # label, tool, env...
  label=$1; tool=$2; shift 2
  log=$(env "$@" compute-sanitizer --tool $tool python tools/sanitize_cases.py 2>&1)
  r=$(echo "$log" | grep -E "ERROR SUMMARY|RACECHECK SUMMARY" | tail -1 | sed 's/=* //')
  done_=$(echo "$log" | grep -c "sanitize cases done")
  echo "| $label | $r | $([ "$done_" = 1 ] && echo yes || echo NO) |"
}
for t in memcheck racecheck synccheck initcheck; do run $t $t CS_NONE=1; done
run "racecheck, 2 KB staged boxes" racecheck CS_STAGED_SMEM_KB=2
run "memcheck, Ax layer pieces (CS_MAX_LAYERS=22: nx = ny = 24 in 2 pieces)" memcheck CS_MAX_LAYERS=22
run "memcheck, Ax sub-slabs (CS_TEX_MAX_MB=0.03: 20-plane slab in 10-plane pieces; residual skipped)" memcheck CS_TEX_MAX_MB=0.03 SAN_NO_RESIDUAL=1
run "memcheck, z-layered Ax" memcheck CS_FWD_MLAYER=0
run "racecheck, matched x-major views in their own frame (CS_ST_TRANSPOSE=0)" racecheck CS_ST_TRANSPOSE=0
run "memcheck, matched x-major views in their own frame (CS_ST_TRANSPOSE=0)" memcheck CS_ST_TRANSPOSE=0
run "memcheck, deterministic matched (CS_ST_DETERMINISTIC=1)" memcheck CS_ST_DETERMINISTIC=1
run "racecheck, deterministic matched (CS_ST_DETERMINISTIC=1)" racecheck CS_ST_DETERMINISTIC=1
run "memcheck, deterministic matched with 2 KB boxes (global path)" memcheck CS_ST_DETERMINISTIC=1 CS_STAGED_SMEM_KB=2
} > $out
