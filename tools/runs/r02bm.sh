# the deterministic-mode lines of tools/sanitize_all.sh only
out=gpurun_out/r02bm_sanitizer.md
{
echo "| tool | result | cases completed |"
echo "|---|---|---|"
run() {
  label=$1; tool=$2; shift 2
  log=$(env "$@" compute-sanitizer --tool $tool python tools/sanitize_cases.py 2>&1)
  r=$(echo "$log" | grep -E "ERROR SUMMARY|RACECHECK SUMMARY" | tail -1 | sed 's/=* //')
  done_=$(echo "$log" | grep -c "sanitize cases done")
  echo "| $label | $r | $([ "$done_" = 1 ] && echo yes || echo NO) |"
}
run "memcheck, deterministic matched (CS_ST_DETERMINISTIC=1)" memcheck CS_ST_DETERMINISTIC=1
run "racecheck, deterministic matched (CS_ST_DETERMINISTIC=1)" racecheck CS_ST_DETERMINISTIC=1
run "memcheck, deterministic matched with 2 KB boxes (global path)" memcheck CS_ST_DETERMINISTIC=1 CS_STAGED_SMEM_KB=2
} > $out
cat $out
