# e2e timeline of the staged pipeline over stage schedules (GCABEM_STAGE_*)
mkdir -p gpurun_out
for v in "$@"; do
  echo "== $v"
  env REPS=7 $v timeout 300 python tools/e2e_timeline.py c3 2>/dev/null | grep "total" | tail -6 | awk '{print $3}' | sort -n | tr '\n' ' '; echo
done
