echo "# compute-sanitizer (memcheck + racecheck) over every kernel of the path, reduced budgets"
echo "# tools/sanitizer_workload.py <nodes> <solver path>; B200, final build of round 1"
for cfg in "50 auto" "50 split" "60 auto" "100 auto" "15 generic" "7 split"; do
  for tool in memcheck racecheck; do
    echo "== compute-sanitizer --tool $tool: nodes/path $cfg"
    timeout 600 compute-sanitizer --tool $tool python tools/sanitizer_workload.py $cfg 2>&1 | grep -E "^status|ERROR SUMMARY|RACECHECK SUMMARY|Error|hazard" | head -8
  done
done
