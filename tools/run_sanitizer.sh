echo "# compute-sanitizer (memcheck + racecheck) over every kernel of the path, reduced budgets"
echo "# tools/sanitizer_workload.py <nodes> <solver path>; B200, build of round 2 (discretization in tiles of four"
echo "# intervals with CTA-cooperative chunk copies, latency-mode kernels over 1 / 2 / 8 CTAs, column-sparse kernels:"
echo "# 'fast' = column-sparse + dense behind them for N <= 61 (15: one warp per role, 50 / 61: two with halo lanes),"
echo "# 'dense' = the dense register-resident kernels alone)"
for cfg in "50 fast" "15 fast" "31 fast" "32 fast" "61 fast" "62 fast" "63 fast" "102 fast" "50 dense" "50 latency" "15 latency" "17 latency" "100 latency" "50 split" "60 fast" "100 fast" "15 generic" "7 split"; do
  for tool in memcheck racecheck; do
    echo "== compute-sanitizer --tool $tool: nodes/path $cfg"
    timeout 900 compute-sanitizer --tool $tool python tools/sanitizer_workload.py $cfg 2>&1 | grep -E "^status|ERROR SUMMARY|RACECHECK SUMMARY|Error|hazard" | sed 's/+0x.*//' | sort | uniq -c | head -12
  done
done
