timeout 1500 python -m pytest tests -x -q -m gpu 2>&1 | tail -5 > gpurun_out/g11_tests.log
for cfg in "62 fast" "63 fast" "100 fast" "102 fast" "50 fast" "61 fast"; do
  for tool in memcheck racecheck; do
    echo "== compute-sanitizer --tool $tool: nodes/path $cfg"
    timeout 900 compute-sanitizer --tool $tool python tools/sanitizer_workload.py $cfg 2>&1 | grep -E "^status|ERROR SUMMARY|RACECHECK SUMMARY|Error|hazard" | sed 's/+0x.*//' | sort | uniq -c | head -12
  done
done > gpurun_out/g11_sanitizer.txt 2>&1
timeout 300 python tools/n100_probe.py > gpurun_out/g11_n100.txt 2>&1
cat gpurun_out/g11_tests.log gpurun_out/g11_sanitizer.txt gpurun_out/g11_n100.txt
