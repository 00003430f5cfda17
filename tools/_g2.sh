timeout 300 python tools/_probe100.py 2>&1 | tail -1 > gpurun_out/g8.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "node_count_edges or config5_n100_cluster" 2>&1 | tail -5 >> gpurun_out/g8.txt
cat gpurun_out/g8.txt
