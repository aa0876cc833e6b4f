timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "bc" 2>&1 | tail -1
MG_LIB_PATH=paper_1504_04804_b200/libmgraph_b200_bclr.so timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "bc" 2>&1 | tail -1
for i in 1 2 3; do
timeout 300 python tools/timeline.py bc 24 2>&1 | grep -E "device_ms" | sed "s/^/[cur] /"
MG_LIB_PATH=paper_1504_04804_b200/libmgraph_b200_bclr.so timeout 300 python tools/timeline.py bc 24 2>&1 | grep -E "device_ms" | sed "s/^/[bclr] /"
done
