# same-box A/B vs variant $1 plus the first-pull instruction count of both (source 0)
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "dobfs or bfs or across" 2>&1 | tail -1
bash tools/gpu/ab_multi.sh $1
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum
MG_NO_GRAPH=1 ncu --metrics $M --clock-control none -k regex:"dobfs_pull_thread" -c 1 --csv --log-file gpurun_out/pi_def.csv python tools/dobfs_probe.py 26 0.01 exact 0 > /dev/null 2>&1
MG_LIB_PATH=paper_1504_04804_b200/libmgraph_b200_$1.so MG_NO_GRAPH=1 ncu --metrics $M --clock-control none -k regex:"dobfs_pull_thread" -c 1 --csv --log-file gpurun_out/pi_var.csv python tools/dobfs_probe.py 26 0.01 exact 0 > /dev/null 2>&1
