# per-launch times of one exact-cost DOBFS (source 0, graph loop): session-start vs current library
M=gpu__time_duration.sum,smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum
MG_NO_GRAPH=1 MG_LIB_PATH=paper_1504_04804_b200/libmgraph_b200_old.so ncu --metrics $M --clock-control none --csv --log-file gpurun_out/l_old.csv python tools/dobfs_probe.py 26 0.01 exact 0 > /dev/null 2>&1
MG_NO_GRAPH=1 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/l_cur.csv python tools/dobfs_probe.py 26 0.01 exact 0 > /dev/null 2>&1
ls -la gpurun_out/l_*.csv
