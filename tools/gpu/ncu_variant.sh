# per-launch ncu metrics of the pull kernels (source ${SRC:-0}) for the default build and variant $1
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum
ncu --metrics $M --clock-control none -k regex:"dobfs_pull" --csv --log-file gpurun_out/nv_def.csv python tools/dobfs_probe.py 26 0.01 exact ${SRC:-0} > /dev/null 2>&1
MG_LIB_PATH=paper_1504_04804_b200/libmgraph_b200_$1.so ncu --metrics $M --clock-control none -k regex:"dobfs_pull" --csv --log-file gpurun_out/nv_var.csv python tools/dobfs_probe.py 26 0.01 exact ${SRC:-0} > /dev/null 2>&1
