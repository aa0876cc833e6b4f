M=gpu__time_duration.sum,smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum
MG_NO_GRAPH=1 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/s3_on.csv python tools/dobfs_probe.py 26 0.01 exact 8863776 > gpurun_out/s3_on.log 2>&1
MG_NO_GRAPH=1 MG_DOBFS_DENSE_ARCS=0 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/s3_off.csv python tools/dobfs_probe.py 26 0.01 exact 8863776 > gpurun_out/s3_off.log 2>&1
