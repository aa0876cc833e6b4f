# push iteration: reference-schedule and graph-loop totals over the bench
# sources, SSSP/BC timelines, ncu of the heavy push of source 0
for i in 1 2; do
timeout 300 python tools/graph_probe.py 26 ref 2>&1 | grep ref
timeout 300 python tools/graph_probe.py 26 graph 2>&1 | grep graph
done
timeout 300 python tools/timeline.py sssp 24 2>&1 | grep -E "device_ms|span"
timeout 300 python tools/timeline.py bc 24 2>&1 | grep -E "device_ms|span"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:lb_expand_kernel -s 1 -c 1 \
  -o gpurun_out/prof_push_ref2 python tools/dobfs_probe.py 26 0.01 ref 0 > gpurun_out/prof_push2.log 2>&1
python tools/ncu_summary.py gpurun_out/prof_push_ref2.ncu-rep > gpurun_out/prof_push_ref2.txt 2>&1
