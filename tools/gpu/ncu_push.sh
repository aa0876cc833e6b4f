# dense push: timeline of the reference schedule (source 0), ncu --set full of
# its two first push expansions, the A/B on the bench sources, DOBFS tests
set -x
timeout 300 python tools/timeline.py dobfs 26 0 > gpurun_out/tl_ref_src0.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:lb_expand_kernel -c 2 \
  -o gpurun_out/prof_push_ref python tools/dobfs_probe.py 26 0.01 ref 0 > gpurun_out/prof_push.log 2>&1
python tools/ncu_summary.py gpurun_out/prof_push_ref.ncu-rep > gpurun_out/prof_push_ref.txt 2>&1
for i in 1 2; do
timeout 300 python tools/graph_probe.py 26 ref 2>&1 | grep ref
MG_DOBFS_DENSE_ARCS=0 timeout 300 python tools/graph_probe.py 26 ref 2>&1 | sed 's/^ref/ref-off/' | grep ref
done
timeout 900 python -m pytest tests -m gpu -x -q -k "dobfs or bfs or dense" > gpurun_out/t_push.log 2>&1; tail -5 gpurun_out/t_push.log
