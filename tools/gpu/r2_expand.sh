# expansion rewrite: W case diagnostic, full GPU suite, A/B vs the committed
# numbers (reference schedule, graph loop, SSSP/BC timelines)
python tools/w_case.py > gpurun_out/w_case.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/gputest_exp.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/gputest_exp.log
for i in 1 2; do
timeout 300 python tools/graph_probe.py 26 ref 2>&1 | grep ref
timeout 300 python tools/graph_probe.py 26 graph 2>&1 | grep graph
done
timeout 300 python tools/timeline.py dobfs 26 0 > gpurun_out/tl_ref_src0_b.txt 2>&1
python tools/bench_configs.py > gpurun_out/configs_exp.jsonl 2> gpurun_out/configs_exp.err
