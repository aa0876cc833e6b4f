# full GPU suite, bench N=1 and the per-config lines on the current code
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/gputest_r2b.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/gputest_r2b.log
python bench.py > gpurun_out/bench_n1_b.json 2> gpurun_out/bench_n1_b.err; echo "bench rc=$?"
for i in 1 2; do timeout 300 python tools/graph_probe.py 26 ref 2>&1 | grep ref; done
