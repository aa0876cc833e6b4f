set -x
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/gputest_final.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/gputest_final.log
python bench.py > gpurun_out/bench_n1.json 2> gpurun_out/bench_n1.err; echo "bench rc=$?"
python tools/bench_configs.py > gpurun_out/configs.jsonl 2> gpurun_out/configs.err; echo "configs rc=$?"
python -c "import __graft_entry__ as g; g.smoke()"; echo "smoke rc=$?"
