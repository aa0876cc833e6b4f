# full GPU test suite, then the driver's bench contract at N=1 and the reference arm
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/gputest_r2.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/gputest_r2.log
python bench.py > gpurun_out/bench_n1.json 2> gpurun_out/bench_n1.err; echo "bench rc=$?"
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
