# the driver's bench contract at N=1, then N=2 with both ranks on GPU 0
python bench.py > gpurun_out/bench_n1.json 2> gpurun_out/bench_n1.err; echo "n1 rc=$?"
MG_BENCH_DEVICE=0 timeout 900 python bench.py --gpus 2 --steps 4 --warmup 3 > gpurun_out/bench_n2.json 2> gpurun_out/bench_n2.err; echo "n2 rc=$?"
tail -c 600 gpurun_out/bench_n1.err; tail -c 600 gpurun_out/bench_n2.err
