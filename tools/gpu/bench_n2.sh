# N=2 bench with both ranks on GPU 0: device-driven loop (default) vs host loop
MG_BENCH_DEVICE=0 timeout 900 python bench.py --gpus 2 --steps 4 --warmup 3 > gpurun_out/bench_n2_dev.json 2> gpurun_out/bench_n2_dev.err; echo "dev rc=$?"
MG_MP_GRAPH_LOOP=0 MG_BENCH_DEVICE=0 timeout 900 python bench.py --gpus 2 --steps 4 --warmup 3 > gpurun_out/bench_n2_host.json 2> gpurun_out/bench_n2_host.err; echo "host rc=$?"
