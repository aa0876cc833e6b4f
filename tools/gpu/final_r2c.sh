# session-7 final: full GPU suite, bench N=1, N=2 (one GPU), per-config lines,
# ncu of the first pull (source 0), pull traffic + bench launch list
set -x
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/gputest_final.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/gputest_final.log
python bench.py > gpurun_out/bench_n1.json 2> gpurun_out/bench_n1.err; echo "bench rc=$?"
MG_BENCH_DEVICE=0 timeout 900 python bench.py --gpus 2 --steps 4 --warmup 3 > gpurun_out/bench_n2.json 2> gpurun_out/bench_n2.err; echo "n2 rc=$?"
python tools/bench_configs.py > gpurun_out/configs.jsonl 2> gpurun_out/configs.err; echo "configs rc=$?"
MG_NO_GRAPH=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:dobfs_pull_thread -c 1 -o gpurun_out/pull_0 python tools/dobfs_probe.py 26 0.01 exact 0 > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/pull_0.ncu-rep > gpurun_out/pull_0.txt 2>&1
bash tools/gpu/profile_r2.sh
