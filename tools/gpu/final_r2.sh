# round-2 final: full GPU suite, bench N=1, N=2 on one GPU, reference arm, per-config lines,
# ncu of the pull (sources 0 and 8582448), pull traffic, bench launch list
set -x
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/gputest_final.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/gputest_final.log
python bench.py > gpurun_out/bench_n1.json 2> gpurun_out/bench_n1.err; echo "bench rc=$?"
MG_BENCH_DEVICE=0 timeout 900 python bench.py --gpus 2 --steps 4 --warmup 3 > gpurun_out/bench_n2.json 2> gpurun_out/bench_n2.err; echo "n2 rc=$?"
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
python tools/bench_configs.py > gpurun_out/configs.jsonl 2> gpurun_out/configs.err; echo "configs rc=$?"
bash tools/gpu/ncu_pull.sh
bash tools/gpu/profile_r2.sh
