# compute-sanitizer over the small-graph cases (every primitive at n = 1/2/3,
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -n 2
# the pull kernels, the device loop, the dense exchange) and the two-process
# CUDA-IPC fabric; one log per tool under gpurun_out/
CS="compute-sanitizer --print-limit 50 --target-processes all"
for tool in memcheck synccheck initcheck; do
  timeout 1200 $CS --tool $tool python tools/sanitize_cases.py > gpurun_out/san_$tool.txt 2>&1
  echo "exit $?" >> gpurun_out/san_$tool.txt
done
timeout 1200 $CS --tool memcheck python tools/sanitize_cases.py --mp > gpurun_out/san_memcheck_mp.txt 2>&1
echo "exit $?" >> gpurun_out/san_memcheck_mp.txt
timeout 1800 $CS --tool racecheck --racecheck-report analysis python tools/sanitize_cases.py > gpurun_out/san_racecheck.txt 2>&1
echo "exit $?" >> gpurun_out/san_racecheck.txt
for f in gpurun_out/san_*.txt; do tail -n 3 $f; done
