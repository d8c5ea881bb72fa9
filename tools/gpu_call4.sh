set -x
python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -q -p no:cacheprovider -x -k "checksum or bitexact or golden or time_height" > gpurun_out/r02_pytest_gpu4.log 2>&1; tail -3 gpurun_out/r02_pytest_gpu4.log
python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r02_bench_s20.json 2> gpurun_out/r02_bench_s20.err
python bench.py --steps 64 --warmup 5 --no-cpu-baseline > gpurun_out/r02_bench_s64.json 2> gpurun_out/r02_bench_s64.err
for t in racecheck synccheck memcheck; do
  timeout 900 compute-sanitizer --tool $t --kernel-name-exclude kns=cub python tools/sanitize_cases.py > gpurun_out/r02_sanitize_$t.txt 2>&1
  tail -5 gpurun_out/r02_sanitize_$t.txt
done
