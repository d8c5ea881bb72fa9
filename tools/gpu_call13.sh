python bench.py --workload cfg4 --steps 64 --warmup 5 --no-cpu-baseline > gpurun_out/r02_bench_cfg4.json 2> gpurun_out/r02_bench_cfg4.err
python bench.py --workload cfg5 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/r02_bench_cfg5.json 2> gpurun_out/r02_bench_cfg5.err
free -g > gpurun_out/r02_free.txt
tail -3 gpurun_out/r02_bench_cfg4.err gpurun_out/r02_bench_cfg5.err
