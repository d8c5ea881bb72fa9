set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/r02b_pytest_gpu.log 2>&1; tail -3 gpurun_out/r02b_pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02b_smoke.log 2>&1; tail -2 gpurun_out/r02b_smoke.log
python bench.py --steps 64 --warmup 5 --no-cpu-baseline --workload cfg4 > gpurun_out/r02b_bench_cfg4.json 2> gpurun_out/r02b_bench_cfg4.err
python bench.py --steps 20 --warmup 3 --no-cpu-baseline --workload cfg5 > gpurun_out/r02b_bench_cfg5.json 2> gpurun_out/r02b_bench_cfg5.err
python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r02b_bench_cfg2.json 2> gpurun_out/r02b_bench_cfg2.err
cat gpurun_out/r02b_bench_*.json
