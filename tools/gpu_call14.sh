python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02_pytest_gpu_full.log 2>&1; tail -3 gpurun_out/r02_pytest_gpu_full.log
python bench.py --workload cfg5 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/r02_bench_cfg5b.json 2> gpurun_out/r02_bench_cfg5b.err
python -c "import json; d=json.loads(open('gpurun_out/r02_bench_cfg5b.json').read()); print(d['value'], d['e2e'])"
