# Round-2 evidence: GPU suite, driver-style bench + reference arm, ncu launch
# list and one full capture of the headline kernel (k pinned: the in-run k
# trial times nonsense under a serialising profiler).
set -x
python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02_pytest_gpu_final.log 2>&1; tail -2 gpurun_out/r02_pytest_gpu_final.log
python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r02_bench_cfg2.json 2> gpurun_out/r02_bench_cfg2.err
python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/r02_bench_reference_arm.json 2> gpurun_out/r02_bench_reference_arm.err
python bench.py --steps 512 --warmup 5 --no-cpu-baseline > gpurun_out/r02_bench_cfg2_512.json 2> gpurun_out/r02_bench_cfg2_512.err
/usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02_headline_launches.csv python bench.py --steps 16 --warmup 3 --k 1 --no-e2e --no-cpu-baseline > gpurun_out/r02_ncu_launches.log 2>&1
/usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:acoustic_fused -s 6 -c 1 -o gpurun_out/r02_headline python bench.py --steps 6 --warmup 3 --k 1 --no-e2e --no-cpu-baseline > gpurun_out/r02_ncu_headline.log 2>&1
ls -la gpurun_out/r02_headline.ncu-rep
