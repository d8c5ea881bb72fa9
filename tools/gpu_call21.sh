python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_multi.py tests/test_tune.py -m gpu -q -p no:cacheprovider -x > gpurun_out/r02_pytest_capture.log 2>&1; tail -3 gpurun_out/r02_pytest_capture.log
python bench.py --steps 64 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r02_bench_cap.json 2>/dev/null
STB_NO_CAPTURE=1 python bench.py --steps 64 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r02_bench_nocap.json 2>/dev/null
python - <<'PY'
import json
for f in ("gpurun_out/r02_bench_cap.json", "gpurun_out/r02_bench_nocap.json"):
    d = json.loads(open(f).read())
    print(f, round(d["value"], 1), round(d["roofline"]["frac"], 4), d["gpu_launches"])
PY
