"""bench.py's multi-GPU plumbing on CPU: `--gpus N` outside torchrun starts N
ranks itself (torch.distributed.run, rendezvous on 127.0.0.1) and rank 0
reports n_gpus = N (gloo here; NCCL on a GPU box)."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_gpus_2_self_launches_two_ranks():
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2",
                          "--launch-check"], capture_output=True, text=True, timeout=600,
                         env=env, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [json.loads(x) for x in out.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, out.stdout
    rec = lines[0]
    assert rec["n_gpus"] == 2 and rec["requested"] == 2
    assert rec["rank_sum"] == 1.0          # both ranks joined the group


def test_bench_cpu_info_has_model_and_physical_cores():
    sys.path.insert(0, ROOT)
    import bench
    info = bench.host_cpu_info()
    assert info["logical_cpus"] == os.cpu_count()
    assert info["physical_cores"] is None or 1 <= info["physical_cores"] <= os.cpu_count()
