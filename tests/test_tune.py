"""Tune/bench harness (paper_2010_10248_b200.tune) with the reference's CSV
semantics (cli.py:289-440; mirrors pkg/tests/test_cli.py TestTune/TestBench).

CPU tests drive the harness with a stand-in runner that applies the same
plan legality as the device path (engine._gpu_time_height) and returns a
deterministic report; ``-m gpu`` tests run the real GPU path."""

import csv
import json
import os
from types import SimpleNamespace

import pytest

import paper_2010_10248_b200 as stb
from paper_2010_10248_b200 import engine, tune

BASE = {
    "physics": "acoustic",
    "grid": {"shape": [24, 24, 24], "spacing_m": [10.0, 10.0, 10.0], "boundary_layers": 4},
    "space_order": 4,
    "nt": 16,
    "medium": {"velocity_m_s": 2500.0},
    "schedule": {"kind": "wavefront", "time_height": 2, "tile_shape": [16, 16],
                 "block_shape": [16, 16]},
    "source": {"f0_hz": 14.0, "coords_m": [[115.0, 115.0, 115.0]]},
    "receivers": {"coords_m": [[115.0, 115.0, 75.0]]},
    "precision": 32,
}


def fake_runner(config):
    k = engine._gpu_time_height(config)          # same legality errors as the device path
    rep = SimpleNamespace(gpoints_per_s=1.0 + 0.1 * max(k, 1), elapsed_s=0.01)
    return SimpleNamespace(report=rep)


def write(tmp_path, doc, name):
    p = tmp_path / name
    p.write_text(json.dumps(doc))
    return str(p)


def test_single_candidate(tmp_path):
    cfg = write(tmp_path, dict(BASE, nt=6), "cfg.json")
    sw = write(tmp_path, {"tile_shapes": [[16, 16]], "time_heights": [2], "repetitions": 1,
                          "warmup": 0}, "sweep.json")
    out = tmp_path / "tune.csv"
    assert tune.main(["tune", "--config", cfg, "--sweep", sw, "--out", str(out)],
                     runner=fake_runner) == 0
    lines = out.read_text().splitlines()
    assert lines[0] == ",".join(tune.TUNE_COLUMNS)
    assert len(lines) == 2 and lines[1].endswith(",1")


def test_invalid_candidate_skipped(tmp_path):
    cfg = write(tmp_path, dict(BASE, nt=6), "cfg.json")
    # tile 8 <= skew*T for T=8 at radius 2: skipped, not fatal
    sw = write(tmp_path, {"tile_shapes": [[8, 8], [20, 20]], "time_heights": [8],
                          "repetitions": 1, "warmup": 0}, "sweep.json")
    out = tmp_path / "tune.csv"
    assert tune.main(["tune", "--config", cfg, "--sweep", sw, "--out", str(out)],
                     runner=fake_runner) == 0
    lines = out.read_text().splitlines()
    assert len(lines) == 3
    assert "skipped" in lines[1] and "ok" in lines[2]


def test_three_by_three_and_lf(tmp_path):
    cfg = write(tmp_path, dict(BASE, nt=4), "cfg.json")
    sw = write(tmp_path, {"tile_shapes": [[16, 16], [20, 20], [24, 24]],
                          "time_heights": [1, 2, 4], "repetitions": 1, "warmup": 0},
               "sweep.json")
    out = tmp_path / "tune.csv"
    assert tune.main(["tune", "--config", cfg, "--sweep", sw, "--out", str(out)],
                     runner=fake_runner) == 0
    text = out.read_text()
    assert len(text.splitlines()) == 10 and "\r" not in text
    rows = list(csv.reader(text.splitlines()))[1:]
    assert [r[0] for r in rows] == ["wavefront"] * 9
    assert [int(r[5]) for r in rows] == [1, 2, 4] * 3
    assert sum(r[-1] == "1" for r in rows) == 1


def test_gpu_kind_candidates_and_no_valid_candidate(tmp_path):
    doc = dict(BASE, schedule={"kind": "gpu", "time_height": 0})
    cfg = tune.parse_config(doc)
    rows, best = tune.tune(cfg, tune.SweepSpec([], [], [1, 2, 3], 1, 0), fake_runner)
    assert [r[5] for r in rows] == [1, 2, 3] and rows[best][5] == 3
    rows, best = tune.tune(cfg, tune.SweepSpec([], [], [-1], 1, 0), fake_runner)
    assert best is None and rows[0][6] == "skipped"
    with pytest.raises(stb.ConfigError):
        list(tune.candidates(tune.parse_config(dict(BASE, schedule={"kind": "naive"})),
                             tune.SweepSpec([], [], [1], 1, 0)))


def test_bench_rows(tmp_path):
    cfg_path = write(tmp_path, dict(BASE, nt=6), "cfg.json")
    suite = tmp_path / "suite.json"
    suite.write_text(json.dumps({"rows": [
        {"config": os.path.basename(cfg_path), "blocks": [[16, 16]], "tiles": [[16, 16]],
         "time_heights": [1], "repetitions": 1, "warmup": 0},
        {"config": "missing.json"}]}))
    out = tmp_path / "bench.csv"
    assert tune.main(["bench", "--suite", str(suite), "--out", str(out)],
                     runner=fake_runner) == 0
    with open(out, newline="") as fh:
        rows = list(csv.reader(fh))
    assert rows[0] == tune.BENCH_COLUMNS
    cells = rows[1]
    assert cells[0] == "acoustic" and cells[2] == "24x24x24" and cells[4] == "16x16"
    assert float(cells[8]) == pytest.approx(1.0)
    assert rows[2][-1] and rows[2][0] == ""          # failing row recorded


def test_config_errors_name_fields(tmp_path, capsys):
    bad = dict(BASE, space_order=5)
    assert tune.main(["tune", "--config", write(tmp_path, bad, "c.json"),
                      "--sweep", write(tmp_path, {"time_heights": [1]}, "s.json")],
                     runner=fake_runner) == 2
    assert "space_order" in capsys.readouterr().err
    doc = json.loads(json.dumps(BASE))
    del doc["medium"]["velocity_m_s"]
    with pytest.raises(stb.ConfigError) as e:
        tune.parse_config(doc)
    assert e.value.field == "medium.velocity_m_s"
    with pytest.raises(stb.ConfigError):
        tune.SweepSpec([], [], [], 1, 0)


def test_tti_and_layout_configs():
    doc = dict(BASE, physics="tti", space_order=8,
               medium={"vp_m_s": 2500.0, "epsilon": 0.2, "delta": 0.1, "theta_rad": 0.3},
               source={"f0_hz": 15.0, "layout": {"count": 5, "mode": "plane", "seed": 3}})
    cfg = tune.parse_config(doc)
    assert cfg.physics == "tti" and cfg.medium["epsilon"] == 0.2 and cfg.medium["theta"] == 0.3
    assert cfg.sources.coords.shape == (5, 3)
    assert (cfg.sources.coords[:, 2] == 115.0).all()


@pytest.mark.gpu
def test_gpu_tune_and_bench_real_runs(tmp_path):
    cfg = write(tmp_path, dict(BASE, nt=6), "cfg.json")
    sw = write(tmp_path, {"tile_shapes": [[8, 8], [20, 20]], "time_heights": [1, 4],
                          "repetitions": 1, "warmup": 0}, "sweep.json")
    out = tmp_path / "tune.csv"
    assert tune.main(["tune", "--config", cfg, "--sweep", sw, "--out", str(out)]) == 0
    rows = list(csv.reader(out.read_text().splitlines()))[1:]
    assert [r[6] for r in rows] == ["ok", "skipped", "ok", "ok"]
    assert all(float(r[7]) > 0 for r in rows if r[6] == "ok")
    suite = tmp_path / "suite.json"
    suite.write_text(json.dumps({"rows": [{"config": "cfg.json", "blocks": [[16, 16]],
                                           "tiles": [[16, 16]], "time_heights": [1, 2],
                                           "repetitions": 1, "warmup": 1}]}))
    bout = tmp_path / "bench.csv"
    assert tune.main(["bench", "--suite", str(suite), "--out", str(bout)]) == 0
    cells = list(csv.reader(bout.read_text().splitlines()))[1]
    assert cells[-1] == "" and float(cells[8]) > 0
