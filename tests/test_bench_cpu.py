"""CPU tests of bench.py's launch contract and its reference arm."""
import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402


def _env(**kw):
    env = {k: v for k, v in os.environ.items()
           if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    env.update(kw)
    return env


@pytest.mark.skipif(__import__("torch").cuda.device_count() >= 2, reason="needs a box with < 2 GPUs")
def test_more_gpus_than_visible_is_an_error():
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2"], capture_output=True,
                         text=True, timeout=300, env=_env())
    assert out.returncode == 2
    assert "needs 2 visible GPUs" in out.stderr
    assert out.stdout.strip() == ""


def test_world_size_mismatch_is_an_error():
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "4"], capture_output=True,
                         text=True, timeout=300, env=_env(WORLD_SIZE="2", RANK="0", LOCAL_RANK="0"))
    assert out.returncode == 2 and "WORLD_SIZE 2" in out.stderr


@pytest.mark.parametrize("workload,extra", [("single", ["--rows-per-gpu", "300000"]),
                                            ("c5", ["--c5-rows", "400000"]),
                                            ("batch", ["--batch", "7", "--batch-rows", "30000"])])
def test_reference_arm_prints_our_config(workload, extra):
    """The reference arm's `config` is the object our arm prints for the same
    arguments (bench.workload), so the driver pairs the two lines."""
    argv = ["--impl", "reference", "--workload", workload, "--steps", "1", "--warmup", "0", *extra]
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), *argv], capture_output=True, text=True,
                         timeout=300, env=_env())
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference"
    assert line["config"] == json.loads(json.dumps(bench.workload(bench.parse(argv), 1)))
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["cpu_baseline"]["kind"] == "port"
    assert line["value"] > 0 and line["scaling"] == line["config"]["scaling"]


def test_reference_arm_other_ranks_exit_quietly():
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--gpus", "2"],
                         capture_output=True, text=True, timeout=300,
                         env=_env(WORLD_SIZE="2", RANK="1", LOCAL_RANK="1"))
    assert out.returncode == 0 and out.stdout.strip() == ""


def test_traffic_is_quoted_only_for_its_build(tmp_path, monkeypatch):
    doc = {"build_hash": bench.kernel_build_hash(), "solve_level0_bytes_per_launch": 123}
    (tmp_path / "profiles").mkdir()
    (tmp_path / "profiles" / "ncu_traffic.json").write_text(json.dumps(doc))
    monkeypatch.setattr(bench, "ROOT", tmp_path)
    # the hash covers the real sources; with ROOT moved the sources are absent,
    # so recompute the doc's hash the same way
    doc["build_hash"] = bench.kernel_build_hash()
    (tmp_path / "profiles" / "ncu_traffic.json").write_text(json.dumps(doc))
    assert bench.traffic_for("solve_level0_bytes_per_launch")[0] == 123
    doc["build_hash"] = "0000"
    (tmp_path / "profiles" / "ncu_traffic.json").write_text(json.dumps(doc))
    v, why = bench.traffic_for("solve_level0_bytes_per_launch")
    assert v is None and why.startswith("stale")


def test_stamp_traffic_reads_the_committed_launch_lists(tmp_path):
    """tools/stamp_traffic.py on the committed round-2 launch lists gives the
    per-launch DRAM bytes of the committed stamp (same capture), and the
    level-0 traffic is the algorithmic 32 / 40 B per unknown within 1 %."""
    fin = ROOT / "profiles" / "round2" / "final"
    out = tmp_path / "t.json"
    r = subprocess.run([sys.executable, str(ROOT / "tools" / "stamp_traffic.py"),
                        "--single", str(fin / "launches_single_r2j.csv"),
                        "--batch", str(fin / "launches_batch_r2j.csv"),
                        "--batch-cluster", str(fin / "launches_cluster_r2j.csv"),
                        "--batch-stream", str(fin / "launches_stream_r2j.csv"),
                        "--f32", str(fin / "launches_f32_r2j.csv"), "--out", str(out)],
                       capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stderr
    doc = json.loads(out.read_text())
    ref = json.loads((fin / "ncu_traffic_r2j.json").read_text())
    for k in ("reduce_level0_bytes_per_launch", "solve_level0_bytes_per_launch",
              "batch_solve_level0_bytes_per_launch", "batch_stream_bytes_per_launch"):
        assert doc[k] == ref[k], k
    n = 80_000_000
    assert abs(doc["reduce_level0_bytes_per_launch"] / (32 * n) - 1) < 0.01
    assert abs(doc["solve_level0_bytes_per_launch"] / (40 * n) - 1) < 0.01
    assert abs(doc["solve_level0_f32_bytes_per_launch"] / (20 * n) - 1) < 0.02
    assert doc["build_hash"] == bench.kernel_build_hash()
