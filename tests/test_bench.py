"""CPU: bench.py's contract pieces that run without a GPU.

* its workload table mirrors the library's (shapes, profile files);
* the reference arm loads only oracle/ (never this repo's library or torch),
  honours --steps/--warmup and prints the same config dict our arm builds;
* `python bench.py --gpus N` self-spawns N ranks (torch.distributed.run) and
  rank 0 prints one JSON line; exercised here on gloo with the oracle codec
  injected as the backend (a harness test of the exchange driver, not a
  measurement).
"""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from paper_2407_04272_b200 import workload as W  # noqa: E402


def _json_line(out: str) -> dict:
    lines = [ln for ln in out.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out[-3000:]
    return json.loads(lines[0])


def test_bench_workloads_mirror_library():
    for name, b in bench.BENCH_WORKLOADS.items():
        w = W.WORKLOADS[name]
        for k in ("tables", "dim", "profiles", "global_eb", "desc"):
            assert b[k] == w[k], (name, k)
        for R in (1, 2, 4, 8):
            assert b["batch"](R) == w["batch"](R)
        specs = W.workload_specs(name)
        assert [list(map(float, (s.rows, s.dist, s.mu, s.sigma, s.lo, s.hi, s.zipf))) for s in specs] == \
            [list(map(float, t)) for t in bench.preset_tables(name)]


def test_reference_arm_is_clean_and_same_config(ref):
    code = ("import sys, runpy; sys.argv=['bench.py','--impl','reference','--steps','4','--warmup','3'];"
            "runpy.run_path('bench.py', run_name='__main__');"
            "bad=[m for m in sys.modules if m.startswith('paper_2407_04272_b200') or m=='torch'];"
            "print('LOADED', bad, file=sys.stderr);"
            "maps=open('/proc/self/maps').read();"
            "print('SO', 'libembc_cuda' in maps, file=sys.stderr)")
    r = subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    assert "LOADED []" in r.stderr and "SO False" in r.stderr
    line = _json_line(r.stdout)
    assert line["impl"] == "reference" and line["steps"] == 4 and line["warmup"] == 3
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["cpu_baseline"]["kind"] == "reference"
    # our arm's config for the same workload (profiles read by the library's read_profiles)
    prof = W.workload_profiles("kg")
    step = 26 * 2048 * 16 * 4
    ours = bench.make_config("kg", 1, [prof[t].codec for t in range(26)], [prof[t].eb for t in range(26)],
                             bench.input_sets(step), step)
    assert line["config"] == json.loads(json.dumps(ours))


@pytest.mark.parametrize("world", [2, 3])
def test_multi_rank_spawn_gloo(world):
    cmd = [sys.executable, "bench.py", "--gpus", str(world), "--cpu-test", "--codec-backend",
           "tests/test_exchange_gloo.py:OracleCodec", "--steps", "2", "--warmup", "1", "--workload", "tb"]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    line = _json_line(r.stdout)
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "e2e", "exchange", "clocks", "gpu_launches"):
        assert k in line, k
    assert line["n_gpus"] == world
    ex = line["exchange"]
    assert ex["compression_ratio_fwd"] > 1 and ex["compression_ratio_bwd"] > 1
    assert line["e2e"]["h2d_bytes_per_step"] > 0 and line["e2e"]["d2h_bytes_per_step"] > 0


def test_adaptive_schedule_phases_gloo():
    cmd = [sys.executable, "bench.py", "--gpus", "2", "--cpu-test", "--codec-backend",
           "tests/test_exchange_gloo.py:OracleCodec", "--adaptive", "8"]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    line = _json_line(r.stdout)
    ph = line["phases"]
    assert [ph[f"stair{k}"]["eb_multiplier"] for k in range(4)] == pytest.approx([2.0, 5 / 3, 4 / 3, 1.0])
    assert ph["post_decay"]["iterations"] == 4
    # a larger bound never compresses worse on the same inputs
    assert ph["stair0"]["compression_ratio_bwd"] >= ph["post_decay"]["compression_ratio_bwd"]
