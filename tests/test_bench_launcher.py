"""CPU tests of bench.py's plumbing: `--gpus N` re-launches itself with N
ranks (torch.distributed.run, one process per GPU; gloo here) and reports the
max-over-ranks step time; the reference arm prints the same config dict as the
GPU arm."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def _json_lines(out):
    return [json.loads(ln) for ln in out.splitlines() if ln.startswith("{")]


def test_gpus_flag_launches_n_ranks():
    env = dict(os.environ)
    for k in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        env.pop(k, None)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2",
                        "--launcher-selftest", "--steps", "3"],
                       capture_output=True, text=True, timeout=300, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = _json_lines(r.stdout)
    assert len(lines) == 1                      # rank 0 alone prints
    ln = lines[0]
    assert ln["n_gpus"] == 2
    assert sorted(x["rank"] for x in ln["ranks"]) == [0, 1]
    assert len({x["pid"] for x in ln["ranks"]}) == 2          # one process per rank
    assert ln["ms_per_step"] == max(x["ms"] for x in ln["ranks"])


def test_reference_arm_prints_the_gpu_arm_config(monkeypatch, capsys):
    monkeypatch.setattr(bench, "N_POINTS", 12_000)

    class A:
        steps, warmup, gpus = 1, 0, 1
    bench.run_reference(A, 0, 1)
    ln = _json_lines(capsys.readouterr().out)[0]
    assert ln["impl"] == "reference"
    assert ln["config"] == bench.bench_config(1)
    assert ln["metric"] == bench.METRIC and ln["unit"] == "points/s"
    assert ln["e2e"]["h2d_bytes_per_step"] == 0
    assert ln["cpu_baseline"]["cores"] == (os.cpu_count() or 1)
    assert "no sampling" in ln["cpu_baseline"]["sample"]
