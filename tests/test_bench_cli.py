"""bench.py's process-count contract (CPU): --gpus N is authoritative."""
import json
import os
import subprocess
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, env_extra=None):
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    env.update(env_extra or {})
    return subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), *args],
                          capture_output=True, text=True, env=env, timeout=300)


def test_more_gpus_than_present_fails_loudly():
    # this container has no GPU: --gpus 2 must refuse instead of timing one device
    r = _run(["--gpus", "2", "--steps", "1", "--warmup", "0"])
    assert r.returncode != 0
    assert "refusing to report a 2-GPU number" in r.stderr
    assert '"n_gpus"' not in r.stdout


def test_world_size_must_match_gpus():
    r = _run(["--gpus", "1", "--steps", "1", "--warmup", "0"], {"WORLD_SIZE": "2"})
    assert r.returncode != 0
    assert "--gpus 1 but WORLD_SIZE=2" in r.stderr


def test_reference_arm_config_matches_ours_keys():
    """The reference arm's config carries only workload keys (parallelism is top-level),
    so the driver's same_config check compares like with like."""
    r = _run(["--impl", "reference", "--steps", "1", "--warmup", "0", "--ref-rows", "32",
              "--config", "c1"])
    assert r.returncode == 0, r.stderr
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference"
    assert "parallelism" not in line["config"] and "parallelism" in line
    sys.path.insert(0, REPO)
    import bench

    bench.select_workload("c1")
    assert line["config"] == json.loads(json.dumps(bench.workload_config()))
    assert line["e2e"]["h2d_bytes_per_step"] == 0
