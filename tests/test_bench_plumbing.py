"""bench.py's launch plumbing on CPU: `--gpus 2` without WORLD_SIZE re-launches
itself under torch.distributed.run (2 ranks, gloo in --dry-run), rank 0
prints one JSON line with n_gpus = 2 after barriers and a max-over-ranks
time; and the reference arm prints the contract's line with the same
`config` the GPU arm builds (bench.config_dict)."""

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _last_json(out):
    lines = [ln for ln in out.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out
    return json.loads(lines[0])


@pytest.mark.timeout(300)
def test_bench_relaunches_two_ranks_dry_run():
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--dry-run",
                        "--steps", "3", "--warmup", "1"], capture_output=True, text=True,
                       env=env, timeout=280)
    assert r.returncode == 0, r.stderr[-2000:]
    line = _last_json(r.stdout)
    assert line["n_gpus"] == 2 and line["ranks_reporting"] == 2 and line["dry_run"]
    assert line["steps"] == 3 and line["warmup"] == 1 and line["value"] > 0


@pytest.mark.timeout(600)
def test_reference_arm_line_matches_gpu_arm_config():
    sys.path.insert(0, ROOT)
    import bench
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                        "--steps", "1", "--warmup", "1"], capture_output=True, text=True,
                       timeout=580)
    assert r.returncode == 0, r.stderr[-2000:]
    line = _last_json(r.stdout)
    assert line["impl"] == "reference" and line["unit"] == "interactions/s"
    assert line["cpu_baseline"]["kind"] == "port" and line["cpu_baseline"]["value"] == line["value"]
    assert line["e2e"]["h2d_bytes_per_step"] == 0

    class A:
        theta, seed, default_g, n = 0.5, 3, False, 1_000_000
    want = bench.config_dict(A, 1_000_000, 1_000_000, line["config"]["tree_nodes"], 1)
    assert line["config"] == want
    assert line["config"]["tree_nodes"] == 1479591  # the GPU arm's tree (topology bit-exact)
