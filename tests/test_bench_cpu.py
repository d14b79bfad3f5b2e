"""bench.py's launch contract on CPU: --gpus N outside torchrun re-launches
itself with N ranks (torch.distributed.run, gloo for the dry run), and every
rank computes its z-slab of the configs[3] grid."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run_bench(*args):
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    env.pop("RANK", None)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args],
                         capture_output=True, text=True, timeout=300, env=env, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [json.loads(l) for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout  # rank 0 alone prints
    return lines[0]


@pytest.mark.parametrize("gpus", [1, 2, 4])
def test_gpus_flag_spawns_ranks(gpus):
    d = run_bench("--gpus", str(gpus), "--dry-run")
    assert d["n_gpus"] == gpus and d["config"] == 3
    parts = d["partitions"]
    assert len(parts) == gpus
    assert parts[0]["z0"] == 0 and parts[-1]["z1"] == 512
    assert sum(p["cells"] for p in parts) == d["cells"] == 512 ** 3
    for a, b in zip(parts, parts[1:]):
        assert a["z1"] == b["z0"] and a["cell0"] + a["cells"] == b["cell0"]


def test_reference_arm_dry_run_is_rank0_only():
    d = run_bench("--gpus", "2", "--impl", "reference", "--dry-run")
    assert d["impl"] == "reference" and d["n_gpus"] == 2
