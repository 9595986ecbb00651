"""bench.py's launcher (`python bench.py --gpus N` without torchrun) and the
reference arm's JSON line: N=2 gloo ranks on 127.0.0.1, one JSON line with
n_gpus 2, and the same `config` keys as the GPU arm (static_config)."""
import json
import os
import subprocess
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _json_lines(out):
    return [json.loads(l) for l in out.splitlines() if l.startswith("{")]


def test_launcher_two_ranks_reference_arm():
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    r = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), "--impl", "reference", "--gpus", "2",
                        "--workload", "ntdm", "--steps", "1", "--warmup", "3"],
                       capture_output=True, text=True, env=env, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = _json_lines(r.stdout)
    assert len(lines) == 1, r.stdout
    line = lines[0]
    assert line["impl"] == "reference" and line["n_gpus"] == 2
    assert line["config"]["parallelism"] == "dp2 (system-index sharding)"
    assert line["cpu_baseline"]["cores"] == len(os.sched_getaffinity(0))


def test_world_size_mismatch_fails_loudly():
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), "--impl", "reference", "--gpus", "2",
                        "--workload", "ntdm", "--steps", "1"], capture_output=True, text=True, env=env,
                       timeout=300)
    assert r.returncode != 0 and "WORLD_SIZE=1" in (r.stderr + r.stdout)


@pytest.mark.parametrize("workload", ["npdm", "mnpdm", "ntdm", "ntdm8k", "sip", "stdm", "spdm", "hb", "adi"])
def test_config_is_the_same_for_both_arms(workload):
    sys.path.insert(0, REPO)
    import argparse
    import bench
    a = argparse.Namespace(workload=workload, algo="partitioned", layout="system")
    c1 = bench.static_config(a, 1)
    assert c1["workload"] and c1["parallelism"]
    # the reference arm prints static_config too; nothing data-dependent in it
    assert json.loads(json.dumps(c1)) == c1
