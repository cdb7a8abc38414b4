"""bench.py's CPU-side logic: the bounded reference sample reproduces the
reference solver's own attempts (same block, improved graphs, forbidden
clique), and the JSON contract keys are present in the reference arm's line."""
import json
import os
import subprocess
import sys

import pytest

from conftest import REPO


@pytest.fixture(scope="module")
def bench():
    sys.path.insert(0, REPO)
    import bench as b
    return b


def test_induced_subgraph(bench):
    rows = [0b0110, 0b1001, 0b1001, 0b0110]  # 4-cycle 0-1-3-2-0
    assert bench._induced(rows, [0, 1, 3]) == [0b010, 0b101, 0b010]


def test_reference_sample_matches_reference_solve(bench, ref):
    """The sample's per-k expanded counts are exactly the reference solve's
    attempts on the same graph (solver.cpp:21-67)."""
    from paper_1709_09990_b200 import generators as G
    rows = G.random_graph(1, 24, 0.3)
    got = bench.reference_sample(rows, threads=2, budget_s=1e9)[2]
    r = ref.solve(rows, dedup="exact", threads=2, cap=bench.CAP)
    stats = json.loads(r["stats"])
    comp = max(stats["components"], key=lambda c: len(c["vertices"]))
    want = [(a["k"], sum(l["expanded"] for l in a["layers"])) for a in comp["attempts"]]
    assert [(k, e) for k, e, _ in got] == want


def test_reference_arm_line(ref):
    env = dict(os.environ)
    out = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "1", "--warmup", "0",
                          "--ref-budget", "0.01"], cwd=REPO, capture_output=True, text=True, env=env,
                         timeout=600)
    assert out.returncode == 0, out.stderr[-1000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "impl", "cpu_baseline", "e2e"):
        assert key in line, key
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["e2e"]["h2d_bytes_per_step"] == 0


def test_gpus_flag_relaunches_under_torchrun(bench):
    """`bench.py --gpus N` outside torchrun re-launches itself as N ranks on
    127.0.0.1 (one process per GPU)."""
    argv = bench.torchrun_argv(["--gpus", "4", "--steps", "2"], 4, port=29999)
    assert argv[1:4] == ["-m", "torch.distributed.run", "--nnodes=1"]
    assert "--nproc-per-node=4" in argv and "--master-addr=127.0.0.1" in argv
    assert argv[-4:] == ["--gpus", "4", "--steps", "2"] and argv[-5].endswith("bench.py")


def test_gpus_flag_fails_loudly_without_enough_devices():
    """No silent N=1 number for --gpus 2: with fewer visible GPUs the bench
    exits non-zero and says why (this container has none)."""
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    p = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), "--gpus", "2"],
                       env=env, capture_output=True, text=True, timeout=300)
    assert p.returncode == 2
    line = json.loads(p.stdout.strip().splitlines()[-1])
    assert line["n_gpus"] == 2 and "needs 2 visible CUDA devices" in line["error"]


def test_world_mismatch_is_an_error():
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    p = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), "--gpus", "2"],
                       env=env, capture_output=True, text=True, timeout=300)
    assert p.returncode != 0 and "WORLD_SIZE=1" in p.stderr
