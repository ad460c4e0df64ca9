"""bench.py's reference arm (the CPU leg the driver times beside ours): one
JSON line with the contract's keys, rank 0 only under torchrun."""

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ARGS = ["--impl", "reference", "--tuples", "4000", "--steps", "1", "--cpu-pairs", "400000"]


def _lines(out):
    return [json.loads(x) for x in out.splitlines() if x.startswith("{")]


@pytest.mark.parametrize("workload", ["citation3", "linkage"])
def test_reference_arm_line(workload):
    r = subprocess.run([sys.executable, "bench.py", *ARGS, "--workload", workload], cwd=ROOT,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    (line,) = _lines(r.stdout)
    assert line["impl"] == "reference" and line["unit"] == "pairs/s" and line["value"] > 0
    assert line["warmup"] >= 3 and line["n_gpus"] == 1 and line["higher_is_better"] is True
    assert line["cpu_baseline"]["kind"] == "port" and line["cpu_baseline"]["value"] == line["value"]
    assert line["e2e"] == {"value": line["value"], "unit": "pairs/s", "h2d_bytes_per_step": 0,
                           "d2h_bytes_per_step": 0}
    assert line["config"]["workload"].startswith(workload)


def test_reference_arm_rank0_only_under_torchrun():
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", "29631", "bench.py", *ARGS, "--gpus", "2"],
                       cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    (line,) = _lines(r.stdout)
    assert line["impl"] == "reference" and line["n_gpus"] == 2


def test_gpus_flag_relaunches_under_torchrun():
    """--gpus N without a torchrun environment re-launches N ranks
    (torch.distributed.run on 127.0.0.1); rank 0 prints the one line."""
    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, "bench.py", *ARGS, "--gpus", "2", "--workload", "citation3"], cwd=ROOT,
                       capture_output=True, text=True, timeout=600, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    (line,) = _lines(r.stdout)
    assert line["n_gpus"] == 2 and line["impl"] == "reference" and line["scaling"] == "strong"


def test_default_reference_arm_is_the_metric_config():
    """The default workload is BASELINE config 4 (i) (the metric's own
    configuration); a small relation keeps this test fast."""
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--tuples", "20000", "--steps", "1",
                        "--cpu-pairs", "2000000"], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    (line,) = _lines(r.stdout)
    assert line["config"]["workload"].startswith("person5_pipeline n=20000")
    assert "config 4 (i)" in line["config"]["workload"]


@pytest.mark.gpu
def test_two_ranks_on_one_gpu_strong_scaling():
    """--gpus 2 on a 1-GPU box: both ranks share the GPU and exchange over
    gloo; the line reports both ranks' pairs (strong scaling of one relation)."""
    r = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--tuples", "200000", "--steps", "3",
                        "--no-secondary", "--no-cpu"], cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    (line,) = _lines(r.stdout)
    assert line["n_gpus"] == 2 and line["scaling"] == "strong" and line["value"] > 0
    r1 = subprocess.run([sys.executable, "bench.py", "--tuples", "200000", "--steps", "3", "--no-secondary",
                         "--no-cpu"], cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert r1.returncode == 0, r1.stderr[-3000:]
    (one,) = _lines(r1.stdout)
    assert line["config"]["pairs_per_step"] == one["config"]["pairs_per_step"]  # the same relation, split
