"""CPU checks of the bench.py contract the driver depends on: the metric is BASELINE.json's,
every workload has a config naming it, and the CLI parses (no GPU needed)."""
import json
import os
import subprocess
import sys
from types import SimpleNamespace

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402

WORKLOADS = ["all", "sht", "disco", "disco_t", "block", "decoder", "dist_sht", "dist_disco"]


def test_metric_is_baselines():
    with open(os.path.join(ROOT, "BASELINE.json")) as f:
        assert bench.METRIC == json.load(f)["metric"]


@pytest.mark.parametrize("w", WORKLOADS)
def test_workload_config(w):
    cfg = bench.workload_config(SimpleNamespace(workload=w, gpus=1, decomp=""))
    assert isinstance(cfg, dict) and cfg.get("workload")
    assert not ({"model", "global_batch", "seq_len"} & set(cfg))  # no ML model keys


def test_cli_parses():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--help"], capture_output=True,
                         text=True, timeout=120)
    assert out.returncode == 0
    for flag in ("--gpus", "--steps", "--warmup", "--impl", "--workload"):
        assert flag in out.stdout
