"""bench.py's reference arm (CPU: the reference's own receiver sources, oracle/_ref) keeps the
driver's JSON contract, alone and under torchrun with two ranks (rank 0 prints, the others exit
0).  The GPU arm's line is checked by the round-end bench run itself."""
import json
import os
import subprocess
import sys

import pytest

import oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _lines(cmd):
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    return [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]


def _check(line):
    assert line["impl"] == "reference"
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in line, k
    assert line["value"] > 0 and line["higher_is_better"] is True
    assert line["config"]["workload"].startswith("cfg4")
    cb = line["cpu_baseline"]
    assert cb["kind"] in ("reference", "port") and cb["cores"] >= 1 and cb["value"] == line["value"] and cb["sample"]
    e2e = line["e2e"]
    assert e2e["value"] == line["value"] and e2e["unit"] == line["unit"]
    assert e2e["h2d_bytes_per_step"] == 0 and e2e["d2h_bytes_per_step"] == 0


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
def test_reference_arm_json_contract():
    lines = _lines([sys.executable, "bench.py", "--impl", "reference", "--steps", "1", "--warmup", "1"])
    assert len(lines) == 1
    _check(lines[0])


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
def test_reference_arm_under_torchrun_two_ranks():
    lines = _lines([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                    "--master-addr", "127.0.0.1", "--master-port", "29537", "bench.py", "--impl", "reference",
                    "--gpus", "2", "--steps", "1", "--warmup", "1"])
    assert len(lines) == 1  # rank 0 only
    _check(lines[0])
