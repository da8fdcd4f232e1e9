"""bench.py's reference arm (CPU, oracle/_ref) prints the contract's JSON line: the metric,
unit and workload descriptor of the B200 arm, impl = reference, a cpu_baseline describing
the run and an e2e object with zero host<->device bytes. Small workload so it runs here."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    from oracle.oracle import have_ref
    if not have_ref():
        pytest.skip("oracle/_ref not built")
    out = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--res", "32", "--cin", "8", "--cout",
                          "16", "--shapes-per-gpu", "1", "--steps", "1", "--warmup", "0"], cwd=ROOT,
                         capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference"
    assert line["metric"] == "hash-conv fwd+bwd occupied voxels/sec" and line["unit"] == "voxels/s"
    assert line["higher_is_better"] is True and line["value"] > 0
    for k in ("workload", "res", "shapes_per_gpu", "global_batch", "c_in", "c_out"):
        assert k in line["config"]
    assert line["cpu_baseline"]["kind"] == "reference" and line["cpu_baseline"]["value"] == line["value"]
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["d2h_bytes_per_step"] == 0
