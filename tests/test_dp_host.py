"""The C++ data-parallel host (hosts/dp_conv.cpp): the conv layer step driven from C++ through
the C ABI only (split-precision fwd, dW, dX; NCCL all-reduce of dW on a side stream for
WORLD_SIZE > 1), one process per GPU. One rank here (the box has one GPU)."""
import json
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "hosts", "_build", "dp_conv")


@pytest.mark.gpu
def test_cpp_dp_host_runs_the_layer(cuda):
    if not os.path.exists(BIN):
        pytest.skip("hosts/_build/dp_conv not built")
    env = dict(os.environ, RANK="0", WORLD_SIZE="1", LOCAL_RANK="0")
    r = subprocess.run([BIN, "--res", "64", "--shapes", "4", "--cin", "32", "--cout", "64", "--steps", "3",
                        "--warmup", "3"], capture_output=True, text=True, timeout=300, env=env)
    assert r.returncode == 0, r.stderr
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["n_gpus"] == 1 and line["dtype"] == "f32" and line["value"] > 0
    assert line["voxels_per_gpu"] == 4 * 14120 and line["gpu_launches"] >= 3 * 7


def test_cpp_dp_host_fails_loudly_without_device():
    import torch
    if torch.cuda.is_available() or not os.path.exists(BIN):
        pytest.skip("needs a GPU-less host and the built binary")
    r = subprocess.run([BIN, "--res", "16", "--shapes", "1"], capture_output=True, text=True, timeout=120)
    assert r.returncode != 0 and "dp_conv" in r.stderr
