"""The C++ host driver (host/flexmoe_step.cpp): one process per GPU, NCCL for
the histogram all-gather and gradient all-reduces, the layer's P2P token
transport through the C ABI — no Python in the step. On the single GPU of
the test box it runs at world 1 (its own arena through the P2P path)."""
import json
import os
import subprocess
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


@pytest.mark.timeout(300)
def test_cpp_host_driver_runs_the_p2p_step():
    exe = ROOT / "host" / "bin" / "flexmoe_step"
    if not exe.exists():  # built by __graft_entry__.build() / make -C host driver
        subprocess.run(["make", "-C", str(ROOT / "host"), "driver"], check=True, capture_output=True)
    cmd = [str(exe), "--gpus", "1", "--steps", "5", "--warmup", "2", "--experts", "16", "--topk", "2",
           "--tokens", "8192", "--replicate", "2"]
    # A world-1 run takes seconds and device P2P waits give up after ~20 s: a
    # stall is a bug, not noise — fail on the first one, with NCCL's own log.
    env = dict(os.environ, NCCL_DEBUG="WARN")
    try:
        res = subprocess.run(cmd, capture_output=True, text=True, timeout=120, env=env)
    except subprocess.TimeoutExpired as exc:
        pytest.fail(f"C++ driver stalled > 120 s; stderr tail: {(exc.stderr or b'')[-2000:]!r}")
    assert res.returncode == 0, res.stderr
    line = json.loads(res.stdout.strip().splitlines()[-1])
    assert line["p2p_timeouts"] == 0
    assert line["value"] > 0 and line["n_gpus"] == 1
    assert abs(line["balance_ratio"] - 1.0) < 1e-12  # one GPU receives everything
