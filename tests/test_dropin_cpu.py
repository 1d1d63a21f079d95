"""Drop-in check against the reference's own program (no GPU needed).

host/Makefile builds the reference's tests/acceptance.cpp twice: once on the
unmodified moesim sources, once with proj/src/router.cpp and policy.cpp
replaced by host/moesim_b200 — moesim's routing and placement-policy API
served by libflexmoe_b200.so (route, received_matrix, per_gpu_received,
balance_ratio, make_scheduling_plan, plan_migrations through the C ABI).
Every SimEngine step, policy what-if and oracle call of the acceptance suite
then runs on this framework's host code. The drop-in must pass all ten
criteria with byte-identical output. Needs /root/reference (skipped on the
GPU box, where the reference does not exist)."""
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
REF = Path("/root/reference/proj")

pytestmark = pytest.mark.skipif(not (REF / "tests" / "acceptance.cpp").exists(),
                                reason="reference sources not present")


@pytest.mark.timeout(600)
def test_reference_acceptance_with_b200_router_and_policy():
    lib = ROOT / "paper_2304_03946_b200" / "libflexmoe_b200.so"
    if not lib.exists():
        pytest.skip("native library not built")
    subprocess.run(["make", "-C", str(ROOT / "host"), "-j8"], check=True, capture_output=True, text=True)
    out = {}
    for name in ("acceptance_ref", "acceptance_b200"):
        res = subprocess.run([str(ROOT / "host" / "_build" / name)], capture_output=True, text=True, timeout=300)
        assert res.returncode == 0, f"{name} failed:\n{res.stdout}\n{res.stderr}"
        out[name] = res.stdout
    assert "all criteria passed" in out["acceptance_b200"]
    assert out["acceptance_b200"].count("[PASS]") == 10
    assert out["acceptance_b200"] == out["acceptance_ref"], "drop-in output differs from the reference"
