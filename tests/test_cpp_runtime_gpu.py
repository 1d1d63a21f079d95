"""The C++ training-step runtime (host/flexmoe_runtime.cpp) against the Python
runtime (paper_2304_03946_b200/runtime.py) on one B200: G ranks in process
(loopback: threads sharing the GPU), the same inputs, initial expert weights
and cluster profile. Both drive the same C ABI, so they must take the same
decisions (balance ratio per step bit-exact, the same ops applied / issued /
accepted at the same steps) and produce the same bytes: the last step's y on
every rank and every hosted expert's state (f32 master + Adam m/v) after the
migrations and optimizer steps. Covers both flip modes, the policy inline and
on the scheduler's worker thread, and both token transports."""
import json
import subprocess
from pathlib import Path

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2304_03946_b200 import scheduler as S  # noqa: E402
from paper_2304_03946_b200.distributed import LoopbackHub  # noqa: E402
from paper_2304_03946_b200.pool import ExpertStore  # noqa: E402
from paper_2304_03946_b200.runtime import FlexMoERuntime  # noqa: E402

from tests.test_multigpu_gpu import run_ranks  # noqa: E402

ROOT = Path(__file__).resolve().parents[1]
EXE = ROOT / "host" / "bin" / "flexmoe_runtime"
N, K, D, F, T, G, E, STEPS = 8, 2, 256, 256, 512, 4, 4, 10


def _inputs(dirpath: Path):
    gen = torch.Generator(device="cpu").manual_seed(0)
    wg = torch.randn(N, D, generator=gen) * D**-0.5
    wg[:, 0] = torch.tensor(np.log(1.0 / np.arange(1, N + 1) ** 1.5) * 2 + 3, dtype=torch.float32)
    xs = [torch.randn(T, D, generator=gen).to(torch.bfloat16) for _ in range(G)]
    for x in xs:
        x[:, 0] = 0.5
    dys = [(torch.randn(T, D, generator=gen) * 0.1).to(torch.bfloat16) for _ in range(G)]
    raw = lambda t: t.contiguous().view(torch.int16).numpy().tobytes()  # noqa: E731
    (dirpath / "wg.bin").write_bytes(raw(wg.to(torch.bfloat16)))
    for r in range(G):
        (dirpath / f"x_{r}.bin").write_bytes(raw(xs[r]))
        (dirpath / f"dy_{r}.bin").write_bytes(raw(dys[r]))
    experts = []
    for e in range(N):
        m = ExpertStore.init_expert(e, D, F)
        experts.append(torch.cat([m["w1"].reshape(-1), m["b1"], m["w2"].reshape(-1), m["b2"]]))
    (dirpath / "experts.bin").write_bytes(torch.stack(experts).numpy().astype(np.float32).tobytes())
    return wg, xs, dys


def _python_run(wg, xs, dys, transport, flip, async_policy):
    hub = LoopbackHub(G)

    def rank_fn(r):
        torch.cuda.set_device(0)
        rt = FlexMoERuntime(N, K, D, F, hub.endpoint(r), S.ClusterProfile.reference_default(G, E),
                            max_tokens=T, gate_weight=wg, lr=1e-3, transport=transport, flip=flip,
                            async_policy=async_policy)
        x, dy = xs[r].cuda(), dys[r].cuda()
        log = []
        for _ in range(STEPS):
            out = rt.step(x, dy)
            log.append((out.balance_ratio, [list(o) for o in out.applied], [list(o) for o in out.issued],
                        [list(o) for o in out.accepted]))
        torch.cuda.synchronize()
        states = {e: torch.cat([t.reshape(-1) for t in rt.store.state(e)]).cpu().numpy()
                  for e in rt.layer.local_experts}
        return log, out.y.contiguous().view(torch.int16).cpu().numpy(), states

    return run_ranks(G, rank_fn)


@pytest.mark.timeout(600)
@pytest.mark.parametrize("transport,flip,async_policy", [
    ("p2p", "copy", 1), ("p2p", "modelled", 0), ("nccl", "copy", 0)])
def test_cpp_runtime_matches_python_runtime(tmp_path, transport, flip, async_policy):
    if not EXE.exists():
        subprocess.run(["make", "-C", str(ROOT / "host"), "driver"], check=True, capture_output=True)
    wg, xs, dys = _inputs(tmp_path)
    dump = tmp_path / "dump"
    dump.mkdir()
    cmd = [str(EXE), "--loopback", str(G), "--steps", str(STEPS), "--warmup", "0", "--experts", str(N),
           "--topk", str(K), "--d-model", str(D), "--d-ff", str(F), "--tokens", str(T), "--slots", str(E),
           "--transport", transport, "--flip", flip, "--async-policy", str(async_policy), "--adam", "1",
           "--lr", "1e-3", "--profile", "reference", "--inputs", str(tmp_path), "--dump", str(dump),
           "--log-steps", "1"]
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=300)
    assert res.returncode == 0, res.stderr[-3000:]
    lines = [json.loads(s) for s in res.stdout.strip().splitlines()]
    steps, summary = lines[:-1], lines[-1]
    assert summary["p2p_timeouts"] == 0 and len(steps) == STEPS

    py = _python_run(wg, xs, dys, transport, flip, async_policy)
    log = py[0][0]
    for s in range(STEPS):
        ratio, applied, issued, accepted = log[s]
        assert steps[s]["balance_ratio"] == ratio, s
        assert steps[s]["applied"] == applied, s
        assert steps[s]["issued"] == issued, s
        assert steps[s]["accepted"] == accepted, s
    assert sum(len(st[1]) for st in log) > 0, "the skewed gate should change the placement"
    for r in range(G):
        y_cpp = np.fromfile(dump / f"y_{r}.bin", dtype=np.int16)
        assert np.array_equal(y_cpp, py[r][1].reshape(-1)), f"y differs on rank {r}"
        for e, st in py[r][2].items():
            st_cpp = np.fromfile(dump / f"state_{r}_{e}.bin", dtype=np.float32)
            assert np.array_equal(st_cpp, st), f"expert {e} state differs on rank {r}"
