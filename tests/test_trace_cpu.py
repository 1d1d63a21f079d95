"""Trace export / replay against the reference's own
save_trace / load_trace (proj/src/workload.cpp:175-341, compiled into
oracle/_ref). Cases follow proj/tests/test_workload.cpp:204-270.
"""
import numpy as np
import pytest

from paper_2304_03946_b200 import _lib as L
from paper_2304_03946_b200 import trace as TR

import oracle

ref_missing = not oracle.Reference.available()
needs_ref = pytest.mark.skipif(ref_missing, reason="oracle/_ref not built")


@needs_ref
@pytest.mark.parametrize("N,G,tokens,zipf,drift,seed,steps", [
    (8, 4, 1024, 1.2, 0.03, 3, 5),       # test_workload.cpp:204-224 round trip
    (64, 8, 65536, 1.25, 0.02, 42, 7),   # configs[2] shape
    (128, 8, 262144, 1.8, 0.02, 5, 3),   # configs[4] shape, severe skew
    (16, 1, 131072, 1.25, 0.0, 42, 2),   # configs[1] shape, single GPU
])
def test_save_matches_reference_bytes(tmp_path, N, G, tokens, zipf, drift, seed, steps):
    ref = oracle.Reference()
    tr = ref.generate_trace(N, G, tokens, zipf, drift, seed, steps)
    ours, theirs = tmp_path / "ours.csv", tmp_path / "ref.csv"
    TR.save_trace(tr, ours)
    ref.save_trace(tr, theirs)
    assert ours.read_bytes() == theirs.read_bytes()
    np.testing.assert_array_equal(TR.load_trace(ours), tr)
    np.testing.assert_array_equal(TR.load_trace(theirs, N, G), tr)
    np.testing.assert_array_equal(ref.load_trace(ours), tr)


MALFORMED = {
    "negative_count": "step,expert,gpu,tokens\n0,0,0,5\n0,1,0,-3\n",
    "missing_field": "step,expert,gpu,tokens\n0,0,0\n",
    "extra_field": "step,expert,gpu,tokens\n0,0,0,1,2\n",
    "bad_header": "step,gpu,expert,tokens\n0,0,0,5\n",
    "unsorted": "step,expert,gpu,tokens\n0,1,0,5\n0,0,0,5\n",
    "duplicate": "step,expert,gpu,tokens\n0,1,0,5\n0,1,0,5\n",
    "totals": "step,expert,gpu,tokens\n0,0,0,5\n1,0,0,4\n",
    "bad_integer": "step,expert,gpu,tokens\n0,x,0,5\n",
    "empty_field": "step,expert,gpu,tokens\n0,,0,5\n",
    "negative_id": "step,expert,gpu,tokens\n0,-1,0,5\n",
    "first_step": "step,expert,gpu,tokens\n1,0,0,5\n",
    "zero_total": "step,expert,gpu,tokens\n0,0,0,0\n",
    "no_records": "step,expert,gpu,tokens\n\n",
    "empty_file": "",
}


@needs_ref
@pytest.mark.parametrize("case", sorted(MALFORMED))
def test_loader_errors_match_reference(tmp_path, case):
    p = tmp_path / "t.csv"
    p.write_text(MALFORMED[case])
    with pytest.raises(L.FlexMoEError) as ours:
        TR.load_trace(p)
    with pytest.raises(RuntimeError) as theirs:
        oracle.Reference().load_trace(p)
    assert ours.value.status == L.FM_ERR_RUNTIME
    assert str(ours.value) == str(theirs.value)


@needs_ref
def test_loader_explicit_dimensions(tmp_path):
    p = tmp_path / "t.csv"
    p.write_text("step,expert,gpu,tokens\n0,3,0,5\n")  # test_workload.cpp:265-269
    with pytest.raises(L.FlexMoEError) as ours:
        TR.load_trace(p, 2, 2)
    with pytest.raises(RuntimeError) as theirs:
        oracle.Reference().load_trace(p, 2, 2)
    assert "out of range" in str(ours.value) and str(ours.value) == str(theirs.value)
    p.write_text("step,expert,gpu,tokens\r\n0,0,0,12\r\n\n")  # CRLF + blank line tolerated
    tr = TR.load_trace(p)
    assert tr.shape == (1, 1, 1) and tr[0, 0, 0] == 12
    np.testing.assert_array_equal(tr, oracle.Reference().load_trace(p))
    np.testing.assert_array_equal(TR.load_trace(p, 3, 2)[0], [[12, 0], [0, 0], [0, 0]])


def test_recorder_and_step_ids(tmp_path):
    rec = TR.TraceRecorder()
    rng = np.random.default_rng(0)
    for _ in range(4):
        D = rng.multinomial(200, np.full(6 * 3, 1 / 18)).reshape(6, 3)
        rec.record(D)
    rec.save(tmp_path / "r.csv")
    np.testing.assert_array_equal(TR.load_trace(tmp_path / "r.csv", 6, 3), rec.trace())
    TR.save_trace(rec.trace()[:1], tmp_path / "s.csv", step_ids=[0])
    assert (tmp_path / "s.csv").read_text().splitlines()[0] == "step,expert,gpu,tokens"


@pytest.mark.parametrize("k", [1, 2, 4])
def test_replay_assignment(k):
    rng = np.random.default_rng(k)
    for _ in range(50):
        N, T = int(rng.integers(k, 40)), int(rng.integers(1, 300))
        # random column with every entry <= T and sum T*k
        choice = np.stack([rng.permutation(N)[:k] for _ in range(T)])
        col = np.bincount(choice.reshape(-1), minlength=N)
        a = TR.replay_assignment(col, k)
        assert a.shape == (T, k)
        np.testing.assert_array_equal(np.bincount(a.reshape(-1), minlength=N), col)
        assert all(len(set(r)) == k for r in a.tolist())
    with pytest.raises(L.InvalidArgument):
        TR.replay_assignment([5, 1], 2)  # expert 0 would need 5 of 3 tokens
    with pytest.raises(L.InvalidArgument):
        TR.replay_assignment([3, 2], 2)  # odd total
