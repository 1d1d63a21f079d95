"""Cluster profile JSON (ClusterTopology::from_json / to_json,
proj/src/topology.cpp:64-255) against the reference parser, and the B200
profile builder."""
import json
from pathlib import Path

import numpy as np
import pytest

import oracle
from paper_2304_03946_b200 import _lib as L
from paper_2304_03946_b200 import scheduler as S
from paper_2304_03946_b200.profile import b200_profile

needs_ref = pytest.mark.skipif(not oracle.Reference.available(), reason="oracle/_ref not built")
REF_CONFIGS = Path("/root/reference/proj/configs")


def _same(prof, ref):
    ints, dbl, intra, inter = ref
    assert [prof.num_gpus, prof.gpus_per_node, prof.slots_per_gpu] == ints.tolist()
    assert [prof.intra_node_bandwidth_bps, prof.inter_node_bandwidth_bps, prof.tps, prof.expert_param_bytes,
            prof.expert_state_bytes, prof.token_bytes] == dbl.tolist()
    G, gpn = prof.num_gpus, prof.gpus_per_node
    for n in range(2, G + 1):
        if n <= min(G, gpn):
            assert prof.allreduce_bps_intra[n] == intra[n], n
        if G > gpn:
            assert prof.allreduce_bps_inter[n] == inter[n], n


@needs_ref
@pytest.mark.skipif(not REF_CONFIGS.exists(), reason="reference configs not present")
@pytest.mark.parametrize("name", ["a100_single_node_8gpu.json", "a100_two_node_16gpu.json"])
def test_reference_configs_parse_identically(name, tmp_path):
    path = REF_CONFIGS / name
    prof = S.ClusterProfile.from_json(path)
    _same(prof, oracle.Reference().topology_load(path))
    out = tmp_path / "round.json"
    out.write_text(json.dumps(prof.to_json()))
    _same(S.ClusterProfile.from_json(out), oracle.Reference().topology_load(out))
    assert prof.to_json() == json.loads(path.read_text())


@needs_ref
@pytest.mark.parametrize("G,E", [(1, 4), (4, 2), (8, 16), (16, 4)])
def test_default_profile_roundtrip(G, E, tmp_path):
    prof = S.ClusterProfile.reference_default(G, E)
    p = tmp_path / "d.json"
    p.write_text(json.dumps(prof.to_json()))
    _same(S.ClusterProfile.from_json(p), oracle.Reference().topology_load(p))


BAD = {
    "missing_num_gpus": {"gpus_per_node": 8, "vexperts_per_gpu": 2},
    "bad_multiple": {"num_gpus": 6, "gpus_per_node": 4, "vexperts_per_gpu": 2},
    "zero_vexperts": {"num_gpus": 2, "gpus_per_node": 2, "vexperts_per_gpu": 0},
    "missing_tps": {"num_gpus": 1, "gpus_per_node": 1, "vexperts_per_gpu": 1, "intra_node_bandwidth_bps": 1.0},
    "negative_tps": {"num_gpus": 1, "gpus_per_node": 1, "vexperts_per_gpu": 1, "intra_node_bandwidth_bps": 1.0,
                     "tps": -1, "expert_param_bytes": 1, "expert_state_bytes": 1, "token_bytes": 1},
    "missing_bps": {"num_gpus": 2, "gpus_per_node": 2, "vexperts_per_gpu": 1, "intra_node_bandwidth_bps": 1.0,
                    "tps": 1, "expert_param_bytes": 1, "expert_state_bytes": 1, "token_bytes": 1},
    "increasing_bps": {"num_gpus": 3, "gpus_per_node": 3, "vexperts_per_gpu": 1, "intra_node_bandwidth_bps": 1.0,
                       "tps": 1, "expert_param_bytes": 1, "expert_state_bytes": 1, "token_bytes": 1,
                       "allreduce_bps": {"intra": {"2": 1.0, "3": 2.0}}},
    "missing_entry": {"num_gpus": 3, "gpus_per_node": 3, "vexperts_per_gpu": 1, "intra_node_bandwidth_bps": 1.0,
                      "tps": 1, "expert_param_bytes": 1, "expert_state_bytes": 1, "token_bytes": 1,
                      "allreduce_bps": {"intra": {"2": 1.0}}},
    "inter_missing_bw": {"num_gpus": 4, "gpus_per_node": 2, "vexperts_per_gpu": 1, "intra_node_bandwidth_bps": 1.0,
                         "tps": 1, "expert_param_bytes": 1, "expert_state_bytes": 1, "token_bytes": 1},
    "inter_faster": {"num_gpus": 4, "gpus_per_node": 2, "vexperts_per_gpu": 1, "intra_node_bandwidth_bps": 1.0,
                     "inter_node_bandwidth_bps": 1.0, "tps": 1, "expert_param_bytes": 1, "expert_state_bytes": 1,
                     "token_bytes": 1, "allreduce_bps": {"intra": {"2": 1.0},
                                                         "inter": {"2": 2.0, "3": 1.0, "4": 1.0}}},
}


@needs_ref
@pytest.mark.parametrize("case", sorted(BAD))
def test_invalid_configs_match_reference(case, tmp_path):
    p = tmp_path / "bad.json"
    p.write_text(json.dumps(BAD[case]))
    with pytest.raises(L.InvalidArgument) as ours:
        S.ClusterProfile.from_json(p)
    with pytest.raises(ValueError) as theirs:
        oracle.Reference().topology_load(p)
    assert str(ours.value) == str(theirs.value)


@needs_ref
def test_b200_profile_loads_in_reference(tmp_path):
    prof = b200_profile(8, 4, tps=2.5e7, d=1024, f=4096)
    p = tmp_path / "b200.json"
    p.write_text(json.dumps(prof.to_json()))
    ref = oracle.Reference().topology_load(p)
    _same(S.ClusterProfile.from_json(p), ref)
    assert ref[1][2] == 2.5e7 and ref[1][5] == 2048.0
    assert np.isclose(ref[2][8], 725e9 * 8 / 14)
