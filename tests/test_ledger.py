"""CommLedger: spes_comm_ledger against the ledger of the UNMODIFIED
reference's in-process protocol run (run_inproc, protocol.cpp:368-405, through oracle/_ref):
every (node, round) entry and the totals, sparse and DiLoCo, several node counts; plus the
metrics.csv bytes columns (assemble_run_result, protocol.cpp:357-362)."""
import ctypes as C

import numpy as np
import pytest

import oracle
import paper_2602_11543_b200 as spes
from paper_2602_11543_b200.abi import model_cfg

SMALL = dict(vocab=32, hidden=16, intermediate=32, layers=2, experts_total=4, experts_active=2)


def ref_ledger(cfg, nodes, rounds, diloco):
    cap = nodes * (rounds + 2) + 1
    nd = np.zeros(cap, np.int32)
    rd = np.zeros(cap, np.int32)
    up = np.zeros(cap, np.uint64)
    dn = np.zeros(cap, np.uint64)
    n = C.c_int32(0)
    tot = np.zeros(4, np.uint64)
    rc = oracle.ref().ref_run_inproc_ledger(C.byref(cfg), nodes, rounds, 1, 1, 8,
                                            1 if diloco else 0, 5, nd, rd, up, dn, cap,
                                            C.byref(n), tot)
    assert rc == 0
    k = n.value
    return nd[:k], rd[:k], up[:k], dn[:k], tot


@pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("nodes,rounds,diloco", [(1, 1, False), (2, 2, False), (4, 3, False),
                                                 (3, 2, False), (2, 2, True)])
def test_ledger_matches_reference_run(nodes, rounds, diloco):
    cfg = model_cfg(**SMALL)
    ent, tot = spes.comm_ledger(cfg, nodes, rounds, diloco=diloco)
    nd, rd, up, dn, rtot = ref_ledger(cfg, nodes, rounds, diloco)
    assert np.array_equal(ent["node"], nd) and np.array_equal(ent["round"], rd)
    assert np.array_equal(ent["up"], up) and np.array_equal(ent["down"], dn)
    assert [tot["total_up"], tot["total_down"], tot["pushes"], tot["broadcasts"]] == rtot.tolist()


def test_ledger_shape_and_round_bytes():
    cfg = model_cfg(**SMALL)
    nodes, rounds = 2, 3
    ent, tot = spes.comm_ledger(cfg, nodes, rounds)
    assert ent.size == 1 + nodes * (rounds + 2)  # HELLOs under node -1, rounds 0..R+1
    assert tot["pushes"] == nodes * rounds and tot["broadcasts"] == nodes * (rounds + 1)
    full = spes.model_payload_bytes(cfg) + 18
    for r in range(1, rounds + 1):
        b_up, b_down = spes.round_bytes(ent, r)
        assert b_down == nodes * (full + 18)  # round r's GLOBAL_MODEL + ROUND_DONE
        assert b_up < nodes * full  # sparse updates: shared blocks + owned experts only
    # replicated ownership (r = 2): each update carries twice the expert blocks
    _, t1 = spes.comm_ledger(cfg, 2, 1)
    _, t2 = spes.comm_ledger(cfg, 2, 1, ownership=[[0, 1, 2], [1, 2, 3]])
    assert t2["total_up"] > t1["total_up"]
    with pytest.raises(spes.SpesError):
        spes.comm_ledger(cfg, 5, 1)  # more nodes than experts


@pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built")
def test_metrics_csv_matches_reference_experiment(tmp_path):
    """run_experiment's metrics.csv (SPES paradigm, 2 nodes, 2 rounds) is reproduced byte for
    byte from its RoundMetrics (wall_ms taken from the reference's own file), and its bytes
    columns equal spes_comm_ledger's round sums."""
    cfg = model_cfg(**SMALL)
    nodes, H, rounds, batch, seq = 2, 1, 2, 2, 8
    rows = (spes.RoundMetrics * 8)()
    n = C.c_int32(0)
    tpr = C.c_int64(0)
    rc = oracle.ref().ref_run_experiment(C.byref(cfg), nodes, H, rounds, batch, seq,
                                         str(tmp_path).encode(), b"run", C.cast(rows, C.c_void_p),
                                         8, C.byref(n), C.byref(tpr))
    assert rc == 0 and n.value == rounds
    ref_text = (tmp_path / "run" / "metrics.csv").read_text()
    wall = [float(line.split(",")[-1]) for line in ref_text.splitlines()[1:]]
    ours = spes.metrics_csv(list(rows[: n.value]), tpr.value, wall)
    assert ours == ref_text
    # the reference's per-round bytes == our ledger's
    ent, _ = spes.comm_ledger(cfg, nodes, rounds)
    for r in range(1, rounds + 1):
        assert spes.round_bytes(ent, r) == (rows[r - 1].bytes_up, rows[r - 1].bytes_down)
