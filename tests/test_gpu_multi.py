"""Multi-GPU sparse sync over NCCL (one process per GPU, one SPES node each).

Every rank trains its own shard for a short local round, then spes_sync runs the
owner-set means over NCCL. The synced model must equal the oracle's
Server::aggregate restatement on the gathered pre-sync node models bit-for-bit,
on every rank; the merge warm-up afterwards must be identical on every rank and
equal to the oracle's merge_model. Skipped when fewer GPUs are visible.
"""
import numpy as np
import pytest
import torch.multiprocessing as mp

import oracle
import paper_2602_11543_b200 as spes
from paper_2602_11543_b200.abi import adamw_cfg, merge_sched, model_cfg

pytestmark = pytest.mark.gpu

CFG = dict(vocab=256, hidden=128, intermediate=256, layers=2, experts_total=8, experts_active=2)
# cfg2 shapes: d = f = 1024, 16 experts top-2, one layer
CFG2 = dict(vocab=256, hidden=1024, intermediate=1024, layers=1, experts_total=16,
            experts_active=2)
SCHED = dict(warmup_rounds=4, interval=1, alpha0=0.1, peers=3, source=0)


def _n_gpus():
    try:
        import torch
        return torch.cuda.device_count()
    except Exception:
        return 0


def _rank(rank, world, nccl_id, owned, params, tokens, q, p2p=True, shape=None):
    try:
        import os
        os.environ["SPES_SYNC_P2P"] = "1" if p2p else "0"  # read when the first sync runs
        cfg = model_cfg(**(shape or CFG))
        node = spes.Node(cfg, rank, world, rank, nccl_id)
        node.set_ownership(owned)
        node.load_params(params)
        node.local_round(tokens[rank], adamw_cfg(lr=1e-3))
        pre = node.read_params()
        st = node.sync()
        post = node.read_params()
        # the bf16 GEMM operand copies the sync left must equal a fresh refresh from fp32
        d, f, M = cfg.hidden, cfg.intermediate, cfg.experts_total
        def copies():
            return [node.debug(w, l, np.uint16, None, M * n)
                    for l in range(cfg.layers) for w, n in (("w1", 2 * d * f), ("w2", d * f))]
        synced = copies()
        node.load_params(post)  # rewrites every copy from the fp32 parameters
        fresh = copies()
        if not all(np.array_equal(a, b) for a, b in zip(synced, fresh)):
            raise AssertionError("operand copies after sync differ from a refresh")
        ev, peers = node.merge_model(merge_sched(**SCHED), 0)
        merged = node.read_params()
        node.close()
        q.put((rank, pre, post, merged, st, None))
    except Exception as e:  # pragma: no cover - surfaced by the parent
        q.put((rank, None, None, None, None, repr(e)))


@pytest.mark.parametrize("world,layout,p2p,shape",
                         [(2, "replicated", True, "cfg1"), (2, "partition", True, "cfg1"),
                          (4, "replicated", True, "cfg1"), (4, "partition", True, "cfg1"),
                          (2, "replicated", False, "cfg1"), (4, "replicated", False, "cfg1"),
                          (4, "replicated", True, "cfg2"), (4, "replicated", False, "cfg2"),
                          (2, "replicated", True, "cfg2")])
def test_nccl_sync_matches_oracle(world, layout, p2p, shape):
    """p2p: the primaries read co-owner copies in place over NVLink (CUDA IPC mappings);
    otherwise the copies travel by NCCL send/recv. Same bits either way. cfg2: the float4
    peer pulls and owner means at cfg2 sizes (50 M expert scalars)."""
    if _n_gpus() < world:
        pytest.skip(f"needs {world} GPUs")
    shp = CFG2 if shape == "cfg2" else CFG
    cfg = model_cfg(**shp)
    M = cfg.experts_total
    owned = (spes.replicated_ownership(M, world, 2) if layout == "replicated"
             else spes.param_partition(cfg, world))
    params = oracle.random_params(cfg, 5)
    S = 128 if shape == "cfg2" else 64
    tokens = [oracle.random_tokens(cfg, 2, S, 100 + r, H=2) for r in range(world)]
    nccl_id = spes.nccl_unique_id()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_rank, args=(r, world, nccl_id, owned, params, tokens, q, p2p,
                                             shp))
             for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=300) for _ in range(world)], key=lambda x: x[0])
    for p in procs:
        p.join(timeout=60)
    errs = [r[5] for r in res if r[5]]
    assert not errs, errs
    pre = np.stack([r[1] for r in res])
    expect = oracle.aggregate(cfg, pre, owned, params)
    for rank, _, post, merged, st, _ in res:
        assert np.array_equal(post.view(np.uint32), expect.view(np.uint32)), f"rank {rank}"
        assert st["psi_bytes_in"] > 0
    merged0 = res[0][3]
    for r in res[1:]:
        assert np.array_equal(r[3].view(np.uint32), merged0.view(np.uint32))
    m_ref, _, _ = oracle.merge_model(cfg, expect, merge_sched(**SCHED), 0)
    if shape == "cfg2":  # the synced model's expert blocks really changed
        per = 3 * cfg.hidden * cfg.intermediate
        o = oracle.expert_offset(cfg, 0, 0)
        assert not np.array_equal(pre[0][o:o + per], expect[o:o + per])
    assert np.array_equal(merged0.view(np.uint32), m_ref.view(np.uint32))


def _rank_outer(rank, world, nccl_id, params, tokens, q):
    try:
        cfg = model_cfg(**CFG)
        node = spes.Node(cfg, rank, world, rank, nccl_id)
        node.set_ownership([list(range(cfg.experts_total))] * world)  # TrainMask::all
        node.load_params(params)
        node.outer_begin()
        out = []
        for rnd in range(2):
            node.local_round(tokens[rank][rnd], adamw_cfg(lr=1e-3))
            pre = node.read_params()
            node.outer_sync("nesterov", lr=0.7, momentum=0.9)
            out.append((pre, node.read_params()))
        node.close()
        q.put((rank, out, None))
    except Exception as e:  # pragma: no cover
        q.put((rank, None, repr(e)))


@pytest.mark.parametrize("world", [2, 4])
def test_nccl_outer_sync_matches_oracle(world):
    """DiLoCo outer sync over NCCL (slice exchange + fp64 node-order step + all-gather)
    equals OuterOptimizer::step on the gathered local models, every rank, two rounds."""
    if _n_gpus() < world:
        pytest.skip(f"needs {world} GPUs")
    cfg = model_cfg(**CFG)
    params = oracle.random_params(cfg, 6)
    tokens = [[oracle.random_tokens(cfg, 2, 64, 200 + 10 * r + h, H=2) for h in range(2)]
              for r in range(world)]
    nccl_id = spes.nccl_unique_id()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_rank_outer, args=(r, world, nccl_id, params, tokens, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=300) for _ in range(world)], key=lambda x: x[0])
    for p in procs:
        p.join(timeout=60)
    errs = [r[2] for r in res if r[2]]
    assert not errs, errs
    theta = params.copy()
    buf = np.zeros(theta.size)
    for rnd in range(2):
        locals_ = np.stack([res[r][1][rnd][0] for r in range(world)])
        oracle.outer_step(1, 0.7, 0.9, theta, locals_, buf)
        for r in range(world):
            assert np.array_equal(res[r][1][rnd][1].view(np.uint32), theta.view(np.uint32)), \
                f"round {rnd} rank {r}"
