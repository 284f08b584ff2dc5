"""N > 1 host logic on CPU (gloo, world_size 2..8).

The sparse sync's data movement is planned by spes_sync_plan (the same function
spes_sync uses before issuing NCCL calls). Here every rank follows that plan with
torch.distributed gloo point-to-point and all-gather on CPU tensors — co-owners send
their copy to the primary, the primary takes the fp64 owner-set mean in ascending
node order, every rank receives every expert from its primary, psi is all-gathered
and averaged in node order — and the result must equal the oracle's
Server::aggregate restatement bit-for-bit on every rank.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import paper_2602_11543_b200 as spes
from paper_2602_11543_b200.abi import model_cfg

CFG = dict(vocab=16, hidden=8, intermediate=8, layers=2, experts_total=8, experts_active=2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _mean_in_order(arrs):
    acc = np.zeros_like(arrs[0], dtype=np.float64)
    for a in arrs:
        acc = acc + a.astype(np.float64)
    return (acc * (1.0 / len(arrs))).astype(np.float32)


def _worker(rank, world, port, owned, node_params, glob, out_q, M):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = model_cfg(**dict(CFG, experts_total=M))
    P = node_params.shape[1]
    M, L = cfg.experts_total, cfg.layers
    per = 3 * cfg.hidden * cfg.intermediate
    mine = node_params[rank].copy()
    primary, balanced = spes.sync_plan(M, owned)
    owners = [[n for n in range(world) if e in owned[n]] for e in range(M)]
    psi = oracle.expert_offset(cfg, 0, 0)
    # psi: all-gather + node-order mean
    gathered = [torch.zeros(psi) for _ in range(world)]
    dist.all_gather(gathered, torch.from_numpy(mine[:psi].copy()))
    result = glob.copy()
    result[:psi] = _mean_in_order([g.numpy() for g in gathered])
    # experts: co-owners -> primary, mean at primary
    for l in range(L):
        for e in range(M):
            O = owners[e]
            off = oracle.expert_offset(cfg, l, e)
            if not O:
                continue
            p = int(primary[e])
            assert p in O
            val = mine[off:off + per].copy()
            if rank == p:
                copies = {}
                for o in O:
                    if o == rank:
                        copies[o] = val
                    else:
                        buf = torch.zeros(per)
                        dist.recv(buf, src=o)
                        copies[o] = buf.numpy()
                val = _mean_in_order([copies[o] for o in sorted(O)])
            elif rank in O:
                dist.send(torch.from_numpy(val), dst=p)
            # distribute from the primary
            t = torch.from_numpy(val.copy()) if rank == p else torch.zeros(per)
            dist.broadcast(t, src=p)
            result[off:off + per] = t.numpy()
    out_q.put((rank, result, bool(balanced)))
    dist.barrier()
    dist.destroy_process_group()


# (8, "replicated", 16) is cfg2 / cfg4's topology: 8 nodes, M = 16, r = 2,
# node n owns {(2n + i) mod 16, i < 4}, primary(e) = e // 2, owner pairs {e//2, (e//2 - 1) mod 8}
@pytest.mark.parametrize("world,layout,M", [(2, "partition", 8), (2, "replicated", 8),
                                            (4, "replicated", 8), (3, "irregular", 8),
                                            (8, "replicated", 16)])
def test_sync_plan_gloo_matches_oracle_aggregate(world, layout, M):
    cfg = model_cfg(**dict(CFG, experts_total=M))
    if layout == "partition":
        owned = spes.param_partition(cfg, world)
    elif layout == "replicated":
        owned = spes.replicated_ownership(M, world, 2)
    else:
        owned = [[0, 1, 5], [1, 2], [2, 3, 4, 5]]  # expert 6, 7 unowned; mixed replication
    P = oracle.param_count(cfg)
    rng = np.random.default_rng(world)
    glob = rng.standard_normal(P).astype(np.float32)
    node_params = rng.standard_normal((world, P)).astype(np.float32)
    expect = oracle.aggregate(cfg, node_params, owned, glob)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    if layout == "replicated" and M == 16 and world == 8:
        assert owned == [sorted((2 * n + i) % 16 for i in range(4)) for n in range(8)]
    procs = [ctx.Process(target=_worker, args=(r, world, port, owned, node_params, glob, q, M))
             for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    for rank, res, balanced in results:
        assert np.array_equal(res.view(np.uint32), expect.view(np.uint32)), f"rank {rank}"
        assert balanced == (layout == "replicated" or (layout == "partition" and M % world == 0))


def test_sync_plan_primaries():
    prim, bal = spes.sync_plan(16, spes.replicated_ownership(16, 8, 2))
    assert bal and list(prim) == [e // 2 for e in range(16)]
    prim, bal = spes.sync_plan(8, [[0, 1, 5], [1, 2], [2, 3, 4, 5]])
    assert not bal and list(prim) == [0, 0, 1, 2, 2, 0, -1, -1]
