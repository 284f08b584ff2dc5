"""GPU parity at the bench's own shapes, through the C ABI.

  * a full local step at cfg5 layer shapes (d=4096, f=2048, M=64, k=8; L=2 so a routed
    layer follows a routed layer) against the oracle's build_loss + backward
    (model.hpp:252-374) and MaskedAdamW (trainer.hpp:68-94);
  * merge_model (merging.hpp:55-150) at M=64 (gram_partial_k, merge_apply_k<1>) and at
    M=16 with 9 peers (merge_apply_k<2>), bit-exact.
Host memory: the cfg5-shape case holds four 12.9 GB parameter-sized vectors.
"""
import numpy as np
import pytest

import oracle
import paper_2602_11543_b200 as spes
from paper_2602_11543_b200.abi import adamw_cfg, merge_sched, model_cfg
from test_gpu_parity import (CFG2, CFG4, GRAD_RTOL, LOSS_RTOL, _check_deep_routing,
                             _check_grad_blocks, _check_operand_copies, bitexact)

pytestmark = pytest.mark.gpu

CFG5_L2 = dict(vocab=256, hidden=4096, intermediate=2048, layers=2, experts_total=64,
               experts_active=8)


def big_params(cfg, seed, std=0.02):
    """Seeded N(0, std) parameters generated in float32 chunks (a float64 temporary of a
    3.2 G-scalar model would not fit next to the comparison vectors); gains 1."""
    P = spes.param_count(cfg)
    rng = np.random.default_rng(seed)
    p = np.empty(P, np.float32)
    step = 1 << 26
    for i in range(0, P, step):
        n = min(step, P - i)
        rng.standard_normal(n, dtype=np.float32, out=p[i:i + n])
        p[i:i + n] *= np.float32(std)
    offs = spes.block_offsets(cfg)
    for l in range(cfg.layers):
        o = offs[2 + 2 * l]
        p[o:o + cfg.hidden] = 1.0
    return p


# Gradient bound when layer-1 routing follows the bench's init: measured max 0.203 (an
# expert of ~32 routed rows whose token set differs by a near-tie flip); 2x that.
GRAD_RTOL_FLIPS = 0.4


@pytest.mark.parametrize("layer1_router", ["zero", "bench_init"])
def test_local_step_cfg5_shapes(gpu, layer1_router):
    """Two layers at cfg5 shapes. layer1_router="zero": layer 1's router is all zeros, so its
    probabilities tie exactly and routing is the lowest k experts on both sides whatever the
    bf16 perturbation of h1 (the tie rule of model.hpp:185-216): every gradient block is then
    held to GRAD_RTOL. "bench_init": N(0, 0.02) like the bench; layer-1 top-k near-ties
    flip under the bf16 perturbation of h1 (~6% of tokens at M=64, k=8) and a flipped
    token's gradient differs discretely, so gradients are held to GRAD_RTOL_FLIPS and the
    routing to bit-exactness on the device's own layer-1 input."""
    cfg = model_cfg(**CFG5_L2)
    params = big_params(cfg, 91)
    if layer1_router == "zero":
        o = spes.block_offsets(cfg)[3 + 2 * 1]
        params[o:o + cfg.hidden * cfg.experts_total] = 0.0
    B, S = 1, 256
    T, M, k, L = B * S, cfg.experts_total, cfg.experts_active, cfg.layers
    tokens = oracle.random_tokens(cfg, B, S, 92)[0]
    owned = list(range(4, 12)) + list(range(16, 24))  # 16 experts; 4..7 see layer-1 tokens
    opt = adamw_cfg(lr=1e-3)
    node = spes.Node(cfg)
    node.set_ownership([owned])
    node.load_params(params)
    node.set_fused_optimizer(False)
    node.round_begin()
    losses = np.array(node.local_step(tokens, opt))
    dbg = {name: [node.debug(name, l, dt, None, n) for l in range(L)]
           for name, dt, n in (("topk_idx", np.int32, T * k), ("probs", np.float32, T * M),
                               ("counts", np.int32, M), ("perm", np.int32, T * k))}
    g_gpu = node.read_grads()
    p_gpu = node.read_params()
    l_ref, g_ref, tr = oracle.forward_backward(cfg, params, tokens, owned, trace=True)
    # layer 0: identical inputs -> routing, probabilities, counts, permutation bit-exact
    assert bitexact(dbg["topk_idx"][0], tr["topk_idx"][0].reshape(-1))
    assert bitexact(dbg["probs"][0], tr["probs"][0].reshape(-1))
    assert bitexact(dbg["counts"][0], tr["counts"][0])
    assert bitexact(dbg["perm"][0], tr["perm"][0])
    # layer 1 follows bf16 expert outputs: bit-exact on the device's own input, near-ties
    # only against the oracle's
    _check_deep_routing(cfg, node, params, tr, T, f"cfg5-shape layer-1 router {layer1_router}")
    for i, name in enumerate(("total", "ce", "lb", "moe_z", "z")):
        assert abs(losses[i] - l_ref[i]) <= LOSS_RTOL * abs(l_ref[i]) + 1e-7, name
    node.close()
    _check_grad_blocks(cfg, g_gpu, g_ref, f"cfg5-shape B=1 S=256 layer-1 router {layer1_router}",
                       rtol=GRAD_RTOL if layer1_router == "zero" else GRAD_RTOL_FLIPS)
    del g_ref
    # MaskedAdamW on the device's own gradients == the oracle's element update, block by
    # block (trainable: psi + owned experts); frozen experts bit-identical
    offs = list(spes.block_offsets(cfg)) + [spes.param_count(cfg)]
    n_psi = 2 + 2 * L
    per = 3 * cfg.hidden * cfg.intermediate
    expert0 = offs[n_psi]
    ranges = [(offs[0], expert0)]
    for l in range(L):
        for j in range(M):
            o = expert0 + (l * M + j) * per
            if j in owned:
                ranges.append((o, o + per))
            else:
                assert bitexact(p_gpu[o:o + per], params[o:o + per]), f"frozen expert {l}.{j}"
    for b0, b1 in ranges:
        th = params[b0:b1].copy()
        m = np.zeros_like(th)
        v = np.zeros_like(th)
        oracle.lib().oracle_adamw_array(th, np.ascontiguousarray(g_gpu[b0:b1]), m, v, b1 - b0,
                                        opt, 1)
        assert bitexact(p_gpu[b0:b1], th), f"AdamW block at {b0}"


@pytest.mark.parametrize("shape,peers,source", [(CFG4, 4, 0), (CFG4, 9, 2), (CFG2, 9, 0)])
def test_merge_bitexact_large(gpu, shape, peers, source):
    """M = 64: gram_partial_k + merge_apply_k<1>; M = 16 with K = 9 > 8: merge_apply_k<2>."""
    cfg = model_cfg(**shape)
    params = big_params(cfg, 101 + peers, std=0.05)
    node = spes.Node(cfg)
    node.load_params(params)
    sched = merge_sched(warmup_rounds=4, interval=1, alpha0=0.1, peers=peers, source=source)
    sim_gpu = node.similarity(0, source)
    sim_ref = oracle.similarity(cfg, params, 0, source)
    assert np.allclose(sim_gpu, sim_ref, rtol=1e-12, atol=1e-14)
    ev_gpu, peers_gpu = node.merge_model(sched, 1)
    p_ref, ev_ref, peers_ref = oracle.merge_model(cfg, params, sched, 1)
    assert (peers_gpu == peers_ref).all()
    assert bitexact(node.read_params(), p_ref)
    _check_operand_copies(node, cfg)
    for a, b in zip(ev_gpu, ev_ref):
        assert a[:3] == b[:3]
        assert abs(a[3] - b[3]) <= 1e-9 * abs(b[3])
    node.close()
