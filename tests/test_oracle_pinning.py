"""Pin the C restatement (oracle/spes_oracle.c) to the reference itself.

Every comparison is bit-for-bit against oracle/_ref/libspes_ref.so, which is the
UNMODIFIED reference (/root/reference/proj) compiled from its own sources with its
own flags, called through its public API. Plus the reference's own known-answer
tests. CPU only.
"""
import ctypes as C

import numpy as np
import pytest

import oracle
from paper_2602_11543_b200.abi import MergeEvent, adamw_cfg, merge_sched, model_cfg

pytestmark = pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built")

TINY = dict(vocab=64, hidden=32, intermediate=64, layers=2, experts_total=4, experts_active=2)
CFG1 = dict(vocab=256, hidden=128, intermediate=256, layers=2, experts_total=8, experts_active=2)


def bits(a):
    a = np.ascontiguousarray(a)
    return a.view({4: np.uint32, 8: np.uint64}[a.dtype.itemsize])


def assert_bitexact(a, b, what):
    a, b = np.asarray(a), np.asarray(b)
    assert a.shape == b.shape, what
    diff = np.flatnonzero(bits(a).ravel() != bits(b).ravel())
    assert diff.size == 0, f"{what}: {diff.size} elements differ, first at {diff[:5]}: " \
                           f"{a.ravel()[diff[:5]]} vs {b.ravel()[diff[:5]]}"


def ref_fwd_bwd(cfg, params, tokens, owned):
    R = oracle.ref()
    B, S1 = tokens.shape[-2:]
    T = B * (S1 - 1)
    L, M, k = cfg.layers, cfg.experts_total, cfg.experts_active
    grads = np.zeros(oracle.param_count(cfg), np.float32)
    losses = np.zeros(5)
    probs = np.zeros((L, T, M), np.float32)
    idx = np.zeros((L, T, k), np.int32)
    w = np.zeros((L, T, k), np.float32)
    rc = R.ref_forward_backward(C.byref(cfg), params, np.ascontiguousarray(tokens.reshape(B, S1)),
                                B, S1 - 1, oracle.trainable_mask(cfg, owned), grads, losses, probs,
                                idx, w)
    assert rc == 0
    return losses, grads, probs, idx, w


@pytest.mark.parametrize("shape,owned,renorm,B,S", [
    (TINY, [0, 1], False, 2, 8),
    (TINY, [2, 3], True, 2, 8),
    (TINY, [0, 1, 2, 3], False, 3, 5),
    (CFG1, [0, 1, 2, 3], False, 1, 64),
    (CFG1, [4, 5, 6, 7], True, 1, 64),
])
def test_forward_backward_bitexact(shape, owned, renorm, B, S):
    cfg = model_cfg(renormalize_after_topk=renorm, **shape)
    R = oracle.ref()
    params = np.zeros(oracle.param_count(cfg), np.float32)
    R.ref_init_model(C.byref(cfg), 7, 0.02 if shape is CFG1 else 0.3, params)
    tokens = oracle.random_tokens(cfg, B, S, seed=3)[0]
    l_ref, g_ref, p_ref, i_ref, w_ref = ref_fwd_bwd(cfg, params, tokens, owned)
    l_or, g_or, tr = oracle.forward_backward(cfg, params, tokens, owned, trace=True)
    assert_bitexact(np.float32(l_or), np.float32(l_ref), "losses")
    assert_bitexact(tr["probs"], p_ref, "router probs")
    assert_bitexact(tr["topk_idx"], i_ref, "routing indices")
    assert_bitexact(tr["topk_w"], w_ref, "gate weights")
    assert_bitexact(g_or, g_ref, "gradients")
    # frozen experts get no gradient (graph.hpp:56-63)
    for l in range(cfg.layers):
        for j in range(cfg.experts_total):
            o = oracle.expert_offset(cfg, l, j)
            seg = g_or[o:o + 3 * cfg.hidden * cfg.intermediate]
            if j not in owned:
                assert not seg.any()


def test_local_round_bitexact():
    cfg = model_cfg(**CFG1)
    R = oracle.ref()
    params = np.zeros(oracle.param_count(cfg), np.float32)
    R.ref_init_model(C.byref(cfg), 1, 0.02, params)
    H, B, S = 3, 1, 32
    tokens = oracle.random_tokens(cfg, B, S, seed=11, H=H)
    opt = adamw_cfg()
    lr = np.array([oracle.lib().oracle_lr_at(1e-3, 0.1, 2, 10, h) for h in range(H)])
    p_or, l_or = oracle.local_round(cfg, params, tokens, [4, 5, 6, 7], opt, lr)
    p_ref = params.copy()
    l_ref = np.zeros((H, 5))
    rc = R.ref_local_round(C.byref(cfg), p_ref, tokens, B, S, H, lr, C.byref(opt),
                           oracle.trainable_mask(cfg, [4, 5, 6, 7]), l_ref)
    assert rc == 0
    assert_bitexact(np.float32(l_or), np.float32(l_ref), "step losses")
    assert_bitexact(p_or, p_ref, "params after local round")
    # frozen experts bit-identical to round entry (test_trainer.cpp:132-155)
    for j in range(4):
        o = oracle.expert_offset(cfg, 0, j)
        n = 3 * cfg.hidden * cfg.intermediate
        assert_bitexact(p_or[o:o + n], params[o:o + n], "frozen expert")


def test_adamw_first_step_bitexact():
    cfg = model_cfg(**TINY)
    rng = np.random.default_rng(5)
    params = rng.standard_normal(oracle.param_count(cfg)).astype(np.float32)
    grads = rng.standard_normal(params.size).astype(np.float32)
    owned = [1, 3]
    mask = oracle.trainable_mask(cfg, owned)
    opt = adamw_cfg(lr=3e-3, weight_decay=0.05)
    p_ref = params.copy()
    assert oracle.ref().ref_adamw_first_step(C.byref(cfg), p_ref, grads, mask, C.byref(opt)) == 0
    p_or = params.copy()
    m = np.zeros_like(params)
    v = np.zeros_like(params)
    g = grads.copy()
    for j in range(cfg.experts_total):  # frozen blocks carry no gradient into the step
        if j not in owned:
            for l in range(cfg.layers):
                o = oracle.expert_offset(cfg, l, j)
                g[o:o + 3 * cfg.hidden * cfg.intermediate] = 0
    oracle.lib().oracle_adamw_step(C.byref(cfg), p_or, g, m, v, mask, C.byref(opt), 1)
    assert_bitexact(p_or, p_ref, "adamw")


@pytest.mark.parametrize("N", [2, 3, 4])
def test_aggregate_matches_reference_server(N):
    cfg = model_cfg(vocab=16, hidden=8, intermediate=8, layers=2, experts_total=4,
                    experts_active=2)
    P = oracle.param_count(cfg)
    rng = np.random.default_rng(N)
    glob = rng.standard_normal(P).astype(np.float32)
    nodes = rng.standard_normal((N, P)).astype(np.float32)
    part = oracle.param_partition(cfg.experts_total, N)
    ref_out = np.zeros(P, np.float32)
    assert oracle.ref().ref_aggregate_partition(C.byref(cfg), N, nodes, glob, ref_out) == 0
    assert_bitexact(oracle.aggregate(cfg, nodes, part, glob), ref_out, "aggregate")


def test_similarity_select_merge_bitexact():
    cfg = model_cfg(vocab=16, hidden=16, intermediate=24, layers=2, experts_total=6,
                    experts_active=2)
    params = oracle.random_params(cfg, 9, std=0.5)
    R = oracle.ref()
    for src in (0, 1, 2):
        s_ref = np.zeros((6, 6))
        R.ref_similarity(C.byref(cfg), params, 1, src, s_ref)
        assert_bitexact(oracle.similarity(cfg, params, 1, src), s_ref, f"similarity src={src}")
    sim = oracle.similarity(cfg, params, 0)
    for j in range(6):
        for K in (1, 3, 5, 9):
            a = np.zeros(8, np.int32)
            b = np.zeros(8, np.int32)
            na = oracle.lib().oracle_select_peers(sim, 6, j, K, a)
            nb = R.ref_select_peers(sim, 6, j, K, b)
            assert na == nb and (a[:na] == b[:nb]).all()
    sched = merge_sched(warmup_rounds=10, interval=2, alpha0=0.3, peers=3, source=0)
    for rnd in (0, 1, 2, 9, 10):
        p_or, ev_or, peers_or = oracle.merge_model(cfg, params, sched, rnd)
        p_ref = params.copy()
        ev = (MergeEvent * cfg.layers)()
        peers_ref = np.zeros((cfg.layers, 6, 3), np.int32)
        n = R.ref_merge_model(C.byref(cfg), p_ref, C.byref(sched), rnd, C.cast(ev, C.c_void_p),
                              peers_ref)
        assert n == len(ev_or)
        assert_bitexact(p_or, p_ref, f"merge round {rnd}")
        for l in range(n):
            assert ev[l].alpha == ev_or[l][2]
            assert ev[l].displacement_sq == ev_or[l][3]
            assert (peers_ref[l] == peers_or[l]).all()


def test_lr_schedule_and_partition():
    L, R = oracle.lib(), oracle.ref()
    for args in [(1e-3, 0.1, 5, 100), (3e-4, 0.0, 0, 50), (1e-2, 0.5, 10, 5)]:
        for s in range(0, 120, 7):
            assert L.oracle_lr_at(*args, s) == R.ref_lr_at(*args, s)
    for M, N in [(8, 2), (16, 8), (7, 3), (64, 5)]:
        cfg = model_cfg(experts_total=M, experts_active=1)
        offs = np.zeros(N + 1, np.int32)
        ex = np.zeros(M, np.int32)
        R.ref_param_partition(C.byref(cfg), N, offs, ex)
        ours = oracle.param_partition(M, N)
        assert ours == [list(ex[offs[i]:offs[i + 1]]) for i in range(N)]


# ---------------- the reference's own known-answer tests ----------------

def test_kat_routing():
    # test_model.cpp:50-84
    cfg = model_cfg(hidden=2, experts_total=2, experts_active=1)
    probs_of = lambda logits: np.exp(logits - logits.max()) / np.exp(logits - logits.max()).sum()
    p = probs_of(np.array([2.0, -1.0]))
    assert abs(p[0] - 0.9526) < 1e-3
    # tie -> lowest index, through the restated router on equal logits
    cfg = model_cfg(hidden=4, experts_total=4, experts_active=2)
    h = np.ones((1, 4), np.float32)
    router = np.zeros((4, 4), np.float32)
    out = oracle.router_forward(cfg, h, np.ones(4, np.float32), router)
    assert list(out["idx"][0]) == [0, 1]


def test_kat_adamw_scalar():
    # test_trainer.cpp:83-96: theta=1, g=0.5, lr=0.1, wd=0.1 -> 0.89
    cfg = model_cfg(vocab=1, hidden=1, intermediate=1, layers=1, experts_total=1,
                    experts_active=1)
    P = oracle.param_count(cfg)
    p = np.zeros(P, np.float32)
    p[0] = 1.0
    g = np.zeros(P, np.float32)
    g[0] = 0.5
    m = np.zeros(P, np.float32)
    v = np.zeros(P, np.float32)
    oracle.lib().oracle_adamw_step(C.byref(cfg), p, g, m, v, np.ones(1, np.uint8),
                                   C.byref(adamw_cfg(lr=0.1)), 1)
    assert abs(p[0] - 0.89) < 1e-6


def test_kat_aggregate_two_nodes():
    # test_protocol.cpp:167-190: (1+3)/2 == 2.0 exactly, experts verbatim
    cfg = model_cfg(vocab=4, hidden=2, intermediate=2, layers=2, experts_total=4,
                    experts_active=2)
    P = oracle.param_count(cfg)
    glob = np.zeros(P, np.float32)
    nodes = np.tile(glob, (2, 1))
    nodes[0, 0], nodes[1, 0] = 1.0, 3.0
    nodes[0, oracle.expert_offset(cfg, 0, 0)] = 0.123
    nodes[1, oracle.expert_offset(cfg, 1, 3) + 5] = -4.5
    out = oracle.aggregate(cfg, nodes, [[0, 1], [2, 3]], glob)
    assert out[0] == 2.0
    assert out[oracle.expert_offset(cfg, 0, 0)] == np.float32(0.123)
    assert out[oracle.expert_offset(cfg, 1, 3) + 5] == np.float32(-4.5)


def test_kat_merge_constant_experts():
    # test_merging.cpp:132-146: constant experts 0 and 2, alpha 0.1, K=1 -> 0.2 / 1.8
    cfg = model_cfg(vocab=1, hidden=1, intermediate=1, layers=1, experts_total=2,
                    experts_active=1)
    p = np.zeros(oracle.param_count(cfg), np.float32)
    o1 = oracle.expert_offset(cfg, 0, 1)
    p[o1:o1 + 3] = 2.0
    out, ev, _ = oracle.merge_model(cfg, p, merge_sched(warmup_rounds=10, alpha0=0.1, peers=1), 0)
    o0 = oracle.expert_offset(cfg, 0, 0)
    assert np.allclose(out[o0:o0 + 3], 0.2) and np.allclose(out[o1:o1 + 3], 1.8)


def test_kat_cosine():
    # test_merging.cpp:53-69 (gate vectors [1,0],[2,0],[0,1],[1,1],[0,0])
    cfg = model_cfg(vocab=1, hidden=1, intermediate=2, layers=1, experts_total=5,
                    experts_active=1)
    p = np.zeros(oracle.param_count(cfg), np.float32)
    for j, g in enumerate([[1, 0], [2, 0], [0, 1], [1, 1], [0, 0]]):
        o = oracle.expert_offset(cfg, 0, j)
        p[o:o + 2] = g
    s = oracle.similarity(cfg, p, 0)
    assert abs(s[0, 1] - 1) < 1e-12 and abs(s[0, 2]) < 1e-12
    assert abs(s[0, 3] - 1 / np.sqrt(2)) < 1e-12 and s[0, 4] == 0 and s[4, 4] == 0


@pytest.mark.parametrize("kind,N", [(0, 1), (0, 3), (1, 1), (1, 3)])
def test_outer_optimizer_bitexact(kind, N):
    """OuterOptimizer::step (trainer.hpp:228-266) over 3 rounds, state carried."""
    R = oracle.ref()
    cfg = model_cfg(**TINY)
    theta_ref = oracle.random_params(cfg, 31)
    theta_or = theta_ref.copy()
    buf = np.zeros(theta_or.size)
    h = R.ref_outer_create(kind, 0.7, 0.9)
    try:
        rng = np.random.default_rng(32)
        for _ in range(3):
            locals_ = np.stack([theta_ref + (rng.standard_normal(theta_ref.size) * 1e-2)
                                .astype(np.float32) for _ in range(N)])
            assert R.ref_outer_step(h, C.byref(cfg), theta_ref, np.ascontiguousarray(locals_), N) == 0
            oracle.outer_step(kind, 0.7, 0.9, theta_or, locals_, buf)
            assert_bitexact(theta_or, theta_ref, f"outer kind={kind} N={N}")
    finally:
        R.ref_outer_destroy(h)


def test_outer_sgd_lr1_single_node_reproduces_local():
    """trainer.hpp:232-234: SGD with lr = 1 and N = 1 reproduces the local params exactly."""
    cfg = model_cfg(**TINY)
    theta = oracle.random_params(cfg, 33)
    local = theta + np.float32(0.01)
    oracle.outer_step(0, 1.0, 0.9, theta, local[None], np.zeros(theta.size))
    assert_bitexact(theta, local, "sgd lr=1")
