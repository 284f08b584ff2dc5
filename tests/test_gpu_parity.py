"""GPU parity of the B200 path against the CPU oracle, through the C ABI.

Bar (SURVEY.md §8c / north_star):
  * bit-exact given identical inputs: expf port, router (rmsnorm, logits, softmax,
    top-k indices, weights), counts and token permutation, AdamW update, owner-set
    mean, merge apply and peer sets, embedding gradient;
  * bf16 tensor-core GEMMs feed losses and gradients: stated tolerances below;
  * routing of layers > 0 depends on bf16 expert outputs: reported as an
    agreement rate, every disagreement must be a near-tie under the oracle.
"""
import ctypes as C
import os

import numpy as np
import pytest

import oracle
import paper_2602_11543_b200 as spes
from paper_2602_11543_b200.abi import adamw_cfg, merge_sched, model_cfg

pytestmark = pytest.mark.gpu

CFG1 = dict(vocab=256, hidden=128, intermediate=256, layers=2, experts_total=8, experts_active=2)
CFG2 = dict(vocab=256, hidden=1024, intermediate=1024, layers=1, experts_total=16, experts_active=2)
CFG4 = dict(vocab=256, hidden=2048, intermediate=1024, layers=1, experts_total=64, experts_active=8)

# bf16 operands, fp32 accumulation: relative Frobenius error per gradient block. Measured
# maximum over every block of every local-step case with identical routing (GRADERR lines,
# round 2, B200): 5.18e-3 at cfg1 / cfg2 / cfg4 / non-pow2 / ragged shapes, 8.56e-3 at cfg5
# shapes (test_gpu_large.py, the layer-1 router gradient); the bound is 2x the maximum.
GRAD_RTOL = float(os.environ.get("SPES_GRAD_RTOL", "1.75e-2"))
LOSS_RTOL = 2e-3


def bitexact(a, b):
    a, b = np.ascontiguousarray(a), np.ascontiguousarray(b)
    return a.shape == b.shape and np.array_equal(a.view(np.uint8), b.view(np.uint8))


def rel_err(a, b):
    n = np.linalg.norm(b.astype(np.float64))
    return np.linalg.norm(a.astype(np.float64) - b.astype(np.float64)) / max(n, 1e-30)


# ---------------------------------------------------------------- kernels on identical inputs

def test_expf_port_exhaustive_negative_range(gpu):
    """Device expf port == host glibc expf on every float in [-104, 0]."""
    lo = np.float32(-0.0).view(np.uint32)            # 0x80000000
    hi = np.float32(-104.0).view(np.uint32)          # 0xC2D00000
    chunk = 1 << 27
    bad = 0
    for start in range(int(lo), int(hi) + 1, chunk):
        stop = min(int(hi) + 1, start + chunk)
        x = np.arange(start, stop, dtype=np.uint64).astype(np.uint32).view(np.float32)
        y = np.empty_like(x)
        spes._check(spes.lib().spes_kernel_expf(spes.f32(x), spes.f32(y), x.size, 0))
        bad += oracle.lib().oracle_expf_range_mismatches(start, stop - 1, y)
    assert bad == 0


# the last two: the bench's full token count per step (B*S = 16384) at cfg2 / cfg4 shapes
@pytest.mark.parametrize("shape,T,seed", [(CFG1, 256, 0), (CFG2, 4096, 1), (CFG4, 2048, 2),
                                          (CFG2, 16384, 3), (CFG4, 16384, 4)])
def test_router_kernel_bitexact(gpu, shape, T, seed):
    cfg = model_cfg(**shape)
    rng = np.random.default_rng(seed)
    d, M, k = cfg.hidden, cfg.experts_total, cfg.experts_active
    h = (rng.standard_normal((T, d)) * 0.5).astype(np.float32)
    gain = (1 + 0.1 * rng.standard_normal(d)).astype(np.float32)
    router = (rng.standard_normal((d, M)) * 0.05).astype(np.float32)
    router[:, 1] = router[:, 0]           # exact ties: expert 0 must win over 1
    h[:8] = h[8:16]                        # duplicate tokens
    ref = oracle.router_forward(cfg, h, gain, router)
    out = dict(normed=np.zeros((T, d), np.float32), logits=np.zeros((T, M), np.float32),
               probs=np.zeros((T, M), np.float32), idx=np.zeros((T, k), np.int32),
               w=np.zeros((T, k), np.float32), counts=np.zeros(M, np.int32),
               perm=np.zeros(T * k, np.int32))
    spes._check(spes.lib().spes_kernel_router(
        cfg, spes.f32(h), spes.f32(gain), spes.f32(router), T, spes.f32(out["normed"]),
        spes.f32(out["logits"]), spes.f32(out["probs"]), spes.i32(out["idx"]), spes.f32(out["w"]),
        spes.i32(out["counts"]), spes.i32(out["perm"]), 0))
    for key in ("normed", "logits", "probs", "idx", "w", "counts", "perm"):
        if not bitexact(out[key], ref[key]):
            bad = np.flatnonzero(out[key].reshape(-1).view(np.uint32) !=
                                 ref[key].reshape(-1).view(np.uint32))
            raise AssertionError(f"{key}: {bad.size} entries differ, first at {bad[:8]}: "
                                 f"{out[key].reshape(-1)[bad[:8]]} vs {ref[key].reshape(-1)[bad[:8]]}")


@pytest.mark.parametrize("shape,T", [(CFG1, 256), (CFG4, 16384)])
def test_routing_plan_repeatable(gpu, shape, T):
    """The routing plan (counting sort, model.hpp:314-318) is deterministic: 20 repeated
    launches on the same logits give the same permutation, bit for bit, as the oracle."""
    cfg = model_cfg(**shape)
    rng = np.random.default_rng(5)
    d, M, k = cfg.hidden, cfg.experts_total, cfg.experts_active
    h = (rng.standard_normal((T, d)) * 0.5).astype(np.float32)
    gain = (1 + 0.1 * rng.standard_normal(d)).astype(np.float32)
    router = (rng.standard_normal((d, M)) * 0.05).astype(np.float32)
    ref = oracle.router_forward(cfg, h, gain, router)
    for it in range(20):
        perm = np.zeros(T * k, np.int32)
        counts = np.zeros(M, np.int32)
        idx = np.zeros((T, k), np.int32)
        spes._check(spes.lib().spes_kernel_router(
            cfg, spes.f32(h), spes.f32(gain), spes.f32(router), T, None, None, None,
            spes.i32(idx), None, spes.i32(counts), spes.i32(perm), 0))
        assert bitexact(idx, ref["idx"]), f"launch {it}: top-k indices"
        assert bitexact(counts, ref["counts"]), f"launch {it}: counts"
        bad = np.flatnonzero(perm != ref["perm"])
        assert bad.size == 0, (f"launch {it}: {bad.size} permutation entries differ, first "
                               f"{bad[:8]}: got {perm[bad[:8]]} want {ref['perm'][bad[:8]]}")


def test_adamw_kernel_bitexact(gpu):
    rng = np.random.default_rng(7)
    n = 1 << 20
    th = rng.standard_normal(n).astype(np.float32)
    g = (rng.standard_normal(n) * 1e-3).astype(np.float32)
    g[:1024] = 0.0
    m = (rng.standard_normal(n) * 1e-3).astype(np.float32)
    v = np.abs(rng.standard_normal(n) * 1e-6).astype(np.float32)
    opt = adamw_cfg(lr=3e-4, weight_decay=0.1)
    for step in (1, 2, 37):
        a = [x.copy() for x in (th, g, m, v)]
        b = [x.copy() for x in (th, g, m, v)]
        spes._check(spes.lib().spes_kernel_adamw(spes.f32(a[0]), spes.f32(a[1]), spes.f32(a[2]),
                                                 spes.f32(a[3]), n, opt, step, 0))
        oracle.lib().oracle_adamw_array(b[0], b[1], b[2], b[3], n, opt, step)
        assert bitexact(a[0], b[0]) and bitexact(a[2], b[2]) and bitexact(a[3], b[3])


@pytest.mark.parametrize("r", [1, 2, 3, 8])
def test_owner_mean_bitexact(gpu, r):
    rng = np.random.default_rng(r)
    n = 1 << 18
    x = rng.standard_normal((r, n)).astype(np.float32)
    out = np.zeros(n, np.float32)
    spes._check(spes.lib().spes_kernel_owner_mean(spes.f32(x), r, n, spes.f32(out), 0))
    acc = np.zeros(n, np.float64)
    for i in range(r):
        acc = acc + x[i].astype(np.float64)
    assert bitexact(out, (acc * (1.0 / r)).astype(np.float32))
    if r == 1:
        assert bitexact(out, x[0])  # verbatim copy for a unique owner (protocol.cpp:229-236)


# ---------------------------------------------------------------- full local step

def _check_deep_routing(cfg, node, params, tr, T, label, min_agree=0.9):
    """Layers > 0 take the previous layer's bf16-GEMM output as input. Given the device's own
    layer input h_l, the router is bit-exact (rmsnorm, logits, softmax, top-k, weights);
    against the oracle's own h_l, routing agrees except where the oracle's k-th and
    (k+1)-th probabilities nearly tie (relative gap < 5%)."""
    L, d, M, k = cfg.layers, cfg.hidden, cfg.experts_total, cfg.experts_active
    offs = spes.block_offsets(cfg)
    for l in range(1, L):
        idx = node.debug("topk_idx", l, np.int32, (T, k), T * k)
        probs = node.debug("probs", l, np.float32, (T, M), T * M)
        h_l = node.debug("h", l, np.float32, (T, d), T * d)
        gain = params[offs[2 + 2 * l]:offs[2 + 2 * l] + d]
        router = params[offs[3 + 2 * l]:offs[3 + 2 * l] + d * M].reshape(d, M)
        ref = oracle.router_forward(cfg, h_l, gain, router)
        assert bitexact(idx, ref["idx"]), f"layer {l} routing on the device's own input"
        assert bitexact(probs, ref["probs"]), f"layer {l} probabilities on the device's own input"
        same = (idx == tr["topk_idx"][l]).all(axis=1)
        if k < M:
            p = np.sort(tr["probs"][l], axis=1)[:, ::-1]
            rel_gap = (p[:, k - 1] - p[:, k]) / p[:, k - 1]
            worst = rel_gap[~same].max() if (~same).any() else 0.0
        else:
            worst = 0.0
        print(f"GRADERR {label} layer {l} routing agreement vs oracle {same.mean():.4f}, "
              f"largest relative top-k gap at a disagreement {worst:.3e}")
        assert same.mean() >= min_agree, f"layer {l} routing agreement {same.mean():.4f}"
        assert worst < 0.05, "routing disagreement away from a near-tie"


def _check_grad_blocks(cfg, g_gpu, g_ref, label, rtol=None):
    """Per-block relative Frobenius error against the oracle; frozen blocks exactly zero.
    The observed maximum is printed (GRADERR lines, pytest -s) so GRAD_RTOL stays a
    measured bound rather than a guess."""
    offs = spes.block_offsets(cfg)
    ends = list(offs[1:]) + [spes.param_count(cfg)]
    worst, worst_at = 0.0, None
    for b0, b1 in zip(offs, ends):
        gr, gg = g_ref[b0:b1], g_gpu[b0:b1]
        if not gr.any():
            assert not gg.any(), f"frozen block {b0} got a gradient"
            continue
        e = rel_err(gg, gr)
        if e > worst:
            worst, worst_at = e, b0
        assert e < (rtol or GRAD_RTOL), f"block at {b0}: rel err {e:.3e}"
    print(f"GRADERR {label} d={cfg.hidden} f={cfg.intermediate} M={cfg.experts_total} "
          f"k={cfg.experts_active} L={cfg.layers}: max block rel err {worst:.3e} at {worst_at}")
    return worst


def _node(cfg, params, owned_lists, node=0):
    n = spes.Node(cfg, node=node, n_nodes=1, device=0)
    n.set_ownership([owned_lists[node]] if len(owned_lists) > 1 else owned_lists)
    n.load_params(params)
    return n


def _check_step(cfg, B, S, owned, seed, renorm=False):
    params = oracle.random_params(cfg, seed)
    tokens = oracle.random_tokens(cfg, B, S, seed + 1)[0]
    node = spes.Node(cfg, 0, 1, 0)
    node.set_ownership([owned])
    node.load_params(params)
    node.set_fused_optimizer(False)  # materialize the gradients for the comparison below
    node.round_begin()
    opt = adamw_cfg(lr=1e-3)
    losses = np.array(node.local_step(tokens, opt))
    g_gpu = node.read_grads()
    p_gpu = node.read_params()
    # AdamW fused into the dW GEMM epilogues -> identical bits, same losses
    fused = spes.Node(cfg, 0, 1, 0)
    fused.set_ownership([owned])
    fused.load_params(params)
    fused.set_fused_optimizer(True)
    fused.round_begin()
    assert np.array_equal(np.array(fused.local_step(tokens, opt)), losses)
    assert bitexact(fused.read_params(), p_gpu), "fused optimizer differs from the standalone pass"
    with pytest.raises(spes.SpesError) as e:
        fused.read_grads()
    assert e.value.kind == "logic_error"
    fused.close()
    T = B * S
    l_ref, g_ref, tr = oracle.forward_backward(cfg, params, tokens, owned, trace=True)
    L, M, k, d = cfg.layers, cfg.experts_total, cfg.experts_active, cfg.hidden
    # layer-0 routing: identical inputs (embedding rows) -> bit-exact
    idx0 = node.debug("topk_idx", 0, np.int32, (T, k), T * k)
    assert bitexact(idx0, tr["topk_idx"][0]), "layer-0 routing indices"
    assert bitexact(node.debug("probs", 0, np.float32, (T, M), T * M), tr["probs"][0])
    assert bitexact(node.debug("counts", 0, np.int32, None, M), tr["counts"][0])
    assert bitexact(node.debug("perm", 0, np.int32, None, T * k), tr["perm"][0])
    # layer-0 input h0 = emb[inputs] is read in place (never materialized): the bit-exact
    # layer-0 routing above covers it; debug("h", 0) rebuilds it from the CURRENT embedding
    emb_now = node.read_params()[: cfg.vocab * d].reshape(cfg.vocab, d)
    assert bitexact(node.debug("h", 0, np.float32, (T, d), T * d),
                    emb_now[tokens[:, :-1].reshape(-1)])
    _check_deep_routing(cfg, node, params, tr, T, "cfg1-like" if d == 128 else f"d={d}")
    # losses
    for i, name in enumerate(("total", "ce", "lb", "moe_z", "z")):
        assert abs(losses[i] - l_ref[i]) <= LOSS_RTOL * abs(l_ref[i]) + 1e-7, name
    # gradients, block by block
    offs = spes.block_offsets(cfg)
    ends = list(offs[1:]) + [spes.param_count(cfg)]
    _check_grad_blocks(cfg, g_gpu, g_ref, f"B={B} S={S}")
    # embedding gradient == sequential scatter-add of the device's own grad_h0 rows in
    # token order (graph.hpp:220-229): bit-exact given identical upstream
    gh0 = node.debug("grad_h0", 0, np.float32, (T, d), T * d)
    inputs = tokens[:, :-1].reshape(-1)
    g_emb = np.zeros((cfg.vocab, d), np.float32)
    for t in range(T):
        g_emb[inputs[t]] += gh0[t]  # float32 adds, ascending t
    assert bitexact(g_gpu[: cfg.vocab * d].reshape(cfg.vocab, d), g_emb), "embedding gradient"
    # optimizer: GPU params == oracle AdamW applied to the GPU's own gradients (bit-exact)
    mask = oracle.trainable_mask(cfg, owned)
    p_chk = params.copy()
    m0 = np.zeros_like(params)
    v0 = np.zeros_like(params)
    import ctypes as C
    oracle.lib().oracle_adamw_step(C.byref(cfg), p_chk, g_gpu, m0, v0, mask, C.byref(opt), 1)
    assert bitexact(p_gpu, p_chk), "AdamW update differs from the oracle on identical grads"
    # frozen experts bit-identical (trainer.hpp frozen blocks)
    per = 3 * cfg.hidden * cfg.intermediate
    for l in range(L):
        for j in range(M):
            if j not in owned:
                o = oracle.expert_offset(cfg, l, j)
                assert bitexact(p_gpu[o:o + per], params[o:o + per])
    c = node.counts()
    P = spes.param_count(cfg)
    psi = oracle.expert_offset(cfg, 0, 0)
    assert c["grad_scalars"] == psi + L * len(owned) * per
    assert c["opt_state_scalars"] == 2 * c["grad_scalars"]
    node.close()


@pytest.mark.parametrize("fused", [True, False])
def test_nonfinite_loss_applies_no_update(gpu, fused):
    """trainer.hpp:166-167: a non-finite loss aborts the round before the optimizer step;
    with the fused optimizer the device-side guard skips the in-epilogue update too."""
    cfg = model_cfg(**CFG1)
    params = oracle.random_params(cfg, 3)
    tokens = oracle.random_tokens(cfg, 2, 64, 4)
    params[: cfg.vocab * cfg.hidden] = np.inf  # embedding rows -> non-finite loss
    node = spes.Node(cfg, 0, 1, 0)
    node.set_ownership([[0, 1, 2, 3]])
    node.load_params(params)
    node.set_fused_optimizer(fused)
    with pytest.raises(spes.SpesError) as e:
        node.local_round(tokens, adamw_cfg())
    assert e.value.kind == "runtime_error"
    assert bitexact(node.read_params(), params)
    assert node.counts()["adam_step"] == 0
    node.close()


def test_local_step_cfg1(gpu):
    _check_step(model_cfg(**CFG1), B=4, S=64, owned=[0, 1, 2, 3], seed=10)


def test_local_step_cfg1_renorm(gpu):
    _check_step(model_cfg(renormalize_after_topk=True, **CFG1), B=2, S=64, owned=[4, 5, 6, 7],
                seed=20)


def test_local_step_cfg2_shapes(gpu):
    _check_step(model_cfg(**CFG2), B=1, S=384, owned=[0, 1, 2, 3], seed=30)


def test_local_step_cfg4_shapes(gpu):
    # M = 64, k = 8, d = 2048: the large-M router (4 tokens per lane), k = 8 combine and
    # backward paths, cta_group::2 GEMMs at d = 2048
    _check_step(model_cfg(**CFG4), B=1, S=256, owned=list(range(16)), seed=35)


def test_local_step_non_pow2_experts(gpu):
    # M = 6, k = 3: the integer-division staging paths of the router / norm-gradient kernels
    # (every shipped config has power-of-two M and k, which index by shifts)
    _check_step(model_cfg(vocab=256, hidden=128, intermediate=256, layers=2, experts_total=6,
                          experts_active=3), B=2, S=80, owned=[1, 4, 5], seed=45)


def test_local_step_reference_default_config(gpu):
    # the reference's default ModelConfig (model.hpp:21-31: V=64, d=32, f=64, L=2, M=4, k=2):
    # hidden / intermediate / vocab are zero-padded to the 128-wide tiles on the device
    _check_step(model_cfg(), B=2, S=32, owned=[1, 2], seed=47)


def test_local_step_unaligned_shapes_renorm(gpu):
    # every dimension off the tile grid, renormalized gates, 6 experts
    _check_step(model_cfg(vocab=100, hidden=96, intermediate=200, layers=2, experts_total=6,
                          experts_active=2, renormalize_after_topk=True),
                B=3, S=40, owned=[0, 3, 5], seed=48)


def test_local_step_ragged_T(gpu):
    # T not a multiple of 128, an owned expert that may receive no tokens
    _check_step(model_cfg(**CFG1), B=3, S=37, owned=[0, 7], seed=40)


@pytest.mark.parametrize("shape", ["cfg1", "cfg4"])
def test_router_gradient_paths(gpu, monkeypatch, shape):
    """Both router-gradient paths (SPES_ROUTER_TC: the tensor-core normed^T glog GEMM, the
    default above 16 experts, and the CUDA-core partial kernel) against the oracle; the
    gain gradient and the rest of the step do not depend on the path (identical bits)."""
    cfg = model_cfg(**(CFG1 if shape == "cfg1" else CFG4))
    B, S, owned = (4, 64, [0, 1, 2, 3]) if shape == "cfg1" else (1, 256, list(range(16)))
    params = oracle.random_params(cfg, 57)
    tokens = oracle.random_tokens(cfg, B, S, 58)[0]
    grads = {}
    for tc in ("0", "1"):
        monkeypatch.setenv("SPES_ROUTER_TC", tc)
        node = spes.Node(cfg, 0, 1, 0)
        node.set_ownership([owned])
        node.load_params(params)
        node.set_fused_optimizer(False)
        node.round_begin()
        node.local_step(tokens, adamw_cfg(lr=1e-3))
        grads[tc] = node.read_grads()
        node.close()
    _, g_ref, _ = oracle.forward_backward(cfg, params, tokens, owned, trace=True)
    for tc, g in grads.items():
        _check_grad_blocks(cfg, g, g_ref, f"{shape} router_tc={tc}")
    keep = np.ones(grads["0"].size, bool)
    for l in range(cfg.layers):  # router block of layer l: d x M after its norm gain
        r0 = oracle.lib().oracle_off_router(C.byref(cfg), l)
        keep[r0:r0 + cfg.hidden * cfg.experts_total] = False
    assert bitexact(grads["0"][keep], grads["1"][keep]), "non-router gradients differ by path"


def test_dswiglu_epilogue_variants_identical_bits(gpu, monkeypatch):
    """Every dSwiGLU epilogue (SPES_DSWIGLU_TMA: 0 direct loads, 1 TMA-staged 64-column
    pieces, 3 / 4 TMA-staged 32-column pieces written back in place by TMA) computes the same
    per-element products: identical gradients, bit for bit (cfg2 shapes: pair tiles)."""
    cfg = model_cfg(**CFG2)
    params = oracle.random_params(cfg, 71)
    tokens = oracle.random_tokens(cfg, 1, 384, 72)[0]
    grads = {}
    for v in ("0", "1", "3", "4"):
        monkeypatch.setenv("SPES_DSWIGLU_TMA", v)
        node = spes.Node(cfg, 0, 1, 0)
        node.set_ownership([[0, 1, 2, 3]])
        node.load_params(params)
        node.set_fused_optimizer(False)
        node.round_begin()
        node.local_step(tokens, adamw_cfg(lr=1e-3))
        grads[v] = node.read_grads()
        node.close()
    for v in ("1", "3", "4"):
        assert bitexact(grads[v], grads["0"]), f"variant {v} differs from the direct epilogue"


def test_normed_grad_load_depth_identical_bits(gpu, monkeypatch):
    """normed_grad_k with all k expert pieces in flight (SPES_NG_ALLK=1, the default for
    k > 4) and with the 2-deep loop sum in the same descending order: identical gradients."""
    cfg = model_cfg(**CFG4)
    params = oracle.random_params(cfg, 73)
    tokens = oracle.random_tokens(cfg, 1, 256, 74)[0]
    grads = {}
    for v in ("0", "1"):
        monkeypatch.setenv("SPES_NG_ALLK", v)
        node = spes.Node(cfg, 0, 1, 0)
        node.set_ownership([list(range(16))])
        node.load_params(params)
        node.set_fused_optimizer(False)
        node.round_begin()
        node.local_step(tokens, adamw_cfg(lr=1e-3))
        grads[v] = node.read_grads()
        node.close()
    assert bitexact(grads["0"], grads["1"])


def test_local_round_and_errors(gpu):
    cfg = model_cfg(**CFG1)
    params = oracle.random_params(cfg, 3)
    node = spes.Node(cfg)
    node.load_params(params)
    toks = oracle.random_tokens(cfg, 2, 64, 5, H=4)
    lr = [spes.lr_at(1e-3, 0.1, 2, 8, h) for h in range(4)]
    losses = node.local_round(toks, adamw_cfg(), lr)
    assert losses.shape == (4, 5) and np.isfinite(losses).all()
    assert node.counts()["adam_step"] == 4
    bad = toks.copy()
    bad[0, 0, 3] = cfg.vocab
    with pytest.raises(spes.SpesError) as e:
        node.local_round(bad, adamw_cfg())
    assert e.value.kind == "out_of_range"
    with pytest.raises(spes.SpesError) as e:
        node.local_round(toks[:0], adamw_cfg())
    assert e.value.kind == "invalid_argument"
    node.close()


def test_local_round_matches_oracle_losses(gpu):
    """H steps: per-step losses track the oracle's local_round within tolerance."""
    cfg = model_cfg(**CFG1)
    params = oracle.random_params(cfg, 9)
    toks = oracle.random_tokens(cfg, 2, 64, 11, H=3)
    owned = [2, 3, 4, 5]
    node = spes.Node(cfg)
    node.set_ownership([owned])
    node.load_params(params)
    l_gpu = node.local_round(toks, adamw_cfg(lr=1e-3))
    _, l_ref = oracle.local_round(cfg, params, toks, owned, adamw_cfg(lr=1e-3))
    assert np.allclose(l_gpu[:, 0], l_ref[:, 0], rtol=5e-3)
    node.close()


@pytest.mark.parametrize("shape,owned,B,S", [(CFG1, [2, 3, 4, 5], 2, 64),
                                             (CFG2, list(range(16)), 1, 512)])
def test_stream_overlap_identical_bits(gpu, shape, owned, B, S):
    """The two-stream step (side-stream bucketing, losses, router scalar backward and the
    experts' AdamW) gives the same bits as the one-stream step, eager and graph-replayed."""
    cfg = model_cfg(**shape)
    params = oracle.random_params(cfg, 21)
    toks = oracle.random_tokens(cfg, B, S, 22, H=4)
    out = []
    for overlap in (True, False):
        node = spes.Node(cfg)
        node.set_ownership([owned])
        node.load_params(params)
        node.set_stream_overlap(overlap)
        losses = node.local_round(toks, adamw_cfg(lr=1e-3))  # step 2 captures, 3-4 replay
        out.append((losses, node.read_params()))
        node.close()
    assert np.array_equal(out[0][0], out[1][0])
    assert bitexact(out[0][1], out[1][1])


# ---------------------------------------------------------------- merge warm-up

def _check_operand_copies(node, cfg):
    """The bf16 GEMM operand copies the merge wrote equal a fresh refresh from fp32."""
    d, f, M = cfg.hidden, cfg.intermediate, cfg.experts_total
    def copies():
        return [node.debug(w, l, np.uint16, None, M * n)
                for l in range(cfg.layers) for w, n in (("w1", 2 * d * f), ("w2", d * f))]
    merged = copies()
    node.load_params(node.read_params())  # rewrites every copy from the fp32 parameters
    assert all(np.array_equal(a, b) for a, b in zip(merged, copies())), "operand copies"


def test_merge_bitexact_vs_oracle(gpu):
    cfg = model_cfg(**CFG1)
    params = oracle.random_params(cfg, 13, std=0.05)
    node = spes.Node(cfg)
    node.load_params(params)
    sched = merge_sched(warmup_rounds=10, interval=1, alpha0=0.1, peers=4, source=0)
    sim_gpu = node.similarity(1, 0)
    sim_ref = oracle.similarity(cfg, params, 1, 0)
    assert np.allclose(sim_gpu, sim_ref, rtol=1e-12, atol=1e-14)
    ev_gpu, peers_gpu = node.merge_model(sched, 0)
    p_ref, ev_ref, peers_ref = oracle.merge_model(cfg, params, sched, 0)
    assert (peers_gpu == peers_ref).all()
    assert bitexact(node.read_params(), p_ref)
    _check_operand_copies(node, cfg)
    for a, b in zip(ev_gpu, ev_ref):
        assert a[0] == b[0] and a[1] == b[1] and a[2] == b[2]
        assert abs(a[3] - b[3]) <= 1e-9 * abs(b[3])
    # inactive schedule: no events, params unchanged
    ev, _ = node.merge_model(sched, 10)
    assert ev == []
    node.close()


def test_merge_concat_source_and_cfg2(gpu):
    cfg = model_cfg(**CFG2)
    params = oracle.random_params(cfg, 17, std=0.02)
    node = spes.Node(cfg)
    node.load_params(params)
    sched = merge_sched(warmup_rounds=4, interval=2, alpha0=0.2, peers=3, source=2)
    ev_gpu, peers_gpu = node.merge_model(sched, 2)
    p_ref, ev_ref, peers_ref = oracle.merge_model(cfg, params, sched, 2)
    assert (peers_gpu == peers_ref).all()
    assert bitexact(node.read_params(), p_ref)
    node.close()


@pytest.mark.parametrize("kind", ["sgd", "nesterov"])
def test_outer_sync_single_node_matches_oracle(gpu, kind):
    """DiLoCo baseline (protocol.cpp:199-213): two rounds of local training + outer step on
    one node, bit-exact with OuterOptimizer::step restated (Nesterov state carried)."""
    cfg = model_cfg(**CFG1)
    params = oracle.random_params(cfg, 41)
    node = spes.Node(cfg, 0, 1, 0)
    node.set_ownership([list(range(cfg.experts_total))])
    node.load_params(params)
    node.outer_begin()
    theta = params.copy()
    buf = np.zeros(theta.size)
    k = 0 if kind == "sgd" else 1
    for rnd in range(2):
        node.local_round(oracle.random_tokens(cfg, 2, 64, 42 + rnd, H=2), adamw_cfg(lr=1e-3))
        local = node.read_params()
        node.outer_sync(kind, lr=0.7, momentum=0.9)
        oracle.outer_step(k, 0.7, 0.9, theta, local[None], buf)
        assert bitexact(node.read_params(), theta), f"round {rnd}"
    node.close()


def test_upcycled_model_local_step(gpu):
    """An upcycled model (model.hpp:415-460; renorm on, identical router columns => every
    token's expert probabilities tie exactly) trains on B200 with the oracle's routing
    (stable ties -> lowest indices) bit-exact and losses within tolerance."""
    dense_cfg = model_cfg(vocab=256, hidden=128, intermediate=256, layers=2, experts_total=1,
                          experts_active=1)
    dense = oracle.random_params(dense_cfg, 51)
    ucfg, up = spes.upcycle_from_dense(dense_cfg, dense, 8, 0.5, 0.02, 52)
    ucfg.experts_active = 2
    tokens = oracle.random_tokens(ucfg, 2, 64, 53)[0]
    owned = [0, 1, 2, 3]
    node = spes.Node(ucfg, 0, 1, 0)
    node.set_ownership([owned])
    node.load_params(up)
    node.round_begin()
    losses = node.local_step(tokens, adamw_cfg())
    l_ref, _, tr = oracle.forward_backward(ucfg, up, tokens, owned, trace=True)
    T = 2 * 64
    idx0 = node.debug("topk_idx", 0, np.int32, (T, 2), T * 2)
    assert bitexact(idx0, tr["topk_idx"][0])
    assert (idx0 == np.array([0, 1])).all()  # exact ties -> lowest indices
    assert abs(losses[0] - l_ref[0]) <= LOSS_RTOL * abs(l_ref[0])
    node.close()


# ---------------------------------------------------------------- batch shapes, status, SGD

def test_batch_shape_change_same_token_count(gpu, monkeypatch):
    """(B, S) changes with B*S fixed: the replayed step graph must not split the
    new batch with the old S. A graph-replaying node and an eager node (SPES_STEP_GRAPH=0)
    run the same shape sequence and must agree bit for bit; each step's layer-0 routing is
    checked against the oracle on that step's own (B, S) batch."""
    cfg = model_cfg(**CFG1)
    params = oracle.random_params(cfg, 61)
    shapes = [(4, 64), (4, 64), (4, 64), (8, 32), (8, 32), (8, 32), (2, 128), (4, 64)]
    batches = [oracle.random_tokens(cfg, B, S, 62 + i)[0] for i, (B, S) in enumerate(shapes)]
    out = []
    for graph in ("1", "0"):
        monkeypatch.setenv("SPES_STEP_GRAPH", graph)
        node = spes.Node(cfg)
        node.set_ownership([[0, 1, 2, 3]])
        node.load_params(params)
        node.round_begin()
        losses = []
        for tk in batches:
            p_before = node.read_params()
            losses.append(node.local_step(tk, adamw_cfg(lr=1e-3)))
            T = tk.shape[0] * (tk.shape[1] - 1)
            _, _, tr = oracle.forward_backward(cfg, p_before, tk, [0, 1, 2, 3], trace=True)
            idx = node.debug("topk_idx", 0, np.int32, (T, cfg.experts_active), T * cfg.experts_active)
            assert bitexact(idx, tr["topk_idx"][0]), f"graph={graph}: routing of a {tk.shape} batch"
        out.append((np.array(losses), node.read_params()))
        node.close()
    assert np.array_equal(out[0][0], out[1][0])
    assert bitexact(out[0][1], out[1][1])


def test_device_tokens_status_reported_at_round_end(gpu):
    """Device-resident tokens without loss reads (the bench path): an out-of-vocabulary id
    applies no update (model.hpp:280-281 throws before the step) and is reported when the
    round ends, as out_of_range; the status then clears and training resumes."""
    import torch
    cfg = model_cfg(**CFG1)
    params = oracle.random_params(cfg, 71)
    node = spes.Node(cfg)
    node.load_params(params)
    node.round_begin()
    good = oracle.random_tokens(cfg, 2, 64, 72)[0]
    bad = good.copy()
    bad[1, 5] = cfg.vocab + 3
    d_good = torch.from_numpy(good).cuda()
    d_bad = torch.from_numpy(bad).cuda()
    node.local_step_device(d_good.data_ptr(), 2, 64)
    p1 = node.read_params()
    node.local_step_device(d_bad.data_ptr(), 2, 64)    # no host sync: not raised yet
    node.local_step_device(d_good.data_ptr(), 2, 64)   # after a bad step: no update either
    torch.cuda.synchronize()
    assert bitexact(node.read_params(), p1), "an update was applied after a bad batch"
    with pytest.raises(spes.SpesError) as e:
        node.sync()
    assert e.value.kind == "out_of_range"
    node.round_begin()                                   # cleared: trains again
    node.local_step_device(d_good.data_ptr(), 2, 64)
    node.sync()
    assert not bitexact(node.read_params(), p1)
    # with losses requested, the step itself reports
    node.round_begin()
    with pytest.raises(spes.SpesError) as e:
        node.local_step_device(d_bad.data_ptr(), 2, 64, want_losses=True)
    assert e.value.kind == "out_of_range"
    node.close()


def test_sgd_inner_optimizer(gpu):
    """InnerOpt::SGD (trainer.hpp:197-204): theta -= float(lr) * g on the trainable blocks,
    bit-exact given the device's own gradients; frozen experts untouched; no moments."""
    cfg = model_cfg(**CFG1)
    params = oracle.random_params(cfg, 81)
    tokens = oracle.random_tokens(cfg, 2, 64, 82)[0]
    owned = [1, 2, 5, 6]
    node = spes.Node(cfg)
    node.set_ownership([owned])
    node.load_params(params)
    node.set_inner_optimizer("sgd")
    node.round_begin()
    lr = 0.05
    losses = node.local_step(tokens, adamw_cfg(lr=lr))
    g = node.read_grads()
    p = node.read_params()
    assert bitexact(p, params - np.float32(lr) * g)
    l_ref, g_ref, _ = oracle.forward_backward(cfg, params, tokens, owned, trace=True)
    assert abs(losses[0] - l_ref[0]) <= LOSS_RTOL * abs(l_ref[0])
    assert node.counts()["opt_state_scalars"] == 0
    node.set_fused_optimizer(True)       # no fused placement for SGD: same path
    losses2 = node.local_step(tokens, adamw_cfg(lr=lr))
    assert bitexact(node.read_params(), p - np.float32(lr) * node.read_grads())
    node.close()
