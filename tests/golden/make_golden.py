"""Generate tests/golden/reference_golden.json from the UNMODIFIED reference.

oracle/_ref/libspes_ref.so is the reference (/root/reference/proj) compiled from its own
sources with its own flags (oracle/Makefile) behind a thin C shim. This script runs
its public entry points on small seeded inputs and records the outputs (scalars in
float hex, integer arrays verbatim, large float arrays as sha256 of their bytes), so
the oracle restatement stays pinned on machines where the reference tree is absent
(tests/test_golden.py). Run from the repo root:  python tests/golden/make_golden.py

Entry points recorded (reference file:line):
  build_loss + GraphT::backward   model.hpp:252-373, graph.hpp:340-348
  local_round (AdamW, H steps)    trainer.hpp:143-222
  MaskedAdamW::step               trainer.hpp:56-112
  Server::aggregate               protocol.cpp:197-251
  similarity_matrix / merge_model merging.hpp:55-150
"""
import ctypes as C
import hashlib
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from paper_2602_11543_b200.abi import MergeEvent, adamw_cfg, merge_sched, model_cfg  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "reference_golden.json")

CASES = {
    "tiny": dict(vocab=64, hidden=32, intermediate=64, layers=2, experts_total=4, experts_active=2),
    "tiny_renorm": dict(vocab=64, hidden=32, intermediate=64, layers=2, experts_total=4,
                        experts_active=2, renormalize_after_topk=True),
    "cfg1": dict(vocab=256, hidden=128, intermediate=256, layers=2, experts_total=8,
                 experts_active=2),
}
SEEDS = dict(params=11, tokens=12)


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def fhex(x):
    return float(x).hex()


def inputs(cfg, B, S, H=1):
    params = oracle.random_params(cfg, SEEDS["params"])
    tokens = oracle.random_tokens(cfg, B, S, SEEDS["tokens"], H)
    return params, tokens


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


def main():
    R = oracle.ref()
    R.ref_set_parallel(0)
    g = {"generator": "tests/golden/make_golden.py", "seeds": SEEDS, "cases": {}}
    for name, shape in CASES.items():
        cfg = model_cfg(**shape)
        B, S, H = (2, 8, 3) if name.startswith("tiny") else (1, 64, 2)
        owned = [0, 1] if name.startswith("tiny") else [0, 1, 2, 3]
        params, tokens = inputs(cfg, B, S, H)
        c = {"shape": shape, "B": B, "S": S, "H": H, "owned": owned,
             "params_sha": sha(params), "tokens_sha": sha(tokens)}
        # one forward/backward (first batch)
        losses, grads, probs, idx, w = ref_fwd_bwd(cfg, params, tokens[0], owned)
        c["fwd_bwd"] = {"losses": [fhex(x) for x in losses], "grads_sha": sha(grads),
                        "probs_sha": sha(probs), "topk_idx": idx.tolist(), "topk_w_sha": sha(w)}
        # local_round, constant lr, fresh AdamW state
        opt = adamw_cfg()
        p_ref = params.copy()
        lr = np.full(H, 1e-3)
        l_ref = np.zeros((H, 5))
        rc = R.ref_local_round(C.byref(cfg), p_ref, np.ascontiguousarray(tokens), B, S, H, lr,
                               C.byref(opt), oracle.trainable_mask(cfg, owned), l_ref)
        assert rc == 0
        c["local_round"] = {"losses": [[fhex(x) for x in row] for row in l_ref],
                            "params_sha": sha(p_ref)}
        # Server::aggregate over a 2-node param_partition (node n trained its own shard)
        N = 2
        rng = np.random.default_rng(5)
        nodes = np.stack([params + (rng.standard_normal(params.size) * 1e-3).astype(np.float32)
                          for _ in range(N)])
        agg = np.zeros_like(params)
        assert R.ref_aggregate_partition(C.byref(cfg), N, np.ascontiguousarray(nodes), params,
                                         agg) == 0
        c["aggregate_n2"] = {"out_sha": sha(agg)}
        # merge_model at round 0 on the trained parameters
        sched = merge_sched(warmup_rounds=4, interval=1, alpha0=0.1,
                            peers=min(3, cfg.experts_total - 1))
        p_m = p_ref.copy()
        L, M = cfg.layers, cfg.experts_total
        K = max(1, min(sched.peers, M - 1))
        ev = (MergeEvent * L)()
        peers = np.zeros((L, M, K), np.int32)
        n = R.ref_merge_model(C.byref(cfg), p_m, C.byref(sched), 0, C.cast(ev, C.c_void_p), peers)
        c["merge_round0"] = {"n_events": int(n), "peers": peers[:n].tolist(),
                             "alpha": [fhex(e.alpha) for e in ev[:n]],
                             "displacement_sq": [fhex(e.displacement_sq) for e in ev[:n]],
                             "params_sha": sha(p_m)}
        g["cases"][name] = c
    with open(OUT, "w") as f:
        json.dump(g, f, indent=1)
    print("wrote", OUT)


if __name__ == "__main__":
    main()
