"""Reproduce the (now fixed, profiles/r02/flake_fix) intermittent permutation mismatch of spes_kernel_router."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import oracle
import paper_2602_11543_b200 as spes
from paper_2602_11543_b200.abi import model_cfg

CFG1 = dict(vocab=256, hidden=128, intermediate=256, layers=2, experts_total=8, experts_active=2)
CFG4 = dict(vocab=256, hidden=2048, intermediate=1024, layers=1, experts_total=64, experts_active=8)


def run(shape, T, seed, reps):
    cfg = model_cfg(**shape)
    rng = np.random.default_rng(seed)
    d, M, k = cfg.hidden, cfg.experts_total, cfg.experts_active
    h = (rng.standard_normal((T, d)) * 0.5).astype(np.float32)
    gain = (1 + 0.1 * rng.standard_normal(d)).astype(np.float32)
    router = (rng.standard_normal((d, M)) * 0.05).astype(np.float32)
    ref = oracle.router_forward(cfg, h, gain, router)
    bad_runs = 0
    for it in range(reps):
        out = dict(idx=np.zeros((T, k), np.int32), w=np.zeros((T, k), np.float32),
                   counts=np.zeros(M, np.int32), perm=np.zeros(T * k, np.int32),
                   probs=np.zeros((T, M), np.float32))
        spes._check(spes.lib().spes_kernel_router(
            cfg, spes.f32(h), spes.f32(gain), spes.f32(router), T, None, None,
            spes.f32(out["probs"]), spes.i32(out["idx"]), spes.f32(out["w"]),
            spes.i32(out["counts"]), spes.i32(out["perm"]), 0))
        msg = []
        for key in ("probs", "idx", "w", "counts", "perm"):
            a, b = out[key].reshape(-1), ref[key].reshape(-1)
            bad = np.flatnonzero(a.view(np.uint32) != b.view(np.uint32))
            if bad.size:
                msg.append(f"{key}: {bad.size} differ at {bad[:6]} got {a[bad[:6]]} want {b[bad[:6]]}")
        if msg:
            bad_runs += 1
            print(f"T={T} M={M} rep {it}: " + " | ".join(msg), flush=True)
    print(f"T={T} M={M}: {bad_runs}/{reps} runs with a mismatch", flush=True)


if __name__ == "__main__":
    # heavy allocation churn first, like the test suite's exhaustive expf test
    x = np.linspace(-100, 0, 1 << 27, dtype=np.float32)
    y = np.empty_like(x)
    spes._check(spes.lib().spes_kernel_expf(spes.f32(x), spes.f32(y), x.size, 0))
    run(CFG4, 16384, 4, 3)
    run(CFG1, 256, 5, 200)
    run(CFG4, 16384, 4, 20)
    run(CFG1, 256, 5, 200)
