"""Stress the router-kernel parity case that flaked once (cfg1, T=256): repeat GPU routing
and the oracle, report every disagreement in detail."""
import sys
import numpy as np
import oracle
import paper_2602_11543_b200 as spes
from paper_2602_11543_b200.abi import model_cfg

CFG1 = dict(vocab=256, hidden=128, intermediate=256, layers=2, experts_total=8, experts_active=2)
cfg = model_cfg(**CFG1)
T, d, M, k = 256, 128, 8, 2
rng = np.random.default_rng(0)
h = (rng.standard_normal((T, d)) * 0.5).astype(np.float32)
gain = (1 + 0.1 * rng.standard_normal(d)).astype(np.float32)
router = (rng.standard_normal((d, M)) * 0.05).astype(np.float32)
router[:, 1] = router[:, 0]
h[:8] = h[8:16]
n = int(sys.argv[1]) if len(sys.argv) > 1 else 50
refs = [oracle.router_forward(cfg, h, gain, router) for _ in range(3)]
for r in refs[1:]:
    for key in r:
        if not np.array_equal(r[key].view(np.uint8), refs[0][key].view(np.uint8)):
            print("ORACLE NONDETERMINISTIC", key)
ref = refs[0]
bad_runs = 0
for it in range(n):
    out = dict(normed=np.zeros((T, d), np.float32), logits=np.zeros((T, M), np.float32),
               probs=np.zeros((T, M), np.float32), idx=np.zeros((T, k), np.int32),
               w=np.zeros((T, k), np.float32), counts=np.zeros(M, np.int32),
               perm=np.zeros(T * k, np.int32))
    spes._check(spes.lib().spes_kernel_router(
        cfg, spes.f32(h), spes.f32(gain), spes.f32(router), T, spes.f32(out["normed"]),
        spes.f32(out["logits"]), spes.f32(out["probs"]), spes.i32(out["idx"]), spes.f32(out["w"]),
        spes.i32(out["counts"]), spes.i32(out["perm"]), 0))
    diffs = [key for key in out if not np.array_equal(out[key].view(np.uint8), ref[key].view(np.uint8))]
    if diffs:
        bad_runs += 1
        print(f"iter {it}: differs in {diffs}")
        if "perm" in diffs:
            b = np.flatnonzero(out["perm"] != ref["perm"])
            print("  perm idx", b[:8], "gpu", out["perm"][b[:8]], "ref", ref["perm"][b[:8]])
            for t in set(out["perm"][b[:4]]) | set(ref["perm"][b[:4]]):
                print(f"  token {t}: gpu idx {out['idx'][t]} ref idx {ref['idx'][t]}")
            # recompute the reference perm from the GPU's own idx
            cnt = np.bincount(out["idx"].reshape(-1), minlength=M)
            pos = np.concatenate([[0], np.cumsum(cnt)])[:-1].copy()
            p2 = np.zeros(T * k, np.int32)
            for t in range(T):
                for s in range(k):
                    e = out["idx"][t, s]; p2[pos[e]] = t; pos[e] += 1
            print("  perm from gpu idx == gpu perm:", np.array_equal(p2, out["perm"]),
                  "== ref perm:", np.array_equal(p2, ref["perm"]))
print(f"{bad_runs} of {n} runs differ")
