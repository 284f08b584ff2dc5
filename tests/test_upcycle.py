"""Upcycling: spes_upcycle_from_dense against the UNMODIFIED reference's
upcycle_from_dense (model.hpp:415-460, through oracle/_ref) bit for bit, plus the
reference's own properties (test_model.cpp:240-290)."""
import ctypes as C

import numpy as np
import pytest

import oracle
import paper_2602_11543_b200 as spes
from paper_2602_11543_b200.abi import model_cfg

DENSE = dict(vocab=64, hidden=32, intermediate=64, layers=2, experts_total=1, experts_active=1)


def dense_params(seed=3):
    cfg = model_cfg(**DENSE)
    return cfg, oracle.random_params(cfg, seed)


@pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("m,frac,std,seed", [(4, 0.5, 0.02, 99), (3, 0.0, 5.0, 99), (4, 0.5, 0.0, 7),
                                              (8, 1.0, 0.1, 1)])
def test_upcycle_bitexact_with_reference(m, frac, std, seed):
    cfg, dense = dense_params()
    ucfg, ours = spes.upcycle_from_dense(cfg, dense, m, frac, std, seed)
    ref = np.zeros_like(ours)
    assert oracle.ref().ref_upcycle(C.byref(cfg), dense, m, frac, std, seed, ref) == 0
    assert np.array_equal(ours.view(np.uint32), ref.view(np.uint32))
    assert ucfg.experts_total == m and ucfg.renormalize_after_topk == 1


def test_upcycle_properties():
    cfg, dense = dense_params()
    m = 4
    ucfg, up = spes.upcycle_from_dense(cfg, dense, m, 0.5, 0.0, 99)  # no noise
    offs_d, offs_u = spes.block_offsets(cfg), spes.block_offsets(ucfg)
    d, f, L, V = cfg.hidden, cfg.intermediate, cfg.layers, cfg.vocab
    assert np.array_equal(up[: 2 * V * d], dense[: 2 * V * d])  # emb + head
    for l in range(L):
        rd = dense[offs_d[3 + 2 * l]: offs_d[3 + 2 * l] + d]                  # router d x 1
        ru = up[offs_u[3 + 2 * l]: offs_u[3 + 2 * l] + d * m].reshape(d, m)  # d x m
        assert (ru == rd[:, None]).all()
        e = dense[oracle.expert_offset(cfg, l, 0): oracle.expert_offset(cfg, l, 0) + 3 * d * f]
        for j in range(m):
            o = oracle.expert_offset(ucfg, l, j)
            assert np.array_equal(up[o: o + 3 * d * f], e)  # noise_std 0 -> exact copies
    # with noise: every expert differs from the dense one on about noise_frac of elements
    _, noisy = spes.upcycle_from_dense(cfg, dense, m, 0.5, 0.02, 99)
    o = oracle.expert_offset(ucfg, 0, 1)
    e = dense[oracle.expert_offset(cfg, 0, 0): oracle.expert_offset(cfg, 0, 0) + d * f]
    frac = np.mean(noisy[o: o + d * f] != e)
    assert 0.45 < frac <= 0.5


def test_upcycle_errors_mirror_reference():
    cfg, dense = dense_params()
    with pytest.raises(spes.SpesError) as e:
        spes.upcycle_from_dense(cfg, dense, 1)
    assert e.value.kind == "invalid_argument"
    ucfg, up = spes.upcycle_from_dense(cfg, dense, 2)
    with pytest.raises(spes.SpesError) as e:
        spes.upcycle_from_dense(ucfg, up, 4)  # source must have a single expert
    assert e.value.kind == "invalid_argument"
