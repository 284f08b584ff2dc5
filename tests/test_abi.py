"""CPU-side checks of the C-ABI library: it loads, exports every declared symbol,
and its pure-host helpers agree with the oracle / reference. No device calls."""
import ctypes as C
import os
import re

import numpy as np
import pytest

import oracle
import paper_2602_11543_b200 as spes
from paper_2602_11543_b200.abi import merge_sched, model_cfg

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "spes_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(spes_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    L = spes.lib()
    names = declared_symbols()
    assert len(names) >= 30
    missing = [n for n in names if not hasattr(L, n)]
    assert not missing, missing


def test_param_count_and_offsets_match_oracle():
    for shape in [dict(vocab=256, hidden=128, intermediate=256, layers=2, experts_total=8,
                       experts_active=2),
                  dict(vocab=256, hidden=1024, intermediate=1024, layers=1, experts_total=16,
                       experts_active=2)]:
        cfg = model_cfg(**shape)
        assert spes.param_count(cfg) == oracle.param_count(cfg)
        offs = spes.block_offsets(cfg)
        L, M = cfg.layers, cfg.experts_total
        assert len(offs) == 2 + 2 * L + 3 * L * M  # enumerate_blocks (model.hpp:95-111)
        assert offs[2 + 2 * L] == oracle.expert_offset(cfg, 0, 0)


def test_validate_cfg_errors_mirror_reference():
    L = spes.lib()
    ok = model_cfg(vocab=256, hidden=128, intermediate=256, layers=1, experts_total=8,
                   experts_active=2)
    assert L.spes_validate_cfg(C.byref(ok)) == 0
    bad_k = model_cfg(vocab=256, hidden=128, intermediate=256, layers=1, experts_total=4,
                      experts_active=5)
    assert L.spes_validate_cfg(C.byref(bad_k)) == 1  # invalid_argument (model.hpp:36-37)
    assert b"1 <= k <= M" in L.spes_last_error()
    tied = model_cfg(vocab=256, hidden=128, intermediate=256, layers=1, experts_total=4,
                     experts_active=2)
    tied.tied_head = 1
    assert L.spes_validate_cfg(C.byref(tied)) == 3  # logic_error (model.hpp:361)
    # any hidden / intermediate / vocab size: the device layout pads them to the tcgen05
    # tile; the reference's own default ModelConfig (model.hpp:21-31) is accepted
    odd = model_cfg(vocab=100, hidden=96, intermediate=200, layers=1, experts_total=4,
                    experts_active=2)
    assert L.spes_validate_cfg(C.byref(odd)) == 0
    assert L.spes_validate_cfg(C.byref(model_cfg())) == 0
    big_m = model_cfg(vocab=256, hidden=128, intermediate=256, layers=1, experts_total=65,
                      experts_active=2)
    assert L.spes_validate_cfg(C.byref(big_m)) == 1  # B200 routing limit: M <= 64
    zero = model_cfg(vocab=256, hidden=0, intermediate=256, layers=1, experts_total=4,
                     experts_active=2)
    assert L.spes_validate_cfg(C.byref(zero)) == 1  # model.hpp:33-35


@pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built")
def test_partition_and_lr_schedule_match_reference():
    R = oracle.ref()
    for M, N in [(8, 2), (16, 8), (7, 3), (64, 5), (4, 4)]:
        cfg = model_cfg(experts_total=M, experts_active=1)
        offs = np.zeros(N + 1, np.int32)
        ex = np.zeros(M, np.int32)
        R.ref_param_partition(C.byref(cfg), N, offs, ex)
        assert spes.param_partition(cfg, N) == [list(ex[offs[i]:offs[i + 1]]) for i in range(N)]
    with pytest.raises(spes.SpesError):
        spes.param_partition(model_cfg(experts_total=4, experts_active=1), 5)
    for args in [(1e-3, 0.1, 5, 100), (3e-4, 0.0, 0, 50), (1e-2, 0.5, 10, 5)]:
        for s in range(0, 120, 3):
            assert spes.lr_at(*args, s) == R.ref_lr_at(*args, s)


def test_merge_schedule_helpers():
    L = spes.lib()
    s = merge_sched(warmup_rounds=10, interval=2, alpha0=0.1)
    assert [L.spes_merge_at(C.byref(s), r) for r in range(12)] == \
        [1, 0, 1, 0, 1, 0, 1, 0, 1, 0, 0, 0]
    a = C.c_double()
    assert L.spes_alpha_at(C.byref(s), 5, C.byref(a)) == 0 and abs(a.value - 0.05) < 1e-15
    assert L.spes_alpha_at(C.byref(s), -1, C.byref(a)) == 1  # invalid_argument (merging.hpp:29)


def test_replicated_ownership_layout():
    # node n -> {(2n+i) mod 16, i<4}
    own = spes.replicated_ownership(16, 8, 2)
    assert own[0] == [0, 1, 2, 3] and own[7] == [0, 1, 14, 15]
    counts = np.zeros(16, int)
    for o in own:
        counts[o] += 1
    assert (counts == 2).all()


def test_host_expf_port_matches_glibc_sample():
    """Host twin of the device port vs this host's glibc expf (a stride sample of all
    2^32 floats; the GPU test sweeps [-104, 0] exhaustively on the device)."""
    bits = np.arange(0, 1 << 32, 257, dtype=np.uint64).astype(np.uint32)
    x = bits.view(np.float32)
    x = x[~np.isnan(x)]
    y = np.empty_like(x)
    spes.lib().spes_host_expf_port(spes.f32(x), spes.f32(y), x.size, 0)
    assert oracle.lib().oracle_expf_mismatches(x, y, x.size) == 0
