"""Wire / checkpoint format against the UNMODIFIED reference
(proj/src/wire.cpp through oracle/_ref): byte-identical GLOBAL_MODEL payloads and
checkpoints, both directions, and the reference's decode errors (ProtoError code and
message) on corrupted input."""
import ctypes as C
import os

import numpy as np
import pytest

import oracle
import paper_2602_11543_b200 as spes
from paper_2602_11543_b200.abi import model_cfg

SHAPES = {
    "tiny": dict(vocab=64, hidden=32, intermediate=64, layers=2, experts_total=4, experts_active=2),
    "cfg1": dict(vocab=256, hidden=128, intermediate=256, layers=2, experts_total=8,
                 experts_active=2),
}

needs_ref = pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built")


def ref_encode(cfg, params):
    R = oracle.ref()
    n = R.ref_encode_model(C.byref(cfg), params, None, 0)
    out = np.zeros(n, np.uint8)
    R.ref_encode_model(C.byref(cfg), params, out.ctypes.data_as(C.c_void_p), n)
    return out


def ref_decode(cfg, payload):
    """(params or None, error message or None)"""
    R = oracle.ref()
    out = np.zeros(spes.param_count(cfg), np.float32)
    err = C.create_string_buffer(512)
    rc = R.ref_decode_model(C.byref(cfg), np.ascontiguousarray(payload, np.uint8), payload.size,
                            out, err, 512)
    return (out, None) if rc == 0 else (None, err.value.decode())


@needs_ref
@pytest.mark.parametrize("name", sorted(SHAPES))
def test_payload_bytes_identical_to_reference(name):
    cfg = model_cfg(**SHAPES[name])
    params = oracle.random_params(cfg, 21)
    ours = spes.encode_model(cfg, params)
    ref = ref_encode(cfg, params)
    assert spes.model_payload_bytes(cfg) == ref.size
    assert np.array_equal(ours, ref)
    back = spes.decode_model(cfg, ref)
    assert np.array_equal(back.view(np.uint32), params.view(np.uint32))


@needs_ref
def test_checkpoint_round_trip_with_reference(tmp_path):
    cfg = model_cfg(**SHAPES["cfg1"])
    params = oracle.random_params(cfg, 22)
    R = oracle.ref()
    # reference writes, our codec reads (payload + u64 round trailer, wire.cpp:212-236)
    p_ref = str(tmp_path / "ref.ckpt")
    assert R.ref_write_checkpoint(C.byref(cfg), params, p_ref.encode(), 77) == 0
    raw = np.fromfile(p_ref, np.uint8)
    assert int.from_bytes(raw[-8:].tobytes(), "little") == 77
    assert np.array_equal(spes.decode_model(cfg, raw[:-8]).view(np.uint32), params.view(np.uint32))
    # our bytes == the reference's checkpoint bytes
    assert np.array_equal(np.concatenate([spes.encode_model(cfg, params),
                                          np.frombuffer((77).to_bytes(8, "little"), np.uint8)]),
                          raw)


def _corruptions(payload, cfg):
    """(label, bytes) cases that decode_blocks / blocks_into_model reject"""
    p = payload.copy()
    yield "truncated-header", p[:3]
    yield "truncated-values", p[: p.size - 5]
    yield "trailing-bytes", np.concatenate([p, np.zeros(3, np.uint8)])
    q = p.copy()
    q[6] ^= 0x01  # first block name "psi.emb" -> different name
    yield "renamed-block", q
    q = p.copy()
    nlen = int(p[4]) | int(p[5]) << 8
    q[6 + nlen] = 1  # dtype byte
    yield "bad-dtype", q
    q = p.copy()
    q[6 + nlen + 1] = 0  # rank byte
    yield "bad-rank", q
    q = p.copy()
    q[0] = 1  # block count 1 (then trailing bytes)
    yield "wrong-count", q


@needs_ref
def test_decode_errors_match_reference():
    cfg = model_cfg(**SHAPES["tiny"])
    payload = ref_encode(cfg, oracle.random_params(cfg, 23))
    for label, bad in _corruptions(payload, cfg):
        _, ref_err = ref_decode(cfg, bad)
        assert ref_err is not None, label
        with pytest.raises(spes.SpesError) as e:
            spes.decode_model(cfg, bad)
        assert e.value.kind == "protocol_error", label
        assert str(e.value).endswith(ref_err), (label, str(e.value), ref_err)


@pytest.mark.gpu
def test_device_export_import_and_checkpoint(tmp_path):
    """ctx encode == host encode of the device parameters; the reference reads our
    checkpoint; our ctx reads the reference's checkpoint and trains on it identically."""
    from paper_2602_11543_b200.abi import adamw_cfg
    cfg = model_cfg(**SHAPES["cfg1"])
    params = oracle.random_params(cfg, 24)
    node = spes.Node(cfg, 0, 1, 0)
    try:
        node.set_ownership([[0, 1, 2, 3]])
        node.load_params(params)
        assert np.array_equal(node.encode_model(), spes.encode_model(cfg, params))
        path = str(tmp_path / "b200.ckpt")
        node.write_checkpoint(path, 5)
        if oracle.ref_available():
            out = np.zeros(spes.param_count(cfg), np.float32)
            r = C.c_uint64()
            assert oracle.ref().ref_read_checkpoint(C.byref(cfg), path.encode(), out, C.byref(r),
                                                    None, 0) == 0
            assert r.value == 5 and np.array_equal(out.view(np.uint32), params.view(np.uint32))
        # import into a fresh context, then one step: identical to load_params
        tokens = oracle.random_tokens(cfg, 2, 64, 25)[0]
        other = spes.Node(cfg, 0, 1, 0)
        other.set_ownership([[0, 1, 2, 3]])
        assert other.read_checkpoint(path) == 5
        other.round_begin()
        node.round_begin()
        assert np.array_equal(np.array(other.local_step(tokens, adamw_cfg())),
                              np.array(node.local_step(tokens, adamw_cfg())))
        assert np.array_equal(other.read_params().view(np.uint32),
                              node.read_params().view(np.uint32))
        other.decode_model(spes.encode_model(cfg, params))
        assert np.array_equal(other.read_params().view(np.uint32), params.view(np.uint32))
        other.close()
    finally:
        node.close()
