"""Synthetic corpus and batch streams against the UNMODIFIED reference's
gen_corpus / shard_corpus / make_batch_provider (proj/src/corpus.cpp via oracle/_ref), and
the device-resident corpus path: a local round over corpus rows equals the same round over
host-uploaded tokens bit for bit, and the reference's own batches trained by the oracle
within the loss tolerance."""
import numpy as np
import pytest

import oracle
import paper_2602_11543_b200 as spes
from paper_2602_11543_b200.abi import adamw_cfg, model_cfg

CORPUS = dict(vocab=256, seq=64, sources=4, sequences=96, seed=17)
needs_ref = pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built")


@needs_ref
@pytest.mark.parametrize("skew", [0.0, 1.5])
def test_gen_corpus_bitexact(skew):
    c = CORPUS
    tok, sid = spes.gen_corpus(c["vocab"], c["seq"], c["sources"], c["sequences"], c["seed"], skew)
    rt = np.zeros_like(tok)
    rs = np.zeros_like(sid)
    assert oracle.ref().ref_gen_corpus(c["vocab"], c["seq"], c["sources"], c["sequences"], c["seed"],
                                       skew, rt, rs) == 0
    assert np.array_equal(tok, rt) and np.array_equal(sid, rs)
    assert (sid == np.arange(c["sequences"]) % c["sources"]).all()  # balanced mixture


@needs_ref
@pytest.mark.parametrize("by_source", [False, True])
def test_shards_and_batch_stream_bitexact(by_source):
    c = CORPUS
    tok, sid = spes.gen_corpus(c["vocab"], c["seq"], c["sources"], c["sequences"], c["seed"])
    nodes = 3
    shards = spes.shard_corpus(sid, nodes, by_source, 5)
    order = np.zeros(c["sequences"], np.int64)
    offs = np.zeros(nodes + 1, np.int64)
    oracle.ref().ref_shard_corpus(c["vocab"], c["seq"], c["sources"], c["sequences"], c["seed"],
                                  nodes, 1 if by_source else 0, 5, order, offs)
    for i in range(nodes):
        assert np.array_equal(shards[i], order[offs[i]:offs[i + 1]])
    # the provider's batches over shard 0 across several epochs (wrap-around reshuffles)
    B, H = 8, 12
    stream = spes.BatchStream(shards[0], B, 9)
    ours = np.stack([tok[stream.next()] for _ in range(H)])
    ref = np.zeros((H, B, c["seq"] + 1), np.int32)
    oracle.ref().ref_batches(c["vocab"], c["seq"], c["sources"], c["sequences"], c["seed"],
                             np.ascontiguousarray(shards[0]), shards[0].size, B, 9, H, ref)
    assert np.array_equal(ours, ref)


def test_stream_errors():
    with pytest.raises(spes.SpesError) as e:
        spes.BatchStream(np.zeros(0, np.int64), 4, 1)
    assert e.value.kind == "invalid_argument"
    with pytest.raises(spes.SpesError):
        spes.gen_corpus(4, 8, 8, 2, 1)  # V < C


@pytest.mark.gpu
def test_device_corpus_round_equals_host_tokens():
    cfg = model_cfg(vocab=256, hidden=128, intermediate=256, layers=2, experts_total=8,
                    experts_active=2)
    c = CORPUS
    tok, sid = spes.gen_corpus(c["vocab"], c["seq"], c["sources"], c["sequences"], c["seed"])
    stream = spes.BatchStream(np.arange(c["sequences"]), 4, 3)
    rows = np.stack([stream.next() for _ in range(3)])
    params = oracle.random_params(cfg, 61)
    a = spes.Node(cfg, 0, 1, 0)
    b = spes.Node(cfg, 0, 1, 0)
    try:
        for n in (a, b):
            n.set_ownership([[0, 1, 2, 3]])
            n.load_params(params)
        a.corpus_load(tok)
        la = a.local_round_rows(rows, adamw_cfg())
        lb = b.local_round(tok[rows], adamw_cfg())
        assert np.array_equal(la, lb)
        assert np.array_equal(a.read_params().view(np.uint32), b.read_params().view(np.uint32))
        # against the reference itself: its own provider's batches (make_batch_provider over
        # its gen_corpus, via oracle/_ref) trained by the CPU oracle's local_round
        if oracle.ref_available():
            ref_b = np.zeros((3, 4, c["seq"] + 1), np.int32)
            oracle.ref().ref_batches(c["vocab"], c["seq"], c["sources"], c["sequences"],
                                     c["seed"], np.arange(c["sequences"], dtype=np.int64),
                                     c["sequences"], 4, 3, 3, ref_b)
            assert np.array_equal(ref_b, tok[rows])  # the device gathered the same batches
            _, l_ref = oracle.local_round(cfg, params, ref_b, [0, 1, 2, 3], adamw_cfg())
            assert np.allclose(la[:, 0], l_ref[:, 0], rtol=5e-3)
        with pytest.raises(spes.SpesError) as e:
            a.local_step_rows(np.array([c["sequences"]]))
        assert e.value.kind == "out_of_range"
    finally:
        a.close()
        b.close()


@pytest.mark.gpu
@pytest.mark.parametrize("vocab,seq,sources,sequences,skew", [
    (256, 64, 4, 96, 0.0),     # the CORPUS shape above
    (200, 33, 3, 50, 1.5),     # vocabulary below the model's, skewed bands, ragged sizes
    (256, 1023, 1, 300, 0.0),  # one source, 307k draws (about a thousand engine refills)
])
def test_device_corpus_generation_bitexact(vocab, seq, sources, sequences, skew):
    """spes_corpus_generate (corpus_dev.cu): the engine replayed and the chains sampled on
    the device equal the host transcription and the reference's own gen_corpus."""
    cfg = model_cfg(vocab=256, hidden=128, intermediate=256, layers=2, experts_total=8,
                    experts_active=2)
    node = spes.Node(cfg, 0, 1, 0)
    try:
        tok, sid = node.corpus_generate(vocab, seq, sources, sequences, 23, skew)
        ht, hs = spes.gen_corpus(vocab, seq, sources, sequences, 23, skew)
        assert np.array_equal(tok, ht) and np.array_equal(sid, hs)
        if oracle.ref_available():
            rt = np.zeros_like(tok)
            rs = np.zeros_like(sid)
            assert oracle.ref().ref_gen_corpus(vocab, seq, sources, sequences, 23, skew, rt,
                                               rs) == 0
            assert np.array_equal(tok, rt)
        # the generated corpus is the node's HBM corpus: steps over its rows run
        node.set_ownership([[0, 1, 2, 3]])
        node.load_params(oracle.random_params(cfg, 5))
        la = node.local_round_rows(np.array([[0, sequences - 1]]), adamw_cfg())
        assert np.isfinite(la).all()
        with pytest.raises(spes.SpesError) as e:
            node.corpus_generate(cfg.vocab + 1, 8, 1, 2, 1)
        assert e.value.kind == "invalid_argument"
    finally:
        node.close()
