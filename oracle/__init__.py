"""Python bindings of the CPU oracle. TEST INFRASTRUCTURE ONLY.

Two libraries, both checkers, never part of the product path:
  * liboracle.so        -- the C restatement (spes_oracle.c), always available;
  * _ref/libspes_ref.so -- the unmodified reference compiled from its own sources
                           (built here by oracle/Makefile; the prebuilt file travels
                           to the GPU box, the reference tree does not).
Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference arm
import this module.
"""
import ctypes as C
import os

import numpy as np

from paper_2602_11543_b200.abi import AdamWCfg, MergeEvent, MergeSched, ModelCfg

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libspes_ref.so")

_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
_cfgp = C.POINTER(ModelCfg)


def build():
    import subprocess
    subprocess.check_call(["make", "-s", "-C", HERE], stdout=subprocess.DEVNULL)


def _nullable(ptr_type):
    """ndpointer that also accepts None."""

    class _P(ptr_type):
        @classmethod
        def from_param(cls, obj):
            if obj is None:
                return None
            return ptr_type.from_param(obj)

    return _P


_f32n, _i32n, _f64n = _nullable(_f32p), _nullable(_i32p), _nullable(_f64p)


class OracleTrace(C.Structure):
    _fields_ = [("normed", C.c_void_p), ("logits", C.c_void_p), ("probs", C.c_void_p),
                ("topk_idx", C.c_void_p), ("topk_w", C.c_void_p), ("counts", C.c_void_p),
                ("perm", C.c_void_p), ("h", C.c_void_p), ("head_logits", C.c_void_p),
                ("grad_h", C.c_void_p)]


_lib = None
_ref = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(ORACLE_SO):
            build()
        L = C.CDLL(ORACLE_SO)
        L.oracle_param_count.restype = C.c_int64
        L.oracle_param_count.argtypes = [_cfgp]
        for n in ("oracle_off_norm", "oracle_off_router"):
            getattr(L, n).restype = C.c_int64
            getattr(L, n).argtypes = [_cfgp, C.c_int]
        L.oracle_off_expert.restype = C.c_int64
        L.oracle_off_expert.argtypes = [_cfgp, C.c_int, C.c_int]
        L.oracle_off_head.restype = C.c_int64
        L.oracle_off_head.argtypes = [_cfgp]
        L.oracle_router_forward.argtypes = [_cfgp, _f32p, _f32p, _f32p, C.c_int64, _f32p, _f32p,
                                            _f32p, _i32p, _f32p, _i32p, _i32p]
        L.oracle_forward_backward.restype = C.c_int
        L.oracle_forward_backward.argtypes = [_cfgp, _f32p, _i32p, C.c_int64, C.c_int64, _u8p,
                                              _f32p, _f64p, C.POINTER(OracleTrace)]
        L.oracle_adamw_step.argtypes = [_cfgp, _f32p, _f32p, _f32p, _f32p, _u8p,
                                        C.POINTER(AdamWCfg), C.c_int64]
        L.oracle_adamw_array.argtypes = [_f32p, _f32p, _f32p, _f32p, C.c_int64,
                                         C.POINTER(AdamWCfg), C.c_int64]
        L.oracle_local_round.restype = C.c_int
        L.oracle_local_round.argtypes = [_cfgp, _f32p, _i32p, C.c_int64, C.c_int64, C.c_int32,
                                         _f64n, C.POINTER(AdamWCfg), _u8p, _f64p]
        L.oracle_aggregate.argtypes = [_cfgp, C.c_int32, _f32p, _i32p, _i32p, _f32p, _f32p]
        L.oracle_outer_step.argtypes = [C.c_int32, C.c_double, C.c_double, _f32p, _f32p,
                                        C.c_int32, C.c_int64, _f64p]
        L.oracle_similarity.argtypes = [_cfgp, _f32p, C.c_int32, C.c_int32, _f64p]
        L.oracle_select_peers.restype = C.c_int32
        L.oracle_select_peers.argtypes = [_f64p, C.c_int32, C.c_int32, C.c_int32, _i32p]
        L.oracle_merge_model.restype = C.c_int32
        L.oracle_merge_model.argtypes = [_cfgp, _f32p, C.POINTER(MergeSched), C.c_int32,
                                         C.c_void_p, _i32n]
        L.oracle_lr_at.restype = C.c_double
        L.oracle_lr_at.argtypes = [C.c_double, C.c_double, C.c_int64, C.c_int64, C.c_int64]
        L.oracle_param_partition.argtypes = [C.c_int32, C.c_int32, _i32p, _i32p]
        L.oracle_expf_array.argtypes = [_f32p, _f32p, C.c_int64]
        L.oracle_expf_mismatches.restype = C.c_int64
        L.oracle_expf_mismatches.argtypes = [_f32p, _f32p, C.c_int64]
        L.oracle_expf_range_mismatches.restype = C.c_int64
        L.oracle_expf_range_mismatches.argtypes = [C.c_uint32, C.c_uint32, _f32p]
        _lib = L
    return _lib


def ref_available():
    return os.path.exists(REF_SO)


def ref():
    """The compiled reference (oracle/_ref). Raises if it was never built."""
    global _ref
    if _ref is None:
        if not os.path.exists(REF_SO):
            build()
        R = C.CDLL(REF_SO)
        R.ref_param_count.restype = C.c_int64
        R.ref_param_count.argtypes = [_cfgp]
        R.ref_init_model.argtypes = [_cfgp, C.c_uint64, C.c_double, _f32p]
        R.ref_forward_backward.restype = C.c_int
        R.ref_forward_backward.argtypes = [_cfgp, _f32p, _i32p, C.c_int64, C.c_int64, _u8p, _f32p,
                                           _f64p, _f32n, _i32n, _f32n]
        R.ref_local_round.restype = C.c_int
        R.ref_local_round.argtypes = [_cfgp, _f32p, _i32p, C.c_int64, C.c_int64, C.c_int32,
                                      _f64n, C.POINTER(AdamWCfg), _u8p, _f64p]
        R.ref_local_round_timed.restype = C.c_int
        R.ref_local_round_timed.argtypes = [_cfgp, _f32p, _i32p, C.c_int64, C.c_int64, C.c_int32,
                                            _f64n, C.POINTER(AdamWCfg), _u8p, _f64p,
                                            C.POINTER(C.c_double)]
        R.ref_local_round_pair_timed.restype = C.c_int
        R.ref_local_round_pair_timed.argtypes = [_cfgp, _f32p, _i32p, C.c_int64, _i32p, C.c_int64,
                                                 C.POINTER(AdamWCfg), _u8p, _f64p]
        R.ref_aggregate_partition.restype = C.c_int
        R.ref_aggregate_partition.argtypes = [_cfgp, C.c_int32, _f32p, _f32p, _f32p]
        R.ref_similarity.argtypes = [_cfgp, _f32p, C.c_int32, C.c_int32, _f64p]
        R.ref_select_peers.restype = C.c_int32
        R.ref_select_peers.argtypes = [_f64p, C.c_int32, C.c_int32, C.c_int32, _i32p]
        R.ref_merge_model.restype = C.c_int32
        R.ref_merge_model.argtypes = [_cfgp, _f32p, C.POINTER(MergeSched), C.c_int32, C.c_void_p,
                                      _i32n]
        R.ref_adamw_first_step.restype = C.c_int
        R.ref_adamw_first_step.argtypes = [_cfgp, _f32p, _f32p, _u8p, C.POINTER(AdamWCfg)]
        R.ref_lr_at.restype = C.c_double
        R.ref_lr_at.argtypes = [C.c_double, C.c_double, C.c_int64, C.c_int64, C.c_int64]
        R.ref_param_partition.argtypes = [_cfgp, C.c_int32, _i32p, _i32p]
        _u8 = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
        _i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
        R.ref_gen_corpus.restype = C.c_int
        R.ref_gen_corpus.argtypes = [C.c_int64, C.c_int64, C.c_int32, C.c_int64, C.c_uint64,
                                     C.c_double, _i32p, _i32p]
        R.ref_shard_corpus.argtypes = [C.c_int64, C.c_int64, C.c_int32, C.c_int64, C.c_uint64,
                                       C.c_int32, C.c_int32, C.c_uint64, _i64p, _i64p]
        R.ref_batches.argtypes = [C.c_int64, C.c_int64, C.c_int32, C.c_int64, C.c_uint64, _i64p,
                                  C.c_int64, C.c_int64, C.c_uint64, C.c_int32, _i32p]
        R.ref_upcycle.restype = C.c_int
        R.ref_upcycle.argtypes = [_cfgp, _f32p, C.c_int32, C.c_double, C.c_double, C.c_uint64, _f32p]
        R.ref_outer_create.restype = C.c_void_p
        R.ref_outer_create.argtypes = [C.c_int32, C.c_double, C.c_double]
        R.ref_outer_destroy.argtypes = [C.c_void_p]
        R.ref_outer_step.restype = C.c_int
        R.ref_outer_step.argtypes = [C.c_void_p, _cfgp, _f32p, _f32p, C.c_int32]
        R.ref_encode_model.restype = C.c_int64
        R.ref_encode_model.argtypes = [_cfgp, _f32p, C.c_void_p, C.c_int64]
        R.ref_decode_model.restype = C.c_int
        R.ref_decode_model.argtypes = [_cfgp, _u8, C.c_int64, _f32p, C.c_char_p, C.c_int]
        R.ref_write_checkpoint.restype = C.c_int
        R.ref_write_checkpoint.argtypes = [_cfgp, _f32p, C.c_char_p, C.c_uint64]
        R.ref_read_checkpoint.restype = C.c_int
        R.ref_read_checkpoint.argtypes = [_cfgp, C.c_char_p, _f32p, C.POINTER(C.c_uint64),
                                          C.c_char_p, C.c_int]
        R.ref_set_parallel.argtypes = [C.c_int]
        R.ref_run_experiment.restype = C.c_int
        R.ref_run_experiment.argtypes = [_cfgp, C.c_int32, C.c_int32, C.c_int32, C.c_int64,
                                         C.c_int64, C.c_char_p, C.c_char_p, C.c_void_p, C.c_int32,
                                         C.POINTER(C.c_int32), C.POINTER(C.c_int64)]
        R.ref_run_inproc_ledger.restype = C.c_int
        R.ref_run_inproc_ledger.argtypes = [_cfgp, C.c_int32, C.c_int32, C.c_int32, C.c_int64,
                                            C.c_int64, C.c_int32, C.c_uint64, _i32p, _i32p,
                                            np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS"),
                                            np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS"),
                                            C.c_int32, C.POINTER(C.c_int32),
                                            np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")]
        _ref = R
    return _ref


# ---------------- numpy-level helpers ----------------

def param_count(cfg):
    return lib().oracle_param_count(C.byref(cfg))


def expert_offset(cfg, l, j):
    return lib().oracle_off_expert(C.byref(cfg), l, j)


def random_params(cfg, seed, std=0.02):
    """Seeded synthetic parameters (norm gains 1, like init_model, model.hpp:160-162)."""
    rng = np.random.default_rng(seed)
    p = (rng.standard_normal(param_count(cfg)) * std).astype(np.float32)
    for l in range(cfg.layers):
        o = lib().oracle_off_norm(C.byref(cfg), l)
        p[o:o + cfg.hidden] = 1.0
    return p


def random_tokens(cfg, B, S, seed, H=1):
    rng = np.random.default_rng(seed)
    return rng.integers(0, cfg.vocab, size=(H, B, S + 1), dtype=np.int32)


def trainable_mask(cfg, owned):
    m = np.zeros(cfg.experts_total, np.uint8)
    m[list(owned)] = 1
    return m


def router_forward(cfg, h, gain, router):
    T = h.shape[0]
    d, M, k = cfg.hidden, cfg.experts_total, cfg.experts_active
    out = dict(normed=np.zeros((T, d), np.float32), logits=np.zeros((T, M), np.float32),
               probs=np.zeros((T, M), np.float32), idx=np.zeros((T, k), np.int32),
               w=np.zeros((T, k), np.float32), counts=np.zeros(M, np.int32),
               perm=np.zeros(T * k, np.int32))
    lib().oracle_router_forward(C.byref(cfg), np.ascontiguousarray(h, np.float32),
                                np.ascontiguousarray(gain, np.float32),
                                np.ascontiguousarray(router, np.float32), T, out["normed"],
                                out["logits"], out["probs"], out["idx"], out["w"], out["counts"],
                                out["perm"])
    return out


def forward_backward(cfg, params, tokens, owned, trace=False):
    B, S1 = tokens.shape[-2], tokens.shape[-1]
    S = S1 - 1
    T = B * S
    L, d, M, k, V = cfg.layers, cfg.hidden, cfg.experts_total, cfg.experts_active, cfg.vocab
    grads = np.zeros(param_count(cfg), np.float32)
    losses = np.zeros(5, np.float64)
    tr = None
    arrays = {}
    if trace:
        arrays = dict(normed=np.zeros((L, T, d), np.float32), logits=np.zeros((L, T, M), np.float32),
                      probs=np.zeros((L, T, M), np.float32), topk_idx=np.zeros((L, T, k), np.int32),
                      topk_w=np.zeros((L, T, k), np.float32), counts=np.zeros((L, M), np.int32),
                      perm=np.zeros((L, T * k), np.int32), h=np.zeros((L + 1, T, d), np.float32),
                      head_logits=np.zeros((T, V), np.float32),
                      grad_h=np.zeros((L + 1, T, d), np.float32))
        tr = OracleTrace(**{k_: a.ctypes.data for k_, a in arrays.items()})
    rc = lib().oracle_forward_backward(C.byref(cfg), np.ascontiguousarray(params, np.float32),
                                       np.ascontiguousarray(tokens.reshape(B, S1), np.int32), B, S,
                                       trainable_mask(cfg, owned), grads, losses,
                                       C.byref(tr) if tr is not None else None)
    if rc:
        raise IndexError("batch: token id out of vocabulary")
    return losses, grads, arrays


def local_round(cfg, params, tokens, owned, opt, lr=None):
    """tokens: H x B x (S+1). Returns (new params, losses[H,5])."""
    H, B, S1 = tokens.shape
    p = np.array(params, np.float32, copy=True)
    losses = np.zeros((H, 5), np.float64)
    lr_arr = None if lr is None else np.ascontiguousarray(lr, np.float64)
    rc = lib().oracle_local_round(C.byref(cfg), p, np.ascontiguousarray(tokens, np.int32), B,
                                  S1 - 1, H, lr_arr, C.byref(opt), trainable_mask(cfg, owned),
                                  losses)
    if rc == 2:
        raise IndexError("batch: token id out of vocabulary")
    if rc >= 3:
        raise RuntimeError(f"local_round: non-finite loss at step {rc - 3}")
    return p, losses


def ownership_csr(owned_lists):
    offs = np.zeros(len(owned_lists) + 1, np.int32)
    flat = []
    for n, e in enumerate(owned_lists):
        flat.extend(sorted(e))
        offs[n + 1] = len(flat)
    return offs, np.array(flat if flat else [0], np.int32)


def aggregate(cfg, node_params, owned_lists, global_in):
    N = len(owned_lists)
    offs, flat = ownership_csr(owned_lists)
    out = np.zeros_like(global_in)
    lib().oracle_aggregate(C.byref(cfg), N, np.ascontiguousarray(node_params, np.float32), offs,
                           flat, np.ascontiguousarray(global_in, np.float32), out)
    return out


def outer_step(kind, lr, momentum, theta, locals_, buf):
    """OuterOptimizer::step (trainer.hpp:228-266) restated: theta (in place), locals N x n,
    buf (n doubles, Nesterov state, in place)."""
    N = locals_.shape[0]
    lib().oracle_outer_step(kind, lr, momentum, theta, np.ascontiguousarray(locals_, np.float32),
                            N, theta.size, buf)


def similarity(cfg, params, layer, source=0):
    M = cfg.experts_total
    sim = np.zeros((M, M), np.float64)
    lib().oracle_similarity(C.byref(cfg), np.ascontiguousarray(params, np.float32), layer, source,
                            sim)
    return sim


def merge_model(cfg, params, sched, round0):
    p = np.array(params, np.float32, copy=True)
    L, M = cfg.layers, cfg.experts_total
    K = max(1, min(sched.peers, M - 1))
    events = (MergeEvent * L)()
    peers = np.zeros((L, M, K), np.int32)
    n = lib().oracle_merge_model(C.byref(cfg), p, C.byref(sched), round0, C.cast(events, C.c_void_p),
                                 peers)
    return p, [(e.layer, e.peers_k, e.alpha, e.displacement_sq) for e in events[:n]], peers[:n]


def param_partition(M, N):
    offs = np.zeros(N + 1, np.int32)
    flat = np.zeros(M, np.int32)
    lib().oracle_param_partition(M, N, offs, flat)
    return [list(flat[offs[i]:offs[i + 1]]) for i in range(N)]


def expf(x):
    x = np.ascontiguousarray(x, np.float32)
    y = np.zeros_like(x)
    lib().oracle_expf_array(x, y, x.size)
    return y
