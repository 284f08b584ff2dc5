"""B200-native SPES hot path: Python host mirror over the C ABI (include/spes_b200.h).

The product is libspes_b200.so (C++ host orchestration + sm_100a CUDA kernels +
NCCL); this module only binds it with ctypes and mirrors the reference's
operator interface (proj/include/spes/trainer.hpp, merging.hpp, protocol.cpp):

    Node(cfg, node, n_nodes, device, nccl_id)      one SPES node == one GPU
      .set_ownership(owned_lists)                   ASSIGN / TrainMask (any replication)
      .load_params / read_params                    enumerate_blocks layout, fp32
      .local_round(tokens[H,B,S+1], opt, lr, carry) local_round (trainer.hpp:143-222)
      .local_step(...)                              one build_loss + backward + AdamW step
      .sync()                                       Server::aggregate (protocol.cpp:197-251)
      .merge_model(sched, round0)                   merge_model (merging.hpp:138-150)

There is no CPU fallback: if the shared library is missing, loading fails loudly.
"""
import ctypes as C
import os

import numpy as np

from .abi import (CONFIGS, AdamWCfg, Losses, MergeEvent, MergeSched, ModelCfg, SyncStats,
                  adamw_cfg, merge_sched, model_cfg)

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libspes_b200.so")

SPES_OK = 0
_STATUS = {1: "invalid_argument", 2: "out_of_range", 3: "logic_error", 4: "runtime_error",
           5: "cuda_error", 6: "nccl_error", 7: "protocol_error"}


class SpesError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"[{_STATUS.get(status, status)}] {msg}")
        self.status = status
        self.kind = _STATUS.get(status, "error")


_lib = None


def build():
    import subprocess
    subprocess.check_call(["make", "-s", "-C", os.path.join(HERE, "csrc"), "-j4"])


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} missing: run __graft_entry__.build() (no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        vp, i32, i64, f32p = C.c_void_p, C.c_int32, C.c_int64, C.POINTER(C.c_float)
        cfgp = C.POINTER(ModelCfg)
        L.spes_last_error.restype = C.c_char_p
        L.spes_validate_cfg.argtypes = [cfgp]
        L.spes_param_count.restype = i64
        L.spes_param_count.argtypes = [cfgp]
        L.spes_block_offsets.argtypes = [cfgp, C.POINTER(i64), C.POINTER(i32)]
        L.spes_param_partition.argtypes = [cfgp, i32, C.POINTER(i32), C.POINTER(i32)]
        L.spes_sync_plan.argtypes = [i32, i32, C.POINTER(i32), C.POINTER(i32), C.POINTER(i32),
                                     C.POINTER(i32)]
        L.spes_lr_at.restype = C.c_double
        L.spes_lr_at.argtypes = [C.c_double, C.c_double, i64, i64, i64]
        L.spes_merge_at.restype = i32
        L.spes_merge_at.argtypes = [C.POINTER(MergeSched), i32]
        L.spes_alpha_at.argtypes = [C.POINTER(MergeSched), i32, C.POINTER(C.c_double)]
        L.spes_create.argtypes = [cfgp, i32, i32, i32, vp, C.POINTER(vp)]
        L.spes_destroy.argtypes = [vp]
        L.spes_destroy.restype = None
        L.spes_nccl_unique_id.argtypes = [vp]
        L.spes_set_ownership.argtypes = [vp, C.POINTER(i32), C.POINTER(i32)]
        L.spes_load_params.argtypes = [vp, f32p, i64]
        L.spes_read_params.argtypes = [vp, f32p, i64]
        L.spes_load_params_device.argtypes = [vp, vp, i64]
        L.spes_read_grads.argtypes = [vp, f32p, i64]
        L.spes_set_fused_optimizer.argtypes = [vp, C.c_int32]
        L.spes_set_stream_overlap.argtypes = [vp, C.c_int32]
        L.spes_set_inner_optimizer.argtypes = [vp, C.c_int32]
        L.spes_outer_begin.argtypes = [vp]
        i64p = C.POINTER(C.c_int64)
        L.spes_gen_corpus.argtypes = [i64, i64, C.c_int32, i64, C.c_uint64, C.c_double,
                                      C.POINTER(C.c_int32), C.POINTER(C.c_int32)]
        L.spes_shard_corpus.argtypes = [C.POINTER(C.c_int32), i64, C.c_int32, C.c_int32,
                                        C.c_uint64, i64p, i64p]
        L.spes_batch_stream_create.argtypes = [i64p, i64, i64, C.c_uint64, C.POINTER(vp)]
        L.spes_batch_stream_next.argtypes = [vp, i64p]
        L.spes_batch_stream_destroy.argtypes = [vp]
        L.spes_batch_stream_destroy.restype = None
        L.spes_corpus_load.argtypes = [vp, C.POINTER(C.c_int32), i64, i64]
        L.spes_corpus_generate.argtypes = [vp, i64, i64, C.c_int32, i64, C.c_uint64, C.c_double,
                                           C.POINTER(C.c_int32), C.POINTER(C.c_int32)]
        L.spes_local_step_rows.argtypes = [vp, i64p, i64, C.POINTER(AdamWCfg), C.POINTER(Losses)]
        L.spes_local_round_rows.argtypes = [vp, i64p, i64, C.c_int32, C.POINTER(C.c_double),
                                            C.POINTER(AdamWCfg), C.c_int32, C.POINTER(Losses)]
        L.spes_upcycle_from_dense.argtypes = [C.POINTER(ModelCfg), f32p, C.c_int32, C.c_double,
                                              C.c_double, C.c_uint64, C.POINTER(ModelCfg), f32p]
        L.spes_outer_sync.argtypes = [vp, C.c_int32, C.c_double, C.c_double, C.POINTER(SyncStats)]
        L.spes_metrics_csv.argtypes = [C.c_void_p, C.c_int32, C.c_int64, C.c_void_p, C.c_char_p,
                                       C.c_int64, C.POINTER(C.c_int64)]
        L.spes_comm_ledger.argtypes = [C.POINTER(ModelCfg), C.c_int32, C.c_void_p, C.c_void_p,
                                       C.c_int32, C.c_int32, C.c_void_p, C.c_int32,
                                       C.POINTER(C.c_int32), C.POINTER(C.c_uint64)]
        u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
        L.spes_model_payload_bytes.restype = i64
        L.spes_model_payload_bytes.argtypes = [C.POINTER(ModelCfg)]
        L.spes_encode_model_host.argtypes = [C.POINTER(ModelCfg), f32p, u8p, i64]
        L.spes_decode_model_host.argtypes = [C.POINTER(ModelCfg), u8p, i64, f32p]
        L.spes_encode_model.argtypes = [vp, u8p, i64]
        L.spes_decode_model.argtypes = [vp, u8p, i64]
        L.spes_write_checkpoint.argtypes = [vp, C.c_char_p, C.c_uint64]
        L.spes_read_checkpoint.argtypes = [vp, C.c_char_p, C.POINTER(C.c_uint64)]
        L.spes_round_begin.argtypes = [vp, i32]
        L.spes_local_step.argtypes = [vp, C.POINTER(i32), i64, i64, C.POINTER(AdamWCfg),
                                      C.POINTER(Losses)]
        L.spes_local_step_device.argtypes = [vp, vp, i64, i64, C.POINTER(AdamWCfg),
                                             C.POINTER(Losses)]
        L.spes_local_round.argtypes = [vp, C.POINTER(i32), i64, i64, i32, C.POINTER(C.c_double),
                                       C.POINTER(AdamWCfg), i32, C.POINTER(Losses)]
        L.spes_sync.argtypes = [vp, C.POINTER(SyncStats)]
        L.spes_merge.argtypes = [vp, C.POINTER(MergeSched), i32, C.POINTER(MergeEvent),
                                 C.POINTER(i32), C.POINTER(i32)]
        L.spes_similarity.argtypes = [vp, i32, i32, C.POINTER(C.c_double)]
        L.spes_counts.argtypes = [vp, C.POINTER(i64), C.POINTER(i64), C.POINTER(i64)]
        L.spes_debug_read.argtypes = [vp, C.c_char_p, i32, vp, i64]
        L.spes_stream.restype = vp
        L.spes_stream.argtypes = [vp]
        L.spes_profile.argtypes = [vp, i32]
        L.spes_profile_reset.argtypes = [vp]
        L.spes_profile_count.restype = i32
        L.spes_profile_count.argtypes = [vp]
        L.spes_profile_get.argtypes = [vp, i32, C.c_char_p, C.POINTER(C.c_double),
                                       C.POINTER(i64)]
        L.spes_kernel_launches.restype = i64
        L.spes_kernel_launches.argtypes = [vp]
        L.spes_kernel_router.argtypes = [cfgp, f32p, f32p, f32p, i64, f32p, f32p, f32p,
                                         C.POINTER(i32), f32p, C.POINTER(i32), C.POINTER(i32), i32]
        L.spes_kernel_adamw.argtypes = [f32p, f32p, f32p, f32p, i64, C.POINTER(AdamWCfg), i64, i32]
        L.spes_kernel_owner_mean.argtypes = [f32p, i32, i64, f32p, i32]
        L.spes_kernel_expf.argtypes = [f32p, f32p, i64, i32]
        L.spes_host_expf_port.argtypes = [f32p, f32p, i64, i32]
        L.spes_host_expf_port.restype = None
        L.spes_host_expf_variant.restype = i32
        _lib = L
    return _lib


def _check(status):
    if status != SPES_OK:
        raise SpesError(status, lib().spes_last_error().decode())


def _p(a, ctype):
    return a.ctypes.data_as(C.POINTER(ctype))


def f32(a):
    return _p(a, C.c_float)


def i32(a):
    return _p(a, C.c_int32)


def param_count(cfg):
    return lib().spes_param_count(C.byref(cfg))


def block_offsets(cfg):
    n = C.c_int32()
    _check(lib().spes_block_offsets(C.byref(cfg), None, C.byref(n)))
    out = np.zeros(n.value, np.int64)
    _check(lib().spes_block_offsets(C.byref(cfg), _p(out, C.c_int64), None))
    return out


def param_partition(cfg, n):
    offs = np.zeros(n + 1, np.int32)
    ex = np.zeros(max(cfg.experts_total, 1), np.int32)
    _check(lib().spes_param_partition(C.byref(cfg), n, i32(offs), i32(ex)))
    return [list(ex[offs[i]:offs[i + 1]]) for i in range(n)]


def replicated_ownership(M, N, r=2):
    """node n owns {(s*n + i) mod M, i < E} with s = M/N, E = min(M, r*M/N)."""
    s = M // N
    E = min(M, r * M // N)
    return [sorted({(s * n + i) % M for i in range(E)}) for n in range(N)]


def sync_plan(M, owned_lists):
    """(primary owner per expert, balanced?) exactly as spes_sync uses them."""
    N = len(owned_lists)
    offs = np.zeros(N + 1, np.int32)
    flat = []
    for n, e in enumerate(owned_lists):
        flat.extend(sorted(int(x) for x in e))
        offs[n + 1] = len(flat)
    arr = np.array(flat if flat else [0], np.int32)
    prim = np.zeros(M, np.int32)
    bal = C.c_int32()
    _check(lib().spes_sync_plan(M, N, i32(offs), i32(arr), i32(prim), C.byref(bal)))
    return prim, bool(bal.value)


def nccl_unique_id():
    buf = (C.c_char * 128)()
    _check(lib().spes_nccl_unique_id(buf))
    return bytes(buf)


def lr_at(peak, min_frac, warmup, total, step):
    return lib().spes_lr_at(peak, min_frac, warmup, total, step)


# ---- wire / checkpoint format (proj/src/wire.cpp), byte-identical to the reference ----

def model_payload_bytes(cfg):
    return lib().spes_model_payload_bytes(C.byref(cfg))


def encode_model(cfg, params):
    """encode_blocks(model_to_blocks(params)): the GLOBAL_MODEL payload as bytes (uint8)."""
    out = np.zeros(model_payload_bytes(cfg), np.uint8)
    params = np.ascontiguousarray(params, np.float32)
    _check(lib().spes_encode_model_host(C.byref(cfg), f32(params), out, out.size))
    return out


def decode_model(cfg, payload):
    """blocks_into_model(decode_blocks(payload)) -> flat fp32 parameters."""
    payload = np.ascontiguousarray(np.frombuffer(bytes(payload), np.uint8) if not
                                   isinstance(payload, np.ndarray) else payload, np.uint8)
    out = np.zeros(param_count(cfg), np.float32)
    _check(lib().spes_decode_model_host(C.byref(cfg), payload, payload.size, f32(out)))
    return out


# ---- CommLedger (protocol.hpp:29-52): the reference protocol's byte accounting ----

_LEDGER_DT = np.dtype([("node", np.int32), ("round", np.int32), ("up", np.uint64),
                       ("down", np.uint64)])


def comm_ledger(cfg, n_nodes, rounds, diloco=False, ownership=None):
    """CommLedger of a SPES run under the reference's protocol (spes_comm_ledger).

    Returns (entries, totals): entries a structured array (node, round, up, down) in
    (node, round) order, node -1 holding the HELLOs; totals a dict with total_up,
    total_down, pushes and broadcasts. ownership: list of per-node expert lists, or None
    for param_partition."""
    offs = exps = None
    if ownership is not None:
        offs = np.zeros(len(ownership) + 1, np.int32)
        for i, o in enumerate(ownership):
            offs[i + 1] = offs[i] + len(o)
        exps = np.ascontiguousarray(np.concatenate([np.asarray(o, np.int32) for o in ownership]),
                                    np.int32)
    n = C.c_int32(0)
    tot = (C.c_uint64 * 4)()
    cap = n_nodes * (rounds + 2) + 1
    ent = np.zeros(cap, _LEDGER_DT)
    _check(lib().spes_comm_ledger(C.byref(cfg), n_nodes,
                                  None if offs is None else offs.ctypes.data_as(C.c_void_p),
                                  None if exps is None else exps.ctypes.data_as(C.c_void_p),
                                  rounds, 1 if diloco else 0, ent.ctypes.data_as(C.c_void_p), cap,
                                  C.byref(n), tot))
    return ent[:n.value], dict(total_up=tot[0], total_down=tot[1], pushes=tot[2],
                               broadcasts=tot[3])


class RoundMetrics(C.Structure):
    """spes_round_metrics == RoundMetrics (protocol.hpp:132-137)."""
    _fields_ = [("round", C.c_int32), ("mean_total", C.c_double), ("mean_ce", C.c_double),
                ("mean_lb", C.c_double), ("mean_moe_z", C.c_double), ("mean_z", C.c_double),
                ("merge_displacement_sq", C.c_double), ("bytes_up", C.c_uint64),
                ("bytes_down", C.c_uint64)]


def metrics_csv(rows, tokens_per_round, wall_ms=None):
    """metrics.csv text of an experiment (experiment.cpp:376-385) from RoundMetrics rows."""
    arr = (RoundMetrics * max(1, len(rows)))(*rows)
    wall = None
    if wall_ms is not None:
        wall = np.ascontiguousarray(wall_ms, np.float64)
    n = C.c_int64(0)
    L = lib()
    wp = None if wall is None else wall.ctypes.data_as(C.c_void_p)
    _check(L.spes_metrics_csv(arr, len(rows), tokens_per_round, wp, None, 0, C.byref(n)))
    buf = C.create_string_buffer(n.value + 1)
    _check(L.spes_metrics_csv(arr, len(rows), tokens_per_round, wp, buf, n.value, C.byref(n)))
    return buf.raw[:n.value].decode()


def round_bytes(entries, rnd):
    """RoundMetrics.bytes_up / bytes_down of round rnd (assemble_run_result,
    protocol.cpp:357-362): the ledger entries of that round summed over nodes."""
    sel = entries[entries["round"] == rnd]
    return int(sel["up"].sum()), int(sel["down"].sum())


# ---- synthetic corpus / batch streams (proj/src/corpus.cpp), bit-identical ----

def _i64(a):
    return _p(a, C.c_int64)


def gen_corpus(vocab, seq, sources, sequences, seed, skew=0.0):
    """gen_corpus (corpus.cpp:49-79) -> (tokens [sequences, seq+1] int32, source_id int32)."""
    tok = np.zeros((sequences, seq + 1), np.int32)
    sid = np.zeros(sequences, np.int32)
    _check(lib().spes_gen_corpus(vocab, seq, sources, sequences, seed, skew, i32(tok), i32(sid)))
    return tok, sid


def shard_corpus(source_id, nodes, by_source, seed):
    """shard_corpus (corpus.cpp:107-128) -> list of per-node row index arrays."""
    source_id = np.ascontiguousarray(source_id, np.int32)
    order = np.zeros(source_id.size, np.int64)
    offs = np.zeros(nodes + 1, np.int64)
    _check(lib().spes_shard_corpus(i32(source_id), source_id.size, nodes, 1 if by_source else 0,
                                   seed, _i64(order), _i64(offs)))
    return [order[offs[i]:offs[i + 1]] for i in range(nodes)]


class BatchStream:
    """make_batch_provider's row stream (corpus.cpp:130-149): shuffled epochs, wrap-around."""

    def __init__(self, shard, batch, seed):
        shard = np.ascontiguousarray(shard, np.int64)
        self.batch = batch
        self._s = C.c_void_p()
        _check(lib().spes_batch_stream_create(_i64(shard), shard.size, batch, seed,
                                              C.byref(self._s)))

    def next(self):
        rows = np.zeros(self.batch, np.int64)
        _check(lib().spes_batch_stream_next(self._s, _i64(rows)))
        return rows

    def __del__(self):
        if getattr(self, "_s", None):
            lib().spes_batch_stream_destroy(self._s)
            self._s = None


def upcycle_from_dense(dense_cfg, dense_params, m, noise_frac=0.5, noise_std=0.02, seed=1):
    """upcycle_from_dense (model.hpp:415-460) -> (cfg with m experts and renorm, params)."""
    out_cfg = ModelCfg()
    probe = ModelCfg.from_buffer_copy(dense_cfg)
    probe.experts_total = m
    out = np.zeros(param_count(probe), np.float32)
    dense_params = np.ascontiguousarray(dense_params, np.float32)
    _check(lib().spes_upcycle_from_dense(C.byref(dense_cfg), f32(dense_params), m, noise_frac,
                                         noise_std, seed, C.byref(out_cfg), f32(out)))
    return out_cfg, out


class Node:
    """One SPES node on one GPU."""

    def __init__(self, cfg, node=0, n_nodes=1, device=0, nccl_id=None):
        self.cfg = cfg
        self.node, self.n_nodes, self.device = node, n_nodes, device
        self._ctx = C.c_void_p()
        idbuf = None
        if nccl_id is not None:
            idbuf = C.create_string_buffer(bytes(nccl_id), 128)
        _check(lib().spes_create(C.byref(cfg), node, n_nodes, device,
                                 C.cast(idbuf, C.c_void_p) if idbuf is not None else None,
                                 C.byref(self._ctx)))
        self.P = param_count(cfg)

    def close(self):
        if self._ctx:
            lib().spes_destroy(self._ctx)
            self._ctx = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def ctx(self):
        return self._ctx

    def set_ownership(self, owned_lists):
        offs = np.zeros(len(owned_lists) + 1, np.int32)
        flat = []
        for n, e in enumerate(owned_lists):
            flat.extend(sorted(int(x) for x in e))
            offs[n + 1] = len(flat)
        arr = np.array(flat if flat else [0], np.int32)
        _check(lib().spes_set_ownership(self._ctx, i32(offs), i32(arr)))

    def load_params(self, p):
        p = np.ascontiguousarray(p, np.float32)
        _check(lib().spes_load_params(self._ctx, f32(p), p.size))

    def load_params_device(self, dev_ptr, n):
        """Parameters from a device buffer (n fp32 scalars in enumerate_blocks order)."""
        _check(lib().spes_load_params_device(self._ctx, C.c_void_p(dev_ptr), n))

    def read_params(self):
        out = np.zeros(self.P, np.float32)
        _check(lib().spes_read_params(self._ctx, f32(out), out.size))
        return out

    def set_fused_optimizer(self, on):
        """Owned experts' AdamW inside the dW GEMM epilogue, or (default) as a separate pass
        with materialized gradients (needed by read_grads); identical bits either way."""
        _check(lib().spes_set_fused_optimizer(self._ctx, 1 if on else 0))

    def set_inner_optimizer(self, kind):
        """LocalRoundConfig::inner (trainer.hpp:116-121): "adamw" (default) or "sgd"
        (theta -= float(lr) * g on the trainable blocks, trainer.hpp:197-204)."""
        k = {"adamw": 0, "sgd": 1}.get(kind, kind)
        _check(lib().spes_set_inner_optimizer(self._ctx, k))

    def set_stream_overlap(self, on):
        """Second low-priority stream for the step's off-critical-path work (default on);
        identical bits either way."""
        _check(lib().spes_set_stream_overlap(self._ctx, 1 if on else 0))

    def corpus_load(self, tokens):
        """Upload a corpus [sequences, S+1] to HBM once (token ids validated here)."""
        tokens = np.ascontiguousarray(tokens, np.int32)
        _check(lib().spes_corpus_load(self._ctx, i32(tokens), tokens.shape[0], tokens.shape[1] - 1))

    def corpus_generate(self, vocab, seq, sources, sequences, seed, skew=0.0, fetch=True):
        """gen_corpus (corpus.cpp:49-79) generated on the device into this node's HBM corpus;
        returns (tokens [sequences, seq+1], source_id) when fetch, else None."""
        tok = np.zeros((sequences, seq + 1), np.int32) if fetch else None
        sid = np.zeros(sequences, np.int32) if fetch else None
        _check(lib().spes_corpus_generate(self._ctx, vocab, seq, sources, sequences, seed, skew,
                                          i32(tok) if fetch else None,
                                          i32(sid) if fetch else None))
        return (tok, sid) if fetch else None

    def local_step_rows(self, rows, opt=None):
        rows = np.ascontiguousarray(rows, np.int64)
        lo = Losses()
        _check(lib().spes_local_step_rows(self._ctx, _i64(rows), rows.size,
                                          C.byref(opt or adamw_cfg()), C.byref(lo)))
        return (lo.total, lo.ce, lo.lb, lo.moe_z, lo.z)

    def local_round_rows(self, rows, opt=None, lr=None, carry_state=False):
        """rows: H x B corpus row indices; returns losses [H, 5]."""
        rows = np.ascontiguousarray(rows, np.int64)
        H, B = rows.shape
        out = (Losses * H)()
        lr_p = None
        if lr is not None:
            lr_arr = (C.c_double * H)(*lr)
            lr_p = C.cast(lr_arr, C.POINTER(C.c_double))
        _check(lib().spes_local_round_rows(self._ctx, _i64(rows), B, H, lr_p,
                                           C.byref(opt or adamw_cfg()), 1 if carry_state else 0,
                                           out))
        return np.array([(o.total, o.ce, o.lb, o.moe_z, o.z) for o in out])

    def outer_begin(self):
        """DiLoCo baseline: snapshot the round-start global model (this rank's slice)."""
        _check(lib().spes_outer_begin(self._ctx))

    def outer_sync(self, kind="nesterov", lr=0.7, momentum=0.9):
        """DiLoCo outer step over the full model (collective; protocol.cpp:199-213)."""
        st = SyncStats()
        k = {"sgd": 0, "nesterov": 1}[kind] if isinstance(kind, str) else int(kind)
        _check(lib().spes_outer_sync(self._ctx, k, lr, momentum, C.byref(st)))
        return dict(bytes_in=st.expert_bytes_in, ms=st.ms)

    def encode_model(self):
        out = np.zeros(model_payload_bytes(self.cfg), np.uint8)
        _check(lib().spes_encode_model(self._ctx, out, out.size))
        return out

    def decode_model(self, payload):
        payload = np.ascontiguousarray(payload, np.uint8)
        _check(lib().spes_decode_model(self._ctx, payload, payload.size))

    def write_checkpoint(self, path, round_no):
        _check(lib().spes_write_checkpoint(self._ctx, str(path).encode(), round_no))

    def read_checkpoint(self, path):
        r = C.c_uint64()
        _check(lib().spes_read_checkpoint(self._ctx, str(path).encode(), C.byref(r)))
        return r.value

    def read_grads(self):
        out = np.zeros(self.P, np.float32)
        _check(lib().spes_read_grads(self._ctx, f32(out), out.size))
        return out

    def round_begin(self, carry_state=False):
        _check(lib().spes_round_begin(self._ctx, int(carry_state)))

    def local_step(self, tokens, opt=None, want_losses=True):
        tokens = np.ascontiguousarray(tokens, np.int32)
        B, S1 = tokens.shape[-2:]
        lo = Losses()
        _check(lib().spes_local_step(self._ctx, i32(tokens), B, S1 - 1,
                                     C.byref(opt or adamw_cfg()),
                                     C.byref(lo) if want_losses else None))
        return lo.as_tuple() if want_losses else None

    def local_step_device(self, dev_ptr, B, S, opt=None, want_losses=False):
        lo = Losses()
        _check(lib().spes_local_step_device(self._ctx, C.c_void_p(dev_ptr), B, S,
                                            C.byref(opt or adamw_cfg()),
                                            C.byref(lo) if want_losses else None))
        return lo.as_tuple() if want_losses else None

    def local_round(self, tokens, opt=None, lr=None, carry_state=False):
        """tokens: H x B x (S+1) int32; returns losses [H, 5] (total, ce, lb, moe_z, z)."""
        tokens = np.ascontiguousarray(tokens, np.int32)
        H, B, S1 = tokens.shape
        losses = (Losses * H)()
        lr_arr = None
        if lr is not None:
            lr_arr = np.ascontiguousarray(lr, np.float64)
        _check(lib().spes_local_round(self._ctx, i32(tokens), B, S1 - 1, H,
                                      _p(lr_arr, C.c_double) if lr_arr is not None else None,
                                      C.byref(opt or adamw_cfg()), int(carry_state), losses))
        return np.array([l.as_tuple() for l in losses])

    def sync(self):
        st = SyncStats()
        _check(lib().spes_sync(self._ctx, C.byref(st)))
        return dict(psi_bytes_in=st.psi_bytes_in, expert_bytes_in=st.expert_bytes_in, ms=st.ms)

    def merge_model(self, sched, round0):
        L, M = self.cfg.layers, self.cfg.experts_total
        K = max(1, min(sched.peers, M - 1))
        ev = (MergeEvent * L)()
        peers = np.zeros((L, M, K), np.int32)
        n = C.c_int32()
        _check(lib().spes_merge(self._ctx, C.byref(sched), round0, ev, i32(peers), C.byref(n)))
        return [(e.layer, e.peers_k, e.alpha, e.displacement_sq) for e in ev[:n.value]], \
            peers[:n.value]

    def similarity(self, layer, source=0):
        M = self.cfg.experts_total
        out = np.zeros((M, M), np.float64)
        _check(lib().spes_similarity(self._ctx, layer, source, _p(out, C.c_double)))
        return out

    def counts(self):
        a, b, c = C.c_int64(), C.c_int64(), C.c_int64()
        _check(lib().spes_counts(self._ctx, C.byref(a), C.byref(b), C.byref(c)))
        return dict(opt_state_scalars=a.value, grad_scalars=b.value, adam_step=c.value)

    def debug(self, name, layer=0, dtype=np.float32, shape=None, count=None):
        cfg = self.cfg
        if count is None:
            raise ValueError("count required")
        out = np.zeros(count, dtype)
        _check(lib().spes_debug_read(self._ctx, name.encode(), layer, out.ctypes.data,
                                     out.nbytes))
        return out.reshape(shape) if shape is not None else out

    def profile(self, enable=True, reset=False):
        if reset:
            _check(lib().spes_profile_reset(self._ctx))
        _check(lib().spes_profile(self._ctx, int(enable)))

    def profile_stats(self):
        """{kernel family: (total device ms, launches)} from live CUDA-event timing."""
        L = lib()
        out = {}
        n = L.spes_profile_count(self._ctx)
        for i in range(n):
            name = C.create_string_buffer(64)
            ms, cnt = C.c_double(), C.c_int64()
            _check(L.spes_profile_get(self._ctx, i, name, C.byref(ms), C.byref(cnt)))
            out[name.value.decode()] = (ms.value, cnt.value)
        return out

    def stream(self):
        return lib().spes_stream(self._ctx)

    def kernel_launches(self):
        return lib().spes_kernel_launches(self._ctx)
