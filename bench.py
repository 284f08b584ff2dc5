#!/usr/bin/env python
"""SPES hot-path benchmark (BASELINE.json metric) on 1..8 B200s.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg5] [--impl ours|reference]

One bench step = one SPES round of the configuration: H local training steps
(forward + backward + masked AdamW over psi and the owned experts) on every node,
then the sparse synchronization (owner-set means over NCCL), plus the expert merge
when the configuration has the warm-up active. Metric = training tokens/s
(all nodes) = N * H * B * S / round time; the sync is therefore amortised over H
exactly as in the metric's definition. For N > 1 launch with torchrun; one process
per GPU; timing = CUDA events on the library's stream, max over ranks.

Default workload: cfg5 (BASELINE.json configs[4], the largest configuration that fits one
B200: d=4096, f=2048, L=4, 64 experts top-8, seq 4096, H=50); cfg2..cfg4 via --config.

Timed arms:
  value : tokens already resident in HBM, no host sync inside a round except the sync step;
  e2e   : the public C-ABI call with HOST tokens (H2D each step) and the losses read back
          (D2H each step), wall clock, max over ranks.
--impl reference times the reference's own CPU implementation (oracle/_ref, compiled
from /root/reference sources) on this host's cores, on a bounded sample extrapolated to the
configuration (cpu_reference_sample).
"""
import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "training tokens/sec per SPES step (local + amortised sync) at 1/2/4/8 B200"
UNIT = "tokens/s"


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="cfg5")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--H", type=int, default=None, help="override sync interval")
    ap.add_argument("--prof-rounds", type=int, default=1,
                    help="rounds after the timed region with per-family CUDA-event profiling")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return rank, world, local


class Dist:
    """torch.distributed over gloo (CPU) for the launcher plumbing only: NCCL id
    exchange, barriers and the max-over-ranks of the measured times."""

    def __init__(self, rank, world):
        self.rank, self.world = rank, world
        self.pg = None
        if world > 1:
            import torch.distributed as td
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            td.init_process_group("gloo", rank=rank, world_size=world)
            self.td = td

    def barrier(self):
        if self.world > 1:
            self.td.barrier()

    def bcast(self, obj):
        if self.world == 1:
            return obj
        lst = [obj]
        self.td.broadcast_object_list(lst, src=0)
        return lst[0]

    def max(self, x):
        if self.world == 1:
            return x
        import torch
        t = torch.tensor([float(x)], dtype=torch.float64)
        self.td.all_reduce(t, op=self.td.ReduceOp.MAX)
        return float(t.item())

    def sum(self, x):
        if self.world == 1:
            return x
        import torch
        t = torch.tensor([float(x)], dtype=torch.float64)
        self.td.all_reduce(t, op=self.td.ReduceOp.SUM)
        return float(t.item())


def workload(name, N, H_override=None):
    from paper_2602_11543_b200.abi import CONFIGS, model_cfg
    import paper_2602_11543_b200 as spes
    c = dict(CONFIGS[name])
    cfg = model_cfg(**c["model"])
    M = cfg.experts_total
    if name == "cfg1":
        owned = spes.param_partition(cfg, N) if N <= M else None
        repl = 1
    else:
        owned = spes.replicated_ownership(M, N, 2)
        repl = 2
    H = H_override or c["H"]
    desc = {
        "cfg1": "cfg1 tiny MoE: V=256 d=128 f=256 L=2, 8 experts top-2, disjoint ownership",
        "cfg2": "cfg2 single MoE block d=1024 f=1024, 16 experts top-2, V=256, 2x replicated "
                "ownership (8 nodes x 4 owned at N=8), seq 2048, sync every 50 steps",
        "cfg3": "cfg3 = cfg2 shapes with sync + expert-merging warm-up every round (H=1)",
        "cfg4": "cfg4 2B-class layer d=2048 f=1024, 64 experts top-8, 2x replicated ownership, "
                "seq 4096",
        "cfg5": "cfg5 7B-class stack d=4096 f=2048 L=4, 64 experts top-8, 2x replicated, seq 4096",
    }[name]
    return cfg, owned, H, c["B"], c["S"], bool(c.get("merge")), repl, desc


def expert_flops_per_step(cfg, counts_by_layer, owned):
    """Algorithmic tensor FLOPs of one local step:
    6*d*f*(2*sum_j n_j + sum_{owned} n_j) per layer + head 3 * 2*T*d*V."""
    d, f = cfg.hidden, cfg.intermediate
    tot = 0.0
    for cnt in counts_by_layer:
        cnt = np.asarray(cnt, np.float64)
        tot += 6.0 * d * f * (2.0 * cnt.sum() + cnt[list(owned)].sum())
    return tot


def clocks_sampler():
    """nvidia-smi clocks + throttle reasons during the timed region."""
    q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    try:
        p = subprocess.Popen(["nvidia-smi", f"--query-gpu={q}", "--format=csv,noheader,nounits",
                              "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL,
                             text=True)
    except Exception:
        return None
    lines = []

    def rd():
        for ln in p.stdout:
            lines.append(ln.strip())

    t = threading.Thread(target=rd, daemon=True)
    t.start()
    return p, lines


def clocks_summary(handle, device):
    if handle is None:
        return None
    p, lines = handle
    time.sleep(0.3)
    p.terminate()
    try:
        p.wait(timeout=5)
    except Exception:
        p.kill()
    sm, mx, reasons = [], 0, set()
    names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
    for ln in lines:
        parts = [x.strip() for x in ln.split(",")]
        if len(parts) < 9 or not parts[0].isdigit() or int(parts[0]) != device:
            continue
        try:
            sm.append(float(parts[1]))
            mx = max(mx, float(parts[2]))
        except ValueError:
            continue
        for nm, v in zip(names, parts[5:9]):
            if v.lower() == "active":
                reasons.add(nm)
    if not sm:
        return None
    loaded = [x for x in sm if x > 0.5 * mx] or sm
    return {"sm_mhz": float(np.median(loaded)), "sm_max_mhz": mx, "reasons": sorted(reasons),
            "samples": len(sm)}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return p["bf16_tflops"], p["bf16_tflops_sustained"], p["hbm_gbs"], "measured"
    except Exception:
        return 1590.0, 1400.0, 6650.0, "fallback (B200_PROFILING.md)"


def hbm_rooflines(fam, cfg, counts, owned, G, T, hbm_peak, steps):
    """HBM-bound kernel families: algorithmic bytes per step (SURVEY.md §8(d) formulas, with
    this implementation's element widths) over the family's measured CUDA-event time per step
    (profiled round). T tokens, R = T*k routed rows, R_own rows of owned experts, per layer:
      router_fwd     h (fp32) read, normed (bf16) + logits + probs (fp32) + top-k (idx, w) +
                     3 per-token scalars written: 6Td + 8TM + 8Tk + 12T
      permute        normed rows read once, gathered rows written: 2Td + 2Rd
      combine_fwd    expert rows (fp32) + residual read, next input written: 4Rd + 8Td
      combine_bwd    upstream grad + expert rows read, bf16 row grads + gate grads written:
                     4Td + 4Rd + 2Rd + 4R
      router_bwd     expert-input grads (fp32) + h read, normed grad written, plus the
                     router's per-token scalars (probs read, logit grads written):
                     4Rd + 8Td + 8TM
      norm_router    h + normed grad read, residual grad written: 12Td (+ 4TM logit grads)
      embed_grad     layer-0 grad rows read, embedding grad written: 4Td + 4Vd
      adamw          theta, g, m, v read; theta, m, v written (fp32); bf16 copy of expert /
                     head scalars written: 28 B per trainable scalar + 2 B per copied one"""
    d, f, M, k, V, L = (cfg.hidden, cfg.intermediate, cfg.experts_total, cfg.experts_active,
                        cfg.vocab, cfg.layers)
    R = T * k
    by = {
        "router_fwd": L * (6 * T * d + 8 * T * M + 8 * T * k + 12 * T),
        "permute": L * (2 * T * d + 2 * R * d),
        "combine_fwd": L * (4 * R * d + 8 * T * d),
        "combine_bwd": L * (4 * T * d + 6 * R * d + 4 * R),
        "router_bwd": L * (4 * R * d + 8 * T * d + 8 * T * M),
        "norm_router_grads": L * (12 * T * d + 4 * T * M),
        "embed_grad": 4 * T * d + 4 * V * d,
    }
    psi_no_copy = V * d + L * (d + d * M)  # embedding, norms, routers: no bf16 copy
    by["adamw"] = 28.0 * G + 2.0 * (G - psi_no_copy)
    out = {}
    for k_, b in by.items():
        if k_ not in fam:
            continue
        ms = fam[k_][0] / steps
        gbs = b / (ms / 1e3) / 1e9
        out[k_] = {"bytes_per_step": float(b), "ms_per_step": ms, "achieved": gbs,
                   "peak": hbm_peak, "unit": "GB/s", "frac": gbs / hbm_peak}
    return out


def gemm_rooflines(fam, cfg, counts, owned, T, peak, steps):
    """Per expert-GEMM family: algorithmic FLOPs per step from the routing counts (R rows,
    R_own rows of owned experts) over its CUDA-event time per step."""
    d, f = cfg.hidden, cfg.intermediate
    R = float(sum(np.sum(c) for c in counts))
    R_own = float(sum(np.asarray(c)[list(owned)].sum() for c in counts))
    fl = {"gemm_fwd_gate_up": 4 * R * d * f, "gemm_fwd_down": 2 * R * d * f,
          "gemm_bwd_dh": 2 * R * d * f, "gemm_bwd_dx": 4 * R * d * f,
          "gemm_bwd_dw_gate_up": 4 * R_own * d * f, "gemm_bwd_dw_down": 2 * R_own * d * f,
          # router weight gradient normed^T glog (tensor cores above 16 experts): 2 T d M per
          # layer of algorithmic work (the device pads M to 128 columns)
          "router_grad_gemm": 2.0 * T * d * cfg.experts_total * cfg.layers}
    # the fused placement (SPES_FUSED_OPT=1) times the dW GEMMs with their MaskedAdamW
    for k_ in list(fl):
        if k_ + "+adamw" in fam:
            fl[k_ + "+adamw"] = fl[k_]
    out = {}
    for k_, x in fl.items():
        if k_ not in fam:
            continue
        ms = fam[k_][0] / steps
        tf = x / (ms / 1e3) / 1e12
        out[k_] = {"tflop_per_step": x / 1e12, "ms_per_step": ms, "achieved": tf, "peak": peak,
                   "unit": "TFLOP/s", "frac": tf / peak}
    return out


def sync_roofline(st, N):
    """The last round's sparse sync on this rank: inbound bytes (psi copies + expert copies
    read over NVLink / received over NCCL) over its device time, against the 900 GB/s per
    direction NVLink 5 gives each B200."""
    if not st or N < 2 or not st.get("ms"):
        return None
    b = float(st["psi_bytes_in"]) + float(st["expert_bytes_in"])
    gbs = b / (st["ms"] / 1e3) / 1e9
    return {"bound": "nvlink", "ms": st["ms"], "bytes_in": b, "achieved": gbs, "peak": 900.0,
            "unit": "GB/s", "frac": gbs / 900.0,
            "note": "rank 0; ms runs from the moment every node has arrived (waiting for slower "
                    "nodes' local rounds excluded) and includes the owner means, pulls, barrier "
                    "and operand-copy writes"}


def ncu_traffic(cfg_name):
    """DRAM bytes per launch of the grouped GEMM measured by ncu --set full on this
    configuration (profiles/ncu_traffic.json, written from the committed capture), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as fh:
            e = json.load(fh).get(cfg_name)
        return None if e is None else e.get("gemm_dram_bytes_per_launch")
    except Exception:
        return None


# ------------------------------------------------------------------ CPU reference

def _ref_pair_seconds(R, cfg, owned, S1, S2, rng, parallel):
    """Two reference local_round steps (H=1, B=1) from one global model, at S1 and S2 tokens:
    wall time of each local_round call itself (the shim's flat -> ModelParams conversion,
    done once, excluded)."""
    import ctypes as C
    import oracle
    from paper_2602_11543_b200.abi import adamw_cfg
    P = oracle.param_count(cfg)
    params = np.empty(P, np.float32)
    for i in range(0, P, 1 << 26):
        n = min(1 << 26, P - i)
        rng.standard_normal(n, dtype=np.float32, out=params[i:i + n])
        params[i:i + n] *= np.float32(0.02)
    t1 = rng.integers(0, cfg.vocab, size=(S1 + 1,), dtype=np.int32)
    t2 = rng.integers(0, cfg.vocab, size=(S2 + 1,), dtype=np.int32)
    sec = np.zeros(2, np.float64)
    R.ref_set_parallel(1 if parallel else 0)
    rc = R.ref_local_round_pair_timed(C.byref(cfg), params, t1, S1, t2, S2, C.byref(adamw_cfg()),
                                      oracle.trainable_mask(cfg, owned), sec)
    R.ref_set_parallel(1)
    assert rc == 0, rc
    return float(sec[0]), float(sec[1])


def cpu_reference_sample(cfg_name, N, parallel=True):
    """The reference's own CPU path (oracle/_ref = /root/reference compiled from its sources)
    on this host, as a bounded sample extrapolated to the configuration's step:
      * one layer (L=1) of the configuration's d, f, V and top-k; for M > 16 the sample keeps
        M_s = k experts (every token then visits as many experts, so the per-token expert work
        is the configuration's) and node 0's owned fraction of them;
      * two local_round steps (H=1, B=1) at S1 and S2 tokens give the per-token time a and the
        per-step constant b (MaskedAdamW, parameter copies) of that layer;
      * step(T) = L * (a*T + b * P_layer / P_layer_sample) (the constant scales with the
        layer's parameters), plus Server::aggregate's cost at N nodes amortised over H
        (negligible: measured at the sample's size and scaled the same way).
    Returns (tokens/s, seconds per sampled pair, threads, description)."""
    import oracle
    from paper_2602_11543_b200.abi import model_cfg
    cfg, owned, H, B, S, merge, repl, desc = workload(cfg_name, N)
    d, f, M, k, V, L = (cfg.hidden, cfg.intermediate, cfg.experts_total, cfg.experts_active,
                        cfg.vocab, cfg.layers)
    Ms = M if M <= 16 else k
    own_frac = len(owned[0]) / M
    owned_s = list(range(max(1, round(Ms * own_frac))))
    scfg = model_cfg(vocab=V, hidden=d, intermediate=f, layers=1, experts_total=Ms,
                     experts_active=k)
    S1, S2 = (16, 64) if d * f >= 2048 * 1024 else (128, 384)
    R = oracle.ref()
    rng = np.random.default_rng(1)
    t0 = time.perf_counter()
    t1, t2 = _ref_pair_seconds(R, scfg, owned_s, S1, S2, rng, parallel)
    wall = time.perf_counter() - t0
    a = max((t2 - t1) / (S2 - S1), 1e-12)
    b = max(t1 - a * S1, 0.0)
    p_layer = d * (M + 1) + 3.0 * d * f * M
    p_sample = d * (Ms + 1) + 3.0 * d * f * Ms
    T = B * S
    step = L * (a * T + b * p_layer / p_sample)
    threads = int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1)) if parallel else 1
    sample = (f"{cfg_name}: reference local_round (H=1, B=1) at S={S1} and S={S2} tokens on one "
              f"layer with d={d} f={f} V={V} k={k}, {Ms} experts ({len(owned_s)} owned); per-token "
              f"{a:.4g} s, per-step constant {b:.4g} s; extrapolated to L={L}, M={M}, T={T} "
              f"tokens: {step:.4g} s per step; OpenMP threads={threads}")
    return T / step, wall, threads, sample


def reference_arm(args):
    rank, world, local = dist_env()
    if rank != 0:
        return 0
    # all host cores for the one process that runs (torchrun sets OMP_NUM_THREADS=1 for its
    # ranks; the reference's OpenMP runtime reads it when oracle/_ref is first loaded)
    os.environ["OMP_NUM_THREADS"] = str(os.cpu_count() or 1)
    vals = []
    # a CPU sample needs no more than one warm-up (page-in); each step is one bounded sample
    warm = min(args.warmup, 1)
    for i in range(warm + args.steps):
        v, sec, threads, sample = cpu_reference_sample(args.config, args.gpus)
        if i >= warm:
            vals.append((v, sec))
    value = float(np.mean([v for v, _ in vals]))
    ms = float(np.mean([s for _, s in vals])) * 1e3
    cfg, owned, H, B, S, merge, repl, desc = workload(args.config, args.gpus)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic", "impl": "reference",
        "config": {"workload": desc, "name": args.config,
                   "sample": "bounded CPU sample extrapolated to the configuration (see "
                             "cpu_baseline.sample); ms_per_step = wall time of one sample"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference",
                         "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    emit(line)
    return 0


# ------------------------------------------------------------------ our arm

def our_arm(args):
    import torch
    import paper_2602_11543_b200 as spes
    from paper_2602_11543_b200.abi import adamw_cfg, merge_sched
    rank, world, local = dist_env()
    if world != args.gpus:
        log(f"warning: --gpus {args.gpus} but WORLD_SIZE={world}; using {world}")
    N = world
    dist = Dist(rank, world)
    cfg, owned, H, B, S, merge, repl, desc = workload(args.config, N, args.H)
    torch.cuda.set_device(local)
    nccl_id = dist.bcast(spes.nccl_unique_id() if rank == 0 else None) if N > 1 else None
    node = spes.Node(cfg, node=rank, n_nodes=N, device=local, nccl_id=nccl_id)
    node.set_ownership(owned)
    # synthetic init N(0, 0.02), norm gains 1 (init_model, model.hpp:153-173), drawn on the
    # device from one seed, so every node starts from the identical global model (a 26 GB
    # cfg5 model is not staged through host memory)
    P = spes.param_count(cfg)
    gen = torch.Generator(device=f"cuda:{local}")
    gen.manual_seed(1)
    params = torch.empty(P, dtype=torch.float32, device=f"cuda:{local}")
    for i in range(0, P, 1 << 28):
        n = min(1 << 28, P - i)
        params[i:i + n].normal_(0.0, 0.02, generator=gen)
    offs = spes.block_offsets(cfg)
    for l in range(cfg.layers):
        o = int(offs[2 + 2 * l])
        params[o:o + cfg.hidden] = 1.0
    torch.cuda.synchronize(local)
    node.load_params_device(params.data_ptr(), P)
    del params
    torch.cuda.empty_cache()
    trng = np.random.default_rng(1000 + rank)  # per-node data shard
    toks_host = trng.integers(0, cfg.vocab, size=(H, B, S + 1), dtype=np.int32)
    toks_dev = torch.from_numpy(toks_host).to(f"cuda:{local}")
    ptrs = [toks_dev[h].data_ptr() for h in range(H)]
    opt = adamw_cfg(lr=1e-4)
    sched = merge_sched(warmup_rounds=10 ** 6, interval=1, alpha0=0.1, peers=4, source=0)
    stream = torch.cuda.ExternalStream(node.stream(), device=f"cuda:{local}")

    round_no = [0]
    last_sync = [None]

    def spes_round(host=False):
        node.round_begin()
        for h in range(H):
            if host:
                node.local_step(toks_host[h], opt)  # H2D tokens + D2H losses every step
            else:
                node.local_step_device(ptrs[h], B, S, opt)
        last_sync[0] = node.sync()
        if merge:
            node.merge_model(sched, round_no[0])
        round_no[0] += 1

    for _ in range(args.warmup):
        spes_round()
    torch.cuda.synchronize(local)
    dist.barrier()

    # ---- timed region: K rounds, device-resident tokens, no profiling events (the local
    # step replays as one CUDA graph) ----
    clk = clocks_sampler() if rank == 0 else None
    launches0 = node.kernel_launches()
    dist.barrier()
    torch.cuda.synchronize(local)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        spes_round()
    e1.record(stream)
    torch.cuda.synchronize(local)
    dist.barrier()
    ms = dist.max(e0.elapsed_time(e1))
    launches = node.kernel_launches() - launches0
    clocks = clocks_summary(clk, local) if rank == 0 else None

    # ---- kernel-family breakdown: CUDA events bracket every family on the context's
    # stream during PROF_ROUNDS extra rounds (eager launches); rates below are per launch
    node.profile(True, reset=True)
    for _ in range(args.prof_rounds):
        spes_round()
    torch.cuda.synchronize(local)
    node.profile(False)
    fam = node.profile_stats()
    sync_st = last_sync[0]  # the last device-resident round's sync (the e2e rounds' include host skew)

    tokens = N * H * B * S * args.steps
    value = tokens / (ms / 1e3)

    # ---- e2e: public API with host tokens and losses read back every step ----
    # (--e2e-steps 0 skips it: sweeps only)
    ke = max(1, min(args.steps, 3)) if args.e2e_steps is None else args.e2e_steps
    e2e_value = None
    if ke > 0:
        dist.barrier()
        torch.cuda.synchronize(local)
        t0 = time.perf_counter()
        for _ in range(ke):
            spes_round(host=True)
        torch.cuda.synchronize(local)
        t_e2e = dist.max(time.perf_counter() - t0)
        e2e_value = N * H * B * S * ke / t_e2e

    # ---- rooflines from the profiled round: the grouped tcgen05 GEMM (dominant kernel)
    # and every HBM-bound family ----
    T = B * S
    counts = [node.debug("counts", l, np.int32, None, cfg.experts_total) for l in range(cfg.layers)]
    gemm_fams = [k for k in fam if k.startswith("gemm_")]
    gemm_ms = sum(fam[k][0] for k in gemm_fams)
    gemm_launches = sum(fam[k][1] for k in gemm_fams)
    steps_prof = H * args.prof_rounds
    expert_flops = expert_flops_per_step(cfg, counts, owned[rank]) * steps_prof
    burst, sustained, hbm, peak_src = peaks()
    achieved = expert_flops / (gemm_ms / 1e3) / 1e12 if gemm_ms > 0 else 0.0
    G = node.counts()["grad_scalars"]
    hbm_lines = hbm_rooflines(fam, cfg, counts, owned[rank], G, T, hbm, steps_prof)
    gemm_lines = gemm_rooflines(fam, cfg, counts, owned[rank], T, sustained, steps_prof)
    step_ms_total = sum(v[0] for v in fam.values())
    if rank == 0:
        log(f"kernel family breakdown (device ms over {args.prof_rounds} profiled round(s) after "
            "the timed region, share of profiled time):")
        for k, (t, n) in sorted(fam.items(), key=lambda kv: -kv[1][0]):
            extra = ""
            if k in hbm_lines:
                extra = f"  {hbm_lines[k]['achieved']:8.1f} GB/s ({hbm_lines[k]['frac']:.2f} of HBM)"
            elif k in gemm_lines:
                extra = (f"  {gemm_lines[k]['achieved']:8.1f} TFLOP/s "
                         f"({gemm_lines[k]['frac']:.2f} of sustained bf16)")
            log(f"  {k:24s} {t:10.3f} ms  {n:6d} launches  "
                f"{100 * t / max(step_ms_total, 1e-9):5.1f}%{extra}")
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": N, "steps": args.steps,
        "value_per_gpu": value / N,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
        "config": {"workload": desc, "name": args.config, "d": cfg.hidden, "f": cfg.intermediate,
                   "layers": cfg.layers, "experts": cfg.experts_total, "top_k": cfg.experts_active,
                   "vocab": cfg.vocab, "B": B, "S": S, "H": H, "global_batch": N * B,
                   "seq_len": S, "nodes": N, "replication": repl,
                   "owned_per_node": len(owned[rank]), "merge_every_round": merge,
                   "parallelism": f"spes-dp{N} (expert ownership, sparse sync)",
                   "step": f"one SPES round = {H} local steps + sparse sync"
                           + (" + merge" if merge else ""),
                   "l2": "inputs larger than L2: per-step activations >> 126 MB, no flush"},
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(H * B * (S + 1) * 4),
                "d2h_bytes_per_step": int(H * 5 * 8), "steps": ke},
        "gpu_launches": int(dist.sum(launches)),
        "roofline": {"bound": "tensor", "kernel": "grouped_gemm_2cta_kernel (tcgen05 cta_group::2/TMEM/TMA, "
                                                   "6 expert contractions)",
                     "achieved": achieved, "peak": sustained, "unit": "TFLOP/s",
                     "frac": achieved / sustained if sustained else None,
                     "peak_kind": f"bf16 sustained ({peak_src})",
                     "frac_of_burst": achieved / burst if burst else None,
                     "traffic": ncu_traffic(args.config), "launches": int(gemm_launches),
                     "flops_source": "6*d*f*(2*sum n_j + sum_owned n_j) per layer, last step's "
                                     "routing counts",
                     "timing": "CUDA events around every GEMM launch on the context stream, "
                               f"{args.prof_rounds} profiled round(s) right after the timed "
                               "region (the timed region itself runs unprofiled)"},
        "roofline_gemm": gemm_lines,
        "roofline_hbm": hbm_lines,
        "roofline_hbm_peak": f"{hbm:.1f} GB/s copy bandwidth ({peak_src})",
        "sync": sync_roofline(sync_st, N),
        "kernels_ms": {k: round(v[0], 4) for k, v in fam.items()},
        "clocks": clocks,
    }
    if rank == 0 and N == 1 and not args.no_cpu_baseline:
        try:
            v, sec, threads, sample = cpu_reference_sample(args.config, N)
            line["cpu_baseline"] = {"value": v, "unit": UNIT, "cores": threads,
                                    "kind": "reference", "sample": sample}
            if cfg.hidden * cfg.intermediate <= 1024 * 1024:
                # also the reference single-threaded (OpenMP off), same sample
                v1, _, _, _ = cpu_reference_sample(args.config, N, parallel=False)
                line["cpu_baseline"]["single_thread"] = {"value": v1, "unit": UNIT, "cores": 1}
        except Exception as e:  # the reference lib is test infra; report, don't fail
            line["cpu_baseline"] = {"value": None, "unit": UNIT, "cores": 0, "kind": "reference",
                                    "sample": f"unavailable: {e}"}
    if rank == 0:
        emit(line)
    node.close()
    return 0


_JSON_OUT = None


def emit(line):
    """The bench's one JSON line, on the real stdout."""
    out = _JSON_OUT or sys.stdout
    out.write(json.dumps(line) + "\n")
    out.flush()


def main():
    global _JSON_OUT
    os.environ.setdefault("OMP_NUM_THREADS", str(os.cpu_count() or 1))
    # stdout carries only the JSON line: native libraries' prints (e.g. NCCL's "NCCL
    # version" banner) are sent to stderr by pointing fd 1 at fd 2
    sys.stdout.flush()
    _JSON_OUT = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)
    args = parse()
    if args.impl == "reference":
        return reference_arm(args)
    return our_arm(args)


if __name__ == "__main__":
    sys.exit(main())
