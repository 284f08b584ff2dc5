"""ctypes mirror of include/spes_b200.h (types only; no library loading here)."""
import ctypes as C


class ModelCfg(C.Structure):
    """spes_model_cfg == ModelConfig + LossCoeffs (proj/include/spes/model.hpp:14-41)."""

    _fields_ = [
        ("vocab", C.c_int64),
        ("hidden", C.c_int64),
        ("intermediate", C.c_int64),
        ("layers", C.c_int32),
        ("experts_total", C.c_int32),
        ("experts_active", C.c_int32),
        ("renormalize_after_topk", C.c_int32),
        ("tied_head", C.c_int32),
        ("_pad", C.c_int32),
        ("coeff_ce", C.c_double),
        ("coeff_lb", C.c_double),
        ("coeff_moe_z", C.c_double),
        ("coeff_z", C.c_double),
        ("rms_eps", C.c_float),
        ("_pad2", C.c_float),
    ]


class AdamWCfg(C.Structure):
    """spes_adamw_cfg == AdamWConfig (proj/include/spes/trainer.hpp:45-51)."""

    _fields_ = [("lr", C.c_double), ("beta1", C.c_double), ("beta2", C.c_double),
                ("eps", C.c_double), ("weight_decay", C.c_double)]


class MergeSched(C.Structure):
    """spes_merge_sched == MergeSchedule (proj/include/spes/merging.hpp:14-25)."""

    _fields_ = [("warmup_rounds", C.c_int32), ("interval", C.c_int32), ("alpha0", C.c_double),
                ("peers", C.c_int32), ("source", C.c_int32)]


class Losses(C.Structure):
    """spes_losses == LossBundle (proj/include/spes/model.hpp:376-378)."""

    _fields_ = [("total", C.c_double), ("ce", C.c_double), ("lb", C.c_double),
                ("moe_z", C.c_double), ("z", C.c_double)]

    def as_tuple(self):
        return (self.total, self.ce, self.lb, self.moe_z, self.z)


class MergeEvent(C.Structure):
    """spes_merge_event == MergeEvent (proj/include/spes/merging.hpp:97-102)."""

    _fields_ = [("layer", C.c_int32), ("peers_k", C.c_int32), ("alpha", C.c_double),
                ("displacement_sq", C.c_double)]


class SyncStats(C.Structure):
    _fields_ = [("psi_bytes_in", C.c_double), ("expert_bytes_in", C.c_double), ("ms", C.c_double)]


def model_cfg(vocab=64, hidden=32, intermediate=64, layers=2, experts_total=4, experts_active=2,
              renormalize_after_topk=False, coeffs=(1.0, 0.01, 0.001, 1e-5), rms_eps=1e-5):
    """Defaults are the reference's ModelConfig defaults (model.hpp:21-31)."""
    return ModelCfg(vocab, hidden, intermediate, layers, experts_total, experts_active,
                    int(bool(renormalize_after_topk)), 0, 0, coeffs[0], coeffs[1], coeffs[2],
                    coeffs[3], rms_eps, 0.0)


def adamw_cfg(lr=1e-3, beta1=0.9, beta2=0.95, eps=1e-8, weight_decay=0.1):
    return AdamWCfg(lr, beta1, beta2, eps, weight_decay)


def merge_sched(warmup_rounds=0, interval=1, alpha0=0.1, peers=4, source=0):
    return MergeSched(warmup_rounds, interval, alpha0, peers, source)


# Named configurations of BASELINE.json (shapes fixed in SURVEY.md §8d).
CONFIGS = {
    # cfg1: tiny MoE, CPU-runnable oracle case
    "cfg1": dict(model=dict(vocab=256, hidden=128, intermediate=256, layers=2, experts_total=8,
                            experts_active=2), nodes=2, owned=4, H=4, B=4, S=64),
    # cfg2: single MoE block d=1024, 16 experts top-2, 8 nodes x 4 owned (r=2), seq 2048, H=50
    "cfg2": dict(model=dict(vocab=256, hidden=1024, intermediate=1024, layers=1, experts_total=16,
                            experts_active=2), nodes=8, owned=4, H=50, B=8, S=2048),
    # cfg3: cfg2 with a merge every round (H=1)
    "cfg3": dict(model=dict(vocab=256, hidden=1024, intermediate=1024, layers=1, experts_total=16,
                            experts_active=2), nodes=8, owned=4, H=1, B=8, S=2048, merge=True),
    # cfg4: 2B-class layer d=2048, 64 experts top-8, ffn 1024, 8 nodes x 16 owned, seq 4096
    "cfg4": dict(model=dict(vocab=256, hidden=2048, intermediate=1024, layers=1, experts_total=64,
                            experts_active=8), nodes=8, owned=16, H=50, B=4, S=4096),
    # cfg5: 7B-class stack d=4096, 64 experts top-8, ffn 2048, L=4 (chosen), seq 4096
    "cfg5": dict(model=dict(vocab=256, hidden=4096, intermediate=2048, layers=4, experts_total=64,
                            experts_active=8), nodes=8, owned=16, H=50, B=4, S=4096),
}
