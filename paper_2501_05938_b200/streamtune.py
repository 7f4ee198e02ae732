"""Python view of the streamtune C++ API through include/streamtune_c.h.

Every call runs the C++ implementation in libpm_tridiag.so (no Python
re-implementation): timing identities (timing_model.hpp:117-146), the
predictor, regression and the dataset
loaders / Eq. 5 batch step.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .errors import raise_for
from .solver import StageTimings

ModelBundleC = _lib.ModelBundleC
CANDIDATES = (2, 4, 8, 16, 32)


def _err():
    return C.create_string_buffer(512)


def _call(fn, *args):
    e = _err()
    st = fn(*args, e, len(e))
    if st != 0:
        raise_for(st, e.value.decode(errors="replace"))


def _st(t: StageTimings):
    return _lib.StageTimingsC(int(t.slae_size), t.t1_h2d, t.t1_comp, t.t1_d2h, t.t2_comp, t.t3_h2d,
                              t.t3_comp, t.t3_d2h)


@dataclass
class ModelBundle:
    """streamtune::ModelBundle; keys as SPEC.md:316 (sum, overhead_small, overhead_big)."""
    sum_a: float = 0.0
    sum_b: float = 0.0
    small_a: float = 0.0
    small_b: float = 0.0
    small_c: float = 0.0
    big_a: float = 0.0
    big_b: float = 0.0
    big_c: float = 0.0
    size_threshold: int = 1_000_000
    candidates: tuple = CANDIDATES
    provenance: dict = field(default_factory=dict)

    @staticmethod
    def paper() -> "ModelBundle":
        c = ModelBundleC()
        _lib.load().pm_paper_bundle(C.byref(c))
        return ModelBundle.from_c(c, provenance={"fitted_on": "RTX 2080 Ti (paper Eq. 4 / Eq. 7)"})

    @staticmethod
    def b200() -> "ModelBundle":
        c = ModelBundleC()
        _lib.load().pm_b200_bundle(C.byref(c))
        return ModelBundle.from_c(c, provenance={"fitted_on": "NVIDIA B200 re-fit (refit/pooled/)"})

    @staticmethod
    def from_c(c, provenance=None) -> "ModelBundle":
        return ModelBundle(c.sum_a, c.sum_b, c.small_a, c.small_b, c.small_c, c.big_a, c.big_b, c.big_c,
                           int(c.size_threshold), tuple(c.candidates[k] for k in range(c.num_candidates)),
                           provenance or {})

    def to_c(self):
        c = ModelBundleC(self.sum_a, self.sum_b, self.small_a, self.small_b, self.small_c, self.big_a,
                         self.big_b, self.big_c, int(self.size_threshold), len(self.candidates))
        for k, v in enumerate(self.candidates):
            c.candidates[k] = int(v)
        return c

    def to_document(self) -> dict:
        """Serialisation with the SPEC.md:316 key names (>= 15 significant digits)."""
        return {
            "sum": {"a": repr(self.sum_a), "b": repr(self.sum_b)},
            "overhead_small": {"a": repr(self.small_a), "b": repr(self.small_b), "c": repr(self.small_c)},
            "overhead_big": {"a": repr(self.big_a), "b": repr(self.big_b), "c": repr(self.big_c)},
            "size_threshold": int(self.size_threshold),
            "candidates": list(self.candidates),
            "provenance": self.provenance,
        }

    @staticmethod
    def from_document(doc: dict) -> "ModelBundle":
        f = float
        return ModelBundle(f(doc["sum"]["a"]), f(doc["sum"]["b"]), f(doc["overhead_small"]["a"]),
                           f(doc["overhead_small"]["b"]), f(doc["overhead_small"]["c"]),
                           f(doc["overhead_big"]["a"]), f(doc["overhead_big"]["b"]),
                           f(doc["overhead_big"]["c"]), int(doc.get("size_threshold", 1_000_000)),
                           tuple(doc.get("candidates", CANDIDATES)), doc.get("provenance", {}))


# ---- timing_model ---------------------------------------------------------------
def stream_count_is_valid(n: int) -> bool:
    return bool(_lib.load().st_stream_count_is_valid(int(n)))


def validate_stage_timings(t: StageTimings) -> None:
    s = _st(t)
    _call(_lib.load().st_validate_stage_timings, C.byref(s))


def total_unstreamed(t: StageTimings) -> float:
    s = _st(t)
    return _lib.load().st_total_unstreamed(C.byref(s))


def overlap_sum(t: StageTimings) -> float:
    s = _st(t)
    return _lib.load().st_overlap_sum(C.byref(s))


def streamed_lower_bound(t: StageTimings, n: int, overhead_ms: float) -> float:
    s, out = _st(t), C.c_double()
    _call(_lib.load().st_streamed_lower_bound, C.byref(s), int(n), float(overhead_ms), C.byref(out))
    return out.value


def overhead_from_measurement(t_str: float, t_non_str: float, n: int, sum_ms: float) -> float:
    out = C.c_double()
    _call(_lib.load().st_overhead_from_measurement, t_str, t_non_str, int(n), sum_ms, C.byref(out))
    return out.value


def overlap_benefit(n: int, sum_ms: float, overhead_ms: float) -> float:
    out = C.c_double()
    _call(_lib.load().st_overlap_benefit, int(n), sum_ms, overhead_ms, C.byref(out))
    return out.value


# ---- predictor ---------------------------------------------------------------------
def predict_sum(bundle: ModelBundle, n: int) -> float:
    b, out = bundle.to_c(), C.c_double()
    _call(_lib.load().st_predict_sum, C.byref(b), int(n), C.byref(out))
    return out.value


def predict_overhead(bundle: ModelBundle, n: int, streams: int) -> float:
    b, out = bundle.to_c(), C.c_double()
    _call(_lib.load().st_predict_overhead, C.byref(b), int(n), int(streams), C.byref(out))
    return out.value


@dataclass
class Recommendation:
    slae_size: int
    chosen: int
    benefits: list
    overheads: list
    predicted_sum: float
    model_used: str


def recommend(bundle: ModelBundle, n: int) -> Recommendation:
    b = bundle.to_c()
    chosen, used, psum = C.c_int(), C.c_int(), C.c_double()
    ben, ovh = (C.c_double * 5)(), (C.c_double * 5)()
    _call(_lib.load().st_recommend, C.byref(b), int(n), C.byref(chosen), ben, ovh, C.byref(psum),
          C.byref(used))
    k = len(bundle.candidates)
    return Recommendation(int(n), chosen.value, list(ben)[:k], list(ovh)[:k], psum.value,
                          "small" if used.value == 0 else "big")


def recommend_fp32(bundle: ModelBundle, n: int) -> int:
    b, out = bundle.to_c(), C.c_int()
    _call(_lib.load().st_recommend_fp32, C.byref(b), int(n), C.byref(out))
    return out.value


def gomez_luna_optimum(sum_ms: float, tau_ms: float) -> float:
    out = C.c_double()
    _call(_lib.load().st_gomez_luna_optimum, float(sum_ms), float(tau_ms), C.byref(out))
    return out.value


# ---- regression -----------------------------------------------------------------------
def train_test_split(n: int, train_fraction: float = 0.75, shuffle: bool = True, seed: int = 42):
    order = (C.c_int * max(n, 1))()
    nt = C.c_int()
    _call(_lib.load().st_train_test_split, int(n), float(train_fraction), int(shuffle), int(seed), order,
          C.byref(nt))
    idx = list(order)[:n]
    return idx[: nt.value], idx[nt.value:]


def fit_least_squares(X, y) -> np.ndarray:
    X = np.ascontiguousarray(X, np.float64)
    y = np.ascontiguousarray(y, np.float64)
    beta = np.zeros(X.shape[1])
    D = C.POINTER(C.c_double)
    _call(_lib.load().st_fit_least_squares, X.ctypes.data_as(D), y.ctypes.data_as(D), X.shape[0],
          X.shape[1], beta.ctypes.data_as(D))
    return beta


def metrics(predicted, actual) -> dict:
    p = np.ascontiguousarray(predicted, np.float64)
    a = np.ascontiguousarray(actual, np.float64)
    out = np.zeros(3)
    D = C.POINTER(C.c_double)
    _call(_lib.load().st_metrics, p.ctypes.data_as(D), a.ctypes.data_as(D), len(a), out.ctypes.data_as(D))
    return {"r_squared": out[0], "mse": out[1], "rmse": out[2]}


@dataclass
class FitReport:
    coefficients: list
    train: dict
    test: dict
    n_train: int


def fit_model(kind: str, sizes, target, streams=None, train_fraction=0.75, shuffle=True,
              seed=42) -> FitReport:
    """kind: 'sum' (Eq. 4), 'small' / 'big' (Eq. 7)."""
    k = {"sum": 0, "small": 1, "big": 2}[kind]
    rows = len(sizes)
    sz = (C.c_uint64 * max(rows, 1))(*[int(s) for s in sizes])
    ns = (C.c_int * max(rows, 1))(*([int(s) for s in streams] if streams is not None else [1] * rows))
    tg = (C.c_double * max(rows, 1))(*[float(t) for t in target])
    coef = (C.c_double * 3)()
    met = (C.c_double * 6)()
    nt = C.c_int()
    _call(_lib.load().st_fit_model, k, sz, ns, tg, rows, float(train_fraction), int(shuffle), int(seed),
          coef, met, C.byref(nt))
    names = ("r_squared", "mse", "rmse")
    return FitReport(list(coef)[: (2 if k == 0 else 3)], dict(zip(names, list(met)[:3])),
                     dict(zip(names, list(met)[3:])), nt.value)


# ---- dataset -----------------------------------------------------------------------------
def load_stage_timings(csv_text: str) -> list[StageTimings]:
    rows = (_lib.StageTimingsC * 4096)()
    n = C.c_int()
    _call(_lib.load().st_load_stage_timings, csv_text.encode(), rows, 4096, C.byref(n))
    return [StageTimings(*[getattr(rows[k], f) for f, _ in _lib.StageTimingsC._fields_])
            for k in range(min(n.value, 4096))]


def load_streamed_runs(csv_text: str) -> list[tuple[int, int, float]]:
    cap = 65536
    sz, ns, ts = (C.c_uint64 * cap)(), (C.c_int * cap)(), (C.c_double * cap)()
    n = C.c_int()
    _call(_lib.load().st_load_streamed_runs, csv_text.encode(), sz, ns, ts, cap, C.byref(n))
    return [(int(sz[k]), int(ns[k]), float(ts[k])) for k in range(min(n.value, cap))]


def derive_overhead_rows(stage_csv: str, runs_csv: str) -> list[tuple[int, int, float]]:
    cap = 65536
    sz, ns, ov = (C.c_uint64 * cap)(), (C.c_int * cap)(), (C.c_double * cap)()
    n = C.c_int()
    _call(_lib.load().st_derive_overhead_rows, stage_csv.encode(), runs_csv.encode(), sz, ns, ov, cap,
          C.byref(n))
    return [(int(sz[k]), int(ns[k]), float(ov[k])) for k in range(min(n.value, cap))]


def fit_bundle(stage_csv: str, runs_csv: str, size_threshold: int = 1_000_000, seed: int = 42,
               anchored: bool = False):
    """cmd_fit: returns (ModelBundle, metrics dict).
    anchored=True: the B200 re-fit's constrained overhead forms
    (T_overhead(N, 1) = 0, coefficients >= 0; st_fit_bundle_anchored)."""
    b = ModelBundleC()
    met = (C.c_double * 18)()
    fn = _lib.load().st_fit_bundle_anchored if anchored else _lib.load().st_fit_bundle
    _call(fn, stage_csv.encode(), runs_csv.encode(), int(size_threshold), int(seed),
          C.byref(b), met)
    names = ("r_squared", "mse", "rmse")
    m = {}
    for i, model in enumerate(("sum", "small", "big")):
        m[model] = {"train": dict(zip(names, list(met)[6 * i: 6 * i + 3])),
                    "test": dict(zip(names, list(met)[6 * i + 3: 6 * i + 6]))}
    return ModelBundle.from_c(b, provenance={"seed": seed, "metrics": m}), m


# ---- simulator -----------------------------------------------------
ENGINES = ("h2d", "comp", "d2h")


@dataclass
class PipelineSpec:
    """streamtune::PipelineSpec: per-stage (h2d, comp, d2h) ms, the CPU Stage 2, n, tau."""
    stage1: tuple = (0.0, 0.0, 0.0)
    cpu_ms: float = 0.0
    stage3: tuple = (0.0, 0.0, 0.0)
    num_streams: int = 1
    tau_ms: float = 0.0
    hw_queues: int = 32

    def _stages(self):
        return (C.c_double * 7)(*[float(v) for v in (*self.stage1, self.cpu_ms, *self.stage3)])

    def timings(self, slae_size: int = 1) -> StageTimings:
        return StageTimings(slae_size, *self.stage1, self.cpu_ms, *self.stage3)


@dataclass
class SimResult:
    total_ms: float
    stage1_makespan_ms: float
    stage3_makespan_ms: float
    trace: list  # (engine, stream, stage, start_ms, end_ms)


def simulate(spec: PipelineSpec, trace: bool = True) -> SimResult:
    out = (C.c_double * 3)()
    cap = 6 * max(1, int(spec.num_streams)) if trace else 0
    tr = (C.c_double * max(1, 5 * cap))()
    ne = C.c_int()
    _call(_lib.load().st_simulate, spec._stages(), int(spec.num_streams), float(spec.tau_ms),
          int(spec.hw_queues), out, tr if trace else None, cap, C.byref(ne))
    events = []
    for k in range(min(ne.value, cap)):
        e, s, g, t0, t1 = tr[5 * k: 5 * k + 5]
        events.append((ENGINES[int(e)], int(s), int(g), t0, t1))
    return SimResult(out[0], out[1], out[2], events)


def verify_lower_bound(spec: PipelineSpec) -> tuple[bool, bool]:
    """(simulate.total >= Eq. 2 bound - 1e-9, dominance regime holds)."""
    h, d = C.c_int(), C.c_int()
    _call(_lib.load().st_verify_lower_bound, spec._stages(), int(spec.num_streams), float(spec.tau_ms),
          C.byref(h), C.byref(d))
    return bool(h.value), bool(d.value)


# ---- bundle document / report harness -----------------------------
def bundle_to_json(bundle: ModelBundle) -> str:
    b = bundle.to_c()
    need = C.c_int()
    buf = C.create_string_buffer(4096)
    _call(_lib.load().st_bundle_to_json, C.byref(b), buf, len(buf), C.byref(need))
    return buf.value.decode()


def bundle_from_json(doc: str) -> ModelBundle:
    b = ModelBundleC()
    _call(_lib.load().st_bundle_from_json, doc.encode(), C.byref(b))
    return ModelBundle.from_c(b)


STATUS = ("PASS", "FAIL", "KNOWN")


def report_table(bundle: ModelBundle, table: str) -> dict:
    b = bundle.to_c()
    p, f, k, nc = C.c_int(), C.c_int(), C.c_int(), C.c_int()
    cells = (C.c_double * (4 * 64))()
    _call(_lib.load().st_report_table, C.byref(b), table.encode(), C.byref(p), C.byref(f), C.byref(k),
          cells, 64, C.byref(nc))
    rows = [(cells[4 * i], cells[4 * i + 1], cells[4 * i + 2], STATUS[int(cells[4 * i + 3])])
            for i in range(min(nc.value, 64))]
    return {"passed": p.value, "failed": f.value, "known": k.value, "cells": rows}


def dump_reference(table: str) -> str:
    need = C.c_int()
    buf = C.create_string_buffer(8192)
    _call(_lib.load().st_dump_reference, table.encode(), buf, len(buf), C.byref(need))
    return buf.value.decode()
