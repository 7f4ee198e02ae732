"""Property-based tests (hypothesis) of the SPEC's stated invariants for the
timing model, the predictor and the
simulator, through the C ABI of the C++ implementation."""
import math

import pytest
from hypothesis import given, settings
from hypothesis import strategies as S

from paper_2501_05938_b200 import streamtune as st
from paper_2501_05938_b200.solver import StageTimings

durations = S.floats(min_value=0.0, max_value=1e4, allow_nan=False, allow_infinity=False)
counts = S.sampled_from([1, 2, 4, 8, 16, 32])
PAPER = st.ModelBundle.paper()


def timings(vals):
    return StageTimings(1000, *vals)


@settings(max_examples=300, deadline=None, derandomize=True)
@given(S.lists(durations, min_size=7, max_size=7), S.integers(0, 6),
       S.floats(min_value=0.0, max_value=100.0))
def test_total_is_additive_and_bounds_the_overlap_sum(vals, k, delta):
    t = timings(vals)
    base = st.total_unstreamed(t)
    bumped = list(vals)
    bumped[k] += delta
    assert st.total_unstreamed(timings(bumped)) == pytest.approx(base + delta, rel=1e-12, abs=1e-9)
    assert st.overlap_sum(t) <= base + 1e-9


@settings(max_examples=300, deadline=None, derandomize=True)
@given(S.lists(durations, min_size=7, max_size=7), S.floats(min_value=0.0, max_value=10.0))
def test_lower_bound_decreases_in_n(vals, ovh):
    t = timings(vals)
    prev = math.inf
    s = st.overlap_sum(t)
    rest = st.total_unstreamed(t) - s + ovh
    for n in (1, 2, 4, 8, 16, 32):
        lb = st.streamed_lower_bound(t, n, ovh)
        assert lb <= prev
        if s > 1e-9 * (rest + 1.0):  # strictly, when the 1/n term is representable
            assert lb < prev
        prev = lb
    assert st.streamed_lower_bound(t, 1, 0.0) == pytest.approx(st.total_unstreamed(t), rel=1e-12)


@settings(max_examples=300, deadline=None, derandomize=True)
@given(durations, durations, counts, durations)
def test_overhead_then_benefit_is_the_measured_saving(t_str, t_non, n, s):
    ovh = st.overhead_from_measurement(t_str, t_non, n, s)
    assert st.overlap_benefit(n, s, ovh) == pytest.approx(t_non - t_str, rel=1e-12, abs=1e-9)


@settings(max_examples=200, deadline=None, derandomize=True)
@given(S.floats(min_value=0.0, max_value=1e3), S.floats(min_value=1e-6, max_value=1.0))
def test_gomez_luna_identity(s, tau):
    g = st.gomez_luna_optimum(s, tau)
    assert g * g * tau == pytest.approx(s, rel=1e-12, abs=1e-15)


@settings(max_examples=200, deadline=None, derandomize=True)
@given(S.integers(1_000, 100_000_000), S.floats(min_value=0.05, max_value=20.0))
def test_recommend_scale_invariant_and_fp32_halves(n, k):
    base = st.recommend(PAPER, n)
    scaled = st.ModelBundle(*(k * v for v in (PAPER.sum_a, PAPER.sum_b, PAPER.small_a, PAPER.small_b,
                                              PAPER.small_c, PAPER.big_a, PAPER.big_b, PAPER.big_c)))
    assert st.recommend(scaled, n).chosen == base.chosen
    f32 = st.recommend_fp32(PAPER, n)
    assert f32 in (1, 2, 4, 8, 16, 32) and f32 == max(1, base.chosen // 2)
    qual = [b > 0 for b in base.benefits]
    assert (base.chosen == 1) == (not any(qual))


@settings(max_examples=200, deadline=None, derandomize=True)
@given(S.tuples(durations, durations, durations), durations, S.tuples(durations, durations, durations),
       counts, S.floats(min_value=0.0, max_value=0.1))
def test_simulator_bounds(s1, cpu, s3, n, tau):
    spec = st.PipelineSpec(stage1=s1, cpu_ms=cpu, stage3=s3, num_streams=n, tau_ms=tau)
    r = st.simulate(spec, trace=False)
    holds, dom = st.verify_lower_bound(spec)
    assert holds
    assert r.stage1_makespan_ms >= max(s1) - 1e-9 and r.stage3_makespan_ms >= max(s3) - 1e-9
    assert r.total_ms <= st.total_unstreamed(spec.timings()) + n * tau + 1e-6
