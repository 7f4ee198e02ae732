"""CPU tests of the simulator, the ModelBundle document
(SPEC.md:316), the report harness and the `streamtune` CLI.

The simulator is checked three ways: against the SPEC's worked examples,
against the closed-form stage makespan (h+c+d)/n + (n-1)max/n,
and against an independent event-by-event pipeline enumeration written here
in Python (a checker only).  Acceptance criterion 5: 10^4 random
specs satisfy simulate.total >= Eq. 2 - 1e-9, with equality to 1e-12 in the
dominance regime.
"""
import json
import random
import subprocess
from pathlib import Path

import pytest

from paper_2501_05938_b200 import errors
from paper_2501_05938_b200 import streamtune as st

ROOT = Path(__file__).resolve().parents[1]
CLI = ROOT / "paper_2501_05938_b200" / "bin" / "streamtune"
PAPER = st.ModelBundle.paper()


def enumerate_pipeline(stage, n):
    """Independent checker: per-engine serial, per-chunk FIFO H2D->COMP->D2H."""
    free = [0.0, 0.0, 0.0]
    end = 0.0
    for _ in range(n):
        ready = 0.0
        for e in range(3):
            start = max(free[e], ready)
            free[e] = ready = start + stage[e] / n
        end = max(end, ready)
    return end


def test_simulate_spec_examples():
    r = st.simulate(st.PipelineSpec(stage1=(4, 2, 1), num_streams=4))
    assert r.stage1_makespan_ms == pytest.approx(4.75, abs=1e-12)
    assert r.total_ms == pytest.approx(4.75, abs=1e-12)
    # n = 1, tau = 0: Eq. 1
    spec = st.PipelineSpec(stage1=(1.0, 2.0, 3.0), cpu_ms=0.5, stage3=(0.25, 1.5, 2.0))
    assert st.simulate(spec).total_ms == pytest.approx(st.total_unstreamed(spec.timings()), abs=1e-12)
    # n = 1 with tau: Eq. 1 + tau, and the bound holds with equality
    spec.tau_ms = 0.01
    r = st.simulate(spec)
    assert r.total_ms == pytest.approx(st.total_unstreamed(spec.timings()) + 0.01, abs=1e-12)
    assert st.verify_lower_bound(spec)[0]


def test_simulate_trace_invariants():
    spec = st.PipelineSpec(stage1=(3.0, 1.0, 2.0), cpu_ms=0.7, stage3=(0.5, 2.5, 1.5), num_streams=8,
                           tau_ms=0.004448)
    r = st.simulate(spec)
    assert len(r.trace) == 6 * 8
    for eng in st.ENGINES:
        for stage in (1, 3):
            iv = sorted((a, b) for (e, s, g, a, b) in r.trace if e == eng and g == stage)
            # engine exclusivity
            assert all(iv[k][1] <= iv[k + 1][0] + 1e-12 for k in range(len(iv) - 1))
            # chunk conservation
            comp = {"h2d": 0, "comp": 1, "d2h": 2}[eng]
            total = (spec.stage1 if stage == 1 else spec.stage3)[comp]
            assert sum(b - a for a, b in iv) == pytest.approx(total, rel=1e-12)
    for s in range(8):  # per-stream order H2D -> COMP -> D2H
        for stage in (1, 3):
            ev = {e: (a, b) for (e, ss, g, a, b) in r.trace if ss == s and g == stage}
            assert ev["h2d"][1] <= ev["comp"][0] + 1e-12 and ev["comp"][1] <= ev["d2h"][0] + 1e-12
    # stage 3 starts after stage 1, the CPU stage and stream creation
    s3_start = min(a for (e, s, g, a, b) in r.trace if g == 3)
    assert s3_start == pytest.approx(8 * spec.tau_ms + r.stage1_makespan_ms + spec.cpu_ms, rel=1e-12)


def test_simulate_matches_enumeration_and_closed_form():
    rng = random.Random(7)
    for _ in range(300):
        s1 = tuple(rng.uniform(0, 5) for _ in range(3))
        s3 = tuple(rng.uniform(0, 5) for _ in range(3))
        n = rng.choice([1, 2, 4, 8, 16, 32])
        r = st.simulate(st.PipelineSpec(stage1=s1, cpu_ms=1.0, stage3=s3, num_streams=n), trace=False)
        for got, stage in ((r.stage1_makespan_ms, s1), (r.stage3_makespan_ms, s3)):
            assert got == pytest.approx(enumerate_pipeline(stage, n), rel=1e-12, abs=1e-12)
            closed = sum(stage) / n + (n - 1) * max(stage) / n
            assert got == pytest.approx(closed, rel=1e-12, abs=1e-12)


def test_lower_bound_criterion_5():
    """SPEC criterion 5: 10^4 random specs."""
    rng = random.Random(42)
    strict_seen = False
    for k in range(10_000):
        s1 = [rng.uniform(0, 10) for _ in range(3)]
        s3 = [rng.uniform(0, 10) for _ in range(3)]
        dominant = k % 2 == 0
        if dominant:  # stage-1 max is H2D, stage-3 max is D2H
            s1[0] = max(s1) + rng.uniform(0, 1)
            s3[2] = max(s3) + rng.uniform(0, 1)
        n = rng.choice([1, 2, 4, 8, 16, 32])
        spec = st.PipelineSpec(stage1=tuple(s1), cpu_ms=rng.uniform(0, 3), stage3=tuple(s3), num_streams=n,
                               tau_ms=rng.uniform(0, 0.01))
        holds, dom = st.verify_lower_bound(spec)
        assert holds
        assert dom == (dominant or (s1[0] >= max(s1) and s3[2] >= max(s3)))
        if dominant:
            r = st.simulate(spec, trace=False)
            bound = st.streamed_lower_bound(spec.timings(), n, n * spec.tau_ms)
            assert r.total_ms == pytest.approx(bound, rel=1e-12)
        elif n > 1 and not dom:
            r = st.simulate(spec, trace=False)
            bound = st.streamed_lower_bound(spec.timings(), n, n * spec.tau_ms)
            strict_seen |= r.total_ms > bound + 1e-9
    assert strict_seen  # outside the dominance regime the bound is strict for some n


def test_makespan_monotone_in_n():
    stage = (2.0, 3.0, 1.0)
    prev = float("inf")
    for n in (1, 2, 4, 8, 16, 32):
        r = st.simulate(st.PipelineSpec(stage1=stage, num_streams=n), trace=False)
        assert r.stage1_makespan_ms <= prev + 1e-12
        assert r.stage1_makespan_ms >= max(stage) - 1e-12
        prev = r.stage1_makespan_ms


def test_hw_queue_serialisation():
    # fewer hardware queues than streams: streams sharing a queue serialise
    free = st.simulate(st.PipelineSpec(stage1=(4, 4, 4), num_streams=8), trace=False)
    one = st.simulate(st.PipelineSpec(stage1=(4, 4, 4), num_streams=8, hw_queues=1), trace=False)
    assert one.stage1_makespan_ms == pytest.approx(12.0)
    assert free.stage1_makespan_ms == pytest.approx(12 / 8 + 7 * 4 / 8)


def test_simulate_validation():
    with pytest.raises(errors.InvalidStreamCountError):
        st.simulate(st.PipelineSpec(num_streams=3))
    with pytest.raises(errors.NegativeDurationError):
        st.simulate(st.PipelineSpec(stage1=(-1.0, 0.0, 0.0)))


# ---- ModelBundle document ------------------------------------------------------------
def test_bundle_document_round_trip():
    for b in (PAPER, st.ModelBundle.b200()):
        doc = st.bundle_to_json(b)
        d = json.loads(doc)
        assert set(d) >= {"sum", "overhead_small", "overhead_big", "size_threshold", "candidates"}
        back = st.bundle_from_json(doc)
        for f in ("sum_a", "sum_b", "small_a", "small_b", "small_c", "big_a", "big_b", "big_c"):
            assert getattr(back, f) == getattr(b, f)  # bit-exact (17 digits)
        assert back.candidates == b.candidates and back.size_threshold == b.size_threshold
    # the Python mirror's document (repr strings) loads in C++
    back = st.bundle_from_json(json.dumps(PAPER.to_document()))
    assert back.sum_a == PAPER.sum_a and back.big_c == PAPER.big_c


@pytest.mark.parametrize("doc", [
    "{}", "not json", '{"sum": {"a": 1}}',
    '{"sum": {"a": 1, "b": 2}, "overhead_small": {"a": 0, "b": 0, "c": 0}, '
    '"overhead_big": {"a": 0, "b": 0, "c": "x"}}',
    '{"sum": {"a": 1, "b": 2}, "overhead_small": {"a": 0, "b": 0, "c": 0}, '
    '"overhead_big": {"a": 0, "b": 0, "c": 0}, "candidates": [2, 3]}',
])
def test_bundle_document_malformed(doc):
    with pytest.raises(errors.ValidationError):
        st.bundle_from_json(doc)


# ---- report harness ----------------------------------------------------------------------
def test_report_tables_paper_bundle():
    t1 = st.report_table(PAPER, "table1")
    assert t1["failed"] == 0 and t1["passed"] == 10
    t2 = st.report_table(PAPER, "table2")
    assert t2["failed"] == 0 and t2["passed"] == 11
    t4 = st.report_table(PAPER, "table4")
    assert (t4["passed"], t4["failed"], t4["known"]) == (24, 0, 1)  # 8e4: SURVEY.md App. B.1
    t5 = st.report_table(PAPER, "table5")
    assert t5["failed"] == 0
    # the halving rule on Table 5's own FP64 column: every "half" row passes,
    # the 9 "same" rows are the paper's documented deviations
    rule = [c for i, c in enumerate(t5["cells"]) if i % 2 == 0]
    assert sum(c[3] == "KNOWN" for c in rule) == 9
    with pytest.raises(errors.ValidationError):
        st.report_table(PAPER, "table3")


def test_report_detects_perturbed_bundle():
    bad = st.ModelBundle(**{**PAPER.__dict__, "sum_b": PAPER.sum_b + 1.0})
    assert st.report_table(bad, "table4")["failed"] > 0


def test_dump_reference():
    t2 = st.dump_reference("table2").strip().splitlines()
    assert t2[0] == "num_streams,t_str,t_non_str,sum,overhead,benefit"
    assert t2[3].startswith("8,7.401472,8.81744,2.433568,0.713404,1.415968")
    assert len(st.dump_reference("table4").strip().splitlines()) == 26
    assert float(st.dump_reference("tau").split()[1]) == 0.004448


# ---- the CLI --------------------------------------------------------------------------------
def run(*args):
    assert CLI.exists(), "streamtune CLI not built (build.py build_cli)"
    p = subprocess.run([str(CLI), *map(str, args)], capture_output=True, text=True, timeout=60)
    return p.returncode, p.stdout, p.stderr


def test_cli_predict_and_report():
    rc, out, _ = run("predict", "--model", "paper", "--sizes", "1000,100000,500000,1000000", "--json")
    assert rc == 0
    got = [p["chosen"] for p in json.loads(out)["predictions"]]
    assert got == [1, 2, 4, 8]
    rc, out, _ = run("predict", "--model", "paper", "--sizes", "1e6", "--precision", "fp32", "--json")
    assert rc == 0 and json.loads(out)["predictions"][0]["chosen"] == 4
    rc, out, _ = run("report", "--model", "paper", "--reference", "table2", "--json")
    assert rc == 0 and json.loads(out)["failed"] == 0
    rc, _, _ = run("report", "--model", "paper", "--reference", "table4")
    assert rc == 0


def test_cli_fit_then_predict(tmp_path):
    # noiseless forward-generated dataset (SPEC cmd_fit example): coefficients recovered
    sa, sb = 2.0e-6, 0.15
    sm = (1.0e-7, 0.6, 0.05)
    bg = (2.0e-8, 0.03, 0.2)
    sizes = [1000, 4000, 10000, 40000, 100000, 400000, 1000000, 2500000, 5000000, 10000000, 40000000,
             80000000]
    import math
    stage = ["slae_size,t1_h2d,t1_comp,t1_d2h,t2_comp,t3_h2d,t3_comp,t3_d2h"]
    runs = ["slae_size,num_streams,t_str"]
    for N in sizes:
        s = sa * N + sb
        t_non = 3 * s  # t1_h2d = s, overlap fields sum to s, t3_d2h = s
        stage.append(f"{N},{s!r},{s / 4!r},{s / 4!r},0,{s / 4!r},{s / 4!r},{s!r}")
        runs.append(f"{N},1,{t_non!r}")
        for n in (2, 4, 8, 16, 32):
            if N <= 1000000:
                ovh = sm[0] * N + sm[1] * math.log10(n) + sm[2]
            else:
                ovh = (bg[0] * N + bg[1]) * (4 / 3) * math.log2(n) + bg[2]
            t_str = t_non - (n - 1) / n * s + ovh
            runs.append(f"{N},{n},{t_str!r}")
    (tmp_path / "stage.csv").write_text("\n".join(stage) + "\n")
    (tmp_path / "runs.csv").write_text("\n".join(runs) + "\n")
    model = tmp_path / "model.json"
    rc, out, err = run("fit", "--stage-csv", tmp_path / "stage.csv", "--runs-csv", tmp_path / "runs.csv",
                       "--out", model)
    assert rc == 0, err
    b = st.bundle_from_json(model.read_text())
    assert b.sum_a == pytest.approx(sa, rel=1e-9) and b.sum_b == pytest.approx(sb, rel=1e-9)
    assert (b.small_a, b.small_b, b.small_c) == pytest.approx(sm, rel=1e-8)
    assert (b.big_a, b.big_b, b.big_c) == pytest.approx(bg, rel=1e-8)
    rc, out, _ = run("predict", "--model", model, "--sizes", "1000000", "--json")
    assert rc == 0
    assert json.loads(out)["predictions"][0]["chosen"] == st.recommend(b, 10**6).chosen
    # only n = 1 runs -> no overhead observations -> exit 2
    (tmp_path / "runs1.csv").write_text("\n".join(r for r in runs if r.count(",1,") or r.startswith("slae"))
                                         + "\n")
    rc, _, err = run("fit", "--stage-csv", tmp_path / "stage.csv", "--runs-csv", tmp_path / "runs1.csv")
    assert rc == 2, err
    rc, _, err = run("fit", "--stage-csv", tmp_path / "missing.csv", "--runs-csv", tmp_path / "runs.csv")
    assert rc == 1 and "missing.csv" in err


def test_cli_baseline_and_simulate(tmp_path):
    rows = ["slae_size,t1_h2d,t1_comp,t1_d2h,t2_comp,t3_h2d,t3_comp,t3_d2h"]
    rows.append("4000,0.1,0.221312,0.014848,0.01,0.006592,0.030688,0.1")
    rows.append("40000000,50,17.4515,38.8368,1,9.60672,20.9816,20")
    (tmp_path / "s.csv").write_text("\n".join(rows) + "\n")
    rc, out, _ = run("baseline", "--stage-csv", tmp_path / "s.csv", "--tau", "0.004448", "--json")
    assert rc == 0
    gl = [r["gomez_luna"] for r in json.loads(out)["rows"]]
    assert gl == pytest.approx([7.8, 139.8], abs=0.05)
    rc, _, _ = run("baseline", "--stage-csv", tmp_path / "s.csv", "--tau", "0")
    assert rc == 2
    (tmp_path / "empty.csv").write_text(rows[0] + "\n")
    rc, _, _ = run("baseline", "--stage-csv", tmp_path / "empty.csv", "--tau", "0.004448")
    assert rc == 0
    rc, out, _ = run("simulate", "--h2d1", 4, "--comp1", 2, "--d2h1", 1, "--streams", 4, "--json",
                     "--trace", tmp_path / "t.csv")
    assert rc == 0
    d = json.loads(out)
    assert d["total_ms"] == pytest.approx(4.75) and d["lower_bound_holds"] and d["dominance"]
    assert (tmp_path / "t.csv").read_text().splitlines()[0] == "engine,stream,start_ms,end_ms"
    rc, _, _ = run("simulate", "--streams", 3)
    assert rc == 1
    rc, out, _ = run("dump-reference", "--reference", "table1")
    assert rc == 0 and out.startswith("slae_size,")
    rc, _, _ = run("bogus")
    assert rc == 1


def test_reference_data_checksums():
    """the embedded ReferenceData (Tables 1, 2, 4, 5 and tau of
    /root/reference/PAPER.md, transcribed in csrc/streamtune/dataset.cpp) is
    pinned by checksums taken at transcription time (the values themselves
    are cross-checked against PAPER.md literals in test_streamtune.py)."""
    import hashlib

    pinned = {
        "table1": "5ae56b65daaf9b0bb856aaf6ff9f98cdca761061f5eca26d992f66d32c15aa61",
        "table2": "c8e38d21a1bcabf83590a4c285e50d8933e5b8d187f6aa887d5d8c10b05b019d",
        "table4": "bc5a47d50445b9aade880334c68f8a340c1c5d3d8f67246c47f3ef9dcc6c43b8",
        "table5": "2f360de02e62f49496a95ef74354e1505b49831ff5fbb8f7ccfb27f52438b53c",
        "tau": "75bbd116ec994e2656babefec8c787a2361b9d15944f266b947801a5678e5c27",
    }
    for table, digest in pinned.items():
        assert hashlib.sha256(st.dump_reference(table).encode()).hexdigest() == digest, table
    t5 = st.dump_reference("table5").strip().splitlines()[1:]
    assert len(t5) == 17 and sum(r.endswith(",half") for r in t5) == 7  # "7 out of 16"
