"""SLO-aware batching scheduler:
the library's host scheduler vs the exhaustive-search / AIMD oracle (oracle/slo.py), the
SPEC worked examples, and the oracle's own pins (no GPU)."""
import random

import pytest

from oracle import slo as O
from paper_2511_07399_b200 import build
from paper_2511_07399_b200.sdv2 import SDV2Error, SloAdapter, slo_fit, slo_select


@pytest.fixture(scope="module", autouse=True)
def _built():
    build.build()


def _table(rnd, Ts=(1, 2, 4), Bs=(1, 2, 3, 4, 6, 8)):
    """Latency grows with B T (memory-bound model of P:178) plus noise; sometimes a knee."""
    a, b = rnd.uniform(0.002, 0.02), rnd.uniform(0.0005, 0.01)
    knee = rnd.choice([None, 4, 8])
    tab = {}
    for t in Ts:
        for bb in Bs:
            if rnd.random() < 0.2:
                continue
            x = bb * t
            lat = a + b * x + (0.0 if knee is None or x <= knee else 3 * b * (x - knee))
            tab[(t, bb)] = round(lat * rnd.uniform(0.9, 1.1), 6)
    tab.setdefault((1, 1), a + b)
    return tab


def test_select_matches_exhaustive_oracle_200_fixtures():
    rnd = random.Random(0)
    for _ in range(200):
        tab = _table(rnd)
        f_slo = rnd.choice([4.0, 8.0, 16.0, 30.0, 60.0])
        dl = rnd.choice([1.0 / f_slo, 2.0 / f_slo, 0.5 / f_slo])
        buf = rnd.randint(1, 40)
        bmax = rnd.randint(1, 8)
        exp = O.select_batch(tab, f_slo, dl, buf, bmax)
        got = slo_select(tab, f_slo, dl, buf, bmax)
        assert (got["T"], got["B"], got["feasible"]) == (exp["T"], exp["B"], exp["feasible"]), (tab, f_slo, buf, bmax)
        assert got["fps"] == pytest.approx(exp["fps"], rel=1e-12)
        assert got["B"] * got["T"] <= buf                       # P:177 invariant


def test_select_examples():
    # monotone throughput, loose SLO -> B = min(b_max, buffered / T)  (SPEC S:133 example 1)
    tab = {(1, b): 0.01 + 0.001 * b for b in range(1, 9)}
    assert slo_select(tab, 1.0, 10.0, 5, 8)["B"] == 5
    assert slo_select(tab, 1.0, 10.0, 40, 6)["B"] == 6
    # buffered = 7 latent frames, T = 4 -> B = 1
    tab4 = {(4, b): 0.05 * b for b in range(1, 5)}
    d = slo_select(tab4, 1.0, 10.0, 7, 4)
    assert d["B"] == 1 and d["T"] == 4
    # not enough input -> error
    with pytest.raises(SDV2Error):
        slo_select(tab4, 1.0, 10.0, 3, 4)
    # infeasible SLO is reported, not relaxed
    d = slo_select(tab, 1e6, 10.0, 8, 8)
    assert not d["feasible"] and d["B"] == 1
    # the knee: past it, latency grows faster than B and throughput drops
    knee = {(1, b): 0.01 * (1 if b <= 4 else (b - 3)) for b in range(1, 9)}
    assert slo_select(knee, 1.0, 10.0, 16, 8)["B"] == 4


def test_adapt_examples_and_oracle():
    # violation with B = 8 -> 4; compliant streak at 4 -> 5; B = 1 violating stays 1, infeasible
    a = SloAdapter(8, 1, 8, 3, 16.0, 1.0 / 16)
    assert a.adapt(1.0)["B"] == 4
    for _ in range(2):
        assert a.adapt(0.01)["B"] == 4
    assert a.adapt(0.01)["B"] == 5
    one = SloAdapter(1, 1, 8, 3, 16.0, 1.0 / 16)
    r = one.adapt(1.0)
    assert r["B"] == 1 and r["infeasible"]
    # random histories: library == oracle step by step, never B < 1 or > b_max
    rnd = random.Random(1)
    for _ in range(50):
        bmax, streak, T = rnd.randint(1, 8), rnd.randint(1, 5), rnd.choice([1, 2, 4])
        f, dl = rnd.choice([8.0, 16.0]), rnd.choice([1 / 8, 1 / 16])
        lib_a = SloAdapter(bmax, T, bmax, streak, f, dl)
        ora = O.AimdState(bmax, T, bmax, streak)
        for _ in range(60):
            lat = rnd.uniform(0.05, 1.5) * 4 * T / f
            g, e = lib_a.adapt(lat), ora.adapt(lat, f, dl)
            assert g == e and 1 <= g["B"] <= bmax


def test_adapt_converges_under_constant_latency_model():
    """with latency L(B) = a + b B and an SLO the knee B* satisfies, AIMD settles
    into the cycle B* <-> B*+1 (the +1 probe violates and halves back) within b_max +
    streak b_max iterations; it never leaves [1, b_max]."""
    a_, b_ = 0.01, 0.01
    f = 4.0 * 1 / (a_ + b_ * 4.5)          # B = 4 meets f, B = 5 does not
    ad = SloAdapter(1, 1, 8, 2, f, 10.0)
    seen = []
    for _ in range(8 + 2 * 8 + 20):
        B = ad.st.streams
        seen.append(B)
        ad.adapt(a_ + b_ * B)
    assert max(seen[-10:]) <= 5 and 4 in seen[-10:]


def test_latency_model_fit():
    tab = {(t, b): 0.004 + 0.0025 * b * t for t in (1, 2) for b in (1, 2, 4)}
    a, b = slo_fit(tab)
    assert a == pytest.approx(0.004, abs=1e-12) and b == pytest.approx(0.0025, abs=1e-12)
    assert O.fit_latency_model(tab) == pytest.approx((a, b), abs=1e-12)


def test_oracle_pins():
    """The oracle's own closed forms: a single feasible point is chosen; equal throughput
    ties go to the smaller B; the AIMD sequence of SPEC S:143-145 by hand."""
    assert O.select_batch({(1, 1): 0.1}, 1.0, 1.0, 1, 1)["B"] == 1
    tie = {(1, 2): 0.02, (1, 4): 0.04}            # both 100 frames/s per ... 4*2/0.02 == 4*4/0.04
    assert O.select_batch(tie, 1.0, 10.0, 8, 8)["B"] == 2
    s = O.AimdState(8, 1, 8, 2)
    assert [s.adapt(x, 16.0, 1 / 16)["B"] for x in (1.0, 0.01, 0.01, 1.0, 0.01)] == [4, 4, 5, 2, 2]
