"""Online DiT-block scheduler: the
library policy (sdv2_rebalance) vs the brute-force oracle (oracle/balance.py), the SPEC
examples and invariants (no GPU)."""
import random

import pytest

from oracle import balance as OB
from oracle import control as C
from paper_2511_07399_b200 import build
from paper_2511_07399_b200.sdv2 import rebalance


@pytest.fixture(scope="module", autouse=True)
def _built():
    build.build()


def _uniform(nb, K):
    q, r = divmod(nb, K)
    b = [0]
    for s in range(K):
        b.append(b[-1] + q + (1 if s < r else 0))
    return b


def test_matches_oracle_random():
    rnd = random.Random(3)
    for _ in range(300):
        nb = rnd.randint(2, 14)
        K = rnd.randint(1, min(nb, 5))
        cur = _uniform(nb, K)
        ema_l = [0.0] * nb
        ema_o = [0.0] * nb
        for step in range(4):
            meas = [rnd.choice([1.0, 1.0, 2.0, rnd.random() * 3]) for _ in range(nb)]
            ef, el = rnd.random(), rnd.random()
            a, hy = rnd.choice([0.3, 0.5, 1.0]), rnd.choice([0.0, 0.05, 0.2])
            nbd, ch, pc, pn = rebalance(meas, K, cur, ema_l, ef, el, a, hy)
            ema_o, och, opc, opn = OB.rebalance_online(meas, K, cur, ema_o, ef, el, a, hy)
            assert ema_l == pytest.approx(ema_o, abs=1e-12)
            assert ch == och and pc == pytest.approx(opc, abs=1e-12) and pn == pytest.approx(opn, abs=1e-12)
            assert pn <= pc + 1e-12                                       # never worse
            assert max(C.stage_times(ema_l, nbd, ef, el)) == pytest.approx(pn, abs=1e-12)
            assert nbd[0] == 0 and nbd[-1] == nb and all(nbd[i] < nbd[i + 1] for i in range(K))
            if not ch:
                assert nbd == cur
            cur = nbd


def test_spec_examples():
    # measured == previous profile -> unchanged (already optimal uniform split of equal blocks)
    ema = [0.0] * 8
    b, ch, _, _ = rebalance([1.0] * 8, 2, [0, 4, 8], ema)
    assert not ch and b == [0, 4, 8]
    b, ch, _, _ = rebalance([1.0] * 8, 2, [0, 4, 8], ema)
    assert not ch and b == [0, 4, 8]
    # doubled cost on one middle block -> its stage shrinks by >= 1 block (improvement > hysteresis)
    ema = [0.0] * 9
    meas = [1.0] * 9
    meas[4] = 3.0
    b, ch, pc, pn = rebalance(meas, 3, [0, 3, 6, 9], ema, alpha=1.0, hysteresis=0.05)
    assert ch and (b[2] - b[1]) < 3 and pn < pc
    # improvement below hysteresis -> unchanged
    ema = [0.0] * 9
    b, ch, pc, pn = rebalance(meas, 3, [0, 3, 6, 9], ema, alpha=1.0, hysteresis=0.5)
    assert not ch and b == [0, 3, 6, 9] and pn == pc
    # VAE-like endpoint extras move blocks off the first and last stages
    ema = [0.0] * 12
    b, ch, _, _ = rebalance([1.0] * 12, 3, [0, 4, 8, 12], ema, extra_first=3.0, extra_last=3.0, alpha=1.0)
    assert ch and b[1] - b[0] < 4 and b[3] - b[2] < 4 and b[2] - b[1] > 4


def test_ema_smooths_spikes():
    """One noisy sample does not flip the partition when alpha is small."""
    ema = [0.0] * 6
    b, ch, _, _ = rebalance([1.0] * 6, 2, [0, 3, 6], ema, alpha=0.2, hysteresis=0.05)
    spike = [1.0] * 6
    spike[0] = 2.0
    b, ch, _, _ = rebalance(spike, 2, [0, 3, 6], ema, alpha=0.2, hysteresis=0.1)
    assert not ch and ema[0] == pytest.approx(1.2)
