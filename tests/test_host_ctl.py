"""Host control plane of the library (libsdv2_ctl.so, no GPU) vs the oracle's control
plane: Appendix A trace, long-horizon replay, R2 schedule invariants, partition DP vs
brute force (SURVEY.md §8(c) pins P3, P6, P13)."""
import json
import os
import random

import numpy as np
import pytest

import synthgen as sg
from oracle import control as C
from paper_2511_07399_b200 import build
from paper_2511_07399_b200.sdv2 import HostControl, partition


@pytest.fixture(scope="module", autouse=True)
def _built():
    build.build()


def _oracle_lane_states(geom, T_reset, tau, hs):
    ctl = C.ControlPlane(geom, T_reset, tau)
    lane = C.LaneCache(geom.sink_chunks, geom.window_chunks, T_reset)
    out = []
    for X, h in enumerate(hs):
        act = ctl.admit(X, h)
        lane.apply(act, None, None, geom.chunk_frames)
        out.append((act, lane.state(), lane.evictions))
    return out


def _check_lane(st, ostate, oevict, S):
    tags = [st.tag[s] for s in range(S)]
    for s in range(S):
        if s in ostate:
            assert tags[s] == ostate[s][0]
            assert st.pos[s] == ostate[s][1][0]
        else:
            assert tags[s] == -1
    assert st.evictions == oevict
    assert st.num_valid == len(ostate)
    assert sorted(ostate) == list(range(len(ostate)))       # valid slots form a prefix


def test_appendix_a_trace_library(golden_dir):
    g = json.load(open(os.path.join(golden_dir, "appendixA_trace.json")))
    p = g["params"]
    hc = HostControl(p["T"], p["m"], p["W"], 1, 1, 0, p["T_reset"], p["tau"])
    for row in g["rows"]:
        hc.set_prompt_mean(p["h_before_6"] if row["X"] < 6 else p["h_from_6"], 0 if row["X"] < 6 else 1)
        na, ents, _ = hc.call()
        e = ents[0]
        assert e["X"] == row["X"] and e["pos"][0] == row["qpos"]
        assert bool(e["rebase"]) == row["rebase"]
        assert [bool(e["refresh_mask"] & 1)] == row["refresh"]
        st = hc.lane_state(0)
        assert [[st.tag[0], st.pos[0]]] == row["sinks"]
        ring = [[st.tag[1 + i], st.pos[1 + i]] if st.tag[1 + i] >= 0 else None for i in range(p["W"])]
        assert ring == row["ring"]
        assert st.evictions == row["evict"] and st.resets == row["r"]


@pytest.mark.parametrize("T,m,W,T_reset,n,K", [(1, 1, 4, 240, 4, 1), (1, 1, 4, 240, 4, 8), (2, 2, 3, 8, 2, 2),
                                               (1, 0, 2, 3, 1, 1), (3, 1, 2, 7, 3, 4)])
def test_long_replay_matches_oracle(T, m, W, T_reset, n, K):
    """10k-chunk metadata replay (configs[4]-style: resets, evictions, prompt switches)."""
    geom = sg.Geometry(8, 8, T, n, m, W)
    rng = np.random.default_rng(7)
    prompts = [rng.standard_normal(5) for _ in range(6)]
    N = 3000 if K > 1 else 10000
    sw = sorted(set(int(x) for x in rng.integers(1, N, size=5)))
    pidx = [sum(1 for s in sw if X >= s) for X in range(N)]
    hs = [prompts[pidx[X] % len(prompts)] for X in range(N)]
    ref = _oracle_lane_states(geom, T_reset, 0.95, hs)
    hc = HostControl(T, m, W, n, K, 0, T_reset, 0.95)
    S = m + W
    for c in range(N):
        hc.set_prompt_mean(hs[c], pidx[c])
        na, ents, oc = hc.call()
        # R2: active entries are the prefix j with c - jK >= 0
        assert na == sum(1 for j in range(n) if c - j * K >= 0)
        assert oc == (c - (n - 1) * K if c - (n - 1) * K >= 0 else -1)
        for j in range(n):
            X = c - j * K
            e = ents[j]
            assert e["active"] == (X >= 0)
            if X < 0:
                continue
            act = ref[X][0]
            assert e["X"] == X and e["pos"][:T] == act["pos"] and bool(e["rebase"]) == act["rebase"]
            assert e["pver"] == pidx[X]
            assert e["refresh_mask"] == sum(1 << i for i, r in enumerate(act["refresh"]) if r)
            if c % 97 == 0 or act["rebase"] or e["refresh_mask"]:
                _check_lane(hc.lane_state(j), ref[X][1], ref[X][2], S)


@pytest.mark.parametrize("n", [1, 2, 4])
@pytest.mark.parametrize("K", [1, 2, 4, 8])
def test_r2_schedule_invariants(n, K):
    """Appendix B check 1: dependencies met, lanes in chunk order, one clean chunk per
    stage-tick in steady state, first clean chunk at stage-tick nK - 1."""
    hc = HostControl(1, 1, 2, n, K, 0, 1000, 0.95)
    hc.set_prompt_mean([1.0], 0)
    done_at = {}        # (X, j) -> global tick its last stage finishes
    last_lane = [-1] * n
    outs = []
    for c in range(60):
        _, ents, oc = hc.call()
        # rank 0 runs call c at global tick c; the last stage at tick c + K - 1
        for e in ents:
            if not e["active"]:
                continue
            X, j = e["X"], e["j"]
            if j > 0:
                assert done_at[(X, j - 1)] < c          # predecessor left the last stage
            assert X == last_lane[j] + 1                # lane j sees chunks in order
            last_lane[j] = X
            done_at[(X, j)] = c + K - 1
        if oc >= 0:
            outs.append((c + K - 1, oc))
    assert outs[0] == (n * K - 1, 0)
    assert [o for _, o in outs] == list(range(len(outs)))
    assert [t for t, _ in outs] == list(range(n * K - 1, n * K - 1 + len(outs)))


def test_partition_examples_and_bruteforce(golden_dir):
    ex = json.load(open(os.path.join(golden_dir, "spec_examples.json")))["balance"]
    b, mx = partition([1.0] * 30, 4)
    assert [b[i + 1] - b[i] for i in range(4)] == ex[0]["expect_sizes"] and mx == ex[0]["expect_max"]
    _, mx = partition([3, 1, 1, 1, 3], 2)
    assert mx == ex[1]["expect_max"]
    _, mx = partition([1.0, 2.0, 3.0], 1, 0.5, 0.25)
    assert mx == pytest.approx(6.75)
    rnd = random.Random(0)
    for _ in range(300):
        B = rnd.randint(1, 12)
        K = rnd.randint(1, min(B, 5))
        costs = [rnd.choice([0.0, 1.0, 2.0, rnd.random() * 3]) for _ in range(B)]
        ef, el = rnd.random() * 2, rnd.random() * 2
        bounds, mx = partition(costs, K, ef, el)
        assert mx == pytest.approx(C.brute_force_partition(costs, K, ef, el), abs=1e-12)
        assert max(C.stage_times(costs, bounds, ef, el)) == pytest.approx(mx, abs=1e-12)
        assert bounds[0] == 0 and bounds[-1] == B and all(bounds[i] < bounds[i + 1] for i in range(K))
    with pytest.raises(Exception):
        partition([1.0, 1.0], 3)


@pytest.mark.parametrize("T,m,W,T_reset,n,K,B", [(1, 1, 4, 6, 2, 1, 3), (2, 2, 3, 8, 2, 2, 2), (1, 1, 2, 3, 1, 1, 8),
                                                 (1, 0, 2, 4, 4, 1, 4)])
def test_multi_stream_replay_matches_independent_oracles(T, m, W, T_reset, n, K, B):
    """B streams batched per call (SLO batch; "different colors denote distinct
    latent streams", Fig. parallel): entry e = j B + b of the library's call equals stream b's
    own oracle control plane at chunk c - jK (each stream has its own prompts, so its own
    sink refreshes and prompt versions), and lane e holds stream b's lane state."""
    geom = sg.Geometry(8, 8, T, n, m, W)
    rng = np.random.default_rng(11 + B)
    N = 400
    prompts = [rng.standard_normal(4) for _ in range(5)]
    hs, pidx, refs = [], [], []
    for b in range(B):
        sw = sorted(set(int(x) for x in rng.integers(1, N, size=4)))
        pi = [sum(1 for s in sw if X >= s) for X in range(N)]
        h = [prompts[(pi[X] + b) % len(prompts)] for X in range(N)]
        hs.append(h)
        pidx.append(pi)
        refs.append(_oracle_lane_states(geom, T_reset, 0.95, h))
    hc = HostControl(T, m, W, n, K, 0, T_reset, 0.95, B=B)
    S = m + W
    for c in range(N):
        for b in range(B):
            hc.set_prompt_mean(hs[b][c], pidx[b][c], stream=b)
        na, ents, oc = hc.call()
        assert na == B * sum(1 for j in range(n) if c - j * K >= 0)
        assert oc == (c - (n - 1) * K if c - (n - 1) * K >= 0 else -1)
        for j in range(n):
            X = c - j * K
            for b in range(B):
                e = ents[j * B + b]
                assert e["active"] == (X >= 0) and e["stream"] == b and e["j"] == j
                if X < 0:
                    continue
                act = refs[b][X][0]
                assert e["X"] == X and e["pos"][:T] == act["pos"] and bool(e["rebase"]) == act["rebase"]
                assert e["pver"] == pidx[b][X] and e["xslot"] == 2 * b + (pidx[b][X] & 1)
                assert e["refresh_mask"] == sum(1 << i for i, r in enumerate(act["refresh"]) if r)
                if c % 31 == 0 or act["rebase"] or e["refresh_mask"]:
                    _check_lane(hc.lane_state(j * B + b), refs[b][X][1], refs[b][X][2], S)
    with pytest.raises(Exception):
        HostControl(T, m, W, 8, K, 0, T_reset, 0.95, B=3)      # 24 entries > 16
