"""Visual chunk embedding for the sink refresh ("given a new chunk
embedding h_t"): the library's host helper vs the oracle's definition, and the control plane
driven by per-chunk visual embeddings vs the oracle control plane (no GPU)."""
import numpy as np
import pytest

import synthgen as sg
from oracle import control as C
from paper_2511_07399_b200 import build
from paper_2511_07399_b200.sdv2 import HostControl, chunk_embedding, ctl_lib


@pytest.fixture(scope="module", autouse=True)
def _built():
    build.build()


def test_chunk_embedding_closed_form_and_oracle():
    v = np.zeros((4, 2, 8, 8), np.float32)
    for c in range(4):
        v[c] = c - 1.5                                     # constant channel -> its value
    assert np.array_equal(chunk_embedding(v), np.array([-1.5, -0.5, 0.5, 1.5]))
    r = np.random.default_rng(0).standard_normal((16, 1, 60, 104)).astype(np.float32)
    assert chunk_embedding(r) == pytest.approx(C.visual_embedding(r), rel=1e-12, abs=1e-15)


def _scene_chunks(n, cut):
    a = sg.LatentStream(4, 8, 8, seed=1, speeds=(0.0,))      # a static scene (noise only) ...
    b = sg.LatentStream(4, 8, 8, seed=9, speeds=(0.0,))      # ... cut to another one
    return [(a if X < cut else b).chunk(X, 1) + (0.0 if X < cut else 0.7) for X in range(n)]


def test_visual_refresh_matches_oracle():
    """Scene cut at chunk 9: the visual embedding of the new scene is far from the sinks,
    which are refreshed; before the cut the static scene keeps them."""
    geom = sg.Geometry(8, 8, 1, 2, 2, 3)
    chunks = _scene_chunks(20, 9)
    ctl = C.ControlPlane(geom, 6, 0.9)
    hc = HostControl(1, 2, 3, 2, 1, 0, 6, 0.9)
    refreshed = []
    for X, v in enumerate(chunks):
        h = C.visual_embedding(v)
        act = ctl.admit(X, h)
        emb = np.ascontiguousarray(chunk_embedding(v))
        import ctypes
        assert hc.L.sdv2ctl_set_chunk_embedding(ctypes.c_void_p(hc.h), 0,
                                                emb.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), emb.size) == 0
        na, ents, _ = hc.call()
        e = ents[0]
        assert e["refresh_mask"] == sum(1 << i for i, r in enumerate(act["refresh"]) if r), X
        refreshed.append(e["refresh_mask"])
    assert refreshed[9] == 3 and not any(refreshed[2:9]) and not any(refreshed[10:])
