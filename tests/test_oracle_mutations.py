"""Mutation check of the closed-form pins (no GPU): each plausible misreading of an oracle
function (a dropped term, a swapped row, a wrong index law) is patched in and the pin
that guards that function must FAIL.  A pin that still passes under its mutation does
not pin anything."""
import numpy as np
import pytest

import test_oracle_closed_forms as T
from oracle import control as C
from oracle import model as M
from oracle import stream as S


def _time_embed_variant(t_scale=1000.0, silu1=True, silu2=True, transpose=False):
    def f(sigma, W, md, dt):
        emb = M.sinusoid(t_scale * float(sigma), md.freq_dim).astype(dt)
        h = M.linear(emb, W["t1_w"], W["t1_b"])
        e = M.linear(M.silu(h) if silu1 else h, W["t2_w"], W["t2_b"])
        e0 = M.linear(M.silu(e) if silu2 else e, W["tp_w"], W["tp_b"])
        return e, (e0.reshape(md.dim, 6).T if transpose else e0.reshape(6, md.dim))
    return f


def _sin_first(t, dim):
    half = dim // 2
    arg = float(t) * np.power(10000.0, -np.arange(half, dtype=np.float64) / half)
    return np.concatenate([np.sin(arg), np.cos(arg)])


def _rms_g_per_head(y, g, eps, hd=64):
    out = np.empty_like(y)
    for c in range(0, y.shape[-1], hd):
        out[..., c:c + hd] = M.rms_norm(y[..., c:c + hd], eps)
    return g * out


def _rope_angles_2i(hd, pt, ph, pw):
    ct, ch, cw = M.rope_split(hd)
    ws = [np.power(10000.0, -2.0 * np.arange(c, dtype=np.float64) / c) for c in (ct, ch, cw)]
    ps = [np.asarray(p, dtype=np.float64)[:, None] for p in (pt, ph, pw)]
    return np.concatenate([p * w[None] for p, w in zip(ps, ws)], axis=1)


def _rope_angles_shared(hd, pt, ph, pw):
    ct, ch, cw = M.rope_split(hd)
    w = np.power(10000.0, -np.arange(hd // 2, dtype=np.float64) / (hd // 2))
    pos = np.concatenate([np.repeat(np.asarray(p, np.float64)[:, None], c, 1) for p, c in ((pt, ct), (ph, ch), (pw, cw))], 1)
    return pos * w[None]


def _rope_angles_hwt(hd, pt, ph, pw):
    return M.rope_angles.__wrapped__(hd, ph, pw, pt) if hasattr(M.rope_angles, "__wrapped__") else _orig_rope(hd, ph, pw, pt)


_orig_rope = M.rope_angles


def _rope_apply_halves(x, phi):
    h = x.shape[1] // 2
    x0, x1 = x[:, :h].astype(np.float64), x[:, h:].astype(np.float64)
    c, s = np.cos(phi), np.sin(phi)
    return np.concatenate([x0 * c - x1 * s, x0 * s + x1 * c], axis=1).astype(x.dtype)


_orig_positions = M.token_positions


def _positions_swapped(md, geom, frame_pos):
    pt, ph, pw = _orig_positions(md, geom, frame_pos)
    return pt, pw, ph


def _positions_transposed_scan(md, geom, frame_pos):
    hn, wn = geom.latent_h // md.patch_h, geom.latent_w // md.patch_w
    pt, ph, pw = [], [], []
    for f in range(geom.chunk_frames // md.patch_t):
        for jj in range(wn):
            for i in range(hn):
                pt.append(frame_pos[f]); ph.append(i); pw.append(jj)
    return np.array(pt), np.array(ph), np.array(pw)


def _text_embed_no_gelu(P, W, dt):
    return M.linear(M.linear(P.astype(dt), W["txt1_w"], W["txt1_b"]), W["txt2_w"], W["txt2_b"])


def _prompt_kv_no_norm(ctx, W, b, md, dt):
    p = f"blocks.{b}."
    return (W[p + "gck"] * M.linear(ctx, W[p + "wck"], W[p + "bck"]),
            M.linear(ctx, W[p + "wcv"], W[p + "bcv"]))


def _head_swapped(x, e, W, md, dt):
    mod = W["head_mod"].astype(dt) + e[None, :]
    sc, sh = mod[0], mod[1]
    return M.linear(M.norm(x, md) * (1 + sc) + sh, W["head_w"], W["head_b"])


def _head_no_e(x, e, W, md, dt):
    mod = W["head_mod"].astype(dt)
    sh, sc = mod[0], mod[1]
    return M.linear(M.norm(x, md) * (1 + sc) + sh, W["head_w"], W["head_b"])


def _permuted_oracle(perm):
    class Mut(S.StreamOracle):
        def block(self, x, e0, b, lane, act):
            key = f"blocks.{b}.mod"
            orig = self.W[key]
            self.W = dict(self.W)
            self.W[key] = orig[perm]
            try:
                return super().block(x, e0[perm], b, lane, act)
            finally:
                self.W[key] = orig
    return Mut


class _NoRebaseLane(C.LaneCache):
    def apply(self, act, k, v, T):
        act = dict(act)
        act["rebase"] = False
        super().apply(act, k, v, T)


class _NoWrapControl(C.ControlPlane):
    def admit(self, X, h):
        act = super().admit(X, h)
        act["pos"] = [X * self.g.chunk_frames + f for f in range(self.g.chunk_frames)]
        return act


def _cross_variant(kind):
    """Oracle whose cross-attention sub-block is rebuilt with one misreading."""
    class Mut(S.StreamOracle):
        def block(self, x, e0, b, lane, act):
            Wt = self.W
            p = f"blocks.{b}."
            x1 = super().block(x, e0, b, lane, dict(act, ctx_kv={b: (np.zeros_like(act["ctx_kv"][b][0]),
                                                                  np.zeros_like(act["ctx_kv"][b][1]))}))
            # recompute the cross contribution with the misreading and add it back
            n3b = 0.0 if kind == "no_n3_bias" else Wt[p + "n3_b"]
            n3g = (1 + Wt[p + "n3_g"]) if kind == "one_plus_g" else Wt[p + "n3_g"]
            a3 = M.norm(x, self.md) * n3g + n3b
            qc = M.linear(a3, Wt[p + "wcq"], Wt[p + "bcq"])
            if kind != "no_q_rms":
                qc = M.rms_g(qc, Wt[p + "gcq"], self.md.eps)
            Kc, Vc = act["ctx_kv"][b]
            hd = self.md.head_dim
            oc = np.zeros_like(x)
            for hh in range(self.md.num_heads):
                cs = slice(hh * hd, (hh + 1) * hd)
                oc[:, cs] = M.attention(qc[:, cs], Kc[:, cs], Vc[:, cs])
            y = M.linear(oc, Wt[p + "wco"], Wt[p + "bco"])
            gate = (Wt[p + "mod"][0] + e0[0]) if kind == "gated" else 1.0
            # x1 already holds the zero-K/V cross term (uniform over zero V = b_co only)
            return x1 - Wt[p + "bco"] + gate * y
    return Mut


MUTATIONS = [
    # (pin, [(module, attribute, replacement)], what it models)
    ("pin_time_embed", [(M, "time_embed", _time_embed_variant(t_scale=1.0))], "timestep t = sigma"),
    ("pin_time_embed", [(M, "time_embed", _time_embed_variant(silu1=False))], "no SiLU before t2"),
    ("pin_time_embed", [(M, "time_embed", _time_embed_variant(silu2=False))], "no SiLU before tp"),
    ("pin_time_embed", [(M, "time_embed", _time_embed_variant(transpose=True))], "e0 viewed [d, 6]"),
    ("pin_time_embed", [(M, "sinusoid", _sin_first)], "sin before cos"),
    ("pin_text_embed_and_prompt_kv", [(M, "text_embed", _text_embed_no_gelu)], "no GELU in text MLP"),
    ("pin_text_embed_and_prompt_kv", [(M, "prompt_kv", _prompt_kv_no_norm)], "no RMS on cross K"),
    ("pin_text_embed_and_prompt_kv", [(M, "rms_g", _rms_g_per_head)], "cross-K RMS per head"),
    ("pin_rms_g_full_dim", [(M, "rms_g", _rms_g_per_head)], "qk-norm per head"),
    ("pin_rope_frequency_law", [(M, "rope_angles", _rope_angles_2i)], "omega = 10000^(-2i/c)"),
    ("pin_rope_frequency_law", [(M, "rope_angles", _rope_angles_shared)], "one omega law over all pairs"),
    ("pin_rope_frequency_law", [(M, "rope_angles", _rope_angles_hwt)], "groups ordered (h, w, t)"),
    ("pin_rope_frequency_law", [(M, "rope_apply", _rope_apply_halves)], "rotate halves, not pairs"),
    ("pin_token_positions", [(M, "token_positions", _positions_swapped)], "height/width swapped"),
    ("pin_token_positions", [(M, "token_positions", _positions_transposed_scan)], "column-major scan"),
    ("pin_block_wiring", [(T, "StreamOracle", _permuted_oracle([1, 0, 2, 3, 4, 5]))], "sh1 <-> sc1"),
    ("pin_block_wiring", [(T, "StreamOracle", _permuted_oracle([0, 1, 5, 3, 4, 2]))], "g1 <-> g2"),
    ("pin_block_wiring", [(T, "StreamOracle", _permuted_oracle([3, 4, 2, 0, 1, 5]))], "msa <-> mlp shift/scale"),
    ("pin_block_wiring", [(M, "gelu_tanh", lambda z: z / (1 + np.exp(-1.702 * z)))], "sigmoid GELU"),
    ("pin_block_wiring", [(M, "norm", lambda x, md: M.layer_norm(x, md.eps))], "LayerNorm for RMSNorm"),
    ("pin_cross_wiring", [(T, "StreamOracle", _cross_variant("no_n3_bias"))], "norm3 without shift"),
    ("pin_cross_wiring", [(T, "StreamOracle", _cross_variant("one_plus_g"))], "norm3 scale 1 + g"),
    ("pin_cross_wiring", [(T, "StreamOracle", _cross_variant("no_q_rms"))], "cross q without RMS"),
    ("pin_cross_wiring", [(T, "StreamOracle", _cross_variant("gated"))], "gated cross residual"),
    ("pin_head", [(M, "head", _head_swapped)], "head sh <-> sc"),
    ("pin_head", [(M, "head", _head_no_e)], "head ignores e"),
    ("pin_reset_invariance", [(S, "LaneCache", _NoRebaseLane)], "window keys not re-based"),
    ("pin_reset_invariance", [(S, "ControlPlane", _NoWrapControl)], "query positions not reset"),
]


@pytest.mark.parametrize("pin,patches,what", MUTATIONS, ids=[m[2] for m in MUTATIONS])
def test_pin_catches_mutation(monkeypatch, pin, patches, what):
    for mod, attr, rep in patches:
        monkeypatch.setattr(mod, attr, rep)
    with pytest.raises(AssertionError):
        getattr(T, pin)()


def test_cross_variant_reproduces_oracle():
    """The mutation harness with no misreading reproduces the oracle (so its failures are the
    misreadings', not the harness's)."""
    import numpy as _np
    Mut = _cross_variant("none")
    orig = T.StreamOracle
    try:
        T.StreamOracle = Mut
        T.pin_cross_wiring()
    finally:
        T.StreamOracle = orig


def test_pins_pass_unmutated():
    for pin in sorted({m[0] for m in MUTATIONS}):
        getattr(T, pin)()
