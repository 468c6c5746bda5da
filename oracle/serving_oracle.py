"""CPU oracle of the two-stage serving path — TEST INFRASTRUCTURE ONLY (tests/ and bench.py's
c4 CPU baseline); never imported by the product package.

A batched float64 restatement of ``longrec.serving`` (the reference, pure Python/NumPy):

* ``build_cache`` ≙ ``build_cache`` (pkg/src/longrec/serving.py:84-144): the candidate-free part
  of the forward — per layer the key / value rows of every row but the target (the cross layer's
  merged rows + the m-1 non-target globals, each self layer's k sequence queries + m-1 globals),
  the target's visibility row (non-pad keys, every global, itself), the last layer's CLS row and
  the user-side head features;
* ``score`` ≙ ``score_with_cache`` (serving.py:147-167) with ``attention_block_cached``
  (pkg/src/longrec/attention.py:215-236): only the target row runs through the blocks, against
  the cached rows with its own key and value appended last.

Pinned by tests/test_serving_oracle.py against tests/golden/serving_*.npz, which
make_serving_golden.py produced with the reference's own build_cache / score_with_cache.
"""
from __future__ import annotations

import math

import numpy as np

from . import longer_oracle as O


def build_cache(P, cfg, users):
    """users: batch dict in the C-ABI layout (dt measured from each user's scoring time)."""
    B = len(users["uid"])
    b = dict(users)
    b["cand_item"] = np.zeros(B, dtype=np.int64)          # any candidate: its row is dropped
    _, c = O.forward(P, cfg, b)
    k, m, G = cfg.k, cfg.m, cfg.merged_len
    layers = [(c["c_cross"]["Kh"][:, :, :-1], c["c_cross"]["Vh"][:, :, :-1])]
    layers += [(cs["Kh"][:, :, :-1], cs["Vh"][:, :, :-1]) for cs in c["c_self"]]
    npg = c["npg"]
    qg = c["qg"]
    kpad = np.arange(G)[None, :] < npg[:, None]                               # [B, G]
    qpad = O.query_pad(cfg, npg, qg)                                          # [B, k]
    ones = np.ones((B, m - 1 + 1), dtype=bool)                                # globals + own key
    vis_cross = np.concatenate([~kpad, ones], axis=1)                         # [B, G + m]
    vis_self = np.concatenate([~qpad, ones], axis=1)                          # [B, k + m]
    u_d = np.concatenate([P["tables.uid_table"][c["uid"]], P["tables.profile_table"][c["prof"]]], axis=-1)
    return dict(layers=layers, vis_cross=vis_cross, vis_self=vis_self, cls=c["layers"][-1][:, k + 1],
                u_d=u_d)


def _cached_block(P, pre, g, Kc, Vc, vis, heads):
    """attention_block_cached for [U, C, D] target rows; Kc / Vc [U, H, n, dh]."""
    U, C, D = g.shape
    dh = D // heads
    qn, _ = O.ln_fwd(g, P[pre + "ln1_g"], P[pre + "ln1_b"])
    q = O.lin(qn, P[pre + "w_q"], P[pre + "b_q"]).reshape(U, C, heads, dh).transpose(0, 2, 1, 3)
    ko = O.lin(qn, P[pre + "w_k"], P[pre + "b_k"]).reshape(U, C, heads, dh).transpose(0, 2, 1, 3)
    vo = O.lin(qn, P[pre + "w_v"], P[pre + "b_v"]).reshape(U, C, heads, dh).transpose(0, 2, 1, 3)
    scale = 1.0 / math.sqrt(dh)
    s_c = (q * scale) @ Kc.transpose(0, 1, 3, 2)                             # [U, H, C, n]
    s_o = np.sum(q * scale * ko, axis=-1, keepdims=True)                     # [U, H, C, 1]
    s = np.concatenate([s_c, s_o], axis=-1)
    p = O.masked_softmax_fwd(s, vis[:, None, None, :])
    ctx = p[..., :-1] @ Vc + p[..., -1:] * vo                                # [U, H, C, dh]
    ctx = ctx.transpose(0, 2, 1, 3).reshape(U, C, D)
    x1 = g + O.lin(ctx, P[pre + "w_o"], P[pre + "b_o"])
    x1n, _ = O.ln_fwd(x1, P[pre + "ln2_g"], P[pre + "ln2_b"])
    f1 = O.lin(x1n, P[pre + "w1"], P[pre + "b1"])
    gf, _ = O.gelu_fwd(f1)
    return x1 + O.lin(gf, P[pre + "w2"], P[pre + "b2"])


def score(P, cfg, cache, cand):
    """cand [U, C] candidate items (timestamp = the cache's scoring time) → p [U, C]."""
    cand = np.asarray(cand, dtype=np.int64)
    U, C = cand.shape
    tfeat = np.concatenate([P["tables.item_table"][cand], np.zeros((U, C, cfg.d_act)),
                            np.broadcast_to(P["tables.time_bucket_table"][0], (U, C, cfg.d_time))], axis=-1)
    td = O.lin(tfeat, P["tables.mlp.tok_proj_w"], P["tables.mlp.tok_proj_b"])
    g = O.lin(td, P["tables.mlp.lift_w"], P["tables.mlp.lift_b"])
    ga = O.lin(g, P["tables.mlp.glob_w1"], P["tables.mlp.glob_b1"])
    gg, _ = O.gelu_fwd(ga)
    g = O.lin(gg, P["tables.mlp.glob_w2"], P["tables.mlp.glob_b2"])
    Kc, Vc = cache["layers"][0]
    g = _cached_block(P, "cross.", g, Kc, Vc, cache["vis_cross"], cfg.heads)
    for i in range(cfg.N):
        Kc, Vc = cache["layers"][1 + i]
        g = _cached_block(P, f"self.{i}.", g, Kc, Vc, cache["vis_self"], cfg.heads)
    cl = np.broadcast_to(cache["cls"][:, None, :], g.shape)
    ud = np.broadcast_to(cache["u_d"][:, None, :], (U, C, cache["u_d"].shape[-1]))
    hin = np.concatenate([g, cl, g * cl, g * g, ud], axis=-1)
    z1 = O.lin(hin, P["head.w1"], P["head.b1"])
    hg, _ = O.gelu_fwd(z1)
    z = O.lin(hg, P["head.w2"], P["head.b2"])[..., 0]
    return O.sigmoid(z)
