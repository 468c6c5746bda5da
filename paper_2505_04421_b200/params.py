"""Parameter inventory and initialisation, bit-identical to the reference.

Names, shapes and order follow ``LongRecModel.params()`` (``pkg/src/longrec/model.py:252-263``,
``inputs.py:340-390``, ``attention.py:131-137``).  :func:`init_params` replays the reference's
single ``default_rng(seed)`` stream in the reference's draw order
(``EmbeddingTables.create`` → inner blocks → cross → self blocks → query bank → head,
``model.py:185-207``) and then applies the identity-biased init (``model.py:209-245``), so
``LongerModel(cfg, seed)`` starts from exactly the weights ``LongRecModel(cfg, seed)`` has.
"""
from __future__ import annotations

import math
from collections import OrderedDict

import numpy as np

from .config import ModelConfig

BLOCK_ORDER = ("w_q", "b_q", "w_k", "b_k", "w_v", "b_v", "w_o", "b_o",
               "w1", "b1", "w2", "b2", "ln1_g", "ln1_b", "ln2_g", "ln2_b")
MLP_ORDER = ("tok_proj_w", "tok_proj_b", "seq_w1", "seq_b1", "seq_w2", "seq_b2",
             "lift_w", "lift_b", "glob_w1", "glob_b1", "glob_w2", "glob_b2")

_QK_GAIN = 1.5
_WO_SCALE_CROSS = 0.3
_WO_SCALE_SELF = 0.1
_FFN_OUT_DAMP = 0.05
_SIDE_EMB_STD = 0.05
_HEAD_DAMP = 0.05
_HEAD_PRIME_IN = 0.5
_HEAD_PRIME_OUT = 0.15


def block_shapes(w: int):
    return OrderedDict([("w_q", (w, w)), ("b_q", (w,)), ("w_k", (w, w)), ("b_k", (w,)),
                        ("w_v", (w, w)), ("b_v", (w,)), ("w_o", (w, w)), ("b_o", (w,)),
                        ("w1", (w, 4 * w)), ("b1", (4 * w,)), ("w2", (4 * w, w)), ("b2", (w,)),
                        ("ln1_g", (w,)), ("ln1_b", (w,)), ("ln2_g", (w,)), ("ln2_b", (w,))])


def param_shapes(cfg: ModelConfig) -> "OrderedDict[str, tuple]":
    d, D, F = cfg.d, cfg.D, cfg.feat_width
    out = OrderedDict()
    out["tables.item_table"] = (cfg.vocab, cfg.d_item)
    out["tables.action_table"] = (cfg.n_actions, cfg.d_act)
    out["tables.time_bucket_table"] = (cfg.n_time_buckets, cfg.d_time)
    out["tables.uid_table"] = (cfg.n_users, d)
    out["tables.profile_table"] = (cfg.n_profiles, d)
    out["tables.abs_pos_table"] = (cfg.L, d)
    out["tables.cls_vector"] = (cfg.m - 2, D)
    mlp = {"tok_proj_w": (F, d), "tok_proj_b": (d,), "seq_w1": (d, 2 * D), "seq_b1": (2 * D,),
           "seq_w2": (2 * D, d), "seq_b2": (d,), "lift_w": (d, D), "lift_b": (D,),
           "glob_w1": (D, 2 * D), "glob_b1": (2 * D,), "glob_w2": (2 * D, D), "glob_b2": (D,)}
    for n in MLP_ORDER:
        out[f"tables.mlp.{n}"] = mlp[n]
    if cfg.merge_mode == "inner":
        for i in range(cfg.inner_layers):
            for n, s in block_shapes(d).items():
                out[f"inner.{i}.{n}"] = s
    for n, s in block_shapes(D).items():
        out[f"cross.{n}"] = s
    for i in range(cfg.N):
        for n, s in block_shapes(D).items():
            out[f"self.{i}.{n}"] = s
    if cfg.query_strategy == "learnable":
        out["query_bank"] = (cfg.k, D)
    h_in = 4 * D + 2 * d
    out["head.w1"] = (h_in, cfg.head_hidden)
    out["head.b1"] = (cfg.head_hidden,)
    out["head.w2"] = (cfg.head_hidden, 1)
    out["head.b2"] = (1,)
    return out


def _block_init(rng, w: int, prefix: str, out: dict) -> None:
    """``BlockParams.create`` draw order (attention.py:112-129)."""
    def wt(fi, fo):
        return rng.normal(0.0, 1.0 / math.sqrt(fi), size=(fi, fo))
    out[prefix + "w_q"] = wt(w, w); out[prefix + "b_q"] = np.zeros(w)
    out[prefix + "w_k"] = wt(w, w); out[prefix + "b_k"] = np.zeros(w)
    out[prefix + "w_v"] = wt(w, w); out[prefix + "b_v"] = np.zeros(w)
    out[prefix + "w_o"] = wt(w, w); out[prefix + "b_o"] = np.zeros(w)
    out[prefix + "w1"] = wt(w, 4 * w); out[prefix + "b1"] = np.zeros(4 * w)
    out[prefix + "w2"] = wt(4 * w, w); out[prefix + "b2"] = np.zeros(w)
    out[prefix + "ln1_g"] = np.ones(w); out[prefix + "ln1_b"] = np.zeros(w)
    out[prefix + "ln2_g"] = np.ones(w); out[prefix + "ln2_b"] = np.zeros(w)


def _identity_mlp(P, w1, b1, w2, b2, width):
    for n in (w1, b1, w2, b2):
        P[n][...] = 0.0
    for i in range(width):
        P[w1][i, i] = 1.0
        P[w1][i, width + i] = -1.0
        P[w2][i, i] = 1.0
        P[w2][width + i, i] = -1.0


def init_params(cfg: ModelConfig, seed: int = 0) -> "OrderedDict[str, np.ndarray]":
    cfg.validate()
    rng = np.random.default_rng(seed)
    d, D, F = cfg.d, cfg.D, cfg.feat_width
    P = {}
    emb = lambda r, c: rng.normal(0.0, 0.3, size=(r, c))
    wt = lambda fi, fo: rng.normal(0.0, 1.0 / np.sqrt(fi), size=(fi, fo))
    # EmbeddingTables.create (inputs.py:372-382), then InputMLP.create (inputs.py:336-346)
    P["tables.item_table"] = emb(cfg.vocab, cfg.d_item)
    P["tables.action_table"] = emb(cfg.n_actions, cfg.d_act)
    P["tables.time_bucket_table"] = emb(cfg.n_time_buckets, cfg.d_time)
    P["tables.uid_table"] = emb(cfg.n_users, d)
    P["tables.profile_table"] = emb(cfg.n_profiles, d)
    P["tables.abs_pos_table"] = emb(cfg.L, d)
    P["tables.cls_vector"] = emb(cfg.m - 2, D)
    P["tables.mlp.tok_proj_w"] = wt(F, d); P["tables.mlp.tok_proj_b"] = np.zeros(d)
    P["tables.mlp.seq_w1"] = wt(d, 2 * D); P["tables.mlp.seq_b1"] = np.zeros(2 * D)
    P["tables.mlp.seq_w2"] = wt(2 * D, d); P["tables.mlp.seq_b2"] = np.zeros(d)
    P["tables.mlp.lift_w"] = wt(d, D); P["tables.mlp.lift_b"] = np.zeros(D)
    P["tables.mlp.glob_w1"] = wt(D, 2 * D); P["tables.mlp.glob_b1"] = np.zeros(2 * D)
    P["tables.mlp.glob_w2"] = wt(2 * D, D); P["tables.mlp.glob_b2"] = np.zeros(D)
    if cfg.merge_mode == "inner":
        for i in range(cfg.inner_layers):
            _block_init(rng, d, f"inner.{i}.", P)
    _block_init(rng, D, "cross.", P)
    for i in range(cfg.N):
        _block_init(rng, D, f"self.{i}.", P)
    if cfg.query_strategy == "learnable":
        P["query_bank"] = rng.normal(0.0, 0.3, size=(cfg.k, D))
    h_in = 4 * D + 2 * d
    P["head.w1"] = rng.normal(0.0, 1.0 / math.sqrt(h_in), size=(h_in, cfg.head_hidden))
    P["head.b1"] = np.zeros(cfg.head_hidden)
    P["head.w2"] = rng.normal(0.0, 1.0 / math.sqrt(cfg.head_hidden), size=(cfg.head_hidden, 1))
    P["head.b2"] = np.zeros(1)

    # _identity_biased_init (model.py:209-245)
    for name in ("tables.item_table", "tables.cls_vector"):
        norms = np.linalg.norm(P[name], axis=1, keepdims=True)
        P[name] /= np.maximum(norms, 1e-12)
    for name in ("tables.action_table", "tables.time_bucket_table", "tables.abs_pos_table"):
        P[name] *= _SIDE_EMB_STD / 0.3
    P["tables.mlp.tok_proj_w"] *= 0.1
    for i in range(min(cfg.d_item, d)):
        P["tables.mlp.tok_proj_w"][i, i] = 1.0
    _identity_mlp(P, "tables.mlp.seq_w1", "tables.mlp.seq_b1", "tables.mlp.seq_w2", "tables.mlp.seq_b2", d)
    _identity_mlp(P, "tables.mlp.glob_w1", "tables.mlp.glob_b1", "tables.mlp.glob_w2", "tables.mlp.glob_b2", D)
    P["tables.mlp.lift_w"] *= 0.1
    for s in range(cfg.K):
        for i in range(d):
            P["tables.mlp.lift_w"][i, s * d + i] = 1.0
    for pre in ["cross."] + [f"self.{i}." for i in range(cfg.N)]:
        wq = P[pre + "w_q"]
        P[pre + "w_k"] = wq * _QK_GAIN
        P[pre + "w_q"] = wq * _QK_GAIN
        P[pre + "w_v"] = np.eye(D)
        scale = _WO_SCALE_CROSS if pre == "cross." else _WO_SCALE_SELF
        P[pre + "w_o"] = np.eye(D) * scale
        P[pre + "w2"] = P[pre + "w2"] * _FFN_OUT_DAMP
    P["head.w1"] *= _HEAD_DAMP
    P["head.w2"] *= _HEAD_DAMP
    readers = ((2 * D, 0, 1.0), (2 * D, 1, -1.0), (3 * D, 2, 1.0), (3 * D, 3, -1.0))
    for offset, col, sign in readers:
        if col >= cfg.head_hidden:
            break
        for j in range(D):
            P["head.w1"][offset + j, col] += sign * _HEAD_PRIME_IN
        P["head.w2"][col, 0] = sign * _HEAD_PRIME_OUT
    shapes = param_shapes(cfg)
    out = OrderedDict()
    for n, s in shapes.items():
        a = np.asarray(P[n], dtype=np.float64)
        assert a.shape == tuple(s), (n, a.shape, s)
        out[n] = a
    return out


def count_params(cfg: ModelConfig) -> int:
    return int(sum(int(np.prod(s)) for s in param_shapes(cfg).values()))
