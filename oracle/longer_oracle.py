"""CPU oracle — TEST INFRASTRUCTURE ONLY.

A float64 NumPy restatement of the reference LONGER encoder (``longrec``, the pure-Python
package under ``/root/reference/pkg``), batched over samples, with a hand-derived backward
pass.  It is the parity checker for the sm_100a path and the CPU arm of ``bench.py``; it is
never imported by the product package (``paper_2505_04421_b200``), which fails loudly
without its CUDA library.

Parity pin: ``tests/test_oracle.py`` checks this module against golden vectors produced by
running the reference itself (``tests/golden/make_golden.py`` imports ``longrec`` from
``/root/reference/pkg/src``): per-sample probabilities, batch-mean BCE and every parameter
gradient, to 1e-9.

Batch layout (shared with the product's host code): token arrays are ``[B, L]``,
right-aligned like ``encode_events`` (``pkg/src/longrec/inputs.py:457-482``) — sample b's
``n_b`` real events occupy columns ``L-n_b .. L-1`` — plus per-sample ``uid``, ``profile``,
``cand_item`` and ``label``.  ``dt`` holds ``candidate_ts - event_ts`` (non-negative).
Parameters are a dict keyed by the reference ``LongRecModel.params()`` names
(``pkg/src/longrec/model.py:252-263``).
"""
from __future__ import annotations

import math

import numpy as np

GELU_C = math.sqrt(2.0 / math.pi)   # pkg/src/longrec/tensors.py:36
GELU_A = 0.044715                   # pkg/src/longrec/tensors.py:37
PROB_EPS = 1e-12                    # pkg/src/longrec/tensors.py:38
LN_EPS = 1e-12                      # pkg/src/longrec/tensors.py:39


# ----------------------------------------------------------------- elementwise pieces

def time_bucket(dt, n_buckets):
    """``min(bit_length(dt), n_buckets-1)`` (pkg/src/longrec/inputs.py:307-315), exact for int64."""
    dt = np.asarray(dt, dtype=np.int64)
    if (dt < 0).any():
        raise ValueError("future event: negative time delta")
    bl = np.zeros(dt.shape, dtype=np.int64)
    for i in range(63):
        bl += (dt >= (np.int64(1) << np.int64(i)))
    return np.minimum(bl, n_buckets - 1)


def gelu_fwd(x):
    """tanh-GELU (pkg/src/longrec/tensors.py:292-304); returns (y, t) with t kept for bw."""
    t = np.tanh(GELU_C * (x + GELU_A * x ** 3))
    return 0.5 * x * (1.0 + t), t


def gelu_bwd(dy, x, t):
    du = GELU_C * (1.0 + 3.0 * GELU_A * x ** 2)
    return dy * (0.5 * (1.0 + t) + 0.5 * x * (1.0 - t ** 2) * du)


def sigmoid(z):
    """Two-branch stable sigmoid (pkg/src/longrec/tensors.py:307-317)."""
    e = np.exp(-np.abs(z))
    return np.where(z >= 0, 1.0 / (1.0 + e), e / (1.0 + e))


def ln_fwd(x, g, b):
    """Row layer norm, biased variance, eps 1e-12 (pkg/src/longrec/tensors.py:354-381)."""
    mu = x.mean(axis=-1, keepdims=True)
    var = ((x - mu) ** 2).mean(axis=-1, keepdims=True)
    inv = 1.0 / np.sqrt(var + LN_EPS)
    xhat = (x - mu) * inv
    return xhat * g + b, (xhat, inv)


def ln_bwd(dy, g, saved):
    xhat, inv = saved
    ghat = dy * g
    m1 = ghat.mean(axis=-1, keepdims=True)
    m2 = (ghat * xhat).mean(axis=-1, keepdims=True)
    dx = (ghat - m1 - xhat * m2) * inv
    w = dy.shape[-1]
    return dx, (dy * xhat).reshape(-1, w).sum(0), dy.reshape(-1, w).sum(0)


def lin(x, W, b):
    return x @ W + b


def lin_bwd(dy, x, W, grads, wname, bname):
    """y = x·W + b (pkg/src/longrec/tensors.py:209-228,387-388): accumulate dW, db; return dx."""
    fin, fout = W.shape
    _acc(grads, wname, x.reshape(-1, fin).T @ dy.reshape(-1, fout))
    if bname is not None:
        _acc(grads, bname, dy.reshape(-1, fout).sum(0))
    return dy @ W.T


def _acc(grads, name, value):
    if name in grads:
        grads[name] = grads[name] + value
    else:
        grads[name] = np.array(value, dtype=np.float64)


def masked_softmax_fwd(s, vis):
    """Interpreted-mask softmax; masked → exactly 0; fully masked row → zeros
    (pkg/src/longrec/tensors.py:323-351)."""
    z = np.where(vis, s, -np.inf)
    rowmax = z.max(axis=-1, keepdims=True)
    rowmax = np.where(np.isfinite(rowmax), rowmax, 0.0)
    e = np.exp(np.where(vis, s - rowmax, 0.0)) * vis
    tot = e.sum(axis=-1, keepdims=True)
    return np.divide(e, tot, out=np.zeros_like(e), where=tot > 0)


def masked_softmax_bwd(dp, p):
    return p * (dp - (dp * p).sum(axis=-1, keepdims=True))


# ----------------------------------------------------------------- masks

def group_pad_counts(cfg, n_events):
    """Number of all-pad merged groups per sample (pkg/src/longrec/merge.py:45-62):
    left padding makes them a prefix, ``(L_padded - n) // K``."""
    n = np.minimum(np.asarray(n_events, dtype=np.int64), cfg.L)
    return (cfg.L_padded - n) // cfg.K


def recent_query_groups(cfg):
    """``select_queries(strategy="recent")`` (pkg/src/longrec/model.py:58-123): pad groups are a
    prefix, so the k most recent groups are always G-k .. G-1 (pad ones become pad queries)."""
    G = cfg.merged_len
    return np.arange(G - cfg.k, G)


def _ceil_div(a, b):
    return -(-a // b)


def query_groups(cfg, npg):
    """Merged-group index of every sequence query, [B, k] (``select_queries``,
    pkg/src/longrec/model.py:58-123, all four strategies).  Pad groups are the prefix
    0..npg-1; a chosen pad group is a pad query.  For "learnable" every row is a bank vector at
    the top grid position (returned as G-1) and is never pad."""
    G, k = cfg.merged_len, cfg.k
    B = npg.shape[0]
    out = np.zeros((B, k), dtype=np.int64)
    for b in range(B):
        fv = int(npg[b])
        nonpad = np.arange(fv, G)
        n_m = nonpad.size
        if cfg.query_strategy == "learnable":
            out[b] = G - 1
            continue
        if n_m <= k:
            fill = k - n_m
            chosen = list(range(fv - fill, fv)) + list(nonpad)
        elif cfg.query_strategy == "recent":
            chosen = list(nonpad[-k:])
        elif cfg.query_strategy == "uniform":
            chosen = [int(nonpad[_ceil_div((j + 1) * n_m, k) - 1]) for j in range(k)]
        elif cfg.query_strategy == "recent_uniform":
            r = _ceil_div(k, 2)
            u = k - r
            picked = set(int(i) for i in nonpad[-r:])
            prefix = nonpad[:n_m - r]
            plen = prefix.size
            for j in range(u):
                picked.add(int(prefix[_ceil_div((j + 1) * plen, u) - 1]))
            for idx in reversed(nonpad):
                if len(picked) >= k:
                    break
                picked.add(int(idx))
            chosen = sorted(picked)
        else:
            raise NotImplementedError(cfg.query_strategy)
        out[b] = np.sort(np.asarray(chosen, dtype=np.int64))
    return out


def query_pad(cfg, npg, qg):
    """[B, k] pad flags of the sequence queries (never for "learnable")."""
    if cfg.query_strategy == "learnable":
        return np.zeros(qg.shape, dtype=bool)
    return qg < npg[:, None]


def cross_mask(cfg, npg, qg=None):
    """Visibility of the first layer, [B, q, v] (pkg/src/longrec/attention.py:49-87 with the
    metadata of pkg/src/longrec/model.py:275-293)."""
    G, k, m = cfg.merged_len, cfg.k, cfg.m
    B = npg.shape[0]
    if qg is None:
        qg = np.broadcast_to(recent_query_groups(cfg), (B, k))
    keyg = np.arange(G)
    vis = np.zeros((B, k + m, G + m), dtype=bool)
    nonpad_key = keyg[None, :] >= npg[:, None]                      # [B, G]
    qpad = query_pad(cfg, npg, qg)                                  # [B, k]
    seq = nonpad_key[:, None, :] & (keyg[None, None, :] <= qg[:, :, None]) & ~qpad[:, :, None]
    vis[:, :k, :G] = seq
    vis[:, k:, :G] = nonpad_key[:, None, :]
    r = np.arange(m)
    vis[:, k:, G:] = (r[None, :] <= r[:, None])[None]
    return vis


def self_mask(cfg, npg, qg=None):
    """Visibility among the q retained rows, [B, q, q] (positions of the sequence queries are their
    groups; equal positions see each other, as for the "learnable" bank)."""
    k, m = cfg.k, cfg.m
    B = npg.shape[0]
    if qg is None:
        qg = np.broadcast_to(recent_query_groups(cfg), (B, k))
    qpad = query_pad(cfg, npg, qg)                                  # [B, k]
    vis = np.zeros((B, k + m, k + m), dtype=bool)
    seq = (qg[:, None, :] <= qg[:, :, None]) & ~qpad[:, None, :] & ~qpad[:, :, None]
    vis[:, :k, :k] = seq
    vis[:, k:, :k] = ~qpad[:, None, :]
    r = np.arange(m)
    vis[:, k:, k:] = (r[None, :] <= r[:, None])[None]
    return vis


# ----------------------------------------------------------------- attention block

def block_fwd(P, pre, xq, xkv, vis, heads, self_attn):
    """Pre-norm block (pkg/src/longrec/attention.py:172-212): LN1 on both sources (one shared
    LN for self-attention), Q/K/V, masked MHA with scale 1/sqrt(D/heads), W_o + residual,
    LN2 → FFN(4x, GELU) + residual."""
    c = {}
    qn, c["ln1q"] = ln_fwd(xq, P[pre + "ln1_g"], P[pre + "ln1_b"])
    if self_attn:
        kn = qn
    else:
        kn, c["ln1k"] = ln_fwd(xkv, P[pre + "ln1_g"], P[pre + "ln1_b"])
    Q = lin(qn, P[pre + "w_q"], P[pre + "b_q"])
    K = lin(kn, P[pre + "w_k"], P[pre + "b_k"])
    V = lin(kn, P[pre + "w_v"], P[pre + "b_v"])
    B, nq, D = Q.shape
    nk = K.shape[1]
    dh = D // heads
    scale = 1.0 / math.sqrt(dh)
    Qh = Q.reshape(B, nq, heads, dh).transpose(0, 2, 1, 3)
    Kh = K.reshape(B, nk, heads, dh).transpose(0, 2, 1, 3)
    Vh = V.reshape(B, nk, heads, dh).transpose(0, 2, 1, 3)
    S = (Qh * scale) @ Kh.transpose(0, 1, 3, 2)
    Pm = masked_softmax_fwd(S, vis[:, None])
    ctx = (Pm @ Vh).transpose(0, 2, 1, 3).reshape(B, nq, D)
    x1 = xq + lin(ctx, P[pre + "w_o"], P[pre + "b_o"])
    x1n, c["ln2"] = ln_fwd(x1, P[pre + "ln2_g"], P[pre + "ln2_b"])
    f1 = lin(x1n, P[pre + "w1"], P[pre + "b1"])
    gf, tf = gelu_fwd(f1)
    out = x1 + lin(gf, P[pre + "w2"], P[pre + "b2"])
    c.update(qn=qn, kn=kn, Qh=Qh, Kh=Kh, Vh=Vh, P=Pm, ctx=ctx, x1n=x1n, f1=f1, gf=gf, tf=tf,
             scale=scale, heads=heads, self_attn=self_attn)
    return out, c


def block_bwd(P, pre, dout, c, grads):
    """Returns (d x_q, d x_kv) — for self-attention d x_kv is already folded into d x_q."""
    dx1 = dout.copy()
    dgf = lin_bwd(dout, c["gf"], P[pre + "w2"], grads, pre + "w2", pre + "b2")
    df1 = gelu_bwd(dgf, c["f1"], c["tf"])
    dx1n = lin_bwd(df1, c["x1n"], P[pre + "w1"], grads, pre + "w1", pre + "b1")
    d, dg, db = ln_bwd(dx1n, P[pre + "ln2_g"], c["ln2"])
    _acc(grads, pre + "ln2_g", dg)
    _acc(grads, pre + "ln2_b", db)
    dx1 = dx1 + d
    dxq = dx1.copy()
    dctx = lin_bwd(dx1, c["ctx"], P[pre + "w_o"], grads, pre + "w_o", pre + "b_o")
    B, nq, D = dctx.shape
    heads = c["heads"]
    dh = D // heads
    dctxh = dctx.reshape(B, nq, heads, dh).transpose(0, 2, 1, 3)
    Pm, Qh, Kh, Vh = c["P"], c["Qh"], c["Kh"], c["Vh"]
    dVh = Pm.transpose(0, 1, 3, 2) @ dctxh
    dP = dctxh @ Vh.transpose(0, 1, 3, 2)
    dS = masked_softmax_bwd(dP, Pm)
    dQh = c["scale"] * (dS @ Kh)
    dKh = c["scale"] * (dS.transpose(0, 1, 3, 2) @ Qh)
    nk = Kh.shape[2]
    dQ = dQh.transpose(0, 2, 1, 3).reshape(B, nq, D)
    dK = dKh.transpose(0, 2, 1, 3).reshape(B, nk, D)
    dV = dVh.transpose(0, 2, 1, 3).reshape(B, nk, D)
    dqn = lin_bwd(dQ, c["qn"], P[pre + "w_q"], grads, pre + "w_q", pre + "b_q")
    dkn = lin_bwd(dK, c["kn"], P[pre + "w_k"], grads, pre + "w_k", pre + "b_k")
    dkn = dkn + lin_bwd(dV, c["kn"], P[pre + "w_v"], grads, pre + "w_v", pre + "b_v")
    if c["self_attn"]:
        d, dg, db = ln_bwd(dqn + dkn, P[pre + "ln1_g"], c["ln1q"])
        _acc(grads, pre + "ln1_g", dg)
        _acc(grads, pre + "ln1_b", db)
        return dxq + d, None
    d, dg, db = ln_bwd(dqn, P[pre + "ln1_g"], c["ln1q"])
    _acc(grads, pre + "ln1_g", dg)
    _acc(grads, pre + "ln1_b", db)
    dkv, dg, db = ln_bwd(dkn, P[pre + "ln1_g"], c["ln1k"])
    _acc(grads, pre + "ln1_g", dg)
    _acc(grads, pre + "ln1_b", db)
    return dxq + d, dkv


# ----------------------------------------------------------------- InnerTrans merge

def inner_fwd(P, cfg, h, npg):
    """merge_inner_trans (pkg/src/longrec/merge.py:83-112) with grouped_attention
    (pkg/src/longrec/tensors.py:406-444): full attention inside each K-group at width d."""
    B, Lp, d = h.shape
    K, G = cfg.K, cfg.merged_len
    x = h
    caches = []
    for i in range(cfg.inner_layers):
        pre = f"inner.{i}."
        c = {"x_in": x}
        xn, c["ln1"] = ln_fwd(x, P[pre + "ln1_g"], P[pre + "ln1_b"])
        q = lin(xn, P[pre + "w_q"], P[pre + "b_q"]).reshape(B, G, K, d)
        kk = lin(xn, P[pre + "w_k"], P[pre + "b_k"]).reshape(B, G, K, d)
        v = lin(xn, P[pre + "w_v"], P[pre + "b_v"]).reshape(B, G, K, d)
        scale = 1.0 / math.sqrt(d)
        s = np.einsum("bgqd,bgkd->bgqk", q, kk) * scale
        s = s - s.max(axis=-1, keepdims=True)
        e = np.exp(s)
        p = e / e.sum(axis=-1, keepdims=True)
        ctx = np.einsum("bgqk,bgkd->bgqd", p, v).reshape(B, Lp, d)
        x1 = x + lin(ctx, P[pre + "w_o"], P[pre + "b_o"])
        x1n, c["ln2"] = ln_fwd(x1, P[pre + "ln2_g"], P[pre + "ln2_b"])
        f1 = lin(x1n, P[pre + "w1"], P[pre + "b1"])
        gf, tf = gelu_fwd(f1)
        x = x1 + lin(gf, P[pre + "w2"], P[pre + "b2"])
        c.update(xn=xn, q=q, k=kk, v=v, p=p, ctx=ctx, x1n=x1n, f1=f1, gf=gf, tf=tf, scale=scale)
        caches.append(c)
    keep = (np.arange(G)[None, :] >= npg[:, None]).astype(np.float64)       # all-pad groups → 0
    keep_tok = np.repeat(keep, K, axis=1)[:, :, None]
    return x * keep_tok, (caches, keep_tok)


def inner_bwd(P, cfg, dx, cache, grads):
    caches, keep_tok = cache
    dx = dx * keep_tok
    B, Lp, d = dx.shape
    K, G = cfg.K, cfg.merged_len
    for i in reversed(range(cfg.inner_layers)):
        pre = f"inner.{i}."
        c = caches[i]
        dgf = lin_bwd(dx, c["gf"], P[pre + "w2"], grads, pre + "w2", pre + "b2")
        df1 = gelu_bwd(dgf, c["f1"], c["tf"])
        dx1n = lin_bwd(df1, c["x1n"], P[pre + "w1"], grads, pre + "w1", pre + "b1")
        d1, dg, db = ln_bwd(dx1n, P[pre + "ln2_g"], c["ln2"])
        _acc(grads, pre + "ln2_g", dg)
        _acc(grads, pre + "ln2_b", db)
        dx1 = dx + d1
        dctx = lin_bwd(dx1, c["ctx"], P[pre + "w_o"], grads, pre + "w_o", pre + "b_o")
        g3 = dctx.reshape(B, G, K, d)
        p = c["p"]
        dv = np.einsum("bgqk,bgqd->bgkd", p, g3).reshape(B, Lp, d)
        dp = np.einsum("bgqd,bgkd->bgqk", g3, c["v"])
        ds = (dp - (dp * p).sum(axis=-1, keepdims=True)) * p * c["scale"]
        dq = np.einsum("bgqk,bgkd->bgqd", ds, c["k"]).reshape(B, Lp, d)
        dk = np.einsum("bgqk,bgqd->bgkd", ds, c["q"]).reshape(B, Lp, d)
        dxn = lin_bwd(dq, c["xn"], P[pre + "w_q"], grads, pre + "w_q", pre + "b_q")
        dxn = dxn + lin_bwd(dk, c["xn"], P[pre + "w_k"], grads, pre + "w_k", pre + "b_k")
        dxn = dxn + lin_bwd(dv, c["xn"], P[pre + "w_v"], grads, pre + "w_v", pre + "b_v")
        d0, dg, db = ln_bwd(dxn, P[pre + "ln1_g"], c["ln1"])
        _acc(grads, pre + "ln1_g", dg)
        _acc(grads, pre + "ln1_b", db)
        dx = dx1 + d0
    return dx


# ----------------------------------------------------------------- full model

def forward(P, cfg, batch):
    """Batched ``LongRecModel.forward_tensor`` (pkg/src/longrec/model.py:307-363).

    Returns (p [B], cache).  All four query strategies (``query_groups``).
    """
    items = np.asarray(batch["items"], dtype=np.int64)
    actions = np.asarray(batch["actions"], dtype=np.int64)
    dt = np.asarray(batch["dt"], dtype=np.int64)
    n_ev = np.minimum(np.asarray(batch["n_events"], dtype=np.int64), cfg.L)
    uid = np.asarray(batch["uid"], dtype=np.int64)
    prof = np.asarray(batch["profile"], dtype=np.int64)
    cand = np.asarray(batch["cand_item"], dtype=np.int64)
    B, L = items.shape
    assert L == cfg.L
    d, D, K, G, m, k = cfg.d, cfg.D, cfg.K, cfg.merged_len, cfg.m, cfg.k
    Lp = cfg.L_padded
    extra = Lp - L
    # token grid in L_padded coordinates: the merge pads on the left (merge.py:45-52)
    col = np.arange(Lp)
    real = col[None, :] >= (Lp - n_ev)[:, None]                                  # [B, Lp]
    pad_l = lambda a: np.concatenate([np.zeros((B, extra), a.dtype), a], axis=1)
    it, ac, tdt = pad_l(items), pad_l(actions), pad_l(dt)
    it = np.where(real, it, 0)
    ac = np.where(real, ac, 0)
    bucket = time_bucket(np.where(real, tdt, 0), cfg.n_time_buckets)
    rec = np.where(real, Lp - 1 - col[None, :], 0)                               # recency, 0 = newest
    # _event_features + abs pos + _seq_mlp (inputs.py:434-482)
    feat = np.concatenate([P["tables.item_table"][it], P["tables.action_table"][ac],
                           P["tables.time_bucket_table"][bucket]], axis=-1)      # [B, Lp, F]
    x0 = lin(feat, P["tables.mlp.tok_proj_w"], P["tables.mlp.tok_proj_b"]) + P["tables.abs_pos_table"][rec]
    a1 = lin(x0, P["tables.mlp.seq_w1"], P["tables.mlp.seq_b1"])
    g1, t1 = gelu_fwd(a1)
    h = lin(g1, P["tables.mlp.seq_w2"], P["tables.mlp.seq_b2"]) * real[:, :, None]
    npg = group_pad_counts(cfg, n_ev)
    if cfg.merge_mode == "inner":
        hm, inner_cache = inner_fwd(P, cfg, h, npg)
    else:
        hm, inner_cache = h, None
    merged = hm.reshape(B, G, D)                                                 # merge_concat reshape
    # global tokens [UID, CLS..., target] (inputs.py:500-537)
    uid_emb = P["tables.uid_table"][uid]
    uid_row = lin(uid_emb, P["tables.mlp.lift_w"], P["tables.mlp.lift_b"])
    tfeat = np.concatenate([P["tables.item_table"][cand], np.zeros((B, cfg.d_act)),
                            np.broadcast_to(P["tables.time_bucket_table"][0], (B, cfg.d_time))], axis=-1)
    td = lin(tfeat, P["tables.mlp.tok_proj_w"], P["tables.mlp.tok_proj_b"])
    trow = lin(td, P["tables.mlp.lift_w"], P["tables.mlp.lift_b"])
    raw = np.concatenate([uid_row[:, None], np.broadcast_to(P["tables.cls_vector"], (B, m - 2, D)),
                          trow[:, None]], axis=1)                                # [B, m, D]
    ga = lin(raw, P["tables.mlp.glob_w1"], P["tables.mlp.glob_b1"])
    gg, gt = gelu_fwd(ga)
    glob = lin(gg, P["tables.mlp.glob_w2"], P["tables.mlp.glob_b2"])
    # composite queries and keys (model.py:317-320)
    qg = query_groups(cfg, npg)                                                   # [B, k]
    if cfg.query_strategy == "learnable":
        qrows = np.broadcast_to(P["query_bank"], (B, k, D))
    else:
        qrows = np.take_along_axis(merged, qg[:, :, None], axis=1)
    O = np.concatenate([qrows, glob], axis=1)
    R = np.concatenate([merged, glob], axis=1)
    vis1 = cross_mask(cfg, npg, qg)
    viss = self_mask(cfg, npg, qg)
    x, c_cross = block_fwd(P, "cross.", O, R, vis1, cfg.heads, False)
    c_self, layers = [], [x]
    for i in range(cfg.N):
        x, c = block_fwd(P, f"self.{i}.", x, x, viss, cfg.heads, True)
        c_self.append(c)
        layers.append(x)
    # head (model.py:346-362)
    t = x[:, k + m - 1]
    cl = x[:, k + 1]
    u_d = np.concatenate([uid_emb, P["tables.profile_table"][prof]], axis=-1)
    hin = np.concatenate([t, cl, t * cl, t * t, u_d], axis=-1)
    z1 = lin(hin, P["head.w1"], P["head.b1"])
    hg, ht = gelu_fwd(z1)
    z = lin(hg, P["head.w2"], P["head.b2"])[:, 0]
    p = sigmoid(z)
    cache = dict(it=it, ac=ac, bucket=bucket, rec=rec, real=real, feat=feat, x0=x0, a1=a1, g1=g1, t1=t1,
                 inner=inner_cache, npg=npg, uid=uid, prof=prof, cand=cand, uid_emb=uid_emb, td=td, tfeat=tfeat,
                 raw=raw, ga=ga, gg=gg, gt=gt, c_cross=c_cross, c_self=c_self, x=x, t=t, cl=cl, hin=hin, qg=qg,
                 z1=z1, hg=hg, ht=ht, z=z, p=p, h=h, merged=merged, layers=layers)
    return p, cache


def bce_mean(p, labels):
    """Batch-mean BCE with the 1e-12 clamp (pkg/src/longrec/tensors.py:536-571)."""
    y = np.asarray(labels, dtype=np.float64)
    pc = np.clip(p, PROB_EPS, 1.0 - PROB_EPS)
    return float(np.mean(-(y * np.log(pc) + (1.0 - y) * np.log(1.0 - pc))))


def backward(P, cfg, batch, cache):
    """Gradients of the batch-mean BCE w.r.t. every parameter (train step body,
    pkg/src/longrec/model.py:555-567).  Returns {name: array}."""
    grads = {}
    y = np.asarray(batch["label"], dtype=np.float64)
    p = cache["p"]
    B = p.shape[0]
    k, m, D, d, G = cfg.k, cfg.m, cfg.D, cfg.d, cfg.merged_len
    # bce (clamp gradient is zero outside the open interval) then sigmoid: dz = (p - y) / B
    inr = (p > PROB_EPS) & (p < 1.0 - PROB_EPS)
    dz = np.where(inr, (p - y) / B, 0.0)[:, None]
    dhg = lin_bwd(dz, cache["hg"], P["head.w2"], grads, "head.w2", "head.b2")
    dz1 = gelu_bwd(dhg, cache["z1"], cache["ht"])
    dhin = lin_bwd(dz1, cache["hin"], P["head.w1"], grads, "head.w1", "head.b1")
    t, cl = cache["t"], cache["cl"]
    dt_ = dhin[:, :D] + dhin[:, 2 * D:3 * D] * cl + 2.0 * dhin[:, 3 * D:4 * D] * t
    dcl = dhin[:, D:2 * D] + dhin[:, 2 * D:3 * D] * t
    du = dhin[:, 4 * D:]
    g_uid = np.zeros_like(P["tables.uid_table"])
    g_prof = np.zeros_like(P["tables.profile_table"])
    np.add.at(g_uid, cache["uid"], du[:, :d])
    np.add.at(g_prof, cache["prof"], du[:, d:])
    dx = np.zeros_like(cache["x"])
    dx[:, k + m - 1] += dt_
    dx[:, k + 1] += dcl
    for i in reversed(range(cfg.N)):
        dx, _ = block_bwd(P, f"self.{i}.", dx, cache["c_self"][i], grads)
    dO, dR = block_bwd(P, "cross.", dx, cache["c_cross"], grads)
    dmerged = dR[:, :G].copy()
    if cfg.query_strategy == "learnable":
        _acc(grads, "query_bank", dO[:, :k].sum(axis=0))
    else:
        qg = cache["qg"]
        for b in range(dO.shape[0]):
            np.add.at(dmerged[b], qg[b], dO[b, :k])
    dglob = dR[:, G:] + dO[:, k:]
    # global MLP and its inputs
    dgg = lin_bwd(dglob, cache["gg"], P["tables.mlp.glob_w2"], grads, "tables.mlp.glob_w2", "tables.mlp.glob_b2")
    dga = gelu_bwd(dgg, cache["ga"], cache["gt"])
    draw = lin_bwd(dga, cache["raw"], P["tables.mlp.glob_w1"], grads, "tables.mlp.glob_w1", "tables.mlp.glob_b1")
    duid_emb = lin_bwd(draw[:, 0], cache["uid_emb"], P["tables.mlp.lift_w"], grads,
                       "tables.mlp.lift_w", "tables.mlp.lift_b")
    np.add.at(g_uid, cache["uid"], duid_emb)
    _acc(grads, "tables.cls_vector", draw[:, 1:m - 1].sum(0))
    dtd = lin_bwd(draw[:, m - 1], cache["td"], P["tables.mlp.lift_w"], grads, "tables.mlp.lift_w", "tables.mlp.lift_b")
    dtfeat = lin_bwd(dtd, cache["tfeat"], P["tables.mlp.tok_proj_w"], grads,
                     "tables.mlp.tok_proj_w", "tables.mlp.tok_proj_b")
    g_item = np.zeros_like(P["tables.item_table"])
    g_act = np.zeros_like(P["tables.action_table"])
    g_time = np.zeros_like(P["tables.time_bucket_table"])
    di, da = cfg.d_item, cfg.d_act
    np.add.at(g_item, cache["cand"], dtfeat[:, :di])
    g_time[0] += dtfeat[:, di + da:].sum(0)
    # merge
    dh = dmerged.reshape(B, cfg.L_padded, d)
    if cfg.merge_mode == "inner":
        dh = inner_bwd(P, cfg, dh, cache["inner"], grads)
    dh = dh * cache["real"][:, :, None]                     # pad rows are constants
    dg1 = lin_bwd(dh, cache["g1"], P["tables.mlp.seq_w2"], grads, "tables.mlp.seq_w2", "tables.mlp.seq_b2")
    da1 = gelu_bwd(dg1, cache["a1"], cache["t1"])
    dx0 = lin_bwd(da1, cache["x0"], P["tables.mlp.seq_w1"], grads, "tables.mlp.seq_w1", "tables.mlp.seq_b1")
    dx0 = dx0 * cache["real"][:, :, None]
    g_pos = np.zeros_like(P["tables.abs_pos_table"])
    np.add.at(g_pos, cache["rec"].reshape(-1), dx0.reshape(-1, d))
    dfeat = lin_bwd(dx0, cache["feat"], P["tables.mlp.tok_proj_w"], grads,
                    "tables.mlp.tok_proj_w", "tables.mlp.tok_proj_b")
    np.add.at(g_item, cache["it"].reshape(-1), dfeat[..., :di].reshape(-1, di))
    np.add.at(g_act, cache["ac"].reshape(-1), dfeat[..., di:di + da].reshape(-1, da))
    np.add.at(g_time, cache["bucket"].reshape(-1), dfeat[..., di + da:].reshape(-1, cfg.d_time))
    grads["tables.item_table"] = g_item
    grads["tables.action_table"] = g_act
    grads["tables.time_bucket_table"] = g_time
    grads["tables.uid_table"] = g_uid
    grads["tables.profile_table"] = g_prof
    grads["tables.abs_pos_table"] = g_pos
    return grads


def forward_backward(P, cfg, batch):
    p, cache = forward(P, cfg, batch)
    loss = bce_mean(p, batch["label"])
    return p, loss, backward(P, cfg, batch, cache)


# ----------------------------------------------------------------- optimizer
def adam_step(params, grads, m, v, t, lr):
    """Adam.step (pkg/src/longrec/model.py:467-482): beta1 = 0.9, beta2 = 0.999, eps = 1e-8, bias
    corrections with the step counter t (>= 1).  Arrays are updated in place (float64)."""
    b1, b2, eps = 0.9, 0.999, 1e-8
    c1 = 1.0 - b1 ** t
    c2 = 1.0 - b2 ** t
    m *= b1
    m += (1 - b1) * grads
    v *= b2
    v += (1 - b2) * grads * grads
    params -= lr * (m / c1) / (np.sqrt(v / c2) + eps)

