"""Pin the CPU oracle (oracle/longer_oracle.py) to golden vectors produced by the reference
itself (tests/golden/make_golden.py) — forward probabilities, loss and every gradient."""
import glob
import json
import os

import numpy as np
import pytest

from oracle import longer_oracle as O
from paper_2505_04421_b200.config import ModelConfig
from paper_2505_04421_b200.params import init_params, param_shapes

GOLDEN = sorted(p for p in glob.glob(os.path.join(os.path.dirname(__file__), "golden", "*.npz"))
                if not os.path.basename(p).startswith("serving_"))


def load_golden(path):
    z = np.load(path)
    cfg = ModelConfig(**json.loads(str(z["cfg"])))
    P = {k[2:]: z[k] for k in z.files if k.startswith("P/")}
    G = {k[2:]: z[k] for k in z.files if k.startswith("G/")}
    batch = {k[6:]: z[k] for k in z.files if k.startswith("batch/")}
    return cfg, P, G, batch, z["p"], float(z["loss"]), int(z["seed"])


@pytest.mark.parametrize("path", GOLDEN, ids=[os.path.basename(p)[:-4] for p in GOLDEN])
def test_oracle_matches_reference_golden(path):
    cfg, P, G, batch, p_ref, loss_ref, _ = load_golden(path)
    p, loss, grads = O.forward_backward(P, cfg, batch)
    np.testing.assert_allclose(p, p_ref, rtol=0, atol=1e-10)
    assert abs(loss - loss_ref) <= 1e-10
    assert set(grads) == set(G)
    for n, g in G.items():
        np.testing.assert_allclose(grads[n], g, rtol=1e-8, atol=1e-11, err_msg=n)


@pytest.mark.parametrize("path", GOLDEN, ids=[os.path.basename(p)[:-4] for p in GOLDEN])
def test_init_params_bit_identical_to_reference(path):
    cfg, P, _, _, _, _, seed = load_golden(path)
    mine = init_params(cfg, seed)
    assert list(mine) == list(param_shapes(cfg))
    assert set(mine) == set(P)
    for n, a in mine.items():
        np.testing.assert_array_equal(a, P[n], err_msg=n)


def test_time_bucket_known_answers():
    # pkg/tests/test_inputs.py:93-106 and SPEC.md: 3601 s → 12, 0 → 0, 2^40 → 31
    assert O.time_bucket(np.array([3601, 0, 2 ** 40, 1, 2, 3, 4]), 32).tolist() == [12, 0, 31, 1, 2, 2, 3]
    assert O.time_bucket(np.array([2 ** 40]), 8).tolist() == [7]


REF_SRC = "/root/reference/pkg/src"


@pytest.mark.skipif(not os.path.isdir(REF_SRC), reason="reference package not present")
def test_oracle_adam_matches_reference_adam():
    """oracle.adam_step against longrec's own Adam.step (pkg/src/longrec/model.py:453-482)."""
    import sys
    sys.path.insert(0, REF_SRC)
    try:
        from longrec.model import Adam as RefAdam
        from longrec.tensors import Tensor
    finally:
        sys.path.remove(REF_SRC)
    rng = np.random.default_rng(1)
    w = Tensor(rng.standard_normal((7, 5)))
    ref = RefAdam([("w", w)], lr=3e-3)
    p = w.data.copy()
    m, v = np.zeros_like(p), np.zeros_like(p)
    for t in range(1, 5):
        g = rng.standard_normal(p.shape)
        w.grad = g.copy()
        ref.step()
        O.adam_step(p, g, m, v, t, 3e-3)
        np.testing.assert_allclose(p, w.data, rtol=0, atol=1e-15)
