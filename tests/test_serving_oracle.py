"""Pins the oracle as the serving checker (CPU): the reference's cached scores
(tests/golden/serving_*.npz, made by make_serving_golden.py from longrec.serving) equal the
float64 oracle's full forward of the same (user, candidate) samples — the identity the
reference itself asserts (pkg/src/longrec/serving.py:9-12)."""
import glob
import json
import os

import numpy as np
import pytest

from oracle import longer_oracle as O
from paper_2505_04421_b200 import ModelConfig

SERVING = sorted(glob.glob(os.path.join(os.path.dirname(__file__), "golden", "serving_*.npz")))


@pytest.mark.parametrize("path", SERVING, ids=[os.path.basename(p)[:-4] for p in SERVING])
def test_oracle_full_forward_equals_reference_cached_scores(path):
    z = np.load(path)
    cfg = ModelConfig(**json.loads(str(z["cfg"])))
    P = {k[2:]: z[k] for k in z.files if k.startswith("P/")}
    users = {k[6:]: z[k] for k in z.files if k.startswith("users/")}
    cand = z["cand"]
    U, C = cand.shape
    batch = {f: np.repeat(np.asarray(v), C, axis=0) for f, v in users.items()}
    batch["cand_item"] = cand.reshape(-1)
    p, _ = O.forward(P, cfg, batch)
    np.testing.assert_allclose(p.reshape(U, C), z["p_cached"], rtol=0, atol=1e-10)
    np.testing.assert_allclose(z["p_full"], z["p_cached"], rtol=0, atol=1e-10)


def test_serving_fixtures_exist():
    assert len(SERVING) >= 3


@pytest.mark.parametrize("path", SERVING, ids=[os.path.basename(p)[:-4] for p in SERVING])
def test_serving_oracle_equals_reference_cached_scores(path):
    """oracle/serving_oracle.py (batched build_cache / score_with_cache) against the reference's
    own cached scores."""
    from oracle import serving_oracle as SO
    z = np.load(path)
    cfg = ModelConfig(**json.loads(str(z["cfg"])))
    P = {k[2:]: z[k] for k in z.files if k.startswith("P/")}
    users = {k[6:]: z[k] for k in z.files if k.startswith("users/")}
    cache = SO.build_cache(P, cfg, users)
    p = SO.score(P, cfg, cache, z["cand"])
    np.testing.assert_allclose(p, z["p_cached"], rtol=0, atol=1e-10)
