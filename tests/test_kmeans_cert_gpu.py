"""Certified parallel k-means (kmeans.cu): the k-means++ pick from a parallel prefix
and the interval Lloyd steps must reproduce the reference's sequential fp64 sums'
decisions exactly (quantize.cpp:94-325).  Codebooks are compared bit for bit with
the oracle over inputs chosen to stress the certificates -- heavy ties, zero
weights (sigma = 0 with zero keys), few distinct values, wide dynamic range,
k up to 62 -- and with DQTG_KM_EXACT=1 (every sum sequential).  The stand-alone
C-ABI clustering primitives (dqtg_kmeanspp_init / dqtg_lloyd / dqtg_sq_loss),
dqtg_partition masks and dqtg_proxy_quality are checked against the oracle too."""
import os

import numpy as np
import pytest

from tests.util import CONFIGS, flat, make_tensors

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def eng():
    from paper_2306_11800_b200 import engine

    return engine.Engine(0)


def _cases(seed):
    rng = np.random.default_rng(seed)
    return [
        rng.normal(0, 0.05, 200_000),                                   # C2-like weights
        rng.standard_t(2, 50_000) * 0.01,                               # heavy tails
        np.concatenate([np.zeros(30_000), rng.normal(0, 1e-3, 30_000)]),  # many exact zeros
        np.round(rng.normal(0, 3, 20_000)) * 0.25,                      # few distinct values
        rng.lognormal(-8, 3, 40_000) * rng.choice([-1, 1], 40_000),     # wide dynamic range
        np.concatenate([rng.normal(-1, 1e-4, 5000), rng.normal(1, 1e-4, 5000)]),  # two tight clumps
    ]


@pytest.mark.parametrize("exact", [False, True])
@pytest.mark.parametrize("k", [3, 16, 32, 62])
def test_approx_kmeans_certified(eng, oracle, k, exact):
    if exact:
        os.environ["DQTG_KM_EXACT"] = "1"
    try:
        for trial in range(3):
            for ci, x in enumerate(_cases(100 * k + trial)):
                x = x.astype(np.float32)
                for sigma in (0.2, 0.0, 1.0):
                    a = eng.approx_kmeans(x, k, sigma, 0.01, trial * 7 + ci)
                    b = oracle.approx_kmeans(x, k, sigma, 0.01, trial * 7 + ci)
                    assert a.view(np.uint32).tolist() == b.view(np.uint32).tolist(), (trial, ci, sigma)
    finally:
        os.environ.pop("DQTG_KM_EXACT", None)


def test_clustering_primitives_match_oracle(eng, oracle):
    rng = np.random.default_rng(4)
    for n, k in ((50, 3), (1500, 16), (4000, 32)):
        pts = np.sort(rng.normal(0, 1, n))
        w = rng.random(n)
        w[rng.random(n) < 0.1] = 0.0
        for seed in (1, 2, 3):
            c1 = eng.kmeanspp_init(pts, w, k, seed)
            c2 = oracle.kmeanspp_init(pts, w, k, seed)
            assert c1.tobytes() == c2.tobytes(), (n, k, seed)
            l1, i1 = eng.lloyd(pts, w, c1)
            l2, i2 = oracle.lloyd(pts, w, c2)
            assert l1.tobytes() == l2.tobytes() and i1 == i2, (n, k, seed)
            assert eng.sq_loss(pts, w, l1) == oracle.sq_loss(pts, w, l2)


@pytest.mark.parametrize("ci", range(len(CONFIGS)))
def test_partition_masks_match_oracle(eng, oracle, ci):
    from paper_2306_11800_b200.engine import Config

    cfg = CONFIGS[ci]
    ts = make_tensors(seed=ci)
    rng = np.random.default_rng(ci)
    ema = rng.normal(0, 0.1, flat(ts).size).astype(np.float32)
    sizes = np.cumsum([t.data.size for t in ts])[:-1]
    ck = eng.checkpoint([t.name for t in ts], [t.type for t in ts], [t.shape for t in ts],
                        weights=[t.data for t in ts], ema=np.split(ema, sizes))
    got = np.concatenate(eng.partition(ck, Config(*cfg.astuple())))
    m, s = oracle.scores(flat(ts), ema)
    want = oracle.partition(ts, m, s, cfg)
    assert np.array_equal(got, want)


def test_proxy_quality_matches_oracle(eng, oracle):
    ts = make_tensors(seed=3)
    rng = np.random.default_rng(3)
    recon = [t.data + rng.normal(0, 1e-3, t.data.size).astype(np.float32) for t in ts]
    got = eng.proxy_quality([t.name for t in ts], [t.type for t in ts], [t.shape for t in ts],
                            [t.data for t in ts], recon)
    want = oracle.proxy_quality(ts, np.concatenate(recon))
    assert abs(got - want) <= 1e-12 * max(1.0, abs(want))
