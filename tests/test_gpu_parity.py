"""GPU parity through the C ABI (libdqtg.so) against the oracle.

Bar (task ③): bit-exact for bucket counts, levels, protected entries,
codebooks and record bytes; the oracle is pinned in test_oracle_pin.py.
"""
import zlib

import numpy as np
import pytest

from oracle.oracle import Config as OConfig
from oracle.oracle import QState
from tests.util import CONFIGS, SMALL_LAYOUT, flat, make_tensors, perturb

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def eng():
    from paper_2306_11800_b200 import engine

    return engine.Engine(0)


def _cfg(c: OConfig):
    from paper_2306_11800_b200.engine import Config

    return Config(*c.astuple())


def _qs(h) -> QState:
    return QState(h.step, h.config, h.codebooks, h.names, h.types, h.shapes, h.levels, h.prot_pos,
                  h.prot_val)


@pytest.mark.parametrize("alpha", [0.01, 0.02, 0.05, 1.0 / 3.0, 0.003])
def test_sketch_build_matches_oracle(eng, oracle, alpha):
    rng = np.random.default_rng(3)
    x = np.concatenate([rng.normal(0, 0.05, 200_000), rng.lognormal(0, 4, 50_000) *
                        rng.choice([-1, 1], 50_000), [0.0, -0.0, 1e-13, -1e-13, 1e-12, 3.4e38,
                                                      -3.4e38, 1.1754944e-38]]).astype(np.float32)
    kmin, zero, pos, neg = eng.sketch_build(x, alpha)
    okmin, ozero, opos, oneg = oracle.sketch_dense(x, alpha)
    assert kmin == okmin and zero == ozero
    assert np.array_equal(pos, opos) and np.array_equal(neg, oneg)


@pytest.mark.parametrize("k", [1, 2, 4, 8, 16, 32])
def test_approx_kmeans_matches_oracle(eng, oracle, k):
    rng = np.random.default_rng(k)
    cases = [rng.normal(0, 1, 20000), rng.normal(0, 0.02, 3000), rng.standard_t(3, 5000),
             np.round(rng.normal(0, 2, 400)), np.full(100, 1.0), np.array([0.0, -0.0, 2.0, 2.0])]
    for trial, x in enumerate(cases):
        x = x.astype(np.float32)
        for sigma in (0.2, 1.0, 0.0):
            a = eng.approx_kmeans(x, k, sigma, 0.01, trial + 3)
            b = oracle.approx_kmeans(x, k, sigma, 0.01, trial + 3)
            assert a.view(np.uint32).tolist() == b.view(np.uint32).tolist(), (trial, sigma)


def _run_pair(eng, oracle, cfg, tensors1, tensors2, ema, derived, seed=11):
    names = [t.name for t in tensors1]
    types = [t.type for t in tensors1]
    shapes = [t.shape for t in tensors1]
    out = []
    for step, ts in ((5, tensors1), (6, tensors2)):
        w = [t.data for t in ts]
        m, s = oracle.scores(flat(ts), ema)
        if derived:
            ck = eng.checkpoint(names, types, shapes, weights=w,
                                ema=None if ema is None else np.split(ema, np.cumsum([t.data.size for t in ts])[:-1]))
        else:
            sizes = np.cumsum([t.data.size for t in ts])[:-1]
            ck = eng.checkpoint(names, types, shapes, weights=w, mag=np.split(m, sizes),
                                sens=None if s is None else np.split(s, sizes))
        dq = eng.quantize(ck, _cfg(cfg), seed, step)
        oq = oracle.quantize(ts, step, m, s, cfg, seed)
        assert _qs(dq.download()) == oq, "quantize mismatch"
        out.append((dq, oq))
    (d1, o1), (d2, o2) = out
    full = eng.encode_record(d1, None, 0.25)
    delta = eng.encode_record(d2, d1, 0.5)
    assert full == oracle.encode_record(o1, None, 0.25)
    assert delta == oracle.encode_record(o2, o1, 0.5)


@pytest.mark.parametrize("ci", range(len(CONFIGS)))
@pytest.mark.parametrize("derived", [False, True])
def test_quantize_and_records_match_oracle(eng, oracle, ci, derived):
    cfg = CONFIGS[ci]
    t1 = make_tensors(seed=ci)
    t2 = perturb(t1, seed=100 + ci)
    rng = np.random.default_rng(ci)
    ema = rng.normal(0, 0.1, flat(t1).size).astype(np.float32) if (cfg.metric or ci % 2 == 0) else None
    _run_pair(eng, oracle, cfg, t1, t2, ema, derived)


def test_c1_fingerprint_on_gpu(eng, oracle):
    """SURVEY.md §8c C1 recipe through the device pipeline."""
    layout = oracle.default_layout(11_700_000)
    traj = oracle.generate_trajectory(layout, 2, 1)
    (w1, g1), (w2, g2) = traj
    ema = oracle.ema_update(flat(g1), flat(g2), 0.9)
    names = [n for n, _, _ in layout]
    types = [t for _, t, _ in layout]
    shapes = [s for _, _, s in layout]
    sizes = np.cumsum([int(np.prod(s)) for s in shapes])[:-1]
    from paper_2306_11800_b200.engine import Config
    states = []
    for step, ws in ((1, w1), (2, w2)):
        ck = eng.checkpoint(names, types, shapes, weights=[t.data for t in ws],
                            ema=np.split(ema, sizes))
        states.append(eng.quantize(ck, Config(), 1, step))
    full = eng.encode_record(states[0])
    delta = eng.encode_record(states[1], states[0])
    assert (len(full), zlib.crc32(full)) == (5_785_628, 0xDCF04BBA)
    assert (len(delta), zlib.crc32(delta)) == (802_911, 0xAAAAE4E6)


def test_primitives(eng, oracle):
    assert eng.crc32(b"123456789") == 0xCBF43926
    rng = np.random.default_rng(0)
    for n in (0, 1, 7, 100_003):
        b = rng.integers(0, 256, n, dtype=np.uint8).tobytes()
        assert eng.crc32(b) == zlib.crc32(b)
    p = rng.integers(0, 34, 10000).astype(np.uint16)
    c = rng.integers(0, 34, 10000).astype(np.uint16)
    assert np.array_equal(eng.delta_compute(p, c, 34), oracle.delta_compute(p, c, 34))
    e = rng.normal(0, 1, 100_000).astype(np.float32)
    g = rng.normal(0, 1, 100_000).astype(np.float32)
    assert np.array_equal(eng.ema_update(e, g, 0.9), oracle.ema_update(e, g, 0.9))
    w = rng.normal(0, 1, 100_000).astype(np.float32)
    m1, s1 = eng.compute_scores(w, e)
    m2, s2 = oracle.scores(w, e)
    assert np.array_equal(m1, m2) and np.array_equal(s1, s2)
