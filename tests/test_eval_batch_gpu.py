"""Batched candidate evaluation (EvalCache::prefetch -> dqtg_eval_batch, search.cpp:
107-112, 174-204): candidates sharing a partition (alpha, prune, protect, metric)
share pass B and are evaluated kEvalM at a time per read of the weights.  Every
candidate's result must equal its evaluation alone and the oracle's
quantize -> dequantize -> proxy_quality_delta / estimate_compression:
estimate_compression exactly (integer level counts), quality to 1e-12 relative
(fixed-order parallel sums)."""
import numpy as np
import pytest

from oracle.oracle import Config
from tests.util import flat, make_tensors

pytestmark = pytest.mark.gpu


def _cands():
    out = []
    for prune, prot in ((0.0, 0.005), (0.1, 0.01), (0.0, 0.0005)):
        for bins in (4, 6, 8, 12, 16, 32):
            for emb in (16, 32):
                out.append(Config(bins=bins, embed_bins=emb, prune_frac=prune, protect_frac=prot))
    out.append(Config(bins=8, embed_bins=16, prune_frac=0.2, protect_frac=0.005, metric=1, sigma=0.7))
    out.append(Config(bins=16, embed_bins=32, prune_frac=0.2, protect_frac=0.005, metric=1, sigma=0.1))
    return out


def test_batched_equals_single_and_oracle(oracle):
    from paper_2306_11800_b200 import engine as E

    eng = E.Engine(0)
    ts = make_tensors(seed=51)
    ema = np.random.default_rng(7).normal(0, 0.1, flat(ts).size).astype(np.float32)
    sizes = np.cumsum([t.data.size for t in ts])[:-1]
    m, s = oracle.scores(flat(ts), ema)
    ck = eng.checkpoint([t.name for t in ts], [t.type for t in ts], [t.shape for t in ts],
                        weights=[t.data for t in ts], mag=np.split(m, sizes), sens=np.split(s, sizes))
    cands = _cands()
    seeds = [oracle.quantize_seed(9, c) for c in cands]
    q_all, e_all = eng.eval_batch(ck, [E.Config(*c.astuple()) for c in cands], seeds)
    for i, (c, sd) in enumerate(zip(cands, seeds)):
        q1, e1 = eng.eval_batch(ck, [E.Config(*c.astuple())], [sd])
        assert e_all[i] == e1[0], i
        assert abs(q_all[i] - q1[0]) <= 1e-12 * max(1e-300, abs(q1[0])), i
        qs = oracle.quantize(ts, 0, m, s, c, sd)
        want_q = oracle.proxy_quality(ts, oracle.dequantize(qs))
        want_e = oracle.estimate_compression(ts, qs)
        assert e_all[i] == want_e, (i, e_all[i], want_e)
        assert abs(q_all[i] - want_q) <= 1e-12 * max(1e-300, abs(want_q)), (i, q_all[i], want_q)
