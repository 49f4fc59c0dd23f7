"""Alphabets above 64 levels (quantize.cpp:400-401: u16 levels, codec.cpp:416-417:
B = max levels): bins up to 253 (B up to 255) run the dense tile encoder with 8-bit
keys and global symbol frequencies, the decoder's wide unrearrange, and batched
evaluation with global level counts.  Asserted bit for bit against the oracle:
quantized states, FULL and DELTA records, device decode of the records, the C ABI
compress_step (unfused for B > 64) and the proxy evaluation's estimate."""
import numpy as np
import pytest

from oracle.oracle import Config as OConfig
from oracle.oracle import QState
from tests.util import flat, make_tensors, perturb

pytestmark = pytest.mark.gpu

LAYOUT = [
    ("tok_embed.weight", 4, (400, 150)),
    ("blk.attn.qkv", 2, (300, 200)),
    ("blk.fc1.weight", 1, (250, 240)),
    ("blk.norm.weight", 3, (3000,)),
    ("blk.fc1.bias", 5, (5000,)),
    ("head.weight", 6, (100, 300)),
]


@pytest.fixture(scope="module")
def eng():
    from paper_2306_11800_b200 import engine

    return engine.Engine(0)


def _qs(h) -> QState:
    return QState(h.step, h.config, h.codebooks, h.names, h.types, h.shapes, h.levels, h.prot_pos,
                  h.prot_val)


@pytest.mark.parametrize("bins,embed", [(100, 64), (200, 253), (62, 150)])
def test_large_alphabet_records_match_oracle(eng, oracle, bins, embed):
    from paper_2306_11800_b200.engine import Config

    cfg = OConfig(bins=bins, embed_bins=embed, prune_frac=0.0, protect_frac=0.002)
    t1 = make_tensors(LAYOUT, seed=bins, scale=1.0)
    t2 = perturb(t1, seed=bins + 1, frac=0.2, scale=0.05)
    ema = np.random.default_rng(bins).normal(0, 0.1, flat(t1).size).astype(np.float32)
    names = [t.name for t in t1]
    types = [t.type for t in t1]
    shapes = [t.shape for t in t1]
    sizes = np.cumsum([t.data.size for t in t1])[:-1]
    dev, ref = [], []
    for step, ts in ((1, t1), (2, t2)):
        ck = eng.checkpoint(names, types, shapes, weights=[t.data for t in ts], ema=np.split(ema, sizes))
        dev.append(eng.quantize(ck, Config(*cfg.astuple()), 3, step))
        m, s = oracle.scores(flat(ts), ema)
        ref.append(oracle.quantize(ts, step, m, s, cfg, 3))
        assert _qs(dev[-1].download()) == ref[-1]
    assert ref[1].max_levels() > 64
    full = eng.encode_record(dev[0], None, 0.1)
    delta = eng.encode_record(dev[1], dev[0], 0.2)
    assert full == oracle.encode_record(ref[0], None, 0.1)
    assert delta == oracle.encode_record(ref[1], ref[0], 0.2)
    d0 = eng.decode_record(full)
    d1 = eng.decode_record(delta, base=d0)
    assert _qs(d1.download()) == ref[1]
    # Chain::append through the C ABI (B > 64: pass C + the dense encoder)
    ck = eng.checkpoint(names, types, shapes, weights=[t.data for t in t2], ema=np.split(ema, sizes))
    st, rh = eng.compress_step(ck, Config(*cfg.astuple()), 3, 2, base=dev[0], quality=0.2)
    assert eng.record_bytes(rh) == delta
    assert eng.states_equal(st, dev[1])


def test_large_alphabet_eval_estimate(eng, oracle):
    from paper_2306_11800_b200.engine import Config

    t1 = make_tensors(LAYOUT, seed=9, scale=1.0)
    ema = np.random.default_rng(9).normal(0, 0.1, flat(t1).size).astype(np.float32)
    sizes = np.cumsum([t.data.size for t in t1])[:-1]
    ck = eng.checkpoint([t.name for t in t1], [t.type for t in t1], [t.shape for t in t1],
                        weights=[t.data for t in t1], ema=np.split(ema, sizes))
    cfgs = [OConfig(bins=b, embed_bins=e, protect_frac=0.002) for b, e in ((120, 200), (8, 16), (250, 90))]
    seeds = [oracle.quantize_seed(5, c) for c in cfgs]
    q, est = eng.eval_batch(ck, [Config(*c.astuple()) for c in cfgs], seeds)
    m, s = oracle.scores(flat(t1), ema)
    for i, c in enumerate(cfgs):
        oq = oracle.quantize(t1, 0, m, s, c, seeds[i])
        assert est[i] == oracle.estimate_compression(t1, oq), c
        want = oracle.proxy_quality(t1, oracle.dequantize(oq))
        assert abs(q[i] - want) <= 1e-12 * max(1.0, abs(want)), c


def test_alphabet_above_255_is_rejected(eng, oracle):
    from paper_2306_11800_b200.engine import Config, EngineError

    cfg = Config(bins=254, embed_bins=16, prune_frac=0.0, protect_frac=0.0)
    t1 = make_tensors(LAYOUT, seed=4, scale=1.0)
    ck = eng.checkpoint([t.name for t in t1], [t.type for t in t1], [t.shape for t in t1],
                        weights=[t.data for t in t1])
    st = eng.quantize(ck, cfg, 1, 1)
    with pytest.raises(EngineError, match="255"):
        eng.encode_record(st)
