"""payload_bytes_pe / _rle / _he (codec.cpp:615-646) from the device encoder's
ablation modes against the oracle: small checkpoints for every config, and a
multi-tile checkpoint where runs cross tile boundaries (joined for the RLE
variants, never for the raw-delta variant)."""
import numpy as np
import pytest

from tests.util import CONFIGS, flat, make_tensors, perturb

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def eng():
    from paper_2306_11800_b200 import engine as E

    return E.Engine(0)


def _dev(eng, q):
    from paper_2306_11800_b200 import engine as E

    return eng.upload_state(E.HostState(q.step, q.config, q.codebooks, q.names, q.types, q.shapes,
                                        q.levels, q.prot_pos, q.prot_val))


@pytest.mark.parametrize("ci", range(len(CONFIGS)))
def test_payload_bytes_match_oracle(eng, oracle, ci):
    t1 = make_tensors(seed=30 + ci)
    t2 = perturb(t1, seed=40 + ci, frac=0.2)
    ema = np.random.default_rng(ci).normal(0, 0.1, flat(t1).size).astype(np.float32)
    m1, s1 = oracle.scores(flat(t1), ema)
    m2, s2 = oracle.scores(flat(t2), ema)
    q1 = oracle.quantize(t1, 1, m1, s1, CONFIGS[ci], 1)
    q2 = oracle.quantize(t2, 2, m2, s2, CONFIGS[ci], 1)
    d1, d2 = _dev(eng, q1), _dev(eng, q2)
    for v in range(3):
        assert eng.payload_bytes(d1, d2, v) == oracle.payload_bytes(q1, q2, v), v
        assert eng.payload_bytes(d2, d1, v) == oracle.payload_bytes(q2, q1, v), v
    # identical states: every delta is 0 (one long run per group)
    for v in range(3):
        assert eng.payload_bytes(d1, d1, v) == oracle.payload_bytes(q1, q1, v), v


def test_payload_bytes_multi_tile(eng, oracle):
    from paper_2306_11800_b200 import engine as E

    layout = [("emb", 4, (700, 900)), ("fc", 1, (513, 1001)), ("b", 5, (3,)), ("ln", 3, (77,))]
    names = [n for n, _, _ in layout]
    types = [t for _, t, _ in layout]
    shapes = [s for _, _, s in layout]
    rng = np.random.default_rng(5)
    w1 = [rng.normal(0, 0.05, int(np.prod(s))).astype(np.float32) for s in shapes]
    # sparse changes: long zero-delta runs that cross the 4096-element tiles
    w2 = [x + (rng.random(x.size) < 0.01) * rng.normal(0, 0.05, x.size).astype(np.float32)
          for x in w1]
    st = []
    for step, w in ((1, w1), (2, w2)):
        ck = eng.checkpoint(names, types, shapes, weights=w)
        st.append(eng.quantize(ck, E.Config(), 1, step))
    from oracle.oracle import QState

    def host(d):
        h = d.download()
        return QState(h.step, h.config, h.codebooks, h.names, h.types, h.shapes, h.levels,
                      h.prot_pos, h.prot_val)

    q1, q2 = host(st[0]), host(st[1])
    for v in range(3):
        assert eng.payload_bytes(st[0], st[1], v) == oracle.payload_bytes(q1, q2, v), v
