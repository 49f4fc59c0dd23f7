"""decode_delta_record on the device (decode.cu) against the oracle and the
reference's golden records: levels, protected entries, codebooks and step must
round-trip bit-exactly; corrupt records raise the reference's error types."""
import glob
import os

import numpy as np
import pytest

from tests.util import CONFIGS, flat, make_tensors, perturb

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def eng():
    from paper_2306_11800_b200 import engine as E

    return E.Engine(0)


def host_equal(dev_state, q):
    """DevState (downloaded) == oracle QState."""
    h = dev_state.download()
    assert h.step == q.step
    for lt in range(7):
        np.testing.assert_array_equal(np.asarray(h.codebooks[lt], np.float32),
                                      np.asarray(q.codebooks[lt], np.float32))
    assert h.names == list(q.names)
    assert [tuple(x) for x in h.shapes] == [tuple(x) for x in q.shapes]
    for i, lv in enumerate(h.levels):
        np.testing.assert_array_equal(lv, np.asarray(q.levels[i]).ravel())
        np.testing.assert_array_equal(h.prot_pos[i], np.asarray(q.prot_pos[i], np.uint64))
        np.testing.assert_array_equal(h.prot_val[i], np.asarray(q.prot_val[i], np.uint16))


@pytest.mark.parametrize("ci", range(len(CONFIGS)))
def test_decode_oracle_records(eng, oracle, ci):
    cfg = CONFIGS[ci]
    t1 = make_tensors(seed=10 + ci)
    t2 = perturb(t1, seed=20 + ci, frac=0.2)
    ema = np.random.default_rng(ci).normal(0, 0.1, flat(t1).size).astype(np.float32)
    qs = []
    for step, ts in ((1, t1), (2, t2)):
        m, s = oracle.scores(flat(ts), ema)
        qs.append(oracle.quantize(ts, step, m, s, cfg, 1))
    full = oracle.encode_record(qs[0])
    delta = oracle.encode_record(qs[1], qs[0])
    d1 = eng.decode_record(full)
    host_equal(d1, qs[0])
    d2 = eng.decode_record(delta, base=d1)
    host_equal(d2, qs[1])
    # re-encoding the decoded states reproduces the records byte for byte
    assert eng.encode_record(d1) == full
    assert eng.encode_record(d2, d1) == delta


def test_decode_golden_reference_records(eng):
    files = sorted(glob.glob(os.path.join(HERE, "golden", "golden_case*.npz")))
    assert files
    for f in files:
        g = np.load(f)
        d1 = eng.decode_record(bytes(g["full"]))
        d2 = eng.decode_record(bytes(g["delta"]), base=d1)
        h = d2.download()
        got = np.concatenate([lv.ravel() for lv in h.levels])
        np.testing.assert_array_equal(got, g["levels2"].ravel(), err_msg=f)


def test_decode_chain_roundtrip_large(eng):
    """A longer chain of device-encoded records (many chunks per group)."""
    from paper_2306_11800_b200 import engine as E

    layout = [("emb", 4, (4000, 256)), ("att", 2, (512, 1024)), ("fc", 1, (1024, 700)),
              ("ln", 3, (1024,)), ("b", 5, (3000,))]
    names = [n for n, _, _ in layout]
    types = [t for _, t, _ in layout]
    shapes = [s for _, _, s in layout]
    rng = np.random.default_rng(7)
    w = [rng.normal(0, 0.05, int(np.prod(s))).astype(np.float32) for s in shapes]
    ema = [rng.normal(0, 0.05, x.size).astype(np.float32) for x in w]
    prev_dev, prev_dec = None, None
    for step in range(4):
        ck = eng.checkpoint(names, types, shapes, weights=w, ema=ema)
        st = eng.quantize(ck, E.Config(), 1, step)
        rec = eng.encode_record(st, prev_dev)
        dec = eng.decode_record(rec, base=prev_dec)
        a, b = st.download(), dec.download()
        for x, y in zip(a.levels, b.levels):
            np.testing.assert_array_equal(x, y)
        for x, y in zip(a.prot_pos, b.prot_pos):
            np.testing.assert_array_equal(x, y)
        prev_dev, prev_dec = st, dec
        w = [x - np.float32(0.1 * 0.9 ** step) * (x + 0.0025 * rng.normal(size=x.size)).astype(np.float32)
             for x in w]


def test_decode_errors(eng, oracle):
    from paper_2306_11800_b200 import engine as E

    t1 = make_tensors(seed=3)
    t2 = perturb(t1, seed=4, frac=0.2)
    m1, s1 = oracle.scores(flat(t1), None)
    m2, s2 = oracle.scores(flat(t2), None)
    q1 = oracle.quantize(t1, 1, m1, s1, CONFIGS[0], 1)
    q2 = oracle.quantize(t2, 2, m2, s2, CONFIGS[0], 1)
    full = oracle.encode_record(q1)
    delta = oracle.encode_record(q2, q1)
    d1 = eng.decode_record(full)

    def status(rec, base=None):
        with pytest.raises(E.EngineError) as ex:
            eng.decode_record(rec, base=base)
        return ex.value.status

    assert status(b"XXXX" + full[4:]) == 2                      # BadMagic
    assert status(full[:40]) == 3                               # TruncatedFile
    bad_crc = bytearray(full)
    bad_crc[-1] ^= 0xFF
    assert status(bytes(bad_crc)) == 15                         # ChecksumMismatch
    assert status(delta) == 16                                  # delta without base: ChainCorrupt
    d2 = eng.decode_record(delta, base=d1)
    assert status(delta, base=d2) == 16                         # base step mismatch
    assert status(full + b"\0") == 6                            # trailing bytes: IoError
    # a flipped bit inside the payload is detected (bitstream, index or checksum)
    flip = bytearray(full)
    flip[len(full) // 2] ^= 0x10
    assert status(bytes(flip)) in (3, 13, 14, 15)


def test_decode_fuzzed_records(eng, oracle):
    """Random byte flips anywhere in FULL and DELTA records: the device decoder either
    decodes (a flip inside codebook floats or the quality field can leave a valid
    record) or raises one of the reference's error types; it never faults, and the
    engine keeps decoding the intact records afterwards."""
    from paper_2306_11800_b200 import engine as E

    t1 = make_tensors(seed=8)
    t2 = perturb(t1, seed=9, frac=0.2)
    m1, s1 = oracle.scores(flat(t1), None)
    m2, s2 = oracle.scores(flat(t2), None)
    q1 = oracle.quantize(t1, 1, m1, s1, CONFIGS[0], 1)
    q2 = oracle.quantize(t2, 2, m2, s2, CONFIGS[0], 1)
    full = oracle.encode_record(q1)
    delta = oracle.encode_record(q2, q1)
    base = eng.decode_record(full)
    rng = np.random.default_rng(123)
    allowed = {1, 2, 3, 4, 6, 13, 14, 15, 16}
    for rec, b in ((full, None), (delta, base)):
        for _ in range(120):
            bad = bytearray(rec)
            pos = int(rng.integers(0, len(bad)))
            bad[pos] ^= int(rng.integers(1, 256))
            try:
                eng.decode_record(bytes(bad), base=b)
            except E.EngineError as ex:
                assert ex.status in allowed, (pos, ex)
    host_equal(eng.decode_record(full), q1)
    host_equal(eng.decode_record(delta, base=eng.decode_record(full)), q2)


def test_decode_chain_matches_sequential(oracle):
    """dqtg_decode_chain (host walk of record k+1 overlapping the device decode of k)
    gives the states decode_record gives one by one, and the oracle's."""
    from paper_2306_11800_b200 import engine as E
    from tests.util import CONFIGS, flat, make_tensors, perturb

    eng = E.Engine(0)
    cfg = CONFIGS[1]
    ts = [make_tensors(seed=3)]
    for k in range(4):
        ts.append(perturb(ts[-1], seed=10 + k))
    ema = np.random.default_rng(1).normal(0, 0.1, flat(ts[0]).size).astype(np.float32)
    qs, recs, prev = [], [], None
    for k, t in enumerate(ts):
        m, s = oracle.scores(flat(t), ema)
        q = oracle.quantize(t, k, m, s, cfg, 1)
        recs.append(oracle.encode_record(q, prev))
        qs.append(q)
        prev = q
    seen = []
    last = eng.decode_chain(recs, on_state=lambda k, h: seen.append(k))
    assert seen == list(range(len(recs)))
    got = last.download()
    want = qs[-1]
    assert [x.tolist() for x in got.levels] == [np.asarray(x).tolist() for x in want.levels]
    # the same chain one record at a time
    st = None
    for r in recs:
        st = eng.decode_record(r, base=st)
    assert eng.states_equal(st, last)
    # a corrupt record in the middle: raised after the records before it decoded
    bad = list(recs)
    bad[2] = bad[2][:-5]
    seen.clear()
    with pytest.raises(E.EngineError):
        eng.decode_chain(bad, on_state=lambda k, h: seen.append(k))
    assert seen == [0, 1]
