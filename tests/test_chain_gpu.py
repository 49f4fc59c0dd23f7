"""DeviceChain (paper_2306_11800_b200/chain.py): Chain::append/restore
(src/chain.cpp:86-154) over device states.  Records are the engine's own records
(byte-identical to the oracle's, see test_gpu_parity), the directory is the
reference layout (the drop-in and the reference Chain open and restore it), FULL
every full_every records, and the pipelined append writes the same files as
one-by-one appends."""
import os

import numpy as np
import pytest

from tests.util import make_tensors, perturb

pytestmark = pytest.mark.gpu


def _series(n, seed=11):
    s = [make_tensors(seed=seed)]
    for k in range(n - 1):
        s.append(perturb(s[-1], seed=seed * 100 + k, frac=0.1))
    return s


def _layout(ts):
    return [t.name for t in ts], [t.type for t in ts], [t.shape for t in ts]


def _files(d):
    return {f: open(os.path.join(d, f), "rb").read() for f in sorted(os.listdir(d))
            if f.endswith(".dqdr")}


def _manifest_body(d):
    return open(os.path.join(d, "manifest.txt")).read().split("\n", 1)[1]


@pytest.fixture(scope="module")
def eng():
    from paper_2306_11800_b200 import engine as E

    return E.Engine(0)


def test_device_chain_append_restore(eng, tmp_path):
    from paper_2306_11800_b200 import engine as E
    from paper_2306_11800_b200.chain import DeviceChain

    series = _series(7)
    names, types, shapes = _layout(series[0])
    cfg = E.Config()
    states = []
    for k, ts in enumerate(series):
        ck = eng.checkpoint(names, types, shapes, weights=[t.data for t in ts])
        states.append(eng.quantize(ck, cfg, 1, 10 + k))
    d = str(tmp_path / "c")
    ch = DeviceChain(eng, d, full_every=3)
    for st in states:
        ch.append(st)
    assert [e.full for e in ch.entries] == [True, False, False, True, False, False, True]
    files = _files(d)
    for k, e in enumerate(ch.entries):
        want = eng.encode_record(states[k], None if e.full else states[k - 1])
        assert files[e.filename] == want, e.step
    # device replay restores every step
    for k in (1, 4, 6):
        got, want = ch.restore(10 + k).download(), states[k].download()
        for a, b in zip(got.levels, want.levels):
            np.testing.assert_array_equal(a, b)
    # the drop-in Chain opens the same directory and restores the same levels
    from paper_2306_11800_b200 import dqt

    hc = dqt.Chain.open(d, 3)
    assert [e.step for e in hc.entries] == [e.step for e in ch.entries]
    hc.verify()
    q = hc.restore(15)
    for t, lv in zip(q.tensors, states[5].download().levels):
        np.testing.assert_array_equal(np.asarray(t.levels).ravel(), lv)
    # reopening continues the chain (base restored from the records on the device)
    ch2 = DeviceChain(eng, d, full_every=3)
    ck = eng.checkpoint(names, types, shapes, weights=[t.data for t in perturb(series[-1], seed=5)])
    st8 = eng.quantize(ck, cfg, 1, 17)
    e = ch2.append(st8)
    assert not e.full and e.base_step == 16
    assert _files(d)[e.filename] == eng.encode_record(st8, states[6])
    with pytest.raises(E.EngineError):
        ch2.append(states[0])  # step not after the last one


def test_device_chain_opened_by_reference(eng, tmp_path, ref):
    """The unmodified reference Chain (oracle/_ref) restores the device chain."""
    from paper_2306_11800_b200 import engine as E
    from paper_2306_11800_b200.chain import DeviceChain

    series = _series(4, seed=3)
    names, types, shapes = _layout(series[0])
    d = str(tmp_path / "r")
    ch = DeviceChain(eng, d, full_every=50)
    states = []
    for k, ts in enumerate(series):
        ck = eng.checkpoint(names, types, shapes, weights=[t.data for t in ts])
        states.append(eng.quantize(ck, E.Config(), 1, k + 1))
        ch.append(states[-1])
    R = ref.load()
    rc = R.Chain.open(d, 50)
    rc.verify()
    q = rc.restore(4)
    for t, lv in zip(q.tensors, states[3].download().levels):
        np.testing.assert_array_equal(np.asarray(t.levels).ravel(), lv)


@pytest.mark.parametrize("full_every", [2, 4, 50])
def test_pipelined_append_matches_sequential(eng, tmp_path, full_every):
    from paper_2306_11800_b200 import engine as E
    from paper_2306_11800_b200.chain import DeviceChain
    from paper_2306_11800_b200.pipeline import ChainCompressor

    series = _series(7, seed=21)
    names, types, shapes = _layout(series[0])
    cfg = E.Config()
    cc = ChainCompressor(0, workers=3)
    cks = []
    for ts in series:
        c = cc.checkpoint(names, types, shapes)
        c.set_weights([t.data for t in ts])
        cks.append(c)
    steps = list(range(100, 107))
    dp = str(tmp_path / "p")
    chp = DeviceChain(eng, dp, full_every=full_every)
    chp.append_snapshots(cc, cks[:3], cfg, 1, steps[:3])
    chp.append_snapshots(cc, cks[3:], cfg, 1, steps[3:])
    ds = str(tmp_path / "s")
    chs = DeviceChain(eng, ds, full_every=full_every)
    for c, s in zip(cks, steps):
        chs.append(eng.quantize(c, cfg, 1, s))
    assert _files(dp) == _files(ds)
    assert _manifest_body(dp) == _manifest_body(ds)
