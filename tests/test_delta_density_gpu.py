"""DELTA records across the range of delta densities the sparse encoder
(enc_tile_delta_kernel) must handle: identical states, a few moved levels, half
and all levels moved, every cyclic alphabet width from 2 to 64 levels, ragged
tensors (1, 63, 4095, 4097 elements) and groups without moved elements.
Records are compared byte for byte with the oracle's encode_delta_record
(codec.cpp:398-460) and decoded back on the device."""
import numpy as np
import pytest

from oracle.oracle import QState

pytestmark = pytest.mark.gpu

SIZES = [1, 63, 4095, 4096, 4097, 20000, 70001]


def states(rng, cb_len, density, lt=1, runs=False):
    """Two states of len(SIZES) tensors with levels < cb_len + 2."""
    top = cb_len + 2
    names = [f"t{i}" for i in range(len(SIZES))]
    cbs = [np.zeros(0, np.float32) for _ in range(7)]
    cbs[lt] = np.linspace(-1, 1, cb_len).astype(np.float32)
    prev, cur = [], []
    for n in SIZES:
        if runs:  # long runs of equal levels: runs crossing tile boundaries
            a = np.repeat(rng.integers(0, top, n // 500 + 1), 500)[:n].astype(np.uint16)
        else:
            a = rng.integers(0, top, n).astype(np.uint16)
        b = a.copy()
        m = rng.random(n) < density
        b[m] = rng.integers(0, top, int(m.sum())).astype(np.uint16)
        prev.append(a)
        cur.append(b)
    mk = lambda lv, step: QState(step, (cb_len, cb_len, 0.0, 0.0, 0, 0.2, 0.01), cbs, names,  # noqa: E731
                                 [lt] * len(SIZES), [(n,) for n in SIZES], lv,
                                 [np.zeros(0, np.uint64)] * len(SIZES),
                                 [np.zeros(0, np.uint16)] * len(SIZES))
    return mk(prev, 1), mk(cur, 2)


@pytest.fixture(scope="module")
def eng():
    from paper_2306_11800_b200 import engine as E

    return E.Engine(0)


def host(q):
    from paper_2306_11800_b200 import engine as E

    return E.HostState(q.step, q.config, q.codebooks, q.names, q.types, q.shapes, q.levels,
                       q.prot_pos, q.prot_val)


@pytest.mark.parametrize("cb_len", [0, 1, 8, 32, 62])
@pytest.mark.parametrize("density", [0.0, 0.001, 0.05, 0.5, 1.0])
def test_delta_records_match_oracle(eng, oracle, cb_len, density):
    rng = np.random.default_rng(int(cb_len * 1000 + density * 100))
    for runs in (False, True):
        base, target = states(rng, cb_len, density, runs=runs)
        db, dt = eng.upload_state(host(base)), eng.upload_state(host(target))
        got = eng.encode_record(dt, db)
        want = oracle.encode_record(target, base)
        assert got == want, (cb_len, density, runs, len(got), len(want))
        dec = eng.decode_record(got, base=db).download()
        for x, y in zip(dec.levels, target.levels):
            np.testing.assert_array_equal(x, y)
