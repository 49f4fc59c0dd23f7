"""Hand-built DQDR records at the edges of decode_delta_record (reference
codec.cpp:234-273 huffman_decode, :56-77 unrearrange, :513-597): the device decoder
must accept exactly what the reference (oracle/_ref, compiled from its sources)
accepts and decode it to the same levels.

* a fixed-length code (8 equally likely symbols -> every code 3 bits) over far
  more than 64 bitstream chunks: wrong chunk phases never fall back into step by
  themselves (decode.cu chunk sync)
* an overfull table ({1, 1, 2} bit lengths): Kraft sum > 1 -> CorruptBitstream
* a group without symbols carries a garbage table: the reference never validates it
* groups listed in descending bucket order: the reference accepts any order
* a table entry holding an out-of-range symbol that is never decoded
"""
import struct
import zlib

import numpy as np
import pytest

from oracle.oracle import QState

pytestmark = pytest.mark.gpu


def uv(v):
    out = bytearray()
    while v >= 0x80:
        out.append((v & 0x7F) | 0x80)
        v >>= 7
    out.append(v)
    return bytes(out)


def sv(v):
    return uv(((v << 1) ^ (v >> 63)) & (2**64 - 1))


def record(levels, cb_len, groups, B, has_base=False, base_step=0, step=1, lt=1, prot=()):
    """DQDR v1: one tensor `t` of layer type `lt`; groups =
    [(bucket, elems, nsyms, [(sym, len)...], bytes)]."""
    levels = np.asarray(levels, np.uint16)
    w = bytearray(b"DQDR") + struct.pack("<IBQQI", 1, int(has_base), base_step, step, B)
    w += struct.pack("<IIddBdd", 16, 32, 0.0, 0.005, 0, 0.2, 0.01) + struct.pack("<d", 0.0)
    w += struct.pack("<B", 1) + struct.pack("<BI", lt, cb_len)
    w += np.linspace(-1, 1, cb_len).astype(np.float32).tobytes()
    w += struct.pack("<I", 1) + struct.pack("<H", 1) + b"t" + struct.pack("<BB", lt, 1)
    w += struct.pack("<Q", len(levels)) + uv(len(prot))
    last = 0
    for i, (p, v) in enumerate(prot):
        w += uv(p if i == 0 else p - last) + struct.pack("<H", v)
        last = p
    w += uv(len(groups))
    for bucket, elems, nsyms, table, bits in groups:
        w += uv(bucket) + uv(elems) + uv(nsyms) + uv(len(table))
        for s, ln in table:
            w += sv(s) + struct.pack("<B", ln)
        w += uv(len(bits)) + bytes(bits)
    w += struct.pack("<I", zlib.crc32(levels.astype("<u2").tobytes()) & 0xFFFFFFFF)
    return bytes(w)


def state(levels, cb_len, step, lt=1):
    cbs = [np.zeros(0, np.float32) for _ in range(7)]
    cbs[lt] = np.linspace(-1, 1, cb_len).astype(np.float32)
    lv = np.asarray(levels, np.uint16)
    return QState(step, (16, 32, 0.0, 0.005, 0, 0.2, 0.01), cbs, ["t"], [lt], [(len(lv),)],
                  [lv], [np.zeros(0, np.uint64)], [np.zeros(0, np.uint16)])


def both(eng, ref, rec, base_dev=None, base_ref=None):
    """(device levels or status, reference levels or exception name)"""
    from paper_2306_11800_b200 import engine as E

    d = ref.load()
    try:
        got = eng.decode_record(rec, base=base_dev).download().levels[0]
    except E.EngineError as ex:
        got = ex.kind
    try:
        q = d.decode_delta_record(rec, base_ref) if base_ref is not None else d.decode_delta_record(rec)
        want = np.asarray(q.tensors[0].levels, np.uint16).ravel()
    except Exception as ex:  # noqa: BLE001 - the reference's exception type is the answer
        want = type(ex).__name__
    return got, want


def ref_state(ref, levels, cb_len, step, lt=1):
    """A reference QuantizedCheckpoint holding `levels` (decoded from a record the
    oracle writes)."""
    from oracle import oracle as O

    rec = O.get().encode_record(state(levels, cb_len, step, lt))
    return ref.load().decode_delta_record(rec), rec


@pytest.fixture(scope="module")
def eng():
    from paper_2306_11800_b200 import engine as E

    return E.Engine(0)


def test_fixed_length_code_many_chunks(eng, ref, oracle):
    rng = np.random.default_rng(5)
    n = 1 << 20
    step = rng.integers(1, 8, n).astype(np.uint16)  # never 0: no two neighbours equal
    lv = (np.cumsum(step) % 8).astype(np.uint16)
    q = state(lv, 8, 1)  # B = 10, FULL deltas (10 - l) % 10: 8 symbols, 1 element each
    rec = oracle.encode_record(q)
    got, want = both(eng, ref, rec)
    assert isinstance(want, np.ndarray), want
    np.testing.assert_array_equal(got, want)
    np.testing.assert_array_equal(got, lv)
    # and as a DELTA against a base with a different phase pattern
    lv2 = lv.copy()
    lv2[::3] = (lv2[::3] + 1) % 8
    rec2 = oracle.encode_record(state(lv2, 8, 2), q)
    base_dev = eng.decode_record(rec)
    base_ref, _ = ref_state(ref, lv, 8, 1)
    got, want = both(eng, ref, rec2, base_dev, base_ref)
    assert isinstance(want, np.ndarray), want
    np.testing.assert_array_equal(got, want)
    np.testing.assert_array_equal(got, lv2)


def test_overfull_table_rejected(eng, ref):
    # 4 zero levels, B = 4: symbols [0, 4] ('value 0, run 4'), table lengths {1, 1, 2}
    rec = record([0] * 4, 2, [(0, 4, 2, [(0, 1), (4, 1), (5, 2)], [0x40])], B=4)
    got, want = both(eng, ref, rec)
    assert isinstance(want, str), want  # the module maps CorruptBitstream to dqt.Error
    assert got == "CorruptBitstream"
    # the same stream with a complete table decodes on both sides
    ok = record([0] * 4, 2, [(0, 4, 2, [(0, 1), (4, 1)], [0x40])], B=4)
    got, want = both(eng, ref, ok)
    np.testing.assert_array_equal(got, want)


def test_empty_group_garbage_table_accepted(eng, ref):
    garbage = [(7, 0), (3, 70), (1, 2), (1, 1)]  # zero / too long / non-canonical lengths
    rec = record([0] * 4, 2, [(0, 4, 2, [(0, 1), (4, 1)], [0x40]), (1, 0, 0, garbage, [])], B=4)
    got, want = both(eng, ref, rec)
    assert isinstance(want, np.ndarray), want
    np.testing.assert_array_equal(got, want)


def test_unused_out_of_range_symbol_accepted(eng, ref):
    # codes: -2^40 '00', 0 '01', 4 '10', 2^40 '11'; stream [0, 4] = '0110'
    rec = record([0] * 4, 2, [(0, 4, 2, [(-(1 << 40), 2), (0, 2), (4, 2), (1 << 40, 2)],
                               [0b01100000])], B=4)
    got, want = both(eng, ref, rec)
    assert isinstance(want, np.ndarray), want
    np.testing.assert_array_equal(got, want)


def test_group_order_is_free(eng, ref):
    # base levels [0, 1, 0, 1]; target [1, 1, 0, 0] -> deltas (p - c) mod 4 = [3, 0, 0, 1]
    # groups: bucket 0 -> [3, 0], bucket 1 -> [0, 1]; RLE symbols [-3, 0] and [0, -1]
    base_lv, target = [0, 1, 0, 1], [1, 1, 0, 0]
    base_ref, base_rec = ref_state(ref, base_lv, 2, 1)
    base_dev = eng.decode_record(base_rec)
    tab = [(0, 1), (-3, 2), (-1, 2)]  # codes: 0 -> '0', -3 -> '10', -1 -> '11'
    g0 = (0, 2, 2, tab, [0b10000000])  # -3, 0
    g1 = (1, 2, 2, tab, [0b01100000])  # 0, -1
    for groups in ([g0, g1], [g1, g0]):
        rec = record(target, 2, groups, B=4, has_base=True, base_step=1, step=2)
        got, want = both(eng, ref, rec, base_dev, base_ref)
        assert isinstance(want, np.ndarray), want
        np.testing.assert_array_equal(got, want)
        np.testing.assert_array_equal(got, np.asarray(target, np.uint16))
    dup = record(target, 2, [g0, g0], B=4, has_base=True, base_step=1, step=2)
    got, want = both(eng, ref, dup, base_dev, base_ref)
    assert isinstance(want, str) and isinstance(got, str), (got, want)
