"""DQT1 ingest into HBM (dqtg_ckpt_read_dqt1, ingest.cu) against the drop-in host
reader and the reference's read_checkpoint semantics (src/tensor.cpp:63-75,
110-149; tests/test_tensor.cpp): weights land bit-exactly at the device
checkpoint's padded offsets, step/meta/names/types/shapes round-trip, every
malformed file raises the reference's error type, and a record compressed from
an ingested checkpoint is byte-identical to one from host uploads."""
import struct

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

NON_FINITE, IO, TRUNC, BAD_MAGIC, SHAPE = 5, 6, 3, 2, 4


@pytest.fixture(scope="module")
def eng():
    from paper_2306_11800_b200 import engine as E

    return E.Engine(0)


def dqt1_bytes(tensors, step=0, meta=None, version=1, magic=b"DQT1"):
    """write_checkpoint (src/tensor.cpp:77-98): tensors = [(name, type, shape, f32 array)]."""
    out = [magic, struct.pack("<IQ", version, step)]
    meta = meta or {}
    out.append(struct.pack("<I", len(meta)))
    for k in sorted(meta):
        kb, vb = k.encode(), meta[k].encode()
        out += [struct.pack("<H", len(kb)), kb, struct.pack("<I", len(vb)), vb]
    out.append(struct.pack("<I", len(tensors)))
    for name, lt, shape, data in tensors:
        nb = name.encode()
        out += [struct.pack("<H", len(nb)), nb, struct.pack("<BB", lt, len(shape))]
        out += [struct.pack("<Q", d) for d in shape]
        out.append(np.ascontiguousarray(data, np.float32).tobytes())
    return b"".join(out)


def rand_tensors(seed, n=12, max_numel=50000):
    rng = np.random.default_rng(seed)
    ts = []
    for i in range(n):
        rank = int(rng.integers(1, 4))
        shape = tuple(int(x) for x in rng.integers(1, int(max_numel ** (1 / rank)) + 1, rank))
        # odd-length names misalign the data sections inside the file
        name = f"layer{i}." + "x" * int(rng.integers(0, 7)) + ".weight"
        ts.append((name, int(rng.integers(0, 7)), shape,
                   rng.normal(0, 0.05, int(np.prod(shape))).astype(np.float32)))
    return ts


def check_same(ck, tensors):
    assert ck.meta.names == [t[0] for t in tensors]
    assert ck.meta.types == [t[1] for t in tensors]
    assert ck.meta.shapes == [tuple(t[2]) for t in tensors]
    got = ck.download()
    for (name, _, _, data), g in zip(tensors, got):
        assert g.view(np.uint32).tobytes() == np.asarray(data, np.float32).view(np.uint32).tobytes(), name


@pytest.mark.parametrize("threads", [1, 3, 8])
def test_ingest_roundtrip(eng, tmp_path, threads):
    ts = rand_tensors(threads)
    p = tmp_path / "a.dqt"
    p.write_bytes(dqt1_bytes(ts, step=77, meta={"note": "s1", "beta": "0.9"}))
    ck, step, meta = eng.read_dqt1(str(p), threads=threads)
    assert step == 77 and meta == {"beta": "0.9", "note": "s1"}
    check_same(ck, ts)


def test_ingest_matches_dropin_reader(eng, tmp_path):
    """The host drop-in read_checkpoint (tensor.cpp restatement) sees the same file."""
    from paper_2306_11800_b200 import dqt

    c = dqt.Checkpoint()
    c.step = 5
    c.meta = {"run": "x"}
    rng = np.random.default_rng(2)
    for i, lt in enumerate([dqt.LayerType.EMBEDDING, dqt.LayerType.ATTENTION, dqt.LayerType.NORM]):
        c.add_tensor(f"t{i}", rng.normal(size=(37 + i, 11)).astype(np.float32), lt)
    p = str(tmp_path / "c.dqt")
    dqt.write_checkpoint(p, c)
    ck, step, meta = eng.read_dqt1(p)
    back = dqt.read_checkpoint(p)
    assert step == back.step == 5 and meta == dict(back.meta)
    got = ck.download()
    for t, g in zip(back.tensors, got):
        np.testing.assert_array_equal(np.asarray(t.data, np.float32).ravel(), g)


def test_ingest_large_direct(eng, tmp_path):
    """Hundreds of MiB across many chunks, buffered and O_DIRECT reads."""
    rng = np.random.default_rng(9)
    ts = [("emb", 4, (20000, 1024), rng.normal(0, 0.05, 20000 * 1024).astype(np.float32)),
          ("b", 5, (3,), np.array([1, 2, 3], np.float32)),
          ("fc", 1, (4097, 513), rng.normal(0, 0.05, 4097 * 513).astype(np.float32)),
          ("z", 6, (0, 5), np.zeros(0, np.float32))]
    p = tmp_path / "big.dqt"
    p.write_bytes(dqt1_bytes(ts, step=3))
    for direct in (False, True):
        ck, step, _ = eng.read_dqt1(str(p), direct=direct)
        assert step == 3
        check_same(ck, ts)


def test_ingest_empty_checkpoint(eng, tmp_path):
    p = tmp_path / "e.dqt"
    p.write_bytes(dqt1_bytes([], step=9, meta={"k": ""}))
    ck, step, meta = eng.read_dqt1(str(p))
    assert step == 9 and meta == {"k": ""} and ck.meta.names == []


def test_ingest_errors(eng, tmp_path):
    from paper_2306_11800_b200 import engine as E

    good = [("w", 6, (2,), np.array([1, 2], np.float32)), ("v", 6, (1,), np.array([3], np.float32))]
    nan = np.array([1, np.nan], np.float32)
    inf = np.array([np.inf], np.float32)
    cases = {
        "magic": (dqt1_bytes(good, magic=b"DQT2"), BAD_MAGIC),
        "version": (dqt1_bytes(good, version=2), IO),
        "truncated": (dqt1_bytes(good)[:-3], TRUNC),
        "truncated_header": (dqt1_bytes(good)[:10], TRUNC),
        "trailing": (dqt1_bytes(good) + b"\0", IO),
        "rank0": (dqt1_bytes([("w", 6, (), np.zeros(1, np.float32))]), SHAPE),
        "badtype": (dqt1_bytes([("w", 7, (1,), np.ones(1, np.float32))]), IO),
        "nan": (dqt1_bytes([good[0], ("v", 6, (2,), nan)]), NON_FINITE),
        "inf_last": (dqt1_bytes([good[0], ("v", 6, (1,), inf)]), NON_FINITE),
        "dup": (dqt1_bytes([good[0], ("w", 6, (1,), np.ones(1, np.float32))]), IO),
        "empty_name": (dqt1_bytes([("", 6, (1,), np.ones(1, np.float32))]), IO),
        # validate() walks tensors in order: NaN in tensor 0 wins over a later duplicate,
        # a duplicate at tensor 1 wins over NaN in tensor 2
        "nan_before_dup": (dqt1_bytes([("w", 6, (2,), nan), ("w", 6, (1,), np.ones(1, np.float32))]),
                           NON_FINITE),
        "dup_before_nan": (dqt1_bytes([good[0], ("w", 6, (1,), np.ones(1, np.float32)),
                                       ("n", 6, (2,), nan)]), IO),
        "huge_dims": (dqt1_bytes([("w", 6, (1 << 40, 3), np.ones(1, np.float32))]), TRUNC),
        # the element count wraps to 0 (NamedTensor::size() in u64): the data is trailing
        "wrapped_dims": (dqt1_bytes([("w", 6, (1 << 40, 1 << 30), np.ones(1, np.float32))]), IO),
    }
    for name, (blob, code) in cases.items():
        p = tmp_path / f"{name}.dqt"
        p.write_bytes(blob)
        with pytest.raises(E.EngineError) as ex:
            eng.read_dqt1(str(p))
        assert ex.value.status == code, (name, ex.value)
    with pytest.raises(E.EngineError) as ex:
        eng.read_dqt1(str(tmp_path / "missing.dqt"))
    assert ex.value.status == IO


def test_ingest_dropin_error_types_agree(eng, tmp_path):
    """The drop-in host reader rejects the same files (its module, like the reference's
    py_module.cpp:50-60, surfaces the reader's exceptions as dqt.Error)."""
    from paper_2306_11800_b200 import dqt
    from paper_2306_11800_b200 import engine as E

    good = [("w", 6, (2,), np.array([1, 2], np.float32))]
    for blob, code in ((dqt1_bytes(good, magic=b"XXXX"), BAD_MAGIC), (dqt1_bytes(good)[:-1], TRUNC),
                       (dqt1_bytes(good) + b"!", IO),
                       (dqt1_bytes([("w", 6, (1,), np.array([np.nan], np.float32))]), NON_FINITE)):
        p = str(tmp_path / "x.dqt")
        open(p, "wb").write(blob)
        with pytest.raises(E.EngineError) as ex:
            eng.read_dqt1(p)
        assert ex.value.status == code
        with pytest.raises(dqt.Error):
            dqt.read_checkpoint(p)


def test_ingest_then_compress_matches_upload(eng, tmp_path):
    """quantize + encode from the ingested checkpoint == from host uploads."""
    from paper_2306_11800_b200 import dqt
    from paper_2306_11800_b200 import engine as E

    ts = rand_tensors(5, n=6, max_numel=200000)
    p = tmp_path / "q.dqt"
    p.write_bytes(dqt1_bytes(ts, step=4))
    ck, step, _ = eng.read_dqt1(str(p))
    rules = dqt.default_layer_rules()
    types = [int(dqt.classify_layer_type(n, rules)) for n in ck.meta.names]
    ck.set_types(types)
    ref = eng.checkpoint(ck.meta.names, types, ck.meta.shapes, weights=[t[3] for t in ts])
    cfg = E.Config()
    r1 = eng.encode_record(eng.quantize(ck, cfg, 1, step))
    r2 = eng.encode_record(eng.quantize(ref, cfg, 1, step))
    assert r1 == r2


def test_ema_file_ingest(eng, tmp_path):
    """ema_save (drop-in) -> read_ema_dqt1 -> set_ema_from: the quantized state equals
    the one built from the host EMA arrays; update_ema_from matches host updates."""
    from paper_2306_11800_b200 import dqt
    from paper_2306_11800_b200 import engine as E

    ts = rand_tensors(7, n=5, max_numel=100000)
    names = [t[0] for t in ts]
    rules = dqt.default_layer_rules()
    types = [int(dqt.classify_layer_type(n, rules)) for n in names]
    shapes = [t[2] for t in ts]
    rng = np.random.default_rng(3)
    grads = [rng.normal(0, 0.01, t[3].size).astype(np.float32) for t in ts]
    g = dqt.Checkpoint()
    for (name, _, shape, _), gr, lt in zip(ts, grads, types):
        g.add_tensor(name, gr.reshape(shape), dqt.LayerType(lt))
    ema = dqt.ema_init(0.8)
    dqt.ema_update(ema, g)
    p = str(tmp_path / "ema.dqt")
    dqt.ema_save(p, ema)
    eck, beta, count = eng.read_ema_dqt1(p)
    assert beta == 0.8 and count == 1
    w = [t[3] for t in ts]
    a = eng.checkpoint(names, types, shapes, weights=w)
    a.set_ema_from(eck)
    b = eng.checkpoint(names, types, shapes, weights=w, ema=grads)
    cfg = E.Config(metric=1)
    assert eng.encode_record(eng.quantize(a, cfg, 1, 2)) == eng.encode_record(eng.quantize(b, cfg, 1, 2))
    # a second gradient snapshot from a file, applied on the device
    g2 = [rng.normal(0, 0.01, x.size).astype(np.float32) for x in w]
    p2 = tmp_path / "g2.dqt"
    p2.write_bytes(dqt1_bytes([(n, lt, s, x) for n, lt, s, x in zip(names, types, shapes, g2)]))
    gck, _, _ = eng.read_dqt1(str(p2))
    a.update_ema_from(gck, beta)
    b.update_ema(g2, beta)
    assert eng.encode_record(eng.quantize(a, cfg, 1, 3)) == eng.encode_record(eng.quantize(b, cfg, 1, 3))
    p3 = tmp_path / "nometa.dqt"
    p3.write_bytes(dqt1_bytes([(names[0], 6, shapes[0], w[0])]))
    with pytest.raises(E.EngineError) as ex:
        eng.read_ema_dqt1(str(p3))
    assert ex.value.status == 6
