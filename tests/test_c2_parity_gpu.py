"""Full-size parity at the bench's own configuration (BASELINE.json configs[1], C2:
GPT-2 small, 124,439,808 fp32 params, 148 tensors incl. the 38.6 M-element wte).

The bench's input series (paper_2306_11800_b200/workloads.py) is compressed on
the device and by the reference compiled from its sources (oracle/_ref) on the
SAME bytes: gradient EMA (ema_update, ranker.cpp:21-37), scores (compute_scores,
:79-101), quantize_checkpoint (quantize.cpp:373-425) of three snapshots, then
encode_delta_record (codec.cpp:398-460) FULL(q0), DELTA(q0 -> q1), DELTA(q1 -> q2).
Asserted: the EMA bytes, every tensor's levels, protected entries and codebooks,
and the three records byte for byte; the device decoder restores the reference's
records to the reference's levels.  (~1 min of reference CPU time.)"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_c2_records_match_reference(ref, tmp_path):
    import torch

    from paper_2306_11800_b200 import engine as E
    from paper_2306_11800_b200 import workloads as W

    d = ref.load()
    dev = torch.device("cuda", 0)
    layout = W.gpt2_small_layout()
    names = [n for n, _, _ in layout]
    types = [t for _, t, _ in layout]
    shapes = [s for _, _, s in layout]
    tr = W.Trajectory(torch, W.layout_params(layout), 1234, dev)  # the bench's rank-0 seed
    snaps = [tr.next() for _ in range(3)]
    ema = tr.ema()

    def ref_ckpt(flat_dev, step):
        host = flat_dev.cpu().numpy()
        c = d.Checkpoint()
        c.step = step
        for (name, lt, shape), x in zip(layout, W.split(host, layout)):
            c.add_tensor(name, x.reshape(shape), d.LayerType(lt))
        return c

    # the EMA the bench feeds the engine == the reference's own ema_update of the
    # same gradients (read back through the reference's ema_save / read_checkpoint)
    rema = d.ema_init(0.9)
    for k, g in enumerate(tr.grads):
        d.ema_update(rema, ref_ckpt(g, k + 1))
    path = str(tmp_path / "ema.dqt")
    d.ema_save(path, rema)
    saved = d.read_checkpoint(path)
    for x, t in zip(W.split(ema.cpu().numpy(), layout), saved.tensors):
        assert np.array_equal(x.view(np.uint32),
                              np.asarray(t.data, np.float32).ravel().view(np.uint32)), t.name
    del saved

    eng = E.Engine(0)
    cfg = E.Config()
    rcfg = d.QuantConfig()
    dev_states, ref_states = [], []
    for k, s in enumerate(snaps):
        ck = E.DevCheckpoint(eng, names, types, shapes)
        ck.set_weights(W.tensor_ptrs(s.data_ptr(), layout))
        ck.set_ema(W.tensor_ptrs(ema.data_ptr(), layout))
        dev_states.append(eng.quantize(ck, cfg, 1, k))
        rc = ref_ckpt(s, k)
        ref_states.append(d.quantize_checkpoint(rc, d.compute_scores(rc, rema), rcfg, 1))
        del rc
    torch.cuda.synchronize()

    for k, (ds, rs) in enumerate(zip(dev_states, ref_states)):
        got = ds.download()
        want = ref.qstate(rs)
        assert got.step == want.step
        for lt in range(7):
            np.testing.assert_array_equal(np.asarray(got.codebooks[lt]).view(np.uint32),
                                          np.asarray(want.codebooks[lt]).view(np.uint32))
        for i, name in enumerate(names):
            assert np.array_equal(got.levels[i], want.levels[i]), (k, name)
            assert np.array_equal(got.prot_pos[i], want.prot_pos[i]), (k, name)
            assert np.array_equal(got.prot_val[i], want.prot_val[i]), (k, name)

    pairs = [(0, None), (1, 0), (2, 1)]
    for t, b in pairs:
        ours = eng.encode_record(dev_states[t], None if b is None else dev_states[b])
        theirs = bytes(d.encode_delta_record(ref_states[t], None if b is None else ref_states[b]))
        assert len(ours) == len(theirs), (t, len(ours), len(theirs))
        assert ours == theirs, t
        # the device decoder restores the reference's record
        base = None if b is None else eng.decode_record(
            bytes(d.encode_delta_record(ref_states[b])))
        got = eng.decode_record(theirs, base=base).download()
        want = ref.qstate(ref_states[t])
        for i in range(len(names)):
            assert np.array_equal(got.levels[i], want.levels[i]), (t, names[i])

    # Chain::append through dqtg_compress_step: pass C fused into the DELTA encoder
    # (the levels are computed in the encoder's tile pass and never re-read)
    for t, b in pairs[1:]:
        ck = E.DevCheckpoint(eng, names, types, shapes)
        ck.set_weights(W.tensor_ptrs(snaps[t].data_ptr(), layout))
        ck.set_ema(W.tensor_ptrs(ema.data_ptr(), layout))
        st, rh = eng.compress_step(ck, cfg, 1, t, base=dev_states[b])
        ours = eng.record_bytes(rh)
        theirs = bytes(d.encode_delta_record(ref_states[t], ref_states[b]))
        assert ours == theirs, ("compress_step", t)
        got = st.download()
        want = ref.qstate(ref_states[t])
        for i, name in enumerate(names):
            assert np.array_equal(got.levels[i], want.levels[i]), ("compress_step", t, name)
            assert np.array_equal(got.prot_pos[i], want.prot_pos[i]), ("compress_step", t, name)
            assert np.array_equal(got.prot_val[i], want.prot_val[i]), ("compress_step", t, name)
