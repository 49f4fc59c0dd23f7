"""Corrupt-record parity against the reference's decode_delta_record
(codec.cpp:459-597): 600 single-byte corruptions of a FULL and a DELTA record.
Accept/reject agrees with the reference compiled from its sources (oracle/_ref)
and with the oracle's restatement for EVERY corruption; whenever both accept,
the decoded levels are identical; the error class (the oracle's, the reference
module maps most classes to dqt.Error) agrees for >= 95 % of the rejected ones
(the remaining
cases are corruptions where the reference reports the first failing check in its
sequential tensor order while the device decoder checks all tensors' bitstreams
first, or absurd counts where the reference's reserve() throws std::length_error,
which has no dqt type)."""
import numpy as np
import pytest

from tests.util import CONFIGS, flat, make_tensors, perturb, ref_decode_many

pytestmark = pytest.mark.gpu

# oracle error code -> dqtg_status (include/dqtg.h)
STATUS = {1: 1, 5: 13, 6: 14, 7: 15, 8: 4, 9: 16, 10: 3, 11: 2, 12: 6}


def test_corrupt_records_match_oracle(oracle, ref):  # noqa: ARG001 (ref: oracle/_ref built)
    from oracle import oracle as O
    from paper_2306_11800_b200 import engine as E

    eng = E.Engine(0)
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
    agree = total = 0
    mismatch = []
    for rec, b, qb, base_rec in ((full, None, None, None), (delta, base, q1, full)):
        bads = []
        for _ in range(300):
            bad = bytearray(rec)
            bad[int(rng.integers(0, len(bad)))] ^= int(rng.integers(1, 256))
            bads.append(bytes(bad))
        # the reference itself (oracle/_ref), in a memory-bounded child process
        refs = ref_decode_many(bads, base_rec)
        for bad, r in zip(bads, refs):
            try:
                got = eng.decode_record(bad, base=b).download()
                ours = 0
            except E.EngineError as ex:
                got, ours = None, ex.status
            try:
                want = oracle.decode_record(bad, qb)
                theirs = 0
            except O.OracleError as ex:
                want, theirs = None, STATUS.get(ex.code, 100 + ex.code)
            ref_ok = not isinstance(r, str)
            total += 1
            if (ours == 0) != (theirs == 0) or (ours == 0) != ref_ok:
                mismatch.append((ours, theirs, r if not ref_ok else "accepted"))
            if ours == 0 and ref_ok:
                for x, y in zip(got.levels, r):
                    np.testing.assert_array_equal(x, y)
            if ours == 0 and theirs == 0:
                for x, y in zip(got.levels, want.levels):
                    np.testing.assert_array_equal(x, np.asarray(y).ravel())
            agree += ours == theirs
    assert not mismatch, mismatch  # accept/reject: exact
    assert agree >= 0.95 * total, (agree, total)
