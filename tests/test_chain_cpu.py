"""DeviceChain manifest handling on the host (Chain::open, src/chain.cpp:22-70):
a fresh directory gets the reference header; malformed manifests raise
ChainCorrupt (status 16) for the same conditions as the reference."""
import os

import pytest


def _open(d, text, full_every=50):
    from paper_2306_11800_b200.chain import DeviceChain

    os.makedirs(d, exist_ok=True)
    with open(os.path.join(d, "manifest.txt"), "w") as f:
        f.write(text)
    return DeviceChain(None, d, full_every)


def test_fresh_and_reopen(tmp_path):
    from paper_2306_11800_b200.chain import DeviceChain

    d = str(tmp_path / "c")
    ch = DeviceChain(None, d, 5)
    head = open(os.path.join(d, "manifest.txt")).read()
    assert head == f"# dqt-chain {ch.id}\n" and len(ch.id) == 16 and ch.empty()
    ch2 = _open(d, head + "3,FULL,rec-000000000003.dqdr,\n4,DELTA,rec-000000000004.dqdr,3\n\n")
    assert ch2.id == ch.id and [e.step for e in ch2.entries] == [3, 4]
    assert ch2.entries[1].base_step == 3 and ch2.latest_step() == 4
    assert not ch2._next_is_full()
    ch3 = _open(d, head + "3,FULL,a,\n4,DELTA,b,3\n", full_every=2)
    assert ch3._next_is_full()


@pytest.mark.parametrize("body", [
    "garbage\n",                                   # header missing
    "# dqt-chain x\n1,FULL\n",                     # malformed line
    "# dqt-chain x\n1,HALF,a,\n",                  # unknown kind
    "# dqt-chain x\n1,DELTA,a,0\n",                # first entry not FULL
    "# dqt-chain x\n2,FULL,a,\n1,FULL,b,\n",       # steps not ascending
    "# dqt-chain x\n1,FULL,a,\n3,DELTA,b,2\n",     # delta does not chain
    "# dqt-chain x\n1,FULL,a,\n2,DELTA,b,\n",      # delta without base
])
def test_corrupt_manifests(tmp_path, body):
    from paper_2306_11800_b200.chain import ChainError

    with pytest.raises(ChainError) as ex:
        _open(str(tmp_path / "c"), body)
    assert ex.value.status == 16


def test_full_every_zero(tmp_path):
    from paper_2306_11800_b200.chain import ChainError, DeviceChain

    with pytest.raises(ChainError):
        DeviceChain(None, str(tmp_path / "z"), 0)
