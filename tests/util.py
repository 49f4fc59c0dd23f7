"""Shared test inputs (seeded numpy generators; never /root/reference at run time)."""
import numpy as np

from oracle.oracle import Config, Tensor

# (name, layer type, shape) like tests/helpers.hpp small_checkpoint in the reference
SMALL_LAYOUT = [
    ("tok_embed.weight", 4, (100, 20)),
    ("blk.attn.qkv", 2, (100, 20)),
    ("blk.fc1.weight", 1, (100, 20)),
    ("blk.norm.weight", 3, (500,)),
    ("blk.fc1.bias", 5, (500,)),
    ("stem.conv.weight", 0, (30, 7)),
    ("head.weight", 6, (64, 3)),
]

CONFIGS = [
    Config(),
    Config(bins=8, embed_bins=16, prune_frac=0.1, protect_frac=0.01),
    Config(bins=4, embed_bins=16, prune_frac=0.5, protect_frac=0.0005, metric=1),
    Config(bins=32, embed_bins=32, prune_frac=0.0, protect_frac=0.0),
    Config(bins=6, embed_bins=32, prune_frac=0.3, protect_frac=0.9),   # protect/prune overlap
    Config(bins=12, embed_bins=16, prune_frac=0.2, protect_frac=0.005, metric=1, sigma=0.7,
           alpha=0.02),
]


def make_tensors(layout=SMALL_LAYOUT, seed=0, scale=0.05):
    rng = np.random.default_rng(seed)
    out = []
    for i, (name, lt, shape) in enumerate(layout):
        n = int(np.prod(shape))
        x = rng.normal(0.0, scale * (1 + 0.3 * i), n).astype(np.float32)
        if lt == 3:  # LayerNorm-like weights around 1
            x = (1.0 + 0.1 * rng.normal(size=n)).astype(np.float32)
        out.append(Tensor(name, lt, tuple(shape), x))
    return out


def flat(tensors):
    return np.concatenate([np.ascontiguousarray(t.data, np.float32).ravel() for t in tensors])


def perturb(tensors, seed, frac=0.05, scale=0.01):
    rng = np.random.default_rng(seed)
    out = []
    for t in tensors:
        x = t.data.copy()
        m = rng.random(x.size) < frac
        x[m] += (scale * rng.normal(size=int(m.sum()))).astype(np.float32)
        out.append(Tensor(t.name, t.type, t.shape, x))
    return out


_REF_DECODE_WORKER = r"""
import pickle, resource, sys
import numpy as np
lim = int(sys.argv[2]) << 30
resource.setrlimit(resource.RLIMIT_AS, (lim, lim))
sys.path.insert(0, sys.argv[1])
import dqtref as d
with open(sys.argv[3], "rb") as f:
    base_rec, recs = pickle.load(f)
base = d.decode_delta_record(base_rec) if base_rec is not None else None
out = []
for r in recs:
    try:
        q = d.decode_delta_record(r, base) if base is not None else d.decode_delta_record(r)
        out.append([np.asarray(t.levels, np.uint16).ravel().copy() for t in q.tensors])
    except BaseException as ex:  # noqa: BLE001 - bad_alloc / length_error count as rejects
        out.append(type(ex).__name__)
with open(sys.argv[3] + ".out", "wb") as f:
    pickle.dump(out, f)
"""


def ref_decode_many(records, base_record=None, mem_gb=6):
    """decode_delta_record of the reference (oracle/_ref) over many records in a
    child process with a bounded address space: corrupt counts make the reference
    allocate what the header claims (codec.cpp:541-580), which a memory limit
    turns into std::bad_alloc instead of an out-of-memory kill.  Returns per
    record the decoded levels (list of arrays) or the exception name."""
    import os
    import pickle
    import subprocess
    import sys
    import tempfile

    from oracle import ref as R

    fd, path = tempfile.mkstemp(suffix=".pkl")
    os.close(fd)
    try:
        with open(path, "wb") as f:
            pickle.dump((base_record, list(records)), f)
        subprocess.run([sys.executable, "-c", _REF_DECODE_WORKER, R.REF_DIR, str(mem_gb), path],
                       check=True)
        with open(path + ".out", "rb") as f:
            return pickle.load(f)
    finally:
        for p in (path, path + ".out"):
            if os.path.exists(p):
                os.unlink(p)
