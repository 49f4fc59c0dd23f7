"""DQT1 ingest throughput sweep: reader threads x staging chunk size, buffered and
O_DIRECT reads, on the C2 GPT-2-small snapshot (498 MB file, page cache warm for
buffered reads).  usage: python profiles/ingest_sweep.py"""
import os
import sys
import tempfile
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2306_11800_b200 import engine as E  # noqa: E402

layout = bench.gpt2_small_layout()
N = sum(bench.numel(s) for _, _, s in layout)
flat = np.random.default_rng(0).normal(0, 0.05, N).astype(np.float32)
eng = E.Engine(0)
fd, path = tempfile.mkstemp(suffix=".dqt")
os.close(fd)
bench.write_dqt1(path, layout, flat)
size = os.path.getsize(path)
print(f"file {size / 1e6:.1f} MB")
for chunk in (4, 8, 16, 32):
    os.environ["DQTG_INGEST_CHUNK_MB"] = str(chunk)
    for threads in (1, 2, 4, 8, 16):
        for direct in (False, True):
            eng.read_dqt1(path, direct=direct, threads=threads)
            ts = []
            for _ in range(3):
                t = time.perf_counter()
                ck, _, _ = eng.read_dqt1(path, direct=direct, threads=threads)
                ts.append(time.perf_counter() - t)
                del ck
            print(f"chunk {chunk:2d} MB threads {threads:2d} {'direct' if direct else 'cached'}: "
                  f"{size / min(ts) / 1e9:6.2f} GB/s ({1e3 * min(ts):.1f} ms)", flush=True)
os.unlink(path)
