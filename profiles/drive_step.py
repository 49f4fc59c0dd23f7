"""Small driver for ncu: C2 workload (GPT-2-small layout), FULL + a few DELTA steps.

Usage: python profiles/drive_step.py [steps] — prints per-step wall time and the
engine's per-kernel event profile."""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2306_11800_b200 import workloads as W  # noqa: E402


def main():
    import torch

    from paper_2306_11800_b200 import engine as E

    steps = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    dev = torch.device("cuda", 0)
    stream = torch.cuda.current_stream(dev)
    eng = E.Engine(0, stream.cuda_stream)
    layout = W.gpt2_small_layout()
    names = [n for n, _, _ in layout]
    types = [t for _, t, _ in layout]
    shapes = [s for _, _, s in layout]
    snaps, ema = W.series(torch, layout, steps + 1, 1234, dev)
    torch.cuda.synchronize()
    ck = []
    for s in snaps:
        c = E.DevCheckpoint(eng, names, types, shapes)
        c.set_weights(W.tensor_ptrs(s.data_ptr(), layout))
        c.set_ema(W.tensor_ptrs(ema.data_ptr(), layout))
        ck.append(c)
    cfg = E.Config()
    st = eng.quantize(ck[0], cfg, 1, 0)
    if os.environ.get("DQT_PROFILE"):
        eng.profile(True)
    for i in range(1, steps + 1):
        t = time.perf_counter()
        st2, r = eng.compress_step(ck[i], cfg, 1, i, st)
        eng.sync()
        print(f"step {i}: {1e3 * (time.perf_counter() - t):.2f} ms, record {E.LIB.dqtg_record_size(r)} B")
        E.LIB.dqtg_record_destroy(r)
        st = st2
    if os.environ.get("DQT_PROFILE"):
        for k, v in sorted(eng.profile_report().items(), key=lambda kv: -kv[1][1]):
            print(f"  {k}: {v[0]} launches {v[1]:.3f} ms")


if __name__ == "__main__":
    main()
