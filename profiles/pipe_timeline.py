"""Per-launch timeline of the native pipelined chain (dqtg_pipe_*).
DQTG_TIMELINE=1 WORKERS=4 python profiles/pipe_timeline.py [snapshots] [reps] 2> timeline.txt
prints ms/step per repetition on stdout; launch spans (ms since a process epoch,
per worker stream) on stderr."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def main():
    import torch

    from paper_2306_11800_b200 import engine as E
    from paper_2306_11800_b200.pipeline import ChainCompressor

    n = int(sys.argv[1]) if len(sys.argv) > 1 else 12
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    dev = torch.device("cuda", 0)
    layout = bench.gpt2_small_layout()
    names = [a for a, _, _ in layout]
    types = [t for _, t, _ in layout]
    shapes = [s for _, _, s in layout]
    snaps, ema = bench.gen_series(torch, layout, n, 1234, dev)
    torch.cuda.synchronize()
    cc = ChainCompressor(0, workers=int(os.environ.get("WORKERS", "4")))
    ck = []
    for s in snaps:
        c = cc.checkpoint(names, types, shapes)
        c.set_weights(bench.tensor_ptrs(s.data_ptr(), layout))
        c.set_ema(bench.tensor_ptrs(ema.data_ptr(), layout))
        ck.append(c)
    base = cc.run(ck[:2], E.Config(), 1, [0, 1])
    for r in range(reps):
        t = time.perf_counter()
        cc.run(ck[2:], E.Config(), 1, list(range(2, n)), base=base)
        dt = time.perf_counter() - t
        print(f"rep {r}: {1e3 * dt / (n - 2):.3f} ms/step", flush=True)
        print(f"--- rep {r} end", file=sys.stderr, flush=True)


if __name__ == "__main__":
    main()
