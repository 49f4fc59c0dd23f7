"""Host-side cost of a sequential compress step (C2): wall time per step, host syncs
per step and the time blocked in them; wall - blocked = host work between syncs
(launch overhead, host-side table builds) during which this stream's GPU work is
not queued.  usage: python profiles/host_overhead.py [steps]"""
import os
import platform
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def cpu_info():
    model = ""
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                model = ln.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    t = time.perf_counter()
    x = 0
    for i in range(2_000_000):
        x += i
    return f"{model} | nproc {os.cpu_count()} | load {os.getloadavg()} | py-loop {1e3 * (time.perf_counter() - t):.1f} ms | {platform.release()}"


def main():
    import torch

    from paper_2306_11800_b200 import engine as E

    steps = int(sys.argv[1]) if len(sys.argv) > 1 else 8
    print(cpu_info())
    dev = torch.device("cuda", 0)
    eng = E.Engine(0, torch.cuda.current_stream(dev).cuda_stream)
    layout = bench.gpt2_small_layout()
    names = [n for n, _, _ in layout]
    types = [t for _, t, _ in layout]
    shapes = [s for _, _, s in layout]
    snaps, ema = bench.gen_series(torch, layout, steps + 1, 1234, dev)
    torch.cuda.synchronize()
    ck = []
    for s in snaps:
        c = E.DevCheckpoint(eng, names, types, shapes)
        c.set_weights(bench.tensor_ptrs(s.data_ptr(), layout))
        c.set_ema(bench.tensor_ptrs(ema.data_ptr(), layout))
        ck.append(c)
    cfg = E.Config()
    st = eng.quantize(ck[0], cfg, 1, 0)
    for i in range(1, steps + 1):
        n0, b0 = eng.sync_stats()
        t = time.perf_counter()
        st2, r = eng.compress_step(ck[i], cfg, 1, i, st)
        eng.sync()
        wall = 1e3 * (time.perf_counter() - t)
        n1, b1 = eng.sync_stats()
        print(f"step {i}: wall {wall:.3f} ms, syncs {n1 - n0}, blocked {b1 - b0:.3f} ms, "
              f"host {wall - (b1 - b0):.3f} ms")
        E.LIB.dqtg_record_destroy(r)
        st = st2


if __name__ == "__main__":
    main()
