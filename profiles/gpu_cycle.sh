# GPU round trip used during development: gpu tests, then one bench run, compact output
set -o pipefail
T=$(timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -1)
echo "TESTS: $T"
timeout 600 python bench.py --no-cpu-baseline "$@" > gpurun_out/bench.json 2> gpurun_out/bench.err || tail -5 gpurun_out/bench.err
python - <<'PY'
import json
d = json.load(open("gpurun_out/bench.json"))
k = d["roofline"]["kernels_ms_per_step"]
print("BENCH: value %.1f GB/s  %.3f ms/step  e2e %.1f  restore %s" % (
    d["value"], d["ms_per_step"], d["e2e"]["value"],
    None if not d.get("restore") else round(d["restore"]["value"], 1)))
print("KERNELS:", ", ".join("%s %.3f" % (n.replace("_kernel", ""), v) for n, v in list(k.items())[:12]))
PY
