set -o pipefail
nvidia-smi -L
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -8
timeout 400 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; cat gpurun_out/bench.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('value',d['value'],'ms',d['ms_per_step'],'seq',d['config']['ms_per_step_sequential'],'e2e',d['e2e']['value']); print(d['roofline']['kernels_ms_per_step'])"; tail -3 gpurun_out/bench.err
