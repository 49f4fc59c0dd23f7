# sparse DELTA encoder: parity tests, per-kernel times (sparse vs dense), one ncu capture
python -m pytest tests/test_delta_density_gpu.py tests/test_gpu_parity.py -q -x 2>&1 | tail -2
DQT_PROFILE=1 python profiles/drive_step.py 4 2>&1 | grep -E "step|enc_|pass_"
DQT_PROFILE=1 DQTG_DENSE_DELTA=1 python profiles/drive_step.py 4 2>&1 | grep -E "enc_tile"
ncu --set full --import-source on --clock-control none -k regex:enc_tile_delta -s 1 -c 1 -o gpurun_out/ncu_delta python profiles/drive_step.py 3 > gpurun_out/ncu_delta.log 2>&1
tail -1 gpurun_out/ncu_delta.log
