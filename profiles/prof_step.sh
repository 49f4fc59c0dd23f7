# ncu --set full of the kernels of one C2 DELTA compress_step (profiles/drive_step.py 1:
# step 0 quantize, then compress_step 1), summary + raw CSV (+ profiles/ncu_traffic.json
# for bench.py's roofline); the report is dropped when it would not fit the 64 MiB
# gpurun_out limit.  usage: bash profiles/prof_step.sh TAG [launch-skip]
TAG=${1:-x}
K='regex:enc_tile|enc_huffman|enc_emit|enc_resolve_big|enc_bits|kmeans_restarts|pass_a2|pass_b_kernel|pass_c_kernel|cand_classify'
ncu --set full --import-source on --clock-control none -k "$K" --launch-skip ${2:-4} -c 12 \
    -o gpurun_out/ncu_$TAG python profiles/drive_step.py 1 > gpurun_out/ncu_$TAG.log 2>&1
tail -2 gpurun_out/ncu_$TAG.log
python profiles/ncu_summary.py gpurun_out/ncu_$TAG.ncu-rep gpurun_out/ncu_$TAG.md
ncu -i gpurun_out/ncu_$TAG.ncu-rep --page raw --csv > gpurun_out/ncu_${TAG}_raw.csv
sz=$(stat -c %s gpurun_out/ncu_$TAG.ncu-rep); echo "report bytes $sz"
if [ "$sz" -gt 50000000 ]; then rm gpurun_out/ncu_$TAG.ncu-rep; fi
