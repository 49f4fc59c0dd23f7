# one ncu --set full capture (with source) of kernel regex $1 in a C2 DELTA step:
# profiles/drive_step.py 2 (step 0 quantize, compress_step 1 and 2), launch $2 of the
# matching ones (default 1 = the second); summary + raw CSV + source CSV
K=$1; S=${2:-1}; TAG=${3:-k}
ncu --set full --import-source on --clock-control none -k regex:$K -s $S -c 1 \
    -o gpurun_out/ncu_$TAG python profiles/drive_step.py 2 > gpurun_out/ncu_$TAG.log 2>&1
tail -1 gpurun_out/ncu_$TAG.log
python profiles/ncu_summary.py gpurun_out/ncu_$TAG.ncu-rep gpurun_out/ncu_$TAG.md > /dev/null
ncu -i gpurun_out/ncu_$TAG.ncu-rep --page raw --csv > gpurun_out/ncu_${TAG}_raw.csv
ncu -i gpurun_out/ncu_$TAG.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/ncu_${TAG}_src.csv
rm -f gpurun_out/ncu_$TAG.ncu-rep
