# one ncu --set full capture of kernel $1 (regex) in the C2 step driver
ncu --set full --import-source on --clock-control none -k regex:$1 -s ${2:-1} -c 1 -o gpurun_out/ncu_$1 python profiles/drive_step.py 3 > gpurun_out/ncu_$1.log 2>&1
tail -1 gpurun_out/ncu_$1.log
