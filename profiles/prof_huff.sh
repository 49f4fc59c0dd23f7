ncu --set full --import-source on --clock-control none -k regex:enc_huffman --launch-skip 3 -c 3 -o gpurun_out/ncu_huf python profiles/drive_step.py 2 > gpurun_out/ncu_huf.log 2>&1
tail -1 gpurun_out/ncu_huf.log
python profiles/ncu_summary.py gpurun_out/ncu_huf.ncu-rep gpurun_out/ncu_huf.md > /dev/null
ncu -i gpurun_out/ncu_huf.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/ncu_huf_src.csv
ncu -i gpurun_out/ncu_huf.ncu-rep --page raw --csv > gpurun_out/ncu_huf_raw.csv
rm -f gpurun_out/ncu_huf.ncu-rep
