ncu --set full --clock-control none --import-source on -k regex:psh_kernel -s 16 -c 1 -o gpurun_out/psh_D python tools/psh_bench.py > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/psh_D.ncu-rep
