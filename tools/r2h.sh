ncu --set full --clock-control none --import-source on -k regex:bswin_attn_tc -s 3 -c 1 -o gpurun_out/attn_B_r2 python tools/attn_bench.py --config B --iters 1 > gpurun_out/r2h_ncu_attn.log 2>&1
ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:"psh_kernel|pool_build|gemm_kernel" -c 8 -o gpurun_out/step_B_r2 python tools/prof_step.py > gpurun_out/r2h_ncu_step.log 2>&1
bash tools/sanitize.sh
ls -la gpurun_out/*.ncu-rep
