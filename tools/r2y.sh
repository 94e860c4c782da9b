ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:"bswin_attn_tc|gemm_kernel|psh_kernel|pool_build|pool_reduce|row_ln_vec|scatter_ln_pe|fused_hash|fused_min" -o gpurun_out/step_B_r2b python tools/prof_step.py > gpurun_out/r2y_step.log 2>&1
ncu --set full --clock-control none -k regex:bswin_attn_tc -s 3 -c 1 -o gpurun_out/attn_D_r2 python tools/attn_bench.py --config D --iters 1 > gpurun_out/r2y_attnD.log 2>&1
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2y_train_launches.csv python tools/train_bench.py --scenes 1 --steps 1 --warmup 1 --no-graph > gpurun_out/r2y_train.log 2>&1
ls -la gpurun_out/*.ncu-rep
