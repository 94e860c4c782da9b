mkdir -p gpurun_out
P="ncu --profile-from-start off --set full --clock-control none --import-source on"
$P -k regex:bswin_attn_tc -c 2 -o gpurun_out/z_attn python tools/prof_step.py > /dev/null 2>&1
$P -k regex:gemm_kernel -c 4 -o gpurun_out/z_gemm python tools/prof_step.py > /dev/null 2>&1
$P -k regex:"psh_kernel|fused_hash|fused_min" -c 6 -o gpurun_out/z_psh python tools/prof_step.py > /dev/null 2>&1
$P -k regex:"pool_build|pool_reduce" -c 3 -o gpurun_out/z_pool python tools/prof_step.py > /dev/null 2>&1
$P -k regex:"row_ln_vec|scatter_ln_pe|residual_out" -c 4 -o gpurun_out/z_rows python tools/prof_step.py > /dev/null 2>&1
ncu --set full --clock-control none -k regex:bswin_attn_tc -s 3 -c 1 -o gpurun_out/z_attnD python tools/attn_bench.py --config D --iters 1 > /dev/null 2>&1
for f in gpurun_out/z_*.ncu-rep; do python tools/ncu_summary.py $f > ${f%.ncu-rep}.md; done
ls -la gpurun_out/z_*
du -sh gpurun_out
