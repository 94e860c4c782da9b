python tools/gemm_bench.py 2>&1 | tail -12
for bn in 128 96; do echo "== BN_MAX=$bn"; F3D_GEMM_BN_MAX=$bn python tools/gemm_bench.py 2>&1 | tail -12; done
bash tools/ab_bench.sh "bn256" "bn128 F3D_GEMM_BN_MAX=128" "bn96 F3D_GEMM_BN_MAX=96"
