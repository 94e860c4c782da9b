python tools/gemm_bench.py 2>&1 | tail -4
for bn in 64 128; do echo "== BN_GELU=$bn"; F3D_GEMM_BN_GELU=$bn python tools/gemm_bench.py 2>&1 | grep mlp_in; done
bash tools/ab_bench.sh "gelu96" "gelu64 F3D_GEMM_BN_GELU=64"
