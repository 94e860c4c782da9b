python tools/gemm_bench.py 2>&1 | grep -E "mlp_in|qkv"
echo "== wg4"; F3D_LIB_PATH=tools/exp/libf3d_wg4.so python tools/gemm_bench.py 2>&1 | grep -E "mlp_in|qkv"
echo "== wg4 bn64"; F3D_GEMM_BN_GELU=64 F3D_LIB_PATH=tools/exp/libf3d_wg4.so python tools/gemm_bench.py 2>&1 | grep mlp_in
bash tools/ab_bench.sh "wg3" "wg4 F3D_LIB_PATH=tools/exp/libf3d_wg4.so"
