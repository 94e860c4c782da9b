timeout 600 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_attention_stage.py -q -p no:cacheprovider -x 2>&1 | tail -2
python tools/gemm_bench.py 2>&1
echo "== dense"; F3D_GEMM_DENSE_STAGE=1 python tools/gemm_bench.py 2>&1
echo "== qkv bn96"; F3D_GEMM_BN_MAX=96 python tools/gemm_bench.py 2>&1 | grep qkv
bash tools/ab_bench.sh "swz" "dense F3D_GEMM_DENSE_STAGE=1" "swz_qkv96 F3D_GEMM_BN_MAX=96"
