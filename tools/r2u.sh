timeout 900 python -m pytest tests/test_gpu_attention_stage.py -q -p no:cacheprovider -k "res_ln" 2>&1 | tail -15
timeout 900 python -m pytest tests/test_gpu_headline.py tests/test_gpu_backbone.py tests/test_gpu_attention_stage.py -q -p no:cacheprovider -x 2>&1 | tail -3
bash tools/ab_bench.sh "res_ln" "row_ln F3D_GEMM_RES_LN=0"
