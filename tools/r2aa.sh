timeout 1200 python -m pytest tests/test_gpu_backbone.py tests/test_gpu_attention_stage.py tests/test_gpu_headline.py tests/test_gpu_pool.py tests/test_gpu_psh.py -q -p no:cacheprovider -x 2>&1 | tail -2
bash tools/ab_bench.sh "pdl" "nopdl F3D_PDL=0"
