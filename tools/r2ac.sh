timeout 1500 python -m pytest tests/test_gpu_backbone.py tests/test_gpu_attention_stage.py tests/test_gpu_headline.py tests/test_gpu_train.py -q -p no:cacheprovider -x 2>&1 | tail -2
bash tools/ab_bench.sh "ln8" "ln32 F3D_LN8=0"
