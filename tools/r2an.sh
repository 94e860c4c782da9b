timeout 900 python -m pytest tests/test_gpu_attention_stage.py tests/test_gpu_backbone.py -q -p no:cacheprovider -x 2>&1 | tail -2
for i in 1 2; do echo "== B: $(timeout 300 python tools/attn_bench.py --config B 2>&1 | tail -1 | cut -c100-240)"; done
bash tools/ab_bench.sh "tailskip"
