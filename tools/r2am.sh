timeout 900 python -m pytest tests/test_gpu_psh.py tests/test_gpu_psh_fused.py tests/test_gpu_dropin.py tests/test_gpu_backbone.py -q -p no:cacheprovider -x 2>&1 | tail -2
timeout 300 python tools/psh_bench.py 2>&1 | cut -c1-220
bash tools/ab_bench.sh "fastdiv"
