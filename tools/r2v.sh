timeout 900 python -m pytest tests/test_gpu_psh.py tests/test_gpu_psh_fused.py tests/test_gpu_dropin.py -q -p no:cacheprovider 2>&1 | tail -2
timeout 300 python tools/psh_bench.py 2>&1 | tail -3
bash tools/ab_bench.sh "default"
