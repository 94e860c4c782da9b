timeout 600 python -m pytest tests/test_gpu_backbone.py -q -p no:cacheprovider -k "stream_host" -x 2>&1 | grep -E "Error|assert|^E " | head -20
