timeout 1200 python -m pytest tests/test_gpu_backbone.py tests/test_gpu_psh.py tests/test_gpu_psh_fused.py tests/test_gpu_dropin.py -q -p no:cacheprovider -x 2>&1 | tail -2
bash tools/ab_bench.sh "pdl2" "nopdl F3D_PDL=0"
