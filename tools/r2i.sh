timeout 600 python -m pytest tests/test_gpu_train.py tests/test_gpu_psh.py tests/test_gpu_psh_fused.py tests/test_gpu_pool.py -x -q -p no:cacheprovider > gpurun_out/r2i_tests.log 2>&1; echo "exit $?" >> gpurun_out/r2i_tests.log
tail -4 gpurun_out/r2i_tests.log
grep -E "Error|error|assert" gpurun_out/r2i_tests.log | head -10
timeout 300 python tools/psh_bench.py 2>&1 | tail -8
echo "== train fused"; timeout 600 python tools/train_bench.py --scenes 4 --steps 2 2>&1 | tail -2
echo "== train tiles"; F3D_FUSED_ATTN_BWD=0 timeout 600 python tools/train_bench.py --scenes 4 --steps 2 2>&1 | tail -2
bash tools/ab_bench.sh "default" "unfusedpsh F3D_FUSED_PSH=0"
