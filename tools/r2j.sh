timeout 900 python -m pytest tests/test_gpu_train.py tests/test_gpu_psh.py tests/test_gpu_psh_fused.py tests/test_gpu_pool.py -q -p no:cacheprovider > gpurun_out/r2j_tests.log 2>&1; echo "exit $?" >> gpurun_out/r2j_tests.log
tail -4 gpurun_out/r2j_tests.log
grep -E "^E  |FAILED" gpurun_out/r2j_tests.log | head -10
timeout 300 python tools/psh_bench.py 2>&1 | tail -3
echo "== train fused"; timeout 600 python tools/train_bench.py --scenes 4 --steps 2 2>&1 | tail -1
bash tools/ab_bench.sh "default" "unfusedpsh F3D_FUSED_PSH=0"
