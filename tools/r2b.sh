mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_psh.py tests/test_gpu_psh_fused.py tests/test_gpu_train.py -q -p no:cacheprovider > gpurun_out/r2b_tests.log 2>&1; echo "exit $?" >> gpurun_out/r2b_tests.log
./tools/ubench/mma_ts > gpurun_out/r2b_mma_ts.txt 2>&1
./tools/ubench/sfu_rate > gpurun_out/r2b_sfu.txt 2>&1
bash tools/sanitize.sh > gpurun_out/r2b_sanitize.txt 2>&1
tail -3 gpurun_out/r2b_tests.log; cat gpurun_out/r2b_mma_ts.txt gpurun_out/r2b_sfu.txt gpurun_out/r2b_sanitize.txt
