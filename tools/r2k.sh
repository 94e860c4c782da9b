echo "== cg grid.sync (old) unfused:"; F3D_LIB_PATH=tools/exp/libf3d_cgpsh.so timeout 300 python tools/psh_concurrency.py 300 2>&1 | tail -2
echo "== cg grid.sync (old) fused:"; F3D_FUSED_PSH=1 F3D_LIB_PATH=tools/exp/libf3d_cgpsh.so timeout 300 python tools/psh_concurrency.py 300 2>&1 | tail -2
echo "== own barrier unfused:"; timeout 300 python tools/psh_concurrency.py 300 2>&1 | tail -2
echo "== own barrier fused:"; F3D_FUSED_PSH=1 timeout 300 python tools/psh_concurrency.py 300 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_backbone.py tests/test_gpu_psh.py tests/test_gpu_psh_fused.py -q -p no:cacheprovider > gpurun_out/r2k_tests.log 2>&1; echo "exit $?" >> gpurun_out/r2k_tests.log
tail -3 gpurun_out/r2k_tests.log; grep -E "^E  |FAILED" gpurun_out/r2k_tests.log | head
echo "== old lib two-backbone test:"; F3D_LIB_PATH=tools/exp/libf3d_cgpsh.so timeout 600 python -m pytest tests/test_gpu_backbone.py -q -p no:cacheprovider -k two_backbones 2>&1 | tail -3
