mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_attention_stage.py -x -q -p no:cacheprovider > gpurun_out/r2e_tests.log 2>&1; echo "exit $?" >> gpurun_out/r2e_tests.log
tail -2 gpurun_out/r2e_tests.log
for v in main st400 st900 st1500 p4; do
  lib=""; [ $v != main ] && lib=tools/exp/libf3d_$v.so
  echo "== $v B: $(F3D_LIB_PATH=$lib timeout 300 python tools/attn_bench.py --config B 2>&1 | tail -1 | cut -c1-300)"
done
echo "== main D: $(timeout 300 python tools/attn_bench.py --config D 2>&1 | tail -1)"
F3D_LIB_PATH=tools/exp/libf3d_exp3.so timeout 300 python tools/attn_prof.py --config B 2>&1 | tail -25
