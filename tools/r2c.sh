mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_attention_stage.py tests/test_gpu_headline.py -x -q -p no:cacheprovider > gpurun_out/r2c_tests.log 2>&1; echo "exit $?" >> gpurun_out/r2c_tests.log
for cfg in B D; do
  echo "== main $cfg" >> gpurun_out/r2c_attn.txt
  timeout 300 python tools/attn_bench.py --config $cfg >> gpurun_out/r2c_attn.txt 2>&1
done
for v in p2 p3 p0 nq2; do
  echo "== $v B" >> gpurun_out/r2c_attn.txt
  F3D_LIB_PATH=tools/exp/libf3d_$v.so timeout 300 python tools/attn_bench.py --config B >> gpurun_out/r2c_attn.txt 2>&1
done
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/r2c_bench.json 2> gpurun_out/r2c_bench.err
tail -3 gpurun_out/r2c_tests.log; cat gpurun_out/r2c_attn.txt; tail -c 300 gpurun_out/r2c_bench.json
