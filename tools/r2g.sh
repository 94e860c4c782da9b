timeout 900 python -m pytest tests/test_gpu_attention_stage.py tests/test_gpu_backbone.py -x -q -p no:cacheprovider > gpurun_out/r2g_tests.log 2>&1; echo "exit $?" >> gpurun_out/r2g_tests.log
tail -3 gpurun_out/r2g_tests.log
echo "== main B: $(timeout 300 python tools/attn_bench.py --config B 2>&1 | tail -1 | cut -c1-300)"
echo "== main D: $(timeout 300 python tools/attn_bench.py --config D 2>&1 | tail -1)"
F3D_LIB_PATH=tools/exp/libf3d_exp3.so timeout 300 python tools/attn_prof.py --config B 2>&1 | tail -6
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/r2g_bench.json 2> gpurun_out/r2g_bench.err
python -c "
import json; d=json.loads(open('gpurun_out/r2g_bench.json').read().strip().splitlines()[-1])
print('value', d['value'], 'ms', d['ms_per_step'], 'e2e', d['e2e']['value'], 'attn', d['kernel_ms_per_step'])"
