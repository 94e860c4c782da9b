echo "== stream tests gate off (fixed)"; timeout 600 python -m pytest tests/test_gpu_backbone.py -q -p no:cacheprovider -k "stream_host" 2>&1 | tail -2
echo "== stream tests gate off (fixed), old cg lib"; F3D_LIB_PATH=tools/exp/libf3d_cgpsh.so timeout 600 python -m pytest tests/test_gpu_backbone.py -q -p no:cacheprovider -k "stream_host" 2>&1 | tail -2
echo "== stress 100K"; timeout 300 python tools/stream_gate_stress.py 60 2>&1 | tail -1
for r in 1 2 3; do timeout 600 python -m pytest tests/test_gpu_backbone.py -q -p no:cacheprovider -k "stream_host" 2>&1 | tail -1; done
