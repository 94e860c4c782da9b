echo "== probe"; timeout 600 python tools/g0_overlap_probe.py 60 2>&1 | tail -8
echo "== probe old cg lib"; F3D_LIB_PATH=tools/exp/libf3d_cgpsh.so timeout 600 python tools/g0_overlap_probe.py 60 2>&1 | tail -8
echo "== stream test gate off"; timeout 600 python -m pytest tests/test_gpu_backbone.py -q -p no:cacheprovider -k stream_host 2>&1 | tail -3
echo "== stream test gate off, old lib"; F3D_LIB_PATH=tools/exp/libf3d_cgpsh.so timeout 600 python -m pytest tests/test_gpu_backbone.py -q -p no:cacheprovider -k stream_host 2>&1 | tail -3
echo "== stream test gate on"; F3D_PSH_GATE=1 timeout 600 python -m pytest tests/test_gpu_backbone.py -q -p no:cacheprovider -k stream_host 2>&1 | tail -3
