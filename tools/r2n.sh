echo "== probe"; timeout 600 python tools/g0_overlap_probe.py 40 2>&1 | tail -15
echo "== probe old cg lib"; F3D_LIB_PATH=tools/exp/libf3d_cgpsh.so timeout 600 python tools/g0_overlap_probe.py 40 2>&1 | tail -8
