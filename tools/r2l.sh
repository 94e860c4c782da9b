echo "== old lib, gate off"; F3D_PSH_GATE=0 F3D_LIB_PATH=tools/exp/libf3d_cgpsh.so timeout 300 python tools/stream_gate_stress.py 40 2>&1 | tail -2
echo "== new lib, gate off"; F3D_PSH_GATE=0 timeout 300 python tools/stream_gate_stress.py 40 2>&1 | tail -2
echo "== new lib, gate on"; timeout 300 python tools/stream_gate_stress.py 40 2>&1 | tail -2
bash tools/ab_bench.sh "gate_on" "gate_off F3D_PSH_GATE=0"
