echo "== probe POOL_OVERLAP=0"; F3D_POOL_OVERLAP=0 timeout 600 python tools/g0_overlap_probe.py 40 2>&1 | tail -3
echo "== probe NEXT_PROLOGUE_SIDE=0"; F3D_NEXT_PROLOGUE_SIDE=0 timeout 600 python tools/g0_overlap_probe.py 40 2>&1 | tail -3
echo "== probe CUDA_LAUNCH_BLOCKING"; CUDA_LAUNCH_BLOCKING=1 timeout 600 python tools/g0_overlap_probe.py 40 2>&1 | tail -3
