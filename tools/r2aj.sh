for v in main minb4 minb5; do
  lib=""; [ $v != main ] && lib=tools/exp/libf3d_$v.so
  echo "== $v: $(F3D_LIB_PATH=$lib timeout 600 python tools/train_bench.py --scenes 4 --steps 2 2>&1 | tail -1 | cut -c150-330)"
done
