for v in main ch2 ch4; do
  lib=""; [ $v != main ] && lib=tools/exp/libf3d_$v.so
  echo "== $v"; F3D_LIB_PATH=$lib timeout 300 python tools/psh_bench.py 2>&1 | cut -c1-200
done
