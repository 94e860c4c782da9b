for v in main nq4b48 nq4b32; do
  lib=""; [ $v != main ] && lib=tools/exp/libf3d_$v.so
  echo "== $v B: $(F3D_LIB_PATH=$lib timeout 300 python tools/attn_bench.py --config B 2>&1 | tail -1 | cut -c1-240)"
done
