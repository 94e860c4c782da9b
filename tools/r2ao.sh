for i in 1 2; do for v in main old; do
  lib=""; [ $v != main ] && lib=tools/exp/libf3d_$v.so
  echo "== $v B: $(F3D_LIB_PATH=$lib timeout 300 python tools/attn_bench.py --config B 2>&1 | tail -1 | cut -c100-200)"
done; done
bash tools/ab_bench.sh "tailskip" "old F3D_LIB_PATH=tools/exp/libf3d_old.so"
