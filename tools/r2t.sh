for v in main pool1; do
  lib=""; [ $v != main ] && lib=tools/exp/libf3d_$v.so
  F3D_LIB_PATH=$lib timeout 300 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none -k regex:pool_build --csv --log-file gpurun_out/r2t_$v.csv python tools/prof_step.py > /dev/null 2>&1
  echo "$v: $(grep pool_build gpurun_out/r2t_$v.csv | awk -F'","' '{print $NF}')"
done
bash tools/ab_bench.sh "sep_pools" "shared_pool F3D_SEPARATE_POOLS=0"
