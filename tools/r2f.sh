F3D_LIB_PATH=tools/exp/libf3d_exp3.so timeout 300 python tools/attn_prof.py --config B 2>&1 | tail -12
