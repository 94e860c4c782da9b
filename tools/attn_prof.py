"""Per-role wait-cycle breakdown of the tcgen05 attention kernel.

Needs the F3D_EXPERIMENT=3 build: F3D_LIB_PATH=tools/exp/libf3d_exp3.so
python tools/attn_prof.py --config B|D [--d 512].  Counters are summed over
warps (lane 0 of each warp) and over all CTAs of one launch."""
import ctypes
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2412_16481_b200 import _lib as L  # noqa: E402

NAMES = ["softmax_total", "softmax_wait_S", "softmax_wait_pv_rescale", "softmax_wait_pv_final",
         "mma_wait_q", "mma_wait_kv", "mma_wait_p", "mma_wait_ofree", "mma_total",
         "load_wait_kv_empty", "load_wait_q_empty", "load_total", "softmax_tiles", "rescales",
         "", "", "sm_tmem_ld", "sm_max", "sm_exp_pack", "sm_st_arrive", "sm_decode",
         "sm_epilogue", "sm_busy_span"]

if __name__ == "__main__":
    sys.argv += ["--iters", "1"]
    import tools.attn_bench as AB  # noqa: E402
    lib = L.load()
    buf = (ctypes.c_ulonglong * 24)()
    lib.f3d_attn_prof(buf, 1)
    AB.main()                           # 3 warm-ups + 1 timed launch
    torch.cuda.synchronize()
    lib.f3d_attn_prof(buf, 1)
    vals = list(buf)
    for i, n in enumerate(NAMES):
        if not n:
            continue
        print(f"{n:28s} {vals[i]:>16,d}")
    st = vals[0] or 1
    print("softmax: wait_S %.1f%%  rescale %.1f%%  final %.1f%%" % (100 * vals[1] / st, 100 * vals[2] / st, 100 * vals[3] / st))
    mt = vals[8] or 1
    print("mma: q %.1f%% kv %.1f%% p %.1f%% ofree %.1f%%" % tuple(100 * vals[i] / mt for i in (4, 5, 6, 7)))
    print("softmax phases: ld %.1f%% max %.1f%% exp+pack %.1f%% st+arrive %.1f%%" % tuple(100 * vals[i] / st for i in (16, 17, 18, 19)))
    print("softmax: decode %.1f%% epilogue %.1f%% busy span %.1f%% (rest = tail after the last item)"
          % tuple(100 * vals[i] / st for i in (20, 21, 22)))
    lt = vals[11] or 1
    print("load: kv_empty %.1f%% q_empty %.1f%%" % (100 * vals[9] / lt, 100 * vals[10] / lt))
