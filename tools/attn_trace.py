"""Timeline of the softmax warps of CTA 0 (F3D_EXPERIMENT=4 build):

    F3D_LIB_PATH=tools/exp/libf3d_exp4.so python tools/attn_trace.py --config B

For each SM sub-partition, the exp-phase windows of its softmax warps (one per
Q tile) per key tile, relative to the first S-ready clock: shows whether the
warps sharing a sub-partition's MUFU run their exp phases in lock step."""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2412_16481_b200 import _lib as L  # noqa: E402

if __name__ == "__main__":
    sys.argv += ["--iters", "1"]
    import tools.attn_bench as AB  # noqa: E402
    AB.main()
    torch.cuda.synchronize()
    lib = L.load()
    buf = (ctypes.c_longlong * (16 * 96 * 3 + 16 * 16 * 8))()
    lib.f3d_attn_trace(buf)
    arr = np.array(buf, dtype=np.int64)
    tr = arr[:16 * 96 * 3].reshape(16, 96, 3)
    it = arr[16 * 96 * 3:].reshape(16, 16, 8)
    t0 = tr[4:, 0, 0][tr[4:, 0, 0] > 0].min()
    overlap, tot = 0, 0
    for q in range(4):
        ws = [w for w in range(4, 16) if w % 4 == q]
        print(f"sub-partition {q}: warps {ws}")
        for t in range(0, 24):
            row = []
            for w in ws:
                s, a, b = tr[w, t] - t0
                row.append(f"S{s:7d} e[{a:7d},{b:7d}] ({b - a:5d})")
            print(f"  tile {t:2d}: " + " | ".join(row))
        # pairwise overlap of exp windows over all traced tiles
        for i in range(len(ws)):
            for j in range(i + 1, len(ws)):
                A = tr[ws[i], :, 1:3]
                B = tr[ws[j], :, 1:3]
                for a in A:
                    if a[0] == 0:
                        continue
                    tot += a[1] - a[0]
                    for b in B:
                        if b[0] == 0:
                            continue
                        overlap += max(0, min(a[1], b[1]) - max(a[0], b[0]))
    print("items (warp 4, 8, 12): item start / final-PV wait start / epilogue start / end"
          " / O loaded / row mapped / stored")
    for w in (4, 8, 12):
        for i in range(6):
            if it[w, i, 0]:
                print(f"  w{w} item {i}: " + " ".join(f"{v - t0:7d}" for v in it[w, i][[0, 1, 2, 3]]) + "  |"
                      + " ".join(f"{v - it[w, i, 2]:6d}" for v in it[w, i][[4, 5, 6]]))
    print("exp-window overlap fraction (pairs of warps on one sub-partition): %.2f" % (overlap / max(tot, 1)))
    ex = tr[4:, :, 2] - tr[4:, :, 1]
    per = tr[4:, 1:, 0] - tr[4:, :-1, 0]
    print("mean exp window %.0f clk; mean tile period %.0f clk" % (ex[ex > 0].mean(), per[(per > 0) & (per < 1e5)].mean()))
