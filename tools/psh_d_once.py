import os, sys
sys.path.insert(0, os.getcwd())
import torch
from paper_2412_16481_b200.backbone import Backbone, StageConfig
from paper_2412_16481_b200.geometry import synth_cloud
cfg = StageConfig(voxel=1 / 128, K=1280, S=1024, S_div=1639, W=4, d_model=512)
C = torch.tensor(synth_cloud(7, 1_000_000, "uniform-box").coords, device="cuda")
bb = Backbone.__new__(Backbone)
for _ in range(4):
    Backbone.bucketize(bb, C, cfg)
torch.cuda.synchronize()
