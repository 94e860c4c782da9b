"""Flash3D backbone forward = composition of the reference hot-path ops
(SURVEY.md §7 "Decisions"; bw/cli.py:439-529 demo flow):

    per stage:  voxelize -> remap -> PSH -> scatter -> stage_forward (R rounds)
    between:    pool_stage(rho, mean), then re-bucket the pooled f64 centroids

Every step runs in libf3d kernels on device-resident tensors; the host only
reads the bucket counts once per stage (the attention plan and the pooled row
count depend on them, exactly as the reference needs ``bucket_table``).
"""

from dataclasses import dataclass, field

import numpy as np
import torch
from torch.profiler import record_function

from . import _lib as L
from .attention import DeviceRoundPlan, RoundPlan, plan_arrays, qstep_for, round_members
from .bucketing import BucketAssignment, _run_psh, default_probe_schedule
from .errors import ConfigError, RangeError
from .hashing import HashConfig, raise_range
from .pooling import pool_device
from .stage import StageRunner, init_params


@dataclass(frozen=True)
class StageConfig:
    voxel: float = 1 / 64
    K: int = 256
    S: int = 512
    S_div: int = 1024
    kind: str = "zorder-div"
    W: int = 2
    stride: int = 1
    shift: int = 1
    rounds: int = 2
    d_model: int = 96
    n_heads: int = 4
    pool_rho: int = 2          # 0: no pooling after this stage
    seed: int = 0


def scannet_backbone():
    """Default 2-stage backbone of SURVEY.md §7 (config B)."""
    return (StageConfig(K=256, S=512, S_div=1024, pool_rho=2, seed=0),
            StageConfig(K=128, S=512, S_div=2048, pool_rho=0, seed=1))


@dataclass
class StageTrace:
    n: int
    counts: np.ndarray
    assignment: BucketAssignment
    attention_flops: int
    sweeps: int = 0


def split_table(counts, base, K, S):
    """bucket_table(split_recycle=True) from host counts/base
    (bw/bucketing.py:147-166), vectorised."""
    r = int(counts[K])
    j = np.arange(0, r, S, dtype=np.int64)
    starts = np.concatenate([base[:K], base[K] + j])
    lens = np.concatenate([counts[:K], np.minimum(S, r - j)])
    return starts.astype(np.int64), lens.astype(np.int64)


class Backbone:
    """Device-resident backbone forward.  Parameters are drawn with the
    reference's init_params (bit-identical host RNG) and uploaded once."""

    def __init__(self, stages=None):
        self.stages = tuple(stages) if stages is not None else scannet_backbone()
        self.params = [init_params(s.seed, s.d_model, n_heads=s.n_heads) for s in self.stages]
        d0 = self.stages[0].d_model
        if any(s.d_model != d0 for s in self.stages):
            raise ConfigError("the reference pool preserves width: all stages share d_model")
        self._w = [p.device_weights() for p in self.params]
        self.last_trace = []

    def bucketize(self, coords, cfg: StageConfig):
        """f3d_voxel_hash + f3d_psh_assign on (n,3) f64 device coords."""
        n = coords.shape[0]
        hc = HashConfig(cfg.kind, K=cfg.K, S_div=cfg.S_div)
        vox32 = L.empty((n, 3), torch.int32)
        home = L.empty((n,), torch.int32)
        stats = L.empty((7,), torch.int64)
        ws = L.empty((3,), torch.int64)
        org = (L._F64 * 3)(0.0, 0.0, 0.0)
        L.call("f3d_voxel_hash", L.ptr(coords), None, n, 1, org, float(cfg.voxel), hc.kind_code,
               cfg.K, cfg.S_div, hc.bits_per_axis, L.ptr(vox32), L.ptr(home), L.ptr(stats),
               L.ptr(ws), L.stream())
        ids, offs, counts, base, dest, info = _run_psh(vox32, home, None, 1, n, hc, cfg.S,
                                                       default_probe_schedule())
        host = torch.cat([stats, counts.to(torch.int64), info.to(torch.int64)]).cpu().numpy()
        raise_range(host[:7], hc.bits_per_axis)
        counts_h = host[7:7 + cfg.K + 1]
        a = BucketAssignment(ids, offs, counts, base, cfg.S, cfg.K,
                             _dev={"id": ids, "off": offs, "counts": counts, "base": base,
                                   "batch": None, "dest": dest, "info": info})
        return a, counts_h, int(host[7 + cfg.K + 1])

    def forward_host(self, coords_h, feats_h, out_h=None):
        """End-to-end call with HOST buffers (pinned for async copies):
        coords (n,3) float64, feats (n,d) bf16/float32.  The feature upload
        runs on a side stream and overlaps the first PSH; the result (last
        stage features, bf16) is copied back into ``out_h`` (allocated pinned
        if None) and returned with the stage-2 coordinates left on device."""
        dev = L.device()
        main = torch.cuda.current_stream()
        side = getattr(self, "_side", None)
        if side is None:
            side = self._side = torch.cuda.Stream()
        C = coords_h.to(dev, non_blocking=True)
        side.wait_stream(main)
        with torch.cuda.stream(side):
            X = feats_h.to(dev, non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(side)
        self._feat_event = ev
        f, c = self.forward(C, X)
        fb = f.to(torch.bfloat16)
        if out_h is None or tuple(out_h.shape) != tuple(fb.shape):
            out_h = torch.empty(fb.shape, dtype=fb.dtype).pin_memory()
        out_h.copy_(fb, non_blocking=True)
        X.record_stream(main)
        return out_h, c

    def forward(self, coords, feats, keep_trace=False):
        """coords (n,3) float64, feats (n,d) float32/bf16 CUDA tensors.
        Returns (features, coords) of the last stage in its scattered order."""
        C = coords.to(torch.float64).contiguous()
        X = feats
        trace = []
        for si, cfg in enumerate(self.stages):
            n = C.shape[0]
            with record_function(f"stage{si}.bucketize"):
                a, counts_h, sweeps = self.bucketize(C, cfg)
            base_h = np.zeros_like(counts_h)
            base_h[1:] = np.cumsum(counts_h[:-1])
            with record_function(f"stage{si}.scatter"):
                ev = getattr(self, "_feat_event", None)
                if ev is not None:
                    torch.cuda.current_stream().wait_event(ev)   # features uploaded
                    self._feat_event = None
                dest = a._dev["dest"]
                d = X.shape[1]
                Xf = X.to(torch.float32).contiguous()
                F = torch.empty((n, d), dtype=torch.float32, device=C.device)
                Cs = torch.empty_like(C)
                L.call("f3d_scatter_rows", L.ptr(Xf), L.ptr(dest), n, d * 4, L.ptr(F), L.stream())
                L.call("f3d_scatter_rows", L.ptr(C), L.ptr(dest), n, 24, L.ptr(Cs), L.stream())
            with record_function(f"stage{si}.plan"):
                nb = cfg.K + -(-int(counts_h[cfg.K]) // cfg.S)
                if cfg.W > nb:
                    raise ConfigError(f"window_w ({cfg.W}) exceeds num_buckets ({nb})")
                cd, bd = a._dev["counts"], a._dev["base"]
                qs = qstep_for(cfg.d_model // cfg.n_heads)
                plans = [DeviceRoundPlan(cd, bd, cfg.K, cfg.S, nb, cfg.W, cfg.stride, cfg.shift,
                                         t, n, qstep=qs) for t in range(cfg.rounds)]
                runner = StageRunner(Cs, None, None, self.params[si], n, torch.float32,
                                     weights=self._w[si], plans=plans)
            with record_function(f"stage{si}.run"):
                runner.run(F)
            if keep_trace:
                trace.append(StageTrace(n, counts_h, a, runner.attention_flops(), sweeps))
            if cfg.pool_rho:
                with record_function(f"stage{si}.pool"):
                    X, C, _ = pool_device(F, Cs, counts_h, base_h, cfg.K, cfg.S, 1, cfg.pool_rho,
                                          "mean", check=False, assignment=False,
                                          dev_counts=(a._dev["counts"], a._dev["base"]))
            else:
                X, C = F, Cs
        self.last_trace = trace
        return X, C


def backbone_forward(coords, feats, stages=None):
    """Public entry: host or device arrays in; the caller's array type out."""
    host = L.is_host(coords)
    C = L.to_dev(coords, torch.float64)
    X = L.to_dev(feats, torch.float32) if host else feats.to(L.device())
    bb = Backbone(stages)
    f, c = bb.forward(C, X)
    return L.out(f, host), L.out(c, host)
