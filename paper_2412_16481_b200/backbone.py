"""Flash3D backbone forward = composition of the reference hot-path ops
(SURVEY.md §7 "Decisions"; bw/cli.py:439-529 demo flow):

    per stage:  voxelize -> remap -> PSH -> scatter -> stage_forward (R rounds)
    between:    pool_stage(rho, mean), then re-bucket the pooled f64 centroids

Every step runs in libf3d kernels on device-resident tensors and the whole
forward is enqueued without a single host read-back: data-dependent sizes
(the recycle chunk count, the number of pooled rows) stay on the device, and
each launch is sized for a host-known capacity and reads the true count
(``n_dev`` in include/f3d.h).  Error words (voxel range statistics, PSH
batch errors, planner and pooling flags) are collected on the device and
checked once, after the stream drains, so ``forward`` costs one sync and
``capture`` turns the whole forward into two CUDA graphs (stage-0 bucketing
on the coordinates alone, then everything else), replayed by
``forward_graph`` / ``forward_host``.
"""

import os
from dataclasses import dataclass

import numpy as np
import torch
from torch.profiler import record_function

from . import _lib as L
from .attention import DeviceRoundPlan, qstep_for
from .bucketing import (DEFAULT_MAX_SWEEPS, BucketAssignment, _run_psh, _zero_batch_ids,
                        default_probe_schedule)
from .errors import ConfigError
from .hashing import HashConfig, raise_range
from .pooling import TILE_CAP, _FLAG_MSGS, _build, _reduce
from .stage import LN_EPS, StageRunner, init_params

# The pooling partition, the pooled centroids and the next stage's PSH bucketing
# depend on the coordinates only: by default they run on a side stream under
# the stage's transformer rounds (config B: 1.16 -> 1.12 ms per step for the
# partition alone).  F3D_POOL_OVERLAP=0 keeps them on the main stream.
POOL_OVERLAP = os.environ.get("F3D_POOL_OVERLAP", "1") == "1"
# stream_host runs step i+1's coordinate-only graph g0 on its own stream under
# step i's g1: e2e 1.17 -> 1.10 ms per step.  F3D_G0_CONCURRENT=0 keeps the
# steps serial.  (Round 1 gated g0 behind g1's cooperative stage-1 PSH after
# results came back corrupted.  Root cause, found in round 2: a slot's g0 and
# g1 shared one graph memory pool, so g1's outputs (status words, last-stage
# bf16 features) could occupy memory that g0 uses as scratch, and g0 of step
# i+2 was only ordered after step i's g1 -- not after step i's device-to-host
# read-back of those outputs.  g0 and g1 now capture into separate pools
# (F3D_SEPARATE_POOLS=0: one pool, g0 then waits for the slot's read-back);
# the gate is off by default (F3D_PSH_GATE=1 restores it).
# tools/g0_overlap_probe.py shows concurrent g0/g1 replays themselves agree
# bit for bit; tests/test_gpu_backbone.py covers the pipelined paths.)
# F3D_NEXT_PROLOGUE_SIDE=0 keeps the next stage's PSH/prologue on the main stream.
G0_CONCURRENT = os.environ.get("F3D_G0_CONCURRENT", "1") == "1"
# F3D_SCATTER_LN=0: separate input scatter and first row_ln of each stage
SCATTER_LN = os.environ.get("F3D_SCATTER_LN", "1") == "1"
# F3D_POOL_RESIDUAL=0: a pooled stage's last residual as its own row pass
POOL_RESIDUAL = os.environ.get("F3D_POOL_RESIDUAL", "1") == "1"
NEXT_PROLOGUE_SIDE = os.environ.get("F3D_NEXT_PROLOGUE_SIDE", "1") == "1"
# F3D_FUSED_PSH=1: voxel hash + PSH as one cooperative launch
# (f3d_psh_assign_coords) instead of f3d_voxel_hash + f3d_psh_assign.  Opt-in:
# measured 1.087 vs 1.069 ms per config-B step (its extra grid barrier and
# the all-CTA reduction of the per-CTA extrema cost more than the launches
# the fusion saves)
FUSED_PSH = os.environ.get("F3D_FUSED_PSH", "0") == "1"
# F3D_PSH_GATE=1: hold step i+1's g0 behind step i's cooperative PSH launches
# (the round-1 workaround; see G0_CONCURRENT)
PSH_GATE = os.environ.get("F3D_PSH_GATE", "0") == "1"
SEPARATE_POOLS = os.environ.get("F3D_SEPARATE_POOLS", "1") == "1"


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


def pool_capacity(n_cap: int, nslots: int, rho: int):
    """Upper bounds for the device pooling plan (bw/pooling.py:211-225):
    sum_c ceil(c/1024) < n/1024 + nslots tiles, and sum_tiles ceil(m/rho)
    <= ceil(n/rho) + tiles pooled rows."""
    ntiles = nslots + n_cap // TILE_CAP + 1
    return ntiles, -(-n_cap // rho) + ntiles


class _StageRun:
    """Device state of one enqueued stage (kept alive for the graph)."""

    def __init__(self, si, cfg, n_cap, n_dev):
        self.si, self.cfg, self.n_cap, self.n_dev = si, cfg, n_cap, n_dev


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
        self._graphs = None

    # ------------------------------------------------------------ pieces
    def bucketize(self, coords, cfg: StageConfig, n_cap=None, n_dev=None):
        """Voxelize + remap + hash + PSH on (n,3) f64 device coords, no
        read-back: one fused cooperative launch (f3d_psh_assign_coords) when
        K + 1 <= 12288, else f3d_voxel_hash + f3d_psh_assign.  Returns
        (assignment, stats int64[7], info int32[4])."""
        n = coords.shape[0] if n_cap is None else n_cap
        hc = HashConfig(cfg.kind, K=cfg.K, S_div=cfg.S_div)
        if FUSED_PSH and cfg.K + 1 <= 12288 and n > 0:
            table, P = default_probe_schedule().device_table()
            ids = L.empty((n,), torch.int32)
            offs = L.empty((n,), torch.int32)
            counts = L.empty((cfg.K + 1,), torch.int32)
            base = L.empty((cfg.K + 1,), torch.int32)
            dest = L.empty((n,), torch.int32)
            info = L.empty((4,), torch.int32)
            stats = L.empty((7,), torch.int64)
            ws_bytes = L.load().f3d_psh_coords_workspace_size(n, cfg.K)
            ws = L.empty((ws_bytes,), torch.uint8)
            org = (L._F64 * 3)(0.0, 0.0, 0.0)
            L.call("f3d_psh_assign_coords", L.ptr(coords), n, org, float(cfg.voxel), hc.kind_code,
                   cfg.K, cfg.S, cfg.S_div, hc.bits_per_axis, int(hc.div_overflow == "error"),
                   table.ctypes.data_as(L._P), P, DEFAULT_MAX_SWEEPS, L.ptr(ids), L.ptr(offs),
                   L.ptr(counts), L.ptr(base), L.ptr(dest), L.ptr(info), L.ptr(stats), L.ptr(ws),
                   ws_bytes, L.ptr(n_dev), L.stream())
            a = BucketAssignment(ids, offs, counts, base, cfg.S, cfg.K,
                                 batch_id=_zero_batch_ids(n, ids.device),
                                 _dev={"id": ids, "off": offs, "counts": counts, "base": base,
                                       "batch": None, "dest": dest, "info": info})
            return a, stats, info
        vox32 = L.empty((n, 3), torch.int32)
        home = L.empty((n,), torch.int32)
        stats = L.empty((7,), torch.int64)
        ws = L.empty((3,), torch.int64)
        org = (L._F64 * 3)(0.0, 0.0, 0.0)
        L.call("f3d_voxel_hash", L.ptr(coords), None, n, 1, org, float(cfg.voxel), hc.kind_code,
               cfg.K, cfg.S_div, hc.bits_per_axis, L.ptr(vox32), L.ptr(home), L.ptr(stats),
               L.ptr(ws), L.ptr(n_dev), L.stream())
        ids, offs, counts, base, dest, info = _run_psh(vox32, home, None, 1, n, hc, cfg.S,
                                                       default_probe_schedule(), n_dev=n_dev)
        a = BucketAssignment(ids, offs, counts, base, cfg.S, cfg.K,
                             batch_id=_zero_batch_ids(n, ids.device),
                             _dev={"id": ids, "off": offs, "counts": counts, "base": base,
                                   "batch": None, "dest": dest, "info": info})
        return a, stats, info

    def _stage_prologue(self, r: _StageRun, C):
        """Coordinate-only setup of a bucketed stage: scattered coordinates,
        the device scope plans of every round and the stage runner (buffers,
        coordinate bounding box).  Sets r.Cs, r.plans, r.runner."""
        cfg, si, n, n_dev = r.cfg, r.si, r.n_cap, r.n_dev
        a = r.asg
        with record_function(f"stage{si}.plan"):
            Cs = torch.empty((n, 3), dtype=torch.float64, device=C.device)
            L.call("f3d_scatter_rows", L.ptr(C), L.ptr(a._dev["dest"]), n, 24, L.ptr(Cs),
                   L.ptr(n_dev), L.stream())
            nb_cap = cfg.K + -(-n // cfg.S)
            if cfg.W > nb_cap:
                raise ConfigError(f"window_w ({cfg.W}) exceeds num_buckets ({nb_cap})")
            cd, bd = a._dev["counts"], a._dev["base"]
            qs = qstep_for(cfg.d_model // cfg.n_heads)
            r.plans = DeviceRoundPlan.all_rounds(cd, bd, cfg.K, cfg.S, nb_cap, cfg.W, cfg.stride,
                                                 cfg.shift, cfg.rounds, n, qstep=qs)
            r.runner = StageRunner(Cs, None, None, self.params[si], n, torch.float32,
                                   weights=self._w[si], plans=r.plans, n_dev=n_dev)
            r.Cs = Cs

    @staticmethod
    def _stage_tensors(r: _StageRun):
        """Every device tensor a prepared stage owns (for record_stream)."""
        out = [r.Cs, r.stats, r.info] + [v for v in r.asg._dev.values()
                                         if isinstance(v, torch.Tensor)]
        for p in r.plans:
            out += [v for v in vars(p).values() if isinstance(v, torch.Tensor)]
        out += [v for v in vars(r.runner).values() if isinstance(v, torch.Tensor)]
        return out

    def _stage_body(self, r: _StageRun, C, X):
        """Scatter -> R rounds -> (pool) for one stage whose bucketing is in
        r.asg (and whose prologue may already be enqueued).  Returns the next
        stage's (X, C, n_cap, n_dev)."""
        cfg, si, n, n_dev = r.cfg, r.si, r.n_cap, r.n_dev
        a = r.asg
        if getattr(r, "runner", None) is None:
            self._stage_prologue(r, C)
        Cs = r.Cs
        x_ready = False
        with record_function(f"stage{si}.scatter"):
            dest = a._dev["dest"]
            d = X.shape[1]
            F = torch.empty((n, d), dtype=torch.float32, device=C.device)
            rn = r.runner
            if (SCATTER_LN and d % 12 == 0 and d <= 128
                    and X.is_contiguous()
                    and X.dtype in (torch.bfloat16, torch.float32)):
                # scatter + the stage's first LN1 + PE in one pass (bit-identical)
                w = rn.w
                L.call("f3d_scatter_ln_pe", L.ptr(X), int(X.dtype == torch.float32), X.stride(0),
                       L.ptr(dest), L.ptr(C), L.ptr(rn.lo_ext), 10000.0, L.ptr(w["ln1_g"]),
                       L.ptr(w["ln1_b"]), L.ptr(F), F.stride(0), L.ptr(rn.x), rn.x.stride(0), n,
                       d, LN_EPS, L.ptr(n_dev), L.stream())
                x_ready = True
            elif X.dtype == torch.bfloat16 and d % 8 == 0 and X.is_contiguous():
                # bf16 upload -> fp32 residual stream in the scatter itself
                L.call("f3d_scatter_rows_bf16_f32", L.ptr(X), X.stride(0), L.ptr(dest), n, d,
                       L.ptr(F), F.stride(0), L.ptr(n_dev), L.stream())
            else:
                Xf = (X if X.dtype == torch.float32 else X.to(torch.float32)).contiguous()
                L.call("f3d_scatter_rows", L.ptr(Xf), L.ptr(dest), n, d * 4, L.ptr(F),
                       L.ptr(n_dev), L.stream())
        pool_ev = None
        if cfg.pool_rho and POOL_OVERLAP:
            # the pooling partition, the pooled centroids and the whole
            # coordinate-only prologue of the next stage (PSH bucketing,
            # scattered coordinates, plans, runner) run on a side stream under
            # this stage's transformer rounds
            main = torch.cuda.current_stream()
            side = self._pool_stream = getattr(self, "_pool_stream", None) or torch.cuda.Stream()
            side.wait_stream(main)
            with torch.cuda.stream(side):
                pool_parts = self._pool_partition(cfg, n, a, Cs)
                keep = [t for t in pool_parts if isinstance(t, torch.Tensor)]
                if si + 1 < len(self.stages) and NEXT_PROLOGUE_SIDE:
                    ncfg = self.stages[si + 1]
                    _, _, totals_, np_cap_, _, Cn_ = pool_parts
                    nr = _StageRun(si + 1, ncfg, np_cap_, totals_[1:2])
                    nr.asg, nr.stats, nr.info = self.bucketize(Cn_, ncfg, np_cap_, totals_[1:2])
                    # an external event (a graph event-record node when captured):
                    # with F3D_PSH_GATE=1 stream_host keeps the next scene's
                    # cooperative stage-0 PSH from running while this one is in flight
                    r.psh_event = torch.cuda.Event(external=True)
                    r.psh_event.record(side)
                    self._stage_prologue(nr, Cn_)
                    keep += self._stage_tensors(nr)
                    r.next_run = nr
                pool_ev = torch.cuda.Event()
                pool_ev.record(side)
            for t in keep:
                t.record_stream(main)
        # a pooled stage's last residual (F += y + b_out) is folded into the
        # feature pooling (f3d_pool_reduce_res) instead of its own pass over F
        # (f3d_pool_reduce_res indexes pooled rows x d/4 columns in 32 bits; larger
        # pooled capacities keep the residual in the stage and pool F itself)
        np_cap_ = pool_capacity(n, cfg.K + 1, cfg.pool_rho)[1] if cfg.pool_rho else 0
        defer = (cfg.pool_rho and POOL_RESIDUAL and F.dtype == torch.float32 and d % 4 == 0
                 and np_cap_ * (d // 4) < 2 ** 31)
        r.out_bf16 = None
        if (getattr(self, "_want_out_bf16", False) and si == len(self.stages) - 1
                and not cfg.pool_rho):
            # the graphs read the last stage back in bf16: written with its last residual
            r.out_bf16 = torch.empty((n, d), dtype=torch.bfloat16, device=F.device)
        hook = getattr(self, "round_hook", None)      # test instrumentation (eager only)
        r.runner.round_hook = (None if hook is None else
                               (lambda t, q, k, v, a, _si=si: hook(_si, t, q, k, v, a)))
        with record_function(f"stage{si}.run"):
            r.runner.run(F, x_ready=x_ready, defer_last_residual=defer, out_bf16=r.out_bf16)
        r.F = F
        if not cfg.pool_rho:
            return F, Cs, n, n_dev
        with record_function(f"stage{si}.pool"):
            rho = cfg.pool_rho
            if pool_ev is not None:
                torch.cuda.current_stream().wait_event(pool_ev)
                members, sizes, totals, np_cap, flags, Cn = pool_parts
            else:
                members, sizes, totals, np_cap, flags, Cn = self._pool_partition(cfg, n, a, Cs)
            r.pool_flags = flags
            r.pool_totals = totals
            if defer:
                y = r.runner.y
                Xn = torch.empty((np_cap, d), dtype=torch.float32, device=F.device)
                L.call("f3d_pool_reduce_res", L.ptr(F), F.stride(0), L.ptr(y), y.stride(0),
                       L.ptr(r.runner.w["b_out"]), d, L.ptr(members), L.ptr(sizes), np_cap, rho,
                       1, L.ptr(Xn), Xn.stride(0), L.ptr(totals[1:2]), L.stream())
            else:
                Xn = _reduce(F, members, sizes, np_cap, rho, "mean", npool_dev=totals[1:2])
        return Xn, Cn, np_cap, totals[1:2]

    def _pool_partition(self, cfg, n, a, Cs):
        """Tile table + sub-bucket partition + pooled centroids of one stage
        (depend on the scattered coordinates only)."""
        rho = cfg.pool_rho
        nslots = cfg.K + 1
        nt_cap, np_cap = pool_capacity(n, nslots, rho)
        buf = L.empty((3 * nt_cap + 2,), torch.int32)
        tstart, tm, tout = buf[:nt_cap], buf[nt_cap:2 * nt_cap], buf[2 * nt_cap:3 * nt_cap]
        totals = buf[3 * nt_cap:]
        cd, bd = a._dev["counts"], a._dev["base"]
        L.call("f3d_plan_pool", L.ptr(cd), L.ptr(bd), nslots, TILE_CAP, rho, L.ptr(tstart),
               L.ptr(tm), L.ptr(tout), L.ptr(totals), L.stream())
        plan = _CapPlan(tstart, tm, tout, nt_cap, np_cap)
        members, sizes, _, _, _, flags = _build(Cs, plan, rho, ntiles_dev=totals[0:1])
        Cn = _reduce(Cs, members, sizes, np_cap, rho, "mean", npool_dev=totals[1:2])
        return members, sizes, totals, np_cap, flags, Cn

    def _enqueue_bucketize0(self, C):
        """Stage-0 work that needs only the coordinates: PSH bucketing and the
        stage prologue (graph g0; the feature upload overlaps it)."""
        cfg = self.stages[0]
        r = _StageRun(0, cfg, C.shape[0], None)
        with record_function("stage0.bucketize"):
            r.asg, r.stats, r.info = self.bucketize(C, cfg)
        self._stage_prologue(r, C)
        return r

    def _enqueue_rest(self, r0: _StageRun, C, X):
        """Everything after stage-0 bucketing; returns (X, C, n_dev, runs)."""
        runs = [r0]
        X, C, n_cap, n_dev = self._stage_body(r0, C, X)
        for si in range(1, len(self.stages)):
            cfg = self.stages[si]
            r = _StageRun(si, cfg, n_cap, n_dev)
            prev = runs[-1]
            if getattr(prev, "next_run", None) is not None:
                r = prev.next_run                             # prepared on the side stream
                prev.next_run = None
            else:
                with record_function(f"stage{si}.bucketize"):
                    r.asg, r.stats, r.info = self.bucketize(C, cfg, n_cap, n_dev)
                # this stage's cooperative PSH runs on the main stream with no
                # gating event: stream_host then keeps the next scene's g0 after
                # this whole step (no two cooperative PSH grids in flight)
                r.psh_on_main = True
            runs.append(r)
            X, C, n_cap, n_dev = self._stage_body(r, C, X)
        return X, C, n_dev, runs

    # ------------------------------------------------------------ checks
    @staticmethod
    def _status_vector(runs, n_dev, zero1=None):
        """One int32 device vector holding every error word and the final
        row count, so the host reads it with a single copy.  Layout: the
        7 int64 hash stats of every stage (as int32 pairs), then per stage
        the int32 words [PSH info (4), planner status of each round, pool
        flags], then the row count.  One concatenation kernel (zero1: a
        preallocated int32 zero for unpooled stages, so a captured graph
        holds no fill node)."""
        dev = runs[0].stats.device
        w32 = [r.stats.view(torch.int32) for r in runs]
        for r in runs:
            w32.append(r.info)
            p0 = r.plans[0]
            per = (r.plans[1].live.storage_offset() - p0.live.storage_offset()
                   if len(r.plans) > 1 else 1)
            w32.append(p0.live.as_strided((len(r.plans),), (per,), p0.live.storage_offset() + 3))
            w32.append(r.pool_flags if hasattr(r, "pool_flags")
                       else zero1 if zero1 is not None
                       else torch.zeros(1, dtype=torch.int32, device=dev))
        w32.append(n_dev if n_dev is not None
                   else torch.full((1,), runs[-1].n_cap, dtype=torch.int32, device=dev))
        return torch.cat(w32)

    def _check(self, status_h, runs):
        """Raise the reference exceptions from the status words (same
        conditions and messages as bw/hashing.py:60-75, bw/attention.py:104,
        bw/pooling.py validate); returns the final row count."""
        nr = len(runs)
        s64 = np.ascontiguousarray(status_h[:14 * nr]).view(np.int64)
        o = 14 * nr
        for si, r in enumerate(runs):
            cfg = r.cfg
            stats, info = s64[7 * si:7 * si + 7], status_h[o:o + 4]
            o += 4
            live3 = status_h[o:o + cfg.rounds]
            o += cfg.rounds
            pflags = int(status_h[o])
            o += 1
            raise_range(stats, HashConfig(cfg.kind, K=cfg.K, S_div=cfg.S_div).bits_per_axis)
            if info[2]:
                raise ConfigError(f"PSH input error (code {int(info[2])})")
            if (live3 & 1).any():
                raise ConfigError(f"window_w ({cfg.W}) exceeds num_buckets")
            if (live3 & 6).any():
                raise RuntimeError("attention planner capacity exceeded (internal error)")
            for bit, msg in _FLAG_MSGS:
                if pflags & bit:
                    from .errors import IntegrityError
                    raise IntegrityError(msg)
        return int(status_h[o])

    def _trace(self, runs):
        trace = []
        for r in runs:
            counts_h = r.asg._dev["counts"].cpu().numpy().astype(np.int64)
            n = int(counts_h.sum())
            trace.append(StageTrace(n, counts_h, r.asg, r.runner.attention_flops(),
                                    int(r.info[0].item())))
        return trace

    # ------------------------------------------------------------ eager
    def forward(self, coords, feats, keep_trace=False):
        """coords (n,3) float64, feats (n,d) float32/bf16 CUDA tensors.
        Returns (features, coords) of the last stage in its scattered order.
        The whole forward is enqueued first; the host then reads one status
        vector (one sync) and raises if any stage flagged an error."""
        C = coords.to(torch.float64).contiguous()
        ev = getattr(self, "_feat_event", None)
        r0 = self._enqueue_bucketize0(C)
        if ev is not None:
            torch.cuda.current_stream().wait_event(ev)   # features uploaded (side stream)
            self._feat_event = None
        X, Cn, n_dev, runs = self._enqueue_rest(r0, C, feats)
        status = self._status_vector(runs, n_dev).cpu().numpy()
        n_out = self._check(status, runs)
        self.last_trace = self._trace(runs) if keep_trace else []
        return X[:n_out], Cn[:n_out]

    # ------------------------------------------------------------ graphs
    def _capture_slot(self, n, feat_dtype):
        """Two CUDA graphs over private static buffers: g0 = stage-0
        bucketing + prologue (reads only the coordinates), g1 = the rest."""
        dev = L.device()
        d = self.stages[0].d_model
        coords = torch.zeros((n, 3), dtype=torch.float64, device=dev)
        feats = torch.zeros((n, d), dtype=feat_dtype, device=dev)
        # a real scene to warm up (grid attributes, cuBLAS handles/workspaces)
        rng = np.random.default_rng(0)
        coords.copy_(torch.from_numpy(rng.random((n, 3))))
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            for _ in range(2):
                r0 = self._enqueue_bucketize0(coords)
                self._enqueue_rest(r0, coords, feats)
        torch.cuda.current_stream().wait_stream(side)
        torch.cuda.synchronize()
        # one memory pool per graph: g1's outputs (status words, bf16 features),
        # still being read back by the host stream when stream_host replays the
        # slot's next g0, must not share memory with g0's scratch
        g0, g1 = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
        zero1 = torch.zeros(1, dtype=torch.int32, device=dev)   # outside the capture
        pool0 = torch.cuda.graph_pool_handle()
        pool1 = torch.cuda.graph_pool_handle() if SEPARATE_POOLS else pool0
        with torch.cuda.graph(g0, pool=pool0):
            r0 = self._enqueue_bucketize0(coords)
        with torch.cuda.graph(g1, pool=pool1):
            self._want_out_bf16 = True
            try:
                X, Cn, n_dev, runs = self._enqueue_rest(r0, coords, feats)
            finally:
                self._want_out_bf16 = False
            status = self._status_vector(runs, n_dev, zero1)
            out_bf16 = runs[-1].out_bf16 if runs[-1].out_bf16 is not None \
                else X.to(torch.bfloat16)
        return {"n": n, "g0": g0, "g1": g1, "X": X, "C": Cn, "runs": runs, "status": status,
                "out_bf16": out_bf16, "side": torch.cuda.Stream(), "coords": coords,
                "feats": feats,
                "zero1": zero1,
                "status_h": torch.empty(status.shape, dtype=status.dtype).pin_memory(),
                "out_h": torch.empty(out_bf16.shape, dtype=out_bf16.dtype).pin_memory()}

    def capture(self, n, feat_dtype=torch.bfloat16):
        """Capture the forward for n-point inputs into two CUDA graphs (see
        _capture_slot).  Inputs are the static buffers ``graph_coords`` (n,3)
        f64 and ``graph_feats`` (n,d); replay with ``forward_graph``."""
        self._graphs = self._capture_slot(n, feat_dtype)
        self.graph_coords = self._graphs["coords"]
        self.graph_feats = self._graphs["feats"]
        self._status_host = self._graphs["status_h"]
        return self._graphs

    def stream_host(self, scenes, on_result=None):
        """Pipelined end-to-end forward over a sequence of host scenes
        ``[(coords_h (n,3) f64, feats_h (n,d) bf16), ...]`` (pinned, equal n).
        Two graph slots alternate: step i's upload runs on an H2D stream
        while step i-1 computes, step i's coordinate-only graph g0 runs on its
        own stream under step i-1's g1 (after step i-1's cooperative stage-1
        PSH), and step i-1's read-back (last-stage bf16 features + status
        words) runs on a D2H stream under step i's compute.
        ``on_result(i, feats_host_view, n_out)`` is called in step order once a
        step's read-back landed (the view is reused two steps later); a step's
        errors are raised then, before its slot is reused."""
        n = scenes[0][0].shape[0]
        dt = scenes[0][1].dtype
        slots = getattr(self, "_slots", None)
        if slots is None or slots[0]["n"] != n or slots[0]["feats"].dtype != dt:
            slots = self._slots = [self._capture_slot(n, dt) for _ in range(2)]
            for sl in slots:
                for k in ("ev_c", "ev_in", "ev_g0", "ev_done", "ev_out"):
                    sl[k] = torch.cuda.Event()
                sl["pending"] = None
        if not hasattr(self, "_h2d"):
            self._h2d, self._d2h = torch.cuda.Stream(), torch.cuda.Stream()
            self._g0s = torch.cuda.Stream()
        compute = torch.cuda.current_stream()
        h2d, d2h, g0s = self._h2d, self._d2h, self._g0s

        def finish(sl):
            i = sl["pending"]
            if i is None:
                return
            sl["ev_out"].synchronize()
            sl["pending"] = None
            n_out = self._check(sl["status_h"].numpy(), sl["runs"])
            if on_result is not None:
                on_result(i, sl["out_h"][:n_out], n_out)

        def drain():
            # a previous call that raised may have left a read-back in flight:
            # wait for it and forget its step index before the slots are reused
            for sl in slots:
                if sl["pending"] is not None:
                    sl["ev_out"].synchronize()
                    sl["pending"] = None

        drain()
        try:
            self._stream_steps(scenes, slots, compute, h2d, d2h, g0s, finish)
        finally:
            drain()

    def _stream_steps(self, scenes, slots, compute, h2d, d2h, g0s, finish):
        for i, (ch, fh) in enumerate(scenes):
            sl = slots[i % 2]
            # everything of step i is enqueued before the host blocks on step
            # i-2's read-back, so the upload of step i overlaps step i-1's
            # compute even when the PCIe copies are slower than a step
            if i >= 2:
                h2d.wait_event(sl["ev_done"])            # step i-2's inputs are free
            with torch.cuda.stream(h2d):
                sl["coords"].copy_(ch, non_blocking=True)
                sl["ev_c"].record(h2d)                   # g0 needs the coordinates only
                sl["feats"].copy_(fh, non_blocking=True)
                sl["ev_in"].record(h2d)
            if G0_CONCURRENT:
                # g0 (coordinate-only) on its own stream, under step i-1's g1
                g0s.wait_event(sl["ev_c"])
                if i >= 2:
                    g0s.wait_event(sl["ev_done"])        # step i-2 done with the slot
                    if not SEPARATE_POOLS:               # (round-1 layout: shared pool)
                        g0s.wait_event(sl["ev_out"])
                if i >= 1 and PSH_GATE:                   # not under step i-1's cooperative PSHs
                    prev = slots[(i - 1) % 2]
                    if any(getattr(pr, "psh_on_main", False) for pr in prev["runs"]):
                        g0s.wait_event(prev["ev_done"])   # a PSH without an event: serial
                    for pr in prev["runs"]:
                        pev = getattr(pr, "psh_event", None)
                        if pev is not None:
                            g0s.wait_event(pev)
                with torch.cuda.stream(g0s):
                    sl["g0"].replay()
                    sl["ev_g0"].record(g0s)
                compute.wait_event(sl["ev_g0"])
            else:
                compute.wait_event(sl["ev_c"])
            if i >= 2:
                compute.wait_event(sl["ev_out"])         # step i-2's outputs read out
            if not G0_CONCURRENT:
                sl["g0"].replay()
            compute.wait_event(sl["ev_in"])
            sl["g1"].replay()
            sl["ev_done"].record(compute)
            finish(sl)                                   # step i-2 read back + checked
            d2h.wait_event(sl["ev_done"])
            with torch.cuda.stream(d2h):
                sl["out_h"].copy_(sl["out_bf16"], non_blocking=True)
                sl["status_h"].copy_(sl["status"], non_blocking=True)
                sl["ev_out"].record(d2h)
            sl["pending"] = i
        nxt = len(scenes) % 2                             # drain in step order
        finish(slots[nxt])
        finish(slots[1 - nxt])

    def replay(self):
        """Replay both graphs on the current stream (inputs already in
        graph_coords / graph_feats); no host synchronisation."""
        g = self._graphs
        g["g0"].replay()
        g["g1"].replay()

    def check_graph(self):
        """Read the status words of the last replay (one sync); returns the
        final row count."""
        g = self._graphs
        self._status_host.copy_(g["status"])
        return self._check(self._status_host.numpy(), g["runs"])

    def forward_graph(self, coords, feats):
        """Graph-replayed forward on device inputs of the captured size."""
        g = self._graphs
        if g is None or coords.shape[0] != g["n"]:
            self.capture(coords.shape[0], feats.dtype)
            g = self._graphs
        self.graph_coords.copy_(coords)
        self.graph_feats.copy_(feats)
        self.replay()
        n_out = self.check_graph()
        return g["X"][:n_out], g["C"][:n_out]

    def forward_host(self, coords_h, feats_h, out_h=None):
        """End-to-end call with HOST buffers (pinned for async copies):
        coords (n,3) float64, feats (n,d) bf16.  Coordinates are uploaded and
        stage-0 bucketing (graph g0) starts at once; the feature upload runs
        on a side stream under it; graph g1 then runs the rest and the last
        stage's features (bf16, capacity rows) are copied back into the
        pinned ``out_h`` (a buffer kept with the graphs when None).  One sync (the status read) per call.  Returns
        (out_h[:n_out], n_out)."""
        n = coords_h.shape[0]
        g = self._graphs
        if g is None or g["n"] != n or self.graph_feats.dtype != feats_h.dtype:
            g = self.capture(n, feats_h.dtype)
        main = torch.cuda.current_stream()
        side = g["side"]
        self.graph_coords.copy_(coords_h, non_blocking=True)
        side.wait_stream(main)
        with torch.cuda.stream(side):
            self.graph_feats.copy_(feats_h, non_blocking=True)
        g["g0"].replay()
        main.wait_stream(side)
        g["g1"].replay()
        ob = g["out_bf16"]
        if out_h is None or tuple(out_h.shape) != tuple(ob.shape):
            out_h = g.get("out_h")
            if out_h is None:
                out_h = g["out_h"] = torch.empty(ob.shape, dtype=ob.dtype).pin_memory()
        out_h.copy_(ob, non_blocking=True)
        self._status_host.copy_(g["status"], non_blocking=True)
        main.synchronize()
        n_out = self._check(self._status_host.numpy(), g["runs"])
        return out_h[:n_out], n_out


class _CapPlan:
    """Pool tile table sized for capacity; the device totals hold the
    true tile / pooled-row counts."""

    def __init__(self, tile_start, tile_m, tile_out, ntiles, npool):
        self.tile_start, self.tile_m, self.tile_out = tile_start, tile_m, tile_out
        self.ntiles, self.npool = ntiles, npool


_BACKBONES = {}


def backbone_forward(coords, feats, stages=None):
    """Public entry: host or device arrays in; the caller's array type out
    (features float32, coordinates float64, last stage's scattered order).
    One Backbone per stage configuration is kept, and its forward is captured
    as CUDA graphs per input size and replayed (``Backbone.forward_graph``), so
    repeated calls of one size cost one upload, one replay and one read-back."""
    host = L.is_host(coords)
    key = tuple(stages) if stages is not None else None
    bb = _BACKBONES.get(key)
    if bb is None:
        bb = _BACKBONES[key] = Backbone(stages)
    if host:
        C = torch.from_numpy(np.ascontiguousarray(coords, dtype=np.float64)).to(L.device())
        X = torch.from_numpy(np.ascontiguousarray(feats, dtype=np.float32)).to(L.device())
    else:
        C = coords.to(L.device(), torch.float64)
        X = feats.to(L.device())
        if X.dtype not in (torch.float32, torch.bfloat16):
            X = X.to(torch.float32)
    if C.ndim != 2 or C.shape[1] != 3 or X.ndim != 2 or X.shape[0] != C.shape[0]:
        raise ConfigError("coords must be (N, 3) and feats (N, d) with matching N")
    f, c = bb.forward_graph(C.contiguous(), X.contiguous())
    # the graph's static buffers are overwritten by the next call: copy out
    return (f.cpu().numpy(), c.cpu().numpy()) if host else (f.clone(), c.clone())
