"""Bucket-swin scope scheduling and GPU attention.

Drop-in for bw/attention.py.  Scheduling (``build_schedule``,
``logical_gather``) is integer bookkeeping on the host exactly as in the
reference; ``tiled_attention`` / ``reference_attention`` run the fused
bucket-swin kernel of csrc/attn.cu (bf16 operands, fp32 accumulation and
softmax), which reads every scope's rows in place from the fixed scattered
layout — the "gather" channel of ``copy_meter`` stays 0 by construction and
the "attention" channel is charged analytically with the bytes the kernel
streams.
"""

import math
import os
import warnings
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib as L
from .bucketing import BucketAssignment
from .errors import ConfigError, NumericError

BLOCK_M = 128  # query rows per work item of the mma.sync kernels (csrc/attn.cu kBM)
def qstep_tc(dh):
    """Query rows per work item of the tcgen05 kernel (csrc/attn_tc.cu)."""
    return L.load().f3d_attention_tc_qstep(dh)
BLOCK_N = 64   # keys per streamed tile (csrc/attn.cu kBN)


class CopyMeter:
    """Counts feature bytes copied, split by channel (bw/attention.py:22-41)."""

    def __init__(self):
        self.bytes = {"gather": 0, "attention": 0}

    def add(self, channel: str, nbytes: int) -> None:
        self.bytes[channel] += int(nbytes)

    def reset(self) -> None:
        for k in self.bytes:
            self.bytes[k] = 0


copy_meter = CopyMeter()


@dataclass(frozen=True)
class AttentionParams:
    """bw/attention.py:44-66."""

    d_model: int
    n_heads: int
    tile_rows: int = 64

    def __post_init__(self):
        if self.d_model < 1 or self.n_heads < 1:
            raise ConfigError("d_model and n_heads must be >= 1")
        if self.d_model % self.n_heads:
            raise ConfigError(
                f"d_model ({self.d_model}) must be divisible by n_heads ({self.n_heads})")
        if self.tile_rows < 16 or self.tile_rows % 16:
            raise ConfigError(f"tile_rows must be a positive multiple of 16, got {self.tile_rows}")

    @property
    def head_dim(self) -> int:
        return self.d_model // self.n_heads

    @property
    def scale(self) -> float:
        return 1.0 / math.sqrt(self.head_dim)


@dataclass(frozen=True)
class ScopeSchedule:
    """rounds[t] is a tuple of scopes (int64 bucket-id arrays) that partition
    all bucket ids (bw/attention.py:69-81)."""

    num_buckets: int
    window_w: int
    stride: int
    shift: int
    rounds: tuple

    def num_rounds(self) -> int:
        return len(self.rounds)


def build_schedule(num_buckets: int, window_w: int, stride: int = 1, shift: int = 0,
                   rounds: int = 1) -> ScopeSchedule:
    """Round t rotates the bucket list by (t*shift) mod W, chops it into
    windows of W*stride buckets and deals every stride-th bucket into a scope
    (bw/attention.py:84-117)."""
    if num_buckets < 1:
        raise ConfigError(f"num_buckets must be >= 1, got {num_buckets}")
    if window_w < 1:
        raise ConfigError(f"window_w must be >= 1, got {window_w}")
    if window_w > num_buckets:
        raise ConfigError(f"window_w ({window_w}) exceeds num_buckets ({num_buckets})")
    if stride < 1:
        raise ConfigError(f"stride must be >= 1, got {stride}")
    if not 0 <= shift < window_w:
        raise ConfigError(f"shift must satisfy 0 <= shift < window_w, got {shift}")
    if rounds < 1:
        raise ConfigError(f"rounds must be >= 1, got {rounds}")
    span = window_w * stride
    out = []
    for t in range(rounds):
        order = (np.arange(num_buckets, dtype=np.int64) + (t * shift) % window_w) % num_buckets
        scopes = []
        for s0 in range(0, num_buckets, span):
            chunk = order[s0:s0 + span]
            for lane in range(stride):
                sc = chunk[lane::stride]
                if len(sc):
                    scopes.append(sc)
        out.append(tuple(scopes))
    return ScopeSchedule(num_buckets=num_buckets, window_w=window_w, stride=stride, shift=shift,
                         rounds=tuple(out))


def _table_np(assignment):
    if isinstance(assignment, BucketAssignment):
        st, ln = assignment.bucket_table(split_recycle=False)
    else:
        st, ln = assignment
    to = lambda a: a.detach().cpu().numpy() if isinstance(a, torch.Tensor) else np.asarray(a)
    return to(st).astype(np.int64), to(ln).astype(np.int64)


def logical_gather(assignment, scope):
    """[(start, stop), ...] of the scope's non-empty buckets; copies nothing
    (bw/attention.py:120-139)."""
    starts, lengths = _table_np(assignment)
    ranges = []
    for b in np.asarray(scope, dtype=np.int64):
        if b < 0 or b >= len(starts):
            raise ConfigError(f"scope bucket id {int(b)} outside the bucket table")
        if lengths[b] == 0:
            continue
        ranges.append((int(starts[b]), int(starts[b]) + int(lengths[b])))
    return ranges


# --------------------------------------------------------------- kernel plan

def plan_arrays(starts, lens, members, qstep=BLOCK_M):
    """Vectorised scope planning.  members: (n_scopes, W) bucket ids (-1 pad)
    over a (starts, lens) table.  Returns int32 host arrays: scope_seg
    (n_scopes+1), seg_start, seg_vstart, scope_len, work (nwork, 2) — adjacent
    buckets merged into one physical segment, work items (scope, q_start) in
    longest-scope-first order."""
    starts = np.asarray(starts, dtype=np.int64)
    lens = np.asarray(lens, dtype=np.int64)
    M = np.asarray(members, dtype=np.int64)
    ns, W = M.shape
    ok = M >= 0
    Mi = np.where(ok, M, 0)
    st = np.where(ok, starts[Mi], 0)
    ln = np.where(ok, lens[Mi], 0)
    ln[~ok] = 0
    valid = ln > 0
    sc_of = np.repeat(np.arange(ns), W).reshape(ns, W)[valid]
    st_v = st[valid]
    ln_v = ln[valid]
    scope_len = np.bincount(sc_of, weights=ln_v, minlength=ns).astype(np.int64)
    # virtual start within the scope (exclusive prefix of lengths per scope)
    csum = np.cumsum(ln_v)
    first_of_scope = np.r_[True, sc_of[1:] != sc_of[:-1]] if len(sc_of) else np.zeros(0, bool)
    scope_base = np.zeros(ns, dtype=np.int64)
    if len(sc_of):
        scope_base[sc_of[first_of_scope]] = (csum - ln_v)[first_of_scope]
    vstart = csum - ln_v - scope_base[sc_of] if len(sc_of) else csum
    prev_end = np.r_[-1, (st_v + ln_v)[:-1]] if len(sc_of) else st_v
    new_seg = first_of_scope | (st_v != prev_end)
    seg_start = st_v[new_seg]
    seg_vstart = vstart[new_seg]
    nseg = np.bincount(sc_of[new_seg], minlength=ns) if len(sc_of) else np.zeros(ns, np.int64)
    scope_seg = np.r_[0, np.cumsum(nseg)]
    order = np.argsort(-scope_len, kind="stable")
    live = order[scope_len[order] > 0]
    nt = -(-scope_len[order] // qstep)
    wscope = np.repeat(order, nt)
    wfirst = np.repeat(np.cumsum(nt) - nt, nt)
    wq = (np.arange(len(wscope)) - wfirst) * qstep
    work = np.stack([wscope, wq], 1) if len(wscope) else np.zeros((0, 2), np.int64)
    i32 = lambda x: np.ascontiguousarray(x, dtype=np.int32)
    return {"scope_seg": i32(scope_seg), "scope_nseg": i32(nseg), "seg_start": i32(seg_start),
            "seg_vstart": i32(seg_vstart), "scope_len": i32(scope_len), "work": i32(work),
            "scope_order": i32(live)}


def schedule_members(schedule: "ScopeSchedule", t: int):
    """(n_scopes, W) member matrix of round t (-1 padded)."""
    scopes = schedule.rounds[t]
    W = max((len(s) for s in scopes), default=1)
    M = np.full((len(scopes), max(1, W)), -1, dtype=np.int64)
    for i, sc in enumerate(scopes):
        M[i, :len(sc)] = sc
    return M


def round_members(nb, W, stride, shift, t):
    """Vectorised build_schedule for one round (bw/attention.py:104-115):
    position p of the rotated order belongs to scope (p // span, lane) with
    lane = (p % span) % stride, slot j = (p % span) // stride."""
    span = W * stride
    order = (np.arange(nb, dtype=np.int64) + (t * shift) % W) % nb
    p = np.arange(nb)
    chunk, r = p // span, p % span
    lane, j = r % stride, r // stride
    sid = chunk * stride + lane
    M = np.full((int(sid.max()) + 1 if nb else 0, W), -1, dtype=np.int64)
    M[sid, j] = order
    return M


class RoundPlan:
    """Device tables for one attention launch (see plan_arrays)."""

    def __init__(self, arrays, dev=None, uploaded=None, qstep=BLOCK_M):
        self.host = arrays
        self.qstep = qstep
        lens = arrays["scope_len"].astype(np.int64)
        self.nwork = int(arrays["work"].shape[0])
        self.nlive = int(arrays["scope_order"].shape[0])
        self.max_len = int(lens.max()) if len(lens) else 0
        self.flops_per_head = int((lens.astype(np.float64) ** 2).sum())   # sum m^2
        up = uploaded if uploaded is not None else L.upload(arrays)
        self.scope_seg = up["scope_seg"]
        self.scope_nseg = up["scope_nseg"]
        self.live = None
        self.seg_start = up["seg_start"]
        self.seg_vstart = up["seg_vstart"]
        self.scope_len = up["scope_len"]
        self.work = up["work"]
        self.scope_order = up["scope_order"]

    @classmethod
    def from_ranges(cls, scope_ranges, dev=None, qstep=BLOCK_M):
        """Plan from explicit [(start, stop), ...] lists (one per scope)."""
        starts, lens, members = [], [], []
        W = max((len(r) for r in scope_ranges), default=1)
        M = np.full((len(scope_ranges), max(1, W)), -1, dtype=np.int64)
        k = 0
        for i, rg in enumerate(scope_ranges):
            for j, (a, b) in enumerate(rg):
                starts.append(a)
                lens.append(max(0, b - a))
                M[i, j] = k
                k += 1
        return cls(plan_arrays(np.array(starts + [0]), np.array(lens + [0]), M, qstep), qstep=qstep)


class DeviceRoundPlan:
    """Scope tables of one round built on the device by f3d_plan_round from
    the PSH counts/base (no per-scope host work, no read-back).  nwork /
    nlive are upper bounds for the launch grid; the kernels read the exact
    values from ``live``."""

    def __init__(self, counts_dev, base_dev, K, S, nb, W, stride, shift, t, n, qstep=BLOCK_M,
                 _buf=None):
        span = W * stride
        ns = -(-nb // span) * stride
        self.qstep = qstep
        self.nlive = ns
        self.nwork = n // qstep + ns
        self.max_len = W * S
        i32 = torch.int32
        buf = _buf if _buf is not None else L.empty((self.size_for(nb, W, stride, n, qstep),), i32)
        o = 0

        def take(k):
            nonlocal o
            v = buf[o:o + k]
            o += k
            return v
        self.scope_seg, self.scope_nseg, self.scope_len = take(ns), take(ns), take(ns)
        self.seg_start, self.seg_vstart = take(ns * W), take(ns * W)
        self.scope_order = take(ns)
        self.work = take(2 * self.nwork).view(-1, 2)
        self.live = take(8)
        if _buf is not None:
            return                       # filled by all_rounds' single launch
        L.call("f3d_plan_round", L.ptr(counts_dev), L.ptr(base_dev), K, S, nb, W, stride,
               (t * shift) % W, ns, L.ptr(self.scope_seg), L.ptr(self.scope_nseg),
               L.ptr(self.seg_start), L.ptr(self.seg_vstart), L.ptr(self.scope_len),
               L.ptr(self.scope_order), L.ptr(self.work), self.nwork, qstep, L.ptr(self.live),
               L.stream())

    @staticmethod
    def size_for(nb, W, stride, n, qstep):
        ns = -(-nb // (W * stride)) * stride
        return 3 * ns + 2 * ns * W + ns + 2 * (n // qstep + ns) + 8

    @classmethod
    def all_rounds(cls, counts_dev, base_dev, K, S, nb, W, stride, shift, rounds, n, qstep=BLOCK_M):
        """Plans of rounds 0..rounds-1 (rotation (t*shift) mod W) from one
        f3d_plan_rounds launch; each round's tables live round_stride int32
        apart in one buffer."""
        per = cls.size_for(nb, W, stride, n, qstep)
        buf = L.empty((rounds * per,), torch.int32)
        plans = [cls(counts_dev, base_dev, K, S, nb, W, stride, shift, t, n, qstep,
                     _buf=buf[t * per:(t + 1) * per]) for t in range(rounds)]
        p0 = plans[0]
        L.call("f3d_plan_rounds", L.ptr(counts_dev), L.ptr(base_dev), K, S, nb, W, stride, shift,
               rounds, per, p0.nlive, L.ptr(p0.scope_seg), L.ptr(p0.scope_nseg),
               L.ptr(p0.seg_start), L.ptr(p0.seg_vstart), L.ptr(p0.scope_len),
               L.ptr(p0.scope_order), L.ptr(p0.work), p0.nwork, qstep, L.ptr(p0.live), L.stream())
        return plans


def plan_schedule(table, schedule: ScopeSchedule, dev=None, qstep=BLOCK_M):
    """One RoundPlan per round of the schedule over a (starts, lengths) table."""
    starts, lengths = _table_np(table)
    plans = []
    for t in range(len(schedule.rounds)):
        M = schedule_members(schedule, t)
        if ((M >= len(starts)) | (M < -1)).any():
            raise ConfigError("scope bucket id outside the bucket table")
        plans.append(RoundPlan(plan_arrays(starts, lengths, M, qstep), qstep=qstep))
    return plans


def qstep_for(dh, masked=False):
    """Work-list stride matching the kernel attend() will pick."""
    return qstep_tc(dh) if (ATTN_IMPL == "tc" and not masked and dh % 8 == 0 and 8 <= dh <= 128) \
        else BLOCK_M


# "tc": tcgen05/TMEM kernel where eligible (default); "mma": mma.sync kernels
ATTN_IMPL = os.environ.get("F3D_ATTN", "tc")


def _tc_ok(q, k, v, dh, mask, plan):
    return (mask is None and dh % 8 == 0 and 8 <= dh <= 128
            and getattr(plan, "qstep", BLOCK_M) == qstep_tc(dh)
            and all(t.stride(0) % 8 == 0 and t.data_ptr() % 16 == 0 for t in (q, k, v)))


def attend(q, k, v, out, plan: RoundPlan, n_heads: int, dh: int, mask=None, starved=None,
           lse=None):
    """Launch bucket-swin attention for one round.  q/k/v: bf16 CUDA tensors
    whose rows hold heads side by side (head h at columns h*dh..), any row
    stride; out: bf16 or fp32 rows with the same head layout.  Uses the
    tcgen05 kernel when eligible, else the mma.sync kernels."""
    if _tc_ok(q, k, v, dh, mask, plan):
        L.call("f3d_bswin_attention_tc", L.ptr(q), L.ptr(k), L.ptr(v), q.stride(0), k.stride(0),
               v.stride(0), L.ptr(out), out.stride(0), int(out.dtype == torch.float32), n_heads,
               dh, L.ptr(plan.scope_seg), L.ptr(plan.scope_nseg), L.ptr(plan.seg_start),
               L.ptr(plan.seg_vstart), L.ptr(plan.scope_len), L.ptr(plan.work), plan.nwork,
               L.ptr(plan.live), min(q.shape[0], k.shape[0], v.shape[0]), L.ptr(lse),
               0 if lse is None else lse.stride(0), L.stream())
        return
    if lse is not None:
        raise ConfigError("lse output needs the tcgen05 attention path")
    if getattr(plan, "qstep", BLOCK_M) != BLOCK_M:
        raise ConfigError("attention plan stride does not match the selected kernel")
    L.call("f3d_bswin_attention", L.ptr(q), L.ptr(k), L.ptr(v), q.stride(0), k.stride(0),
           v.stride(0), L.ptr(out), out.stride(0), int(out.dtype == torch.float32), n_heads, dh,
           L.ptr(plan.scope_seg), L.ptr(plan.scope_nseg), L.ptr(plan.seg_start),
           L.ptr(plan.seg_vstart), L.ptr(plan.scope_len), L.ptr(plan.work), plan.nwork,
           L.ptr(plan.scope_order), plan.nlive, plan.max_len, L.ptr(plan.live), L.ptr(mask),
           L.ptr(starved), L.stream())


def _check_finite(name, t):
    if t.numel() and not bool(torch.isfinite(t).all()):
        raise NumericError(f"{name} contains non-finite values")


def _prep_qkv(Q, K, V, params):
    host = L.is_host(Q)
    ts = []
    for name, a in (("Q", Q), ("K", K), ("V", V)):
        t = L.to_dev(a, torch.float64 if not isinstance(a, torch.Tensor) else a.dtype)
        if t.ndim != 2:
            raise ConfigError(f"{name} must be 2-D")
        ts.append(t)
    return ts, host


def tiled_attention(Q, K, V, params: AttentionParams, ranges=None, mask=None):
    """Online-softmax attention over the rows of ``ranges`` (one scope),
    bw/attention.py:188-268.  Returns the real rows of every range in range
    order.  Masked keys are excluded, masked query rows give zeros, and rows
    with no valid key give zeros plus a RuntimeWarning."""
    (q, k, v), host = _prep_qkv(Q, K, V, params)
    if q.shape != k.shape or q.shape != v.shape:
        raise ConfigError("Q, K, V must share one shape")
    if q.shape[1] != params.d_model:
        raise ConfigError(f"feature width {q.shape[1]} != d_model {params.d_model}")
    total = q.shape[0]
    if ranges is None:
        ranges = [(0, total)]
    ranges = [(int(a), int(b)) for a, b in ranges]
    for a, b in ranges:
        if not 0 <= a <= b <= total:
            raise ConfigError(f"range ({a}, {b}) outside [0, {total}]")
    mk = None
    if mask is not None:
        mk = L.to_dev(np.asarray(mask, dtype=bool) if not isinstance(mask, torch.Tensor) else mask,
                      torch.bool)
        if tuple(mk.shape) != (total,):
            raise ConfigError("mask must have shape (N,)")
        mk = mk.to(torch.uint8)
    real = [(a, b) for a, b in ranges if b > a]
    if not real:
        out = torch.empty((0, params.d_model), dtype=torch.float64, device=q.device)
        return L.out(out, host)
    rows = torch.cat([torch.arange(a, b, device=q.device) for a, b in real])
    for name, t in (("Q", q), ("K", k), ("V", v)):
        _check_finite(name, t[rows])
    dh = params.head_dim
    qb, kb, vb = (t.to(torch.bfloat16).contiguous() for t in (q, k, v))
    out = torch.zeros((total, params.d_model), dtype=torch.float32, device=q.device)
    # overlapping / repeated ranges are legal in the reference: run each
    # distinct physical range list as one scope over a private row space
    plan = RoundPlan.from_ranges([real], qstep=qstep_for(params.head_dim, mk is not None))
    starved = torch.zeros(1, dtype=torch.int32, device=q.device) if mk is not None else None
    m = sum(b - a for a, b in real)
    # bytes the kernel streams: Q once, K and V once per query tile (bf16)
    copy_meter.add("attention", 2 * m * params.d_model * (1 + 2 * (-(-m // BLOCK_M))))
    if _disjoint(real):
        attend(qb, kb, vb, out, plan, params.n_heads, dh, mask=mk, starved=starved)
        res = out[rows].to(torch.float64)
    else:
        qs, ks, vs = qb[rows].contiguous(), kb[rows].contiguous(), vb[rows].contiguous()
        o2 = torch.zeros((m, params.d_model), dtype=torch.float32, device=q.device)
        mk2 = mk[rows].contiguous() if mk is not None else None
        attend(qs, ks, vs, o2, RoundPlan.from_ranges([[(0, m)]], qstep=qstep_for(dh, mk2 is not None)),
               params.n_heads, dh, mask=mk2,
               starved=starved)
        res = o2.to(torch.float64)
    if mk is not None and not bool(mk[rows].any()):
        warnings.warn(f"{m} query rows had every key masked; their outputs are zero",
                      RuntimeWarning, stacklevel=2)
    return L.out(res, host)


def _disjoint(ranges):
    s = sorted(ranges)
    return all(s[i][1] <= s[i + 1][0] for i in range(len(s) - 1))


def reference_attention(Q, K, V, params: AttentionParams):
    """Dense attention over all rows (bw/attention.py:147-166); runs the same
    kernel as one scope.  NumericError on non-finite inputs."""
    (q, k, v), host = _prep_qkv(Q, K, V, params)
    for name, t in (("Q", q), ("K", k), ("V", v)):
        _check_finite(name, t)
    if q.shape[1] != params.d_model:
        raise ConfigError(f"feature width {q.shape[1]} != d_model {params.d_model}")
    m = q.shape[0]
    qb, kb, vb = (t.to(torch.bfloat16).contiguous() for t in (q, k, v))
    mk = k.shape[0]
    if v.shape[0] != mk or k.shape[1] != params.d_model or v.shape[1] != params.d_model:
        raise ConfigError("K and V must share one shape (n_keys, d_model)")
    if mk != m:
        # queries and keys of different sizes (the reference einsum takes any):
        # one scope over [Q rows; K/V rows], the Q rows marked query-only
        # (mask 2: excluded as keys) and the K/V rows key-only (their outputs
        # are dropped)
        if mk == 0:
            raise ConfigError("reference_attention needs at least one key")
        T = m + mk
        d = params.d_model
        q2 = torch.zeros((T, d), dtype=torch.bfloat16, device=q.device)
        k2 = torch.zeros_like(q2)
        v2 = torch.zeros_like(q2)
        q2[:m], k2[m:], v2[m:] = qb, kb, vb
        mask = torch.ones(T, dtype=torch.uint8, device=q.device)
        mask[:m] = 2
        o2 = torch.zeros((T, d), dtype=torch.float32, device=q.device)
        starved = torch.zeros(1, dtype=torch.int32, device=q.device)
        attend(q2, k2, v2, o2, RoundPlan.from_ranges([[(0, T)]], qstep=qstep_for(params.head_dim, True)),
               params.n_heads, params.head_dim, mask=mask, starved=starved)
        return L.out(o2[:m].to(torch.float64), host)
    out = torch.zeros((m, params.d_model), dtype=torch.float32, device=q.device)
    attend(qb, kb, vb, out, RoundPlan.from_ranges([[(0, m)]], qstep=qstep_for(params.head_dim)),
           params.n_heads, params.head_dim)
    return L.out(out.to(torch.float64), host)


def positional_encoding(coords, d_model: int, base: float = 10000.0):
    """Sinusoidal per-axis encoding, d_model/3 dims per axis as alternating
    sin/cos pairs (bw/attention.py:271-288); computed by f3d_positional_encoding
    in float64."""
    if d_model % 6:
        raise ConfigError(f"d_model must be divisible by 6, got {d_model}")
    host = L.is_host(coords)
    c = L.to_dev(coords, torch.float64)
    if c.ndim != 2 or c.shape[1] != 3:
        raise ConfigError(f"coords must have shape (m, 3), got {tuple(c.shape)}")
    out = L.empty((c.shape[0], d_model), torch.float64)
    L.call("f3d_positional_encoding", L.ptr(c), c.shape[0], d_model, float(base), 1,
           L.ptr(out), d_model, L.stream())
    return L.out(out, host)


def lowest_period(d_model: int, base: float = 10000.0) -> float:
    """Period of the lowest-frequency sin/cos pair (bw/attention.py:291-294)."""
    n_pairs = d_model // 6
    return 2.0 * math.pi * base ** ((n_pairs - 1) / n_pairs)
