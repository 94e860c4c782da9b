"""Training step of one bucket-swin stage on the GPU (SURVEY.md §8(f) #2,
config E).  The reference has no backward pass; the
forward is bw/stage.py:134-158 exactly as ``StageRunner.run`` executes it,
with the activations each round's backward needs kept in HBM.

Per round, in reverse (F_in -> F_mid -> F_out):

    dF_out        -> db_out = colsum, dW_out = g^T dF, dg = dF W_out^T
    f3d_gelu_bwd  -> du (and db_in),  dW_in = x2^T du,  dx2 = du W_in^T
    f3d_ln_bwd    -> dF_mid = dF_out + LN2'(F_mid) dx2 (and dln2)
                  -> db_o = colsum, dW_o = a^T dF_mid, da = dF_mid W_o^T
    attention bwd -> dq, dk, dv by the fused kernels (f3d_attn_bwd, head dims
                     8..32): P = exp2(S*sl2 - lse) recomputed from the
                     forward kernel's LSE block by block, dS = P (dP - D)
                     with D = sum_j P dP / sum_j P (a first pass of the
                     query-block kernel, which then accumulates dQ); a
                     key-block kernel accumulates dK, dV -- no m x m tile.  Other head
                     dims: padded per-(scope, head) tiles (f3d_softmax_bwd
                     modes 0/1 between cuBLAS bmm's, D = sum_j P dP per row)
                  -> db_qkv = colsum, dW_qkv = x1^T dqkv, dx1 = dqkv W_qkv^T
    f3d_ln_bwd    -> dF_in = dF_mid + LN1'(F_in) dx1 (and dln1)

Weight gradients and the per-tile products are bf16 tensor-core cuBLAS GEMMs
with fp32 outputs (library GEMMs; activation gradients are rounded to bf16 as
GEMM operands, the residual-stream gradient stays fp32); the element-wise and
row work is csrc/train.cu.  ``allreduce_grads``
is the data-parallel exchange: one flat fp32 bucket, all_reduce(SUM)/world
(NCCL on the GPU, gloo in the CPU tests).
"""

import math
import os

import numpy as np
import torch
import torch.distributed as dist

from . import _lib as L
from .attention import ATTN_IMPL, attend
from .errors import ConfigError
from .stage import LN_EPS, StageParams, StageRunner

FUSED_ATTN_BWD = os.environ.get("F3D_FUSED_ATTN_BWD", "1") == "1"

GRAD_NAMES = ("w_q", "w_k", "w_v", "w_o", "b_q", "b_k", "b_v", "b_o", "ln1_gain", "ln1_bias",
              "ln2_gain", "ln2_bias", "w_in", "b_in", "w_out", "b_out")


def scope_index(plan, n: int):
    """Padded physical-row index of one round's scopes from the plan's host
    tables: (idx (ns, M) int64 with pad value n, M the longest scope rounded
    up to 16, lens (ns,) int32), rows in
    the scope's virtual (range) order — the order attention sees them."""
    h = getattr(plan, "host", None)
    if h is None:
        raise ConfigError("training needs host-planned rounds (plan_schedule)")
    seg, nseg = h["scope_seg"].astype(np.int64), h["scope_nseg"].astype(np.int64)
    sst, svs = h["seg_start"].astype(np.int64), h["seg_vstart"].astype(np.int64)
    slen = h["scope_len"].astype(np.int64)
    live = np.flatnonzero(slen > 0)
    ns = len(live)
    M = -(-int(slen.max()) // 16) * 16 if ns else 16          # GEMM / 16 B vector friendly
    idx = np.full((ns, M), n, dtype=np.int64)
    for i, s in enumerate(live):
        a, k = seg[s], nseg[s]
        for j in range(k):
            v0 = svs[a + j]
            v1 = svs[a + j + 1] if j + 1 < k else slen[s]
            idx[i, v0:v1] = sst[a + j] + np.arange(v1 - v0)
    return idx, slen[live].astype(np.int32)


class _ScopeGroup:
    """Scopes of similar length padded to a common M (a multiple of 16):
    per-(scope, head) gather/scatter indices over the (n*H, dh) head-row view,
    bh[b*M + i] = row(scope b//H, i)*H + b%H.  Pad entries (i >= len) point at
    row 0 -- their scores are zeroed by f3d_softmax_bwd, so they never reach a
    gradient -- and are dropped on the scatter back (dummy head row n*3H)."""

    def __init__(self, idx, lens, n, H, dev):
        self.ns, self.M = idx.shape
        valid = idx < n
        idx = np.where(valid, idx, 0)
        bh = (idx[:, None, :] * H + np.arange(H)[None, :, None]).reshape(-1)
        vbh = np.broadcast_to(valid[:, None, :], (self.ns, H, self.M)).reshape(-1)
        self.nvalid = int(vbh.sum())
        self.bh32 = torch.from_numpy(bh.astype(np.int32)).to(dev)
        r, h = bh // H, bh % H        # targets in the (n, 3, H, dh) = (n, 3d) dq|dk|dv layout
        self.dest = [torch.from_numpy(np.where(vbh, r * 3 * H + i * H + h, n * 3 * H)
                                      .astype(np.int32)).to(dev) for i in range(3)]
        self.len_bh = torch.from_numpy(np.repeat(lens, H)).to(dev)      # b = scope*H + h


class _RoundIndex:
    """One round's scopes in length groups: sorted by length and cut where the
    length falls below kRatio of the group's longest, so the padded M x M
    score tiles stay close to the real m x m work (one padded batch over all
    scopes of a config-B round wasted ~70 %)."""

    kRatio = 0.8

    def __init__(self, plan, n, H, dev):
        idx, lens = scope_index(plan, n)
        order = np.argsort(-lens, kind="stable")
        groups, start = [], 0
        for k in range(1, len(order) + 1):
            if k == len(order) or lens[order[k]] < self.kRatio * lens[order[start]]:
                sel = order[start:k]
                M = -(-int(lens[sel[0]]) // 16) * 16
                groups.append(_ScopeGroup(idx[sel, :M], lens[sel], n, H, dev))
                start = k
        self.groups = groups
        if sum(g.nvalid for g in groups) != n * H:
            raise ConfigError("the round's scopes do not cover every row exactly once")


class DeviceWeights:
    """fp32 master copies of a stage's parameters on the device plus the
    bf16/fp32 operand dict the forward reads (StageParams.device_weights
    layout); ``sgd`` updates the masters and re-casts in place, so trainers
    sharing this object (one per scene) see the step with no host traffic."""

    def __init__(self, params: StageParams):
        f = lambda a: L.to_dev(a.detach().cpu().numpy() if isinstance(a, torch.Tensor) else a,
                               torch.float32).contiguous()
        self.master = {k: f(getattr(params, k)) for k in GRAD_NAMES}
        self.d = params.d_model
        self.w = params.device_weights()

    def sync(self):
        m, w, d = self.master, self.w, self.d
        for i, k in enumerate(("w_q", "w_k", "w_v")):
            w["w_qkv"][:, i * d:(i + 1) * d].copy_(m[k])
        for i, k in enumerate(("b_q", "b_k", "b_v")):
            w["b_qkv"][i * d:(i + 1) * d].copy_(m[k])
        for k, mk in (("w_o", "w_o"), ("b_o", "b_o"), ("w_in", "w_in"), ("b_in", "b_in"),
                      ("w_out", "w_out"), ("b_out", "b_out"), ("ln1_g", "ln1_gain"),
                      ("ln1_b", "ln1_bias"), ("ln2_g", "ln2_gain"), ("ln2_b", "ln2_bias")):
            w[k].copy_(m[mk])
        w["w_in_t"].copy_(m["w_in"].t())
        w["w_out_t"].copy_(m["w_out"].t())
        w["w_o_t"].copy_(m["w_o"].t())
        w["w_qkv_t"].copy_(w["w_qkv"].t())
        for i, k in enumerate(("b_q", "b_k", "b_v")):
            w["b_qkv32"][i * d:(i + 1) * d].copy_(m[k])

    def sgd(self, grads, lr: float):
        for k in GRAD_NAMES:
            self.master[k].add_(grads[k], alpha=-lr)
        self.sync()


class StageTrainer:
    """Forward with saved activations and the backward of one stage over a
    fixed scattered layout (host-planned rounds).  Residual stream fp32."""

    def __init__(self, coords, table, schedule, params: StageParams, n: int,
                 weights: DeviceWeights = None):
        if params.d_model % 6:
            raise ConfigError(f"d_model must be divisible by 6, got {params.d_model}")
        self.p = params
        self.n_dev = torch.tensor([n], dtype=torch.int32, device=L.device())
        self.r = StageRunner(coords, table, schedule, params, n, torch.float32, n_dev=self.n_dev,
                             weights=None if weights is None else weights.w)
        self.n, self.d, self.H, self.dh = n, self.r.d, self.r.H, self.r.dh
        # fused attention backward (csrc/attn_bwd.cu) for head dims 8..32, else
        # the padded-tile path (F3D_FUSED_ATTN_BWD=0 forces it; A/B and tests)
        self.fused_bwd = (FUSED_ATTN_BWD and self.dh % 8 == 0 and 8 <= self.dh <= 32
                          and ATTN_IMPL == "tc")
        self.ix = None if self.fused_bwd else [_RoundIndex(p, n, self.H, L.device())
                                               for p in self.r.plans]
        self.saved = None

    def refresh_weights(self):
        """Re-cast the host parameters after a host-side update (sgd_step)."""
        self.r.w = self.p.device_weights()

    # ------------------------------------------------------------------ fwd
    def forward(self, F: torch.Tensor) -> torch.Tensor:
        """F (n, d) fp32 on the device, not modified; returns the stage output."""
        r, w, n, d = self.r, self.r.w, self.n, self.d
        if F.dtype != torch.float32 or tuple(F.shape) != (n, d):
            raise ConfigError("training forward takes fp32 (n, d) features")
        F = F.clone()
        saved = []
        y2 = None
        for t, plan in enumerate(r.plans):
            x1 = L.empty((n, d), torch.bfloat16)
            if t == 0:
                r._row_ln(F, None, None, w["ln1_g"], w["ln1_b"], True, x1)
            else:
                r._row_ln(F, y2, w["b_out"], w["ln1_g"], w["ln1_b"], True, x1)
            F_in = F.clone()
            qkv = torch.addmm(w["b_qkv"], x1, w["w_qkv"])
            q, k, v = (qkv[:, i * d:(i + 1) * d] for i in range(3))
            a = L.empty((n, d), torch.bfloat16)
            lse = L.empty((n, self.H), torch.float32)
            attend(q, k, v, a, plan, self.H, self.dh, lse=lse)
            y = torch.mm(a, w["w_o"])
            x2 = L.empty((n, d), torch.bfloat16)
            r._row_ln(F, y, w["b_o"], w["ln2_g"], w["ln2_b"], None, x2)
            F_mid = F.clone()
            u = torch.mm(x2, w["w_in"])
            g = u.clone()
            L.call("f3d_bias_gelu", L.ptr(g), n, g.shape[1], L.ptr(w["b_in"]), L.stream())
            y2 = torch.mm(g, w["w_out"])
            saved.append(dict(F_in=F_in, x1=x1, qkv=qkv, a=a, lse=lse, F_mid=F_mid, x2=x2, u=u,
                              g=g))
        if y2 is not None:
            r._row_ln(F, y2, w["b_out"], None, None, None, None)
        self.saved = saved
        return F

    # ------------------------------------------------------------------ bwd
    def _attn_bwd_fused(self, plan, qkv, lse, da):
        """dq|dk|dv (n, 3d) fp32 by the fused kernels (csrc/attn_bwd.cu): no
        m x m tile is formed; D = sum_j P dP / sum_j P per row is computed by
        the query-block kernel from the same recomputed P."""
        n, d, H, dh = self.n, self.d, self.H, self.dh
        q, k, v = (qkv[:, i * d:(i + 1) * d] for i in range(3))
        dob = da.to(torch.bfloat16)
        delta = L.empty((n, H), torch.float32)
        out = L.empty((n, 3 * d), torch.float32)
        L.call("f3d_attn_bwd", L.ptr(q), L.ptr(k), L.ptr(v), L.ptr(dob), q.stride(0), k.stride(0),
               v.stride(0), dob.stride(0), L.ptr(lse), lse.stride(0), L.ptr(delta), H,
               L.ptr(out), out.stride(0), L.ptr(out[:, d:]), out.stride(0), L.ptr(out[:, 2 * d:]),
               out.stride(0), H, dh, L.ptr(plan.scope_seg), L.ptr(plan.scope_nseg),
               L.ptr(plan.seg_start), L.ptr(plan.seg_vstart), L.ptr(plan.scope_len),
               int(plan.scope_len.shape[0]), int(plan.max_len), L.stream())
        return out

    def _attn_bwd(self, ix: _RoundIndex, qkv, a, lse, da):
        """dq|dk|dv (n, 3d) fp32 from the saved bf16 q/k/v/out, the LSE and
        da (fp32).  bf16 tensor-core GEMMs with fp32 outputs; P and dS are
        rounded to bf16 as GEMM operands (as the forward kernel rounds P)."""
        n, d, H, dh = self.n, self.d, self.H, self.dh
        bf = torch.bfloat16
        heads = [qkv[:, i * d:(i + 1) * d].contiguous().view(n * H, dh) for i in range(3)]
        heads.append(da.to(bf).view(n * H, dh))
        lse_r = lse.reshape(n * H, 1)
        sl2 = 1.4426950408889634 / math.sqrt(dh)
        out = torch.empty((n * 3 * H + 1, dh), dtype=torch.float32, device=qkv.device)
        for gp in ix.groups:
            ns, M = gp.ns, gp.M
            B = ns * H

            def gather(src):        # src (n*H, w) head rows -> (B*M, w), f3d_gather_rows
                t = torch.empty((B * M, src.shape[1]), dtype=src.dtype, device=src.device)
                L.call("f3d_gather_rows", L.ptr(src), L.ptr(gp.bh32), B * M,
                       src.shape[1] * src.element_size(), L.ptr(t), None, L.stream())
                return t

            Q, K, V, dO = (gather(t).view(B, M, dh) for t in heads)
            lse_b = gather(lse_r).view(B, M)
            S = torch.bmm(Q, K.transpose(1, 2), out_dtype=torch.float32)
            P = torch.empty((B, M, M), dtype=bf, device=qkv.device)
            L.call("f3d_softmax_bwd", L.ptr(S), None, L.ptr(lse_b), L.ptr(gp.len_bh), B, M, sl2,
                   0.0, 0, L.ptr(P), L.stream())
            del S
            dV = torch.bmm(P.transpose(1, 2), dO, out_dtype=torch.float32)
            dP = torch.bmm(dO, V.transpose(1, 2), out_dtype=torch.float32)
            dS = torch.empty_like(P)
            # D = sum_j P dP per row inside the kernel (same bf16 P as dS uses)
            L.call("f3d_softmax_bwd", L.ptr(dP), L.ptr(P), None, L.ptr(gp.len_bh), B, M, sl2,
                   1.0 / math.sqrt(dh), 1, L.ptr(dS), L.stream())
            del dP, P
            dQ = torch.bmm(dS, K, out_dtype=torch.float32)
            dK = torch.bmm(dS.transpose(1, 2), Q, out_dtype=torch.float32)
            for i, t in enumerate((dQ, dK, dV)):
                L.call("f3d_scatter_rows", L.ptr(t), L.ptr(gp.dest[i]), B * M, dh * 4,
                       L.ptr(out), None, L.stream())
        return out[:n * 3 * H].view(n, 3 * d)

    def _ln_bwd(self, x, dy, gain, dres, dgain, dbeta):
        dx = torch.empty_like(x)
        L.call("f3d_ln_bwd", L.ptr(x), x.stride(0), L.ptr(dy), int(dy.dtype == torch.bfloat16),
               dy.stride(0), L.ptr(gain), L.ptr(dres), dres.stride(0), L.ptr(dx), dx.stride(0),
               L.ptr(dgain), L.ptr(dbeta), self.n, self.d, LN_EPS, L.stream())
        return dx

    def _colsum(self, x, out):
        L.call("f3d_colsum", L.ptr(x), int(x.dtype == torch.bfloat16), x.stride(0), x.shape[0],
               x.shape[1], L.ptr(out), L.stream())

    def backward(self, dF: torch.Tensor):
        """dF: gradient of the loss w.r.t. the stage output (n, d) fp32.
        Returns (dF_in, grads) with grads keyed by GRAD_NAMES (fp32, device)."""
        if self.saved is None:
            raise ConfigError("backward() needs a preceding forward()")
        w, n, d = self.r.w, self.n, self.d
        dev = dF.device
        z = lambda *s: torch.zeros(s, dtype=torch.float32, device=dev)
        dhid = self.p.d_hidden
        G = dict(w_qkv=z(d, 3 * d), b_qkv=z(3 * d), w_o=z(d, d), b_o=z(d), ln1_gain=z(d),
                 ln1_bias=z(d), ln2_gain=z(d), ln2_bias=z(d), w_in=z(d, dhid), b_in=z(dhid),
                 w_out=z(dhid, d), b_out=z(d))
        bf = torch.bfloat16
        mm = lambda x, y: torch.mm(x, y, out_dtype=torch.float32)   # bf16 TC, fp32 out
        dF = dF.contiguous().float()
        for t in reversed(range(len(self.r.plans))):
            s = self.saved[t]
            dFb = dF.to(bf)
            self._colsum(dF, G["b_out"])
            G["w_out"] += mm(s["g"].t(), dFb)
            dg = mm(dFb, w["w_out"].t())
            du = torch.empty_like(dg)
            L.call("f3d_gelu_bwd", L.ptr(s["u"]), s["u"].stride(0), L.ptr(w["b_in"]), L.ptr(dg),
                   dg.stride(0), L.ptr(du), du.stride(0), L.ptr(G["b_in"]), n, dhid, L.stream())
            dub = du.to(bf)
            G["w_in"] += mm(s["x2"].t(), dub)
            dx2 = mm(dub, w["w_in"].t())
            dF = self._ln_bwd(s["F_mid"], dx2, w["ln2_g"], dF, G["ln2_gain"], G["ln2_bias"])
            dFb = dF.to(bf)
            self._colsum(dF, G["b_o"])
            G["w_o"] += mm(s["a"].t(), dFb)
            da = mm(dFb, w["w_o"].t())
            if self.fused_bwd:
                dqkv = self._attn_bwd_fused(self.r.plans[t], s["qkv"], s["lse"], da)
            else:
                dqkv = self._attn_bwd(self.ix[t], s["qkv"], s["a"], s["lse"], da)
            self._colsum(dqkv, G["b_qkv"])
            dqb = dqkv.to(bf)
            G["w_qkv"] += mm(s["x1"].t(), dqb)
            dx1 = mm(dqb, w["w_qkv"].t())
            dF = self._ln_bwd(s["F_in"], dx1, w["ln1_g"], dF, G["ln1_gain"], G["ln1_bias"])
        self.saved = None
        grads = {"w_q": G["w_qkv"][:, :d], "w_k": G["w_qkv"][:, d:2 * d],
                 "w_v": G["w_qkv"][:, 2 * d:], "b_q": G["b_qkv"][:d], "b_k": G["b_qkv"][d:2 * d],
                 "b_v": G["b_qkv"][2 * d:]}
        for k in ("w_o", "b_o", "ln1_gain", "ln1_bias", "ln2_gain", "ln2_bias", "w_in", "b_in",
                  "w_out", "b_out"):
            grads[k] = G[k]
        return dF, grads


def accumulate_grads(acc, grads):
    """acc += grads (per-scene gradients of one rank's batch); acc None -> copy."""
    if acc is None:
        return {k: grads[k].clone() for k in GRAD_NAMES}
    for k in GRAD_NAMES:
        acc[k].add_(grads[k])
    return acc


def flatten_grads(grads):
    """One contiguous fp32 bucket in GRAD_NAMES order (the all-reduce message)."""
    return torch.cat([grads[k].reshape(-1).float() for k in GRAD_NAMES])


def unflatten_grads(flat, like):
    out, o = {}, 0
    for k in GRAD_NAMES:
        m = like[k].numel()
        out[k] = flat[o:o + m].view(like[k].shape)
        o += m
    return out


def allreduce_grads(grads, group=None):
    """Data-parallel gradient average: all_reduce(SUM) of one flat bucket,
    divided by the world size.  No-op without a process
    group."""
    if not (dist.is_available() and dist.is_initialized()):
        return grads
    flat = flatten_grads(grads)
    dist.all_reduce(flat, op=dist.ReduceOp.SUM, group=group)
    flat /= dist.get_world_size(group)
    return unflatten_grads(flat, grads)


def sgd_step(params: StageParams, grads, lr: float):
    """In-place SGD on the host-side parameter arrays (or fp32 tensors)."""
    for k in GRAD_NAMES:
        cur = getattr(params, k)
        g = grads[k].detach()
        if isinstance(cur, torch.Tensor):
            cur.sub_(lr * g.to(cur.device, cur.dtype))
        else:
            cur -= lr * g.double().cpu().numpy()


class BackboneTrainer:
    """Training step of the multi-stage backbone (config E uses the B recipe:
    stage 0 -> mean pool (rho) -> re-bucketed stage 1 ...).
    The layout of every stage depends on the coordinates only, so the PSH
    bucketing, scatter maps, pooling partition and scope plans are built once
    per scene here (exactly as Backbone.forward builds them); forward/backward
    then run the stage trainers with the pooling as a fixed linear map:

        pool:    X_{s+1}[p] = mean_{i: parent[i] = p} F_s[i]   (f3d_pool_reduce,
                 members in index order as in the inference path)
        unpool:  dF_s[i] = dX_{s+1}[parent[i]] / size[parent[i]]

    ``stages`` are backbone.StageConfig; ``weights`` one DeviceWeights per stage."""

    def __init__(self, coords, stages, params, weights=None):
        from .backbone import Backbone
        from .pooling import TilePlan, _build
        from .attention import build_schedule
        dev = L.device()
        self.stages = tuple(stages)
        self.params = list(params)
        self.weights = list(weights) if weights is not None else [DeviceWeights(p) for p in params]
        C = L.to_dev(coords, torch.float64).contiguous()
        bb = Backbone(self.stages)
        self.levels = []
        for si, cfg in enumerate(self.stages):
            n = C.shape[0]
            asg, _, _ = bb.bucketize(C, cfg)
            dest = asg._dev["dest"].to(torch.int64)
            table = asg.bucket_table(split_recycle=True)
            sched = build_schedule(len(table[0]), cfg.W, cfg.stride, cfg.shift, cfg.rounds)
            Cs = torch.empty_like(C)
            Cs[dest] = C
            lvl = {"n": n, "dest": dest, "table": table, "schedule": sched, "coords": Cs,
                   "trainer": StageTrainer(Cs, table, sched, self.params[si], n,
                                           weights=self.weights[si])}
            if cfg.pool_rho:
                m = asg._mirrors()
                counts = m["counts"].cpu().numpy().astype(np.int64)
                base = m["base"].cpu().numpy().astype(np.int64)
                plan = TilePlan(counts, base, cfg.pool_rho, dev)
                members, sizes, _, _, _, flags = _build(Cs, plan, cfg.pool_rho)
                if int(flags.item()):
                    raise ConfigError(f"pooling partition failed (flags {int(flags.item())})")
                parent = L.empty((max(1, n),), torch.int32)
                L.call("f3d_pool_parent", L.ptr(members), L.ptr(sizes), plan.npool,
                       cfg.pool_rho, L.ptr(parent), None, L.stream())
                parent = parent[:n].to(torch.int64)
                lvl.update(members=members, sizes=sizes, npool=plan.npool, rho=cfg.pool_rho,
                           parent=parent,
                           inv_size=(1.0 / sizes[:plan.npool].to(torch.float32))[parent, None])
                C = self._pool(Cs, lvl)                    # centroids feed the next stage
            self.levels.append(lvl)

    @staticmethod
    def _pool(x, lvl):
        from .pooling import _reduce
        return _reduce(x, lvl["members"], lvl["sizes"], lvl["npool"], lvl["rho"], "mean")

    def forward(self, X: torch.Tensor) -> torch.Tensor:
        """X: (n0, d) fp32 features in the caller's (unscattered) row order.
        Returns the last stage's output rows in that stage's scattered order."""
        for lvl in self.levels:
            Xs = torch.empty_like(X)
            Xs[lvl["dest"]] = X
            out = lvl["trainer"].forward(Xs)
            X = self._pool(out, lvl) if "parent" in lvl else out
        return X

    def backward(self, dout: torch.Tensor):
        """dout: gradient w.r.t. forward()'s output.  Returns (dX in the
        caller's row order, [grads of stage 0, grads of stage 1, ...])."""
        grads = [None] * len(self.levels)
        d = dout
        for si in reversed(range(len(self.levels))):
            lvl = self.levels[si]
            if "parent" in lvl:                            # through the mean pool
                d = d[lvl["parent"]] * lvl["inv_size"]
            d, grads[si] = lvl["trainer"].backward(d)
            d = d[lvl["dest"]]                             # back through the scatter
        return d, grads

    def sgd(self, grads, lr: float):
        for w, g in zip(self.weights, grads):
            w.sgd(g, lr)
