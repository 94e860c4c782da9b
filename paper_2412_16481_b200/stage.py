"""Pre-norm transformer stage over bucket-swin scopes, on the GPU.

Drop-in for bw/stage.py.  Per round (bw/stage.py:134-158):

    x  = LN1(F) + PE(C)                 f3d_row_ln (fused with the previous
                                        round's MLP residual) -> bf16
    QKV = x @ [Wq|Wk|Wv] + b            one bf16 GEMM (f3d_gemm, tcgen05)
    A  = bucket-swin MHSA per scope     f3d_bswin_attention, one launch/round
    F += A @ Wo + bo ; h = LN2(F)       GEMM + f3d_row_ln (fused residual+LN)
    F += gelu(h @ Win + bin) @ Wout + bout    GEMM, f3d_bias_gelu, GEMM, row_ln

The residual stream F stays in the caller's float precision (float64 for host
float64 input, so zeroed branches leave F byte-identical as in
pkg/tests/test_stage.py:75-84; float32 otherwise); GEMM operands are bf16 with
fp32 accumulation.  Rows never move: attention reads each scope in place.
"""

import os
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib as L
from .attention import AttentionParams, ScopeSchedule, attend, plan_schedule, qstep_for
from .bucketing import BucketAssignment
from .errors import ConfigError

LN_EPS = 1e-12
# The QKV, O-projection and MLP GEMMs run on f3d_gemm (csrc/gemm_tc.cu: TMA-fed
# persistent tcgen05 GEMM, bias / GELU epilogue from TMEM).  F3D_OWN_GEMM=0
# selects the library GEMMs (A/B measurements only).
_OG = os.environ.get("F3D_OWN_GEMM", "qkv,o,in,out")
OWN_GEMM = {k for k in ("qkv", "o", "in", "out")
            if _OG == "1" or k in _OG.split(",")} if _OG != "0" else set()
# F3D_GEMM_RES_LN=1: the O projection and the MLP output GEMMs carry the
# residual + LayerNorm (+PE) row pass in their epilogue (f3d_gemm_res_ln: the
# fp32 residual tile TMA-loaded into shared memory, F and LN(F) leave by TMA
# stores) instead of a separate f3d_row_ln pass.  Correct (tests) but opt-in:
# measured 1.115 vs 1.06 ms per config-B step -- with the accumulator's
# thread-per-row layout, two epilogue warpgroups per SM recycle their residual
# tiles (store, reload) on the critical path of every tile, where the
# separate full-occupancy row pass streams F at HBM speed.
GEMM_RES_LN = os.environ.get("F3D_GEMM_RES_LN", "0") == "1"


@dataclass
class StageParams:
    """Projection, norm and MLP weights for one stage (bw/stage.py:25-54)."""

    attention: AttentionParams
    w_q: np.ndarray
    w_k: np.ndarray
    w_v: np.ndarray
    w_o: np.ndarray
    b_q: np.ndarray
    b_k: np.ndarray
    b_v: np.ndarray
    b_o: np.ndarray
    ln1_gain: np.ndarray
    ln1_bias: np.ndarray
    ln2_gain: np.ndarray
    ln2_bias: np.ndarray
    w_in: np.ndarray
    b_in: np.ndarray
    w_out: np.ndarray
    b_out: np.ndarray
    seed: int = 0

    @property
    def d_model(self) -> int:
        return self.attention.d_model

    @property
    def d_hidden(self) -> int:
        return self.w_in.shape[1]

    def device_weights(self):
        """bf16 GEMM operands and fp32 vectors on the device.  Rebuilt on every
        call so in-place edits of the host arrays are honoured."""
        f = lambda a, dt: L.to_dev(a.detach().cpu().numpy() if isinstance(a, torch.Tensor) else a, dt)
        bf, f32 = torch.bfloat16, torch.float32
        return {
            "w_qkv": torch.cat([f(self.w_q, bf), f(self.w_k, bf), f(self.w_v, bf)], 1).contiguous(),
            "b_qkv": torch.cat([f(self.b_q, bf), f(self.b_k, bf), f(self.b_v, bf)]).contiguous(),
            "w_o": f(self.w_o, bf), "b_o": f(self.b_o, f32),
            "w_in": f(self.w_in, bf), "b_in": f(self.b_in, f32),
            "w_out": f(self.w_out, bf), "b_out": f(self.b_out, f32),
            "w_in_t": f(self.w_in, bf).t().contiguous(), "w_out_t": f(self.w_out, bf).t().contiguous(),
            "w_o_t": f(self.w_o, bf).t().contiguous(),
            "w_qkv_t": torch.cat([f(self.w_q, bf), f(self.w_k, bf), f(self.w_v, bf)], 1).t().contiguous(),
            "b_qkv32": torch.cat([f(self.b_q, f32), f(self.b_k, f32), f(self.b_v, f32)]).contiguous(),
            "ln1_g": f(self.ln1_gain, f32), "ln1_b": f(self.ln1_bias, f32),
            "ln2_g": f(self.ln2_gain, f32), "ln2_b": f(self.ln2_bias, f32),
        }


def init_params(seed: int, d_model: int, d_hidden=None, n_heads: int = 4,
                tile_rows: int = 64) -> StageParams:
    """Seeded init (bw/stage.py:57-81): U(+-sqrt(3/fan_in)) drawn in the order
    q, k, v, o, in, out on the host with the reference's PCG64 stream, so the
    weights are bit-identical; biases zero, LN gains one."""
    if d_hidden is None:
        d_hidden = 4 * d_model
    attn = AttentionParams(d_model=d_model, n_heads=n_heads, tile_rows=tile_rows)
    rng = np.random.default_rng(seed)

    def mat(fan_in, fan_out):
        bound = np.sqrt(3.0 / fan_in)
        return rng.uniform(-bound, bound, size=(fan_in, fan_out))

    return StageParams(
        attention=attn,
        w_q=mat(d_model, d_model), w_k=mat(d_model, d_model),
        w_v=mat(d_model, d_model), w_o=mat(d_model, d_model),
        b_q=np.zeros(d_model), b_k=np.zeros(d_model), b_v=np.zeros(d_model), b_o=np.zeros(d_model),
        ln1_gain=np.ones(d_model), ln1_bias=np.zeros(d_model),
        ln2_gain=np.ones(d_model), ln2_bias=np.zeros(d_model),
        w_in=mat(d_model, d_hidden), b_in=np.zeros(d_hidden),
        w_out=mat(d_hidden, d_model), b_out=np.zeros(d_model), seed=seed)


def layer_norm(x, gain, bias, eps: float = 1e-12):
    """(x - mean) / sqrt(var + eps) * gain + bias, population variance
    (bw/stage.py:84-88); f3d_row_ln in float64 for host float64 input."""
    host = L.is_host(x)
    t = L.to_dev(x, torch.float64).contiguous()
    shp = t.shape
    t2 = t.reshape(-1, shp[-1]).clone()
    n, d = t2.shape
    out = L.empty((n, d), torch.float64)
    g = L.to_dev(gain, torch.float32)
    b = L.to_dev(bias, torch.float32)
    L.call("f3d_row_ln", L.ptr(t2), 1, d, None, 0, None, L.ptr(g), L.ptr(b), None, None, 0.0,
           L.ptr(out), 2, d, n, d, float(eps), L.stream())
    return L.out(out.reshape(shp), host)


def gelu(x):
    """Exact-erf GELU in float64 (bw/stage.py:91-92), f3d_gelu_f64."""
    host = L.is_host(x)
    t = L.to_dev(x, torch.float64).contiguous()
    out = torch.empty_like(t)
    L.call("f3d_gelu_f64", L.ptr(t), t.numel(), L.ptr(out), L.stream())
    return L.out(out, host)


class StageRunner:
    """Device-resident execution of one stage over a fixed scattered layout:
    weights, positional encoding and per-round attention plans are built once;
    ``run(F)`` then executes every round with no host synchronisation."""

    def __init__(self, coords, table, schedule: ScopeSchedule, params: StageParams, n: int,
                 f_dtype=torch.float32, weights=None, plans=None, n_dev=None):
        dev = L.device()
        self.p = params
        self.n = n
        self.d = params.d_model
        self.H = params.attention.n_heads
        self.dh = params.attention.head_dim
        self.w = weights if weights is not None else params.device_weights()
        self.plans = plans if plans is not None else plan_schedule(
            table, schedule, dev, qstep=qstep_for(params.attention.head_dim))
        self.f_dtype = f_dtype
        self.coords = L.to_dev(coords, torch.float64).contiguous()
        ws = L.empty((6 * 296,), torch.float64)
        self.lo_ext = L.empty((6,), torch.float64)
        L.call("f3d_coord_bbox", L.ptr(self.coords), n, L.ptr(ws), L.ptr(self.lo_ext),
               L.ptr(n_dev), L.stream())
        d, dhid = self.d, params.d_hidden
        self.x = L.empty((n, d), torch.bfloat16)
        self.qkv = L.empty((n, 3 * d), torch.bfloat16)
        self.a = L.empty((n, d), torch.bfloat16)
        self.y = L.empty((n, d), torch.bfloat16)
        self.n_dev = n_dev
        self.u = L.empty((n, dhid), torch.bfloat16)
        lib = L.load()
        ok = self.w.get("w_qkv_t") is not None
        self.own = {k for k, (k_, n_) in (("qkv", (d, 3 * d)), ("o", (d, d)), ("in", (d, dhid)),
                                          ("out", (dhid, d)))
                    if ok and k in OWN_GEMM and lib.f3d_gemm_supported(k_, n_)}
        self.own_gemm = bool(self.own)
        self.res_ln = (GEMM_RES_LN and f_dtype == torch.float32 and "o" in self.own
                       and "out" in self.own and bool(lib.f3d_gemm_res_ln_supported(d, d))
                       and bool(lib.f3d_gemm_res_ln_supported(dhid, d)))

    def _gemm(self, X, K, w_t, N, bias, gelu, Y):
        L.call("f3d_gemm", L.ptr(X), X.stride(0), self.n, K, L.ptr(w_t), N, L.ptr(bias),
               int(gelu), L.ptr(Y), Y.stride(0), L.ptr(self.n_dev), L.stream())

    def _gemm_res_ln(self, X, K, w_t, bias, F, g, b, pe, out):
        L.call("f3d_gemm_res_ln", L.ptr(X), X.stride(0), self.n, K, L.ptr(w_t), self.d,
               L.ptr(bias), L.ptr(F), F.stride(0), L.ptr(g), L.ptr(b),
               L.ptr(self.coords) if pe else None, L.ptr(self.lo_ext) if pe else None, 10000.0,
               LN_EPS, L.ptr(out), 0 if out is None else out.stride(0), L.ptr(self.n_dev),
               L.stream())

    def _row_ln(self, F, y, ybias, g, b, pe, out):
        L.call("f3d_row_ln", L.ptr(F), int(F.dtype == torch.float64), F.stride(0), L.ptr(y),
               0 if y is None else y.stride(0), L.ptr(ybias), L.ptr(g), L.ptr(b),
               L.ptr(self.coords) if pe else None, L.ptr(self.lo_ext) if pe else None, 10000.0,
               L.ptr(out), 0, 0 if out is None else out.stride(0), self.n, self.d, LN_EPS,
               L.stream())

    def run(self, F: torch.Tensor, x_ready: bool = False,
            defer_last_residual: bool = False, out_bf16=None) -> torch.Tensor:
        """F: (n, d) residual stream on the device (float32/float64), updated
        in place and returned.  x_ready: self.x already holds LN1(F) + PE
        (written by f3d_scatter_ln_pe together with F).  defer_last_residual:
        the last round's F += y + b_out is left to the consumer (self.y holds
        y; f3d_pool_reduce_res folds it into the pooling).  out_bf16: (n, d)
        bf16 buffer that receives a copy of the final F (same pass as the last
        residual, f3d_residual_out)."""
        w = self.w
        q, k, v = (self.qkv[:, i * self.d:(i + 1) * self.d] for i in range(3))
        if not x_ready:
            self._row_ln(F, None, None, w["ln1_g"], w["ln1_b"], True, self.x)
        R = len(self.plans)
        hook = getattr(self, "round_hook", None)
        d, dhid = self.d, self.p.d_hidden
        own = self.own
        for t, plan in enumerate(self.plans):
            if "qkv" in own:
                self._gemm(self.x, d, w["w_qkv_t"], 3 * d, w["b_qkv32"], False, self.qkv)
            else:
                torch.addmm(w["b_qkv"], self.x, w["w_qkv"], out=self.qkv)
            attend(q, k, v, self.a, plan, self.H, self.dh)
            if hook is not None:
                # test instrumentation (parity on the GPU's own round input):
                # called at enqueue time with the round's bf16 Q/K/V and output
                hook(t, q, k, v, self.a)
            if self.res_ln and F.dtype == torch.float32:
                # F += a W_o + b_o;  x = LN2(F)
                self._gemm_res_ln(self.a, d, w["w_o_t"], w["b_o"], F, w["ln2_g"], w["ln2_b"],
                                  False, self.x)
            else:
                if "o" in own:
                    self._gemm(self.a, d, w["w_o_t"], d, None, False, self.y)
                else:
                    torch.mm(self.a, w["w_o"], out=self.y)
                self._row_ln(F, self.y, w["b_o"], w["ln2_g"], w["ln2_b"], None, self.x)
            if "in" in own:
                self._gemm(self.x, d, w["w_in_t"], dhid, w["b_in"], True, self.u)
            else:
                torch.mm(self.x, w["w_in"], out=self.u)
                L.call("f3d_bias_gelu", L.ptr(self.u), self.n, self.u.shape[1],
                       L.ptr(w["b_in"]), L.stream())
            if t + 1 < R and self.res_ln and F.dtype == torch.float32:
                # F += g W_out + b_out;  x = LN1(F) + PE for the next round
                self._gemm_res_ln(self.u, dhid, w["w_out_t"], w["b_out"], F, w["ln1_g"],
                                  w["ln1_b"], True, self.x)
                continue
            if "out" in own:
                self._gemm(self.u, dhid, w["w_out_t"], d, None, False, self.y)
            else:
                torch.mm(self.u, w["w_out"], out=self.y)
            if t + 1 < R:
                self._row_ln(F, self.y, w["b_out"], w["ln1_g"], w["ln1_b"], True, self.x)
            elif not defer_last_residual:
                if out_bf16 is not None and F.dtype == torch.float32:
                    L.call("f3d_residual_out", L.ptr(F), F.stride(0), L.ptr(self.y),
                           self.y.stride(0), L.ptr(w["b_out"]), L.ptr(out_bf16),
                           out_bf16.stride(0), self.n, self.d, L.stream())
                else:
                    self._row_ln(F, self.y, w["b_out"], None, None, None, None)
        return F

    def attention_flops(self) -> int:
        """Algorithmic attention FLOPs per run: sum over rounds and scopes of
        4 * m_s^2 * d; device plans are read back here
        (bench bookkeeping only, outside the timed region)."""
        tot = 0
        for p in self.plans:
            if hasattr(p, "flops_per_head"):
                tot += p.flops_per_head
            else:
                ln = p.scope_len.to(torch.float64)
                tot += int((ln * ln).sum().item())
        return 4 * tot * self.d


def stage_forward(features, coords, assignment: BucketAssignment, schedule: ScopeSchedule,
                  params: StageParams, threads: int = 1):
    """Run every round of the schedule over scattered features
    (bw/stage.py:99-159); ``threads`` is accepted and ignored."""
    host = L.is_host(features)
    if isinstance(features, torch.Tensor):
        F = features.to(L.device()).clone()
        if F.dtype not in (torch.float32, torch.float64):
            F = F.to(torch.float32)
    else:
        F = L.to_dev(np.array(features, dtype=np.float64, copy=True), torch.float64)
    C = L.to_dev(coords, torch.float64)
    if assignment.num_batches != 1:
        raise ConfigError("stage_forward expects a single-batch assignment; process batches separately")
    if F.ndim != 2 or F.shape[0] != len(assignment):
        raise ConfigError("features must be (N, d) matching the assignment")
    if tuple(C.shape) != (F.shape[0], 3):
        raise ConfigError("coords must be (N, 3) matching features")
    if F.shape[1] != params.d_model:
        raise ConfigError(f"feature width {F.shape[1]} != d_model {params.d_model}")
    if assignment.S % 16:
        raise ConfigError(f"attention consumes buckets in 16-row tiles; "
                          f"S={assignment.S} is not a multiple of 16")
    table = assignment.bucket_table(split_recycle=True)
    if schedule.num_buckets != len(table[0]):
        raise ConfigError(
            f"schedule covers {schedule.num_buckets} buckets but the assignment "
            f"has {len(table[0])} (regular + recycle chunks)")
    if params.d_model % 6:
        raise ConfigError(f"d_model must be divisible by 6, got {params.d_model}")
    runner = StageRunner(C, table, schedule, params, F.shape[0], F.dtype)
    runner.run(F)
    return L.out(F, host)
