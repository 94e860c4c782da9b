"""Training oracle (TEST INFRASTRUCTURE ONLY): a float64 PyTorch restatement
of oracle.restated.stage_forward (bw/stage.py:99-159) whose autograd
gradients are the reference for the GPU backward pass (SURVEY.md §8(f) #2:
"the oracle is torch autograd on a float64 PyTorch restatement of
stage_forward, itself checked against the reference at <= 1e-12").

Parity pinning: tests/test_torch_oracle.py checks the forward of this module
against oracle.restated.stage_forward (itself pinned to reference goldens).
"""

import math

import numpy as np
import torch

from . import restated as R

PARAM_NAMES = ("w_q", "w_k", "w_v", "w_o", "b_q", "b_k", "b_v", "b_o", "ln1_gain", "ln1_bias",
               "ln2_gain", "ln2_bias", "w_in", "b_in", "w_out", "b_out")


def params_to_torch(p):
    """dict of float64 leaf tensors (requires_grad) from an oracle param dict."""
    return {k: torch.tensor(np.asarray(p[k], dtype=np.float64), requires_grad=True)
            for k in PARAM_NAMES}


def _ln(x, g, b, eps=1e-12):
    mu = x.mean(dim=-1, keepdim=True)
    var = ((x - mu) ** 2).mean(dim=-1, keepdim=True)   # population variance
    return (x - mu) / torch.sqrt(var + eps) * g + b


def _gelu(x):
    return 0.5 * x * (1.0 + torch.erf(x / math.sqrt(2.0)))


def _attention(q, k, v, H):
    m, d = q.shape
    dh = d // H
    qh, kh, vh = (t.reshape(m, H, dh).transpose(0, 1) for t in (q, k, v))
    s = qh @ kh.transpose(1, 2) / math.sqrt(dh)
    w = torch.softmax(s, dim=-1)
    return (w @ vh).transpose(0, 1).reshape(m, d)


def scope_rows(table, rounds):
    """Per round, per non-empty scope, the physical rows in range order."""
    out = []
    for scopes in rounds:
        rr = []
        for sc in scopes:
            rg = R.scope_ranges(table, sc)
            if rg:
                rr.append(np.concatenate([np.arange(a, b) for a, b in rg]))
        out.append(rr)
    return out


def stage_forward(F, C, rows_per_round, tp, H):
    """F (n,d) float64 tensor (may require grad), C (n,3) float64 numpy,
    rows_per_round from scope_rows, tp from params_to_torch."""
    C = np.asarray(C, dtype=np.float64)
    d = F.shape[1]
    lo = C.min(axis=0)
    ext = C.max(axis=0) - lo
    ext[ext == 0] = 1.0
    pe = torch.tensor(R.positional_encoding((C - lo) / ext, d))
    for rows_list in rows_per_round:
        x = _ln(F, tp["ln1_gain"], tp["ln1_bias"]) + pe
        Q = x @ tp["w_q"] + tp["b_q"]
        K = x @ tp["w_k"] + tp["b_k"]
        V = x @ tp["w_v"] + tp["b_v"]
        parts, idx = [], []
        for rows in rows_list:
            r = torch.as_tensor(rows)
            parts.append(_attention(Q[r], K[r], V[r], H))
            idx.append(r)
        att = torch.zeros_like(F)
        if parts:
            att = att.index_copy(0, torch.cat(idx), torch.cat(parts))
        F = F + att @ tp["w_o"] + tp["b_o"]
        h = _ln(F, tp["ln2_gain"], tp["ln2_bias"])
        F = F + _gelu(h @ tp["w_in"] + tp["b_in"]) @ tp["w_out"] + tp["b_out"]
    return F
