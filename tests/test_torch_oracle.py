"""The float64 torch training oracle (oracle/torch_stage.py) reproduces the
numpy restatement of stage_forward (pinned to reference goldens) to 1e-12."""
import numpy as np
import torch

from oracle import restated as O
from oracle import torch_stage as T


def _instance(n=700, d=24, seed=3):
    coords = O.synth_cloud(seed, n, "uniform-box")
    vox = O.remap_nonnegative(O.voxelize(coords, (0, 0, 0), 1 / 8))
    K, S = 6, 128
    ids, offs, counts, base = O.psh_assign(vox, None, "zorder-div", K, S, 128)
    dest = O.dest_index(ids, offs, base, K)
    Cs = np.empty_like(coords)
    Cs[dest] = coords
    F = np.random.default_rng(seed).normal(size=(n, d))
    table = O.bucket_table(counts, base, K, S)
    rounds = O.build_schedule(len(table[0]), 2, 1, 1, 2)
    return F, Cs, table, rounds


def test_torch_oracle_matches_numpy_restatement():
    F, Cs, table, rounds = _instance()
    p = O.init_params(0, F.shape[1], n_heads=4)
    p["b_in"] = np.random.default_rng(1).normal(size=p["b_in"].shape) * 0.1
    ref = O.stage_forward(F, Cs, table, rounds, p)
    tp = T.params_to_torch(p)
    out = T.stage_forward(torch.tensor(F), Cs, T.scope_rows(table, rounds), tp, 4)
    rel = np.linalg.norm(out.detach().numpy() - ref) / np.linalg.norm(ref)
    assert rel < 1e-12, rel


def test_torch_oracle_gradients_finite_difference():
    F, Cs, table, rounds = _instance(n=200, d=12, seed=5)
    p = O.init_params(1, 12, n_heads=2)
    tp = T.params_to_torch(p)
    X = torch.tensor(F, requires_grad=True)
    rows = T.scope_rows(table, rounds)
    out = T.stage_forward(X, Cs, rows, tp, 2)
    (0.5 * (out ** 2).sum()).backward()
    g = tp["w_in"].grad[3, 5].item()
    eps = 1e-6
    with torch.no_grad():
        tp["w_in"][3, 5] += eps
        up = 0.5 * (T.stage_forward(torch.tensor(F), Cs, rows, tp, 2) ** 2).sum().item()
        tp["w_in"][3, 5] -= 2 * eps
        dn = 0.5 * (T.stage_forward(torch.tensor(F), Cs, rows, tp, 2) ** 2).sum().item()
    assert abs((up - dn) / (2 * eps) - g) < 1e-4 * max(1.0, abs(g))
