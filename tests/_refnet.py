"""torch fp64 SDNet (library ops) — test-side reference used (1) to pin the oracle's
SDNet forward and (2) to give the conditioning scale of the head dot product
for the bf16 tolerance: S = sum_i |wo_i h_i|."""
import numpy as np
import torch
import torch.nn.functional as F

from mfp_inputs import split_params


def torch_sdnet(flat, gb, queries, d=128, n_hidden=3, return_scale=False, round_to=None, approximate="none"):
    """round_to (e.g. torch.bfloat16): emulate the tensor-core chain's operands — the
    input activations and the weights of every hidden layer rounded (RN) to that
    type, products and sums in fp64; the last hidden layer's output (the head's
    input) stays unrounded, as in the chain.  approximate="tanh": the tensor-core
    paths' GELU form (mfp_sdnet_desc.gelu = 1) instead of the exact erf."""
    p = {k: torch.tensor(v, dtype=torch.float64) for k, v in split_params(np.asarray(flat, np.float64), d, n_hidden).items()}
    x = torch.tensor(np.asarray(gb, np.float64))[:, None, :]
    for l in range(2):
        x = F.gelu(F.conv1d(F.pad(x, (2, 2), mode="circular"), p[f"conv{l}.w"], p[f"conv{l}.b"]), approximate=approximate)
    z = F.linear(x.flatten(1), p["W1"], p["b1"])
    X = torch.tensor(np.asarray(queries, np.float64))
    h = F.gelu(z[:, None, :] + F.linear(X, p["W2"])[None], approximate=approximate)
    for l in range(n_hidden):
        if round_to is not None:
            h = F.gelu(F.linear(h.to(round_to).double(), p[f"h{l}.W"].to(round_to).double(), p[f"h{l}.b"]),
                       approximate=approximate)
        else:
            h = F.gelu(F.linear(h, p[f"h{l}.W"], p[f"h{l}.b"]), approximate=approximate)
    y = (F.linear(h, p["wo"][None], p["bo"])[..., 0]).numpy()
    if return_scale:
        S = (h.abs() @ p["wo"].abs()).numpy()
        return y, S
    return y
