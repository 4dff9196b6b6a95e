"""Plain PyTorch fp32 restatement of the decoder (independent cross-check).

Standard ops (matmul, softmax, torch.exp) -- *not* the canonical arithmetic --
so agreement with the oracle / engine within 1e-3 relative on logits shows
the canonical arithmetic computes the intended transformer.
"""

from __future__ import annotations

import numpy as np
import torch

from paper_2506_07639_b200 import model as M


def build_weights(cfg: M.ModelConfig, seed: int) -> dict:
    d, f = cfg.d_model, cfg.d_ffn
    w = {
        "embed": M.init_linear(seed, M.T_EMBED, cfg.vocab, d),
        "lm_head": M.init_linear(seed, M.T_LM_HEAD, cfg.vocab, d),
        "final_norm": M.init_norm(seed, M.T_FINAL_NORM, d),
        "layers": [],
    }
    for l in range(cfg.n_layers):
        t = lambda k: M.layer_tensor(l, k)
        w["layers"].append({
            "attn_norm": M.init_norm(seed, t(M.L_ATTN_NORM), d),
            "wq": M.init_linear(seed, t(M.L_WQ), d, d),
            "wk": M.init_linear(seed, t(M.L_WK), d, d),
            "wv": M.init_linear(seed, t(M.L_WV), d, d),
            "wo": M.init_linear(seed, t(M.L_WO), d, d),
            "ffn_norm": M.init_norm(seed, t(M.L_FFN_NORM), d),
            "wg": M.init_linear(seed, t(M.L_WGATE), f, d),
            "wu": M.init_linear(seed, t(M.L_WUP), f, d),
            "wd": M.init_linear(seed, t(M.L_WDOWN), d, f),
        })
    return w


def _tt(a):
    return torch.from_numpy(np.asarray(a, dtype=np.float32))


def forward_logits(cfg: M.ModelConfig, w: dict, ids, vseed: int) -> torch.Tensor:
    """Logits [n, vocab] of every position of `ids` (teacher forced)."""
    ids = list(ids)
    n, d, H, hd = len(ids), cfg.d_model, cfg.n_heads, cfg.head_dim
    vis = M.vision_embeddings(vseed, cfg.n_vision, d)
    x = torch.stack([_tt(vis[p - 1]) if t == M.VIS_ID else _tt(w["embed"][t]) for p, t in enumerate(ids)])
    rope = _tt(M.rope_table(cfg))[:n]
    cos, sin = rope[:, 0, :], rope[:, 1, :]

    def rms(v, g):
        return v * torch.rsqrt(v.pow(2).mean(-1, keepdim=True) + cfg.rms_eps) * _tt(g)

    def rot(v):  # [n, H, hd]
        a, b = v[..., : hd // 2], v[..., hd // 2:]
        c, s = cos[:, None, :], sin[:, None, :]
        return torch.cat([a * c - b * s, b * c + a * s], dim=-1)

    mask = torch.full((n, n), float("-inf")).triu(1)
    for ly in w["layers"]:
        xn = rms(x, ly["attn_norm"])
        q = rot((xn @ _tt(ly["wq"]).T).view(n, H, hd))
        k = rot((xn @ _tt(ly["wk"]).T).view(n, H, hd))
        v = (xn @ _tt(ly["wv"]).T).view(n, H, hd)
        s = torch.einsum("qhd,khd->hqk", q, k) / np.sqrt(hd) + mask
        a = torch.einsum("hqk,khd->qhd", torch.softmax(s, -1), v).reshape(n, d)
        x = x + a @ _tt(ly["wo"]).T
        xn = rms(x, ly["ffn_norm"])
        g, u = xn @ _tt(ly["wg"]).T, xn @ _tt(ly["wu"]).T
        x = x + (torch.nn.functional.silu(g) * u) @ _tt(ly["wd"]).T
    return rms(x, w["final_norm"]) @ _tt(w["lm_head"]).T
