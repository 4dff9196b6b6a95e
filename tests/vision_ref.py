"""Independent float64 numpy restatement of the vision tower + projector
(definition: oracle/oracle.c `or_vision_encode`; engine: csrc/vision.cu) --
test infrastructure that pins the C oracle's restatement."""

import numpy as np

from paper_2506_07639_b200.model import (LINEAR_MULT, NORM_MULT, get_config, get_vision, tensor_key,
                                         uniform_centered)

T_IMAGE, T_VB = 5, 1 << 20


def _lin(seed, tid, n):
    return uniform_centered(tensor_key(seed, tid), 0, n).astype(np.float64) * float(LINEAR_MULT)


def _norm(seed, tid, n):
    return 1.0 + uniform_centered(tensor_key(seed, tid), 0, n).astype(np.float64) * float(NORM_MULT)


def _ln(x, g, b, eps):
    mu = x.mean(axis=1, keepdims=True)
    var = ((x - mu) ** 2).mean(axis=1, keepdims=True)
    return (x - mu) / np.sqrt(var + eps) * g + b


def _gelu(z):
    return z / (1.0 + np.exp(-1.702 * z))


def vision_rows(llm: str, vision, seed: int, vseed: int) -> np.ndarray:
    cfg, v = get_config(llm), get_vision(vision, llm)
    g, P, d = v.img // v.patch, v.patches, v.d
    kp = (3 * v.patch * v.patch + 127) // 128 * 128
    img = uniform_centered(tensor_key(vseed, T_IMAGE), 0, 3 * v.img * v.img).astype(np.float64) * 2.0
    img = img.reshape(3, v.img, v.img)
    patches = np.zeros((P, kp))
    for p in range(P):
        gy, gx = divmod(p, g)
        patches[p, : 3 * v.patch ** 2] = img[:, gy * v.patch:(gy + 1) * v.patch,
                                             gx * v.patch:(gx + 1) * v.patch].reshape(-1)
    x = patches @ _lin(seed, T_VB + 0, d * kp).reshape(d, kp).T + _lin(seed, T_VB + 1, d)
    x = x + _lin(seed, T_VB + 2, P * d).reshape(P, d)
    hd = d // v.heads
    for layer in range(v.layers):
        b = T_VB + 16 + 16 * layer
        h = _ln(x, _norm(seed, b + 0, d), _lin(seed, b + 1, d), v.eps)
        qkv = h @ _lin(seed, b + 2, 3 * d * d).reshape(3 * d, d).T + _lin(seed, b + 3, 3 * d)
        att = np.zeros((P, d))
        for hh in range(v.heads):
            q = qkv[:, hh * hd:(hh + 1) * hd]
            k = qkv[:, d + hh * hd: d + (hh + 1) * hd]
            vv = qkv[:, 2 * d + hh * hd: 2 * d + (hh + 1) * hd]
            s = q @ k.T / np.sqrt(hd)
            s = np.exp(s - s.max(axis=1, keepdims=True))
            att[:, hh * hd:(hh + 1) * hd] = (s / s.sum(axis=1, keepdims=True)) @ vv
        x = x + att @ _lin(seed, b + 4, d * d).reshape(d, d).T + _lin(seed, b + 5, d)
        h = _ln(x, _norm(seed, b + 6, d), _lin(seed, b + 7, d), v.eps)
        h = _gelu(h @ _lin(seed, b + 8, v.mlp * d).reshape(v.mlp, d).T + _lin(seed, b + 9, v.mlp))
        x = x + h @ _lin(seed, b + 10, d * v.mlp).reshape(d, v.mlp).T + _lin(seed, b + 11, d)
    h = _ln(x, _norm(seed, T_VB + 3, d), _lin(seed, T_VB + 4, d), v.eps)
    h = _gelu(h @ _lin(seed, T_VB + 5, v.proj_hidden * d).reshape(v.proj_hidden, d).T
              + _lin(seed, T_VB + 6, v.proj_hidden))
    od = cfg.d_model
    return h @ _lin(seed, T_VB + 7, od * v.proj_hidden).reshape(od, v.proj_hidden).T + _lin(seed, T_VB + 8, od)
