"""Variant oracle — TEST INFRASTRUCTURE ONLY (same rules as
efunc_oracle.py: only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference legs may use it; the product package never imports it).

The model families of Table 3 written out in float64 over ALL keys (global
support, as efunc_oracle.py):
  * polynomial degree 0, 1, 2 of Eq. poly-func:
      f(x) = circ + x^T diamond + 1/2 x^T square x,   x = q - k_i (shift invariance, L397-399),
    square symmetric, stored as its 6 unique entries (Hxx, Hyy, Hzz, Hxy, Hxz, Hyz) — Table 3
    "Deg 2, # 10" (1 + 3 + 6);
  * key banks: the fixed grid O (Eq. func-interp), the offset-only O^Delta with
    learnable keys k_n + Delta_n (Eq. func-with-offset; Table 3 Full-1/2), and their
    union O^{+Delta} (Eq. func-offset; Table 3 Full-3/4); every bank has a learnable
    scale s = ln beta (reading R-3, Table 3 "Scale L").
Channel layout per node (bank order grid, offset): grid bank [s, c, g(3) if deg >= 1,
H(6) if deg >= 2]; offset bank [Delta(3), s, c, g(3), H(6)]. Degree 1 with both banks is the
13-channel layout of efunc_oracle.py (Table 3 Full-4).

Forward: O = sum_i p_i f_i, G = sum_i p_i [df_i/dq + 2 beta_i d (O - f_i)] (Eq. func-normal,
L425-436, "valid for any choice of f"), df/dx = diamond + square x.
Backward (MSE upstream r = dL/dO, Alg. 2 L540-568 with the degree-2 factor df/dsquare):
  dO/dc = p, dO/dg = p d, dO/dH_aa = p d_a^2 / 2, dO/dH_ab = p d_a d_b (a != b),
  dO/ds = -p a (f - O), dO/dk = p [ -df/dx + 2 beta d (f - O) ]  (-> dO/dDelta for the offset bank).

Pins (tests/test_oracle_variants.py): reduces to efunc_oracle at degree 1 / both banks;
partition of unity with a shared global quadratic P (c_i = P(k_i), g_i = grad P(k_i), H_i = hess P):
O == P(q) and G == grad P(q) for any beta and Delta; degree 0 == normalised RBF (Eq. nrbf);
G against central differences of O; the MSE gradient against central differences of the loss;
Table 3 parameter counts.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .efunc_oracle import _chunks, node_positions

GRID, OFFSET = 1, 2
BOTH = GRID | OFFSET
NCOEF = {0: 1, 1: 4, 2: 10}
# unique entries of the symmetric square: (a, b) per stored slot
H_IDX = ((0, 0), (1, 1), (2, 2), (0, 1), (0, 2), (1, 2))


def bank_channels(degree: int) -> int:
    return 1 + NCOEF[degree]


def n_channels(banks: int, degree: int) -> int:
    """Channels per node: Table 3 "Ch" for learnable scales."""
    n = 0
    if banks & GRID:
        n += bank_channels(degree)
    if banks & OFFSET:
        n += 3 + bank_channels(degree)
    return n


def layout(banks: int, degree: int) -> dict:
    """Channel offsets: {'grid': s index or None, 'off': s index or None, 'delta': index or None}."""
    lay = {"grid": None, "off": None, "delta": None, "nch": n_channels(banks, degree)}
    o = 0
    if banks & GRID:
        lay["grid"] = o
        o += bank_channels(degree)
    if banks & OFFSET:
        lay["delta"] = o
        lay["off"] = o + 3
    return lay


@dataclass
class VKeys:
    pos: np.ndarray    # [K, 3]
    beta: np.ndarray   # [K]
    c: np.ndarray      # [K]
    g: np.ndarray      # [K, 3]   (zeros at degree 0)
    H: np.ndarray      # [K, 3, 3] symmetric (zeros below degree 2)
    bank: np.ndarray   # [K] GRID or OFFSET
    node: np.ndarray   # [K] node index n


def keys_from_theta(theta, R: int, banks: int, degree: int) -> VKeys:
    lay = layout(banks, degree)
    th = np.asarray(theta, dtype=np.float64).reshape(R ** 3, lay["nch"])
    k = node_positions(R)
    n = R ** 3
    pos, beta, c, g, H, bank, node = [], [], [], [], [], [], []

    def add(s0, p):
        beta.append(np.exp(th[:, s0]))
        c.append(th[:, s0 + 1])
        gg = th[:, s0 + 2:s0 + 5] if degree >= 1 else np.zeros((n, 3))
        HH = np.zeros((n, 3, 3))
        if degree >= 2:
            for slot, (a, b) in enumerate(H_IDX):
                HH[:, a, b] = th[:, s0 + 5 + slot]
                HH[:, b, a] = th[:, s0 + 5 + slot]
        g.append(gg)
        H.append(HH)
        pos.append(p)
    if banks & GRID:
        add(lay["grid"], k)
        bank.append(np.full(n, GRID)); node.append(np.arange(n))
    if banks & OFFSET:
        add(lay["off"], k + th[:, lay["delta"]:lay["delta"] + 3])
        bank.append(np.full(n, OFFSET)); node.append(np.arange(n))
    return VKeys(np.concatenate(pos), np.concatenate(beta), np.concatenate(c), np.concatenate(g),
                 np.concatenate(H), np.concatenate(bank), np.concatenate(node))


def _terms(keys: VKeys, q):
    D = q[:, None, :] - keys.pos[None, :, :]                            # d = q - k
    A = keys.beta[None, :] * np.sum(D * D, axis=2)                      # a = beta |d|^2
    HD = np.einsum("iab,jib->jia", keys.H, D)                           # square d
    F = keys.c[None, :] + np.sum(keys.g[None] * D, axis=2) + 0.5 * np.sum(D * HD, axis=2)
    Fd = keys.g[None] + HD                                              # df/dx = diamond + square d
    return D, A, F, Fd


@dataclass
class VForward:
    O: np.ndarray
    G: np.ndarray
    lam: np.ndarray


def forward(theta, R: int, q, banks: int = BOTH, degree: int = 1) -> VForward:
    """Eq. func-interp / func-with-offset / func-offset with the Eq. poly-func f of `degree`,
    global softmax with the per-query max shift (reading R-5), and Eq. func-normal."""
    q = np.asarray(q, dtype=np.float64).reshape(-1, 3)
    keys = keys_from_theta(theta, R, banks, degree)
    J, K = q.shape[0], keys.pos.shape[0]
    O = np.zeros(J); G = np.zeros((J, 3)); lam = np.zeros(J)
    for j0, j1 in _chunks(J, K):
        D, A, F, Fd = _terms(keys, q[j0:j1])
        m = A.min(axis=1)
        W = np.exp(-(A - m[:, None]))
        Z = W.sum(axis=1)
        P = W / Z[:, None]
        Oc = np.sum(P * F, axis=1)
        U = 2.0 * keys.beta[None, :, None] * D
        G[j0:j1] = np.sum(P[:, :, None] * (Fd + U * (Oc[:, None] - F)[:, :, None]), axis=1)
        O[j0:j1] = Oc
        lam[j0:j1] = -m + np.log(Z)
    return VForward(O, G, lam)


def backward(theta, R: int, q, fwd: VForward, dL_dO, banks: int = BOTH, degree: int = 1) -> np.ndarray:
    """dL/dtheta [R^3, nch] for an upstream r = dL/dO (Alg. 2)."""
    lay = layout(banks, degree)
    q = np.asarray(q, dtype=np.float64).reshape(-1, 3)
    r = np.asarray(dL_dO, dtype=np.float64).reshape(-1)
    keys = keys_from_theta(theta, R, banks, degree)
    K = keys.pos.shape[0]
    dc = np.zeros(K); dg = np.zeros((K, 3)); dH = np.zeros((K, 6)); ds = np.zeros(K); dk = np.zeros((K, 3))
    for j0, j1 in _chunks(q.shape[0], K):
        D, A, F, Fd = _terms(keys, q[j0:j1])
        P = np.exp(-A - fwd.lam[j0:j1, None])
        FmO = F - fwd.O[j0:j1, None]
        rP = r[j0:j1, None] * P
        dc += rP.sum(axis=0)
        dg += np.sum(rP[:, :, None] * D, axis=0)
        for slot, (a, b) in enumerate(H_IDX):
            fac = 0.5 if a == b else 1.0
            dH[:, slot] += fac * np.sum(rP * D[:, :, a] * D[:, :, b], axis=0)
        ds += np.sum(rP * (-A) * FmO, axis=0)
        dk += np.sum(rP[:, :, None] * (-Fd + 2.0 * keys.beta[None, :, None] * D * FmO[:, :, None]), axis=0)
    n = R ** 3
    grad = np.zeros((n, lay["nch"]))

    def put(s0, sel):
        grad[:, s0] = ds[sel]
        grad[:, s0 + 1] = dc[sel]
        if degree >= 1:
            grad[:, s0 + 2:s0 + 5] = dg[sel]
        if degree >= 2:
            grad[:, s0 + 5:s0 + 11] = dH[sel]
    o = 0
    if banks & GRID:
        put(lay["grid"], slice(0, n))
        o = n
    if banks & OFFSET:
        put(lay["off"], slice(o, o + n))
        grad[:, lay["delta"]:lay["delta"] + 3] = dk[o:o + n]
    return grad


# ------------------------------------------------------------------ cosine-series stacks (§4.4)
def cosine_weights(q, B: int):
    """w_b(q) = cos(b pi x) cos(b pi y) cos(b pi z), b = 0 .. B-1, and their q-gradients
    (Eq. cosine-series; reading R-C: the 3-D cosine of "cos(b pi q)" is the
    separable product, and b runs over B terms so that B = 1 is Config G-6).
    Returns (W [B, J], dW [B, J, 3])."""
    q = np.asarray(q, dtype=np.float64).reshape(-1, 3)
    W = np.zeros((B, q.shape[0])); dW = np.zeros((B, q.shape[0], 3))
    for b in range(B):
        c = np.cos(b * np.pi * q); s = np.sin(b * np.pi * q)
        W[b] = c[:, 0] * c[:, 1] * c[:, 2]
        dW[b, :, 0] = -b * np.pi * s[:, 0] * c[:, 1] * c[:, 2]
        dW[b, :, 1] = -b * np.pi * c[:, 0] * s[:, 1] * c[:, 2]
        dW[b, :, 2] = -b * np.pi * c[:, 0] * c[:, 1] * s[:, 2]
    return W, dW


def cosine_forward(thetas, R: int, q, banks: int = GRID, degree: int = 1):
    """S(q) = sum_b w_b(q) O_b(q) and dS/dq = sum_b (dw_b O_b + w_b G_b), each O_b a model of the
    given family. thetas: [B, R^3, nch]. Returns (S, GS, per-band VForward list)."""
    q = np.asarray(q, dtype=np.float64).reshape(-1, 3)
    B = len(thetas)
    W, dW = cosine_weights(q, B)
    fs = [forward(thetas[b], R, q, banks, degree) for b in range(B)]
    S = sum(W[b] * fs[b].O for b in range(B))
    GS = sum(dW[b] * fs[b].O[:, None] + W[b][:, None] * fs[b].G for b in range(B))
    return S, GS, fs


def cosine_backward(thetas, R: int, q, fs, dL_dS, banks: int = GRID, degree: int = 1):
    """dL/dtheta_b = backward of band b with upstream w_b(q_j) dL/dS_j (chain rule). [B, R^3, nch]."""
    q = np.asarray(q, dtype=np.float64).reshape(-1, 3)
    W, _ = cosine_weights(q, len(thetas))
    return np.stack([backward(thetas[b], R, q, fs[b], W[b] * np.asarray(dL_dS, np.float64), banks, degree)
                     for b in range(len(thetas))])
