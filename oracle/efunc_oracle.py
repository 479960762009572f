"""efunc CPU oracle — TEST INFRASTRUCTURE ONLY.

Plain, slow, obviously-correct float64 implementation of what the efunc fit-step
hot path computes (arXiv 2505.21319, "efunc: An Efficient Function Representation
without Neural Networks"). Citations are `PAPER.md:L<n>` into the paper text
(/root/reference/PAPER.md, §/Eq./Alg. named beside each).

Who may use this module: only `tests/`, `__graft_entry__.smoke()` and
`bench.py`'s `cpu_baseline` / `--impl reference` legs. The product path
(`paper_2505_21319_b200`) never imports it, and this module imports nothing from
the product package: the two share no code. The only shared module is
`workloads/` (seeded synthetic inputs, none of the method's arithmetic).

What it computes — the exact GLOBAL-support result (§2.1.1,
Alg. 1 L505-518 loops over all I keys): every query sees all 2R^3 keys of the
O^{+Delta} model (Eq. func-offset), degree-1 polynomial values
(Eq. poly-func), softmax weights (Eq. nrbf / func-interp, L336-347,
L385-392).  `cutoff_T` optionally drops pairs with a_ij - m_j > T so the
truncation error of the GPU's certified cutoff can be measured (DESIGN.md
reading R-1); T=None is the paper's definition.

Layout (= Table 3 row Full-4):
theta is float [R^3, 13], node n = x + R*(y + R*z), channels
  0 s0 | 1 c0 | 2-4 g0 | 5-7 Delta | 8 s1 | 9 c1 | 10-12 g1
grid bank key n:   k_n,           beta = exp(s0), f = c0 + g0.(q - k_n)
offset bank key n: k_n + Delta_n, beta = exp(s1), f = c1 + g1.(q - k_n - Delta_n)
Lattice (reading R-2): k(i) = float32(-1 + 2 i/(R-1)) per axis, [-1,1]^3 inclusive.

Pins: every function here is checked in tests/test_oracle_*.py against things
other than itself (partition of unity, single key, degree-0 == O^nrbf, mpmath
brute force, central finite differences, torch.autograd in float64,
torch.optim.AdamW, the paper's parameter counts). No function is "parity unpinned".
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

NCH = 13
# channel indices (Table 3 Full-4; parameter space 5+|phi|+|phi'|, L456)
S0, C0, G0 = 0, 1, slice(2, 5)
DELTA = slice(5, 8)
S1, C1, G1 = 8, 9, slice(10, 13)

# pairs per numpy chunk (bounds the Jc x I x 3 float64 temporaries to ~100 MB)
_CHUNK_PAIRS = 1 << 22


def param_count(R: int, channels: int = NCH) -> int:
    """Total parameters R^3 * C (PAPER.md:L456 parameter space; Table 2, Table 3)."""
    return R ** 3 * channels


def lattice_1d(R: int) -> np.ndarray:
    """Lattice coordinates per axis: float32(-1 + 2 i/(R-1)) widened to float64 (reading R-2).

    R == 1 is a single key at the origin.
    """
    if R < 1:
        raise ValueError("R must be >= 1")
    if R == 1:
        return np.zeros(1, dtype=np.float64)
    i = np.arange(R, dtype=np.float64)
    return (-1.0 + 2.0 * i / (R - 1)).astype(np.float32).astype(np.float64)


def node_positions(R: int) -> np.ndarray:
    """[R^3, 3] base-lattice key positions k_n, node n = x + R*(y + R*z)."""
    t = lattice_1d(R)
    z, y, x = np.meshgrid(t, t, t, indexing="ij")
    return np.stack([x.ravel(), y.ravel(), z.ravel()], axis=1)


@dataclass
class Keys:
    """The union key set of O^{+Delta} (Eq. func-offset): 2R^3 keys."""
    pos: np.ndarray    # [2I, 3]  k_i  (grid bank first, then k_n + Delta_n)
    beta: np.ndarray   # [2I]     beta_i = exp(s_i)   (reading R-3)
    c: np.ndarray      # [2I]     constant term of f  (Eq. poly-func "circ")
    g: np.ndarray      # [2I, 3]  linear term of f   (Eq. poly-func "diamond")


def keys_from_theta(theta: np.ndarray, R: int) -> Keys:
    theta = np.asarray(theta, dtype=np.float64).reshape(R ** 3, NCH)
    k = node_positions(R)
    pos = np.concatenate([k, k + theta[:, DELTA]], axis=0)
    beta = np.exp(np.concatenate([theta[:, S0], theta[:, S1]]))
    c = np.concatenate([theta[:, C0], theta[:, C1]])
    g = np.concatenate([theta[:, G0], theta[:, G1]], axis=0)
    return Keys(pos, beta, c, g)


def _chunks(J: int, I: int):
    step = max(1, _CHUNK_PAIRS // max(I, 1))
    for j0 in range(0, J, step):
        yield j0, min(J, j0 + step)


def _pair_terms(keys: Keys, q: np.ndarray):
    """Per (query j, key i): d = q_j - k_i, a = beta_i ||d||^2, f = c_i + g_i . d."""
    D = q[:, None, :] - keys.pos[None, :, :]                 # [Jc, I, 3]
    A = keys.beta[None, :] * np.sum(D * D, axis=2)           # [Jc, I]
    F = keys.c[None, :] + np.sum(keys.g[None, :, :] * D, axis=2)
    return D, A, F


@dataclass
class Forward:
    O: np.ndarray        # [J]    O(q_j)                      Eq. func-interp
    G: np.ndarray        # [J,3]  dO/dq_j                     Eq. func-normal
    lam: np.ndarray      # [J]    lambda_j = ln e_j = ln sum_i exp(-a_ij)   (Alg. 1 "save e_j", log domain)
    m: np.ndarray        # [J]    m_j = min_i a_ij (the max-shift, reading R-5)
    ubar: np.ndarray     # [J,3]  sum_i p_ij u_ij, u = 2 beta d (needed by the Eikonal backward)
    kept: np.ndarray     # [J]    number of pairs with a_ij - m_j <= T (all pairs if T is None)


def forward(theta, R: int, q, cutoff_T: float | None = None) -> Forward:
    """Alg. 1 with the per-query max shift (L501), plus Eq. func-normal.

    For every query j over ALL keys i of the union set:
      a_ij = beta_i ||q_j - k_i||^2,  m_j = min_i a_ij
      w_ij = exp(-(a_ij - m_j))                       (exp(-a) scaled by e^{m_j})
      Z_j = sum_i w_ij,  O_j = sum_i w_ij f_ij / Z_j   (Alg. 1: e_j, numerator; O = m_j/e_j)
      lambda_j = -m_j + ln Z_j = ln e_j
      p_ij = w_ij / Z_j                               (softmax, Eq. nrbf)
      G_j = sum_i p_ij [ g_i + 2 beta_i d_ij (O_j - f_ij) ]   (Eq. func-normal)
    """
    q = np.asarray(q, dtype=np.float64).reshape(-1, 3)
    keys = keys_from_theta(theta, R)
    J, I = q.shape[0], keys.pos.shape[0]
    O = np.zeros(J); G = np.zeros((J, 3)); lam = np.zeros(J); mm = np.zeros(J)
    ub = np.zeros((J, 3)); kept = np.zeros(J, dtype=np.int64)
    for j0, j1 in _chunks(J, I):
        D, A, F = _pair_terms(keys, q[j0:j1])
        m = A.min(axis=1)
        W = np.exp(-(A - m[:, None]))
        if cutoff_T is not None:
            keep = (A - m[:, None]) <= cutoff_T
            W = np.where(keep, W, 0.0)
            kept[j0:j1] = keep.sum(axis=1)
        else:
            kept[j0:j1] = I
        Z = W.sum(axis=1)
        Oc = (W * F).sum(axis=1) / Z
        P = W / Z[:, None]
        U = 2.0 * keys.beta[None, :, None] * D                 # u_ij = 2 beta_i d_ij
        Gc = np.sum(P[:, :, None] * (keys.g[None, :, :] + U * (Oc[:, None] - F)[:, :, None]), axis=1)
        O[j0:j1] = Oc
        G[j0:j1] = Gc
        lam[j0:j1] = -m + np.log(Z)
        mm[j0:j1] = m
        ub[j0:j1] = np.sum(P[:, :, None] * U, axis=1)
    return Forward(O, G, lam, mm, ub, kept)


def mse_loss(O, o, J_global: int | None = None):
    """Eq. loss: L = (1/J) sum_j (O_j - o_j)^2; returns (L, dL/dO_j)."""
    O = np.asarray(O, dtype=np.float64); o = np.asarray(o, dtype=np.float64)
    if O.shape != o.shape:
        raise ValueError("length mismatch")
    J = O.size if J_global is None else J_global
    if J < 1:
        raise ValueError("J must be >= 1")
    return float(np.sum((O - o) ** 2) / J), 2.0 * (O - o) / J


def eikonal_loss(G, lam_e: float, J_global: int | None = None):
    """Eikonal term (reading R-12; PAPER.md:L439 states ||dO/dq||=1 as the SDF property):
    L_E = lam_e/J sum_j (||G_j|| - 1)^2; returns (L_E, dL_E/dG_j) with h_j = 0 where ||G_j|| = 0."""
    G = np.asarray(G, dtype=np.float64).reshape(-1, 3)
    J = G.shape[0] if J_global is None else J_global
    n = np.linalg.norm(G, axis=1)
    L = lam_e * float(np.sum((n - 1.0) ** 2)) / J
    with np.errstate(invalid="ignore", divide="ignore"):
        h = np.where(n[:, None] > 0, (2.0 * lam_e / J) * ((n - 1.0) / n)[:, None] * G, 0.0)
    return L, h


def backward(theta, R: int, q, fwd: Forward, dL_dO, dL_dG=None) -> np.ndarray:
    """Alg. 2 and the parameter-gradient equations (L569-598), summed
    over queries j (chain rule, L530-537).  Returns dL/dtheta as float64 [R^3, 13].

    Per pair, with l = p_ij = exp(-a_ij)/e_j = exp(-a_ij - lambda_j) (Alg. 2 "softmax"):
      dO/dphi_i: dO/dc = p,  dO/dg = p d                          (L594-597, df/dphi = (1, d))
      dO/dbeta_i = p (-||d||^2)(f - O)                              (L583-590)
         -> dO/ds_i = beta_i dO/dbeta_i = -p a (f - O)              (s = ln beta, reading R-3)
      dO/dk_i = p [ df/dk + 2 beta_i (f - O) d ], df/dk = -g        (L571-580, reading R-7)
         -> offset bank: dO/dDelta_n = dO/dk_{I+n}; grid keys are fixed (Table 3 "Keys F")
    If dL_dG (h_j = dL/dG_j) is given, the second-order terms of G (Eq. func-normal) are added,
    written out from the same chain rule:
      with u = 2 beta d, ubar = sum_i p u, T = h.G, t_i = h.g_i + (h.u_i)(O - f_i):
      dG-part/dc = p h.(ubar - u)
      dG-part/dg = p [ h + (h.(ubar - u)) d ]
      dG-part/ds = -p a [ (t - T) + (h.ubar)(f - O) ] + p (h.u)(O - f)
      dG-part/dk = p [ u (t - T) + 2 beta (f - O) h + (h.u) g + (h.ubar)(u (f - O) - g) ]
    """
    q = np.asarray(q, dtype=np.float64).reshape(-1, 3)
    r = np.asarray(dL_dO, dtype=np.float64).reshape(-1)
    h = None if dL_dG is None else np.asarray(dL_dG, dtype=np.float64).reshape(-1, 3)
    keys = keys_from_theta(theta, R)
    I2 = keys.pos.shape[0]
    J = q.shape[0]
    dc = np.zeros(I2); dg = np.zeros((I2, 3)); ds = np.zeros(I2); dk = np.zeros((I2, 3))
    for j0, j1 in _chunks(J, I2):
        D, A, F = _pair_terms(keys, q[j0:j1])
        O = fwd.O[j0:j1]
        P = np.exp(-A - fwd.lam[j0:j1, None])                   # l = exp(-beta||q-k||^2)/e_j
        FmO = F - O[:, None]                                    # f_i - O(q_j)
        rP = r[j0:j1, None] * P                                 # dL/dO_j * l
        beta = keys.beta[None, :]
        dc += rP.sum(axis=0)
        dg += np.sum(rP[:, :, None] * D, axis=0)
        ds += np.sum(rP * (-A) * FmO, axis=0)
        dk += np.sum(rP[:, :, None] * (-keys.g[None, :, :] + 2.0 * beta[:, :, None] * D * FmO[:, :, None]),
                     axis=0)
        if h is not None:
            hj = h[j0:j1]
            U = 2.0 * beta[:, :, None] * D
            ub = fwd.ubar[j0:j1]
            Gj = fwd.G[j0:j1]
            hU = np.sum(hj[:, None, :] * U, axis=2)             # h.u_i
            hub = np.sum(hj * ub, axis=1)[:, None]              # h.ubar
            Tj = np.sum(hj * Gj, axis=1)[:, None]               # T = h.G
            t = np.sum(hj[:, None, :] * keys.g[None, :, :], axis=2) - hU * FmO   # h.g + (h.u)(O - f)
            dc += np.sum(P * (hub - hU), axis=0)
            dg += np.sum(P[:, :, None] * (hj[:, None, :] + (hub - hU)[:, :, None] * D), axis=0)
            ds += np.sum(-P * A * ((t - Tj) + hub * FmO) - P * hU * FmO, axis=0)
            dk += np.sum(P[:, :, None] * (U * (t - Tj)[:, :, None]
                                          + 2.0 * beta[:, :, None] * FmO[:, :, None] * hj[:, None, :]
                                          + hU[:, :, None] * keys.g[None, :, :]
                                          + hub[:, :, None] * (U * FmO[:, :, None] - keys.g[None, :, :])),
                         axis=0)
    n = R ** 3
    grad = np.zeros((n, NCH))
    grad[:, S0] = ds[:n]; grad[:, C0] = dc[:n]; grad[:, G0] = dg[:n]
    grad[:, DELTA] = dk[n:]
    grad[:, S1] = ds[n:]; grad[:, C1] = dc[n:]; grad[:, G1] = dg[n:]
    return grad


@dataclass
class AdamW:
    """AdamW hyper-parameters: lr from PAPER.md:L698; the rest are reading R-10 (SPEC D16)."""
    lr: float = 6e-4
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8
    weight_decay: float = 1e-2
    decay_mask: int = (1 << C0) | (0b111 << 2) | (1 << C1) | (0b111 << 10)   # c, g only (SPEC D15)


def adamw_step(theta, grad, m, v, step: int, hp: AdamW):
    """One AdamW update ("AdamW"), torch.optim.AdamW semantics (reading R-10):
      theta <- theta (1 - lr wd mask_c)            (decoupled decay, applied first)
      m <- m + (1 - b1)(g - m);  v <- b2 v + (1 - b2) g^2
      theta <- theta - (lr / bc1) m / (sqrt(v)/sqrt(bc2) + eps),  bc_k = 1 - b_k^step
    `step` is the 1-based step count after increment.  Returns (theta, m, v) in float64."""
    theta = np.asarray(theta, np.float64).reshape(-1, NCH).copy()
    g = np.asarray(grad, np.float64).reshape(-1, NCH)
    m = np.asarray(m, np.float64).reshape(-1, NCH).copy()
    v = np.asarray(v, np.float64).reshape(-1, NCH).copy()
    mask = np.array([(hp.decay_mask >> ch) & 1 for ch in range(NCH)], dtype=np.float64)
    theta = theta * (1.0 - hp.lr * hp.weight_decay * mask[None, :])
    m = m + (1.0 - hp.beta1) * (g - m)
    v = hp.beta2 * v + (1.0 - hp.beta2) * g * g
    bc1 = 1.0 - hp.beta1 ** step
    bc2 = 1.0 - hp.beta2 ** step
    theta = theta - (hp.lr / bc1) * m / (np.sqrt(v) / math.sqrt(bc2) + hp.eps)
    return theta, m, v


def mean_shift_offsets(R: int, surface_pts, bandwidth: float = 100.0) -> np.ndarray:
    """Mean-shift offset initialisation (§3.3, N=16384 in the paper):
      Delta_i = sum_n exp(-100 ||k_i - s_n||^2) s_n / sum_n exp(-100 ||k_i - s_n||^2) - k_i
    evaluated with the per-key max shift (the weights otherwise underflow far from the surface).
    Returns [R^3, 3]."""
    s = np.asarray(surface_pts, dtype=np.float64).reshape(-1, 3)
    if s.shape[0] < 1:
        raise ValueError("N must be >= 1")
    k = node_positions(R)
    out = np.zeros_like(k)
    step = max(1, _CHUNK_PAIRS // s.shape[0])
    for i0 in range(0, k.shape[0], step):
        kk = k[i0:i0 + step]
        E = bandwidth * np.sum((kk[:, None, :] - s[None, :, :]) ** 2, axis=2)
        W = np.exp(-(E - E.min(axis=1, keepdims=True)))
        out[i0:i0 + step] = (W @ s) / W.sum(axis=1, keepdims=True) - kk
    return out
