"""CPU oracle of the NEXT-N2 actor-critic update (A2C) -- plain numpy, fp64.

*** TEST INFRASTRUCTURE ONLY. ***  Same rule as ``oracle/__init__.py``: only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py`` may import this module; it never imports the
product package and shares no code with it.

What it computes (SPEC a2c_update S:402-406: "single gradient step on loss =
-mean(log pi * A_hat) + c_v * mean((V - returns)^2) - c_e * mean(entropy), advantages
normalized to zero mean / unit std per batch; gradient global-norm clipped; Adam applied";
P:41 "supports actor-critic algorithms for both discrete and continuous actions"; DESIGN
reading R31 for every point the SPEC leaves open):

* network (R29 policy + a value head on the shared hidden layer, R31):
      h = relu(W1^T o + b1),  logits = W2^T h + b2,  pi = softmax(logits),  V = wv^T h + bv
  packed params  W1 [D][H] | b1 [H] | W2 [H][n] | b2 [n] | wv [H] | bv [1]
  (the prefix W1..b2 is exactly the R29 policy that ws_rollout_policy reads);
* batch = B rows (obs, act, adv, ret); a row whose action is outside [0, n) (R13 invalid
  row, act = -1) contributes nothing; the means divide by the caller's B (the global batch);
* advantage normalisation: A_hat = (A - mu) / sigma with mu, sigma the mean and population
  standard deviation over the batch; if sigma < 1e-8 normalisation is skipped (A_hat = A);
* returns and A_hat are constants (no gradient flows into them);
* clip: g <- g * max_norm / ||g||_2 when ||g||_2 > max_norm;
* Adam (Kingma & Ba 2015, Algorithm 1) at step k >= 1 with bias correction.

Plain fp64 evaluation in the order the definitions are written; the backward pass is the
hand-derived chain rule of the loss above.  Pins (tests/test_oracle_a2c.py): central finite
differences of ``loss``, torch autograd (fp64) of an independently written network,
torch.optim.Adam + clip_grad_norm_, closed forms (uniform policy entropy = log n, zero
advantages and V == returns -> only the entropy term), the SPEC S:404-406 examples; PPO
(R33) against torch autograd of an independent clipped-surrogate loss and the
SPEC identity / clip-rule examples.
"""
from __future__ import annotations

import numpy as np


def n_params(D: int, H: int, n: int) -> int:
    return D * H + H + H * n + n + H + 1


def unpack(params, D: int, H: int, n: int):
    p = np.asarray(params, dtype=np.float64)
    assert p.size == n_params(D, H, n)
    o = 0
    W1 = p[o:o + D * H].reshape(D, H); o += D * H
    b1 = p[o:o + H]; o += H
    W2 = p[o:o + H * n].reshape(H, n); o += H * n
    b2 = p[o:o + n]; o += n
    wv = p[o:o + H]; o += H
    bv = p[o]
    return W1, b1, W2, b2, wv, bv


def forward(params, obs, D: int, H: int, n: int):
    """Per-row network outputs in fp64: z [B,H], h [B,H], logits [B,n], pi [B,n], V [B]."""
    W1, b1, W2, b2, wv, bv = unpack(params, D, H, n)
    o = np.asarray(obs, dtype=np.float64).reshape(-1, D)
    z = o @ W1 + b1
    h = np.maximum(z, 0.0)
    logits = h @ W2 + b2
    m = logits.max(axis=1, keepdims=True)
    e = np.exp(logits - m)
    pi = e / e.sum(axis=1, keepdims=True)
    V = h @ wv + bv
    return z, h, logits, pi, V


def values(params, obs, D: int, H: int, n: int) -> np.ndarray:
    """V(o) for every row of obs (the critic the GAE consumes)."""
    return forward(params, obs, D, H, n)[4]


def moments(x) -> tuple[float, float]:
    """(sum x, sum x^2) in fp64 -- the per-shard part of the normalisation statistics."""
    x = np.asarray(x, dtype=np.float64).ravel()
    return float(x.sum()), float((x * x).sum())


def normalize(adv, total=None, batch=None) -> np.ndarray:
    """A_hat of R31.  total = (sum, sum of squares) over the global batch of `batch` rows
    (defaults: this array)."""
    a = np.asarray(adv, dtype=np.float64).ravel()
    if total is None:
        total = moments(a)
    if batch is None:
        batch = a.size
    mu = total[0] / batch
    var = max(total[1] / batch - mu * mu, 0.0)
    sigma = np.sqrt(var)
    if sigma < 1e-8:
        return a.copy()
    return (a - mu) / sigma


def _valid(act, n):
    a = np.asarray(act).ravel().astype(np.int64)
    return (a >= 0) & (a < n), np.clip(a, 0, n - 1)


def loss(params, obs, act, adv_hat, ret, D, H, n, c_v, c_e, batch=None):
    """(total, policy term, value term, entropy term) of S:405; the means divide by `batch`
    (default: the number of rows)."""
    _, _, logits, pi, V = forward(params, obs, D, H, n)
    ok, a = _valid(act, n)
    B = len(a) if batch is None else batch
    lse = logits.max(axis=1) + np.log(np.exp(logits - logits.max(axis=1, keepdims=True)).sum(axis=1))
    logp = logits[np.arange(len(a)), a] - lse
    ent = -(pi * np.log(np.maximum(pi, 1e-300))).sum(axis=1)
    Ah = np.asarray(adv_hat, dtype=np.float64).ravel()
    R = np.asarray(ret, dtype=np.float64).ravel()
    pol = -(logp * Ah)[ok].sum() / B
    val = c_v * ((V - R) ** 2)[ok].sum() / B
    entt = -c_e * ent[ok].sum() / B
    return pol + val + entt, pol, val, entt


def grad(params, obs, act, adv_hat, ret, D, H, n, c_v, c_e, batch=None) -> np.ndarray:
    """d loss / d params (packed like params), the chain rule written out:
        dL/dlogit_j = (A_hat/B)(pi_j - [j = a]) + (c_e/B) pi_j (log pi_j + Ent)
        dL/dV       = 2 c_v (V - R) / B
        dL/dh_k     = sum_j W2[k][j] dL/dlogit_j + wv_k dL/dV,   dL/dz_k = [z_k > 0] dL/dh_k
        dW1 = o^T dz, db1 = sum dz, dW2 = h^T dlogit, db2 = sum dlogit, dwv = h^T dV, dbv = sum dV
    (Ent = -sum_j pi_j log pi_j; d Ent / d logit_j = -pi_j (log pi_j + Ent))."""
    W1, b1, W2, b2, wv, bv = unpack(params, D, H, n)
    z, h, logits, pi, V = forward(params, obs, D, H, n)
    o = np.asarray(obs, dtype=np.float64).reshape(-1, D)
    ok, a = _valid(act, n)
    B = len(a) if batch is None else batch
    w = ok.astype(np.float64)
    Ah = np.asarray(adv_hat, dtype=np.float64).ravel()
    R = np.asarray(ret, dtype=np.float64).ravel()
    logpi = np.log(np.maximum(pi, 1e-300))
    ent = -(pi * logpi).sum(axis=1)
    onehot = np.zeros_like(pi)
    onehot[np.arange(len(a)), a] = 1.0
    dlog = (Ah / B)[:, None] * (pi - onehot) + (c_e / B) * pi * (logpi + ent[:, None])
    dlog *= w[:, None]
    dV = 2.0 * c_v * (V - R) / B * w
    dh = dlog @ W2.T + dV[:, None] * wv[None, :]
    dz = dh * (z > 0)
    g = np.concatenate([(o.T @ dz).ravel(), dz.sum(axis=0), (h.T @ dlog).ravel(), dlog.sum(axis=0),
                        h.T @ dV, [dV.sum()]])
    return g


def clip(g, max_norm: float) -> np.ndarray:
    g = np.asarray(g, dtype=np.float64)
    norm = np.sqrt((g * g).sum())
    if max_norm > 0 and norm > max_norm:
        return g * (max_norm / norm)
    return g.copy()


def adam(params, g, m, v, k: int, lr: float, beta1: float = 0.9, beta2: float = 0.999,
         eps: float = 1e-8):
    """One Adam step (k >= 1): returns (params', m', v')."""
    p = np.asarray(params, dtype=np.float64)
    g = np.asarray(g, dtype=np.float64)
    m = beta1 * np.asarray(m, dtype=np.float64) + (1 - beta1) * g
    v = beta2 * np.asarray(v, dtype=np.float64) + (1 - beta2) * g * g
    mhat = m / (1 - beta1 ** k)
    vhat = v / (1 - beta2 ** k)
    return p - lr * mhat / (np.sqrt(vhat) + eps), m, v


def update(params, m, v, k, obs, act, adv, ret, D, H, n, *, c_v=0.5, c_e=0.01, lr=1e-3,
           max_norm=0.5, beta1=0.9, beta2=0.999, eps=1e-8):
    """a2c_update: normalise -> gradient -> clip -> Adam.  Returns
    (params', m', v', gradient before clipping, loss terms before the step)."""
    Ah = normalize(adv)
    g = grad(params, obs, act, Ah, ret, D, H, n, c_v, c_e)
    L = loss(params, obs, act, Ah, ret, D, H, n, c_v, c_e)
    p2, m2, v2 = adam(params, clip(g, max_norm), m, v, k, lr, beta1, beta2, eps)
    return p2, m2, v2, g, L


# ------------------------------------------------------------------------------ PPO (R33)
# SPEC ppo_update: "K epochs x M minibatches of the clipped surrogate
# mean(min(rho A_hat, clip(rho, 1 +- eps) A_hat)) with rho = exp(log pi_new - log pi_old);
# value and entropy terms as in A2C".  Reading R33: the loss minimised is
#   -mean(min(rho A_hat, clip(rho, 1-eps, 1+eps) A_hat)) + c_v mean((V-R)^2) - c_e mean(Ent)
# with log pi_old the behaviour log-probabilities logged by the roll-out (constants).

def ppo_loss(params, obs, act, adv_hat, ret, logp_old, D, H, n, c_v, c_e, eps, batch=None):
    """(total, surrogate term, value term, entropy term)."""
    _, _, logits, pi, V = forward(params, obs, D, H, n)
    ok, a = _valid(act, n)
    B = len(a) if batch is None else batch
    lse = logits.max(axis=1) + np.log(np.exp(logits - logits.max(axis=1, keepdims=True)).sum(axis=1))
    logp = logits[np.arange(len(a)), a] - lse
    rho = np.exp(logp - np.asarray(logp_old, dtype=np.float64).ravel())
    Ah = np.asarray(adv_hat, dtype=np.float64).ravel()
    surr = np.minimum(rho * Ah, np.clip(rho, 1 - eps, 1 + eps) * Ah)
    ent = -(pi * np.log(np.maximum(pi, 1e-300))).sum(axis=1)
    R = np.asarray(ret, dtype=np.float64).ravel()
    pol = -surr[ok].sum() / B
    val = c_v * ((V - R) ** 2)[ok].sum() / B
    entt = -c_e * ent[ok].sum() / B
    return pol + val + entt, pol, val, entt


def ppo_grad(params, obs, act, adv_hat, ret, logp_old, D, H, n, c_v, c_e, eps, batch=None) -> np.ndarray:
    """d ppo_loss / d params: the A2C chain rule with A_hat replaced by rho A_hat on rows
    where the unclipped term is the minimum (rho A_hat <= clip(rho) A_hat), 0 elsewhere."""
    _, _, logits, pi, _ = forward(params, obs, D, H, n)
    ok, a = _valid(act, n)
    lse = logits.max(axis=1) + np.log(np.exp(logits - logits.max(axis=1, keepdims=True)).sum(axis=1))
    logp = logits[np.arange(len(a)), a] - lse
    rho = np.exp(logp - np.asarray(logp_old, dtype=np.float64).ravel())
    Ah = np.asarray(adv_hat, dtype=np.float64).ravel()
    active = rho * Ah <= np.clip(rho, 1 - eps, 1 + eps) * Ah
    return grad(params, obs, act, np.where(active, rho * Ah, 0.0), ret, D, H, n, c_v, c_e, batch)


# ------------------------------------------------------------------------------ Gaussian (R35)
# Continuous actions ("both discrete and continuous actions"): the R34 Gaussian policy
# with the R31 value head.  Packed params  W1 [D][H] | b1 [H] | W2 [H][d] | b2 [d] |
# log_std [d] | wv [H] | bv.  log pi(a|o) = sum_k -(a_k - mu_k)^2 / (2 sigma_k^2) - log sigma_k
# - log(2 pi)/2, entropy = sum_k log sigma_k + log(2 pi e)/2 (state independent); the loss
# is R31's with these.

def n_params_gauss(D: int, H: int, d: int) -> int:
    return D * H + H + H * d + d + d + H + 1


def unpack_gauss(params, D: int, H: int, d: int):
    p = np.asarray(params, dtype=np.float64)
    assert p.size == n_params_gauss(D, H, d)
    o = 0
    W1 = p[o:o + D * H].reshape(D, H); o += D * H
    b1 = p[o:o + H]; o += H
    W2 = p[o:o + H * d].reshape(H, d); o += H * d
    b2 = p[o:o + d]; o += d
    log_std = p[o:o + d]; o += d
    wv = p[o:o + H]; o += H
    return W1, b1, W2, b2, log_std, wv, p[o]


def forward_gauss(params, obs, D, H, d):
    W1, b1, W2, b2, log_std, wv, bv = unpack_gauss(params, D, H, d)
    o = np.asarray(obs, dtype=np.float64).reshape(-1, D)
    z = o @ W1 + b1
    h = np.maximum(z, 0.0)
    return z, h, h @ W2 + b2, log_std, h @ wv + bv


def loss_gauss(params, obs, act, adv_hat, ret, D, H, d, c_v, c_e, batch=None):
    _, _, mu, log_std, V = forward_gauss(params, obs, D, H, d)
    a = np.asarray(act, dtype=np.float64).reshape(-1, d)
    ok = np.isfinite(a).all(axis=1)
    a = np.where(np.isfinite(a), a, 0.0)
    B = len(a) if batch is None else batch
    sig2 = np.exp(2 * log_std)
    logp = (-(a - mu) ** 2 / (2 * sig2) - log_std - 0.5 * np.log(2 * np.pi)).sum(axis=1)
    ent = (log_std + 0.5 * np.log(2 * np.pi * np.e)).sum()
    Ah = np.asarray(adv_hat, dtype=np.float64).ravel()
    R = np.asarray(ret, dtype=np.float64).ravel()
    pol = -(logp * Ah)[ok].sum() / B
    val = c_v * ((V - R) ** 2)[ok].sum() / B
    entt = -c_e * ent * ok.sum() / B
    return pol + val + entt, pol, val, entt


def grad_gauss(params, obs, act, adv_hat, ret, D, H, d, c_v, c_e, batch=None) -> np.ndarray:
    """Chain rule: dL/dmu_k = -(A_hat/B)(a_k - mu_k)/sigma_k^2;
    dL/dlog_sigma_k = sum_rows -(A_hat/B)((a_k - mu_k)^2/sigma_k^2 - 1) - c_e n_valid / B;
    the rest as in `grad` with dL/dlogit replaced by dL/dmu.  Rows with a non-finite action
    contribute nothing."""
    W1, b1, W2, b2, log_std, wv, bv = unpack_gauss(params, D, H, d)
    z, h, mu, _, V = forward_gauss(params, obs, D, H, d)
    o = np.asarray(obs, dtype=np.float64).reshape(-1, D)
    a = np.asarray(act, dtype=np.float64).reshape(-1, d)
    ok = np.isfinite(a).all(axis=1)
    a = np.where(np.isfinite(a), a, 0.0)
    w = ok.astype(np.float64)
    B = len(a) if batch is None else batch
    Ah = np.asarray(adv_hat, dtype=np.float64).ravel()
    R = np.asarray(ret, dtype=np.float64).ravel()
    sig2 = np.exp(2 * log_std)
    dmu = -(Ah / B)[:, None] * (a - mu) / sig2 * w[:, None]
    dls = (-(Ah / B)[:, None] * ((a - mu) ** 2 / sig2 - 1.0) * w[:, None]).sum(axis=0) - c_e * w.sum() / B
    dV = 2.0 * c_v * (V - R) / B * w
    dz = (dmu @ W2.T + dV[:, None] * wv[None, :]) * (z > 0)
    return np.concatenate([(o.T @ dz).ravel(), dz.sum(axis=0), (h.T @ dmu).ravel(), dmu.sum(axis=0), dls,
                           h.T @ dV, [dV.sum()]])
