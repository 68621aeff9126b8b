"""End-to-end decode tolerances DERIVED from bf16 rounding (reading #19).

The paper fixes no arithmetic precision; the exact result of a decode step is
the fp64 decoder (oracle c4, ``round_points=False``), pinned to HF transformers
(tests/test_oracle_decode.py). An implementation that stores bf16 at some of the
materialisation points SURVEY.md §8(c) c4 lists differs from it by propagated
rounding error. The CUDA path stores bf16 at the normalised GEMM inputs, the
K/V cache, the attention output, the FFN activation and the final hidden
(reading #25); ``predict`` models exactly those points by default
(``points="survey"`` models every SURVEY point, an all-bf16 implementation).
Under the first-order model every such point multiplies its
value by (1 + delta), delta independent with RMS <= sigma = 2^-8 / sqrt(3) (the
RMS of a relative error uniform on [-u, u], u = 2^-8 the bf16 unit roundoff, an
upper bound on round-to-nearest's RMS relative error). ``predict`` runs the
exact decoder and a few draws of that noise model (oracle c4 ``noise=``) over the
same token script; the bound on the implementation's error is then

    rel-RMS(got - exact)  <=  K_REL * sqrt(mean over draws of rel-RMS(draw - exact)^2)
    max |got - exact|     <=  K_MAX * max over draws of max |draw - exact|

K_REL = 3 covers the draw-to-draw spread of a rel-RMS over d >= 256 elements
(its relative standard deviation is ~ 1/sqrt(d)); K_MAX = 2 covers the tail of a
maximum over d elements estimated from a few draws. fp32 accumulation
(relative 2^-24 * sqrt(K)) and the attention kernel's hi/lo bf16 q and p
(relative 2^-16) are three orders of magnitude below sigma and are not modelled.

Argmax (``argmax_decidable``): the LM head computes logits_j = E_j . x from the
bf16 final hidden x it also returns. With delta = x_gpu - x_exact,
|logit_gpu_j - logit_exact_j| <= ||E_j||_2 ||delta||_2 + gamma_d sum_i |E_ji x_gpu_i|
(Cauchy-Schwarz plus the fp32 dot-product error bound, gamma_d = d u32 / (1 - d u32),
u32 = 2^-24), so the GPU's argmax must equal the exact argmax wherever the exact
top-2 margin exceeds twice that bound. Rows below it are not decidable and are
skipped.
"""
import numpy as np

from oracle.decode import Decoder

SIGMA = 2.0 ** -8 / np.sqrt(3.0)
K_REL, K_MAX = 3.0, 2.0


def rel_rms(a, b):
    return float(np.sqrt(((a - b) ** 2).mean() / (b ** 2).mean()))


def predict(shape, layers, glob, script, draws=4, seed=0, points="product"):
    """script(dec) -> list of (hidden [rows, d], logits [rows, V]) per step.
    Returns (exact steps, [(rel bound, max-abs bound)] per step)."""
    exact = script(Decoder(shape, layers, glob, round_points=False))
    noisy = [script(Decoder(shape, layers, glob,
                            noise=(SIGMA, np.random.default_rng(seed * 1000 + k), points)))
             for k in range(draws)]
    bounds = []
    for t, (hx, _) in enumerate(exact):
        if hx is None:             # a step whose hidden state the script does not report
            bounds.append(None)
            continue
        rel = np.sqrt(np.mean([rel_rms(n[t][0], hx) ** 2 for n in noisy]))
        mx = max(float(np.abs(n[t][0] - hx).max()) for n in noisy)
        bounds.append((K_REL * rel, K_MAX * mx))
    return exact, bounds


def check(got, exact_hidden, bound, what=""):
    rel = rel_rms(got, exact_hidden)
    mx = float(np.abs(got - exact_hidden).max())
    assert rel <= bound[0] and mx <= bound[1], (what, rel, bound[0], mx, bound[1])
    return rel, mx


def lm_head(shape, glob):
    from synth import models
    E = glob["embed"] if shape.family == models.OPT else glob["lm_head"]
    return E.double().numpy() if hasattr(E, "double") else np.asarray(E, np.float64)


def argmax_decidable(E, x_gpu, x_exact, logits_exact):
    """Per row: True where the exact top-2 margin exceeds twice the logit error bound."""
    d = E.shape[1]
    u32 = 2.0 ** -24
    gamma = d * u32 / (1 - d * u32)
    row_norm = np.sqrt((E * E).sum(1)).max()
    absE = np.abs(E)
    out = []
    for xg, xe, lg in zip(np.atleast_2d(x_gpu), np.atleast_2d(x_exact), np.atleast_2d(logits_exact)):
        bound = row_norm * np.sqrt(((xg - xe) ** 2).sum()) + gamma * float((absE @ np.abs(xg)).max())
        s = np.sort(lg)
        out.append(bool(s[-1] - s[-2] > 2 * bound))
    return out
