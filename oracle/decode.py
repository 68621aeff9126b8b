"""c4 — one decode step of an OPT- or Llama-shaped decoder (oracle).
TEST INFRASTRUCTURE ONLY.

The paper treats the decoder as standard (PAPER.md:100 fn., :131-138 §2.1: the
decode phase generates one token per step reusing the KV cache) and MIRAGE
"requires no changes to CUDA kernels": the remap changes where
weights/KV live, never the arithmetic. This module therefore writes out the
public decoder definitions (HF OPT with pre-LN, ReLU, learned positions with
offset 2, tied LM head; HF Llama with RMSNorm, rotate-half RoPE, SiLU-gated MLP,
untied LM head) in fp64, one token per sequence, over a logical per-sequence KV
cache. Attention uses oracle.attention.attend (c3's definition).

The paper fixes no arithmetic precision (it runs vLLM's bf16 models unchanged,
PAPER.md:635, :874), so the AUTHORITATIVE result is the exact decoder
(``round_points=False``, fp64, pinned to HF transformers). Two bf16 models of an
implementation sit beside it:

* ``round_points=True`` rounds to bf16 where the CUDA path stores bf16 (the
  normalised GEMM inputs x, the K/V written to the cache, the attention output
  and the FFN activation; reading #25). A diagnostic twin only: its
  choice of points is not pinned by the paper.
* ``noise=(sigma, rng, points)`` is the first-order bf16 rounding-noise model
  used to DERIVE the end-to-end tolerance (reading #19): at each
  materialisation point, x -> x * (1 + sigma * xi) with xi ~ U(-sqrt 3, sqrt 3)
  i.i.d. (unit variance). With sigma = 2^-8 / sqrt 3 -- the RMS of a relative
  error uniform on [-u, u], u = 2^-8 the bf16 unit roundoff, an upper bound on
  the RMS of round-to-nearest's relative error -- the spread of the outputs over
  a few draws predicts how far an implementation storing bf16 at those points
  sits from the exact decoder. ``points="product"``: the points above (where the
  CUDA path stores bf16); ``points="survey"``: every point SURVEY.md §8(c) c4
  lists (also the embedding sum, qkv, O-projection and FC outputs and the
  residual sums: an all-bf16 implementation such as vLLM's).

Pins (tests/test_oracle_decode.py): token-by-token decode equals a one-shot
causal forward of the HF transformers reference models in float64 on the same
weights (round_points=False), for both families.
"""
import numpy as np

from .attention import attend
from .bf16 import round_bf16

OPT, LLAMA = 0, 1
OPT_POS_OFFSET = 2


def _np(t):
    return t.double().numpy() if hasattr(t, "double") else np.asarray(t, np.float64)


class Decoder:
    def __init__(self, shape, layers, glob, round_points=True, noise=None):
        """shape: synth.models.ModelShape; layers: list of dicts of tensors;
        glob: dict of non-layer tensors (names as synth.weights specs);
        noise: None or (sigma, numpy Generator, "product" | "survey") -- the
        rounding-noise model (implies round_points=False)."""
        self.m = shape
        self.L = [{k: _np(v) for k, v in lw.items()} for lw in layers]
        self.G = {k: _np(v) for k, v in glob.items()}
        self.rp = round_points and noise is None
        self.noise = noise
        self.kv = {}          # seq -> list over layers of (K [H_kv, T, D], V [H_kv, T, D])

    def _perturb(self, x):
        sigma, rng, _ = self.noise
        return x * (1.0 + sigma * rng.uniform(-np.sqrt(3.0), np.sqrt(3.0), np.shape(x)))

    def _s(self, x):
        """A SURVEY §8(c) c4 point where the product keeps fp32: perturbed only
        under the noise model with points="survey"."""
        if self.noise is None or self.noise[2] != "survey":
            return x
        return self._perturb(x)

    def _r(self, x):
        """A point where the product stores bf16 (also a SURVEY point)."""
        if self.noise is not None:
            return self._perturb(x)
        return round_bf16(x) if self.rp else x

    # --- cache -------------------------------------------------------------
    def cache_len(self, seq):
        return self.kv[seq][0][0].shape[1] if seq in self.kv else 0

    def set_kv(self, seq, per_layer):
        """per_layer: list over layers of (K [H_kv,T,D], V [H_kv,T,D]) bf16 values."""
        self.kv[seq] = [(np.asarray(k, np.float64).copy(), np.asarray(v, np.float64).copy())
                        for k, v in per_layer]

    def _append(self, seq, layer, k, v):
        m = self.m
        if seq not in self.kv:
            z = np.zeros((m.n_kv_heads, 0, m.head_dim))
            self.kv[seq] = [(z, z) for _ in range(m.n_layers)]
        K, V = self.kv[seq][layer]
        self.kv[seq][layer] = (np.concatenate([K, k[:, None]], 1), np.concatenate([V, v[:, None]], 1))

    # --- pieces ------------------------------------------------------------
    def _layernorm(self, h, g, b):
        mu = h.mean()
        var = ((h - mu) ** 2).mean()
        return (h - mu) / np.sqrt(var + self.m.norm_eps) * g + b

    def _rmsnorm(self, h, g):
        return h / np.sqrt((h * h).mean() + self.m.norm_eps) * g

    def _rope(self, x, pos):
        """rotate-half RoPE on [heads, D]; inv_freq_i = theta^(-2i/D)."""
        D = x.shape[-1]
        i = np.arange(D // 2, dtype=np.float64)
        ang = pos * self.m.rope_theta ** (-2.0 * i / D)
        c, s = np.cos(ang), np.sin(ang)
        x1, x2 = x[:, : D // 2], x[:, D // 2:]
        return np.concatenate([x1 * c - x2 * s, x2 * c + x1 * s], axis=-1)

    # --- one token -----------------------------------------------------------
    def step_one(self, seq, token, pos):
        """Run one token of `seq` at position `pos` (== cached length). Returns
        (final normalised hidden [d], logits [vocab])."""
        m = self.m
        assert pos == self.cache_len(seq), (pos, self.cache_len(seq))
        H, Hk, D = m.n_heads, m.n_kv_heads, m.head_dim
        g = H // Hk
        if m.family == OPT:
            h = self._s(self.G["embed"][token] + self.G["pos_embed"][pos + OPT_POS_OFFSET])
        else:
            h = self.G["embed"][token].copy()
        for li, W in enumerate(self.L):
            x = self._r(self._layernorm(h, W["ln1_g"], W["ln1_b"]) if m.family == OPT
                        else self._rmsnorm(h, W["rms1_g"]))
            qkv = W["w_qkv"] @ x
            if m.family == OPT:
                qkv = qkv + W["b_qkv"]
            qkv = self._s(qkv)
            q = qkv[: H * D].reshape(H, D)
            k = qkv[H * D: (H + Hk) * D].reshape(Hk, D)
            v = qkv[(H + Hk) * D:].reshape(Hk, D)
            if m.family == LLAMA:
                q, k = self._rope(q, pos), self._rope(k, pos)
            self._append(seq, li, self._r(k), self._r(v))
            K, V = self.kv[seq][li]
            a = np.concatenate([attend(q[hh], K[hh // g], V[hh // g]) for hh in range(H)])
            a = self._r(a)
            o = W["w_o"] @ a
            if m.family == OPT:
                o = o + W["b_o"]
            h = self._s(h + self._s(o))
            if m.family == OPT:
                x = self._r(self._layernorm(h, W["ln2_g"], W["ln2_b"]))
                f = self._r(np.maximum(self._s(W["w_fc1"] @ x + W["b_fc1"]), 0.0))
                h = self._s(h + self._s(W["w_fc2"] @ f + W["b_fc2"]))
            else:
                x = self._r(self._rmsnorm(h, W["rms2_g"]))
                gu = self._s(W["w_gateup"] @ x)
                gate, up = gu[: m.ffn_dim], gu[m.ffn_dim:]
                f = self._r(gate / (1.0 + np.exp(-gate)) * up)
                h = self._s(h + self._s(W["w_down"] @ f))
        if m.family == OPT:
            xf = self._r(self._layernorm(h, self.G["lnf_g"], self.G["lnf_b"]))
            logits = self.G["embed"] @ xf
        else:
            xf = self._r(self._rmsnorm(h, self.G["normf_g"]))
            logits = self.G["lm_head"] @ xf
        return xf, logits

    def step(self, seqs, tokens, positions):
        """Batch decode step; returns (hidden [B,d], logits [B,V], argmax [B]).
        argmax takes the lowest index on ties."""
        hs, ls = [], []
        for s, t, p in zip(seqs, tokens, positions):
            x, lg = self.step_one(int(s), int(t), int(p))
            hs.append(x)
            ls.append(lg)
        ls = np.array(ls)
        return np.array(hs), ls, np.argmax(ls, axis=1)
