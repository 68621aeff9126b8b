"""Head-sharded tensor parallelism: the per-rank shards
the harness builds recombine into the full layer -- the O-projection and the
down-projection are sums of rank partials, which is exactly what the decode
step's ncclAllReduce computes. CPU only (one GPU per box: the NCCL path itself
is exercised on one rank in tests/test_gpu_tp.py)."""
import numpy as np
import pytest

import harness
from synth import models, weights


@pytest.mark.parametrize("tp", [2, 4])
def test_shards_recombine_to_full_layer(tp):
    shape = models.ModelShape("tp-toy", models.LLAMA, 1, 256, 8, 4, 32, 512, 64, 128)
    t = {k: v.double() for k, v in weights.layer_tensors(shape, 0, seed=3).items()}
    rng = np.random.default_rng(0)
    x = rng.standard_normal(shape.d_model)
    H, Hk, D, f = shape.n_heads, shape.n_kv_heads, shape.head_dim, shape.ffn_dim
    a = rng.standard_normal(H * D)          # attention output, all heads
    full_o = t["w_o"].numpy() @ a
    gu = t["w_gateup"].numpy() @ x
    act = gu[:f] / (1 + np.exp(-gu[:f])) * gu[f:]
    full_down = t["w_down"].numpy() @ act
    qkv = t["w_qkv"].numpy() @ x
    o_sum = np.zeros(shape.d_model)
    d_sum = np.zeros(shape.d_model)
    h, hk, fs = H // tp, Hk // tp, f // tp
    for r in range(tp):
        sh = {k: v.numpy() for k, v in harness.shard_layer(shape, t, r, tp).items()}
        o_sum += sh["w_o"] @ a[r * h * D:(r + 1) * h * D]
        g = sh["w_gateup"] @ x
        d_sum += sh["w_down"] @ (g[:fs] / (1 + np.exp(-g[:fs])) * g[fs:])
        q_r = sh["w_qkv"] @ x
        np.testing.assert_allclose(q_r[:h * D], qkv[r * h * D:(r + 1) * h * D], rtol=1e-12, atol=1e-12)
        np.testing.assert_allclose(q_r[h * D:(h + hk) * D], qkv[H * D + r * hk * D:H * D + (r + 1) * hk * D],
                                   rtol=1e-12, atol=1e-12)
        # a rank's q heads h_r * g .. map onto its own kv heads under kv = q // g
        assert (r * h) // (H // Hk) == r * hk
    np.testing.assert_allclose(o_sum, full_o, rtol=1e-10, atol=1e-10)
    np.testing.assert_allclose(d_sum, full_down, rtol=1e-10, atol=1e-10)


def test_shard_sizes_match_library():
    from paper_2507_11507_b200 import _lib
    m = models.LLAMA_70B
    for tp in (1, 2, 4, 8):
        S, G, BB = _lib.model_sizes(harness.shard_shape(m, tp))
        assert BB == m.n_layers * (m.n_kv_heads // tp) * 2 * 16 * 128 * 2
        assert S * tp == weights.layer_bytes(m) + (tp - 1) * 2 * 2 * m.d_model  # norms replicated
