"""Pins for oracle c3 (paged attention): library routine (torch SDPA, float64),
closed forms and special cases. CPU only."""
import numpy as np
import pytest
import torch

from oracle import attention as OA
from oracle import kvgen


def make_pool(rng, B, lens, L, Hk, D, shuffle=True):
    """Build a pool with a random physical placement; return pool, tables, K, V."""
    n_blocks = [(l + 15) // 16 for l in lens]
    ids = list(range(sum(n_blocks) + 5))
    if shuffle:
        rng.shuffle(ids)
    pool, tables, Ks, Vs = {}, [], [], []
    it = iter(ids)
    for b, l in enumerate(lens):
        t = [next(it) for _ in range(n_blocks[b])]
        tables.append(t)
        K = rng.standard_normal((L, Hk, l, D))
        V = rng.uniform(-1, 1, (L, Hk, l, D))
        Ks.append(K)
        Vs.append(V)
        for j, bid in enumerate(t):
            tile = np.zeros((L, Hk, 2, 16, D))
            seg = slice(j * 16, min(l, (j + 1) * 16))
            n = seg.stop - seg.start
            tile[:, :, 0, :n] = K[:, :, seg]
            tile[:, :, 1, :n] = V[:, :, seg]
            pool[bid] = tile
    return pool, tables, Ks, Vs


@pytest.mark.parametrize("H,Hk,D", [(4, 4, 64), (8, 2, 128), (8, 1, 32)])
def test_vs_torch_sdpa(H, Hk, D):
    rng = np.random.default_rng(0)
    lens = [1, 15, 16, 17, 40]
    L = 2
    pool, tables, Ks, Vs = make_pool(rng, len(lens), lens, L, Hk, D)
    q = rng.standard_normal((len(lens), H, D))
    for layer in range(L):
        o = OA.paged_attention(q, pool, tables, lens, layer)
        for b, l in enumerate(lens):
            qt = torch.from_numpy(q[b])[:, None, :]                       # [H,1,D]
            k = torch.from_numpy(Ks[b][layer]).repeat_interleave(H // Hk, 0)  # [H,l,D]
            v = torch.from_numpy(Vs[b][layer]).repeat_interleave(H // Hk, 0)
            ref = torch.nn.functional.scaled_dot_product_attention(qt, k, v)[:, 0]
            np.testing.assert_allclose(o[b], ref.numpy(), atol=1e-12, rtol=1e-12)


def test_placement_does_not_change_result():
    rng = np.random.default_rng(3)
    lens = [33, 70]
    pool, tables, _, _ = make_pool(np.random.default_rng(5), 2, lens, 1, 2, 16, shuffle=False)
    q = rng.standard_normal((2, 2, 16))
    o1 = OA.paged_attention(q, pool, tables, lens, 0)
    perm = {bid: 1000 + i for i, bid in enumerate(sorted(pool, reverse=True))}
    pool2 = {perm[k]: v for k, v in pool.items()}
    tables2 = [[perm[i] for i in t] for t in tables]
    o2 = OA.paged_attention(q, pool2, tables2, lens, 0)
    assert np.array_equal(o1, o2)


def test_special_cases():
    rng = np.random.default_rng(1)
    D = 8
    V = rng.uniform(-1, 1, (5, D))
    # L = 1 -> o = v_0
    assert np.allclose(OA.attend(rng.standard_normal(D), rng.standard_normal((1, D)), V[:1]), V[0])
    # equal keys or q = 0 -> uniform softmax -> mean(V)
    K = np.tile(rng.standard_normal(D), (5, 1))
    assert np.allclose(OA.attend(rng.standard_normal(D), K, V), V.mean(0))
    assert np.allclose(OA.attend(np.zeros(D), rng.standard_normal((5, D)), V), V.mean(0))
    # dominant logit -> that row
    K = np.zeros((5, D))
    K[3, 0] = 1.0
    q = np.zeros(D)
    q[0] = 200.0 * np.sqrt(D)
    assert np.allclose(OA.attend(q, K, V), V[3], atol=1e-12)


def test_gqa_identical_heads():
    rng = np.random.default_rng(2)
    pool, tables, _, _ = make_pool(rng, 1, [50], 1, 2, 16)
    q = rng.standard_normal((1, 8, 16))
    q[0, 1:4] = q[0, 0]
    o = OA.paged_attention(q, pool, tables, [50], 0)
    assert np.array_equal(o[0, 0], o[0, 3])


def test_kvgen_splitmix_reference_vector():
    # splitmix64 from state 0: first output 0xE220A8397B1DCDAF, second 0x6E789E6AA1B965F4
    assert int(kvgen.splitmix64(np.uint64(0))) == 0xE220A8397B1DCDAF
    assert int(kvgen.splitmix64(np.uint64(0x9E3779B97F4A7C15))) == 0x6E789E6AA1B965F4


def test_kvgen_distribution_and_bf16():
    k = kvgen.kv_values(1, 3, 2, 4, 128, 1, 2, 0, range(512))
    v = kvgen.kv_values(1, 3, 2, 4, 128, 1, 2, 1, range(512))
    assert abs(k.mean()) < 0.05 and abs(k.var() - 1.0) < 0.05
    assert v.min() >= -1 and v.max() <= 1   # bf16 rounding may reach 1.0
    for x in (k, v):   # exactly bf16-representable
        b = x.astype(np.float32).view(np.uint32)
        assert np.all(b & 0xFFFF == 0)
    assert not np.array_equal(k, kvgen.kv_values(2, 3, 2, 4, 128, 1, 2, 0, range(512)))


def test_bf16_rounding_matches_torch():
    """oracle.bf16.round_bf16 (round-half-even on 8 significant bits) vs torch's
    fp32 -> bfloat16 conversion (library routine), including exact ties."""
    from oracle.bf16 import round_bf16
    rng = np.random.default_rng(0)
    x = np.concatenate([rng.standard_normal(20000) * 10 ** rng.uniform(-3, 3, 20000),
                        np.array([1 + 2 ** -8, 1 + 3 * 2 ** -8, -(1 + 2 ** -8), 2 ** -7 * 1.5, 0.0])])
    x32 = x.astype(np.float32)
    ref = torch.from_numpy(x32).to(torch.bfloat16).double().numpy()
    np.testing.assert_array_equal(round_bf16(x32.astype(np.float64)), ref)
