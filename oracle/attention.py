"""c3 — paged-attention decode over block tables (oracle). TEST INFRASTRUCTURE ONLY.

What it computes is the plain definition of single-query softmax attention
(the decode step of PagedAttention, §2.2; north_star "QK^T, online
softmax, PV"): for sequence s and query head h with KV head h' = floor(h/g),
g = H / H_kv (reading #17):
    s_j = scale * <q, K_j>,  j < L_s,   scale = 1/sqrt(D)   (reading #16)
    p   = softmax(s),        o = sum_j p_j V_j.
K_j / V_j are found through the block table: block T[s][j // 16], row j % 16
(reading #11). The pool maps a block id to its [L][H_kv][2][16][D] tile; whether
that id lives in the native pool or in a reclaimed parameter region does not
enter the arithmetic (remapping moves memory, not math: PAPER.md:88-91, :874).
fp64 throughout.

Pins (tests/test_oracle_attention.py): dense twin vs torch SDPA in float64;
L=1 -> o = v_0; equal keys -> mean(V); a dominant logit -> that row of V;
identical q heads in a group -> identical outputs.
"""
import numpy as np

BLOCK_TOKENS = 16


def gather_kv(pool, table, length, layer, kv_head):
    """Logical K, V [L_s, D] of one (sequence, kv head) gathered via the table."""
    rows_k, rows_v = [], []
    for j in range(length):
        tile = pool[table[j // BLOCK_TOKENS]]
        rows_k.append(tile[layer, kv_head, 0, j % BLOCK_TOKENS])
        rows_v.append(tile[layer, kv_head, 1, j % BLOCK_TOKENS])
    return np.array(rows_k, dtype=np.float64), np.array(rows_v, dtype=np.float64)


def attend(q, K, V):
    """o = softmax(q K^T / sqrt(D)) V for one query vector (fp64)."""
    D = q.shape[-1]
    s = (K @ q) * (1.0 / np.sqrt(D))
    p = np.exp(s - s.max())
    return (p @ V) / p.sum()


def paged_attention(q, pool, tables, lengths, layer):
    """q [B, H, D]; pool {block_id: array [L, H_kv, 2, 16, D]}; tables [B][...];
    lengths [B]. Returns o [B, H, D] fp64."""
    q = np.asarray(q, dtype=np.float64)
    B, H, D = q.shape
    H_kv = next(iter(pool.values())).shape[1] if pool else H
    g = H // H_kv
    out = np.zeros((B, H, D))
    for b in range(B):
        for hk in range(H_kv):
            K, V = gather_kv(pool, tables[b], lengths[b], layer, hk)
            for h in range(hk * g, (hk + 1) * g):
                out[b, h] = attend(q[b, h], K, V)
    return out


def dense_attention(q, K, V):
    """Dense twin: q [B,H,D], K/V lists of [H_kv, L_b, D] per sequence."""
    q = np.asarray(q, dtype=np.float64)
    B, H, D = q.shape
    out = np.zeros((B, H, D))
    for b in range(B):
        H_kv = K[b].shape[0]
        g = H // H_kv
        for h in range(H):
            out[b, h] = attend(q[b, h], np.asarray(K[b][h // g], np.float64),
                               np.asarray(V[b][h // g], np.float64))
    return out
