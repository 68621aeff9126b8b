"""Counter-based synthetic KV generator (oracle's own implementation).
TEST INFRASTRUCTURE ONLY.

Defines the KV values that ``mirage_fill_kv`` writes (include/mirage.h). The
CUDA fill kernel implements the same function independently; the two share no
code. For element (seq, layer, kv_head, kv, pos, d) of a model with L layers,
H_kv kv heads and head dim D:
    idx = ((((seq * L + layer) * H_kv + kv_head) * 2 + kv) * 2^20 + pos) * D + d
    h   = splitmix64(idx XOR (seed * 0x9E3779B97F4A7C15))      (all mod 2^64)
    u   = (h >> 40) * 2^-24                                       in [0, 1)
    x   = fp32(2u - 1) * fp32(1.7320508)   for K   (unit variance)
        = fp32(2u - 1)                     for V   (bf16 may round to +1.0)
    value = bf16_rne(x)
"""
import numpy as np

M64 = (1 << 64) - 1
GOLD = 0x9E3779B97F4A7C15


def splitmix64(x):
    x = np.asarray(x, dtype=np.uint64)
    with np.errstate(over="ignore"):
        x = x + np.uint64(GOLD)
        x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        x = x ^ (x >> np.uint64(31))
    return x


def _bf16_rne_f32(x32):
    b = np.asarray(x32, dtype=np.float32).view(np.uint32).astype(np.uint64)
    b = (b + np.uint64(0x7FFF) + ((b >> np.uint64(16)) & np.uint64(1))) >> np.uint64(16)
    return (b << np.uint64(16)).astype(np.uint32).view(np.float32).astype(np.float64)


def kv_values(seed, seq, n_layers, n_kv_heads, head_dim, layer, kv_head, kv, positions):
    """Values [len(positions), D] (fp64 holding bf16 values)."""
    pos = np.asarray(positions, dtype=np.uint64)[:, None]
    d = np.arange(head_dim, dtype=np.uint64)[None, :]
    base = (((seq * n_layers + layer) * n_kv_heads + kv_head) * 2 + kv)
    with np.errstate(over="ignore"):
        idx = (np.uint64(base) * np.uint64(1 << 20) + pos) * np.uint64(head_dim) + d
        key = np.uint64((seed * GOLD) & M64)
    h = splitmix64(idx ^ key)
    u = (h >> np.uint64(40)).astype(np.float32) * np.float32(2.0 ** -24)
    x = np.float32(2.0) * u - np.float32(1.0)
    if kv == 0:
        x = x * np.float32(1.7320508)
    return _bf16_rne_f32(x)
