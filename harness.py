"""Glue used by tests, bench.py and __graft_entry__: builds libmirage contexts
and models from the seeded synthetic inputs in ``synth``. No method arithmetic
(that lives in libmirage's kernels); no oracle imports."""
import torch

from paper_2507_11507_b200 import _lib
from synth import weights


def layer_bytes_tensor(shape, layer, seed, model_idx, device="cpu"):
    t = weights.layer_tensors(shape, layer, seed, model_idx, device)
    return _lib.tensors_to_bytes(t, [n for n, _, _ in weights.layer_spec(shape)])


def global_bytes_tensor(shape, seed, model_idx, device="cpu"):
    t = weights.global_tensors(shape, seed, model_idx, device)
    return _lib.tensors_to_bytes(t, [n for n, _, _ in weights.global_spec(shape)])


def make_blob(shape, seed=0, model_idx=0, gen_device="cpu"):
    """Pinned host blob in the include/mirage.h layout. For large shapes pass
    gen_device='cuda' (values then come from torch's CUDA generator)."""
    S, G, _ = _lib.model_sizes(shape)
    blob = torch.empty(shape.n_layers * S + G, dtype=torch.uint8, pin_memory=True)
    for l in range(shape.n_layers):
        blob[l * S:(l + 1) * S].copy_(layer_bytes_tensor(shape, l, seed, model_idx, gen_device))
    blob[shape.n_layers * S:].copy_(global_bytes_tensor(shape, seed, model_idx, gen_device))
    return blob


def arena_for(shapes_and_pools, max_batch, max_ctx, slack=64 << 20):
    return sum(_lib.model_arena_bytes(s, n, max_batch, max_ctx) for s, n in shapes_and_pools) + slack


def blocks_for(tokens):
    return (tokens + _lib.BLOCK_TOKENS - 1) // _lib.BLOCK_TOKENS


def shard_shape(shape, tp):
    """This rank's model shape under head-sharded tensor parallelism."""
    from dataclasses import replace
    return replace(shape, n_heads=shape.n_heads // tp, n_kv_heads=shape.n_kv_heads // tp,
                   ffn_dim=shape.ffn_dim // tp, name=f"{shape.name}-tp{tp}")


def shard_layer(shape, t, rank, tp):
    """Slice one Llama layer's full tensors into rank `rank`'s shard (include/mirage.h)."""
    H, Hk, D, f = shape.n_heads, shape.n_kv_heads, shape.head_dim, shape.ffn_dim
    h, hk, fs = H // tp, Hk // tp, f // tp
    q = t["w_qkv"][rank * h * D:(rank + 1) * h * D]
    k = t["w_qkv"][H * D + rank * hk * D:H * D + (rank + 1) * hk * D]
    v = t["w_qkv"][(H + Hk) * D + rank * hk * D:(H + Hk) * D + (rank + 1) * hk * D]
    return {
        "w_qkv": torch.cat([q, k, v]), "w_o": t["w_o"][:, rank * h * D:(rank + 1) * h * D],
        "w_gateup": torch.cat([t["w_gateup"][rank * fs:(rank + 1) * fs], t["w_gateup"][f + rank * fs:f + (rank + 1) * fs]]),
        "w_down": t["w_down"][:, rank * fs:(rank + 1) * fs], "rms1_g": t["rms1_g"], "rms2_g": t["rms2_g"],
    }


def make_shard_blob(shape, rank, tp, seed=0, model_idx=0):
    """Pinned blob of rank `rank`'s shard of the full seeded model (CPU generation)."""
    sh = shard_shape(shape, tp)
    S, G, _ = _lib.model_sizes(sh)
    blob = torch.empty(shape.n_layers * S + G, dtype=torch.uint8, pin_memory=True)
    order = [n for n, _, _ in weights.layer_spec(sh)]
    for l in range(shape.n_layers):
        t = shard_layer(shape, weights.layer_tensors(shape, l, seed, model_idx), rank, tp)
        blob[l * S:(l + 1) * S].copy_(_lib.tensors_to_bytes({k: v.contiguous() for k, v in t.items()}, order))
    blob[shape.n_layers * S:].copy_(global_bytes_tensor(shape, seed, model_idx))
    return blob


def gpu_numa_node(index):
    """NUMA node of CUDA device `index` (its PCI function's numa_node in sysfs;
    0 when unknown or on a single-node host)."""
    try:
        p = torch.cuda.get_device_properties(index)
        path = "/sys/bus/pci/devices/%04x:%02x:%02x.0/numa_node" % (p.pci_domain_id, p.pci_bus_id, p.pci_device_id)
        return max(0, int(open(path).read().strip()))
    except Exception:
        return 0


def _node_cpus(node):
    out = set()
    try:
        for part in open(f"/sys/devices/system/node/node{node}/cpulist").read().strip().split(","):
            lo, _, hi = part.partition("-")
            out.update(range(int(lo), int(hi or lo) + 1))
    except Exception:
        pass
    return out


class numa_bind:
    """Bind the calling thread to the CPUs of NUMA node `node` for the block, so
    host pages it first-touches (a pinned blob's allocation, a shared blob's
    writes) land on that node; restores the previous affinity."""

    def __init__(self, node):
        self.cpus = _node_cpus(node) if node is not None else set()

    def __enter__(self):
        import os
        self.prev = None
        if self.cpus and hasattr(os, "sched_setaffinity"):
            try:
                self.prev = os.sched_getaffinity(0)
                os.sched_setaffinity(0, self.cpus & self.prev or self.cpus)
            except OSError:
                self.prev = None
        return self

    def __exit__(self, *exc):
        import os
        if self.prev is not None:
            os.sched_setaffinity(0, self.prev)
        return False


def shared_blob(shape, seed, model_idx, tag, creator, barrier, gen_device="cpu", numa_node=None):
    """A weight blob in a file mapping shared by the replicas of one NUMA node
    (the paper's single host copy of the parameters, PAPER.md:555 fn., kept
    local to the socket whose PCIe root the GPUs use), page-locked in every
    process. `creator` generates it with its thread bound to `numa_node`;
    `barrier()` syncs."""
    import os
    S, G, _ = _lib.model_sizes(shape)
    n = shape.n_layers * S + G
    shm = "/dev/shm"
    try:
        st = os.statvfs(shm)
        base = shm if st.f_bavail * st.f_frsize > n + (1 << 30) else "/tmp"
    except OSError:
        base = "/tmp"
    path = os.path.join(base, f"mirage_blob_{tag}_{shape.name}_{seed}_{model_idx}.bin")
    if creator:
        with open(path, "wb") as f:
            f.truncate(n)
        with numa_bind(numa_node):
            t = torch.from_file(path, shared=True, size=n, dtype=torch.uint8)
            for l in range(shape.n_layers):
                t[l * S:(l + 1) * S].copy_(layer_bytes_tensor(shape, l, seed, model_idx, gen_device))
            t[shape.n_layers * S:].copy_(global_bytes_tensor(shape, seed, model_idx, gen_device))
            del t
    barrier()
    t = torch.from_file(path, shared=True, size=n, dtype=torch.uint8)
    _lib.host_register(t)
    return t
