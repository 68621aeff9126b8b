"""ctypes binding of libmirage.so — argument marshalling only.

Every function here forwards to the C-ABI declared in include/mirage.h with the
same name (without the ``mirage_`` prefix on methods). Device memory, pinned
host memory and streams come from PyTorch (plumbing); every step of the decode
path runs inside libmirage's kernels. There is no fallback: if the shared
library is missing or fails to load, importing this module raises.
"""
import ctypes as C
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libmirage.so")

OK, ERR_CONFIG, ERR_CAPACITY, ERR_RANGE, ERR_STATE = 0, -1, -2, -3, -4
ERR_NO_BLOCKS, ERR_DOUBLE_FREE, ERR_INFEASIBLE, ERR_PRESSURE, ERR_CUDA, ERR_NCCL = -5, -6, -7, -8, -9, -10
FAMILY_OPT, FAMILY_LLAMA = 0, 1
BETA_1, BETA_2, BETA_DYNAMIC = 1, 2, 3
BLOCK_TOKENS = 16
FLAG_TIME_ATTN = 1
FLAG_HOST_ONLY = 2
FLAG_SLOT_TAGS = 4
FLAG_CUDA_GRAPHS = 8
FLAG_TP_IPC = 16
FLAG_POISON = 32
FLAG_TC_GEMM = 64
MAX_CYCLE = 256

_NAMES = {ERR_CONFIG: "CONFIG", ERR_CAPACITY: "CAPACITY", ERR_RANGE: "RANGE", ERR_STATE: "STATE",
          ERR_NO_BLOCKS: "NO_BLOCKS", ERR_DOUBLE_FREE: "DOUBLE_FREE", ERR_INFEASIBLE: "INFEASIBLE",
          ERR_PRESSURE: "PRESSURE", ERR_CUDA: "CUDA", ERR_NCCL: "NCCL"}


class MirageError(RuntimeError):
    def __init__(self, code, msg, shortfall=0):
        super().__init__(f"mirage {_NAMES.get(code, code)}: {msg}")
        self.code = code
        self.shortfall = shortfall


class InitCfg(C.Structure):
    _fields_ = [("device", C.c_int32), ("dev_arena", C.c_void_p), ("dev_arena_bytes", C.c_uint64),
                ("block_tokens", C.c_int32), ("compute_stream", C.c_void_p), ("copy_stream", C.c_void_p),
                ("max_batch", C.c_int32), ("max_ctx", C.c_int32), ("flags", C.c_uint32),
                ("tp_rank", C.c_int32), ("tp_size", C.c_int32), ("nccl_id", C.c_void_p)]


class ModelCfg(C.Structure):
    _fields_ = [("family", C.c_int32), ("n_layers", C.c_int32), ("d_model", C.c_int32),
                ("n_heads", C.c_int32), ("n_kv_heads", C.c_int32), ("head_dim", C.c_int32),
                ("ffn_dim", C.c_int32), ("vocab", C.c_int32), ("max_pos", C.c_int32),
                ("norm_eps", C.c_float), ("rope_theta", C.c_float)]


class Region(C.Structure):
    _fields_ = [("donor", C.c_int32), ("first_layer", C.c_int32), ("n_layers", C.c_int32),
                ("first_id", C.c_int32), ("n_blocks", C.c_int32), ("n_free", C.c_int32),
                ("cycle", C.c_int32), ("retired", C.c_int32)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class Stats(C.Structure):
    _fields_ = [("native_blocks", C.c_int64), ("total_blocks", C.c_int64), ("free_blocks", C.c_int64),
                ("layer_bytes", C.c_uint64), ("block_bytes", C.c_uint64),
                ("reclaimed_bytes", C.c_uint64), ("donated_bytes", C.c_uint64),
                ("m", C.c_int32), ("beta", C.c_int32), ("active", C.c_int32), ("n_seqs", C.c_int32),
                ("cycle", C.c_int32 * MAX_CYCLE), ("uses", C.c_uint64), ("h2d_copies", C.c_uint64),
                ("h2d_bytes", C.c_uint64), ("h2d_ms", C.c_double), ("last_step_ms", C.c_double),
                ("steps", C.c_int64), ("attn_launches", C.c_int64), ("attn_ms", C.c_double),
                ("attn_bytes", C.c_uint64), ("last_meta_h2d_bytes", C.c_uint64),
                ("last_attn_units", C.c_int32), ("last_split_blocks", C.c_int32),
                ("slot_tag_errors", C.c_int64), ("tp_peer_timeouts", C.c_int64),
                ("stall_waits", C.c_int64), ("stall_ms", C.c_double)]

    def as_dict(self):
        d = {k: getattr(self, k) for k, _ in self._fields_ if k != "cycle"}
        d["cycle"] = list(self.cycle[: self.m])
        return d


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} not built: run `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = C.CDLL(LIB_PATH)
    P, I32, I64, U64 = C.c_void_p, C.c_int32, C.c_int64, C.c_uint64
    pI32, pI64, pU64 = C.POINTER(C.c_int32), C.POINTER(C.c_int64), C.POINTER(C.c_uint64)
    sig = {
        "mirage_model_sizes": (I32, [C.POINTER(ModelCfg), pU64, pU64, pU64]),
        "mirage_model_arena_bytes": (I32, [C.POINTER(ModelCfg), I64, I32, I32, pU64]),
        "mirage_init": (I32, [C.POINTER(InitCfg), C.POINTER(P)]),
        "mirage_destroy": (None, [P]),
        "mirage_last_error": (C.c_char_p, [P]),
        "mirage_add_model": (I32, [P, C.POINTER(ModelCfg), P, U64, I64, pI32]),
        "mirage_plan": (I32, [I32, I32, I32, U64, U64, I32, pI32, pI32, pI32]),
        "mirage_predict_stall": (I32, [I32, pI32, I32, I32, U64, U64, pI64]),
        "mirage_remap_layers": (I32, [P, I32, I32, pI32, I32, I32, pI64, pU64]),
        "mirage_set_active": (I32, [P, I32, I32]),
        "mirage_alloc_blocks": (I32, [P, I32, I64, I32, pI32, pI32]),
        "mirage_free_blocks": (I32, [P, I32, I64]),
        "mirage_get_block_table": (I32, [P, I32, I64, pI32, I32, pI32]),
        "mirage_block_location": (I32, [P, I32, I32, pI32, pU64]),
        "mirage_seq_len": (I32, [P, I32, I64, pI32]),
        "mirage_decode_step": (I32, [P, I32, I32, pI64, pI32, pI32, P, pI32]),
        "mirage_prefill": (I32, [P, I32, I32, pI64, pI32, pI32, pI32]),
        "mirage_query": (I32, [P, I32, C.POINTER(Stats)]),
        "mirage_slot_log": (I32, [P, I32, pI64, I32, pI32]),
        "mirage_sync": (I32, [P]),
        "mirage_attn_only": (I32, [P, I32, I32, I32, pI64, P, P, I32, I32]),
        "mirage_fill_kv": (I32, [P, I32, I64, I32, U64]),
        "mirage_write_kv": (I32, [P, I32, I64, I32, P]),
        "mirage_kernel_launches": (I64, [P]),
        "mirage_attn_trace": (I32, [P, pU64, I32, pI32]),
        "mirage_decode_gemm": (I32, [P, P, I32, I32, P, I32, P, I32, I32, I32, pI32]),
        "mirage_sk_gemm": (I32, [P, P, I32, I32, P, I32, P, P, P, I32]),
        "mirage_set_flags": (I32, [P, C.c_uint32, C.c_uint32]),
        "mirage_nccl_unique_id": (I32, [P]),
        "mirage_host_register": (I32, [P, U64]),
        "mirage_region_count": (I32, [P, I32, pI32]),
        "mirage_region_info": (I32, [P, I32, I32, C.POINTER(Region)]),
        "mirage_unremap": (I32, [P, I32, I32]),
        "mirage_migrate_region": (I32, [P, I32, I32, pI32]),
        "mirage_swap_out": (I32, [P, I32, I64, P, U64]),
        "mirage_swap_in": (I32, [P, I32, I64, P]),
        "mirage_set_weight_source": (I32, [P, I32, P, U64]),
        "mirage_tp_export": (I32, [P, I32, P]),
        "mirage_tp_import": (I32, [P, I32, P]),
        "mirage_host_unregister": (I32, [P]),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    return lib


LIB = _load()
EXPORTED = [
    "mirage_model_sizes", "mirage_model_arena_bytes", "mirage_init", "mirage_destroy", "mirage_last_error",
    "mirage_add_model", "mirage_plan", "mirage_remap_layers", "mirage_set_active", "mirage_alloc_blocks",
    "mirage_free_blocks", "mirage_get_block_table", "mirage_block_location", "mirage_seq_len",
    "mirage_decode_step", "mirage_query", "mirage_slot_log", "mirage_sync", "mirage_attn_only",
    "mirage_fill_kv", "mirage_write_kv", "mirage_kernel_launches", "mirage_nccl_unique_id",
    "mirage_host_register", "mirage_host_unregister", "mirage_region_count", "mirage_region_info",
    "mirage_unremap", "mirage_swap_out", "mirage_swap_in", "mirage_set_weight_source", "mirage_tp_export",
    "mirage_tp_import", "mirage_prefill", "mirage_migrate_region", "mirage_predict_stall",
    "mirage_attn_trace", "mirage_decode_gemm", "mirage_sk_gemm", "mirage_set_flags"]


def model_cfg(shape):
    """mirage_model_cfg from any object with the synth.models.ModelShape fields."""
    return ModelCfg(shape.family, shape.n_layers, shape.d_model, shape.n_heads, shape.n_kv_heads,
                    shape.head_dim, shape.ffn_dim, shape.vocab, shape.max_pos, shape.norm_eps,
                    shape.rope_theta)


def model_sizes(shape):
    S, G, BB = C.c_uint64(), C.c_uint64(), C.c_uint64()
    cfg = model_cfg(shape)
    rc = LIB.mirage_model_sizes(C.byref(cfg), C.byref(S), C.byref(G), C.byref(BB))
    if rc:
        raise MirageError(rc, "model_sizes")
    return S.value, G.value, BB.value


def model_arena_bytes(shape, native_blocks, max_batch, max_ctx):
    out = C.c_uint64()
    cfg = model_cfg(shape)
    rc = LIB.mirage_model_arena_bytes(C.byref(cfg), native_blocks, max_batch, max_ctx, C.byref(out))
    if rc:
        raise MirageError(rc, "model_arena_bytes")
    return out.value


def plan(n_layers, alpha, beta_policy, t_transfer_ns, t_compute_layer_ns, anchor=0):
    cyc = (C.c_int32 * max(n_layers, 1))()
    m, beta = C.c_int32(), C.c_int32()
    rc = LIB.mirage_plan(n_layers, alpha, beta_policy, int(t_transfer_ns), int(t_compute_layer_ns), anchor,
                         cyc, C.byref(m), C.byref(beta))
    if rc:
        raise MirageError(rc, "plan")
    return list(cyc[: m.value]), m.value, beta.value


def predict_stall(n_layers, cycle, beta, t_transfer_ns, t_compute_layer_ns):
    """Predicted steady-state stall per step (ns) of an explicit cycle (mirage_predict_stall)."""
    out = C.c_int64()
    rc = LIB.mirage_predict_stall(n_layers, _i32(cycle) if cycle else None, len(cycle), beta, int(t_transfer_ns),
                                  int(t_compute_layer_ns), C.byref(out))
    if rc:
        raise MirageError(rc, "predict_stall")
    return out.value


def decode_gemm(w, x, splits=0, stream=None, reduce=False, col_groups=0):
    """Y slices [splits][B][N] fp32 of x [B][K] @ w[N][K]^T on the tcgen05 decode GEMM
    (mirage_decode_gemm); both bf16 CUDA tensors. reduce: the splits are summed in
    the kernel (one slice). Returns (slices, number of slices)."""
    assert w.dtype == torch.bfloat16 and x.dtype == torch.bfloat16 and w.is_cuda and x.is_cuda
    w, x = w.contiguous(), x.contiguous()
    N, K = w.shape
    B = x.shape[0]
    n = splits or 16
    y = torch.empty((n, B, N), dtype=torch.float32, device=w.device)
    got = C.c_int32()
    st = stream if stream is not None else torch.cuda.current_stream(w.device)
    rc = LIB.mirage_decode_gemm(st.cuda_stream, w.data_ptr(), N, K, x.data_ptr(), B, y.data_ptr(), int(splits),
                                int(bool(reduce)), int(col_groups), C.byref(got))
    if rc:
        raise MirageError(rc, "decode_gemm")
    return y[: got.value], got.value


def sk_gemm(w, x, bias=None, relu=False, out_bf16=False, stream=None):
    """y [B][N] = epilogue(x [B][K] @ w[N][K]^T) on the persistent stream-K tcgen05
    GEMM (mirage_sk_gemm); bf16 CUDA tensors; fp32 output unless out_bf16."""
    assert w.dtype == torch.bfloat16 and x.dtype == torch.bfloat16 and w.is_cuda and x.is_cuda
    w, x = w.contiguous(), x.contiguous()
    N, K = w.shape
    B = x.shape[0]
    y = torch.empty((B, N), dtype=torch.bfloat16 if out_bf16 else torch.float32, device=w.device)
    st = stream if stream is not None else torch.cuda.current_stream(w.device)
    rc = LIB.mirage_sk_gemm(st.cuda_stream, w.data_ptr(), N, K, x.data_ptr(), B,
                            None if out_bf16 else y.data_ptr(), y.data_ptr() if out_bf16 else None,
                            None if bias is None else bias.contiguous().data_ptr(), int(bool(relu)))
    if rc:
        raise MirageError(rc, "sk_gemm")
    return y


def nccl_unique_id():
    """128-byte ncclUniqueId (TP rank 0), to broadcast to the other ranks."""
    buf = C.create_string_buffer(128)
    rc = LIB.mirage_nccl_unique_id(buf)
    if rc:
        raise MirageError(rc, "nccl_unique_id")
    return buf.raw


def host_register(tensor):
    """Page-lock a CPU tensor's memory in place (e.g. a shared file mapping)."""
    rc = LIB.mirage_host_register(tensor.data_ptr(), tensor.numel() * tensor.element_size())
    if rc:
        raise MirageError(rc, "host_register")


def _i32(seq):
    return (C.c_int32 * len(seq))(*[int(x) for x in seq])


def _i64(seq):
    return (C.c_int64 * len(seq))(*[int(x) for x in seq])


def pack_blob(layers_bytes, global_bytes):
    """Pinned host blob = concatenation of per-layer byte images + globals
    (include/mirage.h "Weight blob layout"). Inputs are uint8 CPU tensors."""
    total = sum(int(t.numel()) for t in layers_bytes) + int(global_bytes.numel())
    blob = torch.empty(total, dtype=torch.uint8, pin_memory=True)
    off = 0
    for t in list(layers_bytes) + [global_bytes]:
        n = int(t.numel())
        blob[off: off + n].copy_(t)
        off += n
    return blob


def tensors_to_bytes(named, order):
    """Concatenate bf16 tensors in the documented order into one uint8 tensor."""
    return torch.cat([named[n].contiguous().view(torch.uint8).reshape(-1) for n in order])


class Context:
    """One mirage_ctx on one GPU. Owns (keeps alive) the arena, the streams and
    the host blobs it was given."""

    @classmethod
    def host_only(cls, arena_bytes, max_batch, max_ctx, arena_base=1 << 40):
        """A device-less context (MIRAGE_FLAG_HOST_ONLY): allocator, remap and
        tables only; the arena is a virtual address range never dereferenced."""
        self = cls.__new__(cls)
        self.device, self.arena, self.stream, self._blobs = None, None, None, []
        self._arena_ptr = arena_base
        cfg = InitCfg(0, arena_base, int(arena_bytes), BLOCK_TOKENS, None, None, max_batch, max_ctx,
                      FLAG_HOST_ONLY, 0, 1, None)
        self._ctx = C.c_void_p()
        rc = LIB.mirage_init(C.byref(cfg), C.byref(self._ctx))
        if rc:
            raise MirageError(rc, "init(host_only)")
        self.max_batch, self.max_ctx = max_batch, max_ctx
        return self

    def add_model_host_only(self, shape, native_blocks):
        """add_model on a host-only context (no blob is read)."""
        S, G, _ = model_sizes(shape)
        cfg = model_cfg(shape)
        mid = C.c_int32()
        dummy = C.create_string_buffer(1)
        rc = LIB.mirage_add_model(self._ctx, C.byref(cfg), C.addressof(dummy), shape.n_layers * S + G,
                                  int(native_blocks), C.byref(mid))
        self._check(rc, "add_model")
        return mid.value

    def __init__(self, arena_bytes, max_batch, max_ctx, device=0, stream=None, flags=0, tp_rank=0, tp_size=1,
                 nccl_id=None):
        self.device = torch.device("cuda", device)
        self.arena = torch.empty(int(arena_bytes) + 256, dtype=torch.uint8, device=self.device)
        base = self.arena.data_ptr()
        self._arena_ptr = (base + 255) // 256 * 256
        self.stream = stream if stream is not None else torch.cuda.Stream(self.device)
        self._blobs = []
        self._nccl_id = C.create_string_buffer(bytes(nccl_id), 128) if nccl_id is not None else None
        cfg = InitCfg(device, self._arena_ptr, int(arena_bytes), BLOCK_TOKENS, self.stream.cuda_stream,
                      None, max_batch, max_ctx, flags, tp_rank, tp_size,
                      C.addressof(self._nccl_id) if self._nccl_id is not None else None)
        self._ctx = C.c_void_p()
        rc = LIB.mirage_init(C.byref(cfg), C.byref(self._ctx))
        if rc:
            raise MirageError(rc, "init")
        self.max_batch, self.max_ctx = max_batch, max_ctx

    # -- errors ---------------------------------------------------------------
    def _check(self, rc, what, shortfall=0):
        if rc:
            raise MirageError(rc, f"{what}: {LIB.mirage_last_error(self._ctx).decode()}", shortfall)

    def close(self):
        if self._ctx:
            LIB.mirage_destroy(self._ctx)
            self._ctx = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- API ------------------------------------------------------------------
    def add_model(self, shape, host_blob, native_blocks):
        self._blobs.append(host_blob)
        cfg = model_cfg(shape)
        mid = C.c_int32()
        rc = LIB.mirage_add_model(self._ctx, C.byref(cfg), host_blob.data_ptr(), host_blob.numel(),
                                  int(native_blocks), C.byref(mid))
        self._check(rc, "add_model")
        return mid.value

    def remap_layers(self, donor, recipient, cycle, beta):
        gained, rb = C.c_int64(), C.c_uint64()
        rc = LIB.mirage_remap_layers(self._ctx, donor, recipient, _i32(cycle), len(cycle), beta,
                                     C.byref(gained), C.byref(rb))
        self._check(rc, "remap_layers")
        return gained.value, rb.value

    def regions(self, model):
        n = C.c_int32()
        self._check(LIB.mirage_region_count(self._ctx, model, C.byref(n)), "region_count")
        out = []
        for i in range(n.value):
            r = Region()
            self._check(LIB.mirage_region_info(self._ctx, model, i, C.byref(r)), "region_info")
            out.append(r.as_dict())
        return out

    def tp_export(self, model):
        buf = C.create_string_buffer(64)
        self._check(LIB.mirage_tp_export(self._ctx, model, buf), "tp_export")
        return buf.raw

    def tp_import(self, model, handles):
        """handles: list of the tp ranks' 64-byte handles, in rank order."""
        blob = C.create_string_buffer(b"".join(handles), 64 * len(handles))
        self._check(LIB.mirage_tp_import(self._ctx, model, blob), "tp_import")

    def set_weight_source(self, model, src):
        """src: a uint8 tensor (pinned CPU or CUDA, this or a peer GPU) holding the blob."""
        self._blobs.append(src)
        self._check(LIB.mirage_set_weight_source(self._ctx, model, src.data_ptr(), src.numel()), "set_weight_source")

    def swap_out(self, model, seq_id, host_buf):
        """host_buf: pinned uint8 CPU tensor with room for the sequence's blocks."""
        self._check(LIB.mirage_swap_out(self._ctx, model, int(seq_id), host_buf.data_ptr(), host_buf.numel()),
                    "swap_out")

    def swap_in(self, model, seq_id, host_buf):
        self._check(LIB.mirage_swap_in(self._ctx, model, int(seq_id), host_buf.data_ptr()), "swap_in")

    def unremap(self, recipient, region):
        self._check(LIB.mirage_unremap(self._ctx, recipient, region), "unremap")

    def migrate_region(self, model, region):
        n = C.c_int32()
        self._check(LIB.mirage_migrate_region(self._ctx, model, region, C.byref(n)), "migrate_region")
        return n.value

    def set_active(self, model, active):
        self._check(LIB.mirage_set_active(self._ctx, model, int(active)), "set_active")

    def alloc_blocks(self, model, seq_id, n):
        ids = (C.c_int32 * max(n, 1))()
        short = C.c_int32()
        rc = LIB.mirage_alloc_blocks(self._ctx, model, int(seq_id), int(n), ids, C.byref(short))
        self._check(rc, "alloc_blocks", short.value)
        return list(ids[:n])

    def free_blocks(self, model, seq_id):
        self._check(LIB.mirage_free_blocks(self._ctx, model, int(seq_id)), "free_blocks")

    def block_table(self, model, seq_id):
        n = C.c_int32()
        LIB.mirage_get_block_table(self._ctx, model, int(seq_id), None, 0, C.byref(n))
        buf = (C.c_int32 * max(n.value, 1))()
        rc = LIB.mirage_get_block_table(self._ctx, model, int(seq_id), buf, n.value, C.byref(n))
        self._check(rc, "get_block_table")
        return list(buf[: n.value])

    def block_location(self, model, block_id):
        d, off = C.c_int32(), C.c_uint64()
        self._check(LIB.mirage_block_location(self._ctx, model, block_id, C.byref(d), C.byref(off)),
                    "block_location")
        return d.value, off.value

    def seq_len(self, model, seq_id):
        n = C.c_int32()
        self._check(LIB.mirage_seq_len(self._ctx, model, int(seq_id), C.byref(n)), "seq_len")
        return n.value

    def decode_step(self, model, seq_ids, tokens, positions, hidden_out=None, argmax=True):
        B = len(seq_ids)
        am = (C.c_int32 * B)() if argmax else None
        hp = hidden_out.data_ptr() if hidden_out is not None else None
        rc = LIB.mirage_decode_step(self._ctx, model, B, _i64(seq_ids), _i32(tokens), _i32(positions),
                                    hp, am)
        self._check(rc, "decode_step")
        return am

    def prefill(self, model, seq_ids, prompts, argmax=True):
        """prompts: list of token lists, one per seq (appended at the cached length).
        Returns the greedy next token per seq (synchronises) or None."""
        n = len(seq_ids)
        lens = [len(p) for p in prompts]
        flat = [int(t) for p in prompts for t in p]
        am = (C.c_int32 * n)() if argmax else None
        rc = LIB.mirage_prefill(self._ctx, model, n, _i64(seq_ids), _i32(lens), _i32(flat), am)
        self._check(rc, "prefill")
        return list(am) if argmax else None

    def decode_step_raw(self, model, B, seq_ids_c, tokens_c, positions_c, hidden_ptr, argmax_c):
        """Pre-marshalled variant (ctypes arrays) for timed loops."""
        rc = LIB.mirage_decode_step(self._ctx, model, B, seq_ids_c, tokens_c, positions_c, hidden_ptr,
                                    argmax_c)
        self._check(rc, "decode_step")

    def query(self, model):
        st = Stats()
        self._check(LIB.mirage_query(self._ctx, model, C.byref(st)), "query")
        return st.as_dict()

    def slot_log(self, model):
        n = C.c_int32()
        LIB.mirage_slot_log(self._ctx, model, None, 0, C.byref(n))
        buf = (C.c_int64 * max(5 * n.value, 1))()
        self._check(LIB.mirage_slot_log(self._ctx, model, buf, n.value, C.byref(n)), "slot_log")
        v = list(buf[: 5 * n.value])
        return [tuple(v[i: i + 5]) for i in range(0, len(v), 5)]

    def sync(self):
        self._check(LIB.mirage_sync(self._ctx), "sync")

    def set_flags(self, flags, mask):
        """Switch FLAG_TIME_ATTN / FLAG_CUDA_GRAPHS on a live context (mirage_set_flags)."""
        self._check(LIB.mirage_set_flags(self._ctx, int(flags), int(mask)), "set_flags")

    def attn_only(self, model, layer, seq_ids, q, out, split_tokens=0):
        assert q.dtype == torch.float32 and q.is_cuda and q.is_contiguous()
        rc = LIB.mirage_attn_only(self._ctx, model, layer, len(seq_ids), _i64(seq_ids), q.data_ptr(),
                                  out.data_ptr(), int(out.dtype == torch.float32), int(split_tokens))
        self._check(rc, "attn_only")

    def fill_kv(self, model, seq_id, n_tokens, seed):
        self._check(LIB.mirage_fill_kv(self._ctx, model, int(seq_id), int(n_tokens), int(seed)), "fill_kv")

    def write_kv(self, model, seq_id, kv):
        """kv: bf16 CPU tensor [L][H_kv][2][n][D]."""
        kv = kv.contiguous()
        self._check(LIB.mirage_write_kv(self._ctx, model, int(seq_id), int(kv.shape[3]), kv.data_ptr()),
                    "write_kv")

    def kernel_launches(self):
        return LIB.mirage_kernel_launches(self._ctx)

    def attn_trace(self):
        """[n_ctas][16] %globaltimer slots of the last attn_only launch (MIRAGE_ATTN_TRACE)."""
        n = C.c_int32()
        LIB.mirage_attn_trace(self._ctx, None, 0, C.byref(n))
        buf = (C.c_uint64 * max(16 * n.value, 1))()
        self._check(LIB.mirage_attn_trace(self._ctx, buf, n.value, C.byref(n)), "attn_trace")
        v = list(buf[: 16 * n.value])
        return [v[i: i + 16] for i in range(0, len(v), 16)]
