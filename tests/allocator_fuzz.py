"""Seeded allocator op logs replayed through libmirage (host-only context) and
through oracle c2; shared by the single- and multi-rank CPU tests."""
import hashlib
import random

from oracle import allocator as OA
from synth import models, weights


def bb(m):
    return m.n_layers * m.n_kv_heads * 2 * 16 * m.head_dim * 2


def make_log(seed, n_ops=300, n_seqs=12):
    """Op log over two tenants (0 = recipient, 1 = donor that goes inactive)."""
    rng = random.Random(seed)
    log = [("add", 0, 40), ("add", 1, 0), ("set_active", 1, 0)]
    remapped = set()
    self_cycle = False
    for _ in range(n_ops):
        r = rng.random()
        if r < 0.05 and len(remapped) < models.TOY.n_layers:
            # donor gives a random subset of its remaining layers (beta = 0)
            cand = [l for l in range(models.TOY.n_layers) if l not in remapped]
            C = sorted(rng.sample(cand, rng.randint(1, len(cand))))
            remapped |= set(C)
            log.append(("remap", 1, 0, tuple(C), 0))
        elif r < 0.07 and not self_cycle:
            self_cycle = True
            log.append(("remap", 0, 0, (0, 1), 1))
        elif r < 0.09:   # Dynamic Reversion: move a region's live blocks out, then revert it
            log.append(("migrate", 0, rng.randrange(4)))
        elif r < 0.11:
            log.append(("unremap", 0, rng.randrange(4)))
        elif r < 0.6:
            log.append(("alloc", 0, rng.randrange(n_seqs), rng.randint(0, 9)))
        else:
            log.append(("free", 0, rng.randrange(n_seqs)))
    return log


def replay_lib(log, shape=models.TOY, max_ctx=4096):
    from paper_2507_11507_b200 import _lib
    ctx = _lib.Context.host_only(1 << 36, 64, max_ctx)
    out = []
    for op in log:
        try:
            if op[0] == "add":
                out.append(("ok", ctx.add_model_host_only(shape, op[2])))
            elif op[0] == "set_active":
                ctx.set_active(op[1], op[2])
                out.append(("ok",))
            elif op[0] == "remap":
                g, _ = ctx.remap_layers(op[1], op[2], list(op[3]), op[4])
                out.append(("ok", g))
            elif op[0] == "alloc":
                out.append(("ok", tuple(ctx.alloc_blocks(op[1], op[2], op[3]))))
            elif op[0] == "free":
                ctx.free_blocks(op[1], op[2])
                out.append(("ok",))
            elif op[0] == "migrate":
                out.append(("ok", ctx.migrate_region(op[1], op[2])))
            elif op[0] == "unremap":
                ctx.unremap(op[1], op[2])
                out.append(("ok",))
        except _lib.MirageError as e:
            out.append(("err", e.code, e.shortfall))
    state = {}
    for m in (0, 1):
        st = ctx.query(m)
        tabs = {}
        for s in range(64):
            try:
                tabs[s] = tuple(ctx.block_table(m, s))
            except _lib.MirageError:
                pass
        locs = tuple(ctx.block_location(m, b) for b in range(st["total_blocks"]))
        state[m] = (st["total_blocks"], st["free_blocks"], st["reclaimed_bytes"], tabs, locs)
    ctx.close()
    return out, state


def replay_oracle(log, shape=models.TOY, max_ctx=4096):
    from paper_2507_11507_b200 import _lib   # error codes only
    al = OA.Allocator(max_blocks=max_ctx // 16)
    S, BB = weights.layer_bytes(shape), bb(shape)
    out = []
    for op in log:
        try:
            if op[0] == "add":
                out.append(("ok", al.add_model(shape.n_layers, S, BB, op[2])))
            elif op[0] == "set_active":
                al.set_active(op[1], op[2])
                out.append(("ok",))
            elif op[0] == "remap":
                out.append(("ok", al.remap(op[1], op[2], list(op[3]), op[4])))
            elif op[0] == "alloc":
                out.append(("ok", tuple(al.alloc(op[1], op[2], op[3]))))
            elif op[0] == "free":
                al.free_seq(op[1], op[2])
                out.append(("ok",))
            elif op[0] == "migrate":
                try:
                    out.append(("ok", len(al.migrate(op[1], op[2]))))
                except OA.NoBlocks:          # the C-ABI reports no shortfall for migrate
                    out.append(("err", _lib.ERR_NO_BLOCKS, 0))
            elif op[0] == "unremap":
                al.unremap(op[1], op[2])
                out.append(("ok",))
        except OA.NoBlocks as e:
            out.append(("err", _lib.ERR_NO_BLOCKS, e.shortfall))
        except OA.DoubleFree:
            out.append(("err", _lib.ERR_DOUBLE_FREE, 0))
        except OA.StateError:
            out.append(("err", _lib.ERR_STATE, 0))
        except OA.RangeError:
            out.append(("err", _lib.ERR_RANGE, 0))
        except OA.Pressure:
            out.append(("err", _lib.ERR_PRESSURE, 0))
    state = {}
    for m in (0, 1):
        M = al.models[m]
        tabs = {s: tuple(t) for s, t in M.tables.items()}
        locs = tuple((-1, off) if d == "native" else (d, off)
                     for d, off in (M.block_loc[b] for b in range(M.next_id)))
        state[m] = (M.next_id, len(M.free), M.reclaimed_bytes, tabs, locs)
    return out, state


def state_hash(state):
    canon = [(m, (v[0], v[1], v[2], sorted(v[3].items()), v[4])) for m, v in sorted(state.items())]
    return hashlib.sha256(repr(canon).encode()).hexdigest()
