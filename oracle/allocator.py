"""c2 — remap / alloc / free block allocator (oracle). TEST INFRASTRUCTURE ONLY.

Follows PAPER.md:306-308 (Remapping Controller "reclaims a portion of the
parameter memory to expand KV cache capacity"), :492 ("marks the GPU memory
previously occupied by parameters as available for KV cache"), :558-564 §6
("Once parameter tensors are released, the KV cache engine can immediately
reuse the freed physical memory"), Alg. 1 :509/:529-531, and PagedAttention's
block tables. Unstated details follow SURVEY.md §8(c) c2 and
readings #1, #11-#15 (listed in DESIGN.md):

* per recipient model r: native ids [0, N0); reclaimed ids appended
  monotonically (next_id), runs ascending, never reused;
* remap(d, r, C, beta): R = sorted(C[beta:]) split into maximal runs of
  consecutive layer ids; each run of |run| * S_d bytes yields floor(len / BB_r)
  blocks at byte offsets first*S_d + i*BB_r of the donor's weight arena;
* alloc(r, seq, n): the n lowest free ids, ascending, all-or-nothing; a
  sequence's table never exceeds max_blocks = max_ctx / 16 ids (RangeError,
  checked after the free-count check and before any state changes, like every
  other error: a failed call leaves the state exactly as it was);
* free(r, seq): return all of seq's blocks; unknown seq -> DoubleFree.

* unremap(r, region) (NEXT-1, Dynamic Reversion): all of the region's ids free
  -> retired (never reused), donor layers resident again; PRESSURE otherwise.
* migrate(r, region) (reading #29; the paper restores reclaimed memory "when KV
  cache space is sufficient", and is silent on blocks still
  live in it): the region's live ids (a streaming cycle: all its regions'),
  ascending, take the lowest free ids outside it, ascending, one for one; every
  table entry is renamed in place and the old ids become free. NoBlocks when
  fewer free ids lie outside than are live. The product copies each moved
  block's bytes; the oracle only renames.

Pins: worked examples (toy layer -> 48 blocks; SPEC 2 GB / 16 MB -> 128),
invariants I1-I4 and an exhaustive comparison against an independent set-based
model in tests/test_oracle_allocator.py.
"""

RESIDENT, SLOT, RECLAIMED = 0, 1, 2


class StateError(RuntimeError):
    pass


class RangeError(ValueError):
    pass


class NoBlocks(RuntimeError):
    def __init__(self, shortfall):
        super().__init__(f"shortfall {shortfall}")
        self.shortfall = shortfall


class DoubleFree(RuntimeError):
    pass


class Pressure(RuntimeError):
    def __init__(self, used):
        super().__init__(f"{used} blocks still hold KV")
        self.used = used


class Model:
    def __init__(self, n_layers, layer_bytes, block_bytes, n_native):
        self.n_layers = n_layers
        self.S = layer_bytes
        self.BB = block_bytes
        self.n_native = n_native
        self.next_id = n_native
        self.free = set(range(n_native))
        self.tables = {}
        self.layer_state = [RESIDENT] * n_layers
        self.cycle = []
        self.beta = 0
        self.reclaimed_bytes = 0          # bytes of R carved into this model's pool
        self.donated_bytes = 0            # bytes of this model's layers reclaimed
        self.block_loc = {i: ("native", i * block_bytes) for i in range(n_native)}
        self.regions = []                 # dicts: donor, first_layer, n_layers, first_id, n_blocks, cycle, retired
        self.active = True


class Allocator:
    def __init__(self, max_blocks=None):
        """max_blocks: cap on one sequence's table (max_ctx / 16); None = no cap."""
        self.models = []
        self.max_blocks = max_blocks

    def add_model(self, n_layers, layer_bytes, block_bytes, n_native):
        self.models.append(Model(n_layers, layer_bytes, block_bytes, n_native))
        return len(self.models) - 1

    def set_active(self, model, active):
        """A model can run only if every reclaimed layer of it is streamed through
        its own cycle (its other reclaimed bytes are somebody's KV blocks)."""
        m = self.models[model]
        if active and not m.active:
            for l, st in enumerate(m.layer_state):
                if st == RECLAIMED and l not in m.cycle:
                    raise StateError(f"layer {l} is reclaimed outside the model's cycle")
        m.active = bool(active)

    def remap(self, donor, recipient, C, beta):
        """Returns the number of blocks added to the recipient's pool."""
        if not (0 <= donor < len(self.models) and 0 <= recipient < len(self.models)):
            raise RangeError("model id")
        d, r = self.models[donor], self.models[recipient]
        m = len(C)
        if not (0 <= beta <= m) or any(not (0 <= l < d.n_layers) for l in C):
            raise RangeError("cycle")
        if len(set(C)) != m or list(C) != sorted(C):
            raise RangeError("cycle must be strictly ascending")
        if any(d.layer_state[l] != RESIDENT for l in C):
            raise StateError("layer already cycled or reclaimed")
        if beta == 0 and d.active:
            raise StateError("beta=0 needs an inactive donor")
        if beta > 0 and donor != recipient:
            raise StateError("streaming remap must be a self-remap")
        if beta > 0 and d.cycle:
            raise StateError("donor already has a cycle")
        R = sorted(C[beta:])
        gained = 0
        runs = []
        for l in R:
            if runs and runs[-1][-1] == l - 1:
                runs[-1].append(l)
            else:
                runs.append([l])
        for run in runs:
            off = run[0] * d.S
            length = len(run) * d.S
            k = length // r.BB
            first = r.next_id
            for i in range(k):
                bid = r.next_id
                r.next_id += 1
                r.free.add(bid)
                r.block_loc[bid] = (donor, off + i * r.BB)
            r.regions.append(dict(donor=donor, first_layer=run[0], n_layers=len(run), first_id=first,
                                  n_blocks=k, cycle=beta > 0, retired=False))
            gained += k
        r.reclaimed_bytes += len(R) * d.S
        d.donated_bytes += len(R) * d.S
        for l in C[:beta]:
            d.layer_state[l] = SLOT
        for l in R:
            d.layer_state[l] = RECLAIMED
        if beta > 0:
            d.cycle = list(C)
            d.beta = beta
        return gained

    def unremap(self, recipient, region):
        """Dynamic Reversion: the region's blocks must
        all be free; its ids are retired (never handed out again); the donor's
        layers become resident. A streaming cycle's region reverts the whole cycle
        (all its regions; slot holders become plain resident layers)."""
        r = self.models[recipient]
        if not (0 <= region < len(r.regions)):
            raise RangeError("region")
        reg = r.regions[region]
        if reg["retired"]:
            raise StateError("already reverted")
        d = self.models[reg["donor"]]
        if reg["cycle"]:
            which = [g for g in r.regions if g["cycle"] and g["donor"] == reg["donor"] and not g["retired"]]
        else:
            which = [reg]
        ids = [i for g in which for i in range(g["first_id"], g["first_id"] + g["n_blocks"])]
        busy = [i for i in ids if i not in r.free]
        if busy:
            raise Pressure(len(busy))
        for i in ids:
            r.free.discard(i)
        for g in which:
            g["retired"] = True
            r.reclaimed_bytes -= g["n_layers"] * d.S
            d.donated_bytes -= g["n_layers"] * d.S
            for l in range(g["first_layer"], g["first_layer"] + g["n_layers"]):
                d.layer_state[l] = RESIDENT
        if reg["cycle"]:
            for l in d.cycle[: d.beta]:
                d.layer_state[l] = RESIDENT
            d.cycle, d.beta = [], 0

    def _region_ids(self, r, region):
        reg = r.regions[region]
        if reg["cycle"]:
            which = [g for g in r.regions if g["cycle"] and g["donor"] == reg["donor"] and not g["retired"]]
        else:
            which = [reg]
        return {i for g in which for i in range(g["first_id"], g["first_id"] + g["n_blocks"])}

    def migrate(self, recipient, region):
        """Move the region's live blocks to free ids outside it (reading #29).
        Returns the moves [(old, new)] in ascending old-id order."""
        r = self.models[recipient]
        if not (0 <= region < len(r.regions)):
            raise RangeError("region")
        if r.regions[region]["retired"]:
            raise StateError("already reverted")
        X = self._region_ids(r, region)
        live = sorted(i for i in X if i not in r.free)
        outside = sorted(i for i in r.free if i not in X)
        if len(outside) < len(live):
            raise NoBlocks(len(live) - len(outside))
        moves = list(zip(live, outside[: len(live)]))
        ren = dict(moves)
        for seq in r.tables:
            r.tables[seq] = [ren.get(i, i) for i in r.tables[seq]]
        for old, new in moves:
            r.free.remove(new)
            r.free.add(old)
        return moves

    def alloc(self, model, seq, n):
        r = self.models[model]
        if n < 0:
            raise RangeError("n")
        if n > len(r.free):
            raise NoBlocks(n - len(r.free))
        if self.max_blocks is not None and len(r.tables.get(seq, [])) + n > self.max_blocks:
            raise RangeError(f"table of seq {seq} would exceed max_ctx")
        ids = sorted(r.free)[:n]
        for i in ids:
            r.free.remove(i)
        r.tables.setdefault(seq, []).extend(ids)
        return ids

    def free_seq(self, model, seq):
        r = self.models[model]
        if seq not in r.tables:
            raise DoubleFree(f"seq {seq}")
        r.free.update(r.tables.pop(seq))

    def table(self, model, seq):
        return list(self.models[model].tables[seq])

    def n_free(self, model):
        return len(self.models[model].free)

    def n_total(self, model):
        return self.models[model].next_id
